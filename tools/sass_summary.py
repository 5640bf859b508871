"""Per-kernel SASS instruction summary of libihs.so's objects (cuobjdump -sass):
counts of the instructions that show which hardware path a kernel uses --
DMMA (fp64 tensor), UTMALDG / UBLKCP (TMA tensor / bulk copies), REDG (L2
reductions), ATOMS (shared atomics), LDS / STS, MATCH, multimem -- written to
profiles/<round>/sass_summary.json.

  python tools/sass_summary.py r02
"""
import collections
import glob
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["DMMA", "HMMA", "UTCHMMA", "UTMALDG", "UTMASTG", "UBLKCP", "REDG", "RED", "ATOMS", "ATOMG", "ATOM", "LDS",
        "STS", "LDG", "STG", "SHFL", "MATCH", "VOTE", "DFMA", "DADD", "DMUL", "MUFU", "SYNCS", "BAR", "UCGABAR",
        "LDTM", "STTM", "CCTL", "MEMBAR", "ERRBAR", "LDGMC"]


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        return name


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
    out = {}
    for obj in sorted(glob.glob(os.path.join(ROOT, "paper_1910_14166_b200", "build", "*.o"))):
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        cur = None
        for line in sass.splitlines():
            m = re.search(r"Function : (\S+)", line)
            if m:
                cur = demangle(m.group(1))
                cur = re.sub(r"\(.*", "", cur.replace("(anonymous namespace)::", "").replace("void ", ""))
                out.setdefault(os.path.basename(obj), {}).setdefault(cur, collections.Counter())
                continue
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", line)
            if m and cur:
                op = m.group(1)
                if op in KEYS:
                    out[os.path.basename(obj)][cur][op] += 1
    js = {o: {k: dict(v) for k, v in fns.items() if v} for o, fns in out.items()}
    dst = os.path.join(ROOT, "profiles", rnd, "sass_summary.json")
    os.makedirs(os.path.dirname(dst), exist_ok=True)
    with open(dst, "w") as f:
        json.dump(js, f, indent=1, sort_keys=True)
    tot = collections.Counter()
    for fns in js.values():
        for v in fns.values():
            tot.update(v)
    print(dst, dict(tot.most_common(12)))


if __name__ == "__main__":
    main()
