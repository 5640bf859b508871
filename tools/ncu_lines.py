"""Per-source-line warp-stall samples of one kernel in an ncu report (built with
-lineinfo, captured with --import-source on):
  python tools/ncu_lines.py <report.ncu-rep> [kernel-substring] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
path, fn, out = None, None, []
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No" or not r[0].strip().isdigit() or (kfilter and kfilter not in (fn or "")):
        continue
    try:
        s = int(r[4])
    except (ValueError, IndexError):
        continue
    if s > 0:
        out.append((s, path, int(r[0]), r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
for s, p, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  {p}:{ln}  {src}")
print("total samples", tot)
