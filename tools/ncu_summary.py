"""Summarise ncu output for profiles/ (run here, on the CPU box, on files gpurun brought back).

  python tools/ncu_summary.py launches <launches.csv> [--skip-warmup-steps W --steps K]
      per-kernel launch count / average / share of the library's kernel time
      (ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised)
  python tools/ncu_summary.py full <report.ncu-rep>
      headline counters of each captured kernel (ncu --set full), incl. DRAM bytes per launch
      and the top warp-stall reasons
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

OURS = ("cs_", "scan_", "gram", "chol", "potrf", "trsm", "syrk", "backsolve", "aug_fill", "reduce_rows", "sjlt", "small_",
        "sum_splits", "csr_", "pg_", "grad_", "scale_", "sqnorm", "hash_", "ols_", "axpy")


def ours(name: str) -> bool:
    short = name.split("(")[0].split("::")[-1].split("<")[0]
    return short.startswith(OURS)


def launches(path: str) -> dict:
    rows = []
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        rows.append((r["Kernel Name"], us))
    agg = collections.OrderedDict()
    for name, us in rows:
        if not ours(name):
            continue
        short = name.split("(")[0].replace("void ", "").replace("ihs::", "").replace("<unnamed>::", "")
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
    total = sum(v[1] for v in agg.values()) or 1.0
    return {"kernels": [{"kernel": k, "launches": v[0], "avg_us": round(v[1] / v[0], 2),
                         "share_of_libihs_time": round(v[1] / total, 4)} for k, v in agg.items()],
            "libihs_total_us": round(total, 1)}


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "lts__t_sectors_op_red.sum",
           "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"]


def full(path: str) -> list:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        rec = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in hdr:
                rec[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(r[i].replace(",", "")))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        rec["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in
                                 sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        res.append(rec)
    return res


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if kind == "launches" else full(path), indent=1))
