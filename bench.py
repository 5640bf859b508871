#!/usr/bin/env python
"""Benchmark of the IHS hot path on B200 (BASELINE.json metric: "sketch rows/sec &
HBM GB/s vs peak; IHS time-to-1e-10 rel error, 1/2/4/8 GPU").

A step is one IHS iteration over the whole configuration:
hash + stable bucket sort (a1), fused sketch + gradient over A (a2 + a5), the
all-reduce of [SA | g] across ranks (a3), the DMMA Gram (a4) and the Cholesky
update (a6).  Default workload: BASELINE.json configs[1] (C2, dense OLS,
A 2^22 x 128 fp64 AR(1) rows, CountSketch m = 1024), row-sharded over the N
ranks (strong scaling: the problem is fixed, N GPUs share its rows).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl product|reference]

Prints ONE JSON line on rank 0.  value = rows of A sketched per second over the
whole job (n_global * K / max-over-ranks device time).  The oracle (oracle/) is
executed only by the cpu_baseline leg and by --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sketch rows/sec & HBM GB/s vs peak; IHS time-to-1e-10 rel error, 1/2/4/8 GPU"
UNIT = "rows/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-1e-10 solve")
    ap.add_argument("--allreduce", default="nccl", choices=["nccl", "nvls"],
                    help="N > 1: the [SA | g] exchange through NCCL (default) or the library's NVLS multimem kernel")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--lookahead", type=int, default=-1, choices=[-1, 0, 1],
                    help="force the look-ahead schedule off / on (default: the library's rule)")
    ap.add_argument("--la-gram-sms", type=int, default=-1,
                    help="SMs of the wide look-ahead Gram (ctx option la_gram_sms; default: the library's rule)")
    ap.add_argument("--la-gram-tile", type=int, default=-1, help="ctx option la_gram_tile (64 or 128)")
    ap.add_argument("--step-sync-flush", action="store_true",
                    help="L2-flushed configs: time each step alone between a flush and a sync (side-stream work "
                         "that outlives the step's update is then NOT timed) instead of K consecutive steps")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: host-staged all-reduce, for testing the "
                         "sharded path with IHS_BENCH_SHARE_GPU=1 on one GPU)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config_obj(cfg, world, extra=None):
    o = {"workload": f"{cfg.name}: {'CSR' if cfg.layout == 'csr' else 'dense'} OLS A {cfg.n}x{cfg.d} fp64 "
                     f"({cfg.dist}), {cfg.family} m={cfg.m} s={cfg.s}",
         "n": cfg.n, "d": cfg.d, "m": cfg.m, "s": cfg.s, "sketch": cfg.family,
         "parallelism": f"row-shard x{world} + allreduce[SA|g]" if world > 1 else "single GPU",
         "l2": ("inputs larger than L2 (A = %.2f GiB per step)" % (cfg.a_bytes / 2**30))
         if (cfg.a_bytes >= 2 * (126 << 20) and cfg.layout != "csr")
         else ("L2 flushed before every step (512 MiB write; A = %.1f MiB)"
               % (cfg.a_bytes / 2**20))}
    if extra:
        o.update(extra)
    return o


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg_name: str, group: str):
    """DRAM read+write bytes per launch of the group's dominant kernel, from the
    committed `ncu --set full` summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(cfg_name, {}).get(group)
    except Exception:
        return None


DMMA_TFLOPS = 36.8  # fp64 DMMA peak measured on this pool's B200 (tools/probe/probe.cu, profiles/r01/probe.txt)
RED_GPS = 179.5  # fp64 RED.ADD throughput into an L2-resident 64 MB array, G/s (same probe)


def algorithmic(cfg, group, n_loc, nnz_loc, steps_launches):
    """(bytes or flops per step, kind, kernel label) of one kernel group, from
    SURVEY.md 8(d)'s per-unit figures."""
    d, m, s = cfg.d, cfg.m, cfg.s
    M = m // s
    if group == "sketch":
        # A read ONCE per iteration (8d B per row) + b and the
        # perm entry per row + the SA / gradient-partial writes.  For an SJLT
        # (s > 1) the design reads A s times (one bucket-ordered pass per
        # block), which shows up as DRAM traffic ~s x
        # the algorithmic bytes, not as algorithmic work.
        b = 8 * n_loc * d + 12 * n_loc + 8 * M * d + 8 * m * d
        label = "cs_gather_tma_kernel (bucket-ordered sketch, gradient fused)"
        if s > 1:
            label += f"; SJLT: {s} bucket-ordered passes over A (A read {s}x)"
        return b, "hbm", label
    if group == "sjlt":
        # one-read SJLT (sjlt_onepass.cu): A once + the SA write
        return 8 * n_loc * d + 8 * m * d, "hbm", "sjlt_onepass_kernel (one read of A; column-slice CTAs)"
    if group == "grad":
        return 8 * n_loc * d + 8 * n_loc, "hbm", "grad_dense_kernel"
    if group == "csr":  # bound by the s fp64 reductions per nonzero into the L2-resident SA
        return float(s) * nnz_loc, "l2_red", "csr_sketch_grad_kernel (REDG.ADD.F64 into L2-resident SA)"
    if group == "gram":
        return float(m) * d * d, "tensor", "gram_kernel (DMMA m8n8k4 f64, symmetric half)"
    return None, "latency", group


def roofline(prof, cfg, n_loc, nnz_loc, steps):
    """Achieved vs peak for the dominant kernel group of the step: algorithmic
    bytes (flops) per launch / the group's average launch time from the
    library's CUDA events on its stream."""
    peaks, peak_src = measured_peaks()
    groups = {k: v for k, v in prof.items() if v[1] > 0}
    # the sort prefetch and the look-ahead factor run on side streams beside
    # the pass (their event times include waiting for SM slots): not candidates
    main = {k: v for k, v in groups.items() if k not in ("sort", "factor")} or groups
    if not groups:
        return None
    name = max(main, key=lambda k: main[k][0])
    tot, k = groups[name]
    per_step = tot / steps
    avg = tot / k
    launches_per_step = k / steps
    alg, kind, label = algorithmic(cfg, name, n_loc, nnz_loc, launches_per_step)
    out = {"kernel_group": name, "kernel": label, "avg_launch_ms": avg, "launches_per_step": launches_per_step,
           "ms_per_step": per_step}
    if alg is None:
        out.update({"bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None})
    elif kind == "hbm":
        per_launch = alg / launches_per_step
        ach = per_launch / (avg / 1e3) / 1e9
        out.update({"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / peaks["hbm_gbs"], "algorithmic_bytes_per_launch": per_launch,
                    "peak_source": f"{peak_src} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)"})
        if ach > peaks["hbm_gbs"]:
            out["peak_note"] = ("the peak is a measured COPY (half reads, half writes); this kernel's traffic is "
                                "almost all reads, which HBM3e serves slightly faster than a read/write mix, so the "
                                "fraction can exceed 1 by a fraction of a percent")
    elif kind == "l2_red":
        per_launch = alg / launches_per_step
        ach = per_launch / (avg / 1e3) / 1e9
        out.update({"bound": "l2_red", "achieved": ach, "peak": RED_GPS, "unit": "G red/s",
                    "frac": ach / RED_GPS, "algorithmic_reds_per_launch": per_launch,
                    "peak_source": "measured fp64 RED.ADD throughput, random addresses in 64 MB (tools/probe/probe.cu)"})
    else:
        per_launch = alg / launches_per_step
        ach = per_launch / (avg / 1e3) / 1e12
        out.update({"bound": "tensor", "achieved": ach, "peak": DMMA_TFLOPS, "unit": "TFLOP/s",
                    "frac": ach / DMMA_TFLOPS, "algorithmic_flops_per_launch": per_launch,
                    "peak_source": "measured fp64 DMMA m8n8k4 throughput (tools/probe/probe.cu)"})
    tr = ncu_traffic(cfg.name, name)
    traffic = tr.get("dram_bytes_per_launch") if isinstance(tr, dict) else tr
    if traffic is not None and cfg.layout == "dense" and n_loc != cfg.n:
        # the committed capture is of the single-GPU run; a rank streams n_loc of the n rows
        traffic = traffic * n_loc / cfg.n
        out["traffic_scaled_to_rank"] = f"single-GPU ncu bytes x {n_loc}/{cfg.n} rows"
    out["traffic"] = traffic
    if isinstance(tr, dict):
        out["traffic_source"] = tr.get("source")
    if name == "csr" and kind == "l2_red":
        # the same pass against HBM: the CSR stream (8 B row_ptr + 8 B b per row, 12 B per nonzero), x and the SA write
        hb = 16.0 * n_loc + 12.0 * nnz_loc + 8.0 * cfg.m * cfg.d
        ach_h = hb / (avg / 1e3) / 1e9
        out["hbm"] = {"achieved": ach_h, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ach_h / peaks["hbm_gbs"],
                      "algorithmic_bytes_per_launch": hb}
    if name == "sjlt" and kind == "hbm":
        # the pass is bound by shared-memory bandwidth, not HBM: every element of A is
        # written to shared memory once (TMA) and read once per SJLT block by its bucket's owner thread
        smem_bytes = (8.0 + 8.0 * s_of(cfg)) * n_loc * cfg.d
        clk = CLOCK_MHZ[0] or 1965.0
        peak = 128.0 * NUM_SMS[0] * clk * 1e6 / 1e9
        ach = smem_bytes / (avg / 1e3) / 1e9
        out["onchip"] = {"bound": "smem", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "algorithmic_bytes_per_launch": smem_bytes,
                         "peak_source": f"128 B/clk/SM x {NUM_SMS[0]} SMs x {clk:.0f} MHz (median SM clock of the run)"}
    return out


CLOCK_MHZ = [None]
NUM_SMS = [148]


def s_of(cfg):
    return cfg.s


def nccl_summary(path):
    """What NCCL's INFO log says about the communicator (ranks, NVLS), or None."""
    if not path or not os.path.exists(path):
        return None
    nranks, nvls, version = None, False, None
    with open(path, errors="replace") as f:
        for ln in f:
            if "nRanks" in ln and nranks is None:
                try:
                    nranks = int(ln.split("nRanks")[1].split()[0])
                except (IndexError, ValueError):
                    pass
            if "NVLS" in ln and ("enabled" in ln.lower() or "multicast" in ln.lower() or "comm" in ln):
                nvls = True
            if "NCCL version" in ln and version is None:
                version = ln.split("NCCL version", 1)[1].strip().split()[0]
    return {"version": version, "nranks": nranks, "nvls_mentioned": nvls, "log": path}


# ----------------------------------------------------------------------------- host / cpu baseline
def host_info():
    model, mem = None, None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    mem = int(ln.split()[1]) * 1024
                    break
    except OSError:
        pass
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"cpu_model": model, "host_cores": cores, "ram_bytes": mem}


def cpu_baseline(cfg, A_np, b_np, radius, seconds):
    """The oracle as it stands on the host (rank 0, N = 1): whole IHS iterations
    single-threaded on the full rows for about `seconds`, then one call of each
    phase (sketch, gradient, Gram, inner solve), and the OpenMP
    timing variants of the two row-parallel phases on all host cores."""
    import numpy as np

    import oracle
    d = cfg.d
    kw = dict(constraint=cfg.constraint, tau=radius) if cfg.constraint in ("l1ball", "lasso") else {}
    x = np.zeros(d)
    it = 0
    t0 = time.perf_counter()
    while True:
        xh_o, _ = oracle.ihs_solve(A_np, b_np, seed=cfg.hash_seed, m=cfg.m, s=cfg.s, T=1, iter0=it, x0=x, **kw)
        x = xh_o[-1]
        it += 1
        el = time.perf_counter() - t0
        if el >= seconds or it >= 50:
            break

    def timed(fn):
        t = time.perf_counter()
        r = fn()
        return r, 1e3 * (time.perf_counter() - t)

    SA, t_sk = timed(lambda: oracle.sketch_dense(A_np, cfg.hash_seed, it, cfg.m, cfg.s))
    g, t_gr = timed(lambda: oracle.grad_dense(A_np, b_np, x))
    H, t_gm = timed(lambda: oracle.gram(SA))
    if cfg.constraint == "ols":
        _, t_so = timed(lambda: oracle.ols_step(H, g, x))
    elif cfg.constraint == "l1ball":
        _, t_so = timed(lambda: oracle.l1ball_step(H, g, x, radius))
    else:
        _, t_so = timed(lambda: oracle.lasso_step(H, g, x, radius))
    threads = oracle.omp_threads()
    oracle.grad_dense_omp(A_np[:4096], b_np[:4096], x)  # thread pool warm-up
    _, t_sko = timed(lambda: oracle.sketch_dense_omp(A_np, cfg.hash_seed, it, cfg.m, cfg.s))
    _, t_gro = timed(lambda: oracle.grad_dense_omp(A_np, b_np, x))
    t_omp = t_sko + t_gro + t_gm + t_so
    out = {"value": cfg.n * it / el, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"full {cfg.name} rows ({cfg.n}x{d}), {it} oracle IHS iterations, single thread, {el:.1f} s",
           "per_phase_ms_single_thread": {"sketch": t_sk, "gradient": t_gr, "gram": t_gm, "solve": t_so},
           "openmp": {"cores": threads, "sketch_ms": t_sko, "gradient_ms": t_gro,
                      "iteration_rows_per_s": cfg.n / (t_omp / 1e3),
                      "note": "row-parallel phases (sketch, gradient) on all host cores, partials merged in "
                              "thread order (oracle/ihs_oracle_omp.c); Gram and solve single-threaded"}}
    out.update(host_info())
    return out


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    import synthetic
    cfg = synthetic.CONFIGS[args.config]
    if cfg.layout != "dense":
        print(json.dumps({"impl": "reference", "unavailable": "reference arm implemented for dense configs"}))
        return 0
    # the full configuration (same rows as the product arm: same_config); one
    # oracle IHS iteration (~1.6 s single-threaded for C2) per step
    rows = cfg.n
    prob = synthetic.problem(cfg, "cpu")
    A, b = prob["A"].numpy(), prob["b"].numpy()
    kw = {}
    if cfg.constraint != "ols":
        kw = dict(constraint=cfg.constraint, tau=float(prob["tau"]) if cfg.constraint == "l1ball" else cfg.lam)
    x = np.zeros(cfg.d)
    for w in range(args.warmup):
        xh, _ = oracle.ihs_solve(A, b, seed=cfg.hash_seed, m=cfg.m, s=cfg.s, T=1, iter0=w, x0=x, **kw)
        x = xh[-1]
    t0 = time.perf_counter()
    for k in range(args.steps):
        xh, _ = oracle.ihs_solve(A, b, seed=cfg.hash_seed, m=cfg.m, s=cfg.s, T=1, iter0=args.warmup + k, x0=x,
                                 **kw)
        x = xh[-1]
    el = time.perf_counter() - t0
    value = rows * args.steps / el
    sample = f"all {rows} rows of {cfg.name} ({rows}x{cfg.d}), one single-threaded oracle IHS iteration per step"
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded, BASELINE.json recipe)", "config": config_obj(cfg, 1),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


# ----------------------------------------------------------------------------- product arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_1910_14166_b200 as P
    import synthetic
    from paper_1910_14166_b200.dist import CudaOps, ShardedIHS, shard_rows

    rank, world, local = dist_env()
    if os.environ.get("IHS_BENCH_SHARE_GPU") == "1":  # test mode: every rank on cuda:0
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl = args.dist_backend == "nccl"
    nccl_log = None
    if world > 1:
        if nccl:
            # NCCL's own INFO log (ranks, transports, NVLS) to a file, read back below
            nccl_log = f"/tmp/ihs_bench_nccl.{os.getpid()}.log"
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV,NVLS")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/ihs_bench_nccl.%p.log")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    cfg = synthetic.CONFIGS[args.config]
    r0, r1 = shard_rows(cfg.n, rank, world)
    # ---- inputs, resident in HBM before timing
    xs = synthetic.x_star(cfg, dev)
    radius = float(xs.abs().sum()) if cfg.constraint == "l1ball" else (cfg.lam if cfg.constraint == "lasso" else 0.0)
    if cfg.layout == "dense":
        A = synthetic.dense_A(cfg, dev, rows=(r0, r1))
        b = (A @ xs + synthetic.noise(cfg, dev)[r0:r1]).contiguous()
        Am = P.Dense(A, row_offset=r0)
        nnz = n_loc_nnz = None
    else:  # CSR: every rank draws the whole structure once and keeps its row block
        rp, cl, vl = synthetic.csr_A(cfg, dev)
        b = (synthetic.csr_matvec(rp, cl, vl, xs) + synthetic.noise(cfg, dev))[r0:r1].contiguous()
        e0, e1 = int(rp[r0]), int(rp[r1])
        Am = P.Csr((rp[r0:r1 + 1] - e0).contiguous(), cl[e0:e1].contiguous(), vl[e0:e1].contiguous(), cfg.d,
                   row_offset=r0)
        nnz = int(rp[-1])
        n_loc_nnz = e1 - e0
        del rp, cl, vl
        A = None
    del xs
    ctx = P.Context(local)
    if args.la_gram_sms >= 0:
        ctx.set_option("la_gram_sms", args.la_gram_sms)
    if args.la_gram_tile >= 0:
        ctx.set_option("la_gram_tile", args.la_gram_tile)
    spec = P.Spec(m=cfg.m, s=cfg.s, seed=cfg.hash_seed)
    exch = None
    if world > 1 and args.allreduce == "nvls":
        from paper_1910_14166_b200.dist import NvlsAllreduce
        exch = NvlsAllreduce(cfg.m * cfg.d + cfg.d, dev, ctx=ctx)
    S = ShardedIHS(Am, b, spec, ops=CudaOps(ctx), constraint=cfg.constraint, radius=radius, allreduce=exch,
                   lookahead=None if args.lookahead < 0 else bool(args.lookahead))
    d = cfg.d
    xa = torch.zeros(d, dtype=torch.float64, device=dev)
    xb = torch.empty_like(xa)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            if nccl:
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    # configs whose inputs (nearly) fit in the 126 MB L2 are timed step by step
    # with L2 flushed between steps (a 512 MiB write outside the timed events)
    flush = cfg.layout == "csr" or cfg.a_bytes < 2 * (126 << 20)
    fbuf = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if flush else None
    t = 0
    flush_info = None
    for _ in range(max(args.warmup, 3) if args.warmup >= 0 else 3):
        S.step(t, xa, xb)
        xa, xb = xb, xa
        t += 1
    barrier()
    x_start, t_start = xa.clone(), t  # the profiled pass below replays these steps
    l0 = ctx.kernel_launches
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    # a latency-bound small problem on one rank: the K steps are ONE public
    # ihs_solve_ols call (one launch per iteration there, small_step.cu), after
    # an L2 flush; Python call overhead per step would otherwise be timed as
    # GPU idle time
    solve_mode = world == 1 and cfg.layout == "dense" and cfg.constraint == "ols" and cfg.a_bytes < (16 << 20)
    if solve_mode:
        xo_dev = torch.empty(d, dtype=torch.float64, device=dev)
        xh_dev = torch.empty((args.steps + 1, d), dtype=torch.float64, device=dev)
        for _ in range(2):
            P.ihs_solve_ols(Am, b, spec, args.steps, iter0=t, x0=xa, ctx=ctx, x_out=xo_dev, x_hist=xh_dev)
        reps = []
        for _ in range(5):
            fbuf.zero_()
            e0.record(stream)
            P.ihs_solve_ols(Am, b, spec, args.steps, iter0=t, x0=xa, ctx=ctx, x_out=xo_dev, x_hist=xh_dev)
            e1.record(stream)
            e1.synchronize()
            reps.append(e0.elapsed_time(e1))
        ms_local = statistics.median(reps)
        xa.copy_(xo_dev)
        t += args.steps
    elif flush and args.step_sync_flush:
        ms_local = 0.0
        for _ in range(args.steps):
            fbuf.zero_()
            e0.record(stream)
            S.step(t, xa, xb)
            e1.record(stream)
            e1.synchronize()
            ms_local += e0.elapsed_time(e1)
            xa, xb = xb, xa
            t += 1
    elif flush:
        # K consecutive steps with the L2 flush INSIDE the timed region (stream-ordered
        # between steps), so work a step leaves on the side streams (the look-ahead Gram)
        # is timed too; the flush's own time (measured alone) is subtracted afterwards
        fl = []
        for _ in range(5):
            e0.record(stream)
            fbuf.zero_()
            e1.record(stream)
            e1.synchronize()
            fl.append(e0.elapsed_time(e1))
        flush_ms = statistics.median(fl)
        e0.record(stream)
        for _ in range(args.steps):
            fbuf.zero_()
            S.step(t, xa, xb)
            xa, xb = xb, xa
            t += 1
        e1.record(stream)
        e1.synchronize()
        ms_incl_flush = e0.elapsed_time(e1)
        ms_local = ms_incl_flush - args.steps * flush_ms
        flush_info = {"flush_ms": flush_ms, "ms_per_step_incl_flush": ms_incl_flush / args.steps}
    else:
        e0.record(stream)
        for _ in range(args.steps):
            S.step(t, xa, xb)
            xa, xb = xb, xa
            t += 1
        e1.record(stream)
        e1.synchronize()
        ms_local = e0.elapsed_time(e1)
    barrier()
    clk = clocks.stop()
    launches = ctx.kernel_launches - l0
    # every rank must hold the same x (replicated deterministic a4/a6 on the all-reduced [SA | g])
    ranks_same = None
    if world > 1:
        xs = xa.cpu() if not nccl else xa
        allx = [torch.empty_like(xs) for _ in range(world)]
        dist.all_gather(allx, xs)
        ranks_same = all(torch.equal(allx[0], v) for v in allx)
    mt = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
    ms = float(mt.item())
    ms_step = ms / args.steps
    value = cfg.n * args.steps / (ms / 1e3)
    # ---- per-kernel-group breakdown: the same K steps (same iterations, same
    # starting x) replayed with the library's CUDA events around every group,
    # kept out of the timed loop above
    xa.copy_(x_start)
    t = t_start
    S.prime(t)  # the look-ahead prologue (a no-op otherwise), outside the profiled steps
    ctx.set_profiling(True)
    ctx.profile_reset()
    barrier()
    if solve_mode:
        P.ihs_solve_ols(Am, b, spec, args.steps, iter0=t, x0=xa, ctx=ctx, x_out=xo_dev, x_hist=xh_dev)
    else:
        for _ in range(args.steps):
            S.step(t, xa, xb)
            xa, xb = xb, xa
            t += 1
    barrier()
    prof = {name: ctx.profile(k) for k, name in enumerate(P.KERNEL_GROUPS)}
    ctx.set_profiling(False)
    # ---- roofline of the dominant kernel group (C2: the fused sketch+gradient gather)
    n_loc = r1 - r0
    CLOCK_MHZ[0] = clk.get("sm_mhz") if clk else None
    NUM_SMS[0] = torch.cuda.get_device_properties(dev).multi_processor_count
    roof = roofline(prof, cfg, n_loc, n_loc_nnz, args.steps)
    breakdown = {name: {"ms_per_step": v[0] / args.steps, "launches": v[1]} for name, v in prof.items() if v[1]}
    if roof and roof.get("kernel_group") == "csr" and S.lookahead:
        # in the look-ahead schedule the pass shares the SMs with the Gram of the next sketch, so its
        # in-situ launch time is not the kernel's own: time the same call alone (nothing on the side
        # streams, L2 flushed before each launch) and rate it next to the in-situ figure
        torch.cuda.synchronize()
        al = []
        for k in range(5):
            fbuf.zero_()
            e0.record(stream)
            S.ops.sketch_grad(S.A, S.spec, t + 100 + k, S.b, xa, S.SA, S.g)
            e1.record(stream)
            e1.synchronize()
            al.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        alone = statistics.median(al)
        roof["in_situ"] = "beside the look-ahead Gram of the next sketch (shared SMs)"
        roof["alone"] = {"avg_launch_ms": alone, "achieved": roof["algorithmic_reds_per_launch"] / (alone / 1e3) / 1e9,
                         "unit": roof["unit"], "frac": roof["algorithmic_reds_per_launch"] / (alone / 1e3) / 1e9
                         / roof["peak"], "timing": "median of 5 launches alone, L2 flushed before each"}
    # ---- time to 1e-10 (IHS solve from x^0 = 0; errors post hoc, outside the timing)
    ttt = None
    if not args.no_ttt and (cfg.layout == "dense" or cfg.constraint == "ols"):
        if cfg.constraint != "ols":
            xopt = S.exact_constrained()
        else:  # CSR: no dense Gram of A; CG on the normal equations through the gradient kernel
            xopt = S.exact_ols() if cfg.layout == "dense" else S.exact_ols_normal_cg()
        Tmax = 60 if cfg.constraint == "ols" else 40
        xh = S.solve(Tmax, iter0=1000)
        err = S.pred_errors(xh, xopt).cpu().tolist()
        tstar = next((k for k, e in enumerate(err) if e <= 1e-10), None)
        ttt = {"target": 1e-10, "iterations": tstar, "err_at_20": err[20], "err_final": err[-1],
               "errors_first": [float("%.3e" % e) for e in err[:tstar + 1 if tstar else 31]]}
        if tstar:
            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x0 = torch.zeros(d, dtype=torch.float64, device=dev)
            xh2 = torch.zeros((tstar + 1, d), dtype=torch.float64, device=dev)
            f0.record(stream)
            for k in range(tstar):
                S.step(1000 + k, xh2[k], xh2[k + 1])
            f1.record(stream)
            f1.synchronize()
            tt = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ttt["ms"] = float(tt.item())
            ttt["bitwise_same_as_first_run"] = bool(torch.equal(xh2[tstar], xh[tstar]))
            if cfg.constraint != "ols":
                # the PG step bound L comes from a power iteration warm-started from the
                # context's previous update (ihs_inner_cfg.warm_power_iters, "pg_warm"): the
                # second run starts from the first run's vector, so its iterates agree to
                # rounding (same minimiser), not bitwise; "pg_warm" 0 makes them bitwise
                ttt["rel_diff_vs_first_run"] = float(
                    (xh2[tstar] - xh[tstar]).norm() / xh[tstar].norm().clamp_min(1e-300))
            del x0
        del xh
    # ---- e2e: the public solve call with HOST (pinned) buffers, copies inside
    e2e = None
    if not args.no_e2e and world > 1 and not nccl:
        e2e = {"value": None, "unit": UNIT, "error": "the e2e solve all-reduces through NCCL; skipped with gloo"}
    elif not args.no_e2e and cfg.layout == "dense" and cfg.constraint == "ols":
        try:
            T_e2e = (ttt or {}).get("iterations") or 30
            A_h = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
            A_h.copy_(A)
            b_h = torch.empty(b.shape, dtype=torch.float64, pin_memory=True)
            b_h.copy_(b)
            ctx2 = P.Context(local)
            if world > 1:
                uid = [P.nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                ctx2.set_comm(rank, world, uid[0])
            xo_h = torch.empty(d, dtype=torch.float64, pin_memory=True)
            P.ihs_solve_ols(P.Dense(A_h, row_offset=r0), b_h, spec, T_e2e, iter0=1000, ctx=ctx2, x_out=xo_h,
                            x_hist=torch.empty((T_e2e + 1, d), dtype=torch.float64, device=dev))
            barrier()
            reps = 3
            times = []
            for _ in range(reps):
                barrier()
                t0 = time.perf_counter()
                P.ihs_solve_ols(P.Dense(A_h, row_offset=r0), b_h, spec, T_e2e, iter0=1000, ctx=ctx2, x_out=xo_h,
                                x_hist=torch.empty((T_e2e + 1, d), dtype=torch.float64, device=dev))
                times.append(time.perf_counter() - t0)
            te = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            sec = float(te.item())
            e2e = {"value": cfg.n * T_e2e / sec, "unit": UNIT, "h2d_bytes_per_step": 8 * n_loc * d + 8 * n_loc,
                   "d2h_bytes_per_step": 8 * d, "ms_per_step": sec * 1e3,
                   "step": f"one ihs_solve_ols call ({T_e2e} IHS iterations) on host-pinned A, b; x read back",
                   # the solve call's last pass forms g alone (no sketch to look ahead to), so x^T
                   # agrees with the step-by-step device run to rounding, not bit for bit
                   "x_rel_diff_vs_device_run": float(torch.linalg.norm(xo_h.to(dev) - xh2[T_e2e])
                                                     / torch.linalg.norm(xh2[T_e2e]))
                   if ttt and ttt.get("iterations") and T_e2e == ttt["iterations"] else None}
            ctx2.close()
            del A_h, b_h
        except Exception as ex:  # report, do not hide
            e2e = {"value": None, "unit": UNIT, "error": repr(ex)[:300]}
    # ---- cpu baseline: the oracle, as it stands, rank 0 at N = 1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and cfg.layout == "dense":
        A_np = A.cpu().numpy()
        cpu = cpu_baseline(cfg, A_np, b.cpu().numpy(), radius, args.cpu_seconds)
        del A_np
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json recipe)",
               "timing": ("median of 5 public ihs_solve_ols calls of K iterations each (device events around the "
                          "call, L2 flushed before it)") if solve_mode else
                         ("K steps, device events per step (flush, step, sync), L2 flushed between steps"
                          if flush and args.step_sync_flush else
                          "K consecutive steps between two device events with an L2 flush (512 MiB write) before "
                          "every step INSIDE the region; K x the flush's own time (measured alone) subtracted"
                          if flush else "K consecutive steps between two device events"),
               "config": config_obj(cfg, world, {"per_gpu_rows": n_loc, "schedule": (
                   "one-launch small step per iteration (small_step.cu)" if solve_mode else
                   ("look-ahead Gram (H_{t+1} after the CG update of t, beside the next pass; DESIGN.md section 9)"
                    if cfg.constraint == "ols" else
                    "look-ahead Gram (H_{t+1} beside the update of t; DESIGN.md section 9)")
                   if S.lookahead and S.la_gram_only else
                   "look-ahead (H^-1 of the next sketch beside the pass; DESIGN.md section 9)" if S.lookahead
                   else "plain")}),
               "hbm_GBps_step": (cfg.a_bytes / world) / (ms_step / 1e3) / 1e9,
               "roofline": roof, "breakdown_ms": breakdown, "time_to_1e-10": ttt, "e2e": e2e,
               "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clk,
               "gpu": torch.cuda.get_device_name(dev)}
        if flush_info:
            out["l2_flush"] = flush_info
        if world > 1:
            out["ranks_bitwise_identical_x"] = ranks_same
            out["dist_backend"] = args.dist_backend
            out["exchange"] = ("NVLS multimem kernel (ihs_allreduce_multimem)" if args.allreduce == "nvls"
                               else "NCCL all-reduce")
            out["nccl"] = nccl_summary(nccl_log)
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
