"""PG inner-step time on C4 / C4P (the l1-ball and LASSO inner solver, pg.cu):
a traced C-ABI solve reports, per IHS iteration, the inner iteration count and
the device time of the update; their ratio is the time per inner step.  Not a
bench line (bench.py is).  usage: python tools/pg_probe.py [C4|C4P] [T]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_14166_b200 as P  # noqa: E402
import synthetic  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 12
cfg = synthetic.PRESETS[name] if hasattr(synthetic, "PRESETS") else synthetic.CONFIGS[name]
dev = torch.device("cuda", 0)
pb = synthetic.problem(cfg, dev)
spec = P.Spec(m=cfg.m, s=cfg.s)
for cl in (0, 4, 8):
    ctx = P.Context(0)
    ctx.set_profiling(True)
    if cl:
        ctx.set_option("pg_cluster", cl)
    for rep in range(2):
        if cfg.constraint == "lasso":
            out = P.ihs_solve_lasso(pb["A"], pb["b"], pb["lam"], spec, T, trace=True, ctx=ctx)
        else:
            out = P.ihs_solve_l1ball(pb["A"], pb["b"], pb["tau"], spec, T, trace=True, ctx=ctx)
        ctx.synchronize()
    tr = out["trace"]
    inner = [r["inner_iters"] for r in tr]
    ts = [r["t_solve"] for r in tr]
    per = [1e3 * t / max(k, 1) for t, k in zip(ts, inner)]
    print(f"{name} pg_cluster={cl or 'default'}: inner {inner}")
    print(f"   t_solve ms {[round(t, 4) for t in ts]}")
    print(f"   us/inner step {[round(p, 3) for p in per]}  (t >= 3 mean {sum(per[3:]) / max(1, len(per[3:])):.3f})")
    ctx.close()
