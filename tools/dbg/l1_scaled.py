import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synthetic, paper_1910_14166_b200 as P
cfg = synthetic.CONFIGS["C4"].scaled(1 << 15)
prob = synthetic.problem(cfg, "cpu")
dev = torch.device("cuda", 0)
ctx = P.Context(0)
A, b, tau = prob["A"].to(dev), prob["b"].to(dev), prob["tau"]
S = None
for T in (1, 2, 4, 8):
    t0 = time.time()
    out = P.ihs_solve_l1ball(A, b, tau, P.Spec(m=cfg.m), T, trace=True, ctx=ctx)
    torch.cuda.synchronize()
    print(T, time.time() - t0, [r["inner_iters"] for r in out["trace"]], [r["status"] for r in out["trace"]], flush=True)
