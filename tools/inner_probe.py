"""Inner PG steps per IHS iteration on C4 (l1 ball) and C4P (LASSO), full size,
through ShardedIHS / CudaOps (the bench's path).  python tools/inner_probe.py"""
import sys, torch
sys.path.insert(0, '.')
import paper_1910_14166_b200 as P, synthetic
from paper_1910_14166_b200.dist import CudaOps, ShardedIHS
dev = torch.device('cuda', 0)
for name in ['C4', 'C4P']:
    cfg = synthetic.CONFIGS[name]
    A = synthetic.dense_A(cfg, dev); xs = synthetic.x_star(cfg, dev)
    b = (A @ xs + synthetic.noise(cfg, dev)).contiguous()
    radius = float(xs.abs().sum()) if cfg.constraint == 'l1ball' else cfg.lam
    ctx = P.Context(0)
    S = ShardedIHS(P.Dense(A), b, P.Spec(m=cfg.m), ops=CudaOps(ctx), constraint=cfg.constraint, radius=radius)
    x = torch.zeros(cfg.d, dtype=torch.float64, device=dev); xn = torch.empty_like(x)
    its = []
    for t in range(25):
        S.step(t, x, xn); torch.cuda.synchronize(); its.append(int(S.inner.item())); x, xn = xn, x
    print(name, its, flush=True)
    del A, b, S
    torch.cuda.empty_cache()
