"""Per-kernel microbenchmarks through the C ABI (CUDA events, warm)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1910_14166_b200 as P

def bench(fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us

dev = torch.device("cuda", 0)
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("chol", "all"):
    for d in (10, 96, 128, 160, 256, 1024):
        Q, _ = torch.linalg.qr(torch.randn(d, d, dtype=torch.float64, device=dev))
        H = (Q * torch.linspace(1, 13, d, dtype=torch.float64, device=dev)) @ Q.T
        g = torch.randn(d, dtype=torch.float64, device=dev); x = torch.zeros_like(g); xn = torch.empty_like(g)
        print(f"chol d={d}: {bench(lambda: P.ihs_ols_update(H, g, x, out=xn)):.1f} us")
if what in ("gram", "all"):
    for m, d in ((1024, 128), (2048, 256), (4096, 96), (8192, 1024)):
        SA = torch.randn(m, d, dtype=torch.float64, device=dev); Hh = torch.empty(d, d, dtype=torch.float64, device=dev)
        us = bench(lambda: P.ihs_gram(SA, out=Hh), reps=10)
        print(f"gram m={m} d={d}: {us:.1f} us  {m*d*d/us/1e6:.2f} TFLOP/s (sym) ")
if what in ("pg", "all"):
    d = 256
    Q, _ = torch.linalg.qr(torch.randn(d, d, dtype=torch.float64, device=dev))
    H = (Q * torch.linspace(1, 13, d, dtype=torch.float64, device=dev)) @ Q.T * 1e4
    g = torch.randn(d, dtype=torch.float64, device=dev) * 100; x = torch.zeros_like(g); xn = torch.empty_like(g)
    inner = torch.zeros(1, dtype=torch.int32, device=dev)
    us = bench(lambda: P.ihs_l1ball_update(H, g, x, 10.0, out=xn, inner=inner), reps=5)
    print(f"pg d=256: {us:.1f} us, inner iters {int(inner.item())}, {us/max(1,int(inner.item())):.2f} us/step")
