"""Time the dense SJLT sketch at C5's shape (2^25 x 96, m = 4096, s = 8): the
one-read path (default) against the s sorted passes (IHS_SJLT=passes), with the
library's per-group CUDA events.  Not a bench line (bench.py is)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_14166_b200 as P  # noqa: E402

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 25
d, m, s = 96, 4096, 8
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
A = torch.randn((n, d), dtype=torch.float64, device=dev, generator=g)
b = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
x = torch.randn(d, dtype=torch.float64, device=dev, generator=g) * 0.1
spec = P.Spec(m=m, s=s)
res = {}
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["onepass", "gradpass", "passes"]
for mode in modes:
    os.environ["IHS_SJLT"] = mode
    ctx = P.Context(0)
    ctx.set_profiling(True)
    for grad in (False, True):
        for _ in range(2):
            if grad:
                P.ihs_sketch_grad(A, spec, 1, b, x, ctx=ctx)
            else:
                P.ihs_sketch(A, spec, 1, ctx=ctx)
        ctx.synchronize()
        ctx.profile_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            if grad:
                _, SA, gg = P.ihs_sketch_grad(A, spec, 1, b, x, ctx=ctx)
            else:
                SA = P.ihs_sketch(A, spec, 1, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        groups = {name: ctx.profile(k) for k, name in enumerate(P.KERNEL_GROUPS)}
        line = " ".join(f"{k}={v[0] / reps:.3f}" for k, v in groups.items() if v[1])
        print(f"{mode:8s} grad={grad}: {e0.elapsed_time(e1) / reps:.3f} ms/call  [{line}]", flush=True)
        res[(mode, grad)] = SA.clone()
        ctx.profile_reset()
    ctx.close()
ref = res[(modes[-1], False)]
for mode in modes[:-1]:
    da = (res[(mode, True)] - ref).norm() / ref.norm()
    print(f"{mode} vs {modes[-1]} rel fro {da.item():.3e}")
