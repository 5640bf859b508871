"""Small-shape driver for compute-sanitizer (racecheck / synccheck / memcheck):
one call of every kernel family of the hot path through the C ABI, each on a
shape that still exercises its multi-CTA / cluster / pipeline structure.
Run plain first (it must exit 0), then under ONE sanitizer tool per call:

  compute-sanitizer --tool racecheck --error-exitcode 7 python tools/sanitize_run.py

Kernels covered: hash export; counting sort (hist, scan,
scatter); cs_gather_tma_kernel (TMA bulk ring, fused gradient, SJLT batches);
sjlt_lists_kernel + sjlt_onepass_kernel (TMA tensor ring); CSR sketch+grad;
gram (split-K and stream-K); gram_ols_kernel (cluster, DSMEM); the look-ahead
factor cluster + reduce_rows_last_kernel (apply in the last CTA); chol blocked;
ols_large_kernel (cooperative CG, and the in-launch Cholesky fallback); the
pg_warp_kernel cluster (l1 ball, LASSO, warm power); the host-pointer e2e solve.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_14166_b200 as P  # noqa: E402

DEV = torch.device("cuda", 0)


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def main():
    rng = np.random.default_rng(0)
    ctx = P.Context(0)
    # a1 hash export, a2 CountSketch (sort + TMA gather, fused gradient), SJLT batches
    A = rng.standard_normal((20_000, 64))
    b = rng.standard_normal(20_000)
    x = rng.standard_normal(64) * 0.1
    P.ihs_hash(P.Spec(m=256, s=4), 1, 0, 1000, ctx=ctx)
    P.ihs_sketch_grad(t(A), P.Spec(m=256), 1, t(b), t(x), ctx=ctx)
    c0 = P.Context(0)
    c0.set_option("sjlt_onepass", 0)
    P.ihs_sketch(t(A), P.Spec(m=512, s=4), 2, ctx=c0)
    # one-read SJLT (lists + onepass, ragged last chunk), gradient beside it
    P.ihs_sketch_grad(t(A[:9_001]), P.Spec(m=1024, s=8), 3, t(b[:9_001]), t(x), ctx=ctx)
    # CSR sketch + gradient
    n, d = 5000, 40
    nnz_row = rng.integers(0, 4, n)
    rp = np.concatenate([[0], np.cumsum(nnz_row)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(d, k, replace=False)) for k in nnz_row]).astype(np.int32)
    vals = rng.standard_normal(int(rp[-1]))
    P.ihs_sketch_grad((t(rp), t(cols), t(vals), d), P.Spec(m=128, s=4), 1, t(b[:n]), t(x[:d]), ctx=ctx)
    # Gram: split-K and stream-K (many tiles)
    P.ihs_gram(t(rng.standard_normal((512, 96))), ctx=ctx)
    P.ihs_gram(t(rng.standard_normal((1024, 640))), ctx=ctx)
    # a4 + a6 fused cluster (d <= 64), look-ahead factor cluster + apply in the last reducing CTA
    SA = t(rng.standard_normal((512, 48)))
    P.ihs_gram_ols_update(SA, t(rng.standard_normal(48)), t(np.zeros(48)), ctx=ctx)
    Hinv = P.ihs_ols_factor(t(rng.standard_normal((1024, 128))), ctx=ctx)
    ctx.synchronize()  # (the driver reads Hinv next)
    Hinv2 = torch.empty_like(Hinv)
    P.ihs_ols_lookahead_step(t(A[:, :64].copy()), P.Spec(m=256), 2, t(b), t(x), Hinv[:64, :64].contiguous(),
                             SA_next=torch.empty((256, 64), dtype=torch.float64, device=DEV),
                             Hinv_next=Hinv2[:64, :64].contiguous(), ctx=ctx)
    # Cholesky (one CTA) and the large-d cooperative solve: CG, then the Cholesky fallback
    Q, _ = np.linalg.qr(rng.standard_normal((200, 200)))
    Hs = (Q * np.geomspace(1, 50, 200)) @ Q.T
    P.ihs_ols_update(t(Hs[:100, :100] + 100 * np.eye(100)), t(rng.standard_normal(100)), t(np.zeros(100)), ctx=ctx)
    P.ihs_ols_update(t(Hs), t(rng.standard_normal(200)), t(np.zeros(200)), ctx=ctx)
    c2 = P.Context(0)
    c2.set_option("ols_large", 2)
    P.ihs_ols_update(t(Hs), t(rng.standard_normal(200)), t(np.zeros(200)), ctx=c2)
    # PG cluster: l1 ball twice (warm power iteration) and LASSO
    Hp = t((Q[:64, :64] * np.geomspace(1, 10, 64)) @ Q[:64, :64].T + np.eye(64))
    gp = t(rng.standard_normal(64) * 10)
    for _ in range(2):
        P.ihs_l1ball_update(Hp, gp, t(np.zeros(64)), 2.0, ctx=ctx)
    P.ihs_lasso_update(Hp, gp, t(np.zeros(64)), 1.0, ctx=ctx)
    # the look-ahead l1 loop and the host-pointer (e2e) OLS solve
    Ah = torch.from_numpy(A[:, :32].copy()).pin_memory()
    bh = torch.from_numpy(b).pin_memory()
    cl = P.Context(0)
    cl.set_option("lookahead", 1)
    P.ihs_solve_l1ball(t(A[:, :32].copy()), t(b), 3.0, P.Spec(m=256), 4, ctx=cl)
    P.ihs_solve_ols(Ah, bh, P.Spec(m=256), 4, ctx=ctx)
    for c in (ctx, c0, c2, cl):
        c.synchronize()
    torch.cuda.synchronize()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
