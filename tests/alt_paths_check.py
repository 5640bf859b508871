"""Parity checks of the option-selected alternative paths (ihs_ctx_set_option,
DESIGN.md section 1), run on one context by tests/test_gpu_alt_paths.py (or as
a script with the IHS_* environment).  Raises on the first failure.  Uses the
oracle (test infrastructure)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1910_14166_b200 as P  # noqa: E402
import synthetic  # noqa: E402

DEV = torch.device("cuda", 0)


def rel_fro(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def check(name, ok, detail=""):
    print(f"{name}: {'ok' if ok else 'FAIL'} {detail}", flush=True)
    if not ok:
        raise AssertionError(f"{name} {detail}")


def spd(rng, d, cond=13.0):
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    return (Q * np.geomspace(1.0, cond, d)) @ Q.T * 50.0


def main(ctx=None):
    oracle.build()
    ctx = ctx or P.Context(0)
    rng = np.random.default_rng(7)
    # a2 dense SJLT and CountSketch (+ fused gradient)
    for n, d, m, s in [(40_001, 97, 4096, 8), (20_000, 10, 200, 4), (30_000, 40, 512, 2), (9_000, 128, 1024, 1)]:
        A = rng.standard_normal((n, d))
        SA = P.ihs_sketch(torch.from_numpy(A).to(DEV), P.Spec(m=m, s=s, seed=0), 4, ctx=ctx).cpu().numpy()
        ref = oracle.sketch_dense(A, 0, 4, m, s)
        check(f"sketch n={n} d={d} m={m} s={s}", rel_fro(SA, ref) <= 1e-12, f"{rel_fro(SA, ref):.2e}")
    cfg, = [synthetic.CONFIGS["C2"].scaled(40_000)]
    prob = synthetic.problem(cfg, "cpu")
    A, b = prob["A"].numpy(), prob["b"].numpy()
    x = rng.standard_normal(cfg.d) * 0.1
    _, SA, g = P.ihs_sketch_grad(prob["A"].to(DEV), P.Spec(m=cfg.m), 3, prob["b"].to(DEV), torch.from_numpy(x).to(DEV),
                                 ctx=ctx)
    ok = np.array_equal(SA.cpu().numpy(), oracle.sketch_dense(A, 0, 3, cfg.m, 1))
    r = b - A @ x
    gb = 1e-12 * (np.abs(A) * np.abs(r)[:, None]).sum(0) + 1e-300
    check("fused sketch+grad (C2 shape)", ok and (np.abs(g.cpu().numpy() - oracle.grad_dense(A, b, x)) <= gb).all())
    # a6 OLS (Cholesky / CG), both sides of d = 160
    for d in (96, 160, 300):
        H = spd(rng, d)
        gv, xv = rng.standard_normal(d), rng.standard_normal(d)
        xn = P.ihs_ols_update(torch.from_numpy(H).to(DEV), torch.from_numpy(gv).to(DEV), torch.from_numpy(xv).to(DEV),
                              ctx=ctx)
        xo = oracle.ols_step(H, gv, xv)
        err = np.linalg.norm((xn.cpu().numpy() - xv) - (xo - xv)) / np.linalg.norm(xo - xv)
        check(f"ols update d={d}", err <= 1e-12, f"{err:.2e}")
    # a4 + a6 fused (fuse_max_d = 128 forces the cluster kernel up to d = 128)
    for m, d in ((1024, 128), (4096, 96)):
        SAm = rng.standard_normal((m, d))
        gv, xv = rng.standard_normal(d), rng.standard_normal(d)
        xn, Hg = P.ihs_gram_ols_update(torch.from_numpy(SAm).to(DEV), torch.from_numpy(gv).to(DEV),
                                       torch.from_numpy(xv).to(DEV), ctx=ctx)
        Ho = oracle.gram(SAm)
        xo = oracle.ols_step(Ho, gv, xv)
        err = np.linalg.norm((xn.cpu().numpy() - xv) - (xo - xv)) / np.linalg.norm(xo - xv)
        check(f"gram+ols d={d}", rel_fro(Hg.cpu().numpy(), Ho) <= 1e-12 and err <= 1e-11, f"{err:.2e}")
    # a6 l1 ball
    for d, tau in [(256, 10.0), (64, 2.0)]:
        H = spd(rng, d)
        gv = rng.standard_normal(d) * 10
        x0 = np.zeros(d)
        for rep in range(2):  # the second call exercises the warm-started power iteration
            xn = P.ihs_l1ball_update(torch.from_numpy(H).to(DEV), torch.from_numpy(gv).to(DEV),
                                     torch.from_numpy(x0).to(DEV), tau, ctx=ctx).cpu().numpy()
            xo, _, st = oracle.l1ball_step(H, gv, x0, tau)
            err = np.linalg.norm(xn - xo) / max(1.0, np.linalg.norm(xo))
            check(f"l1ball update d={d} call {rep}", st == oracle.OK and err <= 1e-10, f"{err:.2e}")
    # a1-a7: a short IHS solve (exercises the sort prefetch across iterations)
    cfg = synthetic.CONFIGS["C2"].scaled(1 << 15)
    prob = synthetic.problem(cfg, "cpu")
    A, b = prob["A"].numpy(), prob["b"].numpy()
    out = P.ihs_solve_ols(prob["A"].to(DEV), prob["b"].to(DEV), P.Spec(m=cfg.m), 6, ctx=ctx)
    xo, _ = oracle.ihs_solve(A, b, m=cfg.m, s=1, T=6)
    worst = max(oracle.pred_rel_err(a, c, A) for a, c in zip(out["x_hist"].cpu().numpy()[1:], xo[1:]))
    check("ihs solve C2 scaled", worst <= 1e-9, f"{worst:.2e}")
    # short solves (look-ahead: T = 1 is the prologue + one gradient-only pass)
    for T in (1, 2):
        out = P.ihs_solve_ols(prob["A"].to(DEV), prob["b"].to(DEV), P.Spec(m=cfg.m), T, iter0=5, ctx=ctx)
        xo, _ = oracle.ihs_solve(A, b, m=cfg.m, s=1, T=T, iter0=5)
        worst = max(oracle.pred_rel_err(a, c, A) for a, c in zip(out["x_hist"].cpu().numpy()[1:], xo[1:]))
        check(f"ihs solve C2 scaled T={T}", worst <= 1e-9, f"{worst:.2e}")
    print("ALL OK")


if __name__ == "__main__":
    main()
