"""GPU parity at BASELINE.json's FULL sizes (configs[1..4]), in the launch
configuration bench.py times (ShardedIHS.step through the C ABI), checked on
outputs the oracle can compute one by one:
  - buckets/signs of whole row windows (bit-exact),
  - sampled SA rows (oracle scans every row of A for the sampled buckets),
  - the full gradient (componentwise bound of reading R12),
  - the Gram of the GPU sketch and the inner update from the GPU (H, g),
  - one whole IHS step against the oracle where it finishes in seconds.
"""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1910_14166_b200 as P
    P.lib()
    return P


def rel_fro(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def grad_bound_chunked(A, b, x, chunk=1 << 20):
    tot = np.zeros(A.shape[1])
    for i in range(0, A.shape[0], chunk):
        Ai = A[i:i + chunk]
        r = b[i:i + chunk] - Ai @ x
        tot += np.abs(Ai).T @ np.abs(r)
    return 1e-12 * tot


def dense_full(name):
    cfg = synthetic.CONFIGS[name]
    prob = synthetic.problem(cfg, DEV)
    return cfg, prob


def check_hash(P, oracle_mod, cfg, t, windows):
    spec = P.Spec(m=cfg.m, s=cfg.s)
    for r0, cnt in windows:
        bg, sg = P.ihs_hash(spec, t, r0, cnt)
        bo, so = oracle_mod.hash_rows(0, t, cfg.m, cfg.s, r0, cnt)
        np.testing.assert_array_equal(bg.cpu().numpy(), bo)
        np.testing.assert_array_equal(sg.cpu().numpy(), so)


@pytest.mark.parametrize("name", ["C2", "C2-plain", "C4", "C5", "C4P"])
def test_dense_full_size(P, oracle_mod, name):
    """One step in the bench's launch configuration (C2, C4, C4P: the look-ahead
    schedule by default; C2-plain and C5 (SJLT): the plain one)."""
    from paper_1910_14166_b200.dist import CudaOps, ShardedIHS
    plain = name.endswith("-plain")
    name = name.split("-")[0]
    cfg, prob = dense_full(name)
    n, d = cfg.n, cfg.d
    t = 3
    check_hash(P, oracle_mod, cfg, t, [(0, 1 << 20), (n - (1 << 20), 1 << 20), (n // 2 + 12345, 99_999)])
    ctx = P.Context(0)
    spec = P.Spec(m=cfg.m, s=cfg.s)
    S = ShardedIHS(P.Dense(prob["A"]), prob["b"], spec, ops=CudaOps(ctx), constraint=cfg.constraint,
                   radius=prob["lam"] if cfg.constraint == "lasso" else prob["tau"], lookahead=False if plain else None)
    assert S.lookahead == (cfg.s == 1 and not plain)
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal(d) * 0.1).to(DEV)
    xn = torch.empty_like(x)
    S.step(t, x, xn)  # the bench's launch configuration
    torch.cuda.synchronize()
    assert ctx.status() == P.OK
    A = prob["A"].cpu().numpy()
    m = cfg.m
    if S.lookahead:  # prologue: S^t A in packs[0]; the step: [S^{t+1} A | g^t] in packs[1]
        SA, g = S.packs[0][: m * d].view(m, d).cpu().numpy(), S.packs[1][m * d:].cpu().numpy()
        SA1 = S.packs[1][: m * d].view(m, d).cpu().numpy()
        H = oracle_mod.gram(SA)
        if cfg.constraint == "ols":  # H^{-1} of S^t A
            assert rel_fro(S.Hinv[0].cpu().numpy() @ H, np.eye(d)) <= 1e-11
        else:  # the look-ahead Gram of S^t A (what the update used)
            H = S.Hinv[0].cpu().numpy()
            assert rel_fro(H, oracle_mod.gram(SA)) <= 1e-12
        rows1 = np.array([0, m - 1, m // 3])
        ref1 = oracle_mod.sketch_dense_rows(A, 0, t + 1, m, cfg.s, rows1)
        if cfg.s == 1:
            np.testing.assert_array_equal(SA1[rows1], ref1)
        else:
            assert rel_fro(SA1[rows1], ref1) <= 1e-12
    else:
        SA, g, H = S.SA.cpu().numpy(), S.g.cpu().numpy(), S.H.cpu().numpy()
    b = prob["b"].cpu().numpy()
    xh = x.cpu().numpy()
    # sampled SA rows, including the first/last bucket of a block
    edges = [0, cfg.m - 1] + ([cfg.m // cfg.s] if cfg.s > 1 else [])
    rows = np.unique(np.concatenate([edges, rng.integers(0, cfg.m, 5)]))
    ref = oracle_mod.sketch_dense_rows(A, 0, t, cfg.m, cfg.s, rows)
    if cfg.s == 1:
        np.testing.assert_array_equal(SA[rows], ref)  # same left-to-right order: bit-exact
    else:
        assert rel_fro(SA[rows], ref) <= 1e-12
    go = oracle_mod.grad_dense(A, b, xh)
    assert (np.abs(g - go) <= grad_bound_chunked(A, b, xh)).all()
    assert rel_fro(H, oracle_mod.gram(SA)) <= 1e-12
    if cfg.constraint == "ols":
        xo = oracle_mod.ols_step(H, g, xh)
    elif cfg.constraint == "lasso":
        xo, _, st = oracle_mod.lasso_step(H, g, xh, prob["lam"])
        assert st == oracle_mod.OK
    else:
        xo, _, st = oracle_mod.l1ball_step(H, g, xh, prob["tau"])
        assert st == oracle_mod.OK
    assert np.linalg.norm(xn.cpu().numpy() - xo) <= 1e-10 * np.linalg.norm(xo - xh) + 1e-14 * np.linalg.norm(xo)
    if name in ("C2", "C4", "C4P"):  # one whole oracle IHS step at full size (seconds)
        kw = {"l1ball": dict(constraint="l1ball", tau=prob["tau"]),
              "lasso": dict(constraint="lasso", tau=prob["lam"])}.get(cfg.constraint, {})
        xh_o, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=cfg.s, T=1, iter0=t, x0=xh, **kw)
        assert oracle_mod.pred_rel_err(xn.cpu().numpy(), xh_o[1], A) <= 1e-9


def test_csr_full_size(P, oracle_mod):
    cfg = synthetic.CONFIGS["C3"]
    prob = synthetic.problem(cfg, DEV)
    rp, cl, vl = prob["csr"]
    n, d, t = cfg.n, cfg.d, 2
    check_hash(P, oracle_mod, cfg, t, [(0, 1 << 18), (n - 4096, 4096)])
    ctx = P.Context(0)
    from paper_1910_14166_b200.dist import CudaOps, ShardedIHS
    spec = P.Spec(m=cfg.m, s=cfg.s)
    S = ShardedIHS(P.Csr(rp, cl, vl, d), prob["b"], spec, ops=CudaOps(ctx), lookahead=False)
    x = torch.from_numpy(np.random.default_rng(1).standard_normal(d) * 0.1).to(DEV)
    xn = torch.empty_like(x)
    S.step(t, x, xn)
    torch.cuda.synchronize()
    assert ctx.status() == P.OK
    rph, clh, vlh, bh, xh = rp.cpu().numpy(), cl.cpu().numpy(), vl.cpu().numpy(), prob["b"].cpu().numpy(), x.cpu().numpy()
    SA_o = oracle_mod.sketch_csr(rph, clh, vlh, d, 0, t, cfg.m, cfg.s)
    assert rel_fro(S.SA.cpu().numpy(), SA_o) <= 1e-12
    go = oracle_mod.grad_csr(rph, clh, vlh, d, bh, xh)
    import scipy.sparse as sp
    M = sp.csr_matrix((vlh, clh, rph), shape=(n, d))
    bound = 1e-12 * (abs(M).T @ np.abs(bh - M @ xh))
    assert (np.abs(S.g.cpu().numpy() - go) <= bound).all()
    H_o = oracle_mod.gram(S.SA.cpu().numpy())
    assert rel_fro(S.H.cpu().numpy(), H_o) <= 1e-12
    xo = oracle_mod.ols_step(S.H.cpu().numpy(), S.g.cpu().numpy(), xh)
    assert oracle_mod.pred_rel_err(xn.cpu().numpy(), xo, csr=(rph, clh, vlh), d=d) <= 1e-9


def test_csr_full_size_lookahead(P, oracle_mod):
    """C3 in the bench's launch configuration: the Gram-only look-ahead (the
    prologue's and the step's Grams on the factor stream, 128 x 128-tile
    stream-K beside the pass), the CG update with H_t, and S^{t+1} A."""
    cfg = synthetic.CONFIGS["C3"]
    prob = synthetic.problem(cfg, DEV)
    rp, cl, vl = prob["csr"]
    n, d, m, t = cfg.n, cfg.d, cfg.m, 4
    ctx = P.Context(0)
    from paper_1910_14166_b200.dist import CudaOps, ShardedIHS
    spec = P.Spec(m=m, s=cfg.s)
    S = ShardedIHS(P.Csr(rp, cl, vl, d), prob["b"], spec, ops=CudaOps(ctx))
    assert S.lookahead and S.la_gram_only
    x = torch.from_numpy(np.random.default_rng(2).standard_normal(d) * 0.1).to(DEV)
    xn = torch.empty_like(x)
    S.prime(t)
    cur = S._la_cur
    S.step(t, x, xn)
    ctx.synchronize()
    assert ctx.status() == P.OK
    nxt = 1 - cur
    rph, clh, vlh, bh, xh = rp.cpu().numpy(), cl.cpu().numpy(), vl.cpu().numpy(), prob["b"].cpu().numpy(), x.cpu().numpy()
    SA_t = S.packs[cur][: m * d].view(m, d).cpu().numpy()
    assert rel_fro(SA_t, oracle_mod.sketch_csr(rph, clh, vlh, d, 0, t, m, cfg.s)) <= 1e-12
    H_t = S.Hinv[cur].cpu().numpy()
    assert rel_fro(H_t, oracle_mod.gram(SA_t)) <= 1e-12
    np.testing.assert_array_equal(H_t, H_t.T)
    g_t = S.packs[nxt][m * d:].cpu().numpy()
    go = oracle_mod.grad_csr(rph, clh, vlh, d, bh, xh)
    import scipy.sparse as sp
    M = sp.csr_matrix((vlh, clh, rph), shape=(n, d))
    assert (np.abs(g_t - go) <= 1e-12 * (abs(M).T @ np.abs(bh - M @ xh))).all()
    xo = oracle_mod.ols_step(H_t, g_t, xh)
    assert oracle_mod.pred_rel_err(xn.cpu().numpy(), xo, csr=(rph, clh, vlh), d=d) <= 1e-9
    SA_1 = S.packs[nxt][: m * d].view(m, d).cpu().numpy()
    assert rel_fro(SA_1, oracle_mod.sketch_csr(rph, clh, vlh, d, 0, t + 1, m, cfg.s)) <= 1e-12
    assert rel_fro(S.Hinv[nxt].cpu().numpy(), oracle_mod.gram(SA_1)) <= 1e-12


@pytest.mark.parametrize("name", ["C4", "C4P"])
def test_solve_pg_default_schedule_full_size(P, oracle_mod, name):
    """ihs_solve_l1ball (C4) / ihs_solve_lasso (C4P) at FULL size through the C
    ABI with trace=NULL, T = 5: the default look-ahead schedule
    (pg_lookahead_loop: the Gram of S^{t+1} A and its step bound on the factor
    stream, the warm-started power chain) against the oracle's IHS at every t."""
    cfg, prob = dense_full(name)
    radius = prob["tau"] if cfg.constraint == "l1ball" else prob["lam"]
    ctx = P.Context(0)
    assert ctx.get_option("lookahead") == -1  # by size: n d = 2^29 >= 2^27, T >= 3 -> look-ahead
    T = 5
    fn = P.ihs_solve_l1ball if cfg.constraint == "l1ball" else P.ihs_solve_lasso
    out = fn(P.Dense(prob["A"]), prob["b"], radius, P.Spec(m=cfg.m), T, ctx=ctx)
    assert ctx.status() == P.OK
    xh = out["x_hist"].cpu().numpy()
    A, b = prob["A"].cpu().numpy(), prob["b"].cpu().numpy()
    xo, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=1, T=T, constraint=cfg.constraint, tau=radius)
    for t in range(1, T + 1):
        assert oracle_mod.pred_rel_err(xh[t], xo[t], A) <= 1e-9, t
