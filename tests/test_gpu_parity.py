"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs, at sizes that span several tiles and a
ragged tail.  Tolerances (BASELINE.json north_star):
  buckets/signs          bit-exact
  SA, H                  relative Frobenius <= 1e-12 (dense CountSketch SA: bit-exact)
  g                      |g - g_ora|_c <= 1e-12 * sum_i |A_ic r_i|   (reading R12)
  iterates               ||A(x - x_ora)|| / ||A x_ora|| <= 1e-9      (reading R8(i))
"""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def P():
    import paper_1910_14166_b200 as P
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    P.lib()
    return P


def rel_fro(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def grad_bound(A, b, x):
    r = b - A @ x
    return 1e-12 * (np.abs(A) * np.abs(r)[:, None]).sum(0) + 1e-300


def dense_case(cfg_name, n, seed_shift=0):
    cfg = synthetic.CONFIGS[cfg_name].scaled(n)
    prob = synthetic.problem(cfg, "cpu")
    return cfg, prob["A"].numpy(), prob["b"].numpy(), prob


# ---------------------------------------------------------------- a1 hash
@pytest.mark.parametrize("m,s,row_begin,count", [(200, 1, 0, 2000), (1024, 1, 3, 100_003), (8192, 4, 0, 65_536),
                                                 (2048, 1, (1 << 21) - 77, 77), (4096, 8, (1 << 25) - 1000, 1000),
                                                 (7, 7, 123, 10), (1, 1, 0, 5)])
def test_hash_bit_exact(P, oracle_mod, m, s, row_begin, count):
    for t in (0, 1, 29):
        bg, sg = P.ihs_hash(P.Spec(m=m, s=s, seed=0), t, row_begin, count)
        bo, so = oracle_mod.hash_rows(0, t, m, s, row_begin, count)
        np.testing.assert_array_equal(bg.cpu().numpy(), bo)
        np.testing.assert_array_equal(sg.cpu().numpy(), so)


# ---------------------------------------------------------------- a2 sketch
@pytest.mark.parametrize("n,d,m", [(2000, 10, 200), (65_536 + 77, 128, 1024), (40_000, 256, 2048), (5000, 96, 64),
                                   (3000, 33, 300), (1000, 300, 128), (100, 17, 500), (1, 5, 3), (0, 8, 16)])
def test_countsketch_dense_bit_exact(P, oracle_mod, n, d, m):
    rng = np.random.default_rng(n + d)
    A = rng.standard_normal((n, d))
    for t in (0, 5):
        SA = P.ihs_sketch(torch.from_numpy(A).to(DEV), P.Spec(m=m, s=1, seed=7), t).cpu().numpy()
        np.testing.assert_array_equal(SA, oracle_mod.sketch_dense(A, 7, t, m, 1))


def test_countsketch_row_offset_shards(P, oracle_mod):
    rng = np.random.default_rng(1)
    A = rng.standard_normal((9000, 40))
    Ad = torch.from_numpy(A).to(DEV)
    spec = P.Spec(m=256, s=1, seed=3)
    full = oracle_mod.sketch_dense(A, 3, 2, 256, 1)
    tot = np.zeros_like(full)
    for k in range(0, 9000, 3000):
        part = P.ihs_sketch(P.Dense(Ad[k:k + 3000], row_offset=k), spec, 2).cpu().numpy()
        np.testing.assert_array_equal(part, oracle_mod.sketch_dense(A[k:k + 3000], 3, 2, 256, 1, row_offset=k))
        tot += part
    assert rel_fro(tot, full) <= 1e-12


@pytest.mark.parametrize("n,d,m,s", [(65_536 + 11, 96, 4096, 8), (20_000, 10, 200, 4), (30_000, 40, 512, 2),
                                     (5000, 7, 4096, 8), (257, 3, 64, 64), (0, 4, 16, 2), (40_001, 97, 4096, 8),
                                     (30_000, 13, 256, 16), (1, 5, 16, 8)])
def test_sjlt_dense(P, oracle_mod, n, d, m, s):
    rng = np.random.default_rng(n + m)
    A = rng.standard_normal((n, d))
    SA = P.ihs_sketch(torch.from_numpy(A).to(DEV), P.Spec(m=m, s=s, seed=0), 4).cpu().numpy()
    ref = oracle_mod.sketch_dense(A, 0, 4, m, s)
    assert rel_fro(SA, ref) <= 1e-12


@pytest.mark.parametrize("n,d,m,s", [(1 << 20, 32, 64, 1), (1 << 20, 24, 64, 4), ((1 << 19) + 333, 90, 90, 1)])
def test_gather_segmented_small_m(P, oracle_mod, n, d, m, s):
    """Few buckets with long row lists: each bucket's rows are split into
    segments summed in order (not bit-exact, R3); sketch and fused gradient."""
    rng = np.random.default_rng(n + d)
    A = rng.standard_normal((n, d))
    b = rng.standard_normal(n)
    x = rng.standard_normal(d) * 0.1
    Ad = torch.from_numpy(A).to(DEV)
    _, SA, g = P.ihs_sketch_grad(Ad, P.Spec(m=m, s=s, seed=0), 2, torch.from_numpy(b).to(DEV),
                                 torch.from_numpy(x).to(DEV))
    ref = oracle_mod.sketch_dense(A, 0, 2, m, s)
    assert rel_fro(SA.cpu().numpy(), ref) <= 1e-12
    assert (np.abs(g.cpu().numpy() - oracle_mod.grad_dense(A, b, x)) <= grad_bound(A, b, x)).all()


def csr_case(n, d, p, seed):
    cfg = synthetic.Config("csr", n, d, "csr", "normal", "sjlt", 64, 4, 1, "ols", density=p, data_seed=seed)
    rp, cl, vl = synthetic.csr_A(cfg, "cpu")
    return rp.numpy(), cl.numpy(), vl.numpy()


@pytest.mark.parametrize("n,d,p,m,s", [(65_536, 1024, 1e-3, 8192, 4), (20_000, 50, 0.05, 500, 1),
                                       (3000, 300, 0.04, 3000, 4), (100, 10, 0.0, 8, 2)])
def test_csr_sketch_and_grad(P, oracle_mod, n, d, p, m, s):
    rp, cl, vl = csr_case(n, d, p, 3)
    A = (torch.from_numpy(rp).to(DEV), torch.from_numpy(cl).to(DEV), torch.from_numpy(vl).to(DEV), d)
    spec = P.Spec(m=m, s=s, seed=0)
    SA = P.ihs_sketch(A, spec, 1).cpu().numpy()
    ref = oracle_mod.sketch_csr(rp, cl, vl, d, 0, 1, m, s)
    assert rel_fro(SA, ref) <= 1e-12
    rng = np.random.default_rng(0)
    b = rng.standard_normal(n)
    x = rng.standard_normal(d)
    g = P.ihs_grad(A, torch.from_numpy(b).to(DEV), torch.from_numpy(x).to(DEV)).cpu().numpy()
    go = oracle_mod.grad_csr(rp, cl, vl, d, b, x)
    import scipy.sparse as sp
    M = sp.csr_matrix((vl, cl, rp), shape=(n, d))
    r = b - M @ x
    bound = 1e-12 * (abs(M).T @ np.abs(r)) + 1e-300
    assert (np.abs(g - go) <= bound).all()
    pack, SA2, g2 = P.ihs_sketch_grad(A, spec, 1, torch.from_numpy(b).to(DEV), torch.from_numpy(x).to(DEV))
    assert rel_fro(SA2.cpu().numpy(), ref) <= 1e-12
    assert (np.abs(g2.cpu().numpy() - go) <= bound).all()


# ---------------------------------------------------------------- a5 gradient
@pytest.mark.parametrize("cfg_name,n", [("C1", 2000), ("C2", 70_001), ("C4", 30_000), ("C5", 50_000)])
def test_grad_dense(P, oracle_mod, cfg_name, n):
    cfg, A, b, _ = dense_case(cfg_name, n)
    x = np.random.default_rng(2).standard_normal(cfg.d)
    g = P.ihs_grad(torch.from_numpy(A).to(DEV), torch.from_numpy(b).to(DEV), torch.from_numpy(x).to(DEV))
    go = oracle_mod.grad_dense(A, b, x)
    assert (np.abs(g.cpu().numpy() - go) <= grad_bound(A, b, x)).all()


@pytest.mark.parametrize("n,d,m", [(70_001, 128, 1024), (30_000, 256, 2048), (2000, 10, 200), (9000, 96, 300),
                                   (500, 1, 7)])
def test_fused_sketch_grad(P, oracle_mod, n, d, m):
    rng = np.random.default_rng(d)
    A = rng.standard_normal((n, d))
    b = rng.standard_normal(n)
    x = rng.standard_normal(d)
    pack, SA, g = P.ihs_sketch_grad(torch.from_numpy(A).to(DEV), P.Spec(m=m), 3, torch.from_numpy(b).to(DEV),
                                    torch.from_numpy(x).to(DEV))
    np.testing.assert_array_equal(SA.cpu().numpy(), oracle_mod.sketch_dense(A, 0, 3, m, 1))
    assert (np.abs(g.cpu().numpy() - oracle_mod.grad_dense(A, b, x)) <= grad_bound(A, b, x)).all()


# ---------------------------------------------------------------- a4 Gram
@pytest.mark.parametrize("m,d", [(200, 10), (1024, 128), (2048, 256), (4096, 96), (777, 130), (64, 1), (3, 70),
                                 (8192, 1024), (3000, 400), (2048, 1000), (513, 2000)])
def test_gram(P, oracle_mod, m, d):
    rng = np.random.default_rng(m * d)
    SA = rng.standard_normal((m, d))
    H = P.ihs_gram(torch.from_numpy(SA).to(DEV)).cpu().numpy()
    Ho = oracle_mod.gram(SA)
    assert rel_fro(H, Ho) <= 1e-12
    np.testing.assert_array_equal(H, H.T)
    H2 = P.ihs_gram(torch.from_numpy(SA).to(DEV), scale=0.5).cpu().numpy()
    assert rel_fro(H2, 0.25 * Ho) <= 1e-12


@pytest.mark.parametrize("m,d", [(8192, 1024), (2048, 1000), (1024, 513), (4096, 640), (1500, 777), (3000, 300)])
def test_gram_lookahead_tiles(P, oracle_mod, m, d):
    """The look-ahead Gram (ihs_gram_lookahead, the factor stream): for d >= 512
    the 128 x 128-tile stream-K kernel (one CTA per SM), ragged last tiles
    (513, 640, 777, 1000) and uneven k-chunks; d = 300 takes the 64-tile plan."""
    rng = np.random.default_rng(m + d)
    SA = torch.from_numpy(rng.standard_normal((m, d))).to(DEV)
    ctx = P.Context(0)
    ctx.set_option("la_gram_tile", 128)  # the default for d > 256 is the 64-tile stream-K (next test)
    H = P.ihs_gram_lookahead(SA, scale=0.5, ctx=ctx)
    ctx.synchronize()
    Ho = oracle_mod.gram(SA.cpu().numpy())
    Hn = H.cpu().numpy()
    assert rel_fro(Hn, 0.25 * Ho) <= 1e-12
    np.testing.assert_array_equal(Hn, Hn.T)


@pytest.mark.parametrize("tile,sms", [(0, 0), (64, 100), (64, 70), (128, 84), (128, 148)])
@pytest.mark.parametrize("m,d", [(2048, 1000), (1500, 777)])
def test_gram_lookahead_tile_and_sm_share(P, oracle_mod, m, d, tile, sms):
    """The wide (d > 256) look-ahead Gram by its options: the default (64 x 64-tile
    stream-K on every SM), and either tile on a share of the SMs ("la_gram_sms":
    the rest are left to the pass it runs beside)."""
    rng = np.random.default_rng(m + d + tile + sms)
    SA = torch.from_numpy(rng.standard_normal((m, d))).to(DEV)
    ctx = P.Context(0)
    if tile:
        ctx.set_option("la_gram_tile", tile)
    if sms:
        ctx.set_option("la_gram_sms", sms)
    H = P.ihs_gram_lookahead(SA, scale=2.0, ctx=ctx)
    ctx.synchronize()
    Hn = H.cpu().numpy()
    assert rel_fro(Hn, 4.0 * oracle_mod.gram(SA.cpu().numpy())) <= 1e-12
    np.testing.assert_array_equal(Hn, Hn.T)


# ---------------------------------------------------------------- a6 inner QP
def spd(rng, d, cond=13.0):
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    return (Q * np.geomspace(1.0, cond, d)) @ Q.T * 50.0


@pytest.mark.parametrize("d", [1, 10, 96, 128, 160, 256])
def test_ols_update(P, oracle_mod, d):
    rng = np.random.default_rng(d)
    H = spd(rng, d)
    g = rng.standard_normal(d)
    x = rng.standard_normal(d)
    xn = P.ihs_ols_update(torch.from_numpy(H).to(DEV), torch.from_numpy(g).to(DEV), torch.from_numpy(x).to(DEV))
    xo = oracle_mod.ols_step(H, g, x)
    u, uo = xn.cpu().numpy() - x, xo - x
    assert np.linalg.norm(u - uo) <= 1e-12 * np.linalg.norm(uo)


@pytest.mark.parametrize("m,d", [(200, 10), (1024, 128), (4096, 96), (40, 5), (777, 100), (64, 1), (2048, 33),
                                 (1000, 200)])
def test_gram_ols_fused(P, oracle_mod, m, d):
    """a4 + a6 in one cluster launch (d <= 128; d = 200 takes the two-call path)."""
    rng = np.random.default_rng(m + d)
    SA = rng.standard_normal((m, d))
    g = rng.standard_normal(d)
    x = rng.standard_normal(d)
    xn, H = P.ihs_gram_ols_update(torch.from_numpy(SA).to(DEV), torch.from_numpy(g).to(DEV),
                                  torch.from_numpy(x).to(DEV), scale=0.5)
    Ho = 0.25 * oracle_mod.gram(SA)
    assert rel_fro(H.cpu().numpy(), Ho) <= 1e-12
    xo = oracle_mod.ols_step(Ho, g, x)
    u, uo = xn.cpu().numpy() - x, xo - x
    assert np.linalg.norm(u - uo) <= 1e-11 * np.linalg.norm(uo)


@pytest.mark.parametrize("m,d", [(200, 10), (1024, 128), (4096, 96), (40, 5), (777, 100), (64, 1), (2048, 33),
                                 (3000, 128)])
def test_ols_factor_apply(P, oracle_mod, m, d):
    """Look-ahead OLS: Hinv = (scale^2 SA^T SA)^{-1} on the factor stream, then
    x + Hinv g, against the oracle's Gram and Cholesky step."""
    rng = np.random.default_rng(3 * m + d)
    SA = rng.standard_normal((m, d))
    g = rng.standard_normal(d)
    x = rng.standard_normal(d)
    ctx = P.Context(0)
    Hinv = P.ihs_ols_factor(torch.from_numpy(SA).to(DEV), scale=0.5, ctx=ctx)
    xn = P.ihs_ols_apply(Hinv, torch.from_numpy(g).to(DEV), torch.from_numpy(x).to(DEV), ctx=ctx)
    assert ctx.status() == P.OK
    Ho = 0.25 * oracle_mod.gram(SA)
    Hi = Hinv.cpu().numpy()
    np.testing.assert_array_equal(Hi, Hi.T)
    kappa = np.linalg.cond(Ho)
    assert rel_fro(Hi @ Ho, np.eye(d)) <= 1e-14 * kappa * d
    xo = oracle_mod.ols_step(Ho, g, x)
    u, uo = xn.cpu().numpy() - x, xo - x
    assert np.linalg.norm(u - uo) <= 1e-14 * kappa * d * np.linalg.norm(uo)


def test_ols_factor_not_spd_and_unsupported(P):
    ctx = P.Context(0)
    SA = torch.zeros((4, 6), dtype=torch.float64, device=DEV)
    SA[:4, :4] = torch.eye(4, dtype=torch.float64, device=DEV)  # rank 4 < d = 6
    Hinv = P.ihs_ols_factor(SA, ctx=ctx)
    x = torch.ones(6, dtype=torch.float64, device=DEV)
    xn = P.ihs_ols_apply(Hinv, x, x, ctx=ctx)
    assert ctx.status() == P.ERR_NOT_SPD
    assert torch.equal(Hinv, torch.zeros_like(Hinv)) and torch.equal(xn, x)
    with pytest.raises(P.IhsError):
        P.ihs_ols_factor(torch.ones((300, 129), dtype=torch.float64, device=DEV), ctx=ctx)


@pytest.mark.parametrize("solo", [True, False])
@pytest.mark.parametrize("cfg_name,n,T,iter0", [("C2", 40_000, 6, 0), ("C1", 2000, 5, 3), ("C5", 30_001, 4, 2)])
def test_sharded_lookahead_matches_oracle(P, oracle_mod, cfg_name, n, T, iter0, solo):
    """The look-ahead schedule (S^{t+1} A formed in pass t, H^{-1} beside the
    next pass) reproduces the oracle's iterates; a step whose t does not follow
    the previous one re-runs the prologue.  solo: one fused call per step
    (ihs_ols_lookahead_step); else sketch_grad / all-reduce hook / factor / apply."""
    from paper_1910_14166_b200.dist import CudaOps, ShardedIHS
    cfg, A, b, prob = dense_case(cfg_name, n)
    ctx = P.Context(0)
    S = ShardedIHS(P.Dense(prob["A"].to(DEV)), prob["b"].to(DEV), P.Spec(m=cfg.m, s=cfg.s), ops=CudaOps(ctx),
                   lookahead=True, allreduce=None if solo else (lambda t: None))
    assert S.lookahead and S._solo == solo
    xh = S.solve(T, iter0=iter0).cpu().numpy()
    xo, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=cfg.s, T=T, iter0=iter0)
    for t in range(1, T + 1):
        assert oracle_mod.pred_rel_err(xh[t], xo[t], A) <= 1e-9, t
    # out-of-order step: iteration iter0 + 2 from x^2 again
    x2 = torch.from_numpy(xo[2]).to(DEV)
    xn = torch.empty_like(x2)
    S.step(iter0 + 2, x2, xn)
    assert oracle_mod.pred_rel_err(xn.cpu().numpy(), xo[3], A) <= 1e-9
    assert ctx.status() == P.OK


@pytest.mark.parametrize("constraint", ["l1ball", "lasso"])
def test_sharded_lookahead_pg_matches_oracle(P, oracle_mod, constraint):
    """l1 ball / LASSO look-ahead: H_{t+1} (ihs_gram_lookahead) beside the update of t."""
    from paper_1910_14166_b200.dist import CudaOps, ShardedIHS
    name = "C4" if constraint == "l1ball" else "C4P"
    cfg, A, b, prob = dense_case(name, 20_000)
    radius = prob["tau"] if constraint == "l1ball" else prob["lam"]
    ctx = P.Context(0)
    S = ShardedIHS(P.Dense(prob["A"].to(DEV)), prob["b"].to(DEV), P.Spec(m=cfg.m), ops=CudaOps(ctx),
                   constraint=constraint, radius=radius, lookahead=True)
    assert S.lookahead
    T = 4
    xh = S.solve(T, iter0=1).cpu().numpy()
    xo, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=1, T=T, iter0=1, constraint=constraint, tau=radius)
    for t in range(1, T + 1):
        assert oracle_mod.pred_rel_err(xh[t], xo[t], A) <= 1e-9, t
    assert ctx.status() == P.OK


@pytest.mark.parametrize("kind", ["csr", "dense_d200"])
def test_sharded_lookahead_gram_only_ols(P, oracle_mod, kind):
    """The Gram-only look-ahead for OLS (CSR, or d > 128: H_{t+1} ahead, the
    conjugate-gradient / Cholesky update with H_t) reproduces the oracle."""
    from paper_1910_14166_b200.dist import CudaOps, ShardedIHS
    rng = np.random.default_rng(9)
    T, m = 4, 2048
    if kind == "csr":
        n, d = 40_000, 200
        rp, cl, vl = csr_case(n, d, 0.05, 4)
        A_dev = P.Csr(torch.from_numpy(rp).to(DEV), torch.from_numpy(cl).to(DEV), torch.from_numpy(vl).to(DEV), d)
        import scipy.sparse as sp
        Ad = sp.csr_matrix((vl, cl, rp), shape=(n, d)).toarray()
        okw = dict(csr=(rp, cl, vl), d=d)
        s = 4
    else:
        n, d = 20_000, 200
        Ad = rng.standard_normal((n, d))
        A_dev = P.Dense(torch.from_numpy(Ad).to(DEV))
        okw = dict(A=Ad)
        s = 1
    b = Ad @ rng.standard_normal(d) + rng.standard_normal(n)
    ctx = P.Context(0)
    S = ShardedIHS(A_dev, torch.from_numpy(b).to(DEV), P.Spec(m=m, s=s), ops=CudaOps(ctx), lookahead=True)
    assert S.lookahead and S.la_gram_only
    xh = S.solve(T, iter0=2).cpu().numpy()
    xo, _ = oracle_mod.ihs_solve(b=b, m=m, s=s, T=T, iter0=2, **okw)
    for t in range(1, T + 1):
        assert oracle_mod.pred_rel_err(xh[t], xo[t], Ad) <= 1e-9, t
    assert ctx.status() == P.OK


def test_gram_lookahead(P, oracle_mod):
    rng = np.random.default_rng(5)
    SA = rng.standard_normal((2048, 256))
    ctx = P.Context(0)
    H = P.ihs_gram_lookahead(torch.from_numpy(SA).to(DEV), scale=0.5, ctx=ctx)
    ctx.synchronize()
    assert rel_fro(H.cpu().numpy(), 0.25 * oracle_mod.gram(SA)) <= 1e-12


def test_ols_update_not_spd(P):
    ctx = P.Context(0)
    H = torch.diag(torch.tensor([1.0, -1.0, 2.0], dtype=torch.float64, device=DEV))
    x = torch.ones(3, dtype=torch.float64, device=DEV)
    xn = P.ihs_ols_update(H, x, x, ctx=ctx)
    assert ctx.status() == P.ERR_NOT_SPD
    assert torch.equal(xn, x)
    assert ctx.status() == P.OK  # status is cleared once read


@pytest.mark.parametrize("d", [2, 50, 300])
def test_ols_update_indefinite_positive_diagonal(P, d):
    """Reading R13: an indefinite H whose diagonal is positive reports NOT_SPD
    and leaves x unchanged (Cholesky pivot for d <= 160, non-positive curvature
    p.Hp on the CG path for d > 160)."""
    rng = np.random.default_rng(d)
    if d == 2:
        H = np.array([[1.0, 2.0], [2.0, 1.0]])
    else:
        Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
        ev = np.geomspace(1.0, 10.0, d)
        ev[:3] = -0.5  # three negative eigenvalues; the diagonal stays positive
        H = (Q * ev) @ Q.T
        H = 0.5 * (H + H.T)
        assert np.linalg.eigvalsh(H).min() < 0 < np.diag(H).min()
    ctx = P.Context(0)
    x = torch.ones(d, dtype=torch.float64, device=DEV)
    g = torch.from_numpy(rng.standard_normal(d)).to(DEV)
    xn = P.ihs_ols_update(torch.from_numpy(H).to(DEV), g, x, ctx=ctx)
    assert ctx.status() == P.ERR_NOT_SPD
    assert torch.equal(xn, x)


@pytest.mark.parametrize("d,tau", [(16, 1.0), (256, 10.0), (64, 1e9), (5, 0.0), (100, 3.0), (200, 5.0)])
def test_l1ball_update(P, oracle_mod, d, tau):
    rng = np.random.default_rng(d)
    H = spd(rng, d)
    g = rng.standard_normal(d) * 10
    x = np.zeros(d)
    inner = torch.zeros(1, dtype=torch.int32, device=DEV)
    xn = P.ihs_l1ball_update(torch.from_numpy(H).to(DEV), torch.from_numpy(g).to(DEV), torch.from_numpy(x).to(DEV),
                             tau, inner=inner).cpu().numpy()
    xo, it, st = oracle_mod.l1ball_step(H, g, x, tau)
    assert st == oracle_mod.OK
    assert np.linalg.norm(xn - xo) <= 1e-10 * max(1.0, np.linalg.norm(xo))
    assert int(inner.item()) >= 1
    assert np.abs(xn).sum() <= tau * (1 + 1e-12) + 1e-300


# ---------------------------------------------------------------- a1-a7 IHS loops
def iterate_parity(A, xg, xo, oracle_mod):
    return max(oracle_mod.pred_rel_err(a, b, A) for a, b in zip(xg[1:], xo[1:]))


def test_ihs_ols_C1_full(P, oracle_mod):
    cfg = synthetic.CONFIGS["C1"]
    prob = synthetic.problem(cfg, "cpu")
    A, b = prob["A"].numpy(), prob["b"].numpy()
    out = P.ihs_solve_ols(prob["A"].to(DEV), prob["b"].to(DEV), P.Spec(m=cfg.m), cfg.T, trace=True)
    xh = out["x_hist"].cpu().numpy()
    xo, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=1, T=cfg.T)
    assert iterate_parity(A, xh, xo, oracle_mod) <= 1e-9
    xopt = oracle_mod.exact_ols(A, b)
    e = [oracle_mod.pred_rel_err(x, xopt, A) for x in xh]
    assert e[-1] < 1e-4 and all(e[t + 1] < e[t] for t in range(4))
    assert len(out["trace"]) == cfg.T and all(r["status"] == 0 for r in out["trace"])


_C3_ORACLE = {}


def c3_scaled_oracle(oracle_mod, prob, cfg, T):
    """The oracle's iterates for the scaled C3 instance (~2.5 minutes of plain C at
    d = 1024): computed once and shared by the two tests that solve that instance
    with the same seed, m, s and T (device buffers / host buffers)."""
    key = (cfg.n, cfg.d, cfg.m, cfg.s, T)
    if key not in _C3_ORACLE:
        rp, cl, vl = (t.numpy() for t in prob["csr"])
        _C3_ORACLE[key] = oracle_mod.ihs_solve(b=prob["b"].numpy(), csr=(rp, cl, vl), d=cfg.d, m=cfg.m, s=cfg.s,
                                               T=T)[0]
    return _C3_ORACLE[key]


@pytest.mark.parametrize("cfg_name,n,T", [("C2", 1 << 16, 8), ("C5", 1 << 15, 6), ("C3", 1 << 16, 4)])
def test_ihs_ols_scaled_configs(P, oracle_mod, cfg_name, n, T):
    cfg = synthetic.CONFIGS[cfg_name].scaled(n)
    prob = synthetic.problem(cfg, "cpu")
    spec = P.Spec(m=cfg.m, s=cfg.s)
    b = prob["b"].numpy()
    if cfg.layout == "dense":
        A = prob["A"].numpy()
        out = P.ihs_solve_ols(prob["A"].to(DEV), prob["b"].to(DEV), spec, T)
        xo, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=cfg.s, T=T)
        par = iterate_parity(A, out["x_hist"].cpu().numpy(), xo, oracle_mod)
    else:
        rp, cl, vl = (t.numpy() for t in prob["csr"])
        Ad = tuple(t.to(DEV) for t in prob["csr"]) + (cfg.d,)
        out = P.ihs_solve_ols(Ad, prob["b"].to(DEV), spec, T)
        xo = c3_scaled_oracle(oracle_mod, prob, cfg, T)
        xg = out["x_hist"].cpu().numpy()
        par = max(oracle_mod.pred_rel_err(a, c, csr=(rp, cl, vl), d=cfg.d) for a, c in zip(xg[1:], xo[1:]))
    assert par <= 1e-9


def test_ihs_l1ball_scaled_C4(P, oracle_mod):
    cfg = synthetic.CONFIGS["C4"].scaled(1 << 15)
    prob = synthetic.problem(cfg, "cpu")
    A, b, tau = prob["A"].numpy(), prob["b"].numpy(), prob["tau"]
    T = 8
    out = P.ihs_solve_l1ball(prob["A"].to(DEV), prob["b"].to(DEV), tau, P.Spec(m=cfg.m), T, trace=True)
    xo, inner = oracle_mod.ihs_solve(A, b, m=cfg.m, s=1, T=T, constraint="l1ball", tau=tau)
    assert iterate_parity(A, out["x_hist"].cpu().numpy(), xo, oracle_mod) <= 1e-9
    its = [r["inner_iters"] for r in out["trace"]]
    assert all(i >= 1 for i in its)


@pytest.mark.parametrize("d,lam", [(16, 0.5), (256, 5.0), (64, 50.0), (5, 0.0), (100, 1e6)])
def test_lasso_update(P, oracle_mod, d, lam):
    """NEXT-2 inner step (reading R23) against the oracle's proximal gradient."""
    rng = np.random.default_rng(d + 1)
    H = spd(rng, d)
    g = rng.standard_normal(d) * 10
    x = rng.standard_normal(d) * 0.1
    inner = torch.zeros(1, dtype=torch.int32, device=DEV)
    xn = P.ihs_lasso_update(torch.from_numpy(H).to(DEV), torch.from_numpy(g).to(DEV), torch.from_numpy(x).to(DEV),
                            lam, inner=inner).cpu().numpy()
    xo, it, st = oracle_mod.lasso_step(H, g, x, lam)
    assert st == oracle_mod.OK
    assert np.linalg.norm(xn - xo) <= 1e-10 * max(1.0, np.linalg.norm(xo))
    assert ((xn == 0) == (xo == 0)).all()  # the same support (exact zeros from the soft threshold)
    assert int(inner.item()) >= 1


def test_lasso_update_unsupported_d(P):
    d = 300
    H = torch.eye(d, dtype=torch.float64, device=DEV)
    v = torch.zeros(d, dtype=torch.float64, device=DEV)
    with pytest.raises(P.IhsError):
        P.ihs_lasso_update(H, v, v, 1.0)


def test_ihs_lasso_scaled_C4P(P, oracle_mod):
    """NEXT-2: the penalised LASSO loop (lambda = 5) against the oracle."""
    cfg = synthetic.CONFIGS["C4P"].scaled(1 << 15)
    prob = synthetic.problem(cfg, "cpu")
    A, b = prob["A"].numpy(), prob["b"].numpy()
    T = 8
    out = P.ihs_solve_lasso(prob["A"].to(DEV), prob["b"].to(DEV), cfg.lam, P.Spec(m=cfg.m), T, trace=True)
    xo, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=1, T=T, constraint="lasso", tau=cfg.lam)
    assert iterate_parity(A, out["x_hist"].cpu().numpy(), xo, oracle_mod) <= 1e-9
    assert all(r["inner_iters"] >= 1 for r in out["trace"])


def test_solve_with_host_buffers(P, oracle_mod):
    """e2e path: host A/b/x, copies inside the call."""
    cfg = synthetic.CONFIGS["C1"]
    prob = synthetic.problem(cfg, "cpu")
    A = prob["A"].pin_memory()
    b = prob["b"].pin_memory()
    out = P.ihs_solve_ols(A, b, P.Spec(m=cfg.m), cfg.T)
    assert out["x"].device.type == "cpu"
    xo, _ = oracle_mod.ihs_solve(A.numpy(), b.numpy(), m=cfg.m, s=1, T=cfg.T)
    assert oracle_mod.pred_rel_err(out["x"].numpy(), xo[-1], A.numpy()) <= 1e-9


def test_solve_csr_with_host_buffers(P, oracle_mod):
    """e2e path for CSR: host row_ptr / cols / values and b, copied inside the
    call; iterates against the oracle (R8), and the solve's look-ahead Gram
    schedule (d > 256) runs on the staged copies."""
    cfg = synthetic.CONFIGS["C3"].scaled(1 << 16)
    prob = synthetic.problem(cfg, "cpu")
    rp, cl, vl = (t.pin_memory() for t in prob["csr"])
    b = prob["b"].pin_memory()
    T = 4
    out = P.ihs_solve_ols(P.Csr(rp, cl, vl, cfg.d), b, P.Spec(m=cfg.m, s=cfg.s), T)
    assert out["x"].device.type == "cpu"
    csr = (rp.numpy(), cl.numpy(), vl.numpy())
    xo = c3_scaled_oracle(oracle_mod, prob, cfg, T)
    xg = out["x_hist"].numpy()
    par = max(oracle_mod.pred_rel_err(a, c, csr=csr, d=cfg.d) for a, c in zip(xg[1:], xo[1:]))
    assert par <= 1e-9


def test_pred_err2(P, oracle_mod):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((50_000, 128))
    X = rng.standard_normal((4, 128))
    xr = rng.standard_normal(128)
    e2, r2 = P.ihs_pred_err2(torch.from_numpy(A).to(DEV), torch.from_numpy(X).to(DEV), torch.from_numpy(xr).to(DEV))
    e = np.sqrt(e2.cpu().numpy() / r2.item())
    ref = np.array([oracle_mod.pred_rel_err(x, xr, A) for x in X])
    np.testing.assert_allclose(e, ref, rtol=1e-11)


def test_invalid_arguments(P):
    A = torch.zeros((10, 4), dtype=torch.float64, device=DEV)
    with pytest.raises(P.IhsError) as e:
        P.ihs_sketch(A, P.Spec(m=10, s=3, family=P.SJLT), 0)
    assert e.value.status == P.ERR_DIMENSION_MISMATCH
    with pytest.raises(P.IhsError):
        P.ihs_sketch(A, P.Spec(m=10, s=2, family=P.COUNTSKETCH), 0)
    with pytest.raises(P.IhsError):
        P.ihs_sketch(A, P.Spec(m=0), 0)


def test_deterministic_rerun(P):
    rng = np.random.default_rng(9)
    A = torch.from_numpy(rng.standard_normal((100_000, 96))).to(DEV)
    a = P.ihs_sketch(A, P.Spec(m=4096, s=8), 2)
    b = P.ihs_sketch(A, P.Spec(m=4096, s=8), 2)
    assert torch.equal(a, b)
    H1 = P.ihs_gram(a)
    H2 = P.ihs_gram(b)
    assert torch.equal(H1, H2)


# ---------------------------------------------------------------- round 2: the C-ABI defaults and the large-d OLS
def test_ctx_options(P):
    ctx = P.Context(0)
    for name, vals in {"lookahead": (-1, 0, 1), "sjlt_onepass": (0, 1), "ols_large": (0, 1, 2),
                       "fuse_max_d": (0, 64, 128), "pg_warm": (0, 1), "prefetch": (0, 1)}.items():
        for v in vals:
            ctx.set_option(name, v)
            assert ctx.get_option(name) == v
    with pytest.raises(P.IhsError):
        ctx.set_option("no_such_option", 1)
    with pytest.raises(P.IhsError):
        ctx.set_option("ols_large", 3)


@pytest.mark.parametrize("constraint", ["l1ball", "lasso"])
def test_solve_pg_lookahead_c_abi_scaled(P, oracle_mod, constraint):
    """ihs_solve_l1ball / ihs_solve_lasso through the C ABI with trace=NULL and
    the look-ahead forced (option lookahead = 1): pg_lookahead_loop (the
    default schedule at full C4 / C4P), its warm-started power chain and the
    look-ahead step bound, against the oracle at every t (reading R8)."""
    name = "C4" if constraint == "l1ball" else "C4P"
    cfg = synthetic.CONFIGS[name].scaled(1 << 15)
    prob = synthetic.problem(cfg, "cpu")
    A, b = prob["A"].numpy(), prob["b"].numpy()
    radius = prob["tau"] if constraint == "l1ball" else cfg.lam
    T = 6
    for la in (1, 0):
        ctx = P.Context(0)
        ctx.set_option("lookahead", la)
        fn = P.ihs_solve_l1ball if constraint == "l1ball" else P.ihs_solve_lasso
        out = fn(prob["A"].to(DEV), prob["b"].to(DEV), radius, P.Spec(m=cfg.m), T, iter0=1, ctx=ctx)
        assert ctx.status() == P.OK
        xo, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=1, T=T, iter0=1, constraint=constraint, tau=radius)
        assert iterate_parity(A, out["x_hist"].cpu().numpy(), xo, oracle_mod) <= 1e-9, la


def spd_kappa(rng, d, kappa):
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    H = (Q * np.geomspace(1.0, kappa, d)) @ Q.T
    return 0.5 * (H + H.T)


@pytest.mark.parametrize("d", [256, 1024])
@pytest.mark.parametrize("kappa", [1e4, 1e8])
def test_ols_large_high_kappa(P, oracle_mod, d, kappa):
    """d > 160 OLS step at high condition number (reading R22) against the
    oracle's Cholesky step, for the default (CG, then the Cholesky in the same
    launch when CG does not finish) and the Cholesky-only option.  Bar: the
    forward error of a backward-stable solve, 1e-15 kappa d relative."""
    rng = np.random.default_rng(d + int(np.log10(kappa)))
    H = spd_kappa(rng, d, kappa)
    g = rng.standard_normal(d)
    x = rng.standard_normal(d)
    xo = oracle_mod.ols_step(H, g, x)
    uo = xo - x
    for mode in (1, 2):
        ctx = P.Context(0)
        ctx.set_option("ols_large", mode)
        xn = P.ihs_ols_update(torch.from_numpy(H).to(DEV), torch.from_numpy(g).to(DEV), torch.from_numpy(x).to(DEV),
                              ctx=ctx)
        assert ctx.status() == P.OK, mode
        u = xn.cpu().numpy() - x
        assert np.linalg.norm(u - uo) <= max(1e-12, 1e-15 * kappa * d) * np.linalg.norm(uo), mode


def test_ols_large_cg_cap(P, oracle_mod):
    """The CG cap min(2000, 4d): CG alone (option ols_large = 0) on a kappa = 1e8
    matrix stops there with IHS_ERR_NOT_CONVERGED and x + (its last u); the
    default continues with the Cholesky and returns the oracle's step."""
    d = 256
    rng = np.random.default_rng(11)
    H = spd_kappa(rng, d, 1e8)
    g = rng.standard_normal(d)
    x = np.zeros(d)
    Hd, gd, xd = (torch.from_numpy(v).to(DEV) for v in (H, g, x))
    ctx = P.Context(0)
    ctx.set_option("ols_large", 0)
    xn = P.ihs_ols_update(Hd, gd, xd, ctx=ctx)
    assert ctx.status() == P.ERR_NOT_CONVERGED
    u = xn.cpu().numpy()
    assert np.all(np.isfinite(u)) and 0.5 * u @ H @ u - g @ u < 0.0  # a partial solve: CG lowers the energy
    ctx.set_option("ols_large", 1)
    xn = P.ihs_ols_update(Hd, gd, xd, ctx=ctx)
    assert ctx.status() == P.OK
    uo = oracle_mod.ols_step(H, g, x)
    assert np.linalg.norm(xn.cpu().numpy() - uo) <= 1e-15 * 1e8 * d * np.linalg.norm(uo)


@pytest.mark.parametrize("d", [300, 1024])
def test_ols_large_indefinite_g_in_positive_space(P, oracle_mod, d):
    """An indefinite H with a positive diagonal and g inside the positive
    eigenspace, where CG can finish without meeting p.Hp <= 0 (reading R22: CG
    certifies definiteness only on the Krylov space it explores).  The
    Cholesky-only option reports IHS_ERR_NOT_SPD and leaves x, as the oracle
    does; the default returns either that or a solution of H u = g."""
    rng = np.random.default_rng(d)
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    ev = np.geomspace(1.0, 10.0, d)
    ev[:3] = -0.5
    H = (Q * ev) @ Q.T
    H = 0.5 * (H + H.T)
    assert np.diag(H).min() > 0
    g = Q[:, 3:] @ rng.standard_normal(d - 3)
    x = rng.standard_normal(d)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.ols_step(H, g, x)
    Hd, gd, xd = (torch.from_numpy(v).to(DEV) for v in (H, g, x))
    ctx = P.Context(0)
    ctx.set_option("ols_large", 2)
    xn = P.ihs_ols_update(Hd, gd, xd, ctx=ctx)
    assert ctx.status() == P.ERR_NOT_SPD
    assert torch.equal(xn, xd)
    ctx.set_option("ols_large", 1)
    xn = P.ihs_ols_update(Hd, gd, xd, ctx=ctx)
    st = ctx.status()
    if st == P.OK:
        u = xn.cpu().numpy() - x
        assert np.linalg.norm(H @ u - g) <= 1e-12 * np.linalg.norm(g)
    else:
        assert st == P.ERR_NOT_SPD and torch.equal(xn, xd)


def test_reduce_argument_single_rank(P):
    """ihs_sketch / ihs_grad / ihs_sketch_grad with reduce = 1 on one rank: the
    all-reduce is a no-op, results equal reduce = 0 (ihs.h)."""
    rng = np.random.default_rng(3)
    A = torch.from_numpy(rng.standard_normal((20_000, 64))).to(DEV)
    b = torch.from_numpy(rng.standard_normal(20_000)).to(DEV)
    x = torch.from_numpy(rng.standard_normal(64)).to(DEV)
    for spec in (P.Spec(m=512), P.Spec(m=512, s=4)):
        assert torch.equal(P.ihs_sketch(A, spec, 2, reduce=True), P.ihs_sketch(A, spec, 2))
        p1, _, _ = P.ihs_sketch_grad(A, spec, 2, b, x, reduce=True)
        p0, _, _ = P.ihs_sketch_grad(A, spec, 2, b, x)
        assert torch.equal(p1, p0)
    assert torch.equal(P.ihs_grad(A, b, x, reduce=True), P.ihs_grad(A, b, x))


@pytest.mark.parametrize("n,d,m,s", [(70_001, 98, 4096, 8), (9_999, 10, 256, 2), (4_097, 6, 2048, 4),
                                     (30_001, 34, 1536, 8), (5_000, 18, 384, 4), (12_345, 66, 1152, 6),
                                     (3_000, 12, 3 * 170, 3), (1_025, 2, 16, 8), (2_049, 100, 4096, 8)])
def test_sjlt_onepass_vs_passes(P, oracle_mod, n, d, m, s):
    """The one-read SJLT sketch against the s sorted passes (bit-identical to
    the oracle) and the oracle: ragged last chunks, d not a multiple of 4, the
    M = m / s range 2 .. 512, s in 2 .. 8."""
    rng = np.random.default_rng(n + d)
    A = rng.standard_normal((n, d))
    Ad = torch.from_numpy(A).to(DEV)
    ref = oracle_mod.sketch_dense(A, 0, 3, m, s)
    outs = {}
    for opt in (0, 1):
        ctx = P.Context(0)
        ctx.set_option("sjlt_onepass", opt)
        outs[opt] = P.ihs_sketch(Ad, P.Spec(m=m, s=s), 3, ctx=ctx).cpu().numpy()
        assert ctx.status() == P.OK
    np.testing.assert_array_equal(outs[0], ref)
    assert rel_fro(outs[1], ref) <= 1e-12
    # sketch + gradient, the gradient in its own pass (1) or co-resident beside the sketch pass (2)
    b = rng.standard_normal(n)
    x = rng.standard_normal(d)
    bd, xd = torch.from_numpy(b).to(DEV), torch.from_numpy(x).to(DEV)
    go = oracle_mod.grad_dense(A, b, x)
    for opt in (1, 2):
        ctx = P.Context(0)
        ctx.set_option("sjlt_onepass", opt)
        _, SA, g = P.ihs_sketch_grad(Ad, P.Spec(m=m, s=s), 3, bd, xd, ctx=ctx)
        assert ctx.status() == P.OK
        assert rel_fro(SA.cpu().numpy(), ref) <= 1e-12, opt
        assert (np.abs(g.cpu().numpy() - go) <= grad_bound(A, b, x)).all(), opt


@pytest.mark.parametrize("n,d,m,s", [(2000, 10, 200, 1), (3001, 32, 512, 4), (500, 1, 7, 1), (40, 5, 64, 8)])
def test_small_step_solve(P, oracle_mod, n, d, m, s):
    """ihs_solve_ols on a small dense problem: one launch per iteration
    (small_step.cu) against the oracle and against the general path."""
    rng = np.random.default_rng(n + d)
    A = rng.standard_normal((n, d))
    b = A @ rng.standard_normal(d) + rng.standard_normal(n)
    T = 6
    xo, _ = oracle_mod.ihs_solve(A, b, m=m, s=s, T=T, iter0=2)
    outs = []
    for small in (1, 0):
        ctx = P.Context(0)
        ctx.set_option("small_step", small)
        out = P.ihs_solve_ols(torch.from_numpy(A).to(DEV), torch.from_numpy(b).to(DEV), P.Spec(m=m, s=s), T, iter0=2,
                              ctx=ctx)
        assert ctx.status() == P.OK
        xh = out["x_hist"].cpu().numpy()
        assert iterate_parity(A, xh, xo, oracle_mod) <= 1e-9, small
        outs.append(xh)
    assert np.abs(outs[0] - outs[1]).max() <= 1e-10 * max(1.0, np.abs(outs[1]).max())


@pytest.mark.parametrize("n,d,m,s", [(2000, 10, 200, 1), (40, 5, 64, 8), (500, 32, 64, 4), (500, 1, 7, 1)])
def test_small_step_intermediates(P, oracle_mod, n, d, m, s):
    """ihs_small_step's SA (bit-exact for CountSketch), g, H and step against the oracle."""
    rng = np.random.default_rng(n * d)
    A = rng.standard_normal((n, d))
    b = rng.standard_normal(n)
    x = rng.standard_normal(d) * 0.1
    xn, SA, g, H = P.ihs_small_step(torch.from_numpy(A).to(DEV), torch.from_numpy(b).to(DEV), P.Spec(m=m, s=s), 3,
                                    torch.from_numpy(x).to(DEV), intermediates=True)
    SAo = oracle_mod.sketch_dense(A, 0, 3, m, s)
    assert rel_fro(SA.cpu().numpy(), SAo) <= 1e-12
    if s == 1:
        np.testing.assert_array_equal(SA.cpu().numpy(), SAo)
    assert (np.abs(g.cpu().numpy() - oracle_mod.grad_dense(A, b, x)) <= grad_bound(A, b, x)).all()
    Ho = oracle_mod.gram(SAo)
    assert rel_fro(H.cpu().numpy(), Ho) <= 1e-12
    xo = oracle_mod.ols_step(Ho, oracle_mod.grad_dense(A, b, x), x)
    assert np.linalg.norm(xn.cpu().numpy() - xo) <= 1e-11 * np.linalg.norm(xo - x)
