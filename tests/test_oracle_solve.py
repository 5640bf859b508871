"""Pins for the oracle's inner QP (a6) and the IHS loop / exact reference (a7, O10).

Against: numpy/LAPACK (cholesky, solve, lstsq, eigvalsh), brute-force
enumeration of the l1-ball projection, KKT certificates, special cases with
closed forms (H = I, noiseless design, inactive constraint), and Theorem 1's
geometric decay with SPEC.md:469's acceptance rule.
"""
import itertools

import numpy as np
import pytest


def spd(rng, d, cond=10.0):
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    ev = np.geomspace(1.0, cond, d)
    return (Q * ev) @ Q.T


def test_cholesky_vs_lapack(oracle_mod):
    rng = np.random.default_rng(0)
    H = spd(rng, 12)
    L = oracle_mod.cholesky(H)
    np.testing.assert_allclose(L, np.linalg.cholesky(H), rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(L @ L.T, H, atol=1e-13)
    g = rng.standard_normal(12)
    np.testing.assert_allclose(oracle_mod.chol_solve(L, g), np.linalg.solve(H, g), rtol=1e-11)


def test_cholesky_rejects_indefinite(oracle_mod):
    H = np.diag([1.0, -1.0, 2.0])
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.cholesky(H)
    assert e.value.status == oracle_mod.ERR_NOT_SPD
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.ols_step(np.zeros((2, 2)), np.ones(2), np.zeros(2))


def test_identity_hessian_step(oracle_mod, golden):
    ex = golden("spec_worked_examples.json")["identity_hessian"]
    g = np.array(ex["g"])
    np.testing.assert_array_equal(oracle_mod.ols_step(np.eye(3), g, np.zeros(3)), ex["x_next"])


def test_exact_hessian_step_is_least_squares(oracle_mod):
    """One Newton step with the exact Hessian A^T A from any x gives x_OPT
    (Eq. (2) with S^T S = I); composed from the oracle's own gram/grad."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((300, 8))
    b = rng.standard_normal(300)
    x0 = rng.standard_normal(8)
    H = oracle_mod.gram(A)  # "SA" := A gives A^T A
    x1 = oracle_mod.ols_step(H, oracle_mod.grad_dense(A, b, x0), x0)
    np.testing.assert_allclose(x1, np.linalg.lstsq(A, b, rcond=None)[0], rtol=1e-10, atol=1e-12)


def test_exact_ols_vs_lstsq_and_noiseless(oracle_mod):
    rng = np.random.default_rng(2)
    A = rng.standard_normal((2000, 10))
    xs = rng.standard_normal(10)
    b = A @ xs + rng.standard_normal(2000)
    x = oracle_mod.exact_ols(A, b)
    ref = np.linalg.lstsq(A, b, rcond=None)[0]
    assert oracle_mod.pred_rel_err(x, ref, A) < 1e-13
    # noiseless design => x_OPT = x*
    x = oracle_mod.exact_ols(A, A @ xs)
    np.testing.assert_allclose(x, xs, rtol=1e-12, atol=1e-13)


def test_project_l1_hand_cases(oracle_mod, golden):
    ex = golden("spec_worked_examples.json")["project_l1"]
    np.testing.assert_array_equal(oracle_mod.project_l1(ex["v"], ex["tau"]), ex["out"])
    v = np.array([0.1, -0.2, 0.3])
    np.testing.assert_array_equal(oracle_mod.project_l1(v, 1.0), v)  # interior: unchanged
    np.testing.assert_array_equal(oracle_mod.project_l1(v, 0.0), np.zeros(3))


def brute_project_l1(v, tau):
    """min ||x - v|| s.t. ||x||_1 <= tau by enumerating every face of the ball:
    support S and signs sigma, x_S = v_S - lam sigma_S with sum sigma_S x_S = tau."""
    d = v.size
    best, bx = np.inf, None
    if np.abs(v).sum() <= tau:
        return v.copy()
    for pat in itertools.product((-1, 0, 1), repeat=d):
        sg = np.array(pat, float)
        S = sg != 0
        if not S.any():
            cand = np.zeros(d)
        else:
            lam = (sg[S] @ v[S] - tau) / S.sum()
            cand = np.zeros(d)
            cand[S] = v[S] - lam * sg[S]
            if (np.sign(cand[S]) * sg[S] < -1e-12).any():
                continue
        if np.abs(cand).sum() > tau + 1e-12:
            continue
        dist = np.linalg.norm(cand - v)
        if dist < best:
            best, bx = dist, cand
    return bx


@pytest.mark.parametrize("seed", range(12))
def test_project_l1_brute_force(oracle_mod, seed):
    rng = np.random.default_rng(seed)
    d = 1 + seed % 5
    v = rng.standard_normal(d) * 2
    tau = float(rng.uniform(0.1, 2.0))
    np.testing.assert_allclose(oracle_mod.project_l1(v, tau), brute_project_l1(v, tau), atol=1e-12)


def test_power_lmax(oracle_mod):
    rng = np.random.default_rng(3)
    H = spd(rng, 20, cond=13)
    assert abs(oracle_mod.power_lmax(H, 500) - np.linalg.eigvalsh(H).max()) < 1e-9


def kkt_residual(H, g, x, xt, tau):
    """KKT of min 1/2 (y-xt)^T H (y-xt) - g^T (y-xt) s.t. ||y||_1 <= tau:
    -grad = theta sign(y) on supp(y), |grad_j| <= theta off it, theta >= 0,
    theta (||y||_1 - tau) = 0."""
    grad = H @ (x - xt) - g
    supp = np.abs(x) > 1e-12
    if np.abs(x).sum() < tau - 1e-9:
        return np.abs(grad).max(), 0.0
    theta = np.mean(-grad[supp] * np.sign(x[supp]))
    r = np.abs(-grad[supp] - theta * np.sign(x[supp])).max()
    r = max(r, max(0.0, (np.abs(grad[~supp]) - theta).max() if (~supp).any() else 0.0))
    return r, theta


def test_l1ball_step_kkt_and_inactive_case(oracle_mod):
    rng = np.random.default_rng(4)
    d = 16
    H = spd(rng, d, cond=13)
    xt = rng.standard_normal(d) * 0.1
    g = rng.standard_normal(d)
    tau = 1.0
    x, it, st = oracle_mod.l1ball_step(H, g, xt, tau)
    assert st == oracle_mod.OK and it > 1
    assert abs(np.abs(x).sum() - tau) < 1e-12
    r, theta = kkt_residual(H, g, x, xt, tau)
    assert theta > 0 and r < 1e-10 * max(1.0, theta)
    # tau >= ||Newton step||_1: the constraint is inactive and PG returns x + H^{-1} g
    xn = xt + np.linalg.solve(H, g)
    x2, _, st = oracle_mod.l1ball_step(H, g, xt, np.abs(xn).sum() * 1.5)
    np.testing.assert_allclose(x2, xn, atol=1e-11)
    # cap reached -> NOT_CONVERGED with the last iterate
    _, it3, st3 = oracle_mod.l1ball_step(H, g, xt, tau, max_inner=3)
    assert st3 == oracle_mod.ERR_NOT_CONVERGED and it3 == 3


def test_exact_l1ball(oracle_mod):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((400, 12))
    xs = np.zeros(12)
    xs[[1, 4, 7]] = [1.0, -1.0, 1.0]
    b = A @ xs + 0.5 * rng.standard_normal(400)
    tau = 3.0
    x = oracle_mod.exact_l1ball(A, b, tau)
    r, theta = kkt_residual(A.T @ A, A.T @ b, x, np.zeros(12), tau)
    assert r < 1e-9 * max(1.0, theta)
    # noiseless with tau = ||x*||_1 => x_OPT = x*
    x = oracle_mod.exact_l1ball(A, A @ xs, tau)
    np.testing.assert_allclose(x, xs, atol=1e-10)
    # inactive constraint => least squares
    xl = np.linalg.lstsq(A, b, rcond=None)[0]
    x = oracle_mod.exact_l1ball(A, b, np.abs(xl).sum() + 1.0)
    np.testing.assert_allclose(x, xl, atol=1e-10)


def test_ihs_geometric_decay_theorem1(oracle_mod):
    """Theorem 1: e_t <= eps0^t with eps0 = 1/2 for every recorded t
    in >= 8 of 10 seeds, CountSketch m = 10d on 2048 x 16 Gaussian design."""
    good = 0
    for seed in range(10):
        rng = np.random.default_rng(100 + seed)
        A = rng.standard_normal((2048, 16))
        b = A @ rng.standard_normal(16) + rng.standard_normal(2048)
        xo = oracle_mod.exact_ols(A, b)
        xh, _ = oracle_mod.ihs_solve(A, b, seed=seed, m=160, s=1, T=12)
        e = np.array([oracle_mod.pred_rel_err(x, xo, A) for x in xh])
        assert e[0] == pytest.approx(1.0)
        floor = 1e-13
        good += all(e[t] <= max(0.5 ** t, floor) for t in range(len(e)))
    assert good >= 8


def test_ihs_fixed_point_and_machine_precision(oracle_mod):
    """x^t = x_OPT is a fixed point of Eq. (2); IHS reaches ~1e-10 error
    within 40 steps (SPEC.md ihs_solve example)."""
    rng = np.random.default_rng(7)
    A = rng.standard_normal((3000, 10))
    b = A @ rng.standard_normal(10) + rng.standard_normal(3000)
    xo = oracle_mod.exact_ols(A, b)
    xh, _ = oracle_mod.ihs_solve(A, b, m=200, s=1, T=3, x0=xo)
    assert max(oracle_mod.pred_rel_err(x, xo, A) for x in xh) < 1e-13
    xh, _ = oracle_mod.ihs_solve(A, b, m=200, s=4, T=40)
    assert oracle_mod.pred_rel_err(xh[-1], xo, A) < 1e-10


def test_ihs_l1ball_converges(oracle_mod):
    rng = np.random.default_rng(8)
    A = rng.standard_normal((3000, 20)) / np.sqrt(rng.chisquare(3, (3000, 20)) / 3)  # Student-t(3)
    xs = np.zeros(20)
    xs[rng.choice(20, 4, replace=False)] = rng.choice([-1.0, 1.0], 4)
    b = A @ xs + rng.standard_normal(3000)
    tau = 4.0
    xo = oracle_mod.exact_l1ball(A, b, tau)
    xh, inner = oracle_mod.ihs_solve(A, b, m=200, s=1, T=25, constraint="l1ball", tau=tau)
    assert (inner > 0).all()
    assert oracle_mod.pred_rel_err(xh[-1], xo, A) < 1e-9
    assert (np.abs(xh[1:]).sum(1) <= tau * (1 + 1e-12)).all()


def test_ihs_csr_matches_dense(oracle_mod):
    import scipy.sparse as sp
    rng = np.random.default_rng(9)
    M = sp.random(4000, 12, density=0.2, format="csr", random_state=10, data_rvs=rng.standard_normal)
    M.sort_indices()
    b = M @ rng.standard_normal(12) + rng.standard_normal(4000)
    csr = (M.indptr.astype(np.int64), M.indices, M.data)
    xa, _ = oracle_mod.ihs_solve(b=b, csr=csr, d=12, m=128, s=4, T=6)
    xb, _ = oracle_mod.ihs_solve(M.toarray(), b, m=128, s=4, T=6)
    np.testing.assert_allclose(xa, xb, rtol=1e-11, atol=1e-12)
    xo = oracle_mod.exact_ols(b=b, csr=csr, d=12)
    np.testing.assert_allclose(xo, np.linalg.lstsq(M.toarray(), b, rcond=None)[0], rtol=1e-10)


# ---------------------------------------------------------------- NEXT-2: penalised LASSO
def lasso_kkt(H, g, y, xt, lam):
    """Optimality of min 1/2 (y-xt)^T H (y-xt) - g^T (y-xt) + lam ||y||_1:
    r = H(y - xt) - g must equal -lam sign(y_i) where y_i != 0 and satisfy
    |r_i| <= lam where y_i = 0.  Returns the largest violation."""
    r = H @ (y - xt) - g
    on = y != 0
    v_on = np.abs(r[on] + lam * np.sign(y[on])).max(initial=0.0)
    v_off = np.maximum(np.abs(r[~on]) - lam, 0.0).max(initial=0.0)
    return max(v_on, v_off)


def test_lasso_spec_worked_example(oracle_mod):
    """A = I, b = (3, -1), lambda = 1 -> x = (2, 0) (soft threshold)."""
    x = oracle_mod.exact_lasso(np.eye(2), np.array([3.0, -1.0]), 1.0)
    np.testing.assert_allclose(x, [2.0, 0.0], atol=1e-12)


def test_lasso_step_identity_is_soft_threshold(oracle_mod):
    """H = I: the step's minimiser is the l1 prox S_lam(x + g) in closed form
    (SPEC.md:237), a formula independent of the iteration."""
    rng = np.random.default_rng(3)
    d = 40
    g, xt = rng.standard_normal(d) * 3, rng.standard_normal(d)
    lam = 1.3
    y, _, st = oracle_mod.lasso_step(np.eye(d), g, xt, lam)
    v = xt + g
    ref = np.sign(v) * np.maximum(np.abs(v) - lam, 0.0)
    assert st == oracle_mod.OK
    np.testing.assert_allclose(y, ref, atol=1e-13)


def test_lasso_step_kkt_and_special_cases(oracle_mod):
    rng = np.random.default_rng(4)
    d = 30
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    H = (Q * np.geomspace(1.0, 20.0, d)) @ Q.T
    g, xt = rng.standard_normal(d) * 5, rng.standard_normal(d) * 0.1
    lam = 2.0
    y, it, st = oracle_mod.lasso_step(H, g, xt, lam)
    assert st == oracle_mod.OK and it > 1
    assert lasso_kkt(H, g, y, xt, lam) <= 1e-9 * max(1.0, np.abs(g).max())
    assert (y == 0).sum() > 0  # the penalty is active
    # lambda = 0: the Newton step of OLS
    y0, _, st0 = oracle_mod.lasso_step(H, g, xt, 0.0)
    np.testing.assert_allclose(y0, xt + np.linalg.solve(H, g), rtol=1e-9, atol=1e-11)
    # lambda >= ||H xt + g||_inf: y = 0 satisfies the optimality conditions
    big = 1.01 * np.abs(H @ xt + g).max()
    yb, _, stb = oracle_mod.lasso_step(H, g, xt, big)
    assert stb == oracle_mod.OK and np.abs(yb).max() == 0.0
    # the cap reports NOT_CONVERGED with the last iterate
    _, it3, st3 = oracle_mod.lasso_step(H, g, xt, lam, max_inner=3)
    assert st3 == oracle_mod.ERR_NOT_CONVERGED and it3 == 3


def test_exact_lasso_kkt(oracle_mod):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((300, 12))
    b = A @ np.r_[np.ones(3), np.zeros(9)] + 0.5 * rng.standard_normal(300)
    lam = 5.0  # the paper's value
    x = oracle_mod.exact_lasso(A, b, lam)
    G, c = A.T @ A, A.T @ b
    assert lasso_kkt(G, c, x, np.zeros(12), lam) <= 1e-9 * np.abs(c).max()


def test_ihs_lasso_converges(oracle_mod):
    """Theorem 1 on the penalised form."""
    rng = np.random.default_rng(6)
    n, d = 2048, 16
    A = rng.standard_normal((n, d))
    b = A @ rng.standard_normal(d) + rng.standard_normal(n)
    xo = oracle_mod.exact_lasso(A, b, 5.0)
    xh, inner = oracle_mod.ihs_solve(A, b, m=160, s=1, T=30, constraint="lasso", tau=5.0)
    errs = [oracle_mod.pred_rel_err(x, xo, A) for x in xh]
    assert errs[-1] <= 1e-10
    assert sum(e <= 0.5 ** t for t, e in enumerate(errs) if e > 1e-12) >= 0.8 * sum(e > 1e-12 for e in errs)
