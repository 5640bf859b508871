"""Pins for the oracle's sketch (a2), gradient (a5), Gram (a4) and error norm (a7).

Each check compares against something other than the oracle itself: the SPEC's
worked example, an explicitly materialised dense S multiplied by numpy (brute
force), the paper's appendix lemmas (exact and Monte Carlo), numpy / scipy
library routines, and finite differences.
"""
import numpy as np
import pytest
import scipy.sparse as sp


def dense_S(oracle_mod, seed, t, m, s, n, row_offset=0):
    """Materialise S (m x n) from the oracle's exported (h, sigma): entries +-1/sqrt(s)."""
    b, g = oracle_mod.hash_rows(seed, t, m, s, row_offset, n)
    S = np.zeros((m, n))
    for j in range(s):
        S[b[:, j], np.arange(n)] += g[:, j] / np.sqrt(s)
    return S


def test_spec_worked_example(oracle_mod, golden):
    ex = golden("spec_worked_examples.json")["countsketch_identity"]
    SA = oracle_mod.sketch_dense_hs(np.array(ex["A"], float), ex["m"], ex["bucket"], ex["sign"])
    np.testing.assert_array_equal(SA, np.array(ex["SA"], float))


def test_spec_matvec_example(oracle_mod, golden):
    ex = golden("spec_worked_examples.json")["matvec"]
    np.testing.assert_array_equal(oracle_mod.matvec_dense(np.array(ex["A"], float), ex["x"]), ex["y"])


@pytest.mark.parametrize("m,s,n,d", [(200, 1, 2000, 10), (64, 4, 777, 7), (96, 8, 1500, 5), (50, 1, 30, 3)])
def test_sketch_equals_dense_S_times_A(oracle_mod, m, s, n, d):
    """SA == densify(S) @ A (SPEC.md:143 brute force); also the column structure of S:
    exactly s nonzeros +-1/sqrt(s), one per block."""
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((n, d))
    S = dense_S(oracle_mod, 3, 1, m, s, n)
    assert ((S != 0).sum(0) == s).all()
    assert np.allclose(np.abs(S[S != 0]), 1 / np.sqrt(s))
    np.testing.assert_allclose(np.linalg.norm(S, axis=0), 1.0, rtol=1e-15)
    SA = oracle_mod.sketch_dense(A, 3, 1, m, s)
    ref = S @ A
    assert np.linalg.norm(SA - ref) <= 1e-14 * np.linalg.norm(ref)


def test_sketch_is_sum_of_shards(oracle_mod):
    """Linearity + global-row hashing: sum_k S_k A_k == S A (row sharding)."""
    rng = np.random.default_rng(0)
    A = rng.standard_normal((1000, 6))
    full = oracle_mod.sketch_dense(A, 0, 4, 128, 4)
    parts = sum(oracle_mod.sketch_dense(A[k:k + 250], 0, 4, 128, 4, row_offset=k) for k in range(0, 1000, 250))
    assert np.linalg.norm(parts - full) <= 1e-14 * np.linalg.norm(full)


def test_sketch_rows_matches_full(oracle_mod):
    rng = np.random.default_rng(1)
    A = rng.standard_normal((3000, 9))
    full = oracle_mod.sketch_dense(A, 0, 2, 512, 8)
    rows = np.array([0, 5, 511, 300, 64])
    np.testing.assert_array_equal(oracle_mod.sketch_dense_rows(A, 0, 2, 512, 8, rows), full[rows])


def test_linearity_S_Ax(oracle_mod):
    """S (A x) == (S A) x."""
    rng = np.random.default_rng(2)
    A = rng.standard_normal((2000, 8))
    x = rng.standard_normal(8)
    SA = oracle_mod.sketch_dense(A, 0, 0, 100, 1)
    SAx = oracle_mod.sketch_dense((A @ x)[:, None], 0, 0, 100, 1)[:, 0]
    np.testing.assert_allclose(SAx, SA @ x, rtol=0, atol=1e-12 * np.abs(SA @ x).max())


def test_SSt_diagonal_lemma(oracle_mod):
    """Lemma: S S^T is diagonal with (S S^T)_ii = N_i."""
    n, m = 5000, 64
    S = dense_S(oracle_mod, 0, 9, m, 1, n)
    G = S @ S.T
    N = (S != 0).sum(1)
    np.testing.assert_array_equal(G, np.diag(N.astype(float)))


def test_E_SSt_and_E_StS_lemmas(oracle_mod):
    """E[S S^T] = (n/m) I and E[S^T S] = I,
    Monte Carlo over iterations t with the SPEC.md:466 bound 5/sqrt(trials)."""
    n, m, trials = 100, 10, 2000
    acc_sst = np.zeros((m, m))
    acc_sts = np.zeros((n, n))
    for t in range(trials):
        S = dense_S(oracle_mod, 11, t, m, 1, n)
        acc_sst += S @ S.T
        acc_sts += S.T @ S
    assert np.abs(acc_sts / trials - np.eye(n)).max() <= 5 / np.sqrt(trials)
    # diagonal of S S^T is Binomial(n, 1/m): mean n/m, sd sqrt(n/m) per draw
    dev = np.abs(acc_sst / trials - (n / m) * np.eye(m)).max()
    assert dev <= 5 * np.sqrt(n / m) / np.sqrt(trials)


def test_csr_sketch_matches_dense(oracle_mod):
    rng = np.random.default_rng(3)
    M = sp.random(3000, 40, density=0.05, format="csr", random_state=4, data_rvs=rng.standard_normal)
    M.sort_indices()
    dense = M.toarray()
    for s in (1, 4):
        a = oracle_mod.sketch_csr(M.indptr.astype(np.int64), M.indices, M.data, 40, 0, 2, 64, s)
        b = oracle_mod.sketch_dense(dense, 0, 2, 64, s)
        np.testing.assert_array_equal(a, b)  # adding explicit zeros changes nothing
        S = dense_S(oracle_mod, 0, 2, 64, s, 3000)
        assert np.linalg.norm(a - S @ dense) <= 1e-14 * np.linalg.norm(a)


def test_gradient_against_numpy_and_finite_differences(oracle_mod):
    """g = A^T (b - A x) = -grad f, f(x) = 1/2 ||Ax - b||^2 (Eq. (1), (2); reading R21)."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((500, 6))
    b = rng.standard_normal(500)
    x = rng.standard_normal(6)
    g = oracle_mod.grad_dense(A, b, x)
    ref = A.T @ (b - A @ x)
    np.testing.assert_allclose(g, ref, rtol=1e-12, atol=1e-12 * np.abs(A).sum())
    f = lambda z: 0.5 * np.sum((A @ z - b) ** 2)
    h = 1e-5
    fd = np.array([(f(x + h * e) - f(x - h * e)) / (2 * h) for e in np.eye(6)])
    np.testing.assert_allclose(-g, fd, rtol=1e-6)


def test_gradient_csr(oracle_mod):
    rng = np.random.default_rng(6)
    M = sp.random(2000, 30, density=0.04, format="csr", random_state=7, data_rvs=rng.standard_normal)
    M.sort_indices()
    b = rng.standard_normal(2000)
    x = rng.standard_normal(30)
    g = oracle_mod.grad_csr(M.indptr.astype(np.int64), M.indices, M.data, 30, b, x)
    np.testing.assert_allclose(g, M.T @ (b - M @ x), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle_mod.matvec_csr(M.indptr.astype(np.int64), M.indices, M.data, x), M @ x,
                               rtol=1e-13, atol=1e-13)


def test_gram_against_numpy(oracle_mod):
    rng = np.random.default_rng(8)
    SA = rng.standard_normal((300, 17))
    H = oracle_mod.gram(SA)
    np.testing.assert_array_equal(H, H.T)
    ref = SA.T @ SA
    assert np.linalg.norm(H - ref) <= 1e-14 * np.linalg.norm(ref)


def test_gram_collision_identity(oracle_mod):
    """(SA)^T SA - A^T A = sum_{i != k, h_i = h_k} s_i s_k a_i a_k^T  (exact structure of
    one CountSketch draw; the off-diagonal terms of S^T S)."""
    rng = np.random.default_rng(9)
    n, d, m = 120, 4, 16
    A = rng.standard_normal((n, d))
    bk, sg = oracle_mod.hash_rows(0, 0, m, 1, 0, n)
    bk, sg = bk[:, 0], sg[:, 0].astype(float)
    H = oracle_mod.gram(oracle_mod.sketch_dense(A, 0, 0, m, 1))
    extra = np.zeros((d, d))
    for i in range(n):
        for k in range(n):
            if i != k and bk[i] == bk[k]:
                extra += sg[i] * sg[k] * np.outer(A[i], A[k])
    np.testing.assert_allclose(H - A.T @ A, extra, atol=1e-11)


def test_unbiased_hessian(oracle_mod):
    """E[(SA)^T SA] = A^T A (named in the north star): the mean over
    T_mc fresh sketches approaches A^T A like sqrt((d+1)/(m T_mc))."""
    rng = np.random.default_rng(10)
    A = rng.standard_normal((2000, 5))
    G = A.T @ A
    for s in (1, 4):
        acc = np.zeros_like(G)
        T = 400
        for t in range(T):
            acc += oracle_mod.gram(oracle_mod.sketch_dense(A, 0, t, 64, s))
        rel = np.linalg.norm(acc / T - G) / np.linalg.norm(G)
        assert rel < 4 * np.sqrt(6 / (64 * T)), (s, rel)
        single = np.linalg.norm(oracle_mod.gram(oracle_mod.sketch_dense(A, 0, 0, 64, s)) - G) / np.linalg.norm(G)
        assert single > rel  # averaging helps: the estimator is noisy per draw, unbiased in mean


def test_pred_rel_err(oracle_mod):
    rng = np.random.default_rng(11)
    A = rng.standard_normal((400, 7))
    x, y = rng.standard_normal(7), rng.standard_normal(7)
    ref = np.linalg.norm(A @ (x - y)) / np.linalg.norm(A @ y)
    assert abs(oracle_mod.pred_rel_err(x, y, A) - ref) <= 1e-13 * ref
    assert oracle_mod.pred_rel_err(y, y, A) == 0.0


def test_openmp_timing_variants_match_serial(oracle_mod):
    """The OpenMP timing variants (bench.py cpu_baseline) compute the serial
    oracle's S A and A^T(b - Ax) up to rounding (thread partials added in order)."""
    import numpy as np
    rng = np.random.default_rng(12)
    A = rng.standard_normal((5003, 17))
    b = rng.standard_normal(5003)
    x = rng.standard_normal(17)
    for m, s in ((256, 1), (512, 8)):
        ref = oracle_mod.sketch_dense(A, 3, 2, m, s, row_offset=11)
        got = oracle_mod.sketch_dense_omp(A, 3, 2, m, s, row_offset=11)
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    g = oracle_mod.grad_dense(A, b, x)
    go = oracle_mod.grad_dense_omp(A, b, x)
    bound = 1e-12 * (np.abs(A) * np.abs(b - A @ x)[:, None]).sum(0)
    assert (np.abs(go - g) <= bound).all()
    assert oracle_mod.omp_threads() >= 1
