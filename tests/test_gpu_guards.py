"""In-house memory and race checks (compute-sanitizer is closed on this GPU
pool: profiles/r02/sanitizer_closed.txt).

  * guard zones: every output is a window of a larger buffer whose head and
    tail are filled with a sentinel bit pattern; after the call the sentinels
    must be intact (a write past either end of an output fails);
  * inputs unchanged: every input is compared bit for bit with a copy taken
    before the call (a kernel writing to an input fails);
  * races: the deterministic kernels (everything but the CSR scatter, whose
    L2 reductions have no fixed order) are run repeatedly and must return
    bitwise-identical results (an unsynchronised shared-memory or grid-level
    race shows up as run-to-run differences).
Small shapes that still span several CTAs, clusters and pipeline stages.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)
GUARD = 4096  # doubles of guard before and after each output
SENTINEL = -7.77e300


@pytest.fixture(scope="module")
def P():
    import paper_1910_14166_b200 as P
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    P.lib()
    return P


def guarded(shape):
    n = int(np.prod(shape))
    buf = torch.full((GUARD + n + GUARD,), SENTINEL, dtype=torch.float64, device=DEV)
    return buf, buf[GUARD:GUARD + n].view(shape)


def intact(buf):
    return bool((buf[:GUARD] == SENTINEL).all()) and bool((buf[-GUARD:] == SENTINEL).all())


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def run_checked(fn, inputs, outs, reps=3):
    """Run fn() reps times; check guards, inputs, and bitwise repeatability."""
    before = [x.clone() for x in inputs]
    results = []
    for _ in range(reps):
        fn()
        torch.cuda.synchronize()
        results.append([o[1].clone() for o in outs])
        for buf, _ in outs:
            assert intact(buf), "output guard overwritten"
    for x, y in zip(inputs, before):
        assert torch.equal(x, y), "input modified"
    return results


@pytest.mark.parametrize("n,d,m,s", [(20_000, 64, 256, 1), (9_001, 96, 4096, 8), (30_000, 10, 512, 4),
                                     (5_000, 130, 300, 1), (70_000, 98, 2048, 8)])
def test_sketch_grad_guards_and_repeatability(P, n, d, m, s):
    rng = np.random.default_rng(n + m)
    A, b, x = t(rng.standard_normal((n, d))), t(rng.standard_normal(n)), t(rng.standard_normal(d))
    sab, SA = guarded((m, d))
    gb, g = guarded((d,))
    ctx = P.Context(0)
    res = run_checked(lambda: P.ihs_sketch_grad(A, P.Spec(m=m, s=s), 2, b, x, SA=SA, g=g, ctx=ctx), [A, b, x],
                      [(sab, SA), (gb, g)])
    for r in res[1:]:
        assert torch.equal(r[0], res[0][0]) and torch.equal(r[1], res[0][1]), "not repeatable"


def test_csr_guards(P):
    rng = np.random.default_rng(4)
    n, d = 20_000, 300
    cnt = rng.binomial(d, 0.01, n)
    rp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    cl = np.concatenate([np.sort(rng.choice(d, k, replace=False)) for k in cnt]).astype(np.int32)
    vl = rng.standard_normal(int(rp[-1]))
    Ac = (t(rp), t(cl), t(vl), d)
    b, x = t(rng.standard_normal(n)), t(rng.standard_normal(d))
    sab, SA = guarded((512, d))
    gb, g = guarded((d,))
    ctx = P.Context(0)
    run_checked(lambda: P.ihs_sketch_grad(Ac, P.Spec(m=512, s=4), 1, b, x, SA=SA, g=g, ctx=ctx),
                [Ac[0], Ac[1], Ac[2], b, x], [(sab, SA), (gb, g)])


@pytest.mark.parametrize("m,d", [(512, 96), (2048, 256), (1024, 640), (200, 10)])
def test_gram_guards_and_repeatability(P, m, d):
    rng = np.random.default_rng(m + d)
    SA = t(rng.standard_normal((m, d)))
    hb, H = guarded((d, d))
    res = run_checked(lambda: P.ihs_gram(SA, out=H), [SA], [(hb, H)])
    assert all(torch.equal(r[0], res[0][0]) for r in res)


@pytest.mark.parametrize("d", [10, 64, 128, 160, 300, 1024])
def test_ols_update_guards_and_repeatability(P, d):
    rng = np.random.default_rng(d)
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    H = t((Q * np.geomspace(1.0, 30.0, d)) @ Q.T)
    g, x = t(rng.standard_normal(d)), t(rng.standard_normal(d))
    for mode in (1, 2):
        ctx = P.Context(0)
        ctx.set_option("ols_large", mode)
        xb, xn = guarded((d,))
        res = run_checked(lambda: P.ihs_ols_update(H, g, x, out=xn, ctx=ctx), [H, g, x], [(xb, xn)])
        assert all(torch.equal(r[0], res[0][0]) for r in res)
        assert ctx.status() == P.OK


@pytest.mark.parametrize("m,d", [(1024, 128), (512, 48), (4096, 96)])
def test_factor_and_fused_guards(P, m, d):
    rng = np.random.default_rng(m * d)
    SA = t(rng.standard_normal((m, d)))
    g, x = t(rng.standard_normal(d)), t(rng.standard_normal(d))
    ctx = P.Context(0)
    hb, Hinv = guarded((d, d))
    xb, xn = guarded((d,))
    res = run_checked(lambda: (P.ihs_ols_factor(SA, out=Hinv, ctx=ctx), P.ihs_ols_apply(Hinv, g, x, out=xn, ctx=ctx)),
                      [SA, g, x], [(hb, Hinv), (xb, xn)])
    assert all(torch.equal(r[0], res[0][0]) and torch.equal(r[1], res[0][1]) for r in res)
    hb2, H2 = guarded((d, d))
    xb2, xn2 = guarded((d,))
    ctx.set_option("fuse_max_d", 128)
    res = run_checked(lambda: P.ihs_gram_ols_update(SA, g, x, out=xn2, H=H2, ctx=ctx), [SA, g, x],
                      [(hb2, H2), (xb2, xn2)])
    assert all(torch.equal(r[1], res[0][1]) for r in res)


@pytest.mark.parametrize("d,kind", [(64, "l1"), (256, "l1"), (256, "lasso"), (300, "l1")])
def test_pg_guards_and_repeatability(P, d, kind):
    rng = np.random.default_rng(d + len(kind))
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    H = t((Q * np.geomspace(1.0, 10.0, d)) @ Q.T + np.eye(d))
    g, x = t(rng.standard_normal(d) * 10), t(np.zeros(d))
    ctx = P.Context(0)
    ctx.set_option("pg_warm", 0)  # every call the same cold power iteration: repeatable
    xb, xn = guarded((d,))
    fn = P.ihs_l1ball_update if kind == "l1" else P.ihs_lasso_update
    res = run_checked(lambda: fn(H, g, x, 2.0, out=xn, ctx=ctx), [H, g, x], [(xb, xn)])
    assert all(torch.equal(r[0], res[0][0]) for r in res)


def test_solve_history_guards(P):
    rng = np.random.default_rng(2)
    n, d, T = 40_000, 32, 5
    A, b = t(rng.standard_normal((n, d))), t(rng.standard_normal(n))
    for la in (0, 1):
        ctx = P.Context(0)
        ctx.set_option("lookahead", la)
        hb, xh = guarded((T + 1, d))
        xb, xo = guarded((d,))
        res = run_checked(lambda: P.ihs_solve_ols(A, b, P.Spec(m=512), T, ctx=ctx, x_out=xo, x_hist=xh), [A, b],
                          [(hb, xh), (xb, xo)])
        assert all(torch.equal(r[0], res[0][0]) for r in res)
