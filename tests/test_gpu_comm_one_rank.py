"""The in-library NCCL path on one GPU (SURVEY 8(e), a3 = the all-reduce of
[SA | g], exact by linearity of S).

A ctx given a ONE-rank communicator (ihs_ctx_set_comm(ctx, 0, 1, uid), include/
ihs.h) takes the solve calls' collective schedules: the rank-count all-reduce
of the schedule decision, the [S A | g] all-reduces between the pass and the
factor, the separate apply / PG launches -- every NCCL call the multi-GPU run
makes, over one rank.  Results must match the oracle at every iterate (reading
R8) like the single-rank schedules.  What this cannot check: sums over several
ranks (this pool gives one GPU per call; those are covered by the gloo tests
with the oracle as arithmetic, tests/test_dist_gloo.py)."""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def P():
    import paper_1910_14166_b200 as P

    return P


def iterate_parity(A, xg, xo, oracle_mod):
    """The largest relative prediction-norm error over the iterates (reading R8)."""
    return max(oracle_mod.pred_rel_err(a, b, A) for a, b in zip(xg[1:], xo[1:]))


def comm_ctx(P, **opts):
    ctx = P.Context(0)
    ctx.set_comm(0, 1, P.nccl_unique_id())
    for k, v in opts.items():
        ctx.set_option(k, v)
    return ctx


def test_set_comm_once(P):
    ctx = comm_ctx(P)
    with pytest.raises(P.IhsError):
        ctx.set_comm(0, 1, P.nccl_unique_id())
    ctx.close()


@pytest.mark.parametrize("lookahead", [1, 0])
def test_solve_ols_one_rank_comm(P, oracle_mod, lookahead):
    """ihs_solve_ols through the collective schedules (look-ahead: the [S^{t+1}
    A | g^t] all-reduce, the factor and the apply as separate launches; plain:
    the all-reduce of [SA | g] per iteration) against the oracle, and against
    the same call without a communicator."""
    cfg = synthetic.CONFIGS["C2"].scaled(1 << 16)
    prob = synthetic.problem(cfg, "cpu")
    A, b = prob["A"].numpy(), prob["b"].numpy()
    T = 5
    outs = []
    for comm in (True, False):
        ctx = comm_ctx(P, lookahead=lookahead) if comm else P.Context(0)
        if not comm:
            ctx.set_option("lookahead", lookahead)
        out = P.ihs_solve_ols(prob["A"].to(DEV), prob["b"].to(DEV), P.Spec(m=cfg.m), T, iter0=1, ctx=ctx)
        assert ctx.status() == P.OK
        outs.append(out["x_hist"].cpu().numpy())
        ctx.close()
    xo, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=1, T=T, iter0=1)
    assert iterate_parity(A, outs[0], xo, oracle_mod) <= 1e-9
    assert iterate_parity(A, outs[0], outs[1], oracle_mod) <= 1e-12


@pytest.mark.parametrize("constraint", ["l1ball", "lasso"])
def test_solve_pg_one_rank_comm(P, oracle_mod, constraint):
    """ihs_solve_l1ball / ihs_solve_lasso with the look-ahead Gram schedule and
    a one-rank communicator against the oracle at every t."""
    name = "C4" if constraint == "l1ball" else "C4P"
    cfg = synthetic.CONFIGS[name].scaled(1 << 15)
    prob = synthetic.problem(cfg, "cpu")
    A, b = prob["A"].numpy(), prob["b"].numpy()
    radius = prob["tau"] if constraint == "l1ball" else cfg.lam
    T = 5
    ctx = comm_ctx(P, lookahead=1)
    fn = P.ihs_solve_l1ball if constraint == "l1ball" else P.ihs_solve_lasso
    out = fn(prob["A"].to(DEV), prob["b"].to(DEV), radius, P.Spec(m=cfg.m), T, iter0=1, ctx=ctx)
    assert ctx.status() == P.OK
    ctx.close()
    xo, _ = oracle_mod.ihs_solve(A, b, m=cfg.m, s=1, T=T, iter0=1, constraint=constraint, tau=radius)
    assert iterate_parity(A, out["x_hist"].cpu().numpy(), xo, oracle_mod) <= 1e-9


def test_allreduce_and_reduce_argument_one_rank_comm(P):
    """ihs_allreduce_sum and the reduce argument of ihs_sketch / ihs_grad
    through NCCL over one rank: the identity."""
    rng = np.random.default_rng(11)
    A = torch.from_numpy(rng.standard_normal((20_000, 64))).to(DEV)
    b = torch.from_numpy(rng.standard_normal(20_000)).to(DEV)
    x = torch.from_numpy(rng.standard_normal(64)).to(DEV)
    ctx = comm_ctx(P)
    buf = torch.from_numpy(rng.standard_normal(1 << 16)).to(DEV)
    ref = buf.clone()
    P.ihs_allreduce_sum(buf, ctx=ctx)
    ctx.synchronize()
    assert torch.equal(buf, ref)
    spec = P.Spec(m=512, s=4)
    assert torch.equal(P.ihs_sketch(A, spec, 2, reduce=True, ctx=ctx), P.ihs_sketch(A, spec, 2))
    assert torch.equal(P.ihs_grad(A, b, x, reduce=True, ctx=ctx), P.ihs_grad(A, b, x))
    ctx.close()
