"""x_OPT for a CSR A (the reference point of bench.py's time-to-1e-10 run on C3):
ShardedIHS.exact_ols_normal_cg -- conjugate gradients on the normal equations
A^T A x = A^T b with the a5 gradient kernel as the operator (the linear term of
Eq. (2)) -- against the textbook least-squares solution
(numpy.linalg.lstsq on the densified matrix: a library routine, not the oracle
and not the CUDA path), and the dense path's exact_ols against the same."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def random_csr(n, d, density, seed):
    rng = np.random.default_rng(seed)
    nnz_row = rng.binomial(d, density, size=n)
    nnz_row[0] = 0  # an empty row
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(nnz_row, out=rp[1:])
    col = np.concatenate([np.sort(rng.choice(d, size=k, replace=False)) for k in nnz_row]).astype(np.int32)
    val = rng.standard_normal(rp[-1])
    return rp, col, val


@pytest.mark.parametrize("n,d,density", [(20000, 64, 0.05), (50001, 200, 0.02)])
def test_exact_ols_normal_cg_matches_lstsq(n, d, density):
    import paper_1910_14166_b200 as P
    from paper_1910_14166_b200.dist import CudaOps, ShardedIHS

    rp, col, val = random_csr(n, d, density, seed=n + d)
    rng = np.random.default_rng(7)
    Ad = np.zeros((n, d))
    rows = np.repeat(np.arange(n), np.diff(rp))
    Ad[rows, col] = val
    b = Ad @ rng.standard_normal(d) + rng.standard_normal(n)
    xref = np.linalg.lstsq(Ad, b, rcond=None)[0]
    ctx = P.Context(0)
    A = P.Csr(torch.from_numpy(rp).to(DEV), torch.from_numpy(col).to(DEV), torch.from_numpy(val).to(DEV), d)
    S = ShardedIHS(A, torch.from_numpy(b).to(DEV), P.Spec(m=8 * d, s=4), ops=CudaOps(ctx), lookahead=False)
    x = S.exact_ols_normal_cg().cpu().numpy()
    assert ctx.status() == P.OK
    # relative prediction-norm error ||A(x - xref)|| / ||A xref||
    err = np.linalg.norm(Ad @ (x - xref)) / np.linalg.norm(Ad @ xref)
    assert err < 1e-12, err
    # and through the product's own bookkeeping call (a7)
    e = S.pred_errors(torch.from_numpy(x[None, :]).to(DEV), torch.from_numpy(xref).to(DEV)).cpu().numpy()
    assert e[0] < 1e-12
    ctx.close()
