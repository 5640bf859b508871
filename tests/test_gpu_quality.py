"""NEXT-3 (Appendix B): the sketch-quality sweep's error
values computed through the C ABI equal the oracle's (oracle sketch + oracle
Gram, numpy for the exact A^T A) on a small CSR and a dense instance, and the
error shrinks as gamma grows (E ~ sqrt((d+1)/m))."""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1910_14166_b200 as P
    P.lib()
    return P


@pytest.mark.parametrize("layout", ["csr", "dense"])
def test_quality_errors_match_oracle(P, oracle_mod, layout):
    from paper_1910_14166_b200.quality import sketch_quality
    n, d = 3000, 40
    cfg = synthetic.Config("q", n, d, layout, "normal", "countsketch", 1, 1, 1, "ols", density=0.05, data_seed=9)
    if layout == "csr":
        rp, cl, vl = synthetic.csr_A(cfg, "cpu")
        A = np.zeros((n, d))
        rows = np.repeat(np.arange(n), np.diff(rp.numpy()))
        A[rows, cl.numpy()] = vl.numpy()
        Ag = P.Csr(rp.to(DEV), cl.to(DEV), vl.to(DEV), d)
    else:
        A = synthetic.dense_A(cfg, "cpu").numpy()
        Ag = P.Dense(torch.from_numpy(A).to(DEV))
    G = A.T @ A
    for fam, s, gammas in (("countsketch", 1, [1, 2, 10]), ("sjlt", 4, [1, 5])):
        res = sketch_quality(Ag, fam, s, gammas, trials=3)
        for r in res:
            ref = []
            for t in range(3):
                if layout == "csr":
                    SA = oracle_mod.sketch_csr(rp.numpy(), cl.numpy(), vl.numpy(), d, 0, t, r["m"], s)
                else:
                    SA = oracle_mod.sketch_dense(A, 0, t, r["m"], s)
                ref.append(np.linalg.norm(oracle_mod.gram(SA) - G) / np.linalg.norm(G))
            np.testing.assert_allclose(r["errs"], ref, rtol=1e-9)
        errs = [r["err_mean"] for r in res]
        assert errs[-1] < errs[0]  # more rows, smaller distortion
