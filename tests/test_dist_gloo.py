"""The N > 1 path on CPU: world_size-2 gloo process groups drive
paper_1910_14166_b200.dist.ShardedIHS (row sharding with global-row hashing,
the packed [SA | g] all-reduce, replicated Gram + inner solve).  The arithmetic
backend is the oracle here (tests may use it; the product passes CudaOps), so
these tests check the host-side logic: shard ranges, row offsets, packing and
the exchange, against the unsharded oracle run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleOps:
    """CudaOps' interface implemented with the CPU oracle (test backend only)."""

    def __init__(self):
        import oracle
        self.o = oracle

    def sketch_grad(self, A, spec, t, b, x, SA, g):
        SA.copy_(torch.from_numpy(self.o.sketch_dense(A.A.numpy(), spec.seed, t, spec.m, spec.s,
                                                      row_offset=A.row_offset)))
        g.copy_(torch.from_numpy(self.o.grad_dense(A.A.numpy(), b.numpy(), x.numpy())))

    def grad(self, A, b, x, g):
        g.copy_(torch.from_numpy(self.o.grad_dense(A.A.numpy(), b.numpy(), x.numpy())))

    def gram(self, SA, H, scale=1.0):
        H.copy_(torch.from_numpy(self.o.gram(SA.numpy())) * scale * scale)

    def ols(self, H, g, x, xn):
        xn.copy_(torch.from_numpy(self.o.ols_step(H.numpy(), g.numpy(), x.numpy())))

    def l1(self, H, g, x, tau, cfg, xn, inner):
        xo, it, _ = self.o.l1ball_step(H.numpy(), g.numpy(), x.numpy(), tau)
        xn.copy_(torch.from_numpy(xo))
        inner.fill_(it)

    def err2(self, A, X, xref):
        An = A.A.numpy()
        e = [float(np.sum((An @ (xk - xref.numpy())) ** 2)) for xk in X.numpy()]
        return torch.tensor(e, dtype=torch.float64), torch.tensor([float(np.sum((An @ xref.numpy()) ** 2))],
                                                                 dtype=torch.float64)


class OracleLookaheadOps(OracleOps):
    """+ the look-ahead OLS calls (sketch only, H^{-1}, apply), test backend only."""

    def sketch(self, A, spec, t, SA):
        SA.copy_(torch.from_numpy(self.o.sketch_dense(A.A.numpy(), spec.seed, t, spec.m, spec.s,
                                                      row_offset=A.row_offset)))

    def ols_factor(self, SA, Hinv):
        Hinv.copy_(torch.from_numpy(np.linalg.inv(self.o.gram(SA.numpy()))))

    def ols_apply(self, Hinv, g, x, xn):
        xn.copy_(x + Hinv @ g)

    def gram_lookahead(self, SA, H):
        H.copy_(torch.from_numpy(self.o.gram(SA.numpy())))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1910_14166_b200 as P
        from paper_1910_14166_b200.dist import ShardedIHS, shard_rows
        import synthetic
        cfg = synthetic.CONFIGS[case["cfg"]].scaled(case["n"])
        prob = synthetic.problem(cfg, "cpu")
        r0, r1 = shard_rows(cfg.n, rank, world)
        A = P.Dense(prob["A"][r0:r1].contiguous(), row_offset=r0)
        b = prob["b"][r0:r1].contiguous()
        la = case.get("lookahead", False)
        S = ShardedIHS(A, b, P.Spec(m=case["m"], s=case["s"]), ops=OracleLookaheadOps() if la else OracleOps(),
                       constraint=case["constraint"], radius=prob["tau"], lookahead=la)
        assert S.lookahead == la
        xh = S.solve(case["T"], iter0=case["iter0"])
        xopt = S.exact_ols() if case["constraint"] == "ols" else None
        errs = S.pred_errors(xh, xopt) if xopt is not None else None
        out[rank] = {"xh": xh.numpy().copy(), "rows": (r0, r1), "xopt": None if xopt is None else xopt.numpy().copy(),
                     "errs": None if errs is None else errs.numpy().copy()}
    finally:
        dist.destroy_process_group()


def run_world(case, world=2):
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, case, out), nprocs=world, join=True)
    return dict(out)


def test_shard_rows_partition():
    from paper_1910_14166_b200.dist import shard_rows
    for n in (1, 7, 2000, 1 << 20):
        for world in (1, 2, 3, 8):
            parts = [shard_rows(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


@pytest.mark.parametrize("case", [
    {"cfg": "C1", "n": 2000, "m": 200, "s": 1, "T": 6, "iter0": 0, "constraint": "ols"},
    {"cfg": "C5", "n": 3001, "m": 256, "s": 8, "T": 4, "iter0": 7, "constraint": "ols"},
    {"cfg": "C4", "n": 4000, "m": 512, "s": 1, "T": 4, "iter0": 0, "constraint": "l1ball"},
    {"cfg": "C2", "n": 5001, "m": 256, "s": 1, "T": 5, "iter0": 2, "constraint": "ols", "lookahead": True},
    {"cfg": "C4", "n": 4000, "m": 512, "s": 1, "T": 4, "iter0": 1, "constraint": "l1ball", "lookahead": True},
])
def test_sharded_ihs_matches_unsharded_oracle(oracle_mod, case):
    import synthetic
    res = run_world(case)
    # every rank holds a bitwise-identical iterate history (replicated Gram + solve)
    np.testing.assert_array_equal(res[0]["xh"], res[1]["xh"])
    assert res[0]["rows"][1] == res[1]["rows"][0]
    cfg = synthetic.CONFIGS[case["cfg"]].scaled(case["n"])
    prob = synthetic.problem(cfg, "cpu")
    A, b = prob["A"].numpy(), prob["b"].numpy()
    kw = dict(constraint="l1ball", tau=prob["tau"]) if case["constraint"] == "l1ball" else {}
    xo, _ = oracle_mod.ihs_solve(A, b, m=case["m"], s=case["s"], T=case["T"], iter0=case["iter0"], **kw)
    for t in range(1, case["T"] + 1):
        assert oracle_mod.pred_rel_err(res[0]["xh"][t], xo[t], A) <= 1e-11
    if res[0]["xopt"] is not None:
        xl = np.linalg.lstsq(A, b, rcond=None)[0]
        assert oracle_mod.pred_rel_err(res[0]["xopt"], xl, A) <= 1e-12
        e_ref = np.array([oracle_mod.pred_rel_err(x, res[0]["xopt"], A) for x in res[0]["xh"]])
        np.testing.assert_allclose(res[0]["errs"], e_ref, rtol=1e-9, atol=1e-15)
