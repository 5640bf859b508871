"""Row-sharded IHS across ranks (BASELINE.json north_star).

Rank k of P holds the contiguous rows [k n/P, (k+1) n/P) of A and b and hashes
with GLOBAL row indices, so by linearity sum_k S_k A_k = S A and
sum_k A_k^T (b_k - A_k x) = A^T (b - A x).  Per iteration the only exchange is
one all-reduce of the packed buffer [SA | g] (m*d + d doubles); the Gram and
the inner QP are then replicated (deterministic kernels on identical inputs, so
every rank holds a bitwise-identical x^{t+1}).

torch.distributed (NCCL on GPUs) is the plumbing for the exchange; every step
of the arithmetic runs in libihs.so through ``CudaOps``.  The ``ops`` and
``allreduce`` hooks exist so the host-side sharding logic can be exercised with
a CPU backend under gloo in tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

import paper_1910_14166_b200 as P


def shard_rows(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row block of rank `rank` (sizes differ by at most one row)."""
    return n * rank // world, n * (rank + 1) // world


def torch_allreduce(buf: torch.Tensor, group=None) -> None:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)


class CudaOps:
    """The product backend: every call goes to the C ABI."""

    def __init__(self, ctx: P.Context):
        self.ctx = ctx

    def sketch_grad(self, A, spec, t, b, x, SA, g):
        P.ihs_sketch_grad(A, spec, t, b, x, SA=SA, g=g, ctx=self.ctx)

    def gram(self, SA, H, scale=1.0):
        P.ihs_gram(SA, scale=scale, out=H, ctx=self.ctx)

    def grad(self, A, b, x, g):
        P.ihs_grad(A, b, x, out=g, ctx=self.ctx)

    def ols(self, H, g, x, xn):
        P.ihs_ols_update(H, g, x, out=xn, ctx=self.ctx)

    def gram_ols(self, SA, g, x, xn, H):
        P.ihs_gram_ols_update(SA, g, x, out=xn, H=H, ctx=self.ctx)

    def l1(self, H, g, x, tau, cfg, xn, inner):
        P.ihs_l1ball_update(H, g, x, tau, cfg=cfg, out=xn, inner=inner, ctx=self.ctx)

    def lasso(self, H, g, x, lam, cfg, xn, inner):
        P.ihs_lasso_update(H, g, x, lam, cfg=cfg, out=xn, inner=inner, ctx=self.ctx)

    def err2(self, A, X, xref):
        return P.ihs_pred_err2(A, X, xref, ctx=self.ctx)


class ShardedIHS:
    """One rank's view of the row-sharded IHS problem."""

    def __init__(self, A, b: torch.Tensor, spec: P.Spec, *, constraint: str = "ols", radius: float = 0.0,
                 cfg=None, ops=None, allreduce=None, group=None):
        self.A = A
        self.b = b
        self.spec = spec
        self.constraint = constraint
        self.radius = radius
        self.cfg = cfg
        self.group = group
        self.ops = ops if ops is not None else CudaOps(P.default_context(b.device))
        self.allreduce = allreduce if allreduce is not None else (lambda t: torch_allreduce(t, group))
        d, m = A.d, spec.m
        dev = b.device
        self.d, self.m = d, m
        self.pack = torch.empty(m * d + d, dtype=torch.float64, device=dev)
        self.SA = self.pack[: m * d].view(m, d)
        self.g = self.pack[m * d:]
        self.H = torch.empty((d, d), dtype=torch.float64, device=dev)
        self.inner = torch.zeros(1, dtype=torch.int32, device=dev)

    def step(self, t: int, x: torch.Tensor, xn: torch.Tensor) -> torch.Tensor:
        """x^{t+1} from x^t: a1-a2+a5 (local), a3 (all-reduce), a4, a6 (replicated)."""
        self.ops.sketch_grad(self.A, self.spec, t, self.b, x, self.SA, self.g)
        self.allreduce(self.pack)
        if self.constraint == "ols" and hasattr(self.ops, "gram_ols"):  # a4 + a6 fused (one launch)
            self.ops.gram_ols(self.SA, self.g, x, xn, self.H)
            return xn
        self.ops.gram(self.SA, self.H)
        if self.constraint == "ols":
            self.ops.ols(self.H, self.g, x, xn)
        elif self.constraint == "lasso":  # NEXT-2: radius carries lambda
            self.ops.lasso(self.H, self.g, x, self.radius, self.cfg, xn, self.inner)
        else:
            self.ops.l1(self.H, self.g, x, self.radius, self.cfg, xn, self.inner)
        return xn

    def solve(self, T: int, iter0: int = 0, x0: torch.Tensor | None = None) -> torch.Tensor:
        xh = torch.zeros((T + 1, self.d), dtype=torch.float64, device=self.b.device)
        if x0 is not None:
            xh[0].copy_(x0)
        for t in range(T):
            self.step(iter0 + t, xh[t], xh[t + 1])
        return xh

    def exact_ols(self) -> torch.Tensor:
        """x_OPT of Eq. (1) with C = R^d (dense A): G = A^T A on the DMMA Gram kernel,
        c = A^T b, one Cholesky solve and one refinement step; all-reduced."""
        d = self.d
        dev = self.b.device
        buf = torch.empty(d * d + d, dtype=torch.float64, device=dev)
        G, c = buf[: d * d].view(d, d), buf[d * d:]
        zero = torch.zeros(d, dtype=torch.float64, device=dev)
        self.ops.gram(self.A.A if isinstance(self.A, P.Dense) else self.A, G)
        self.ops.grad(self.A, self.b, zero, c)
        self.allreduce(buf)
        x = torch.empty(d, dtype=torch.float64, device=dev)
        self.ops.ols(G, c, zero, x)
        self.ops.grad(self.A, self.b, x, c)
        self.allreduce(c)
        x2 = torch.empty_like(x)
        self.ops.ols(G, c, x, x2)
        return x2

    def pred_errors(self, X: torch.Tensor, xref: torch.Tensor) -> torch.Tensor:
        """e_k = ||A(X_k - xref)|| / ||A xref|| over all ranks (a7, post hoc)."""
        err2, ref2 = self.ops.err2(self.A, X, xref)
        buf = torch.cat([err2, ref2])
        self.allreduce(buf)
        return torch.sqrt(buf[:-1] / buf[-1])
