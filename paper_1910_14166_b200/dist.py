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


class NvlsAllreduce:
    """a3 through NVLink SHARP: the [SA | g] sum as one library kernel
    (ihs_allreduce_multimem: multimem.ld_reduce.add.f64 + multimem.st on the
    multicast address) on a torch symmetric-memory buffer -- torch provides
    the buffer, its multicast mapping and the signal pads (plumbing).  Use as
    ShardedIHS(allreduce=NvlsAllreduce(m * d + d, device)).  Raises when the
    system gives no multicast mapping (then NCCL, the default, stays)."""

    def __init__(self, numel: int, device, group=None, ctx: "P.Context | None" = None):
        import torch.distributed._symmetric_memory as symm_mem
        self.ctx = ctx or P.default_context(device)
        self.buf = symm_mem.empty(numel, dtype=torch.float64, device=device)
        grp = group if group is not None else dist.group.WORLD
        self.h = symm_mem.rendezvous(self.buf, grp.group_name)
        if not self.h.multicast_ptr:
            raise RuntimeError("no NVLS multicast mapping for this group")
        self.pads = torch.tensor(list(self.h.signal_pad_ptrs), dtype=torch.int64, device=device)
        self.pad_slots = int(self.h.signal_pad_size) // 4

    def __call__(self, t: torch.Tensor) -> None:
        n = t.numel()
        flat = t.view(-1)
        self.buf[:n].copy_(flat)
        P.ihs_allreduce_multimem(int(self.h.multicast_ptr), self.pads, int(self.h.rank), int(self.h.world_size), n,
                                 self.pad_slots, ctx=self.ctx)
        flat.copy_(self.buf[:n])


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

    def sketch(self, A, spec, t, SA):
        P.ihs_sketch(A, spec, t, out=SA, ctx=self.ctx)

    def ols_factor(self, SA, Hinv):
        P.ihs_ols_factor(SA, out=Hinv, ctx=self.ctx)

    def ols_apply(self, Hinv, g, x, xn):
        P.ihs_ols_apply(Hinv, g, x, out=xn, ctx=self.ctx)

    def gram_lookahead(self, SA, H):
        P.ihs_gram_lookahead(SA, out=H, ctx=self.ctx)

    def lookahead_step(self, A, spec, t_next, b, x, Hinv, SA_next, Hinv_next, g, xn):
        P.ihs_ols_lookahead_step(A, spec, t_next, b, x, Hinv, SA_next=SA_next, Hinv_next=Hinv_next, g=g, out=xn,
                                 ctx=self.ctx)

    def l1(self, H, g, x, tau, cfg, xn, inner):
        P.ihs_l1ball_update(H, g, x, tau, cfg=cfg, out=xn, inner=inner, ctx=self.ctx)

    def lasso(self, H, g, x, lam, cfg, xn, inner):
        P.ihs_lasso_update(H, g, x, lam, cfg=cfg, out=xn, inner=inner, ctx=self.ctx)

    def err2(self, A, X, xref):
        return P.ihs_pred_err2(A, X, xref, ctx=self.ctx)


def lookahead_default(A, d: int, spec: P.Spec, constraint: str = "ols", rows: int | None = None) -> bool:
    """The look-ahead schedule pays when one pass over A is long next to the
    d x d work it hides (dense, CountSketch, rows * d >= 2^27 per rank; OLS:
    d <= 128); IHS_LOOKAHEAD=0/1 overrides (the rule of ihs_solve_*, api.cu).
    `rows` must be the same on every rank (ceil(n_global / world), see
    ShardedIHS): a per-rank size could put ranks on different schedules, whose
    collectives differ."""
    import os
    env = os.environ.get("IHS_LOOKAHEAD")
    if env is not None:  # forced: any matrix (OLS with d > 128 or CSR: the Gram-only form)
        return d >= 1 and env != "0"
    if constraint == "ols" and d > 256:  # the Gram-only look-ahead, when the Gram is long (C3; api.cu)
        return spec.m * d * d >= (1 << 32)
    ok = isinstance(A, P.Dense) and d >= 1 and (d <= 128 or constraint != "ols")
    return ok and spec.s == 1 and (A.n if rows is None else rows) * d >= (1 << 27)


class ShardedIHS:
    """One rank's view of the row-sharded IHS problem.

    OLS look-ahead (``lookahead``): the sketch S^{t+1}
    does not depend on x, so the pass over A that forms g^t also forms
    S^{t+1} A, the all-reduce carries [S^{t+1} A | g^t], and H_{t+1}^{-1}
    (Gram + Cholesky + inverse, ``ols_factor``) is computed on a side stream
    during the NEXT pass; the step itself only applies x^{t+1} = x^t +
    H_t^{-1} g^t (``ols_apply``).  Same iterates as the plain schedule (each
    iteration still uses its own S^t), to rounding.  For the l1 ball / LASSO
    only the Gram looks ahead (``gram_lookahead``: H_{t+1} beside the PG
    update of t).  A step whose t does not follow the previous one first
    sketches S^t A (the prologue)."""

    def __init__(self, A, b: torch.Tensor, spec: P.Spec, *, constraint: str = "ols", radius: float = 0.0,
                 cfg=None, ops=None, allreduce=None, group=None, lookahead: bool | None = None):
        self.A = A
        self.b = b
        self.spec = spec
        self.constraint = constraint
        self.radius = radius
        self.cfg = cfg
        self.group = group
        self.ops = ops if ops is not None else CudaOps(P.default_context(b.device))
        self.allreduce = allreduce if allreduce is not None else (lambda t: torch_allreduce(t, group))
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        # one rank and the default exchange: nothing to all-reduce, so the
        # look-ahead step can be the single fused call (ihs_ols_lookahead_step)
        self._solo = allreduce is None and world == 1
        d, m = A.d, spec.m
        dev = b.device
        self.d, self.m = d, m
        self.pack = torch.empty(m * d + d, dtype=torch.float64, device=dev)
        self.SA = self.pack[: m * d].view(m, d)
        self.g = self.pack[m * d:]
        self.H = torch.empty((d, d), dtype=torch.float64, device=dev)
        self.inner = torch.zeros(1, dtype=torch.int32, device=dev)
        if lookahead is None and hasattr(self.ops, "ctx"):  # the context's option (ihs_ctx_set_option), if set
            opt = self.ops.ctx.get_option("lookahead")
            if opt >= 0:
                lookahead = bool(opt)
        if lookahead is None:
            # the same decision on every rank: rows per rank from the global n
            nt = torch.tensor([float(A.n)], dtype=torch.float64, device=dev)
            if not self._solo:
                self.allreduce(nt)
            rows = -(-int(nt.item()) // world)
            lookahead = lookahead_default(A, d, spec, constraint, rows=rows)
        # Gram-only look-ahead (H_{t+1} formed ahead, the update then solves with
        # H_t): the l1 / LASSO updates, and OLS where the fused H^{-1} factor does
        # not apply (d > 128 or a CSR matrix: the conjugate-gradient update)
        self.la_gram_only = constraint != "ols" or d > 128 or not isinstance(A, P.Dense)
        need = "gram_lookahead" if self.la_gram_only else "ols_factor"
        self.lookahead = bool(lookahead) and hasattr(self.ops, need)
        self._la_t = None  # iteration whose H^{-1} is in self.Hinv[self._la_cur]
        if self.lookahead:
            self.packs = torch.empty((2, m * d + d), dtype=torch.float64, device=dev)
            self.Hinv = torch.empty((2, d, d), dtype=torch.float64, device=dev)  # H^{-1} (OLS) or H
            self._la_cur = 1  # the first prime() fills slot 0

    def prime(self, t: int) -> None:
        """Look-ahead prologue: S^t A (all-reduced) and its H^{-1}, so that step(t) is one pass."""
        if not self.lookahead or self._la_t == t:
            return
        m, d = self.m, self.d
        # into the slot the last update read (its factor was joined by that
        # update); the other slot may still be read by a pending factor / Gram
        k = 1 - self._la_cur
        pk = self.packs[k]
        self.ops.sketch(self.A, self.spec, t, pk[: m * d].view(m, d))
        self.allreduce(pk[: m * d])
        if self.la_gram_only:
            self.ops.gram_lookahead(pk[: m * d].view(m, d), self.Hinv[k])
        else:
            self.ops.ols_factor(pk[: m * d].view(m, d), self.Hinv[k])
        self._la_t, self._la_cur = t, k

    def step(self, t: int, x: torch.Tensor, xn: torch.Tensor) -> torch.Tensor:
        """x^{t+1} from x^t: a1-a2+a5 (local), a3 (all-reduce), a4, a6 (replicated)."""
        if self.lookahead:
            self.prime(t)
            m, d = self.m, self.d
            cur, nxt = self._la_cur, 1 - self._la_cur
            pk = self.packs[nxt]
            SAn, gn = pk[: m * d].view(m, d), pk[m * d:]
            if self.la_gram_only:  # only the Gram looks ahead
                self.ops.sketch_grad(self.A, self.spec, t + 1, self.b, x, SAn, gn)
                self.allreduce(pk)
                H = self.Hinv[cur]
                if self.constraint == "ols":
                    # the CG update first; the next Gram then runs beside the next pass
                    self.ops.ols(H, gn, x, xn)
                    self.ops.gram_lookahead(SAn, self.Hinv[nxt])
                    self._la_t, self._la_cur = t + 1, nxt
                    return xn
                self.ops.gram_lookahead(SAn, self.Hinv[nxt])  # beside this update
                if self.constraint == "lasso":
                    self.ops.lasso(H, gn, x, self.radius, self.cfg, xn, self.inner)
                else:
                    self.ops.l1(H, gn, x, self.radius, self.cfg, xn, self.inner)
                self._la_t, self._la_cur = t + 1, nxt
                return xn
            if self._solo and hasattr(self.ops, "lookahead_step"):
                self.ops.lookahead_step(self.A, self.spec, t + 1, self.b, x, self.Hinv[cur], SAn, self.Hinv[nxt], gn,
                                        xn)
                self._la_t, self._la_cur = t + 1, nxt
                return xn
            self.ops.sketch_grad(self.A, self.spec, t + 1, self.b, x, SAn, gn)  # S^{t+1} A and g^t
            self.allreduce(pk)
            self.ops.ols_factor(SAn, self.Hinv[nxt])  # beside the next pass (placed before its gather)
            self.ops.ols_apply(self.Hinv[cur], gn, x, xn)
            self._la_t, self._la_cur = t + 1, nxt
            return xn
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

    def exact_ols_normal_cg(self, max_iters: int = 200, tol: float = 1e-15, restarts: int = 2) -> torch.Tensor:
        """x_OPT of Eq. (1) with C = R^d when A^T A cannot be formed by the dense Gram kernel
        (CSR A): conjugate gradients on the normal equations A^T A x = A^T b with the a5
        kernel as the operator (A^T A p = -ihs_grad(A, b = 0, x = p); all-reduced over
        ranks), restarted from the true residual A^T(b - A x).  Bench / test bookkeeping
        (the reference point of the time-to-1e-10 run), not a step of the hot path: only
        the d-vector recurrences run in torch."""
        d, dev = self.d, self.b.device
        zb = torch.zeros_like(self.b)
        x = torch.zeros(d, dtype=torch.float64, device=dev)
        r = torch.empty(d, dtype=torch.float64, device=dev)
        Ap = torch.empty(d, dtype=torch.float64, device=dev)
        r0n = None
        for _ in range(restarts):
            self.ops.grad(self.A, self.b, x, r)
            self.allreduce(r)
            rs = torch.dot(r, r)
            if r0n is None:
                r0n = torch.sqrt(rs)
            p = r.clone()
            for _k in range(max_iters):
                if float(torch.sqrt(rs)) <= tol * float(r0n):
                    break
                self.ops.grad(self.A, zb, p, Ap)
                self.allreduce(Ap)
                Ap.neg_()
                alpha = rs / torch.dot(p, Ap)
                x.add_(p, alpha=float(alpha))
                r.sub_(Ap, alpha=float(alpha))
                rs_new = torch.dot(r, r)
                p.mul_(float(rs_new / rs)).add_(r)
                rs = rs_new
        return x

    def exact_constrained(self, refine: int = 4) -> torch.Tensor:
        """x_OPT of the l1 ball (constraint "l1ball", radius tau) or the penalised
        LASSO ("lasso", radius = lambda) for dense A, the reference of the
        time-to-1e-10 runs: with G = A^T A (DMMA Gram of A itself) and
        c = A^T (b - A x), the inner update at (H = G, g = c) minimises exactly
        1/2 ||A y - b||^2 (+ lambda ||y||_1) over the set -- the IHS step with the
        exact Hessian -- so one update from 0 is x_OPT; a few more from the
        result remove the rounding of the first (all-reduced over ranks)."""
        d = self.d
        dev = self.b.device
        G = torch.empty((d, d), dtype=torch.float64, device=dev)
        self.ops.gram(self.A.A, G)
        self.allreduce(G.view(-1))
        x = torch.zeros(d, dtype=torch.float64, device=dev)
        c = torch.empty(d, dtype=torch.float64, device=dev)
        for _ in range(refine):
            self.ops.grad(self.A, self.b, x, c)
            self.allreduce(c)
            xn = torch.empty_like(x)
            if self.constraint == "lasso":
                self.ops.lasso(G, c, x, self.radius, self.cfg, xn, self.inner)
            else:
                self.ops.l1(G, c, x, self.radius, self.cfg, xn, self.inner)
            x = xn
        return x

    def pred_errors(self, X: torch.Tensor, xref: torch.Tensor) -> torch.Tensor:
        """e_k = ||A(X_k - xref)|| / ||A xref|| over all ranks (a7, post hoc)."""
        err2, ref2 = self.ops.err2(self.A, X, xref)
        buf = torch.cat([err2, ref2])
        self.allreduce(buf)
        return torch.sqrt(buf[:-1] / buf[-1])
