"""NEXT-3: the Appendix B sketch-quality / sketch-time sweep
(Appendix B): the mean empirical sketch error
``||A^T S^T S A - A^T A||_F / ||A^T A||_F`` and the sketch time over ten
independent sketches, for CountSketch and the SJLT (column sparsities s = 1
and s = 4), at projection dimension m = gamma d (
"RP(gamma)").

Every sketch and Gram runs in libihs.so (ihs_sketch / ihs_gram through the C
ABI); torch only holds the arrays and takes the Frobenius norm of the
difference, which is bookkeeping of the experiment, not part of the IHS path.
For SJLT, m is rounded up to a multiple of s (the SJLT needs s | m).
"""
from __future__ import annotations

import math
import statistics

import torch

import paper_1910_14166_b200 as P


def exact_gram(A, ctx=None) -> torch.Tensor:
    """A^T A on the DMMA Gram kernel (CSR is densified on the device first)."""
    if isinstance(A, P.Csr):
        dense = torch.zeros((A.n, A.d), dtype=torch.float64, device=A.device)
        cnt = A.row_ptr[1:] - A.row_ptr[:-1]
        rows = torch.repeat_interleave(torch.arange(A.n, device=A.device), cnt)
        dense[rows, A.col.long()] = A.val
        A = dense
    elif isinstance(A, P.Dense):
        A = A.A
    return P.ihs_gram(A, ctx=ctx)


def sketch_quality(A, family: str, s: int, gammas, trials: int = 10, seed: int = 0, G=None, ctx=None):
    """[{gamma, m, s, family, err_mean, err_std, errs, ms_mean, ms_std}] over `trials`
    independent sketches (hash iterations 0..trials-1 of `seed`)."""
    A = P.as_matrix(A)
    ctx = ctx or P.default_context(A.device)
    G = exact_gram(A, ctx) if G is None else G
    gn = float(torch.linalg.norm(G))
    out = []
    stream = torch.cuda.current_stream(A.device)
    for gamma in gammas:
        m = int(math.ceil(gamma * A.d / s) * s)
        spec = P.Spec(m=m, s=s, seed=seed)
        errs, ms = [], []
        for t in range(trials):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            SA = P.ihs_sketch(A, spec, t, ctx=ctx)
            e1.record(stream)
            H = P.ihs_gram(SA, ctx=ctx)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
            errs.append(float(torch.linalg.norm(H - G)) / gn)
        out.append({"family": family, "s": s, "gamma": gamma, "m": m, "err_mean": statistics.mean(errs),
                    "err_std": statistics.pstdev(errs), "errs": errs, "ms_mean": statistics.mean(ms[1:] or ms),
                    "ms_std": statistics.pstdev(ms[1:] or ms), "rows_per_s": A.n / (statistics.mean(ms[1:] or ms) / 1e3)})
    return out
