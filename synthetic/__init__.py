"""Seeded synthetic inputs for the IHS workloads -- shared by tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no hashing, sketching, Gram,
gradient or solve).  It only draws the problem instances of BASELINE.json's five
configs (DESIGN.md section 5 states the recipe):

  C1 tiny      dense 2000 x 10, iid N(0,1); x* ~ N(0,I); b = A x* + w, w ~ N(0,1)
  C2 dense     dense 2^22 x 128, rows N(0, Sigma), Sigma_ij = 0.5^|i-j| (AR(1) recursion)
  C3 sparse    CSR 2^23 x 1024, iid Bernoulli(1e-3) mask, values N(0,1)
  C4 lasso     dense 2^21 x 256, iid Student-t(3); x* 10-sparse +-1; tau = ||x*||_1
  C5 large     dense 2^25 x 96, iid N(0,1)
  C4P          C4's data with the penalised LASSO, lambda = 5 (NEXT-2)

Every draw comes from a torch.Generator seeded by (config seed, substream), on
the device the caller names.  The same bytes are handed to both the oracle and
the CUDA path by the caller; nothing here depends on either of them.
"""
from __future__ import annotations

import dataclasses
import math

import torch

# substream ids: A, x*, noise, support, csr-structure
_SUB_A, _SUB_X, _SUB_W, _SUB_SUPP, _SUB_CSR = 1, 2, 3, 4, 5


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    layout: str          # "dense" | "csr"
    dist: str            # "normal" | "ar1" | "student_t3"
    family: str          # "countsketch" | "sjlt"
    m: int
    s: int
    T: int               # IHS iterations named by BASELINE.json
    constraint: str      # "ols" | "l1ball" | "lasso" (NEXT-2)
    density: float = 1.0
    sigma: float = 1.0
    sparse_xstar: int = 0
    hash_seed: int = 0
    data_seed: int = 0
    lam: float = 0.0     # l1 penalty of the "lasso" constraint

    def scaled(self, n: int, **kw) -> "Config":
        """Same recipe at a reduced row count (parity-test sizes)."""
        return dataclasses.replace(self, n=n, name=f"{self.name}@n={n}", **kw)

    @property
    def a_bytes(self) -> int:
        if self.layout == "dense":
            return 8 * self.n * self.d
        nnz = self.n * self.d * self.density
        return int(8 * (self.n + 1) + 12 * nnz)


# BASELINE.json configs[0..4]; data seed = config index (1..5), hash seed 0 (reading R14).
CONFIGS = {
    "C1": Config("C1", 2000, 10, "dense", "normal", "countsketch", 200, 1, 10, "ols", data_seed=1),
    "C2": Config("C2", 1 << 22, 128, "dense", "ar1", "countsketch", 1024, 1, 20, "ols", data_seed=2),
    "C3": Config("C3", 1 << 23, 1024, "csr", "normal", "sjlt", 8192, 4, 15, "ols", density=1e-3, data_seed=3),
    "C4": Config("C4", 1 << 21, 256, "dense", "student_t3", "countsketch", 2048, 1, 25, "l1ball",
                 sparse_xstar=10, data_seed=4),
    "C5": Config("C5", 1 << 25, 96, "dense", "normal", "sjlt", 4096, 8, 20, "ols", data_seed=5),
    # NEXT-2: the paper's penalised objective with lambda = 5.0
    # on C4's data (not a BASELINE.json config)
    "C4P": Config("C4P", 1 << 21, 256, "dense", "student_t3", "countsketch", 2048, 1, 25, "lasso",
                  sparse_xstar=10, data_seed=4, lam=5.0),
}


def _gen(cfg: Config, sub: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((cfg.data_seed * 1_000_003 + sub * 7919) & 0x7FFFFFFFFFFFFFFF)
    return g


def _randn(shape, g, device):
    return torch.randn(shape, generator=g, device=device, dtype=torch.float64)


def dense_A(cfg: Config, device="cpu", rows: tuple[int, int] | None = None) -> torch.Tensor:
    """Row-major fp64 A (n x d).  ``rows`` = (begin, end) draws only that row
    block, in chunks whose seeds depend on the chunk index, so any row block is
    reproducible without drawing the whole matrix."""
    r0, r1 = (0, cfg.n) if rows is None else rows
    out = torch.empty((r1 - r0, cfg.d), dtype=torch.float64, device=device)
    CH = 1 << 16
    c0 = r0 // CH
    for c in range(c0, (r1 + CH - 1) // CH):
        lo, hi = c * CH, min((c + 1) * CH, cfg.n)
        g = torch.Generator(device=device)
        g.manual_seed((cfg.data_seed * 1_000_003 + _SUB_A * 7919 + c * 104729) & 0x7FFFFFFFFFFFFFFF)
        blk = _draw_rows(cfg, hi - lo, g, device)
        a, b = max(lo, r0), min(hi, r1)
        out[a - r0:b - r0] = blk[a - lo:b - lo]
    return out


def _draw_rows(cfg: Config, k: int, g, device) -> torch.Tensor:
    if cfg.dist == "normal":
        return _randn((k, cfg.d), g, device)
    if cfg.dist == "ar1":
        # a_1 = z_1, a_j = 0.5 a_{j-1} + sqrt(0.75) z_j  => Cov = 0.5^|i-j| (reading R16)
        z = _randn((k, cfg.d), g, device)
        a = torch.empty_like(z)
        a[:, 0] = z[:, 0]
        c = math.sqrt(0.75)
        for j in range(1, cfg.d):
            a[:, j] = 0.5 * a[:, j - 1] + c * z[:, j]
        return a
    if cfg.dist == "student_t3":
        # t = Z / sqrt(chi2_3 / 3), chi2_3 = sum of three squared normals (reading R17)
        z = _randn((k, cfg.d), g, device)
        q = _randn((3, k, cfg.d), g, device)
        chi2 = (q * q).sum(0)
        return z / torch.sqrt(chi2 / 3.0)
    raise ValueError(cfg.dist)


def x_star(cfg: Config, device="cpu") -> torch.Tensor:
    if cfg.sparse_xstar:
        g = _gen(cfg, _SUB_SUPP, device)
        supp = torch.randperm(cfg.d, generator=g, device=device)[: cfg.sparse_xstar]
        sg = torch.randint(0, 2, (cfg.sparse_xstar,), generator=g, device=device) * 2 - 1
        x = torch.zeros(cfg.d, dtype=torch.float64, device=device)
        x[supp] = sg.to(torch.float64)
        return x
    return _randn((cfg.d,), _gen(cfg, _SUB_X, device), device)


def tau(cfg: Config, device="cpu") -> float:
    """l1-ball radius t = ||x*||_1 (BASELINE.json configs[3])."""
    return float(x_star(cfg, device).abs().sum())


def noise(cfg: Config, device="cpu") -> torch.Tensor:
    return cfg.sigma * _randn((cfg.n,), _gen(cfg, _SUB_W, device), device)


def csr_A(cfg: Config, device="cpu"):
    """CSR A with iid Bernoulli(density) structure (reading R15): per-row count
    ~ Binomial(d, p), distinct uniformly random columns, sorted; values N(0,1).
    Returns (row_ptr int64 [n+1], col int32 [nnz], val f64 [nnz])."""
    g = _gen(cfg, _SUB_CSR, device)
    cnt = torch.binomial(torch.full((cfg.n,), float(cfg.d), dtype=torch.float64, device=device),
                         torch.full((cfg.n,), cfg.density, dtype=torch.float64, device=device),
                         generator=g).to(torch.int64)
    cnt = cnt.clamp_(max=cfg.d)
    row_ptr = torch.zeros(cfg.n + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(cnt, 0)
    nnz = int(row_ptr[-1])
    rows = torch.repeat_interleave(torch.arange(cfg.n, device=device), cnt)
    col = torch.randint(0, cfg.d, (nnz,), generator=g, device=device)
    for _ in range(64):  # redraw within-row duplicates until the columns are distinct
        key = rows * cfg.d + col
        key, order = torch.sort(key)
        col = col[order]
        dup = torch.zeros(nnz, dtype=torch.bool, device=device)
        if nnz > 1:
            dup[1:] = key[1:] == key[:-1]
        nd = int(dup.sum())
        if nd == 0:
            break
        col[dup] = torch.randint(0, cfg.d, (nd,), generator=g, device=device)
    key = rows * cfg.d + col
    key, order = torch.sort(key)
    col = (key % cfg.d).to(torch.int32)
    val = _randn((nnz,), g, device)
    return row_ptr, col, val


def csr_matvec(row_ptr, col, val, x):
    """y = A x for the CSR instance (input generation only: b = A x* + w)."""
    n = row_ptr.numel() - 1
    cnt = row_ptr[1:] - row_ptr[:-1]
    rows = torch.repeat_interleave(torch.arange(n, device=val.device), cnt)
    y = torch.zeros(n, dtype=torch.float64, device=val.device)
    y.index_add_(0, rows, val * x[col.long()])
    return y


def problem(cfg: Config, device="cpu"):
    """Full instance: dict(A or csr, b, x_star, tau)."""
    xs = x_star(cfg, device)
    w = noise(cfg, device)
    out = {"cfg": cfg, "x_star": xs}
    if cfg.layout == "dense":
        A = dense_A(cfg, device)
        out["A"] = A
        out["b"] = A @ xs + w
    else:
        rp, cl, vl = csr_A(cfg, device)
        out["csr"] = (rp, cl, vl)
        out["b"] = csr_matvec(rp, cl, vl, xs) + w
    out["tau"] = float(xs.abs().sum()) if cfg.constraint == "l1ball" else 0.0
    out["lam"] = cfg.lam
    return out
