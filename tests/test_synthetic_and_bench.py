"""Host-side logic (no GPU): the synthetic input recipes (DESIGN.md section 5,
readings R14-R17) and bench.py's roofline arithmetic and JSON contract pieces."""
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_baseline_configs_match_the_recipes():
    c = synthetic.CONFIGS
    assert (c["C1"].n, c["C1"].d, c["C1"].m, c["C1"].T) == (2000, 10, 200, 10)
    assert (c["C2"].n, c["C2"].d, c["C2"].m, c["C2"].dist) == (1 << 22, 128, 1024, "ar1")
    assert (c["C3"].n, c["C3"].d, c["C3"].m, c["C3"].s, c["C3"].layout) == (1 << 23, 1024, 8192, 4, "csr")
    assert (c["C4"].n, c["C4"].d, c["C4"].m, c["C4"].constraint) == (1 << 21, 256, 2048, "l1ball")
    assert (c["C5"].n, c["C5"].d, c["C5"].m, c["C5"].s) == (1 << 25, 96, 4096, 8)
    assert c["C4P"].constraint == "lasso" and c["C4P"].lam == 5.0
    assert c["C5"].a_bytes == 8 * (1 << 25) * 96


def test_row_blocks_are_reproducible_without_the_whole_matrix():
    cfg = synthetic.CONFIGS["C2"].scaled(200_000)
    full = synthetic.dense_A(cfg)
    for r0, r1 in [(0, 1), (65_535, 65_537), (131_000, 200_000), (77, 77)]:
        assert torch.equal(synthetic.dense_A(cfg, rows=(r0, r1)), full[r0:r1])


def test_ar1_rows_have_the_toeplitz_covariance():
    """R16: a_1 = z_1, a_j = 0.5 a_{j-1} + sqrt(0.75) z_j  =>  Cov_ij = 0.5^|i-j|."""
    cfg = synthetic.Config("t", 400_000, 6, "dense", "ar1", "countsketch", 8, 1, 1, "ols", data_seed=3)
    A = synthetic.dense_A(cfg).numpy()
    emp = A.T @ A / A.shape[0]
    ref = 0.5 ** np.abs(np.subtract.outer(np.arange(6), np.arange(6)))
    assert np.abs(emp - ref).max() < 0.01


def test_student_t3_tails():
    """R17: t_3 has variance 3 and heavy tails (P(|t| > 10) ~ 2e-3)."""
    cfg = synthetic.Config("t", 200_000, 5, "dense", "student_t3", "countsketch", 8, 1, 1, "ols", data_seed=4)
    A = synthetic.dense_A(cfg).numpy().ravel()
    assert abs(np.median(A)) < 0.01
    assert 0.0015 < (np.abs(A) > 10).mean() < 0.0030  # exact: 1.92e-3


def test_csr_recipe():
    """R15: iid Bernoulli(p) mask -> Binomial(d, p) per row, distinct sorted columns."""
    cfg = synthetic.Config("t", 50_000, 300, "csr", "normal", "sjlt", 64, 4, 1, "ols", density=0.01, data_seed=5)
    rp, cl, vl = synthetic.csr_A(cfg)
    rp, cl = rp.numpy(), cl.numpy()
    cnt = np.diff(rp)
    assert abs(cnt.mean() - 3.0) < 0.05 and abs(cnt.var() - 300 * 0.01 * 0.99) < 0.1
    for i in range(0, 50_000, 997):
        row = cl[rp[i]:rp[i + 1]]
        assert (np.diff(row) > 0).all() and (row < 300).all()
    assert vl.dtype == torch.float64 and abs(float(vl.std()) - 1.0) < 0.02


def test_c4_xstar_and_radius():
    cfg = synthetic.CONFIGS["C4"]
    xs = synthetic.x_star(cfg).numpy()
    assert (xs != 0).sum() == 10 and set(np.abs(xs[xs != 0])) == {1.0}
    assert synthetic.tau(cfg) == 10.0


# ------------------------------------------------------------------ bench.py helpers
def test_roofline_arithmetic():
    import bench
    cfg = synthetic.CONFIGS["C2"]
    n = cfg.n
    prof = {"sketch": (7.5, 10), "sort": (0.9, 10), "chol": (0.5, 10)}
    r = bench.roofline(prof, cfg, n, None, steps=10)
    alg = 8 * n * cfg.d + 12 * n + 8 * cfg.m * cfg.d + 8 * cfg.m * cfg.d
    assert r["kernel_group"] == "sketch" and r["bound"] == "hbm"
    assert math.isclose(r["algorithmic_bytes_per_launch"], alg)
    assert math.isclose(r["achieved"], alg / 0.75e-3 / 1e9)
    assert math.isclose(r["frac"], r["achieved"] / r["peak"])
    # SJLT: A counted once although the design reads it s times
    c5 = synthetic.CONFIGS["C5"]
    r5 = bench.roofline({"sketch": (40.0, 4)}, c5, c5.n, None, steps=1)
    assert math.isclose(r5["algorithmic_bytes_per_launch"] * 4,
                        8 * c5.n * c5.d + 12 * c5.n + 8 * (c5.m // c5.s) * c5.d + 8 * c5.m * c5.d)
    # CSR: s reductions per nonzero against the measured L2 RED throughput
    c3 = synthetic.CONFIGS["C3"]
    r3 = bench.roofline({"csr": (3.3, 10)}, c3, c3.n, 8_600_000, steps=10)
    assert r3["bound"] == "l2_red" and math.isclose(r3["achieved"], 4 * 8_600_000 / 0.33e-3 / 1e9)


def test_reference_arm_json_contract(tmp_path):
    """--impl reference (the oracle on the host) prints the
    base contract's line with impl/cpu_baseline/e2e."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
