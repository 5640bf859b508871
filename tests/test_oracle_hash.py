"""Pins for the oracle's counter hash (step a1; reading R1 in DESIGN.md).

The hash is a *definition* (the paper draws h, sigma uniformly at random,
PAPER.md:175-184), so it is pinned by: the published splitmix64 test vector,
values of the definition reproduced independently before this repo existed
(SURVEY.md section 8(c)), and the statistical / structural properties the paper
requires of CountSketch and SJLT.
"""
import numpy as np
import pytest
from scipy import stats


def test_splitmix64_published_stream(oracle_mod, golden):
    kat = golden("splitmix64_kat.json")
    gamma = 0x9E3779B97F4A7C15
    # stream from state 0: the k-th output is SM(k * gamma) (state advances by gamma)
    got = [oracle_mod.splitmix64((k * gamma) & 0xFFFFFFFFFFFFFFFF) for k in range(3)]
    assert got == [int(v, 16) for v in kat["state0_stream"]]


def test_iter_key_and_hash_kat(oracle_mod, golden):
    kat = golden("hash_kat.json")
    assert oracle_mod.iter_key(0, 0) == int(kat["iter_key"]["seed0_t0"], 16)
    assert oracle_mod.iter_key(0, 1) == int(kat["iter_key"]["seed0_t1"], 16)
    for t in (0, 1):
        ref = kat["countsketch_m200"][f"t{t}"]
        b, s = oracle_mod.hash_rows(0, t, 200, 1, 0, 6)
        assert b[:, 0].tolist() == ref["bucket"]
        assert s[:, 0].tolist() == ref["sign"]
    b, s = oracle_mod.hash_rows(0, 0, 8192, 4, 0, 2)
    for r in (0, 1):
        ref = kat["sjlt_m8192_s4_t0"][f"row{r}"]
        assert b[r].tolist() == ref["bucket"]
        assert s[r].tolist() == ref["sign"]


def test_row_offsets_are_global(oracle_mod):
    """hash depends on the global row index only: any sub-range reproduces the slice."""
    b, s = oracle_mod.hash_rows(7, 3, 1000, 4, 0, 5000)
    b2, s2 = oracle_mod.hash_rows(7, 3, 1000, 4, 1234, 777)
    np.testing.assert_array_equal(b[1234:1234 + 777], b2)
    np.testing.assert_array_equal(s[1234:1234 + 777], s2)


def test_sjlt_s1_is_countsketch(oracle_mod):
    """SJLT with s = 1 is a CountSketch."""
    b1, s1 = oracle_mod.hash_rows(0, 5, 333, 1, 0, 4000)
    assert b1.min() >= 0 and b1.max() < 333
    assert set(np.unique(s1).tolist()) == {-1, 1}


def test_sjlt_block_structure(oracle_mod):
    """SJLT: one nonzero per block of m/s rows in every column."""
    m, s = 4096, 8
    b, _ = oracle_mod.hash_rows(0, 2, m, s, 0, 20000)
    M = m // s
    for j in range(s):
        assert (b[:, j] // M == j).all()


@pytest.mark.parametrize("m,s", [(200, 1), (1024, 1), (4096, 8)])
def test_bucket_uniformity_and_sign_balance(oracle_mod, m, s):
    """Buckets uniform over each block (chi^2) and signs fair (binomial z)."""
    n = 200_000
    b, sg = oracle_mod.hash_rows(0, 0, m, s, 0, n)
    M = m // s
    for j in range(s):
        counts = np.bincount(b[:, j] - j * M, minlength=M)
        chi2 = ((counts - n / M) ** 2 / (n / M)).sum()
        p = stats.chi2.sf(chi2, M - 1)
        assert p > 1e-4, (j, chi2, p)
    z = sg.sum() / np.sqrt(sg.size)
    assert abs(z) < 4.5
    # independence of sign and bucket parity (a dropped/shared bit would fail this)
    par = (b[:, 0] & 1) * 2 - 1
    corr = (par * sg[:, 0]).sum() / np.sqrt(n)
    assert abs(corr) < 4.5


def test_iterations_and_seeds_draw_fresh_sketches(oracle_mod):
    """A fresh S every iteration (Theorem 1 'for every iteration')."""
    b0, _ = oracle_mod.hash_rows(0, 0, 1024, 1, 0, 5000)
    b1, _ = oracle_mod.hash_rows(0, 1, 1024, 1, 0, 5000)
    b2, _ = oracle_mod.hash_rows(1, 0, 1024, 1, 0, 5000)
    assert (b0 != b1).mean() > 0.99
    assert (b0 != b2).mean() > 0.99
    # agreement rate of two independent uniform draws ~ 1/m
    assert (b0 == b1).mean() < 5.0 / 1024
