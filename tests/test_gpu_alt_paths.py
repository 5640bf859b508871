"""The alternative kernels selected by IHS_* environment switches (DESIGN.md
section 1: measured slower, kept for comparison) stay parity-correct.  Each
switch set runs tests/alt_paths_check.py in a fresh process (the library reads
the switches once per process)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

SETS = {
    "stream_ldg_chol_plain": {"IHS_SJLT": "stream", "IHS_GATHER": "ldg", "IHS_OLS": "chol", "IHS_PG_PLAIN": "1",
                              "IHS_PG_WARM": "0", "IHS_PREFETCH": "0"},
    "tile_async_pgcta": {"IHS_SJLT": "tile", "IHS_GATHER": "async", "IHS_PG_CTA": "1", "IHS_FUSE": "1"},
    "gather_shapes_nohints": {"IHS_GATHER_CW": "1", "IHS_GATHER_ROWS": "8", "IHS_GATHER_HINT": "0",
                              "IHS_SCATTER_KEEP": "0"},
    "gather_rows8": {"IHS_GATHER_ROWS": "8"},
    "pg_single": {"IHS_PG_SINGLE": "1", "IHS_PREFETCH_ORDER": "before", "IHS_PG_THETA_WARM": "0"},
    "lookahead": {"IHS_LOOKAHEAD": "1", "IHS_LOOKAHEAD_CLUSTER": "4"},
}


@pytest.mark.parametrize("name", sorted(SETS))
def test_alt_paths(name):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, **SETS[name])
    r = subprocess.run([sys.executable, os.path.join(HERE, "alt_paths_check.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
