"""The alternative paths selected by per-context options (ihs_ctx_set_option;
DESIGN.md section 1: measured slower, or certified-exact variants) stay
parity-correct: tests/alt_paths_check.py on a context with each option set."""
import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

SETS = {
    "passes_cholesky_nowarm_noprefetch": {"sjlt_onepass": 0, "ols_large": 2, "pg_warm": 0, "prefetch": 0},
    "cg_only_fuse128": {"ols_large": 0, "fuse_max_d": 128},
    "no_fuse": {"fuse_max_d": 0},
    "lookahead": {"lookahead": 1},
    "plain": {"lookahead": 0},
}


@pytest.mark.parametrize("name", sorted(SETS))
def test_alt_paths(name):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import alt_paths_check
    import paper_1910_14166_b200 as P
    ctx = P.Context(0)
    for k, v in SETS[name].items():
        ctx.set_option(k, v)
    alt_paths_check.main(ctx)
