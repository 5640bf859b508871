"""CPU checks of the boundary: libihs.so loads, exports every symbol include/ihs.h
declares, and fails loudly (no fallback) without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    from paper_1910_14166_b200 import build
    build.build()
    import paper_1910_14166_b200 as P
    return P


def header_symbols():
    with open(os.path.join(ROOT, "include", "ihs.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int64_t|int|ihs_status)\s+(ihs_\w+)\s*\(", text, re.M)))


def test_header_declares_the_north_star_calls():
    syms = header_symbols()
    for name in ("ihs_sketch", "ihs_gram", "ihs_grad", "ihs_solve_ols", "ihs_solve_l1ball", "ihs_hash"):
        assert name in syms


def test_library_exports_every_header_symbol(built):
    lib = ctypes.CDLL(built.LIB_PATH)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(header_symbols()) <= set(built._EXPORTS)


def test_abi_version_and_status_strings(built):
    L = built.lib()
    assert L.ihs_abi_version() == built.ABI_VERSION
    assert L.ihs_status_string(built.ERR_NOT_SPD) == b"Hessian sketch not positive definite"
    assert L.ihs_status_string(0) == b"ok"


def test_no_gpu_means_loud_failure(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = built.lib().ihs_ctx_create(ctypes.byref(h), 0, None)
    assert st == built.ERR_CUDA


def test_product_never_imports_oracle():
    """The product package and bench.py's product leg must not touch oracle/."""
    pkg = os.path.join(ROOT, "paper_1910_14166_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "ihs_oracle" not in src, f
