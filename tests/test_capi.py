"""CPU checks of the C-ABI boundary: the library loads without a GPU, exports
every entry point include/dbp_b200.h declares, and the ctypes argument lists
match the header."""

import os
import re

import pytest

from paper_1808_04473_b200 import _lib

HEADER = os.path.join(os.path.dirname(__file__), os.pardir, "include", "dbp_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(?:int|const char\*)\s+(dbp_\w+)\s*\(([^)]*)\)\s*;", text):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else len(args.split(","))
    return out


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libdbp_b200.so not built (run make)")
    return _lib.load_library()


def test_every_declared_symbol_is_exported(lib):
    fns = header_functions()
    assert len(fns) >= 14
    for name in fns:
        assert hasattr(lib, name), name


def test_ctypes_signatures_match_header():
    fns = header_functions()
    assert set(fns) == set(_lib.SIGNATURES)
    for name, nargs in fns.items():
        assert len(_lib.SIGNATURES[name]) == nargs, (name, nargs, len(_lib.SIGNATURES[name]))


def test_abi_version_and_errors_without_gpu(lib):
    assert lib.dbp_abi_version() == _lib.ABI_VERSION
    # argument validation happens before any CUDA call
    rc = lib.dbp_equalize(9, 0, None, None, 1, 2, 2, 2, 1, 1, None, None, 0, 0.0, None, 1, 1.0, 0, 0.0, 1.0, 1,
                          1.0, None, 0, None, 0, None, None, None, None, None, None, None, None, None, None)
    assert rc == -1
    assert b"architecture" in lib.dbp_last_error()
    # empty batches are a no-op
    assert lib.dbp_gram_mrc(None, None, 0, 2, 2, 2, 1, 1, None, 1, None, None) == 0


def test_product_path_fails_loudly_without_gpu():
    import torch

    import paper_1808_04473_b200 as dbp

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(dbp.BackendError):
        dbp.local_preprocess([[1.0, 0.0], [0.0, 1.0]], [1.0, 2.0])
    with pytest.raises(dbp.BackendError):
        dbp.kernels.backend()
