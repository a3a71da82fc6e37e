"""ctypes binding of libdbp_b200.so (include/dbp_b200.h).

The library is loaded lazily on first use.  There is no CPU fallback: a
missing library, a machine without a CUDA device or a failed launch raise
:class:`BackendError`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import BackendError

_HERE = os.path.dirname(os.path.abspath(__file__))
# DBP_LIB: alternative build of the same library (A/B timing studies only)
LIB_PATH = os.environ.get("DBP_LIB") or os.path.join(_HERE, "libdbp_b200.so")
ABI_VERSION = 1

# status codes (include/dbp_b200.h)
ST_OK, ST_SINGULAR, ST_NEGVAR, ST_DIVERGED, ST_BADVAR = 0, 1, 2, 3, 4
KIND = {"mrc": 0, "zf": 1, "lmmse": 2, "lama": 3}
ARCH_PD, ARCH_FD, ARCH_FD_PARTIAL = 1, 2, 3
# fused kernels (dbp_last_kernel / DBP_OPT_KERNEL)
KERNEL_AUTO, KERNEL_SIMT, KERNEL_TC_TF32, KERNEL_TC_BF16 = 0, 1, 2, 3
# dbp_set_option keys
OPTIONS = {"kernel": 0, "tc_smax_kb": 1, "tc_ns": 2, "tc_pair": 3, "tc_nsolv": 4, "simt_ns": 5,
           "no_wide": 6, "t2_nsplit": 7, "t2_quad": 8, "wide_chunk": 9, "lama_kernel": 10}

_vp, _fp, _i32p, _u8p = C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p
_i64, _i, _f = C.c_int64, C.c_int, C.c_float

# name -> argtypes (pointers to host parameter arrays are passed as c_void_p)
SIGNATURES = {
    "dbp_abi_version": [],
    "dbp_last_error": [],
    "dbp_last_kernel": [],
    "dbp_set_option": [_i, _i],
    "dbp_device_query": [_vp, _vp, _vp, _vp],
    "dbp_gram_mrc": [_vp, _vp, _i64, _i, _i, _i, _i, _i, _vp, _i, _vp, _vp],
    "dbp_gram_mrc_parts": [_vp, _vp, _i64, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, _vp],
    "dbp_equalize_stats": [_vp, _i64, _i, _i, _i, _f, _vp, _i64, _f, _i, _f, _f, _i, _f,
                           _vp, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "dbp_equalize": [_i, _i, _vp, _vp, _i64, _i, _i, _i, _i, _i, _vp, _vp, _i, _f, _vp, _i64,
                     _f, _i, _f, _f, _i, _f, _vp, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                     _vp, _vp, _vp],
    "dbp_fd_finalize": [_vp, _i64, _i, _i, _i, _vp, _i, _vp, _i, _vp, _vp, _vp, _vp],
    "dbp_fd_weights": [_vp, _vp, _i64, _i, _i, _vp, _vp],
    "dbp_posterior": [_vp, _i64, _f, _vp, _i, _vp, _vp, _vp],
    "dbp_hard_detect": [_vp, _i64, _vp, _i, _vp, _vp],
    "dbp_stats_sum": [_vp, _i, _i64, _vp, _vp],
    "dbp_unbias": [_vp, _vp, _vp, _i64, _i, _i, _f, _vp, _vp, _vp, _vp],
    "dbp_fusion_weights": [_vp, _i64, _i, _i, _vp, _vp, _vp],
    "dbp_fuse_estimates": [_vp, _vp, _vp, _i, _i64, _vp, _vp, _vp],
    "dbp_llr": [_vp, _vp, _i64, _i, _i, _i, _vp, _i, _i, _vp, _vp],
    "dbp_gray_bits": [_vp, _i, _i64, _i, _vp, _vp],
    "dbp_quadrature": [_i, _vp, _i64, _vp, _i, _vp, _vp, _i, _vp, _vp],
    "dbp_fixed_point": [_i, _vp, _vp, _vp, _vp, _i64, _vp, _i, _vp, _vp, _i, C.c_double, _i, _vp, _vp, _vp],
    "dbp_comm_unique_id": [_vp],
    "dbp_comm_init": [_vp, _i, _i, _vp],
    "dbp_comm_destroy": [_vp],
    "dbp_pd_reduce_scatter": [_vp, _vp, _vp, _i64, _i, _i, _vp],
    "dbp_fd_reduce_scatter": [_vp, _vp, _vp, _i64, _i, _i, _i, _vp],
    "dbp_allreduce_sum": [_vp, _vp, _i64, _vp],
    "dbp_synthesize": [C.c_uint64, _i64, _i64, _i, _i, _i, _vp, _i, _f, _vp, _i64, _vp, _vp, _vp, _vp],
}

_lock = threading.Lock()
_lib = None


def load_library(path=LIB_PATH):
    """Load the shared library and declare every exported signature (no GPU
    needed for this step)."""
    if not os.path.exists(path):
        raise BackendError(
            f"{path} not found: build it with `make` (or __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = C.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_char_p if name == "dbp_last_error" else C.c_int
    if lib.dbp_abi_version() != ABI_VERSION:
        raise BackendError("libdbp_b200.so ABI version mismatch; rebuild")
    return lib


def lib():
    """The loaded library, after checking that a CUDA device is present."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch

                if not torch.cuda.is_available():
                    raise BackendError("no CUDA device: the sm_100a path has no CPU fallback")
                _lib = load_library()
    return _lib


def check(rc):
    if rc != 0:
        msg = lib().dbp_last_error().decode(errors="replace")
        raise BackendError(f"libdbp_b200 error {rc}: {msg}")


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def host_f32(values):
    """Keep a host float32 parameter array alive and return (array, ptr)."""
    import numpy as np

    arr = np.ascontiguousarray(np.asarray(values, dtype=np.float32).reshape(-1))
    return arr, (arr.ctypes.data_as(C.c_void_p) if arr.size else None)


def host_i32(values):
    import numpy as np

    arr = np.ascontiguousarray(np.asarray(values, dtype=np.int32).reshape(-1))
    return arr, arr.ctypes.data_as(C.c_void_p)


class options:
    """Context manager over dbp_set_option (kernel selection and staging
    overrides for tests and A/B studies), e.g.
    ``with _lib.options(kernel=KERNEL_SIMT): ...``.  Restores the previous
    values on exit."""

    def __init__(self, **kw):
        unknown = set(kw) - set(OPTIONS)
        if unknown:
            raise ValueError(f"unknown options {sorted(unknown)}")
        self.kw = kw
        self.prev = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.prev[k] = lib().dbp_set_option(OPTIONS[k], int(v))
        return self

    def __exit__(self, *exc):
        for k, v in self.prev.items():
            lib().dbp_set_option(OPTIONS[k], v)
        return False
