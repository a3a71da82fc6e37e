"""Device-buffer plumbing for the drop-in API: host arrays are uploaded as
complex64 / float32 torch CUDA tensors, CUDA tensors are used in place, and
results go back in the caller's flavour (NumPy complex128 / float64 for host
inputs, torch CUDA tensors for device inputs)."""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import (
    ConfigError,
    DimensionMismatchError,
    DivergenceError,
    NegativeVarianceError,
    SingularGramError,
)


def torch():
    import torch as _t

    return _t


def is_device(x):
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def to_c64(x):
    """-> (contiguous complex64 CUDA tensor, was_host)."""
    _lib.lib()  # no device / no library -> BackendError before any upload
    t = torch()
    if isinstance(x, t.Tensor):
        host = not x.is_cuda
        y = x.to(device="cuda", dtype=t.complex64).contiguous()
        return y, host
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.complex64))
    return t.from_numpy(arr).to("cuda"), True


def to_f32(x):
    _lib.lib()
    t = torch()
    if isinstance(x, t.Tensor):
        return x.to(device="cuda", dtype=t.float32).contiguous(), not x.is_cuda
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    return t.from_numpy(arr).to("cuda"), True


def empty_c64(shape):
    t = torch()
    return t.empty(tuple(shape), dtype=t.complex64, device="cuda")


def empty_f32(shape):
    t = torch()
    return t.empty(tuple(shape), dtype=t.float32, device="cuda")


def zeros_i32(shape):
    t = torch()
    return t.zeros(tuple(shape), dtype=t.int32, device="cuda")


def out(t_, host, real=False):
    """Return a result tensor in the caller's flavour."""
    if not host:
        return t_
    a = t_.cpu().numpy()
    return a.astype(np.float64 if real else np.complex128)


def raise_status(status, iters=None, what=""):
    """Map the first non-zero per-item status onto the reference's exception
    types (errors.py), as the reference raises on its first failure."""
    st = status.cpu().numpy().reshape(-1)
    bad = np.flatnonzero(st)
    if bad.size == 0:
        return
    i = int(bad[0])
    code = int(st[i])
    where = f"{what} (item {i})" if st.size > 1 else what
    if code == _lib.ST_SINGULAR:
        raise SingularGramError(f"{where}: Gram matrix / signal gain is singular")
    if code == _lib.ST_NEGVAR:
        raise NegativeVarianceError(f"{where}: negative error variance")
    if code == _lib.ST_DIVERGED:
        it = None
        if iters is not None:
            it = int(iters.cpu().numpy().reshape(-1)[i])
        raise DivergenceError(f"{where}: non-finite iterate at t={it}", iteration=it)
    if code == _lib.ST_BADVAR:
        raise ConfigError(f"{where}: fusion weights need strictly positive variances")
    raise DimensionMismatchError(f"{where}: unknown status {code}")


def const_params(constellation):
    """(levels array+ptr, L, symbols array+ptr, M) of a constellation for
    the C ABI; PAM levels only for square-QAM layouts."""
    levels = constellation.pam_levels if getattr(constellation, "is_square_qam", False) else None
    if levels is None:
        lv, lp, L = None, None, 0
    else:
        lv, lp = _lib.host_f32(levels)
        L = len(levels)
    syms = np.asarray(constellation.symbols, dtype=np.complex128)
    sv, sp = _lib.host_f32(np.stack([syms.real, syms.imag], axis=1))
    return (lv, lp, L, sv, sp, syms.size)


def symbols_params(symbols):
    syms = np.asarray(symbols, dtype=np.complex128).reshape(-1)
    sv, sp = _lib.host_f32(np.stack([syms.real, syms.imag], axis=1))
    return sv, sp, syms.size


def pad_even_u(h):
    """Channel tensor [..., B, U] -> (tensor with an even column stride, u_stride)."""
    u = h.shape[-1]
    if u % 2 == 0:
        return h, u
    return _pad_last(h, u + 1), u + 1


def _pad_last(h, new_u):
    t = torch()
    out_ = t.zeros(h.shape[:-1] + (new_u,), dtype=h.dtype, device=h.device)
    out_[..., : h.shape[-1]] = h
    return out_


def pad_clusters(h, y, counts):
    """Zero-pad every cluster to an even row count (zero rows add nothing to
    the Gram or the matched filter).  h [n][B][us], y [n][T][B]."""
    counts = [int(c) for c in counts]
    if all(c % 2 == 0 for c in counts):
        off = np.concatenate(([0], np.cumsum(counts)))
        return h, y, off
    t = torch()
    padded = [c + (c % 2) for c in counts]
    off_new = np.concatenate(([0], np.cumsum(padded)))
    off_old = np.concatenate(([0], np.cumsum(counts)))
    hn = t.zeros((h.shape[0], int(off_new[-1]), h.shape[2]), dtype=h.dtype, device=h.device)
    yn = t.zeros((y.shape[0], y.shape[1], int(off_new[-1])), dtype=y.dtype, device=y.device)
    for c in range(len(counts)):
        a, b = int(off_old[c]), int(off_old[c + 1])
        a2 = int(off_new[c])
        hn[:, a2:a2 + (b - a)] = h[:, a:b]
        yn[:, :, a2:a2 + (b - a)] = y[:, :, a:b]
    return hn, yn, off_new
