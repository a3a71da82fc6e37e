"""Soft outputs: Gray-labelled bit LLRs from the equalizer's (x-hat, sigma2)
(SURVEY.md §8(f) rank 3 -- the paper's downstream use; the
reference itself stops at symbol decisions, equalize.py:262-268).

Model: the decoupled channel x = s + e, e ~ CN(0, sigma2) the equalizer
reports (unbiased linear outputs, or LAMA's z with tau).  Labels are
``model.gray_labels``: symbol k = i*L + j carries (gray(i) << log2 L) |
gray(j), bits MSB first.  LLR = log P(b=0 | x) / P(b=1 | x); ``exact``
selects log-sum-exp over the symbols instead of max-log.  Computed by the
``dbp_llr`` kernel (one thread per symbol, per-dimension factorisation).

``gray_bits`` gives the hard counterpart: the Gray bits of symbol decisions
(``Detection.decisions`` or ``hard_detect_index``), ``dbp_gray_bits``.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib
from .errors import ConfigError, DimensionMismatchError


def llr(xhat, sigma2, constellation, exact=False):
    """Bit LLRs [..., T, U, 2 log2 L] of x-hat [..., T, U].  ``sigma2``:
    per UE [..., U] (linear equalizers) or per symbol [..., T] (LAMA).
    Host arrays in -> NumPy out; CUDA tensors in -> CUDA tensor out."""
    if not getattr(constellation, "is_square_qam", False):
        raise ConfigError("bit LLRs need a square QAM constellation")
    L = len(constellation.pam_levels)
    nbits = 2 * int(round(np.log2(L)))
    x, host = _dev.to_c64(xhat)
    s2, _ = _dev.to_f32(sigma2)
    if x.dim() < 2:
        raise DimensionMismatchError("xhat must be [..., T, U]")
    T, u = x.shape[-2], x.shape[-1]
    lead = tuple(x.shape[:-2])
    n = int(np.prod(lead)) if lead else 1
    if tuple(s2.shape) == lead + (u,):
        per_symbol = 0
    elif tuple(s2.shape) == lead + (T,):
        per_symbol = 1
    else:
        raise DimensionMismatchError("sigma2 must be [..., U] or [..., T]")
    out = _dev.empty_f32(lead + (T, u, nbits))
    lv, lp = _lib.host_f32(constellation.pam_levels)
    _lib.check(_lib.lib().dbp_llr(_lib.ptr(x), _lib.ptr(s2), n, T, u, per_symbol, lp, L, int(bool(exact)),
                                  _lib.ptr(out), _lib.stream_ptr()))
    return _dev.out(out, host, real=True)


def gray_bits(decisions, constellation):
    """Hard Gray bits [..., 2 log2 L] (uint8 0/1, MSB first) of symbol indices
    (k = i*L + j; uint8 detector decisions or int32/int64 hard_detect_index
    output).  Host arrays in -> NumPy out; CUDA tensors in -> CUDA tensor out."""
    if not getattr(constellation, "is_square_qam", False):
        raise ConfigError("Gray bits need a square QAM constellation")
    t = _dev.torch()
    L = len(constellation.pam_levels)
    nbits = 2 * int(round(np.log2(L)))
    _lib.lib()
    host = not _dev.is_device(decisions)
    d = decisions if isinstance(decisions, t.Tensor) else t.from_numpy(np.ascontiguousarray(decisions))
    if d.dtype == t.uint8:
        idx, width = d.to("cuda").contiguous(), 1
    elif d.dtype in (t.int32, t.int64, t.int16):
        idx, width = d.to(device="cuda", dtype=t.int32).contiguous(), 4
    else:
        raise ConfigError("decisions must be integer symbol indices")
    out = t.empty(tuple(idx.shape) + (nbits,), dtype=t.uint8, device="cuda")
    _lib.check(_lib.lib().dbp_gray_bits(_lib.ptr(idx), width, idx.numel(), L, _lib.ptr(out), _lib.stream_ptr()))
    return out.cpu().numpy() if host else out
