"""The reference's kernel seam (kernels.py) bound to the sm_100a library.

``backend()`` names the active implementation; ``posterior_mean_var`` is the
hot-path denoiser (kernels.py:41-50 -> _kernels.pyx:19-71).  The reference's
Gauss-Hermite quadratures (lama_mse, lama_mse_pam, mi_awgn) belong to the
large-system analysis, which is out of scope for this build.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib

BACKEND = "cuda-sm_100a"


def backend():
    """Name of the active kernel implementation.  Loading the library here
    makes a missing build or a missing GPU fail loudly."""
    _lib.lib()
    return BACKEND


def posterior_mean_var(z, tau, symbols):
    """Entry-wise posterior mean F and variance G of a uniform prior over
    ``symbols`` observed through CN(z, tau); preserves the shape of z."""
    zd, host = _dev.to_c64(z)
    shape = tuple(zd.shape)
    flat = zd.reshape(-1)
    f = _dev.empty_c64(flat.shape)
    g = _dev.empty_f32(flat.shape)
    sv, sp, M = _dev.symbols_params(symbols)
    lib = _lib.lib()
    _lib.check(lib.dbp_posterior(_lib.ptr(flat), flat.numel(), float(tau), sp, M, _lib.ptr(f), _lib.ptr(g),
                                 _lib.stream_ptr()))
    del sv
    f = f.reshape(shape)
    g = g.reshape(shape)
    if host:
        return f.cpu().numpy().astype(np.complex128), g.cpu().numpy().astype(np.float64)
    return f, g
