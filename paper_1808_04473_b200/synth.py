"""Seeded synthetic uplink frames with the BASELINE.json shapes.

Stand-in for the paper's LTE/WINNER-II data (not available, and not used by
BASELINE.json): i.i.d. Rayleigh channels CN(0, 1/B) constant over the T OFDM
symbols of a subcarrier, uniform symbol indices over a unit-energy square QAM,
and CN(0, N0) noise with N0 = Es * 10^(-SNR/10) (montecarlo.py:155-156).

Draw order follows the reference's ``run_trial`` (montecarlo.py:154-160):
channel, then symbols, then noise, with CN(0, v) = sqrt(v/2) (N + jN)
(model.py:207-211).  One generator per frame,
``default_rng(SeedSequence((seed, frame)))``, draws the whole frame at once:
H [W][B][U], symbol indices [W][T][U], noise [W][T][B].  Inputs are rounded
to complex64; parity checks feed the *rounded* values to the CPU oracle.
"""

from __future__ import annotations

import numpy as np

from .model import make_constellation


def snr_to_n0(snr_db, es=1.0):
    """N0 = Es / 10^(SNR/10) (montecarlo.py:155-156)."""
    return es / (10.0 ** (np.asarray(snr_db, dtype=float) / 10.0))


def synth_frames(seed, frames, w, t, b, u, constellation="qam16", snr_db=10.0):
    """Return (H [F*W][B][U] c64, Y [F*W][T][B] c64, sym_idx [F*W][T][U] u8,
    n0 [F] f64).  ``snr_db`` may be a scalar or one value per frame."""
    const = (make_constellation(constellation)
             if isinstance(constellation, str) else constellation)
    snr = np.broadcast_to(np.asarray(snr_db, dtype=float), (frames,))
    n0 = snr_to_n0(snr, const.es)
    H = np.empty((frames * w, b, u), dtype=np.complex64)
    Y = np.empty((frames * w, t, b), dtype=np.complex64)
    S = np.empty((frames * w, t, u), dtype=np.uint8)
    m = const.size
    for f in range(frames):
        rng = np.random.default_rng(np.random.SeedSequence((int(seed), f)))
        sc = np.sqrt(1.0 / b / 2.0)
        h = sc * (rng.standard_normal((w, b, u)) + 1j * rng.standard_normal((w, b, u)))
        idx = rng.integers(0, m, size=(w, t, u))
        sn = np.sqrt(n0[f] / 2.0)
        noise = sn * (rng.standard_normal((w, t, b)) + 1j * rng.standard_normal((w, t, b)))
        y = np.einsum("wbu,wtu->wtb", h, const.symbols[idx]) + noise
        sl = slice(f * w, (f + 1) * w)
        H[sl] = h
        Y[sl] = y
        S[sl] = idx
    return H, Y, S, n0


def synth_device(seed, n_items, b, u, t, constellation="qam16", n0=0.1, n0_dev=None, n0_group=1, item0=0,
                 return_symbols=False, stream=None):
    """Generate H [n][B][U], Y [n][T][B] (complex64 CUDA tensors) -- and the
    symbol indices [n][T][U] (uint8) when asked -- on the GPU
    (``dbp_synthesize``, counter-based Philox4x32-10: item i of the batch is
    global item ``item0 + i`` and depends on nothing else).  Same model as
    ``synth_frames`` (H ~ CN(0, 1/B), uniform symbols, CN(0, N0) noise), a
    different random stream."""
    from . import _dev, _lib

    const = (make_constellation(constellation) if isinstance(constellation, str) else constellation)
    t_ = _dev.torch()
    H = t_.empty((n_items, b, u), dtype=t_.complex64, device="cuda")
    Y = t_.empty((n_items, t, b), dtype=t_.complex64, device="cuda")
    S = t_.empty((n_items, t, u), dtype=t_.uint8, device="cuda") if return_symbols else None
    syms = np.ascontiguousarray(np.stack([const.symbols.real, const.symbols.imag], -1).astype(np.float32))
    _lib.check(_lib.lib().dbp_synthesize(
        int(seed), int(n_items), int(item0), int(b), int(u), int(t), syms.ctypes.data, int(const.size),
        float(n0), _lib.ptr(n0_dev), int(n0_group), _lib.ptr(H), _lib.ptr(Y), _lib.ptr(S), _lib.stream_ptr(stream)))
    return (H, Y, S) if return_symbols else (H, Y)
