"""Parity metrics used by the GPU tests (fp32 CUDA path vs the fp64 oracle /
reference golden outputs).

Tolerances (BASELINE.json north star): max normwise relative error <= 1e-4 on
the estimates x-hat (per vector: ||x - x_ref||_inf / ||x_ref||_inf, max over
vectors) and entrywise relative error <= 1e-4 on the fusion weights nu;
hard-decision mismatches <= 1e-5 of the symbols, each at a decision boundary.
"""

import numpy as np

XHAT_TOL = 1e-4
NU_TOL = 1e-4
SIGMA2_TOL = 1e-4
DEC_RATE = 1e-5
# a flipped decision "lies at a decision boundary" when the reference
# estimate is within this multiple of the observed estimate error of the
# midpoint between the two PAM levels involved
BOUNDARY_FACTOR = 4.0


def normwise_rel(x, ref):
    """max over vectors (last axis) of ||x - ref||_inf / ||ref||_inf."""
    x = np.asarray(x)
    ref = np.asarray(ref)
    num = np.max(np.abs(x - ref), axis=-1)
    den = np.maximum(np.max(np.abs(ref), axis=-1), 1e-30)
    return float(np.max(num / den))


def entry_rel(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(x - ref) / np.maximum(np.abs(ref), 1e-30)))


def check_decisions(dec, dec_ref, x_ref, x, levels):
    """Return (n_mismatch, n_total, all_at_boundary)."""
    dec = np.asarray(dec).astype(np.int64)
    dec_ref = np.asarray(dec_ref).astype(np.int64)
    bad = np.argwhere(dec != dec_ref)
    if bad.size == 0:
        return 0, dec.size, True
    L = len(levels)
    mids = 0.5 * (np.asarray(levels)[:-1] + np.asarray(levels)[1:])
    ok = True
    for idx in map(tuple, bad):
        xr, xv = complex(x_ref[idx]), complex(x[idx])
        err = abs(xv - xr)
        for comp, a, b in ((xr.real, dec[idx] // L, dec_ref[idx] // L), (xr.imag, dec[idx] % L, dec_ref[idx] % L)):
            if a != b:
                dist = np.min(np.abs(mids - comp))
                if dist > BOUNDARY_FACTOR * err + 1e-7:
                    ok = False
    return len(bad), dec.size, ok
