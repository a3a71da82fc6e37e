"""Gauss-Hermite quadratures of the large-system analysis on the GPU
(SURVEY.md 8(f) rank 4).

Mirrors the reference's ``dbp.kernels`` quadratures (``lama_mse_pam``,
``lama_mse``, ``mi_awgn``; kernels.py:53-75, _kernels.pyx:74-158) and the
analysis functions built directly on them (asymptotics.py: ``MseSpec``
:29-45, ``psi_mse`` :47-72, ``se_trajectory`` :237-251,
``awgn_mutual_information`` :254-262), with the same names, arguments,
defaults (orders 2048 for the factorised PAM rule, 32 for the 2-D rules) and
errors.  The sums run in fp64 in ``dbp_quadrature`` (one CTA per evaluation
point); every function also takes an ARRAY of points and evaluates them in
one launch, which is where the GPU pays (SNR / rate sweeps).  The
fixed-point, closed-form SINR and rate-search parts of the reference's
analysis stay out of scope (scalar, ms on the host).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .equalize import Equalizer
from .errors import ConfigError

DEFAULT_QUAD_ORDER = 32  # kernels.py:22
DEFAULT_PAM_ORDER = 2048  # kernels.py:25
_KIND = {"pam": 0, "mse2d": 1, "mi": 2}


@lru_cache(maxsize=32)
def gauss_hermite(order):
    """Nodes / weights for the weight exp(-x^2) (kernels.py:34-38; scipy's
    roots_hermite: host-side setup, cached like the reference's)."""
    from scipy.special import roots_hermite

    return roots_hermite(int(order))


@lru_cache(maxsize=32)
def _rule_device(order):
    import torch

    n, w = gauss_hermite(order)
    return (torch.as_tensor(np.ascontiguousarray(n), dtype=torch.float64, device="cuda"),
            torch.as_tensor(np.ascontiguousarray(w), dtype=torch.float64, device="cuda"))


def _quad(kind, xs, values, order):
    import torch

    scalar = np.ndim(xs) == 0
    x = np.atleast_1d(np.asarray(xs, dtype=np.float64))
    if x.size == 0:
        return np.empty(0)
    if kind == "pam":
        vals = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
    else:
        c = np.asarray(values, dtype=np.complex128).reshape(-1)
        vals = np.ascontiguousarray(np.stack([c.real, c.imag], -1).reshape(-1))
    m = vals.size if kind == "pam" else vals.size // 2
    nodes, weights = _rule_device(order)
    xd = torch.as_tensor(np.ascontiguousarray(x.reshape(-1)), device="cuda")
    out = torch.empty_like(xd)
    import ctypes as C

    _lib.check(_lib.lib().dbp_quadrature(_KIND[kind], _lib.ptr(xd), xd.numel(), vals.ctypes.data_as(C.c_void_p), m,
                                         _lib.ptr(nodes), _lib.ptr(weights), int(order), _lib.ptr(out),
                                         _lib.stream_ptr()))
    r = out.cpu().numpy().reshape(x.shape)
    return float(r[0]) if scalar else r


def _check_positive(v, what):
    if np.any(np.asarray(v) <= 0):
        raise ConfigError(f"{what} must be > 0")


def lama_mse_pam(sigma2, levels, order=DEFAULT_PAM_ORDER):
    """Posterior-mean MSE of a square QAM set by the factorised 1-D rule
    (kernels.py:62-67); ``sigma2`` scalar or array."""
    _check_positive(sigma2, "sigma2")
    return _quad("pam", sigma2, levels, order)


def lama_mse(sigma2, symbols, order=DEFAULT_QUAD_ORDER):
    """Posterior-mean MSE by the 2-D rule (kernels.py:53-59)."""
    _check_positive(sigma2, "sigma2")
    return _quad("mse2d", sigma2, symbols, order)


def mi_awgn(noise_var, symbols, order=DEFAULT_QUAD_ORDER):
    """Mutual information (bits) of the uniform input over complex AWGN
    (kernels.py:70-75)."""
    _check_positive(noise_var, "noise variance")
    return _quad("mi", noise_var, symbols, order)


@dataclass(frozen=True)
class MseSpec:
    """asymptotics.py:29-45."""

    kind: Equalizer
    es: float = 1.0
    constellation: object = None
    order: int = None

    def __post_init__(self):
        object.__setattr__(self, "kind", Equalizer(self.kind))
        if self.kind is Equalizer.LAMA and self.constellation is None:
            raise ConfigError("the message-passing MSE function needs a constellation")


def psi_mse(spec, sigma2):
    """asymptotics.py:47-72: MSE of the equalizer's decoupled denoiser."""
    _check_positive(sigma2, "MSE function requires sigma2")
    s = np.asarray(sigma2, dtype=np.float64)
    kind = spec.kind
    if kind is Equalizer.MRC:
        r = np.full(s.shape, float(spec.es))
    elif kind is Equalizer.ZF:
        r = s.copy()
    elif kind is Equalizer.LMMSE:
        r = spec.es * s / (spec.es + s)
    else:
        const = spec.constellation
        if getattr(const, "pam_levels", None) is not None:
            return lama_mse_pam(sigma2, const.pam_levels, spec.order or DEFAULT_PAM_ORDER)
        return lama_mse(sigma2, const.symbols, spec.order or DEFAULT_QUAD_ORDER)
    return float(r) if r.ndim == 0 else r


def se_trajectory(constellation, n0, beta, t, w=1.0, order=None):
    """asymptotics.py:237-251: sigma_1^2 = (N0 + beta Es)/w, then
    sigma_t^2 = (N0 + beta Psi(sigma_{t-1}^2))/w."""
    if t < 1:
        raise ConfigError("trajectory length must be >= 1")
    spec = MseSpec(Equalizer.LAMA, es=constellation.es, constellation=constellation, order=order)
    traj = np.empty(t)
    sigma2 = (n0 + beta * constellation.es) / w
    traj[0] = sigma2
    for i in range(1, t):
        sigma2 = (n0 + beta * psi_mse(spec, sigma2)) / w
        traj[i] = sigma2
    return traj


def awgn_mutual_information(constellation, sinr, order=DEFAULT_QUAD_ORDER):
    """asymptotics.py:254-262 (bits per channel use); ``sinr`` scalar or
    array (SINR 0 gives 0 bits)."""
    s = np.asarray(sinr, dtype=np.float64)
    if np.any(s < 0):
        raise ConfigError("SINR must be nonnegative")
    out = np.zeros(s.shape)
    pos = s > 0
    if np.any(pos):
        out[pos] = np.atleast_1d(mi_awgn(constellation.es / s[pos], constellation.symbols, order))
    return float(out) if out.ndim == 0 else out
