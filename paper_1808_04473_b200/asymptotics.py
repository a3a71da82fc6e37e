"""Large-system analysis on the GPU: the
Gauss-Hermite quadratures of the message-passing MSE / mutual information and
the decoupled fixed points the Monte Carlo driver maps to ``ser_predicted``.

- Quadratures (``lama_mse_pam``, ``lama_mse``, ``mi_awgn``; reference
  kernels.py:53-75, _kernels.pyx:74-158) and ``MseSpec`` / ``psi_mse`` /
  ``se_trajectory`` / ``awgn_mutual_information`` (asymptotics.py:29-72,
  237-262): fp64 sums in ``dbp_quadrature``, one CTA per evaluation point;
  every function takes an array of points (one launch per sweep).
- Fixed points (asymptotics.py:75-129): ``fixed_points`` runs the whole state
  evolution sigma2 <- (N0 + beta Psi(sigma2)) / w ON THE GPU for a batch of
  (N0, beta, w, start) points in one launch (``dbp_fixed_point``, one CTA per
  point iterating to convergence); ``solve_fixed_point`` and
  ``fixed_point_multiplicity`` (both orbits in one launch) are views of it.
- ``asymptotic_sinr`` (asymptotics.py:132-235, 291-316) evaluates whole SNR
  arrays: the linear kinds by their closed forms (vectorized), message passing
  by one batched fixed-point launch over every (SNR, cluster) pair.

The reference's rate searches (``sinr_for_rate``, ``min_antenna_ratio``,
asymptotics.py:265-376) are analysis drivers outside the equalization path
and are not part of this build.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .equalize import Equalizer
from .errors import ConfigError, InvalidRegimeError, NonConvergenceError
from .model import Architecture

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
        raise ConfigError(f"{what} must be > 0, got {v}")


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
    _check_positive(sigma2, "the MSE function's sigma2")
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


_ZF_MARGIN = 1e-9  # ZF needs beta / w < 1 - margin (asymptotics.py:25)
_MAX_ITER = 100_000


@dataclass
class FixedPointResult:
    sigma2: float
    sinr: float
    iterations: int
    converged: bool


def _rule_values(constellation, order):
    """(kind, host values, M, order) of the MSE rule for a constellation:
    the factorised PAM rule when it is a square QAM set."""
    levels = getattr(constellation, "pam_levels", None)
    if levels is not None:
        return 0, np.ascontiguousarray(np.asarray(levels, dtype=np.float64)), len(levels), order or DEFAULT_PAM_ORDER
    c = np.asarray(constellation.symbols, dtype=np.complex128).reshape(-1)
    return 1, np.ascontiguousarray(np.stack([c.real, c.imag], -1).reshape(-1)), c.size, order or DEFAULT_QUAD_ORDER


def fixed_points(constellation, n0, beta, w=1.0, start=None, tol=1e-12, max_iter=_MAX_ITER, order=None):
    """Decoupled-variance fixed points of the message-passing equalizer for a
    batch of points: n0, beta, w (and optionally start) broadcast together.
    Each point iterates sigma2 <- (N0 + beta Psi(sigma2)) / w on the GPU from
    ``start`` (default (N0 + beta Es) / w: the orbit decreases onto the largest
    solution) until |new - old| <= tol old.  Returns (sigma2, iterations);
    iterations < 0 marks a point that did not converge."""
    import ctypes as C

    import torch

    es = float(constellation.es)
    st = np.nan if start is None else start
    a, b, c, s0 = np.broadcast_arrays(np.asarray(n0, dtype=np.float64), np.asarray(beta, dtype=np.float64),
                                      np.asarray(w, dtype=np.float64), np.asarray(st, dtype=np.float64))
    shape = a.shape
    if start is None:
        s0 = (a + b * es) / c
    kind, vals, m, q = _rule_values(constellation, order)
    nodes, weights = _rule_device(q)

    def dev(x):
        return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1)), device="cuda")

    n0d, bd, wd, sd = dev(a), dev(b), dev(c), dev(s0)
    out = torch.empty_like(n0d)
    its = torch.empty(n0d.shape, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().dbp_fixed_point(kind, _lib.ptr(n0d), _lib.ptr(bd), _lib.ptr(wd), _lib.ptr(sd), n0d.numel(),
                                          vals.ctypes.data_as(C.c_void_p), m, _lib.ptr(nodes), _lib.ptr(weights),
                                          int(q), float(tol), int(max_iter), _lib.ptr(out), _lib.ptr(its),
                                          _lib.stream_ptr()))
    return out.cpu().numpy().reshape(shape), its.cpu().numpy().reshape(shape)


def _linear_fixed_point(kind, es, n0, beta, w):
    """Closed-form solutions of w sigma2 = N0 + beta Psi(sigma2) for the
    linear kinds' Psi (psi_mse): MRC Es, ZF sigma2, L-MMSE Es sigma2/(Es + sigma2)
    (the positive root of w s^2 + (w Es - N0 - beta Es) s - N0 Es = 0)."""
    if kind is Equalizer.MRC:
        return (n0 + beta * es) / w
    if kind is Equalizer.ZF:
        return n0 / (w - beta)
    bq = w * es - n0 - beta * es
    return (-bq + np.sqrt(bq * bq + 4.0 * w * n0 * es)) / (2.0 * w)


def _check_regime(kind, n0, beta, w):
    if np.any(np.asarray(n0) <= 0):
        raise ConfigError("fixed point requires N0 > 0")
    if np.any(np.asarray(w) <= 0):
        raise ConfigError("cluster fraction w must be positive")
    if kind is Equalizer.ZF and np.any(np.asarray(beta) / np.asarray(w) >= 1.0 - _ZF_MARGIN):
        raise InvalidRegimeError(f"ZF fixed point needs beta/w < 1, got beta={beta}, w={w}")


def solve_fixed_point(spec, n0, beta, w=1.0, tol=1e-12, max_iter=_MAX_ITER):
    """Largest solution of w sigma2 = N0 + beta Psi(sigma2) (asymptotics.py:82-109)."""
    _check_regime(spec.kind, n0, beta, w)
    if spec.kind is Equalizer.LAMA:
        s2, it = fixed_points(spec.constellation, n0, beta, w, tol=tol, max_iter=max_iter, order=spec.order)
        s2, it = float(s2), int(it)
        if it < 0:
            raise NonConvergenceError(f"fixed point did not converge within {max_iter} iterations "
                                      f"(kind={spec.kind}, beta={beta}, w={w})")
        return FixedPointResult(sigma2=s2, sinr=spec.es / s2, iterations=it, converged=True)
    s2 = float(_linear_fixed_point(spec.kind, float(spec.es), float(n0), float(beta), float(w)))
    return FixedPointResult(sigma2=s2, sinr=spec.es / s2, iterations=0, converged=True)


def fixed_point_multiplicity(spec, n0, beta, w=1.0, rel_tol=1e-6):
    """asymptotics.py:112-129: the orbit from (N0 + beta Es)/w and the one
    from just above the noise floor N0/w, both in one launch; different
    limits mean several solutions.  Returns (multiple, largest, smallest)."""
    _check_regime(spec.kind, n0, beta, w)
    if spec.kind is not Equalizer.LAMA:
        s2 = float(_linear_fixed_point(spec.kind, float(spec.es), float(n0), float(beta), float(w)))
        return False, s2, s2
    starts = np.array([(n0 + beta * spec.es) / w, n0 / w * (1.0 + 1e-9)])
    s2, it = fixed_points(spec.constellation, n0, beta, w, start=starts, order=spec.order)
    if it[0] < 0:
        raise NonConvergenceError("fixed point did not converge")
    largest, other = float(s2[0]), float(s2[1])
    return abs(largest - other) > rel_tol * largest, largest, min(other, largest)


def _lmmse_sinr(g, beta, w):
    """L-MMSE SINR of a cluster holding antenna fraction w (asymptotics.py:148-152):
    the positive root of s^2 + (1 - g (w - beta)) s - g w = 0 (vectorized)."""
    b = 1.0 - g * (w - beta)
    return 0.5 * (np.sqrt(b * b + 4.0 * g * w) - b)


def sinr_pd_closed_form(kind, es_over_n0, beta):
    """asymptotics.py:132-145: PD (= centralized) SINR of the linear kinds."""
    kind = Equalizer(kind)
    g = np.asarray(es_over_n0, dtype=np.float64)
    if kind is Equalizer.MRC:
        r = g / (1.0 + beta * g)
    elif kind is Equalizer.ZF:
        if beta >= 1.0 - _ZF_MARGIN:
            raise InvalidRegimeError(f"ZF closed form needs beta < 1, got {beta}")
        r = g * (1.0 - beta)
    elif kind is Equalizer.LMMSE:
        r = _lmmse_sinr(g, beta, 1.0)
    else:
        raise ConfigError("no closed form for the message-passing equalizer")
    return float(r) if r.ndim == 0 else r


def asymptotic_sinr(kind, architecture, constellation, es_over_n0, beta, weights=None, order=None):
    """Large-system post-equalization SINR of any (equalizer, architecture)
    pair (asymptotics.py:291-316); ``es_over_n0`` scalar or array.

    FD fuses the clusters' estimates with SINR-optimal weights, so the fused
    SINR is the sum of the clusters' SINRs: ZF (Es/N0)(1 - C beta), L-MMSE the
    sum of the per-cluster closed forms, message passing the sum of the
    per-cluster fixed points (all (SNR, cluster) pairs in one GPU launch).
    MRC fuses with the Gram-diagonal weights and equals PD."""
    kind = Equalizer(kind)
    architecture = Architecture(architecture)
    g = np.asarray(es_over_n0, dtype=np.float64)
    es = float(constellation.es) if constellation is not None else 1.0
    if architecture is Architecture.FD and kind is not Equalizer.MRC:
        if weights is None:
            raise ConfigError("the FD architecture needs cluster weights")
        w = np.asarray(weights, dtype=np.float64)
        if w.ndim != 1 or abs(w.sum() - 1.0) > 1e-9 or np.any(w < 0):
            raise ConfigError(f"invalid cluster weights {weights}")
        if kind is Equalizer.ZF:
            if w.size * beta >= 1.0 - _ZF_MARGIN:
                raise InvalidRegimeError(f"ZF-FD needs C*beta < 1, got {w.size * beta}")
            r = g * (1.0 - w.size * beta)
        elif kind is Equalizer.LMMSE:
            r = np.sum(_lmmse_sinr(g[..., None], beta, w), axis=-1)
        else:  # message passing: per-cluster fixed points (empty clusters carry nothing)
            wp = w[w > 0]
            n0 = es / g
            s2, it = fixed_points(constellation, n0[..., None], beta, wp, order=order)
            if np.any(it < 0):
                raise NonConvergenceError("a cluster fixed point did not converge")
            r = np.sum(es / s2, axis=-1)
            if np.any(r <= 0):
                raise InvalidRegimeError("fused SINR is zero; no cluster carries information")
    elif kind is Equalizer.LAMA:
        s2, it = fixed_points(constellation, es / g, beta, 1.0, order=order)
        if np.any(it < 0):
            raise NonConvergenceError("fixed point did not converge")
        r = es / s2
    else:
        return sinr_pd_closed_form(kind, es_over_n0, beta)
    r = np.asarray(r, dtype=np.float64)
    return float(r) if r.ndim == 0 else r
