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
one launch, which is where the GPU pays (SNR / rate sweeps).

On top of them, the decoupled fixed points and the post-equalization SINRs
the Monte Carlo driver maps to ``ser_predicted`` (asymptotics.py:75-111,
132-235, 291-316): ``solve_fixed_point``, ``sinr_pd_closed_form``,
``sinr_fd``, ``sinr_fd_zf_closed``, ``sinr_fd_lmmse_closed``,
``asymptotic_sinr`` -- scalar host iterations whose only heavy step, the
message-passing MSE, is the GPU quadrature; and the rate searches
``sinr_for_rate`` / ``min_antenna_ratio`` (asymptotics.py:265-376), the same
bisections over those functions.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

import math

from . import _lib
from .equalize import Equalizer
from .errors import ConfigError, InfeasibleError, InvalidRegimeError, NonConvergenceError
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


_ZF_MARGIN = 1e-9  # asymptotics.py:25 -- ZF needs beta/w < 1 - margin


@dataclass
class FixedPointResult:
    sigma2: float
    sinr: float
    iterations: int
    converged: bool


def solve_fixed_point(spec, n0, beta, w=1.0, tol=1e-12, max_iter=100_000):
    """asymptotics.py:82-109: largest solution of w sigma2 = N0 + beta
    Psi(sigma2), iterated down from (N0 + beta Es)/w."""
    if n0 <= 0:
        raise ConfigError("fixed point requires N0 > 0")
    if w <= 0:
        raise ConfigError("cluster fraction w must be positive")
    if spec.kind is Equalizer.ZF and beta / w >= 1.0 - _ZF_MARGIN:
        raise InvalidRegimeError(f"ZF fixed point needs beta/w < 1, got beta={beta}, w={w}")
    sigma2 = (n0 + beta * spec.es) / w
    for it in range(1, max_iter + 1):
        nxt = (n0 + beta * psi_mse(spec, sigma2)) / w
        if abs(nxt - sigma2) <= tol * sigma2:
            return FixedPointResult(sigma2=nxt, sinr=spec.es / nxt, iterations=it, converged=True)
        sigma2 = nxt
    raise NonConvergenceError(f"fixed point did not converge within {max_iter} iterations "
                              f"(kind={spec.kind}, beta={beta}, w={w})")


def fixed_point_multiplicity(spec, n0, beta, w=1.0, rel_tol=1e-6):
    """asymptotics.py:112-129: rerun the iteration from just above the noise
    floor; a different limit than the largest fixed point means several
    solutions.  Returns (multiple, largest, smallest)."""
    largest = solve_fixed_point(spec, n0, beta, w=w).sigma2
    sigma2 = n0 / w * (1.0 + 1e-9)
    for _ in range(100_000):
        nxt = (n0 + beta * psi_mse(spec, sigma2)) / w
        done = abs(nxt - sigma2) <= 1e-12 * sigma2
        sigma2 = nxt
        if done:
            break
    return abs(largest - sigma2) > rel_tol * largest, largest, min(sigma2, largest)


def _lmmse_cluster_sinr(g, beta, w):
    """Per-cluster L-MMSE SINR for an antenna fraction w (asymptotics.py:148-152):
    the positive root of s^2 + (1 - g (w - beta)) s - g w = 0."""
    b = 1.0 - g * (w - beta)
    return 0.5 * (math.sqrt(b * b + 4.0 * g * w) - b)


def sinr_pd_closed_form(kind, es_over_n0, beta):
    """asymptotics.py:132-145: PD (= centralized) SINR of the linear kinds."""
    kind = Equalizer(kind)
    g = es_over_n0
    if kind is Equalizer.MRC:
        return g / (1.0 + beta * g)
    if kind is Equalizer.ZF:
        if beta >= 1.0 - _ZF_MARGIN:
            raise InvalidRegimeError(f"ZF closed form needs beta < 1, got {beta}")
        return g * (1.0 - beta)
    if kind is Equalizer.LMMSE:
        return _lmmse_cluster_sinr(g, beta, 1.0)
    raise ConfigError("no closed form for the message-passing equalizer")


def _check_weights(weights):
    w = np.asarray(weights, dtype=float)
    if w.ndim != 1 or abs(w.sum() - 1.0) > 1e-9 or np.any(w < 0):
        raise ConfigError(f"invalid cluster weights {weights}")
    return w


@dataclass
class FdSinrResult:
    per_cluster_sinr: np.ndarray
    sinr: float
    sigma2: float


def sinr_fd(spec, es_over_n0, beta, weights, tol=1e-12):
    """asymptotics.py:161-201: per-cluster fixed points; fused SINR = sum of
    the cluster SINRs, fused variance their harmonic combination, checked
    against N0 + beta sum_c nu_c Psi(sigma_c^2)."""
    weights = _check_weights(weights)
    n0 = spec.es / es_over_n0
    if spec.kind is Equalizer.ZF and np.any(beta / weights[weights > 0] >= 1.0 - _ZF_MARGIN):
        raise InvalidRegimeError("ZF in the FD architecture needs w_c > beta for every cluster")
    per = np.zeros(weights.size)
    s2c = np.full(weights.size, np.inf)
    for i, w in enumerate(weights):
        if w == 0.0:
            continue  # an empty cluster carries no information
        fp = solve_fixed_point(spec, n0, beta, w=w, tol=tol)
        per[i], s2c[i] = fp.sinr, fp.sigma2
    total = float(per.sum())
    if total <= 0:
        raise InvalidRegimeError("fused SINR is zero; no cluster carries information")
    sigma2_fd = spec.es / total
    fin = s2c[np.isfinite(s2c)]
    nu = (1.0 / fin) / np.sum(1.0 / fin)
    psi = np.atleast_1d(psi_mse(spec, fin))
    if abs(n0 + beta * float(np.dot(nu, psi)) - sigma2_fd) > 1e-9 * max(sigma2_fd, 1e-300):
        raise NonConvergenceError("fused-variance identity violated")
    return FdSinrResult(per_cluster_sinr=per, sinr=total, sigma2=sigma2_fd)


def sinr_fd_zf_closed(es_over_n0, beta, c):
    """asymptotics.py:204-209: (Es/N0)(1 - C beta)."""
    if c * beta >= 1.0 - _ZF_MARGIN:
        raise InvalidRegimeError(f"ZF-FD closed form needs C*beta < 1, got {c * beta}")
    return es_over_n0 * (1.0 - c * beta)


@dataclass
class LmmseFdSinr:
    value: float
    uniform_lower_bound: float
    pd_upper_bound: float


def sinr_fd_lmmse_closed(es_over_n0, beta, weights):
    """asymptotics.py:219-235: sum of the per-cluster closed forms, with the
    uniform-allocation lower bound and the PD upper bound."""
    w = _check_weights(weights)
    g = es_over_n0
    value = float(sum(_lmmse_cluster_sinr(g, beta, x) for x in w))
    lower = w.size * _lmmse_cluster_sinr(g, beta, 1.0 / w.size)
    return LmmseFdSinr(value=value, uniform_lower_bound=lower,
                       pd_upper_bound=sinr_pd_closed_form(Equalizer.LMMSE, g, beta))


def asymptotic_sinr(kind, architecture, constellation, es_over_n0, beta, weights=None, order=None):
    """asymptotics.py:291-316: large-system SINR of any (equalizer,
    architecture) pair."""
    kind = Equalizer(kind)
    architecture = Architecture(architecture)
    if architecture is Architecture.FD and kind is not Equalizer.MRC:
        if weights is None:
            raise ConfigError("the FD architecture needs cluster weights")
        weights = np.asarray(weights, dtype=float)
        if kind is Equalizer.ZF:
            return sinr_fd_zf_closed(es_over_n0, beta, weights.size)
        if kind is Equalizer.LMMSE:
            return sinr_fd_lmmse_closed(es_over_n0, beta, weights).value
        spec = MseSpec(Equalizer.LAMA, es=constellation.es, constellation=constellation, order=order)
        return sinr_fd(spec, es_over_n0, beta, weights).sinr
    if kind is Equalizer.LAMA:
        spec = MseSpec(Equalizer.LAMA, es=constellation.es, constellation=constellation, order=order)
        return solve_fixed_point(spec, constellation.es / es_over_n0, beta).sinr
    return sinr_pd_closed_form(kind, es_over_n0, beta)


def sinr_for_rate(constellation, rate, tol_bits=1e-9, order=DEFAULT_QUAD_ORDER):
    """asymptotics.py:265-288: the SINR at which the AWGN mutual information
    of the constellation reaches ``rate`` bits (doubling, then bisection)."""
    max_rate = constellation.bits_per_symbol
    if not 0.0 < rate < max_rate:
        raise ConfigError(f"target rate must lie in (0, {max_rate}), got {rate}")
    hi = 1.0
    for _ in range(80):
        if awgn_mutual_information(constellation, hi, order) >= rate:
            break
        hi *= 2.0
    else:
        raise InfeasibleError(f"rate {rate} not reachable at finite SINR")
    lo = 0.0
    while True:
        mid = 0.5 * (lo + hi)
        mi = awgn_mutual_information(constellation, mid, order)
        if abs(mi - rate) <= tol_bits or (hi - lo) <= 1e-12 * max(hi, 1.0):
            return mid
        if mi < rate:
            lo = mid
        else:
            hi = mid


def min_antenna_ratio(kind, architecture, constellation, target_rate, snr_loss_db, c=1, weights=None,
                      beta_resolution=1e-4, order=None):
    """asymptotics.py:319-376: smallest B/U at which the equalizer, at
    ``snr_loss_db`` above the AWGN SNR for ``target_rate``, still reaches it
    (bisection on beta; LAMA's feasible set is re-checked on a grid)."""
    kind = Equalizer(kind)
    architecture = Architecture(architecture)
    if snr_loss_db < 0:
        raise ConfigError("SNR loss must be nonnegative")
    if weights is None:
        weights = np.full(c, 1.0 / c)
    gamma = sinr_for_rate(constellation, target_rate, order=order or DEFAULT_QUAD_ORDER)
    g = gamma * 10.0 ** (snr_loss_db / 10.0)

    def feasible(beta):
        try:
            return asymptotic_sinr(kind, architecture, constellation, g, beta, weights, order=order) >= gamma
        except InvalidRegimeError:
            return False

    lo = 1e-6
    if not feasible(lo):
        raise InfeasibleError(f"no antenna ratio up to 1e6 achieves rate {target_rate} at {snr_loss_db} dB SNR loss")
    if feasible(1.0):
        return 1.0
    hi = 1.0
    while hi - lo > beta_resolution:
        mid = 0.5 * (lo + hi)
        if feasible(mid):
            lo = mid
        else:
            hi = mid
    if kind is Equalizer.LAMA and any(feasible(b) for b in np.linspace(hi, 1.0, 65)[1:]):
        for b in np.arange(1.0, hi, -beta_resolution):  # disconnected feasible set: fine scan
            if feasible(b):
                return 1.0 / b
    return 1.0 / lo
