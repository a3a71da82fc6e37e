"""Monte Carlo symbol-error-rate experiments on the GPU.

Mirrors the reference driver ``dbp/montecarlo.py`` (``ser_closed_form``
:42-60, ``wilson_interval`` :63-82, ``ExperimentConfig`` :85-118,
``trial_rng`` :117-120, ``run_trial`` :148-162, ``run_experiment``
:195-225) with the same seeding contract: trial ``t`` of SNR point ``k``
draws H ~ CN(0, 1/B), the symbol indices and the noise, in that order, from
``default_rng(SeedSequence((seed, k, t)))`` -- bit-identical inputs to the
reference's.  What changes is the equalization: instead of one Python call
per trial, all trials of an SNR point go through ONE fused launch of the
sm_100a detector (``pipeline.Detector``), and the realizations are drawn once
and shared by every (equalizer, architecture) pair of an experiment set
(``draw_inputs`` / ``run_experiment(..., inputs=...)``), as the reference's
own design intends ("experiments that differ only in the equalizer or
architecture see identical channel, symbol, and noise realizations").

``ser_predicted`` maps the large-system SINR (``asymptotics.asymptotic_sinr``,
the message-passing MSE on the GPU quadratures) through ``ser_closed_form``
as the reference does (montecarlo.py:188-194,217-218).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .equalize import Equalizer
from .errors import ConfigError
from .model import Architecture, ClusterPartition, complex_gaussian

_Z95 = 1.959963984540054  # two-sided 95% normal quantile (montecarlo.py:40)


def ser_closed_form(constellation, sinr):
    """Square-QAM SER over complex AWGN at symbol SNR ``sinr``
    (montecarlo.py:42-60): p = 2 (1 - 1/sqrt(M)) Q(sqrt(3 sinr/(M-1))),
    SER = 1 - (1 - p)^2."""
    m = constellation.size
    root = int(round(math.sqrt(m)))
    if root * root != m:
        raise ConfigError(f"closed-form SER needs a square QAM set, got M={m}")
    if sinr < 0:
        raise ConfigError("SINR must be nonnegative")
    q = 0.5 * math.erfc(math.sqrt(1.5 * sinr / (m - 1)))
    p = 2.0 * (1.0 - 1.0 / root) * q
    return p * (2.0 - p)


def wilson_interval(errors, n, z=_Z95):
    """Wilson score interval of a binomial proportion (montecarlo.py:63-82);
    ``errors`` may be fractional (per-trial mean error count)."""
    if n <= 0:
        raise ConfigError("interval needs at least one observation")
    phat = errors / n
    denom = 1.0 + z * z / n
    center = (phat + z * z / (2 * n)) / denom
    half = z * math.sqrt(phat * (1.0 - phat) / n + z * z / (4.0 * n * n)) / denom
    lo = 0.0 if errors == 0 else max(center - half, 0.0)
    hi = 1.0 if errors == n else min(center + half, 1.0)
    return lo, hi


@dataclass(frozen=True)
class ExperimentConfig:
    """One SER experiment: fixed system and equalizer, swept over SNR
    (montecarlo.py:85-118)."""

    b: int
    u: int
    constellation: object
    partition: ClusterPartition
    equalizer: Equalizer
    architecture: Architecture
    snr_db: tuple
    trials: int
    seed: int
    lama_t_max: int = 10
    lama_damping: float = 1.0

    def __post_init__(self):
        object.__setattr__(self, "equalizer", Equalizer(self.equalizer))
        object.__setattr__(self, "architecture", Architecture(self.architecture))
        object.__setattr__(self, "snr_db", tuple(float(s) for s in self.snr_db))
        if self.trials < 1:
            raise ConfigError("trials must be >= 1")
        if self.seed < 0:
            raise ConfigError("seed must be nonnegative")
        if self.partition.b != self.b:
            raise ConfigError("partition does not match the antenna count")
        if not all(np.isfinite(self.snr_db)):
            raise ConfigError("SNR points must be finite")

    @property
    def beta(self):
        return self.u / self.b

    def lama_params(self):
        return {"t_max": self.lama_t_max, "damping": self.lama_damping}


def trial_rng(config, trial_index, snr_index=0):
    """Deterministic child generator for one (SNR point, trial) pair
    (montecarlo.py:117-120)."""
    return np.random.default_rng(np.random.SeedSequence((config.seed, snr_index, trial_index)))


@dataclass
class TrialInputs:
    """Realizations of one SNR point: H [n][B][U], Y [n][1][B] (complex64,
    the detector's input precision), the transmitted symbol indices [n][U]
    and N0."""

    h: np.ndarray
    y: np.ndarray
    s_idx: np.ndarray
    n0: float


def _draw(config, snr_index, trial_index, n0):
    # the reference's draw order (montecarlo.py:154-160): H, symbols, noise
    rng = trial_rng(config, trial_index, snr_index)
    h = complex_gaussian(rng, (config.b, config.u), 1.0 / config.b)
    idx = rng.integers(0, config.constellation.size, size=config.u)
    y = h @ config.constellation.symbols[idx] + complex_gaussian(rng, config.b, n0)
    return h, idx, y


def draw_inputs(config, snr_index, start=0, stop=None):
    """Draw trials [start, stop) of one SNR point exactly as the reference's
    run_trial does (host NumPy; a few tens of microseconds per trial)."""
    stop = config.trials if stop is None else stop
    es_over_n0 = 10.0 ** (config.snr_db[snr_index] / 10.0)
    n0 = config.constellation.es / es_over_n0
    n = stop - start
    H = np.empty((n, config.b, config.u), np.complex64)
    Y = np.empty((n, 1, config.b), np.complex64)
    S = np.empty((n, config.u), np.int64)
    for k, t in enumerate(range(start, stop)):
        h, idx, y = _draw(config, snr_index, t, n0)
        H[k] = h
        Y[k, 0] = y
        S[k] = idx
    return TrialInputs(H, Y, S, n0)


def _detect(config, inp):
    from . import pipeline

    arch = config.architecture
    counts = list(config.partition.counts) if arch is not Architecture.CENTRALIZED else [config.b]
    # centralized statistics = the PD path with one cluster of all B antennas
    arch_s = "fd" if arch is Architecture.FD else "pd"
    lp = config.lama_params() if config.equalizer is Equalizer.LAMA else None
    return pipeline.detect(arch_s, config.equalizer.value, inp.h, inp.y, inp.n0, counts, config.constellation,
                           lama_params=lp, check=True)


def run_trial(config, trial_index, snr_index=0):
    """One transmission: per-UE symbol-error indicators (montecarlo.py:148-162),
    equalized on the GPU."""
    inp = draw_inputs(config, snr_index, trial_index, trial_index + 1)
    det = _detect(config, inp)
    return np.asarray(det.decisions)[0, 0] != inp.s_idx[0]


@dataclass
class SnrPointResult:
    snr_db: float
    trials: int
    n_symbols: int
    errors: int
    ser: float
    ci_low: float
    ci_high: float
    ser_predicted: float


@dataclass
class SerResult:
    config: ExperimentConfig
    points: list = field(default_factory=list)


def predicted_sinr(config, es_over_n0):
    """Large-system SINR for the experiment's (equalizer, architecture)
    (montecarlo.py:188-194)."""
    from . import asymptotics

    return asymptotics.asymptotic_sinr(config.equalizer, config.architecture, config.constellation, es_over_n0,
                                       config.beta, weights=config.partition.weights)


def count_errors(config, inp):
    """Symbol errors of all trials in ``inp`` (one fused launch)."""
    det = _detect(config, inp)
    return int(np.count_nonzero(np.asarray(det.decisions)[:, 0, :] != inp.s_idx))


def run_experiment(config, inputs=None):
    """Aggregate the trials x SNR points (montecarlo.py:195-225).  ``inputs``:
    optional list (one TrialInputs per SNR point) from ``draw_inputs``, shared
    between experiments that differ only in equalizer / architecture."""
    result = SerResult(config=config)
    n_symbols = config.trials * config.u
    for k, snr_db in enumerate(config.snr_db):
        inp = inputs[k] if inputs is not None else draw_inputs(config, k)
        errors = count_errors(config, inp)
        ci_low, ci_high = wilson_interval(errors / config.u, config.trials)
        ser_pred = ser_closed_form(config.constellation, predicted_sinr(config, 10.0 ** (snr_db / 10.0)))
        result.points.append(SnrPointResult(
            snr_db=snr_db, trials=config.trials, n_symbols=n_symbols, errors=errors,
            ser=errors / n_symbols, ci_low=ci_low, ci_high=ci_high, ser_predicted=ser_pred))
    return result
