"""Drop-in replacement for the reference ``dbp.equalize`` (equalize.py):
preprocessing, PD fusion of partial statistics, MRC / ZF / L-MMSE with exact
per-UE error variances, L-MMSE unbiasing, the Gram-domain LAMA recursion and
nearest-symbol detection -- computed by the sm_100a kernels of
libdbp_b200.so.

Same names, dataclasses, argument meaning and exceptions as the reference.
Extensions: every array may carry leading batch dimensions (channels
[..., B, U]; receive vectors [..., B] or, with T vectors per channel,
[..., T, B]); torch CUDA tensors are accepted as buffers and results then stay
on the device.  Arithmetic is fp32 (complex64): estimates match the
reference's float64 results to ~1e-6 relative (tests state the tolerance).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from math import prod

import numpy as np

from . import _dev, _lib
from .errors import ConfigError, DimensionMismatchError, NegativeVarianceError

_VAR_TOL = 1e-9  # equalize.py:24


class Equalizer(str, Enum):
    MRC = "mrc"
    ZF = "zf"
    LMMSE = "lmmse"
    LAMA = "lama"

    def __str__(self):
        return self.value


@dataclass
class PartialStats:
    """Per-cluster Gram G_c = H_c^H H_c and matched filter y_c^mrc = H_c^H y_c."""

    gram: object
    y_mrc: object


@dataclass
class FusedStats:
    """Sum of the per-cluster statistics (complete Gram and MRC vector)."""

    gram: object
    y_mrc: object

    @property
    def u(self):
        return self.gram.shape[-1]


@dataclass
class EqualizerOutput:
    """Estimate z, per-UE error variances, and the own-signal gain of a biased
    estimator (L-MMSE) or None."""

    z: object
    sigma2: object
    equalizer: Equalizer
    signal_gain: object = None


@dataclass
class LamaState:
    """Per-iteration snapshot of the message-passing recursion."""

    t: int
    z: object
    s: object
    v: object
    phi: object


# ----------------------------------------------------------------- helpers --
def _split_receive(h_shape, y):
    """Classify y against a channel of shape [..., B, U]: returns
    (T, single) where single means one vector per channel."""
    lead, b = tuple(h_shape[:-2]), h_shape[-2]
    ys = tuple(y.shape)
    if ys == lead + (b,):
        return 1, True
    if len(ys) == len(lead) + 2 and ys[:-2] == lead and ys[-1] == b:
        return ys[-2], False
    raise DimensionMismatchError(f"incompatible shapes H_c {tuple(h_shape)}, y_c {ys}")


def _stats_view(gram, y_mrc):
    """Normalise (gram [..., U, U], y_mrc [..., U] or [..., T, U]) to device
    tensors (n, U, T, single, lead, host)."""
    g, host_g = _dev.to_c64(gram)
    m, host_m = _dev.to_c64(y_mrc)
    if g.dim() < 2 or g.shape[-1] != g.shape[-2]:
        raise DimensionMismatchError(f"Gram matrix must be square, got {tuple(g.shape)}")
    u = g.shape[-1]
    lead = tuple(g.shape[:-2])
    if tuple(m.shape) == lead + (u,):
        t_count, single = 1, True
    elif m.dim() == len(lead) + 2 and tuple(m.shape[:-2]) == lead and m.shape[-1] == u:
        t_count, single = m.shape[-2], False
    else:
        raise DimensionMismatchError(f"MRC vector {tuple(m.shape)} does not match Gram {tuple(g.shape)}")
    n = prod(lead) if lead else 1
    return g.reshape(n, u, u), m.reshape(n, t_count, u), n, u, t_count, single, lead, (host_g or host_m)


def _pack_stats(g, m):
    """[n][U][U] + [n][T][U] -> contiguous stats records [n][U*U + T*U]."""
    t = _dev.torch()
    n = g.shape[0]
    return t.cat([g.reshape(n, -1), m.reshape(n, -1)], dim=1).contiguous()


def _shape_vec(x, lead, t_count, single, tail):
    shp = lead + ((tail,) if single else (t_count, tail))
    return x.reshape(shp)


# ------------------------------------------------------ preprocessing (K1) --
def local_preprocess(h_c, y_c):
    """Gram and MRC contributions of one antenna cluster (equalize.py:85-93)."""
    return _gram_mrc(h_c, y_c)


def _gram_mrc(h, y, offsets=None, sum_clusters=True):
    hd, host_h = _dev.to_c64(h)
    yd, host_y = _dev.to_c64(y)
    host = host_h or host_y
    if hd.dim() < 2:
        raise DimensionMismatchError(f"incompatible shapes H_c {tuple(hd.shape)}, y_c {tuple(yd.shape)}")
    t_count, single = _split_receive(hd.shape, yd)
    lead = tuple(hd.shape[:-2])
    b, u = hd.shape[-2], hd.shape[-1]
    n = prod(lead) if lead else 1
    if u > 64:
        raise ConfigError("the sm_100a path supports U <= 64")
    H = hd.reshape(n, b, u)
    Y = yd.reshape(n, t_count, b)
    H, us = _dev.pad_even_u(H)
    counts = [b] if offsets is None else list(np.diff(offsets))
    H, Y, off = _dev.pad_clusters(H, Y, counts)
    grams, mrcs = [], []
    for t0 in range(0, t_count, 16):
        tt = min(16, t_count - t0)
        Yt = Y[:, t0:t0 + tt].contiguous()
        stats = _dev.empty_c64((n, u * u + tt * u))
        o_arr, o_ptr = _lib.host_i32(off)
        lib = _lib.lib()
        _lib.check(lib.dbp_gram_mrc(_lib.ptr(H), _lib.ptr(Yt), n, H.shape[1], u, us, tt, len(counts),
                                    o_ptr, 1 if sum_clusters else 0, _lib.ptr(stats), _lib.stream_ptr()))
        if t0 == 0:
            grams.append(stats[:, : u * u].reshape(n, u, u))
        mrcs.append(stats[:, u * u:].reshape(n, tt, u))
        del o_arr
    t = _dev.torch()
    gram = grams[0]
    mrc = t.cat(mrcs, dim=1) if len(mrcs) > 1 else mrcs[0]
    gram = gram.reshape(lead + (u, u))
    mrc = _shape_vec(mrc, lead, t_count, single, u)
    return PartialStats(gram=_dev.out(gram, host), y_mrc=_dev.out(mrc, host))


def fuse_partials(parts):
    """Feedforward adder tree over the partial statistics (equalize.py:96-107)."""
    parts = list(parts)
    if not parts:
        raise ConfigError("cannot fuse an empty list of partial statistics")
    u = parts[0].gram.shape[-1]
    yshape = tuple(parts[0].y_mrc.shape)
    for p in parts:
        if tuple(p.y_mrc.shape) != yshape or tuple(p.gram.shape[-2:]) != (u, u):
            raise DimensionMismatchError("partial statistics disagree on U")
    host = not _dev.is_device(parts[0].gram)
    t = _dev.torch()
    gs = t.stack([_dev.to_c64(p.gram)[0] for p in parts]).contiguous()
    ms = t.stack([_dev.to_c64(p.y_mrc)[0] for p in parts]).contiguous()
    lib = _lib.lib()
    g_out = _dev.empty_c64(gs.shape[1:])
    m_out = _dev.empty_c64(ms.shape[1:])
    _lib.check(lib.dbp_stats_sum(_lib.ptr(gs), len(parts), g_out.numel(), _lib.ptr(g_out), _lib.stream_ptr()))
    _lib.check(lib.dbp_stats_sum(_lib.ptr(ms), len(parts), m_out.numel(), _lib.ptr(m_out), _lib.stream_ptr()))
    return FusedStats(gram=_dev.out(g_out, host), y_mrc=_dev.out(m_out, host))


def centralized_stats(h, y):
    """Fused statistics of the unpartitioned system (equalize.py:110-112)."""
    p = local_preprocess(h, y)
    return FusedStats(gram=p.gram, y_mrc=p.y_mrc)


def _check_sigma2(sigma2, kind):
    """equalize.py:115-120 (host-side guard kept for API compatibility)."""
    s = np.asarray(sigma2)
    if np.min(s) < -_VAR_TOL:
        raise NegativeVarianceError(f"{kind} produced negative error variance {np.min(s):.3e}")
    return np.maximum(s, 0.0)


# ------------------------------------------------------ central equalizers --
def _run_stats(kind, fused, n0, es, unbias, beta=0.0, scale=1.0, t_max=1, damping=1.0,
               constellation=None, trace=False):
    g, m, n, u, t_count, single, lead, host = _stats_view(fused.gram, fused.y_mrc)
    if u > 64:
        raise ConfigError("the sm_100a path supports U <= 64")
    if t_count > 16:
        raise ConfigError("at most 16 receive vectors per Gram on the stats path")
    stats = _pack_stats(g, m)
    lama = kind is Equalizer.LAMA
    xhat = _dev.empty_c64((n, t_count, u))
    s2 = _dev.empty_f32((n, t_count) if lama else (n, u))
    gain = _dev.empty_f32((n, u)) if kind in (Equalizer.LMMSE, Equalizer.MRC) else None
    status = _dev.zeros_i32((n,))
    iters = _dev.zeros_i32((n,))
    tr = [None] * 4
    if trace:
        tr = [_dev.empty_c64((n, t_max, t_count, u)) for _ in range(3)] + [_dev.empty_f32((n, t_max, t_count))]
    if constellation is not None:
        lv, lp, L, sv, sp, M = _dev.const_params(constellation)
    else:
        lv, lp, L, sv, sp, M = None, None, 0, None, None, 0
    lib = _lib.lib()
    _lib.check(lib.dbp_equalize_stats(
        _lib.ptr(stats), n, u, t_count, _lib.KIND[kind.value], float(n0), None, 1, float(es),
        1 if unbias else 0, float(beta), float(scale), int(t_max), float(damping), lp, L, sp, M,
        _lib.ptr(xhat), _lib.ptr(s2), _lib.ptr(gain), None, _lib.ptr(status), _lib.ptr(iters),
        _lib.ptr(tr[0]), _lib.ptr(tr[1]), _lib.ptr(tr[2]), _lib.ptr(tr[3]), _lib.stream_ptr()))
    del lv, sv
    return dict(xhat=xhat, s2=s2, gain=gain, status=status, iters=iters, trace=tr, n=n, u=u, T=t_count,
                single=single, lead=lead, host=host)


def linear_equalize(kind, fused, n0, es=1.0):
    """MRC, ZF or L-MMSE on fused statistics (equalize.py:130-176).  Returns
    the raw (biased) L-MMSE estimate with its signal gain, like the
    reference; see :func:`unbiased_output`."""
    kind = Equalizer(kind)
    if kind is Equalizer.LAMA:
        raise ConfigError("use lama_equalize for the message-passing equalizer")
    if kind is Equalizer.LMMSE and es <= 0:
        raise ConfigError("L-MMSE requires Es > 0")
    r = _run_stats(kind, fused, n0, es, unbias=False)
    _dev.raise_status(r["status"], what=kind.value)
    lead, single, host, u, T = r["lead"], r["single"], r["host"], r["u"], r["T"]
    z = _dev.out(_shape_vec(r["xhat"], lead, T, True if single else False, u), host)
    s2 = _dev.out(r["s2"].reshape(lead + (u,)), host, real=True)
    gain = None
    if kind is Equalizer.LMMSE:
        gain = _dev.out(r["gain"].reshape(lead + (u,)), host, real=True)
    return EqualizerOutput(z=z, sigma2=s2, equalizer=kind, signal_gain=gain)


def unbiased_output(output, es=1.0):
    """Gain-normalised estimate z/c with variance (sigma2 - (1-c)^2 Es)/c^2
    (equalize.py:179-195); unbiased outputs pass through unchanged."""
    c = output.signal_gain
    if c is None:
        return output
    host = not _dev.is_device(output.z)
    z, _ = _dev.to_c64(output.z)
    s2, _ = _dev.to_f32(output.sigma2)
    gain, _ = _dev.to_f32(c)
    u = s2.shape[-1]
    n = s2.numel() // u
    t_count = z.numel() // (n * u)
    z_out = _dev.empty_c64(z.shape)
    s2_out = _dev.empty_f32(s2.shape)
    status = _dev.zeros_i32((n,))
    lib = _lib.lib()
    _lib.check(lib.dbp_unbias(_lib.ptr(z), _lib.ptr(s2), _lib.ptr(gain), n, t_count, u, float(es),
                              _lib.ptr(z_out), _lib.ptr(s2_out), _lib.ptr(status), _lib.stream_ptr()))
    st = status.cpu().numpy()
    if np.any(st == _lib.ST_SINGULAR):
        from .errors import SingularGramError

        raise SingularGramError("nonpositive signal gain; cannot unbias")
    _dev.raise_status(status, what=output.equalizer.value)
    return EqualizerOutput(z=_dev.out(z_out, host), sigma2=_dev.out(s2_out, host, real=True),
                           equalizer=output.equalizer)


def posterior_stats(z, tau, constellation):
    """Posterior mean/variance of one symbol under CN(z, tau)
    (equalize.py:198-205)."""
    if tau <= 0:
        raise ConfigError(f"posterior variance requires tau > 0, got {tau}")
    from . import kernels

    f, g = kernels.posterior_mean_var(np.array([z], dtype=np.complex128), tau, constellation.symbols)
    return complex(f[0]), float(g[0])


def lama_equalize(fused, constellation, n0, beta, t_max=10, damping=1.0):
    """Gram-domain message passing (equalize.py:208-259): t_max iterations of
        z^t = y_mrc + (I - G) s^t + v^t,  s^{t+1} = F(z^t, N0 + beta phi^t), ...
    started at s = E[S], phi = Var[S], v = 0.  Returns (EqualizerOutput with
    z^{t_max} and sigma2 = N0 + beta phi^{t_max}, per-iteration trace)."""
    if t_max < 1:
        raise ConfigError("t_max must be >= 1")
    if not 0.0 < damping <= 1.0:
        raise ConfigError("damping must lie in (0, 1]")
    r = _run_stats(Equalizer.LAMA, fused, n0, constellation.es, unbias=False, beta=beta, scale=1.0,
                   t_max=t_max, damping=damping, constellation=constellation, trace=True)
    _dev.raise_status(r["status"], r["iters"], what="lama")
    lead, single, host, u, T = r["lead"], r["single"], r["host"], r["u"], r["T"]
    z = _dev.out(_shape_vec(r["xhat"], lead, T, single, u), host)
    s2t = r["s2"]  # [n][T]
    t = _dev.torch()
    s2full = s2t.reshape(r["n"], T, 1).expand(r["n"], T, u).contiguous()
    s2 = _dev.out(_shape_vec(s2full, lead, T, single, u), host, real=True)
    trz, trs, trv, trp = r["trace"]
    trace = []
    for it in range(t_max):
        zi = _dev.out(_shape_vec(trz[:, it].contiguous(), lead, T, single, u), host)
        si = _dev.out(_shape_vec(trs[:, it].contiguous(), lead, T, single, u), host)
        vi = _dev.out(_shape_vec(trv[:, it].contiguous(), lead, T, single, u), host)
        ph = trp[:, it].contiguous()
        if single and not lead:
            phi = float(ph.reshape(-1)[0].item())
        else:
            phi = _dev.out(ph.reshape(lead + (() if single else (T,))), host, real=True)
        trace.append(LamaState(t=it + 1, z=zi, s=si, v=vi, phi=phi))
    del t
    return EqualizerOutput(z=z, sigma2=s2, equalizer=Equalizer.LAMA), trace


def hard_detect(z, constellation):
    """Nearest-symbol decision per entry, ties to the lowest symbol index
    (equalize.py:262-268).  Returns symbol values like the reference."""
    idx = hard_detect_index(z, constellation)
    if _dev.is_device(idx):
        t = _dev.torch()
        syms = t.as_tensor(np.asarray(constellation.symbols, dtype=np.complex64), device="cuda")
        return syms[idx.long()]
    return np.asarray(constellation.symbols)[idx]


def hard_detect_index(z, constellation):
    """Symbol indices (k = i*L + j layout) of the nearest-symbol decisions."""
    if isinstance(z, EqualizerOutput):
        z = z.z
    zd, host = _dev.to_c64(z)
    idx = _dev.torch().empty(zd.shape, dtype=_dev.torch().int32, device="cuda")
    sv, sp, M = _dev.symbols_params(constellation.symbols)
    lib = _lib.lib()
    _lib.check(lib.dbp_hard_detect(_lib.ptr(zd), zd.numel(), sp, M, _lib.ptr(idx), _lib.stream_ptr()))
    del sv
    return idx.cpu().numpy().astype(np.int64) if host else idx
