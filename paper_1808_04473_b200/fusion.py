"""Drop-in replacement for the reference ``dbp.fusion`` (fusion.py): the fully
decentralized (FD) pipeline -- per-cluster equalization on the local channel
block, unbiasing, SINR-optimal (inverse-variance; Gram-diagonal for MRC)
fusion weights and the weighted combination -- on the sm_100a kernels.

``fd_equalize`` runs as ONE fused kernel launch per call: every cluster's
Gram, matched filter, local equalizer, unbiasing and the fusion sums stay on
chip.  ``return_weights=True`` additionally returns the fusion weights nu
(the reference computes them internally but does not return them).
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod

import numpy as np

from . import _dev, _lib
from .equalize import Equalizer, EqualizerOutput
from .errors import ConfigError, DimensionMismatchError

_VARIANCE_FLOOR = 1e-15  # fusion.py:23


@dataclass
class ClusterOutput:
    """Local estimate and per-UE error variances of one cluster
    (fusion.py:26-40)."""

    cluster_id: int
    z: object
    sigma2: object
    equalizer: Equalizer
    mrc_gains: object = None
    signal_gain: object = None


@dataclass
class FusionWeights:
    """C x U per-UE fusion weights, columns sum to one (fusion.py:89-93)."""

    nu: object


@dataclass
class FdOutput(EqualizerOutput):
    """EqualizerOutput of the FD pipeline plus the fusion weights nu
    ([..., C, U])."""

    nu: object = None


def _constellation_args(constellation):
    if constellation is None:
        return None, None, 0, None, None, 0
    return _dev.const_params(constellation)


def run_fused(arch, kind, h, y, counts, n0, es=1.0, constellation=None, lama_params=None, beta=None,
              lama_scale=1.0, unbias=True, want_gain=False, want_dec=False, total_antennas=None,
              n0_dev=None, n0_group=1, check=True):
    """Launch dbp_equalize on (h [..., B, U], y [..., B] or [..., T, B]).

    counts: antenna rows per cluster (sum = B).  Returns a dict of device
    tensors (xhat [n][T][U], sigma2 [n][U] or [n][T], nu [n][C][U|T],
    gain, dec, status) plus shape bookkeeping."""
    kind = Equalizer(kind)
    hd, host_h = _dev.to_c64(h)
    yd, host_y = _dev.to_c64(y)
    from .equalize import _split_receive

    t_count, single = _split_receive(hd.shape, yd)
    lead = tuple(hd.shape[:-2])
    b, u = hd.shape[-2], hd.shape[-1]
    n = prod(lead) if lead else 1
    if u > 64:
        raise ConfigError("the sm_100a path supports U <= 64")
    if t_count > 16:
        raise ConfigError("at most 16 receive vectors per channel on the fused path")
    if sum(counts) != b:
        raise DimensionMismatchError("cluster counts do not sum to B")
    H, us = _dev.pad_even_u(hd.reshape(n, b, u))
    Y = yd.reshape(n, t_count, b)
    H, Y, off = _dev.pad_clusters(H, Y, counts)
    C = len(counts)
    lama = kind is Equalizer.LAMA
    wdim = t_count if lama else u
    xhat = _dev.empty_c64((n, t_count, u))
    s2 = _dev.empty_f32((n, wdim))
    nu = _dev.empty_f32((n, C, wdim)) if arch == _lib.ARCH_FD else None
    gain = _dev.empty_f32((n, u)) if want_gain else None
    dec = _dev.torch().empty((n, t_count, u), dtype=_dev.torch().uint8, device="cuda") if want_dec else None
    status = _dev.zeros_i32((n,))
    iters = _dev.zeros_i32((n,))
    lp = dict(lama_params or {})
    t_max = int(lp.get("t_max", 10))
    damping = float(lp.get("damping", 1.0))
    if lama:
        if constellation is None:
            raise ConfigError("message-passing equalization needs a constellation")
        if t_max < 1:
            raise ConfigError("t_max must be >= 1")
        if not 0.0 < damping <= 1.0:
            raise ConfigError("damping must lie in (0, 1]")
    if kind is Equalizer.LMMSE and es <= 0:
        raise ConfigError("L-MMSE requires Es > 0")
    lv, lptr, L, sv, sptr, M = _constellation_args(constellation)
    es_eff = constellation.es if (lama and constellation is not None) else es
    o_arr, o_ptr = _lib.host_i32(off)
    c_arr, c_ptr = _lib.host_i32(counts)
    lib = _lib.lib()
    _lib.check(lib.dbp_equalize(
        arch, _lib.KIND[kind.value], _lib.ptr(H), _lib.ptr(Y), n, H.shape[1], u, us, t_count, C, o_ptr, c_ptr,
        int(total_antennas or sum(counts)), float(n0), _lib.ptr(n0_dev), int(n0_group), float(es_eff),
        1 if unbias else 0, float(beta if beta is not None else u / b), float(lama_scale), t_max, damping,
        lptr, L, sptr, M, _lib.ptr(xhat), _lib.ptr(s2), _lib.ptr(gain), _lib.ptr(nu), _lib.ptr(dec),
        _lib.ptr(status), _lib.ptr(iters), None, None, _lib.stream_ptr()))
    del lv, sv, o_arr, c_arr
    if check:
        _dev.raise_status(status, iters, what=f"{kind.value}")
    return dict(xhat=xhat, sigma2=s2, nu=nu, gain=gain, dec=dec, status=status, iters=iters, n=n, u=u,
                T=t_count, single=single, lead=lead, host=host_h or host_y, C=C, lama=lama)


def _vec(x, r, tail=None):
    from .equalize import _shape_vec

    return _shape_vec(x, r["lead"], r["T"], r["single"], r["u"] if tail is None else tail)


def _sigma2_per_ue(r):
    """[n][U] (linear) or [n][T] broadcast over U (LAMA) -> API shape."""
    s2 = r["sigma2"]
    if r["lama"]:
        s2 = s2.reshape(r["n"], r["T"], 1).expand(r["n"], r["T"], r["u"]).contiguous()
        return _vec(s2, r)
    return s2.reshape(r["lead"] + (r["u"],))


def cluster_equalize(kind, h_c, y_c, n0, es=1.0, total_antennas=None, constellation=None, lama_params=None,
                     cluster_id=0):
    """One cluster's equalizer on its local statistics (fusion.py:43-75):
    LAMA runs on the system rescaled by w_c = B_c / total_antennas with
    beta_c = U / B_c; linear kinds are rescaling-invariant and run unscaled."""
    kind = Equalizer(kind)
    hshape = h_c.shape
    b_c, u = int(hshape[-2]), int(hshape[-1])
    w_c = b_c / total_antennas if total_antennas else 1.0
    r = run_fused(_lib.ARCH_PD, kind, h_c, y_c, [b_c], n0, es=es, constellation=constellation,
                  lama_params=lama_params, beta=u / b_c, lama_scale=1.0 / w_c, unbias=False,
                  want_gain=kind in (Equalizer.MRC, Equalizer.LMMSE))
    host = r["host"]
    z = _dev.out(_vec(r["xhat"], r), host)
    s2 = _dev.out(_sigma2_per_ue(r), host, real=True)
    gains = sgain = None
    if kind is Equalizer.MRC:
        gains = _dev.out(r["gain"].reshape(r["lead"] + (u,)), host, real=True)
    if kind is Equalizer.LMMSE:
        sgain = _dev.out(r["gain"].reshape(r["lead"] + (u,)), host, real=True)
    return ClusterOutput(cluster_id=cluster_id, z=z, sigma2=s2, equalizer=kind, mrc_gains=gains,
                         signal_gain=sgain)


def _unbias_cluster(out, es):
    """fusion.py:78-86."""
    if out.signal_gain is None:
        return out
    from .equalize import unbiased_output

    fixed = unbiased_output(EqualizerOutput(z=out.z, sigma2=out.sigma2, equalizer=out.equalizer,
                                            signal_gain=out.signal_gain), es)
    return ClusterOutput(cluster_id=out.cluster_id, z=fixed.z, sigma2=fixed.sigma2, equalizer=out.equalizer,
                         mrc_gains=out.mrc_gains)


def optimal_fusion_weights(sigma2):
    """nu_{c,u} proportional to 1/max(sigma2_{c,u}, 1e-15), normalised over
    clusters (fusion.py:96-105).  Accepts [C, U] or batched [..., C, U]."""
    s2, host = _dev.to_f32(sigma2)
    if s2.dim() < 2:
        raise DimensionMismatchError("expected a C x U variance matrix")
    C, u = s2.shape[-2], s2.shape[-1]
    n = s2.numel() // (C * u)
    nu = _dev.empty_f32(s2.shape)
    status = _dev.zeros_i32((n,))
    lib = _lib.lib()
    _lib.check(lib.dbp_fusion_weights(_lib.ptr(s2), n, C, u, _lib.ptr(nu), _lib.ptr(status), _lib.stream_ptr()))
    if int(status.max().item()) == _lib.ST_BADVAR:
        raise ConfigError("fusion weights need strictly positive variances")
    return FusionWeights(nu=_dev.out(nu, host, real=True))


def fuse_estimates(outputs, weights):
    """z = sum_c nu_c z_c; sigma2 = 1 / sum_c 1/max(sigma2_c, 1e-15)
    (fusion.py:108-124)."""
    outputs = list(outputs)
    if not outputs:
        raise ConfigError("cannot fuse an empty list of cluster outputs")
    t = _dev.torch()
    u = outputs[0].z.shape[-1]
    nu_d, host_nu = _dev.to_f32(weights.nu)
    if tuple(nu_d.shape[-2:]) != (len(outputs), u):
        raise DimensionMismatchError(f"weight matrix {tuple(nu_d.shape)} does not match {len(outputs)} x {u}")
    host = not _dev.is_device(outputs[0].z)
    zs = t.stack([_dev.to_c64(o.z)[0] for o in outputs])          # [C, ..., U]
    s2s = t.stack([_dev.to_f32(o.sigma2)[0] for o in outputs])    # [C, ..., U]
    nu_c = nu_d.movedim(-2, 0) if nu_d.dim() > 2 else nu_d       # [C, ..., U]
    shape = t.broadcast_shapes(zs.shape, s2s.shape, nu_c.shape)
    zs = zs.expand(shape).contiguous()
    s2b = s2s.expand(shape).contiguous()
    nub = nu_c.expand(shape).contiguous()
    count = zs[0].numel()
    z_out = _dev.empty_c64(shape[1:])
    s2_out = _dev.empty_f32(shape[1:])
    lib = _lib.lib()
    _lib.check(lib.dbp_fuse_estimates(_lib.ptr(zs), _lib.ptr(s2b), _lib.ptr(nub), len(outputs), count,
                                      _lib.ptr(z_out), _lib.ptr(s2_out), _lib.stream_ptr()))
    s2_res = s2_out  # broadcast shape of (z, sigma2, nu) per cluster
    return EqualizerOutput(z=_dev.out(z_out, host), sigma2=_dev.out(s2_res, host, real=True),
                           equalizer=outputs[0].equalizer)


def fd_equalize(kind, channel, y, n0, es=1.0, constellation=None, lama_params=None, return_weights=False):
    """Full FD pipeline over a partitioned channel (fusion.py:127-154) in one
    fused kernel launch.  With return_weights the result is an FdOutput
    carrying the fusion weights nu [..., C, U]."""
    kind = Equalizer(kind)
    counts = list(channel.partition.counts)
    r = run_fused(_lib.ARCH_FD, kind, channel.h, y, counts, n0, es=es, constellation=constellation,
                  lama_params=lama_params, unbias=True, total_antennas=channel.b)
    host = r["host"]
    z = _dev.out(_vec(r["xhat"], r), host)
    s2 = _dev.out(_sigma2_per_ue(r), host, real=True)
    if not return_weights:
        return EqualizerOutput(z=z, sigma2=s2, equalizer=kind)
    nu = r["nu"]  # [n][C][U] or [n][C][T]
    if r["lama"]:
        nu = nu.reshape(r["n"], r["C"], r["T"], 1).expand(r["n"], r["C"], r["T"], r["u"])
        nu = nu.permute(0, 2, 1, 3).contiguous()  # [n][T][C][U]
        shp = r["lead"] + ((r["C"], r["u"]) if r["single"] else (r["T"], r["C"], r["u"]))
    else:
        shp = r["lead"] + (r["C"], r["u"])
    return FdOutput(z=z, sigma2=s2, equalizer=kind, nu=_dev.out(nu.reshape(shp), host, real=True))
