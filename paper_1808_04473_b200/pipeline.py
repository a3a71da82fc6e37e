"""Batched hot-path API: whole frames of (subcarrier x OFDM symbol) vectors in
one fused kernel launch.

This is the form in which a receiver runs the path (the
Gram per subcarrier reused over the N_sym OFDM symbols, all subcarriers in
parallel); the per-vector reference API in :mod:`.equalize` / :mod:`.fusion`
is a thin view of the same kernels.

Layouts: H [n][B][U] (n = frames x subcarriers), Y [n][T][B], complex64.
Results: xhat [n][T][U] (PD linear: unbiased z/c as montecarlo._equalize
detects on; LAMA: z^{t_max}; FD: fused estimate), sigma2 [n][U] (linear) or
[n][T] (LAMA), nu [n][C][U] / [n][C][T] (FD), decisions [n][T][U] uint8
symbol indices (k = i*L + j; Gray labels via model.gray_labels).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .equalize import Equalizer
from .errors import ConfigError, DimensionMismatchError


@dataclass
class Detection:
    xhat: object
    sigma2: object
    decisions: object
    nu: object = None
    status: object = None
    iters: object = None

    def raise_on_error(self):
        _dev.raise_status(self.status, self.iters, what="detect")
        return self


class Detector:
    """Preallocated single-GPU detector for one configuration.

    arch: "pd" or "fd"; kind: mrc / zf / lmmse / lama; counts: antennas per
    cluster (e.g. ClusterPartition.counts).  ``run`` takes device-resident
    H, Y and launches exactly one kernel; ``run_host`` streams host (pinned)
    buffers through the GPU in chunks with the copies overlapped.

    Any partition the reference accepts works: an odd U or an odd cluster size
    is zero-padded on the device (zero UE columns and zero antenna rows change
    neither G's leading block nor y_mrc), with the real cluster sizes passed
    for the FD weights w_c and beta_c (fusion.py:60-68).  The kernels cover
    U <= 64 and T <= 16.
    """

    def __init__(self, arch, kind, n_items, b, u, t, counts, constellation, es=None, lama_params=None):
        self.arch = {"pd": _lib.ARCH_PD, "fd": _lib.ARCH_FD}[str(arch).lower()]
        self.kind = Equalizer(kind)
        self.n, self.b, self.u, self.t = int(n_items), int(b), int(u), int(t)
        self.counts = [int(c) for c in counts]
        if sum(self.counts) != self.b:
            raise DimensionMismatchError("cluster counts do not sum to B")
        if any(c < 1 for c in self.counts):
            raise ConfigError("every cluster needs at least one antenna")
        # even row / column strides for the kernels (zero padding, see above)
        self.us = self.u + (self.u % 2)
        self.pcounts = [c + (c % 2) for c in self.counts]
        self.pb = sum(self.pcounts)
        self.padded = self.us != self.u or self.pb != self.b
        if self.t > 16 or self.u > 64:
            raise ConfigError("Detector supports T <= 16 and U <= 64")
        self.const = constellation
        self.es = constellation.es if es is None else float(es)
        lp = dict(lama_params or {})
        self.t_max = int(lp.get("t_max", 10))
        self.damping = float(lp.get("damping", 1.0))
        self.lama = self.kind is Equalizer.LAMA
        self.wdim = self.t if self.lama else self.u
        self.C = len(self.counts)
        t_ = _dev.torch()
        self.xhat = _dev.empty_c64((self.n, self.t, self.u))
        self.sigma2 = _dev.empty_f32((self.n, self.wdim))
        self.nu = _dev.empty_f32((self.n, self.C, self.wdim)) if self.arch == _lib.ARCH_FD else None
        self.dec = t_.empty((self.n, self.t, self.u), dtype=t_.uint8, device="cuda")
        self.status = _dev.zeros_i32((self.n,))
        self.iters = _dev.zeros_i32((self.n,))
        self._lv, self._lp, self._L, self._sv, self._sp, self._M = _dev.const_params(constellation)
        self._off, self._offp = _lib.host_i32(np.concatenate(([0], np.cumsum(self.pcounts))))
        self._cnt, self._cntp = _lib.host_i32(self.counts)
        self._lib = _lib.lib()
        self.launches = 0

    def _launch(self, H, Y, n, n0, n0_dev, n0_group, out_off=0, stream=None):
        o = out_off
        xh = self.xhat[o:o + n]
        s2 = self.sigma2[o:o + n]
        nu = self.nu[o:o + n] if self.nu is not None else None
        dec = self.dec[o:o + n]
        st = self.status[o:o + n]
        it = self.iters[o:o + n]
        if self.padded:
            H, Y = self._pad(H, Y, n)
        _lib.check(self._lib.dbp_equalize(
            self.arch, _lib.KIND[self.kind.value], _lib.ptr(H), _lib.ptr(Y), n, self.pb, self.u, self.us, self.t,
            self.C, self._offp, self._cntp, self.b, float(n0), _lib.ptr(n0_dev), int(n0_group), float(self.es), 1,
            float(self.u / self.b), 1.0, self.t_max, self.damping, self._lp, self._L, self._sp, self._M,
            _lib.ptr(xh), _lib.ptr(s2), None, _lib.ptr(nu), _lib.ptr(dec), _lib.ptr(st), _lib.ptr(it), None,
            None, _lib.stream_ptr(stream)))
        self.launches += 1

    def _pad(self, H, Y, n):
        """Zero-padded copies [n][pB][us], [n][T][pB] (odd U / odd clusters)."""
        t_ = _dev.torch()
        hp = t_.zeros((n, self.pb, self.us), dtype=t_.complex64, device=H.device)
        yp = t_.zeros((n, self.t, self.pb), dtype=t_.complex64, device=Y.device)
        a = a2 = 0
        for c, pc in zip(self.counts, self.pcounts):
            hp[:, a2:a2 + c, :self.u] = H[:n, a:a + c]
            yp[:, :, a2:a2 + c] = Y[:n, :, a:a + c]
            a += c
            a2 += pc
        return hp, yp

    def _check_n0(self, n, n0_dev, n0_group):
        if n0_dev is None:
            return
        if n0_group < 1 or n0_dev.numel() * n0_group < n:
            raise DimensionMismatchError(
                f"n0_dev has {n0_dev.numel()} values for {n} items in groups of {n0_group}")

    def run(self, H, Y, n0=0.0, n0_dev=None, n0_group=1, check=False):
        """H [n][B][U], Y [n][T][B] complex64 CUDA tensors (contiguous).
        n0: scalar, or n0_dev float32 CUDA tensor with item i using
        n0_dev[i // n0_group]."""
        if tuple(H.shape) != (self.n, self.b, self.u) or tuple(Y.shape) != (self.n, self.t, self.b):
            raise DimensionMismatchError("H / Y do not match the detector geometry")
        self._check_n0(self.n, n0_dev, n0_group)
        self._launch(H, Y, self.n, n0, n0_dev, n0_group)
        det = Detection(self.xhat, self.sigma2, self.dec, self.nu, self.status, self.iters)
        return det.raise_on_error() if check else det

    def alloc_host_outputs(self):
        """Pinned host buffers for run_host()."""
        t_ = _dev.torch()
        outs = dict(xhat=t_.empty(self.xhat.shape, dtype=t_.complex64, pin_memory=True),
                    sigma2=t_.empty(self.sigma2.shape, dtype=t_.float32, pin_memory=True),
                    dec=t_.empty(self.dec.shape, dtype=t_.uint8, pin_memory=True),
                    status=t_.empty(self.status.shape, dtype=t_.int32, pin_memory=True))
        if self.nu is not None:
            outs["nu"] = t_.empty(self.nu.shape, dtype=t_.float32, pin_memory=True)
        return outs

    def run_host(self, H_host, Y_host, outs, n0=0.0, n0_dev=None, n0_group=1, chunks=8, bufs=None):
        """End-to-end call on pinned host tensors: per chunk of items, H2D on
        one stream, the fused kernel on another, D2H of the results on a
        third, so PCIe traffic overlaps compute.  Returns bytes moved
        (h2d, d2h).  Caller synchronizes."""
        t_ = _dev.torch()
        self._check_n0(self.n, n0_dev, n0_group)
        if bufs is None:
            bufs = self.device_staging(chunks)
        h2d, comp, d2h = bufs["streams"]
        Hd, Yd = bufs["H"], bufs["Y"]
        step = (self.n + chunks - 1) // chunks
        cur = t_.cuda.current_stream()
        h2d.wait_stream(cur)
        bi = bo = 0
        ev_free = bufs["free"]
        for k, a in enumerate(range(0, self.n, step)):
            m = min(step, self.n - a)
            slot = k % 2
            with t_.cuda.stream(h2d):
                h2d.wait_event(ev_free[slot])
                Hd[slot][:m].copy_(H_host[a:a + m], non_blocking=True)
                Yd[slot][:m].copy_(Y_host[a:a + m], non_blocking=True)
                bi += H_host[a:a + m].numel() * 8 + Y_host[a:a + m].numel() * 8
                ev_in = t_.cuda.Event()
                ev_in.record(h2d)
            comp.wait_event(ev_in)
            g = n0_group
            nd = n0_dev
            if n0_dev is not None and n0_group > 1 and a % n0_group:
                raise ConfigError("chunk boundaries must align with the n0 groups")
            if n0_dev is not None:
                nd = n0_dev[a // n0_group:]
            self._launch(Hd[slot][:m], Yd[slot][:m], m, n0, nd, g, out_off=a, stream=comp)
            ev_done = t_.cuda.Event()
            ev_done.record(comp)
            ev_free[slot].record(comp)
            d2h.wait_event(ev_done)
            with t_.cuda.stream(d2h):
                for key in outs:
                    src = getattr(self, key)[a:a + m]
                    outs[key][a:a + m].copy_(src, non_blocking=True)
                    bo += src.numel() * src.element_size()
        cur.wait_stream(d2h)
        return bi, bo

    def device_staging(self, chunks=8):
        t_ = _dev.torch()
        step = (self.n + chunks - 1) // chunks
        return dict(
            streams=(t_.cuda.Stream(), t_.cuda.Stream(), t_.cuda.Stream()),
            H=[_dev.empty_c64((step, self.b, self.u)) for _ in range(2)],
            Y=[_dev.empty_c64((step, self.t, self.b)) for _ in range(2)],
            free=[t_.cuda.Event() for _ in range(2)])


def detect(arch, kind, H, Y, n0, counts, constellation, lama_params=None, n0_group=None, check=True):
    """One-shot batched detection (device or host arrays).  n0 may be a
    scalar or an array with one value per group of ``n0_group`` items
    (default: per item)."""
    Hd, host_h = _dev.to_c64(H)
    Yd, host_y = _dev.to_c64(Y)
    if Hd.dim() != 3 or Yd.dim() != 3:
        raise DimensionMismatchError("detect expects H [n][B][U] and Y [n][T][B]")
    n, b, u = Hd.shape
    t = Yd.shape[1]
    det = Detector(arch, kind, n, b, u, t, counts, constellation, lama_params=lama_params)
    n0a = np.asarray(n0, dtype=np.float32).reshape(-1)
    if n0a.size == 1:
        out = det.run(Hd, Yd, float(n0a[0]))
    else:
        grp = int(n0_group) if n0_group else max(1, n // n0a.size)
        if grp * n0a.size != n:
            raise DimensionMismatchError(f"{n0a.size} noise values do not cover {n} items in groups of {grp}")
        out = det.run(Hd, Yd, 0.0, _dev.to_f32(n0a)[0], grp)
    if check:
        out.raise_on_error()
    host = host_h or host_y
    if host:
        return Detection(xhat=out.xhat.cpu().numpy(), sigma2=out.sigma2.cpu().numpy(),
                         decisions=out.decisions.cpu().numpy(),
                         nu=None if out.nu is None else out.nu.cpu().numpy(),
                         status=out.status.cpu().numpy(), iters=out.iters.cpu().numpy())
    return out
