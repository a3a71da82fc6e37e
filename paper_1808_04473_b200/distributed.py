"""Multi-GPU feedforward fusion: one process per GPU, antenna clusters spread
over ranks, torch.distributed (NCCL over NVLink/NVSwitch) for the one real
exchange step of the path.

The reference runs its clusters sequentially in one process
(montecarlo.py:132-135, fusion.py:141-146); the paper's system runs one
cluster per GPU and fuses with ncclReduce to a master GPU.
Here the fusion is a reduce-scatter by item (subcarrier) block, so the
central work is load-balanced and no rank is a hot spot:

  PD: stats_r = sum_{c on rank r} {G_c, y_c^mrc}       (dbp_gram_mrc_parts, K1)
      reduce_scatter(sum)  -> rank r owns items [r n/G, (r+1) n/G)  (dbp_pd_reduce_scatter)
      central equalizer + unbias + hard demap             (dbp_equalize_stats)
  FD: per local cluster: equalize, unbias, weight w_c     (dbp_equalize FD_PARTIAL)
      partial sums {sum w z, sum w, sum 1/s2}_r
      reduce_scatter(sum)  -> fused xhat, sigma2, decisions (dbp_fd_reduce_scatter, dbp_fd_finalize)
      all_reduce(sum w)    -> nu for the local clusters   (dbp_allreduce_sum, dbp_fd_weights)

The collectives are the library's own NCCL entry points (dbp_comm_*); PyTorch
only provides the process group that shares the 128-byte NCCL id once, and
the buffers.  With chunks > 1 the exchange of one chunk overlaps the local
kernels of the next (two CUDA streams).

Rank layout for G ranks and C clusters: G <= C (C % G == 0) gives each rank
C/G whole clusters; G > C (G % C == 0) forms C cluster groups x G/C item
shards, the exchange running inside each shard's sub-communicator.

The per-rank compute is an ``ops`` object (default: :class:`CudaOps`, the
sm_100a kernels) and the collectives an ``exchange`` (default for CUDA ops:
:class:`NcclExchange`); tests substitute a float64 oracle implementation and
:class:`TorchExchange` to check the collective logic on CPU with the gloo
backend.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .equalize import Equalizer
from .errors import ConfigError


def _dist():
    import torch.distributed as dist

    return dist


@dataclass
class RankPlan:
    world: int
    rank: int
    clusters: list          # global cluster indices owned by this rank
    shard: int              # item shard index (G > C) else 0
    n_shards: int
    group_ranks: list       # ranks taking part in this rank's exchange


def plan_ranks(world, rank, n_clusters):
    if world <= n_clusters:
        if n_clusters % world:
            raise ConfigError(f"C={n_clusters} clusters cannot be split evenly over {world} ranks")
        per = n_clusters // world
        return RankPlan(world, rank, list(range(rank * per, (rank + 1) * per)), 0, 1, list(range(world)))
    if world % n_clusters:
        raise ConfigError(f"{world} ranks cannot be split into C={n_clusters} cluster groups")
    shards = world // n_clusters
    shard, c = rank // n_clusters, rank % n_clusters
    return RankPlan(world, rank, [c], shard, shards, [shard * n_clusters + i for i in range(n_clusters)])


class CudaOps:
    """Per-rank compute on the sm_100a kernels (device tensors)."""

    device = "cuda"

    def __init__(self, kind, u, t, constellation, es=1.0, lama_params=None):
        self.kind = Equalizer(kind)
        self.u, self.t = u, t
        self.const = constellation
        self.es = constellation.es if self.kind is Equalizer.LAMA else es
        lp = dict(lama_params or {})
        self.t_max = int(lp.get("t_max", 10))
        self.damping = float(lp.get("damping", 1.0))
        self.wdim = t if self.kind is Equalizer.LAMA else u
        self._c = _dev.const_params(constellation)
        self.lib = _lib.lib()
        self._bufs = {}
        self._offs = {}
        self.bf16_parts = 0  # statistics kernels' default (3 parts); ClusterGroup may choose 2

    def _buf(self, key, shape, dtype):
        """Reusable device output buffer (a detector step allocates nothing)."""
        import torch

        k = (key, tuple(shape), dtype)
        b = self._bufs.get(k)
        if b is None:
            b = self._bufs[k] = torch.empty(tuple(shape), dtype=dtype, device="cuda")
        return b

    def _off(self, counts):
        k = tuple(counts)
        if k not in self._offs:
            self._offs[k] = (_lib.host_i32(np.concatenate(([0], np.cumsum(counts)))), _lib.host_i32(counts))
        return self._offs[k]

    def stats(self, H, Y, counts, tag=0):
        import torch

        n = H.shape[0]
        u, t = self.u, self.t
        out = self._buf(("stats", tag), (n, u * u + t * u), torch.complex64)
        (o, op), _ = self._off(counts)
        _lib.check(self.lib.dbp_gram_mrc_parts(_lib.ptr(H), _lib.ptr(Y), n, H.shape[1], u, u, t, len(counts), op, 1,
                                               self.bf16_parts, _lib.ptr(out), _lib.stream_ptr()))
        return out

    def solve(self, stats, n0_items, beta, tag=0):
        import torch

        n = stats.shape[0]
        u, t = self.u, self.t
        lama = self.kind is Equalizer.LAMA
        xhat = self._buf(("xhat", tag), (n, t, u), torch.complex64)
        s2 = self._buf(("s2", tag), (n, t if lama else u), torch.float32)
        dec = self._buf(("dec", tag), (n, t, u), torch.uint8)
        status = self._buf(("status", tag), (n,), torch.int32)
        iters = self._buf(("iters", tag), (n,), torch.int32)
        lv, lp, L, sv, sp, M = self._c
        _lib.check(self.lib.dbp_equalize_stats(
            _lib.ptr(stats), n, u, t, _lib.KIND[self.kind.value], 0.0, _lib.ptr(n0_items), 1, float(self.es), 1,
            float(beta), 1.0, self.t_max, self.damping, lp, L, sp, M, _lib.ptr(xhat), _lib.ptr(s2), None,
            _lib.ptr(dec), _lib.ptr(status), _lib.ptr(iters), None, None, None, None, _lib.stream_ptr()))
        return xhat, s2, dec, status, iters

    def fd_partial(self, H, Y, counts, b_total, n0_items, tag=0):
        import torch

        n = H.shape[0]
        u, t, wd = self.u, self.t, self.wdim
        acc = self._buf(("acc", tag), (n, 2 * t * u + 2 * wd), torch.float32)
        wraw = self._buf(("wraw", tag), (n, len(counts), wd), torch.float32)
        status = self._buf(("status_p", tag), (n,), torch.int32)
        iters = self._buf(("iters_p", tag), (n,), torch.int32)
        (o, op), (c, cp) = self._off(counts)
        lv, lp, L, sv, sp, M = self._c
        _lib.check(self.lib.dbp_equalize(
            _lib.ARCH_FD_PARTIAL, _lib.KIND[self.kind.value], _lib.ptr(H), _lib.ptr(Y), n, H.shape[1], u, u, t,
            len(counts), op, cp, int(b_total), 0.0, _lib.ptr(n0_items), 1, float(self.es), 1, 0.0, 1.0, self.t_max,
            self.damping, lp, L, sp, M, None, None, None, None, None, _lib.ptr(status), _lib.ptr(iters),
            _lib.ptr(acc), _lib.ptr(wraw), _lib.stream_ptr()))
        return acc, wraw, status, iters

    def fd_finalize(self, acc, tag=0):
        import torch

        n = acc.shape[0]
        u, t, wd = self.u, self.t, self.wdim
        xhat = self._buf(("xhat", tag), (n, t, u), torch.complex64)
        s2 = self._buf(("s2", tag), (n, wd), torch.float32)
        dec = self._buf(("dec", tag), (n, t, u), torch.uint8)
        lv, lp, L, sv, sp, M = self._c
        _lib.check(self.lib.dbp_fd_finalize(_lib.ptr(acc), n, u, t, wd, lp, L, sp, M, _lib.ptr(xhat), _lib.ptr(s2),
                                            _lib.ptr(dec), _lib.stream_ptr()))
        return xhat, s2, dec

    def fd_weights(self, wraw, den, tag=0):
        import torch

        n, cl, wd = wraw.shape
        nu = self._buf(("nu", tag), (n, cl, wd), torch.float32)
        _lib.check(self.lib.dbp_fd_weights(_lib.ptr(wraw), _lib.ptr(den.contiguous()), n, cl, wd, _lib.ptr(nu),
                                           _lib.stream_ptr()))
        return nu


@dataclass
class ShardResult:
    items: object           # global item indices this rank finalized (int64 array, in output order)
    xhat: object
    sigma2: object
    decisions: object
    nu: object = None       # FD: weights of this rank's clusters, all items [n][C_r][wdim]
    status: object = None


class TorchExchange:
    """The exchange through torch.distributed collectives (CPU gloo tests with
    oracle ops)."""

    def __init__(self, group=None):
        self.group = group

    def reduce_scatter(self, x, g, **_):
        dist = _dist()
        import torch

        n = x.shape[0]
        real = torch.view_as_real(x) if x.is_complex() else x
        out = torch.empty((n // g,) + tuple(real.shape[1:]), dtype=real.dtype, device=real.device)
        dist.reduce_scatter_tensor(out, real.contiguous(), group=self.group)
        return torch.view_as_complex(out) if x.is_complex() else out

    def all_reduce(self, x, **_):
        _dist().all_reduce(x, group=self.group)
        return x

    def close(self):
        pass


class NcclExchange:
    """The exchange through the library's NCCL entry points (dbp_comm_*,
    include/dbp_b200.h): PyTorch only hands over buffers and, once, the
    128-byte NCCL id (broadcast inside the exchange group)."""

    def __init__(self, plan, group=None):
        import ctypes as C

        dist = _dist()
        self.lib = _lib.lib()
        self.g = len(plan.group_ranks)
        self.gr = plan.group_ranks.index(plan.rank)
        idbuf = (C.c_char * 128)()
        if self.gr == 0:
            _lib.check(self.lib.dbp_comm_unique_id(idbuf))
        obj = [bytes(idbuf)]
        dist.broadcast_object_list(obj, src=plan.group_ranks[0], group=group)
        idbuf = (C.c_char * 128).from_buffer_copy(obj[0])
        self.comm = C.c_void_p()
        _lib.check(self.lib.dbp_comm_init(idbuf, self.g, self.gr, C.byref(self.comm)))

    def reduce_scatter(self, x, g, kind="pd", u=0, t=0, wdim=0, stream=None):
        import torch

        n = x.shape[0]
        out = torch.empty((n // g,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        if kind == "pd":
            _lib.check(self.lib.dbp_pd_reduce_scatter(self.comm, _lib.ptr(x), _lib.ptr(out), n // g, u, t,
                                                      _lib.stream_ptr(stream)))
        else:
            _lib.check(self.lib.dbp_fd_reduce_scatter(self.comm, _lib.ptr(x), _lib.ptr(out), n // g, u, t, wdim,
                                                      _lib.stream_ptr(stream)))
        return out

    def all_reduce(self, x, stream=None):
        _lib.check(self.lib.dbp_allreduce_sum(self.comm, _lib.ptr(x), x.numel(), _lib.stream_ptr(stream)))
        return x

    def close(self):
        if self.comm:
            _lib.check(self.lib.dbp_comm_destroy(self.comm))
            self.comm = None


class ClusterGroup:
    """Distributed PD / FD detector over the ranks of the default (or given)
    process group.  Each rank calls :meth:`run` with the rows of H / Y that
    belong to its clusters.

    The fusion runs through ``exchange``: the library's NCCL entry points for
    the CUDA ops (default), torch.distributed collectives otherwise.  With
    ``chunks`` > 1 the items are processed in chunks so that the exchange of
    chunk k overlaps the local statistics / partial sums of chunk k + 1 (two
    CUDA streams); rank r then finalizes block r of every chunk."""

    def __init__(self, arch, kind, counts, u, t, constellation, es=1.0, lama_params=None, ops=None, exchange=None):
        dist = _dist()
        self.arch = str(arch).lower()
        self.kind = Equalizer(kind)
        self.counts = [int(c) for c in counts]
        self.b_total = sum(self.counts)
        self.u, self.t = int(u), int(t)
        world, rank = dist.get_world_size(), dist.get_rank()
        self.plan = plan_ranks(world, rank, len(self.counts))
        self.ops = ops if ops is not None else CudaOps(kind, u, t, constellation, es, lama_params)
        # PD linear equalization of a well-conditioned system (B >= 4 u, as the
        # fused single-GPU PD kernel decides it): two bf16 parts in the partial
        # statistics (cfg2, one rank: 71 -> 50 us per 6,600-item chunk)
        if isinstance(self.ops, CudaOps) and arch == "pd" and Equalizer(kind) is not Equalizer.LAMA \
                and self.b_total >= 4 * u:
            self.ops.bf16_parts = 2
        self.group = None
        if self.plan.n_shards > 1:
            groups = [dist.new_group([s * len(self.counts) + i for i in range(len(self.counts))])
                      for s in range(self.plan.n_shards)]
            self.group = groups[self.plan.shard]
        self.local_counts = [self.counts[c] for c in self.plan.clusters]
        self.g = len(self.plan.group_ranks)
        self.gr = self.plan.group_ranks.index(rank)
        if exchange is None:
            exchange = (NcclExchange(self.plan, self.group) if getattr(self.ops, "device", "cpu") == "cuda"
                        else TorchExchange(self.group))
        self.exchange = exchange

    def local_rows(self):
        """Row range [a, b) of this rank's clusters in the full B axis."""
        off = np.concatenate(([0], np.cumsum(self.counts)))
        return int(off[self.plan.clusters[0]]), int(off[self.plan.clusters[-1] + 1])

    def owned_items(self, n, chunks=1):
        """Global item indices this rank finalizes, in output order."""
        m = n // chunks
        return np.concatenate([k * m + self.gr * (m // self.g) + np.arange(m // self.g) for k in range(chunks)])

    def exchanged_bytes(self, n):
        """Bytes this rank contributes to the exchange for n items (unpacked
        records, the reference's message_volume per cluster group)."""
        u, t = self.u, self.t
        if self.arch == "pd":
            return n * (u * u + t * u) * 8
        wd = t if self.kind is Equalizer.LAMA else u
        return n * (2 * t * u + 2 * wd) * 4 + n * wd * 4

    def run(self, H_local, Y_local, n0_items, chunks=1):
        """H_local [n][B_r][U], Y_local [n][T][B_r] on the ops' device;
        n0_items [n] float32 (this shard's items of the group).  Returns the
        items this rank finalized (and FD weights of its clusters)."""
        n = H_local.shape[0]
        if n % (chunks * self.g):
            raise ConfigError(f"{n} items do not split into {chunks} chunks over {self.g} ranks")
        m = n // chunks
        cuda = getattr(self.ops, "device", "cpu") == "cuda"
        streams = None
        if cuda and chunks > 1:
            import torch

            cur = torch.cuda.current_stream()
            if getattr(self, "_streams", None) is None:
                self._streams = (torch.cuda.Stream(), torch.cuda.Stream())
            streams = self._streams
            for s_ in streams:
                s_.wait_stream(cur)
        outs, nus = [], []
        for k in range(chunks):
            sl = slice(k * m, (k + 1) * m)
            a = k * m + self.gr * (m // self.g)
            mine_n0 = n0_items[a:a + m // self.g].contiguous()
            if streams is None:
                outs.append(self._chunk(H_local[sl], Y_local[sl], n0_items[sl], mine_n0, nus, None, None, k))
            else:
                outs.append(self._chunk(H_local[sl], Y_local[sl], n0_items[sl], mine_n0, nus, *streams, k))
        if streams is not None:
            import torch

            cur = torch.cuda.current_stream()
            for s_ in streams:
                cur.wait_stream(s_)
        items = self.owned_items(n, chunks)
        cat = self._cat
        xhat, s2, dec = cat([o[0] for o in outs]), cat([o[1] for o in outs]), cat([o[2] for o in outs])
        status = cat([o[3] for o in outs])
        nu = cat(nus) if nus else None
        return ShardResult(items, xhat, s2, dec, nu, status)

    @staticmethod
    def _cat(xs):
        import torch

        return xs[0] if len(xs) == 1 else torch.cat(xs, 0)

    def _chunk(self, H, Y, n0_chunk, n0_mine, nus, s_comp, s_comm, tag=0):
        """One chunk: local compute on s_comp, exchange on s_comm (None: the
        current stream), finalize on s_comp."""
        import contextlib

        import torch

        def on(s):
            return torch.cuda.stream(s) if s is not None else contextlib.nullcontext()

        ex = self.exchange
        u, t = self.u, self.t
        if self.arch == "pd":
            with on(s_comp):
                stats = self.ops.stats(H, Y, self.local_counts, **self._tag(tag))
            if s_comm is not None:
                s_comm.wait_stream(s_comp)
            with on(s_comm):
                mine = ex.reduce_scatter(stats, self.g, kind="pd", u=u, t=t, stream=s_comm)
            if s_comm is not None:
                s_comp.wait_stream(s_comm)
            with on(s_comp):
                beta = self.u / self.b_total
                xhat, s2, dec, status, iters = self.ops.solve(mine.contiguous(), n0_mine, beta, **self._tag(tag))
            return xhat, s2, dec, status
        with on(s_comp):
            acc, wraw, status, iters = self.ops.fd_partial(H, Y, self.local_counts, self.b_total, n0_chunk,
                                                           **self._tag(tag))
            wd = wraw.shape[-1]
            tu = 2 * t * u
            den = acc[:, tu:tu + wd].contiguous()
        if s_comm is not None:
            s_comm.wait_stream(s_comp)
        with on(s_comm):
            ex.all_reduce(den, stream=s_comm)
            mine = ex.reduce_scatter(acc, self.g, kind="fd", u=u, t=t, wdim=wd, stream=s_comm)
        if s_comm is not None:
            s_comp.wait_stream(s_comm)
        with on(s_comp):
            nus.append(self.ops.fd_weights(wraw, den, **self._tag(tag)))
            xhat, s2, dec = self.ops.fd_finalize(mine.contiguous(), **self._tag(tag))
        # local fault flags of this rank's clusters for the items it finalizes
        m = H.shape[0]
        a = self.gr * (m // self.g)
        return xhat, s2, dec, (status[a:a + m // self.g] if status is not None else None)

    def _tag(self, k):
        """Per-chunk buffer tag for ops that cache their outputs (CudaOps)."""
        return {"tag": k} if isinstance(self.ops, CudaOps) else {}

    def close(self):
        self.exchange.close()


def bench_main(args, wl, name, bench):
    """torchrun entry of bench.py for N > 1 GPUs (one process per GPU).

    Weak scaling: frames per step grow with the number of cluster groups so
    every rank streams the same bytes of H / Y as the single-GPU run streams
    per frame batch; value = all detected bits / max-over-ranks device time.
    The exchange runs through the library's NCCL entry points, in chunks so it
    overlaps the local kernels.  torch.distributed (NCCL) only shares the NCCL
    id, runs the barriers and the max-over-ranks of the timings."""
    import json
    import os

    import torch

    dist = _dist()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    import paper_1808_04473_b200 as dbp
    from paper_1808_04473_b200.synth import snr_to_n0, synth_device

    const = dbp.make_constellation(bench.CONST[wl["bits"]])
    C = wl["C"]
    counts = [wl["B"] // C] * C
    lp = {"t_max": wl["t_max"]} if wl["kind"] == "lama" else None
    grp = ClusterGroup(wl["arch"], wl["kind"], counts, wl["U"], bench.T, const, lama_params=lp)
    plan = grp.plan
    scale = grp.g
    frames = wl["frames"] * scale
    wl2 = dict(wl, frames=frames, snr=(bench.frame_snrs(wl) * scale)[:frames])
    W, T = bench.W, bench.T
    n_items = frames * W
    chunks = max(1, int(getattr(args, "chunks", 4)))
    while n_items % (chunks * grp.g):
        chunks -= 1
    n0 = snr_to_n0(bench.frame_snrs(wl2), const.es)
    n0_frames = torch.tensor(np.asarray(n0, dtype=np.float32), device="cuda")
    n0_items = torch.repeat_interleave(n0_frames, W)
    a_row, b_row = grp.local_rows()
    # this shard's frames (each item shard of a G > C run has its own), this rank's rows
    Hf, Yf = synth_device(1234 + plan.shard, n_items, wl["B"], wl["U"], T, const, n0_dev=n0_frames, n0_group=W)
    Hd = Hf[:, a_row:b_row].contiguous()
    Yd = Yf[:, :, a_row:b_row].contiguous()
    del Hf, Yf
    for _ in range(args.warmup):
        grp.run(Hd, Yd, n0_items, chunks=chunks)
    torch.cuda.synchronize()
    # one step (all chunks, kernels and NCCL calls on two streams) captured as
    # a CUDA graph: the host cost of the chunked schedule is paid once
    graph = None
    if not getattr(args, "no_graph", False):
        try:
            graph = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                grp.run(Hd, Yd, n0_items, chunks=chunks)  # warm the caching allocator on this stream
            torch.cuda.current_stream().wait_stream(cs)
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=cs):
                grp.run(Hd, Yd, n0_items, chunks=chunks)
            torch.cuda.synchronize()
        except Exception as exc:  # capture unsupported: run eagerly
            if rank == 0:
                print(f"[bench] CUDA graph capture failed ({exc}); eager steps", flush=True)
            graph = None
            torch.cuda.synchronize()

    def step():
        if graph is not None:
            graph.replay()
        else:
            grp.run(Hd, Yd, n0_items, chunks=chunks)

    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        step()
    e.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms_t = torch.tensor([s.elapsed_time(e) / args.steps], device="cuda")
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    bits = frames * W * T * wl["U"] * wl["bits"] * plan.n_shards
    # roofline: this rank's HBM bytes (its H / Y rows, its finalized outputs)
    # and NVLink bytes (what it sends into the exchange, unpacked records)
    b_r = b_row - a_row
    own = n_items // grp.g
    wd = T if wl["kind"] == "lama" else wl["U"]
    hbm = n_items * (8 * b_r * wl["U"] + 8 * T * b_r) + own * (8 * T * wl["U"] + 4 * wd + T * wl["U"] + 4)
    nvl = grp.exchanged_bytes(n_items) * (grp.g - 1) // max(grp.g, 1)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(bench.REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # ---- end to end: pinned host H / Y of this rank -> H2D, run, D2H of its outputs
    Hh = torch.empty(Hd.shape, dtype=torch.complex64, pin_memory=True)
    Yh = torch.empty(Yd.shape, dtype=torch.complex64, pin_memory=True)
    Hh.copy_(Hd)
    Yh.copy_(Yd)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, min(args.steps, 5))
    dist.barrier()
    e0.record()
    xh = dec = None
    for _ in range(reps):
        Hd.copy_(Hh, non_blocking=True)
        Yd.copy_(Yh, non_blocking=True)
        res = grp.run(Hd, Yd, n0_items, chunks=chunks)
        xh = res.xhat.cpu()
        dec = res.decisions.cpu()
    e1.record()
    torch.cuda.synchronize()
    ems_t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
    dist.all_reduce(ems_t, op=dist.ReduceOp.MAX)
    ems = float(ems_t.item())
    cpu = None
    if rank == 0 and not getattr(args, "no_cpu", False):
        Hs = Hh[:2 * W].numpy()
        Ys = Yh[:2 * W].numpy()
        cb = bench.CpuBaseline(dict(wl, B=b_r, C=len(grp.local_counts)), Hs, Ys, np.repeat(n0[:2], W))
        rate, n_s, wall = cb.run(min(args.cpu_seconds, 10.0))
        cb.close()
        cpu = {"value": rate, "unit": "Gb/s", "cores": cb.cores, "kind": "port",
               "sample": f"rank 0's clusters on {n_s} items x {T} symbols through the per-vector oracle port "
                         f"({wall:.1f} s wall, {bench.cpu_model()})"}
    if rank == 0:
        par = (f"{world} ranks: {len(plan.clusters)} cluster(s)/rank, {plan.n_shards} item shard(s); "
               f"{'reduce-scatter of {G_c, y_c^mrc}' if wl['arch'] == 'pd' else 'reduce-scatter of fusion sums'}"
               f" over NCCL (dbp_comm_*), {chunks} chunk(s) overlapped"
               f"{', one CUDA graph per step' if graph is not None else ''}")
        line = {
            "metric": bench.METRIC, "value": bits / (ms * 1e-3) / 1e9, "unit": "Gb/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c64 (fp32 arithmetic)",
            "data": "synthetic i.i.d. Rayleigh, generated on the GPU (dbp_synthesize, seeded)",
            "config": dict(bench.config_dict(name, wl2, par),
                           l2=f"inputs {(Hd.numel() + Yd.numel()) * 8 / 2**20:.0f} MiB/step per rank vs 126 MiB L2; "
                              f"one input set"),
            "roofline": {"bound": "hbm", "achieved": hbm / (ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": hbm / (ms * 1e-3) / 1e9 / hbm_peak, "traffic": None,
                         "algorithmic_bytes_per_launch": hbm, "per": "rank",
                         "nvlink": {"bytes_per_rank": nvl, "achieved": nvl / (ms * 1e-3) / 1e9, "peak": 900.0,
                                    "unit": "GB/s", "peak_source": "nominal NVLink 5 per direction (not measured)"}},
            "cpu_baseline": cpu,
            "e2e": {"value": bits / (ems * 1e-3) / 1e9, "unit": "Gb/s",
                    "h2d_bytes_per_step": int((Hh.numel() + Yh.numel()) * 8),
                    "d2h_bytes_per_step": int(xh.numel() * 8 + dec.numel()), "ms_per_step": ems},
            "gpu_launches": args.steps * chunks * (2 if wl["arch"] == "pd" else 3),
        }
        print(json.dumps(line), flush=True)
    grp.close()
    dist.destroy_process_group()
