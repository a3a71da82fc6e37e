"""Multi-GPU feedforward fusion: one process per GPU, antenna clusters spread
over ranks, torch.distributed (NCCL over NVLink/NVSwitch) for the one real
exchange step of the path.

The reference runs its clusters sequentially in one process
(montecarlo.py:132-135, fusion.py:141-146); the paper's system runs one
cluster per GPU and fuses with ncclReduce to a master GPU.
Here the fusion is a reduce-scatter by item (subcarrier) block, so the
central work is load-balanced and no rank is a hot spot:

  PD: stats_r = sum_{c on rank r} {G_c, y_c^mrc}       (dbp_gram_mrc, K1)
      reduce_scatter(sum)  -> rank r owns items [r n/G, (r+1) n/G)
      central equalizer + unbias + hard demap             (dbp_equalize_stats)
  FD: per local cluster: equalize, unbias, weight w_c     (dbp_equalize FD_PARTIAL)
      partial sums {sum w z, sum w, sum 1/s2}_r
      reduce_scatter(sum)  -> fused xhat, sigma2, decisions (dbp_fd_finalize)
      all_reduce(sum w)    -> nu for the local clusters   (dbp_fd_weights)

Rank layout for G ranks and C clusters: G <= C (C % G == 0) gives each rank
C/G whole clusters; G > C (G % C == 0) forms C cluster groups x G/C item
shards, the exchange running inside each shard's sub-communicator.

The per-rank compute is an ``ops`` object (default: :class:`CudaOps`, the
sm_100a kernels); tests substitute a float64 oracle implementation to check
the collective logic on CPU with the gloo backend.
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

    def stats(self, H, Y, counts):
        n = H.shape[0]
        u, t = self.u, self.t
        out = _dev.empty_c64((n, u * u + t * u))
        o, op = _lib.host_i32(np.concatenate(([0], np.cumsum(counts))))
        _lib.check(self.lib.dbp_gram_mrc(_lib.ptr(H), _lib.ptr(Y), n, H.shape[1], u, u, t, len(counts), op, 1,
                                         _lib.ptr(out), _lib.stream_ptr()))
        del o
        return out

    def solve(self, stats, n0_items, beta):
        n = stats.shape[0]
        u, t = self.u, self.t
        lama = self.kind is Equalizer.LAMA
        xhat = _dev.empty_c64((n, t, u))
        s2 = _dev.empty_f32((n, t if lama else u))
        import torch

        dec = torch.empty((n, t, u), dtype=torch.uint8, device="cuda")
        status = _dev.zeros_i32((n,))
        iters = _dev.zeros_i32((n,))
        lv, lp, L, sv, sp, M = self._c
        _lib.check(self.lib.dbp_equalize_stats(
            _lib.ptr(stats), n, u, t, _lib.KIND[self.kind.value], 0.0, _lib.ptr(n0_items), 1, float(self.es), 1,
            float(beta), 1.0, self.t_max, self.damping, lp, L, sp, M, _lib.ptr(xhat), _lib.ptr(s2), None,
            _lib.ptr(dec), _lib.ptr(status), _lib.ptr(iters), None, None, None, None, _lib.stream_ptr()))
        return xhat, s2, dec, status, iters

    def fd_partial(self, H, Y, counts, b_total, n0_items):
        import torch

        n = H.shape[0]
        u, t, wd = self.u, self.t, self.wdim
        acc = _dev.empty_f32((n, 2 * t * u + 2 * wd))
        wraw = _dev.empty_f32((n, len(counts), wd))
        status = _dev.zeros_i32((n,))
        iters = _dev.zeros_i32((n,))
        o, op = _lib.host_i32(np.concatenate(([0], np.cumsum(counts))))
        c, cp = _lib.host_i32(counts)
        lv, lp, L, sv, sp, M = self._c
        _lib.check(self.lib.dbp_equalize(
            _lib.ARCH_FD_PARTIAL, _lib.KIND[self.kind.value], _lib.ptr(H), _lib.ptr(Y), n, H.shape[1], u, u, t,
            len(counts), op, cp, int(b_total), 0.0, _lib.ptr(n0_items), 1, float(self.es), 1, 0.0, 1.0, self.t_max,
            self.damping, lp, L, sp, M, None, None, None, None, None, _lib.ptr(status), _lib.ptr(iters),
            _lib.ptr(acc), _lib.ptr(wraw), _lib.stream_ptr()))
        del o, c, torch
        return acc, wraw, status, iters

    def fd_finalize(self, acc):
        import torch

        n = acc.shape[0]
        u, t, wd = self.u, self.t, self.wdim
        xhat = _dev.empty_c64((n, t, u))
        s2 = _dev.empty_f32((n, wd))
        dec = torch.empty((n, t, u), dtype=torch.uint8, device="cuda")
        lv, lp, L, sv, sp, M = self._c
        _lib.check(self.lib.dbp_fd_finalize(_lib.ptr(acc), n, u, t, wd, lp, L, sp, M, _lib.ptr(xhat), _lib.ptr(s2),
                                            _lib.ptr(dec), _lib.stream_ptr()))
        return xhat, s2, dec

    def fd_weights(self, wraw, den):
        n, cl, wd = wraw.shape
        nu = _dev.empty_f32((n, cl, wd))
        _lib.check(self.lib.dbp_fd_weights(_lib.ptr(wraw), _lib.ptr(den.contiguous()), n, cl, wd, _lib.ptr(nu),
                                           _lib.stream_ptr()))
        return nu


@dataclass
class ShardResult:
    items: tuple            # [start, stop) of the item shard this rank finalized
    xhat: object
    sigma2: object
    decisions: object
    nu: object = None       # FD: weights of this rank's clusters, all items [n][C_r][wdim]
    status: object = None


class ClusterGroup:
    """Distributed PD / FD detector over the ranks of the default (or given)
    process group.  Each rank calls :meth:`run` with the rows of H / Y that
    belong to its clusters."""

    def __init__(self, arch, kind, counts, u, t, constellation, es=1.0, lama_params=None, ops=None):
        dist = _dist()
        self.arch = str(arch).lower()
        self.kind = Equalizer(kind)
        self.counts = [int(c) for c in counts]
        self.b_total = sum(self.counts)
        self.u, self.t = int(u), int(t)
        world, rank = dist.get_world_size(), dist.get_rank()
        self.plan = plan_ranks(world, rank, len(self.counts))
        self.ops = ops if ops is not None else CudaOps(kind, u, t, constellation, es, lama_params)
        self.group = None
        if self.plan.n_shards > 1:
            groups = [dist.new_group([s * len(self.counts) + i for i in range(len(self.counts))])
                      for s in range(self.plan.n_shards)]
            self.group = groups[self.plan.shard]
        self.local_counts = [self.counts[c] for c in self.plan.clusters]
        self.g = len(self.plan.group_ranks)
        self.gr = self.plan.group_ranks.index(rank)

    def local_rows(self):
        """Row range [a, b) of this rank's clusters in the full B axis."""
        off = np.concatenate(([0], np.cumsum(self.counts)))
        return int(off[self.plan.clusters[0]]), int(off[self.plan.clusters[-1] + 1])

    def _reduce_scatter(self, x):
        """Sum over the exchange group, item-block scattered: x [n][...] ->
        [n/g][...] (n divisible by the group size)."""
        dist = _dist()
        import torch

        n = x.shape[0]
        if n % self.g:
            raise ConfigError(f"{n} items do not split over {self.g} ranks")
        real = torch.view_as_real(x) if x.is_complex() else x
        out = torch.empty((n // self.g,) + tuple(real.shape[1:]), dtype=real.dtype, device=real.device)
        dist.reduce_scatter_tensor(out, real.contiguous(), group=self.group)
        return torch.view_as_complex(out) if x.is_complex() else out

    def run(self, H_local, Y_local, n0_items):
        """H_local [n][B_r][U], Y_local [n][T][B_r] on the ops' device;
        n0_items [n] float32 (this shard's items of the group).  Returns the
        finalized item shard of this rank (and FD weights of its clusters)."""
        dist = _dist()
        n = H_local.shape[0]
        a = self.gr * (n // self.g)
        b = a + n // self.g
        n0_shard = n0_items[a:b].contiguous()
        if self.arch == "pd":
            stats = self.ops.stats(H_local, Y_local, self.local_counts)
            mine = self._reduce_scatter(stats)
            beta = self.u / self.b_total
            xhat, s2, dec, status, iters = self.ops.solve(mine.contiguous(), n0_shard, beta)
            return ShardResult((a, b), xhat, s2, dec, None, status)
        acc, wraw, status, iters = self.ops.fd_partial(H_local, Y_local, self.local_counts, self.b_total, n0_items)
        wd = wraw.shape[-1]
        tu = 2 * self.t * self.u
        den = acc[:, tu:tu + wd].contiguous()
        dist.all_reduce(den, group=self.group)
        nu = self.ops.fd_weights(wraw, den)
        mine = self._reduce_scatter(acc)
        xhat, s2, dec = self.ops.fd_finalize(mine.contiguous())
        return ShardResult((a, b), xhat, s2, dec, nu, status)


def bench_main(args, wl, name, bench):
    """torchrun entry of bench.py for N > 1 GPUs (one process per GPU, NCCL).

    Weak scaling: frames per step grow with the number of cluster groups so
    every rank streams the same bytes of H / Y as the single-GPU run streams
    per frame batch; value = all detected bits / max-over-ranks device time."""
    import json
    import os

    import torch

    dist = _dist()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    import paper_1808_04473_b200 as dbp

    const = dbp.make_constellation(bench.CONST[wl["bits"]])
    C = wl["C"]
    counts = [wl["B"] // C] * C
    lp = {"t_max": wl["t_max"]} if wl["kind"] == "lama" else None
    grp = ClusterGroup(wl["arch"], wl["kind"], counts, wl["U"], bench.T, const, lama_params=lp)
    plan = grp.plan
    # frames per step scale with the ranks sharing one item set, so each rank
    # streams as many H / Y bytes as one GPU does for the base workload
    scale = grp.g
    frames = wl["frames"] * scale
    wl2 = dict(wl, frames=frames, snr=(wl["snr"] * scale)[:frames] if len(wl["snr"]) > 1 else wl["snr"])
    H, Y, n0, uf = bench.make_inputs(wl2, seed=1234 + plan.shard, unique_frames=2 if wl["U"] == 64 else None)
    a_row, b_row = grp.local_rows()
    n_items = frames * bench.W
    Hd = torch.empty((n_items, b_row - a_row, wl["U"]), dtype=torch.complex64, device="cuda")
    Yd = torch.empty((n_items, bench.T, b_row - a_row), dtype=torch.complex64, device="cuda")
    for f in range(frames):
        src = (f % uf) * bench.W
        Hd[f * bench.W:(f + 1) * bench.W].copy_(torch.from_numpy(H[src:src + bench.W, a_row:b_row]))
        Yd[f * bench.W:(f + 1) * bench.W].copy_(torch.from_numpy(np.ascontiguousarray(
            Y[src:src + bench.W, :, a_row:b_row])))
    n0_items = torch.tensor(np.repeat(np.asarray(n0, dtype=np.float32), bench.W), device="cuda")
    for _ in range(args.warmup):
        grp.run(Hd, Yd, n0_items)
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        grp.run(Hd, Yd, n0_items)
    e.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([s.elapsed_time(e) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    bits = frames * bench.W * bench.T * wl["U"] * wl["bits"] * plan.n_shards
    if rank == 0:
        line = {
            "metric": bench.METRIC, "value": bits / (ms * 1e-3) / 1e9, "unit": "Gb/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c64 (fp32 arithmetic)",
            "data": "synthetic i.i.d. Rayleigh (seeded)",
            "config": {"workload": bench.wl_desc(name, wl2), "parallelism":
                       f"{world} ranks: {len(plan.clusters)} cluster(s)/rank, {plan.n_shards} item shard(s); "
                       f"{'reduce-scatter of {G_c, y_c^mrc}' if wl['arch'] == 'pd' else 'reduce-scatter of fusion sums'}"
                       " over NCCL"},
            "gpu_launches": args.steps * (2 if wl["arch"] == "pd" else 3),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
