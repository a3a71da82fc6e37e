"""Multi-rank feedforward fusion (paper_1808_04473_b200.distributed) on CPU
with the gloo backend.  The per-rank kernels are replaced by a float64 oracle
implementation (same contracts as CudaOps), so what is tested here is the
rank plan, the data layout of the exchanged statistics / fusion sums, the
reduce-scatter item sharding and the weight all-reduce: the result on every
rank must equal the single-process reference path on that rank's items."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dbp_oracle as O

T = 3


class OracleOps:
    device = "cpu"

    def __init__(self, kind, u, t, bits, t_max=4):
        self.kind, self.u, self.t = kind, u, t
        self.syms, _ = O.square_qam(bits)
        self.lp = {"t_max": t_max} if kind == "lama" else None
        self.wdim = t if kind == "lama" else u

    def stats(self, H, Y, counts):
        H, Y = H.numpy(), Y.numpy()
        off = np.concatenate(([0], np.cumsum(counts)))
        u, t = self.u, self.t
        out = np.zeros((H.shape[0], u * u + t * u), dtype=np.complex128)
        for n in range(H.shape[0]):
            g = sum(O.gram_mrc(H[n, off[c]:off[c + 1]], Y[n, 0, off[c]:off[c + 1]])[0] for c in range(len(counts)))
            m = [sum(O.gram_mrc(H[n, off[c]:off[c + 1]], Y[n, k, off[c]:off[c + 1]])[1] for c in range(len(counts)))
                 for k in range(t)]
            out[n] = np.concatenate([g.reshape(-1), np.array(m).reshape(-1)])
        return torch.from_numpy(out)

    def solve(self, stats, n0_items, beta):
        st = stats.numpy()
        u, t = self.u, self.t
        n = st.shape[0]
        xh = np.zeros((n, t, u), complex)
        s2 = np.zeros((n, t if self.kind == "lama" else u))
        dec = np.zeros((n, t, u), np.uint8)
        for i in range(n):
            g = st[i, :u * u].reshape(u, u)
            for k in range(t):
                ym = st[i, u * u + k * u:u * u + (k + 1) * u]
                if self.kind == "lama":
                    z, v, _ = O.lama_equalize(g, ym, self.syms, 1.0, float(n0_items[i]), beta, **self.lp)
                    s2[i, k] = v[0]
                else:
                    z, v, c = O.linear_equalize(self.kind, g, ym, float(n0_items[i]))
                    z, v = O.unbias(z, v, c)
                    s2[i] = v
                xh[i, k] = z
                dec[i, k] = O.hard_detect_index(z, self.syms)
        return torch.from_numpy(xh), torch.from_numpy(s2), torch.from_numpy(dec), torch.zeros(n), torch.zeros(n)

    def fd_partial(self, H, Y, counts, b_total, n0_items):
        H, Y = H.numpy(), Y.numpy()
        u, t, wd = self.u, self.t, self.wdim
        off = np.concatenate(([0], np.cumsum(counts)))
        n = H.shape[0]
        acc = np.zeros((n, 2 * t * u + 2 * wd))
        wraw = np.zeros((n, len(counts), wd))
        for i in range(n):
            num = np.zeros((t, u), complex)
            den = np.zeros(wd)
            harm = np.zeros(wd)
            for c in range(len(counts)):
                sl = slice(off[c], off[c + 1])
                for k in range(t):
                    r = O.cluster_equalize(self.kind, H[i, sl], Y[i, k, sl], float(n0_items[i]), 1.0, b_total,
                                           self.syms, self.lp)
                    z, s2 = O.unbias(r["z"], r["sigma2"], r["gain"])
                    if self.kind == "mrc":
                        w = r["mrc_gains"]
                    else:
                        w = 1.0 / np.maximum(s2, O.VARIANCE_FLOOR)
                    num[k] += w * z
                    if self.kind == "lama":
                        den[k] += w[0]
                        harm[k] += 1.0 / max(s2[0], O.VARIANCE_FLOOR)
                        wraw[i, c, k] = w[0]
                    elif k == 0:
                        den += w
                        harm += 1.0 / np.maximum(s2, O.VARIANCE_FLOOR)
                        wraw[i, c] = w
            acc[i, :2 * t * u] = np.stack([num.real, num.imag], -1).reshape(-1)
            acc[i, 2 * t * u:2 * t * u + wd] = den
            acc[i, 2 * t * u + wd:] = harm
        return torch.from_numpy(acc), torch.from_numpy(wraw), torch.zeros(n), torch.zeros(n)

    def fd_finalize(self, acc):
        a = acc.numpy()
        u, t, wd = self.u, self.t, self.wdim
        num = a[:, :2 * t * u].reshape(-1, t, u, 2)
        num = num[..., 0] + 1j * num[..., 1]
        den = a[:, 2 * t * u:2 * t * u + wd]
        harm = a[:, 2 * t * u + wd:]
        xh = num / (den[:, :, None] if self.kind == "lama" else den[:, None, :])
        dec = np.array([[O.hard_detect_index(xh[i, k], self.syms) for k in range(t)] for i in range(xh.shape[0])])
        return torch.from_numpy(xh), torch.from_numpy(1.0 / harm), torch.from_numpy(dec.astype(np.uint8))

    def fd_weights(self, wraw, den):
        return wraw / den[:, None, :]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, arch, kind, C, bits, path, chunks=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1808_04473_b200.distributed import ClusterGroup

    rng = np.random.default_rng(5)
    n, B, U = 4 * chunks, 8 * C, 4
    H = (rng.standard_normal((n, B, U)) + 1j * rng.standard_normal((n, B, U))) / np.sqrt(2 * B)
    Y = rng.standard_normal((n, T, B)) + 1j * rng.standard_normal((n, T, B))
    n0 = rng.uniform(0.05, 0.2, n)
    ops = OracleOps(kind, U, T, bits)
    grp = ClusterGroup(arch, kind, [B // C] * C, U, T, None, ops=ops)
    a, b = grp.local_rows()
    # G > C: each item shard group handles its own frames (shift the seed)
    if grp.plan.n_shards > 1:
        H, Y = H * (1 + grp.plan.shard), Y * (1 + grp.plan.shard)
    res = grp.run(torch.from_numpy(np.ascontiguousarray(H[:, a:b])),
                  torch.from_numpy(np.ascontiguousarray(Y[:, :, a:b])), torch.from_numpy(n0), chunks=chunks)
    np.savez(os.path.join(path, f"r{rank}.npz"), items=np.array(res.items), xhat=res.xhat.numpy(),
             sigma2=res.sigma2.numpy(), dec=res.decisions.numpy(),
             nu=np.zeros(0) if res.nu is None else np.asarray(res.nu), clusters=np.array(grp.plan.clusters),
             shard=grp.plan.shard, H=H, Y=Y, n0=n0)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,arch,kind,C,bits,chunks", [
    (2, "pd", "lmmse", 4, 4, 1), (2, "pd", "zf", 2, 4, 1), (2, "fd", "lmmse", 4, 4, 1), (2, "fd", "mrc", 2, 4, 1),
    (2, "fd", "lama", 2, 2, 1), (2, "pd", "lama", 2, 2, 1), (4, "fd", "zf", 2, 4, 1), (4, "pd", "mrc", 2, 4, 1),
    (2, "pd", "lmmse", 4, 4, 2), (2, "fd", "zf", 2, 4, 3)])
def test_cluster_group_matches_single_process(tmp_path, world, arch, kind, C, bits, chunks):
    """Every rank's finalized items (block r of every chunk) equal the
    single-process reference path on those items."""
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, arch, kind, C, bits, str(tmp_path), chunks), nprocs=world,
                       start_method="spawn")
    syms, _ = O.square_qam(bits)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        items = d["items"]
        B = d["H"].shape[1]
        off = O.uniform_offsets(B, C)
        lp = {"t_max": 4} if kind == "lama" else None
        ref = O.run_batch(arch, kind, d["H"], d["Y"], off, d["n0"], 1.0, syms, lp, items=items)
        assert np.max(np.abs(d["xhat"] - ref["z"])) < 1e-10
        s2 = d["sigma2"]
        if kind == "lama":
            s2 = np.broadcast_to(s2[:, :, None], ref["sigma2"].shape)
        else:
            s2 = np.broadcast_to(s2[:, None, :], ref["sigma2"].shape)
        assert np.max(np.abs(s2 - ref["sigma2"])) < 1e-10
        assert np.array_equal(d["dec"], ref["dec"])
        if arch == "fd":
            full = O.run_batch(arch, kind, d["H"], d["Y"], off, d["n0"], 1.0, syms, lp)
            nu_ref = full["nu"][:, :, d["clusters"], :]          # [n][T][C_r][U]
            nu = d["nu"]                                       # [n][C_r][wdim]
            if kind == "lama":
                nu = np.broadcast_to(np.transpose(nu, (0, 2, 1))[:, :, :, None], nu_ref.shape)
            else:
                nu = np.broadcast_to(nu[:, None], nu_ref.shape)
            assert np.max(np.abs(nu - nu_ref)) < 1e-10


def test_rank_plans():
    from paper_1808_04473_b200.distributed import plan_ranks

    p = plan_ranks(4, 2, 8)
    assert p.clusters == [4, 5] and p.n_shards == 1 and p.group_ranks == [0, 1, 2, 3]
    p = plan_ranks(8, 5, 4)
    assert p.clusters == [1] and p.shard == 1 and p.group_ranks == [4, 5, 6, 7]
    with pytest.raises(Exception):
        plan_ranks(3, 0, 8)
