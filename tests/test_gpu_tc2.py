"""Parity of the split-bf16 tensor-core kernel (csrc/dbp_tc2.cuh, U <= 16
linear PD / FD and statistics) against the CPU oracle (oracle/dbp_oracle.py,
pinned to the reference's golden vectors by tests/test_oracle_golden.py).

Covers the geometry the kernel's TMA tensor maps and 4-unit groups must get
right: tail groups (item counts not a multiple of 4), PD over several 32-antenna
stages including a partial last stage (zero fill), FD with C = 1 / 2 / 4 / 8
(groups of 4 items x 1 cluster, 2 x 2, 1 x 4), U = 8 / 15 / 16 (padded
features), T = 1 / 5 / 14 / 16, MRC / ZF / L-MMSE, 2 and 3 bf16 parts, and
the per-cluster / summed statistics (local_preprocess / fuse_partials)."""

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp
from paper_1808_04473_b200 import _lib
from oracle import dbp_oracle as O
from parity import NU_TOL, SIGMA2_TOL, XHAT_TOL, check_decisions, entry_rel, normwise_rel

pytestmark = pytest.mark.gpu

CONST = {2: "qpsk", 4: "qam16", 6: "qam64"}

# (arch, kind, n_items, B, C, U, T, bits)
CASES = [
    ("pd", "lmmse", 13, 128, 4, 16, 14, 4),   # cfg2 shape, tail group of 1 item
    ("pd", "zf", 6, 128, 4, 16, 14, 6),
    ("pd", "mrc", 5, 128, 4, 16, 14, 6),
    ("pd", "lmmse", 7, 80, 2, 16, 14, 4),     # K = 80: partial last stage (TMA zero fill)
    ("pd", "lmmse", 9, 64, 2, 8, 5, 4),       # U = 8 (padded features), T = 5
    ("pd", "lmmse", 4, 128, 4, 15, 16, 4),    # odd U (u_stride 16), T = 16
    ("pd", "zf", 5, 96, 3, 16, 1, 2),         # T = 1, C = 3 (PD sums every antenna)
    ("fd", "lmmse", 7, 64, 2, 8, 14, 4),      # cfg1 shape: groups of 2 items x 2 clusters
    ("fd", "zf", 5, 256, 8, 16, 14, 6),       # cfg3 shape: 2 groups per item
    ("fd", "mrc", 5, 256, 8, 16, 14, 6),
    ("fd", "lmmse", 6, 128, 4, 16, 14, 4),    # one group per item
    ("fd", "lmmse", 9, 64, 1, 16, 14, 4),     # C = 1: groups of 4 items (FD == centralized)
    ("fd", "zf", 3, 192, 4, 16, 7, 4),        # K = 48 antennas per cluster: 2 stages, partial
]


def _inputs(n, b, u, t, bits, seed):
    rng = np.random.default_rng(seed)
    H = ((rng.standard_normal((n, b, u)) + 1j * rng.standard_normal((n, b, u))) / np.sqrt(2 * b)).astype(np.complex64)
    const = dbp.make_constellation(CONST[bits])
    s = const.symbols[rng.integers(0, len(const.symbols), (n, t, u))]
    n0 = 0.05
    noise = (rng.standard_normal((n, t, b)) + 1j * rng.standard_normal((n, t, b))) * np.sqrt(n0 / 2)
    Y = (np.einsum("nbu,ntu->ntb", H.astype(complex), s) + noise).astype(np.complex64)
    return H, Y, const, n0


@pytest.mark.parametrize("nsplit", [0, 2, 3])
@pytest.mark.parametrize("arch,kind,n,b,c,u,t,bits", CASES)
def test_tc2_matches_oracle(arch, kind, n, b, c, u, t, bits, nsplit):
    H, Y, const, n0 = _inputs(n, b, u, t, bits, 11 * n + b + u + t)
    counts = [b // c] * c
    with _lib.options(t2_nsplit=nsplit):
        det = dbp.detect(arch, kind, H, Y, n0, counts, const)
        assert _lib.lib().dbp_last_kernel() == _lib.KERNEL_TC_BF16
    offs = [0] + list(np.cumsum(counts))
    ref = O.run_batch(arch, kind, H.astype(complex), Y.astype(complex), offs, n0, 1.0, const.symbols)
    assert normwise_rel(det.xhat, ref["z"]) < XHAT_TOL, normwise_rel(det.xhat, ref["z"])
    s2 = np.broadcast_to(det.sigma2[:, None, :], ref["sigma2"].shape)
    assert entry_rel(s2, ref["sigma2"]) < SIGMA2_TOL, entry_rel(s2, ref["sigma2"])
    nbad, ntot, at_boundary = check_decisions(det.decisions, ref["dec"], ref["z"], det.xhat, const.pam_levels)
    assert at_boundary and nbad <= 1, nbad
    if arch == "fd":
        nu = np.broadcast_to(det.nu[:, None], ref["nu"].shape)
        assert entry_rel(nu, ref["nu"]) < NU_TOL, entry_rel(nu, ref["nu"])


def test_tc2_equals_tf32_kernel():
    """The split-bf16 kernel (3 parts) and the 3xTF32 kernel agree to fp32
    rounding on the cfg2 shape."""
    H, Y, const, n0 = _inputs(21, 128, 16, 14, 4, 5)
    with _lib.options(t2_nsplit=3):
        a = dbp.detect("pd", "lmmse", H, Y, n0, [32] * 4, const)
        assert _lib.lib().dbp_last_kernel() == _lib.KERNEL_TC_BF16
    with _lib.options(kernel=_lib.KERNEL_TC_TF32):
        b = dbp.detect("pd", "lmmse", H, Y, n0, [32] * 4, const)
        assert _lib.lib().dbp_last_kernel() == _lib.KERNEL_TC_TF32
    assert normwise_rel(a.xhat, b.xhat) < 1e-5


@pytest.mark.parametrize("summed", [False, True])
@pytest.mark.parametrize("n,b,c,u,t", [(7, 128, 4, 16, 14), (5, 64, 2, 8, 14), (6, 256, 8, 16, 3)])
def test_tc2_statistics(n, b, c, u, t, summed):
    """G_c = H_c^H H_c and y_c^mrc = H_c^H y_c per cluster (local_preprocess)
    or summed over clusters (fuse_partials), against fp64 products."""
    import torch

    H, Y, const, n0 = _inputs(n, b, u, t, 4, 3 * n + b)
    offs = np.array([0] + list(np.cumsum([b // c] * c)), dtype=np.int32)
    ncl = 1 if summed else c
    dH = torch.from_numpy(H).cuda()
    dY = torch.from_numpy(Y).cuda()
    out = torch.empty((n, ncl, u * u + t * u), dtype=torch.complex64, device="cuda")
    offa, offp = _lib.host_i32(offs)
    _lib.check(_lib.lib().dbp_gram_mrc(_lib.ptr(dH), _lib.ptr(dY), n, b, u, u, t, c, offp, int(summed),
                                       _lib.ptr(out), _lib.stream_ptr()))
    assert _lib.lib().dbp_last_kernel() == _lib.KERNEL_TC_BF16
    o = out.cpu().numpy()
    for i in range(n):
        for k in range(ncl):
            sl = slice(0, b) if summed else slice(offs[k], offs[k + 1])
            h = H[i, sl].astype(complex)
            y = Y[i][:, sl].astype(complex)
            G = h.conj().T @ h
            Z = (h.conj().T @ y.T).T
            # three bf16 parts (~2^-24 per product) accumulated in the tensor
            # core's fp32 accumulator over up to 256 antennas
            assert np.abs(o[i, k, :u * u].reshape(u, u) - G).max() < 1e-5 * np.abs(G).max(), (i, k, "G")
            assert np.abs(o[i, k, u * u:].reshape(t, u) - Z).max() < 1e-5 * np.abs(Z).max(), (i, k, "Z")


@pytest.mark.parametrize("t", [None, 1, 3, 16])
@pytest.mark.parametrize("kind", ["zf", "lmmse"])
def test_stats_solve_symbol_counts(kind, t):
    """linear_equalize on fused statistics (the warp-pair solver of
    t2_stats_solve_kernel, whose work areas are sized by T): one receive
    vector per channel (t None) and T = 1 / 3 / 16, odd item count."""
    n, b, u = 9, 64, 16
    H, Y, const, n0 = _inputs(n, b, u, t or 1, 4, 7 + (t or 0))
    if t is None:
        Y = Y[:, 0]
    stats = dbp.centralized_stats(H, Y)
    assert _lib.lib().dbp_last_kernel() == _lib.KERNEL_TC_BF16
    out = dbp.linear_equalize(kind, stats, n0)
    Ys = Y if t is not None else Y[:, None]
    for i in range(n):
        zi = np.asarray(out.z[i]).reshape(-1, u)
        s2i = np.asarray(out.sigma2[i]).reshape(-1, u)
        for tt in range(Ys.shape[1]):
            g, m = O.gram_mrc(H[i].astype(complex), Ys[i, tt].astype(complex))
            z, s2, _ = O.linear_equalize(kind, g, m, n0)
            assert normwise_rel(zi[tt], z) < XHAT_TOL, (i, tt)
            assert entry_rel(s2i[0], s2) < SIGMA2_TOL, (i, tt)


@pytest.mark.parametrize("arch,kind,n,b,c,u,t", [
    ("fd", "lmmse", 9, 64, 2, 8, 14),   # cfg1 shape: two items per pass, odd item count
    ("fd", "zf", 6, 128, 4, 8, 14),     # four clusters: one item per pass
    ("fd", "mrc", 5, 64, 1, 8, 7),      # one cluster: four items per pass
    ("fd", "lmmse", 7, 96, 3, 8, 14),   # three clusters: the two-unit solver (items would straddle a pass)
    ("pd", "lmmse", 11, 64, 2, 8, 14),
    ("pd", "zf", 6, 96, 3, 5, 3),       # odd u
    ("pd", "mrc", 3, 64, 2, 8, 16),
])
def test_quad_solver_matches_pair_and_oracle(arch, kind, n, b, c, u, t):
    """u <= 8: four units per solver pass (t2_solve_quad) against the two-unit
    solver (option t2_quad = 2) and the float64 oracle."""
    H, Y, const, n0 = _inputs(n, b, u, t, 4, 5 * n + b + u)
    counts = [b // c] * c
    q = dbp.detect(arch, kind, H, Y, n0, counts, const)
    assert _lib.lib().dbp_last_kernel() == _lib.KERNEL_TC_BF16
    with _lib.options(t2_quad=2):
        pr = dbp.detect(arch, kind, H, Y, n0, counts, const)
    assert normwise_rel(q.xhat, pr.xhat) < 2e-6, normwise_rel(q.xhat, pr.xhat)
    offs = [0] + list(np.cumsum(counts))
    ref = O.run_batch(arch, kind, H.astype(complex), Y.astype(complex), offs, n0, 1.0, const.symbols)
    assert normwise_rel(q.xhat, ref["z"]) < XHAT_TOL
    s2 = np.broadcast_to(q.sigma2[:, None, :], ref["sigma2"].shape)
    assert entry_rel(s2, ref["sigma2"]) < SIGMA2_TOL
    nbad, ntot, at_boundary = check_decisions(q.decisions, ref["dec"], ref["z"], q.xhat, const.pam_levels)
    assert at_boundary and nbad <= 1, nbad
    if arch == "fd":
        nu = np.broadcast_to(q.nu[:, None], ref["nu"].shape)
        assert entry_rel(nu, ref["nu"]) < NU_TOL
    else:
        assert np.array_equal(q.decisions, pr.decisions) or nbad <= 1
