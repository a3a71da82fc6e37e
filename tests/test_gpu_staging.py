"""Parity of the tensor-core kernel's staging variants (dbp_tc.cuh) against
the CPU oracle (oracle/dbp_oracle.py, the fp64 restatement of the reference's
per-vector path, pinned to the reference's golden vectors by
tests/test_oracle_golden.py).

The launcher picks, per geometry, how many whole items share one shared-memory
stage (ips), whether an item is split into antenna row blocks (spi > 1),
whether two units share one tensor-core tile (pair), and the ring depth.  The
options tc_smax_kb / tc_ns / tc_pair (dbp_set_option) force each variant here
on small inputs, including odd item counts (a null half in the last pair),
paired items in different stages, row blocks whose clusters pair inside one
stage, and an odd cluster count (FD without pairing).  U <= 16 linear
geometries run on the split-bf16 kernel by default (tests/test_gpu_tc2.py);
here the 3xTF32 kernel is forced."""

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp
from paper_1808_04473_b200 import _lib
from oracle import dbp_oracle as O
from parity import NU_TOL, SIGMA2_TOL, XHAT_TOL, check_decisions, entry_rel, normwise_rel

pytestmark = pytest.mark.gpu

# (arch, kind, n_items, B, C, U, T, bits, env)
CASES = [
    ("pd", "lmmse", 7, 128, 4, 16, 14, 4, {}),                        # 2 items/stage, null half at the end
    ("pd", "lmmse", 9, 128, 4, 16, 14, 4, {"tc_smax_kb": 96}),     # 3 items/stage: pairs straddle stages
    ("pd", "lmmse", 5, 128, 4, 16, 14, 4, {"tc_smax_kb": 20}),     # row blocks (spi = 2), paired items
    ("pd", "zf", 6, 128, 4, 16, 14, 6, {"tc_pair": 1}),         # one unit per tile
    ("pd", "lmmse", 6, 96, 3, 8, 5, 4, {}),                            # U = 8 (two units in one 32-row block)
    ("pd", "mrc", 4, 256, 8, 32, 14, 6, {"tc_smax_kb": 40}),       # U = 32, row blocks
    ("fd", "lmmse", 5, 128, 4, 16, 14, 4, {}),                        # clusters paired inside an item
    ("fd", "zf", 4, 256, 8, 16, 14, 6, {"tc_smax_kb": 32, "tc_ns": 3}),  # row blocks at cluster pairs
    ("fd", "mrc", 5, 96, 3, 16, 7, 4, {}),                            # odd cluster count: no pairing
    ("fd", "lmmse", 3, 64, 2, 8, 14, 4, {"tc_ns": 2}),          # cfg1 shape
    ("pd", "lama", 3, 128, 4, 16, 14, 4, {}),                          # LAMA epilogue on a solver warp
    ("fd", "lama", 3, 128, 4, 8, 6, 2, {}),                            # FD LAMA fold
]
CONST = {2: "qpsk", 4: "qam16", 6: "qam64"}


@pytest.mark.parametrize("arch,kind,n,b,c,u,t,bits,env", CASES)
def test_staging_variant_matches_oracle(arch, kind, n, b, c, u, t, bits, env):
    rng = np.random.default_rng(7 * n + b + u + t)
    H = ((rng.standard_normal((n, b, u)) + 1j * rng.standard_normal((n, b, u))) / np.sqrt(2 * b)).astype(np.complex64)
    const = dbp.make_constellation(CONST[bits])
    s = const.symbols[rng.integers(0, len(const.symbols), (n, t, u))]
    n0 = 0.05
    noise = (rng.standard_normal((n, t, b)) + 1j * rng.standard_normal((n, t, b))) * np.sqrt(n0 / 2)
    Y = (np.einsum("nbu,ntu->ntb", H.astype(complex), s) + noise).astype(np.complex64)
    counts = [b // c] * c
    lp = {"t_max": 5} if kind == "lama" else None
    with _lib.options(kernel=_lib.KERNEL_TC_TF32, **env):  # forced: other kernels are the default here
        det = dbp.detect(arch, kind, H, Y, n0, counts, const, lama_params=lp)
        assert _lib.lib().dbp_last_kernel() == _lib.KERNEL_TC_TF32  # the 3xTF32 tensor-core kernel ran
    offs = [0] + list(np.cumsum(counts))
    ref = O.run_batch(arch, kind, H.astype(complex), Y.astype(complex), offs, n0, 1.0, const.symbols,
                      lama_params=lp)
    assert normwise_rel(det.xhat, ref["z"]) < XHAT_TOL, normwise_rel(det.xhat, ref["z"])
    if kind == "lama":
        s2 = np.broadcast_to(det.sigma2[:, :, None], ref["sigma2"].shape)
    else:
        s2 = np.broadcast_to(det.sigma2[:, None, :], ref["sigma2"].shape)
    assert entry_rel(s2, ref["sigma2"]) < SIGMA2_TOL
    nbad, ntot, at_boundary = check_decisions(det.decisions, ref["dec"], ref["z"], det.xhat, const.pam_levels)
    assert at_boundary and nbad <= 1, nbad
    if arch == "fd":
        if kind == "lama":
            nu = np.broadcast_to(np.transpose(det.nu, (0, 2, 1))[:, :, :, None], ref["nu"].shape)
        else:
            nu = np.broadcast_to(det.nu[:, None], ref["nu"].shape)
        assert entry_rel(nu, ref["nu"]) < NU_TOL
