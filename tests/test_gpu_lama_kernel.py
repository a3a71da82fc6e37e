"""GPU parity of the LAMA recursion kernel (csrc/dbp_lama.cuh, lama_kernel):
PD and FD LAMA at 16 < u <= 32 run as tensor-core statistics (PD: split-bf16,
FD: 3xTF32) + lama_kernel
(one warp per unit, G in registers).  Each geometry is checked against the
vectorized float64 oracle (equalize.py:208-259 and fusion.py:127-154
restated) at the parity tolerances, and against the previous recursion inside
the streaming kernels (option lama_kernel=1) -- odd and small T, u < 32 and
odd u (padded), damping, t_max = 1, QPSK / 16-QAM / 64-QAM (packed PAM
posterior) and a non-square set (generic posterior)."""

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp
from oracle import dbp_oracle as O
from paper_1808_04473_b200 import _lib
from paper_1808_04473_b200.model import Constellation
from paper_1808_04473_b200.synth import synth_frames
from parity import DEC_RATE, NU_TOL, SIGMA2_TOL, XHAT_TOL, check_decisions, entry_rel, normwise_rel

pytestmark = pytest.mark.gpu

PSK16 = Constellation("16PSK", np.exp(2j * np.pi * np.arange(16) / 16), 1.0)  # no PAM factorisation

# arch, u, T, cluster sizes, constellation, t_max, damping, snr_db
CASES = [
    ("pd", 32, 14, [32] * 8, "qam16", 10, 1.0, 8.0),   # cfg4 geometry
    ("fd", 32, 14, [32] * 8, "qam16", 10, 1.0, 8.0),
    ("pd", 24, 5, [48, 48], "qpsk", 4, 1.0, 6.0),
    ("fd", 20, 16, [40, 40], "qam64", 6, 0.7, 18.0),
    ("fd", 17, 1, [34, 34, 34], "qam16", 1, 1.0, 10.0),
    ("fd", 32, 9, [64, 32, 64], "qpsk", 3, 1.0, 4.0),
    ("pd", 32, 3, [64], PSK16, 5, 1.0, 12.0),
]


def _const(c):
    return dbp.make_constellation(c) if isinstance(c, str) else c


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-u{c[1]}-T{c[2]}-C{len(c[3])}" for c in CASES])
def test_lama_kernel_matches_oracle_and_streaming_recursion(case):
    arch, u, t, counts, cname, t_max, damping, snr = case
    const = _const(cname)
    b = sum(counts)
    H, Y, _, n0 = synth_frames(7, 1, 96, t, b, u, const, snr)
    lp = {"t_max": t_max, "damping": damping}
    det = dbp.detect(arch, "lama", H, Y, n0[0], counts, const, lama_params=lp)
    if u % 2 == 0 and len(set(counts)) == 1:  # odd u / ragged clusters may take the streaming kernel
        assert _lib.lib().dbp_last_kernel() in (_lib.KERNEL_TC_BF16, _lib.KERNEL_TC_TF32)
    offs = np.concatenate([[0], np.cumsum(counts)])
    ref = O.run_batch_vec(arch, "lama", H.astype(complex), Y.astype(complex), offs, n0[0], const.es,
                          const.symbols, lama_params=lp)
    assert normwise_rel(det.xhat, ref["z"]) < XHAT_TOL, normwise_rel(det.xhat, ref["z"])
    s2 = np.broadcast_to(det.sigma2[:, :, None], ref["sigma2"].shape)
    assert entry_rel(s2, ref["sigma2"]) < SIGMA2_TOL, entry_rel(s2, ref["sigma2"])
    nbad, ntot, at_boundary = check_decisions(det.decisions, ref["dec"], ref["z"], det.xhat,
                                              const.pam_levels if const.pam_levels is not None else [0.0])
    if const.pam_levels is not None:
        assert at_boundary and nbad <= max(1, int(np.ceil(DEC_RATE * ntot))), nbad
    if arch == "fd":
        nu = np.broadcast_to(np.transpose(det.nu, (0, 2, 1))[:, :, :, None], ref["nu"].shape)
        assert entry_rel(nu, ref["nu"]) < NU_TOL, entry_rel(nu, ref["nu"])
    # the recursion inside the streaming / statistics kernels agrees to fp32 rounding
    with _lib.options(lama_kernel=1):
        old = dbp.detect(arch, "lama", H, Y, n0[0], counts, const, lama_params=lp)
    assert normwise_rel(det.xhat, old.xhat) < 2e-5
    assert entry_rel(det.sigma2, old.sigma2) < 2e-5


def test_lama_kernel_per_item_noise_and_many_items():
    """Per-item N0 (one SNR per frame) over several frames: each CTA warp walks
    many items and clusters (grid-stride), FD fusion per item."""
    const = dbp.make_constellation("qam16")
    counts = [32] * 4
    H, Y, _, n0 = synth_frames(3, 4, 300, 14, 128, 32, const, [4.0, 8.0, 12.0, 16.0])
    n0_items = np.repeat(n0, 300)
    lp = {"t_max": 10}
    for arch in ("pd", "fd"):
        det = dbp.detect(arch, "lama", H, Y, n0, counts, const, lama_params=lp, n0_group=300)
        assert _lib.lib().dbp_last_kernel() in (_lib.KERNEL_TC_BF16, _lib.KERNEL_TC_TF32)
        pick = np.arange(0, 1200, 7)
        ref = O.run_batch_vec(arch, "lama", H[pick].astype(complex), Y[pick].astype(complex),
                              O.uniform_offsets(128, 4), n0_items[pick], const.es, const.symbols, lama_params=lp)
        assert normwise_rel(det.xhat[pick], ref["z"]) < XHAT_TOL
        s2 = np.broadcast_to(det.sigma2[pick][:, :, None], ref["sigma2"].shape)
        assert entry_rel(s2, ref["sigma2"]) < SIGMA2_TOL


@pytest.mark.parametrize("u", [24, 32])
def test_lama_kernel_from_statistics_records(u):
    """The multi-GPU PD central solve (dbp_equalize_stats without traces) runs
    lama_kernel on the exchanged statistics, reading G by rows (as the
    reference's i_minus_g @ s does): against the per-vector oracle."""
    import torch

    from paper_1808_04473_b200.distributed import CudaOps

    const = dbp.make_constellation("qam16")
    b, t, n = 4 * u, 14, 64
    H, Y, _, n0 = synth_frames(11, 1, n, t, b, u, const, 9.0)
    g = np.einsum("nbi,nbj->nij", H.conj().astype(complex), H.astype(complex))
    ym = np.einsum("nbi,ntb->nti", H.conj().astype(complex), Y.astype(complex))
    rec = np.concatenate([g.reshape(n, -1), ym.reshape(n, -1)], axis=1).astype(np.complex64)
    ops = CudaOps("lama", u, t, const, lama_params={"t_max": 8})
    beta = u / b
    n0_items = torch.full((n,), float(n0[0]), dtype=torch.float32, device="cuda")
    xhat, s2, dec, status, _ = ops.solve(torch.tensor(rec, device="cuda"), n0_items, beta)
    assert int(status.abs().max()) == 0
    xhat, s2 = xhat.cpu().numpy(), s2.cpu().numpy()
    for i in range(0, n, 9):
        for tt in range(t):
            z, tau, _ = O.lama_equalize(g[i], ym[i, tt], const.symbols, const.es, float(n0[0]), beta, t_max=8)
            assert normwise_rel(xhat[i, tt], z) < XHAT_TOL
            assert entry_rel(s2[i, tt], tau[0]) < SIGMA2_TOL


@pytest.mark.parametrize("arch", ["pd", "fd"])
def test_lama_kernel_divergence_status(arch):
    """A non-finite receive vector makes z^1 non-finite: DivergenceError at
    iteration 1 for that item only (equalize.py:246-249), through the per-warp
    status reduction of lama_kernel; the other items are unaffected."""
    from paper_1808_04473_b200 import DivergenceError

    const = dbp.make_constellation("qam16")
    counts = [32] * 4
    H, Y, _, n0 = synth_frames(5, 1, 40, 14, 128, 32, const, 10.0)
    Y = Y.copy()
    Y[7, 3, 5] = np.nan
    with pytest.raises(DivergenceError) as err:
        dbp.detect(arch, "lama", H, Y, n0[0], counts, const, lama_params={"t_max": 5})
    assert err.value.iteration == 1
    assert "item 7" in str(err.value)
    det = dbp.detect(arch, "lama", H, Y, n0[0], counts, const, lama_params={"t_max": 5}, check=False)
    st = np.asarray(det.status)
    assert st[7] == _lib.ST_DIVERGED and np.count_nonzero(st) == 1
