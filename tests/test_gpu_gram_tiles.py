"""dbp_gram_mrc (kernel K1, the tensor-core Gram/MRC stage) against an fp64
numpy restatement of the per-cluster products G_c = H_c^H H_c, z_c = H_c^H y
(reference dbp/partial.py, Cluster.gram / Cluster.mrc), over the shapes that
exercise the operand-tile layouts: two units paired per tcgen05.mma (a warp
then holds accumulator rows of both units, e.g. Y rows of unit 0 and 1), a
single unit per tile, per-cluster and cluster-summed outputs, odd and tiny
T, U=8/16/32, and U=64 on the wide layout (A = the 128 H features, B = [H | Y],
N = 160), including ragged row chunks and u < 64."""

import numpy as np
import pytest
import torch

from paper_1808_04473_b200 import _lib

pytestmark = pytest.mark.gpu

CASES = [
    # items, B, U, T, offsets, summed
    (3, 32, 16, 14, [0, 32], 1),
    (3, 64, 16, 14, [0, 32, 64], 0),
    (3, 128, 16, 14, [0, 64, 128], 0),
    (3, 64, 16, 4, [0, 32, 64], 0),
    (3, 64, 16, 8, [0, 32, 64], 0),
    (5, 64, 16, 1, [0, 32, 64], 0),
    (3, 64, 8, 14, [0, 32, 64], 0),
    (4, 128, 16, 14, [0, 32, 64, 96, 128], 1),
    (4, 128, 16, 14, [0, 32, 64, 96, 128], 0),
    (3, 64, 16, 14, [0, 64], 0),
    (3, 128, 32, 14, [0, 64, 128], 0),
    (2, 128, 64, 7, [0, 64, 128], 0),
    (7, 96, 16, 3, [0, 32, 64, 96], 1),
    # wide (U = 64): cfg5 geometry summed, one cluster, ragged clusters (SIMT), u < UP, T = 16
    (3, 512, 64, 14, list(range(0, 513, 64)), 1),
    (2, 512, 64, 14, list(range(0, 513, 64)), 0),
    (2, 64, 64, 16, [0, 64], 1),
    (3, 80, 64, 14, [0, 48, 80], 0),
    (2, 256, 62, 5, [0, 128, 256], 1),
]


@pytest.mark.parametrize("n,b,u,t,offs,summed", CASES)
def test_gram_mrc_tiles(n, b, u, t, offs, summed):
    rng = np.random.default_rng(1000 * u + 10 * t + b)
    H = ((rng.standard_normal((n, b, u)) + 1j * rng.standard_normal((n, b, u))) / 8).astype(np.complex64)
    Y = (rng.standard_normal((n, t, b)) + 1j * rng.standard_normal((n, t, b))).astype(np.complex64)
    Hd, Yd = torch.from_numpy(H).cuda(), torch.from_numpy(Y).cuda()
    c = len(offs) - 1
    ncl = 1 if summed else c
    out = torch.full((n, ncl, u * u + t * u), float("nan"), dtype=torch.complex64, device="cuda")
    offa, offp = _lib.host_i32(offs)  # offa keeps the buffer alive
    _lib.check(_lib.lib().dbp_gram_mrc(_lib.ptr(Hd), _lib.ptr(Yd), n, b, u, u, t, c, offp, summed,
                                       _lib.ptr(out), _lib.stream_ptr()))
    o = out.cpu().numpy()
    for i in range(n):
        for k in range(ncl):
            sl = slice(0, b) if summed else slice(offs[k], offs[k + 1])
            h = H[i, sl].astype(complex)
            y = Y[i][:, sl].astype(complex)
            G = h.conj().T @ h
            Z = (h.conj().T @ y.T).T
            scale_g = np.abs(G).max()
            scale_z = np.abs(Z).max()
            # 3xTF32 / fp32 accumulation: ~1e-6 relative to the largest entry
            assert np.abs(o[i, k, :u * u].reshape(u, u) - G).max() < 2e-5 * scale_g, (i, k, "G")
            assert np.abs(o[i, k, u * u:].reshape(t, u) - Z).max() < 2e-5 * scale_z, (i, k, "Z")
    if len(set(np.diff(offs))) == 1:  # uniform clusters run on the tensor cores (ragged: SIMT kernel)
        assert _lib.lib().dbp_last_kernel() in (_lib.KERNEL_TC_TF32, _lib.KERNEL_TC_BF16)


def test_gram_mrc_parts_two_vs_three():
    """dbp_gram_mrc_parts: two bf16 parts stay within ~2^-16 of the three-part
    (~3xTF32) statistics on a well-conditioned PD geometry (the multi-GPU PD
    path's choice), and 0 equals the default entry point bit for bit."""
    import torch
    from paper_1808_04473_b200 import _lib

    rng = np.random.default_rng(5)
    n, b, c, u, t = 64, 128, 4, 16, 14
    H = torch.tensor(((rng.standard_normal((n, b, u)) + 1j * rng.standard_normal((n, b, u))) / np.sqrt(2 * b))
                     .astype(np.complex64), device="cuda")
    Y = torch.tensor((rng.standard_normal((n, t, b)) + 1j * rng.standard_normal((n, t, b))).astype(np.complex64),
                     device="cuda")
    offs_keep, offs = _lib.host_i32(np.arange(0, b + 1, b // c))
    lib = _lib.lib()
    outs = {}
    for parts in (0, 2, 3):
        out = torch.empty((n, u * u + t * u), dtype=torch.complex64, device="cuda")
        _lib.check(lib.dbp_gram_mrc_parts(_lib.ptr(H), _lib.ptr(Y), n, b, u, u, t, c, offs, 1, parts, _lib.ptr(out),
                                          _lib.stream_ptr()))
        outs[parts] = out.cpu().numpy()
    ref = torch.empty((n, u * u + t * u), dtype=torch.complex64, device="cuda")
    _lib.check(lib.dbp_gram_mrc(_lib.ptr(H), _lib.ptr(Y), n, b, u, u, t, c, offs, 1, _lib.ptr(ref), _lib.stream_ptr()))
    assert np.array_equal(outs[0], ref.cpu().numpy())
    assert np.array_equal(outs[0], outs[3])
    scale = np.max(np.abs(outs[3]), axis=1, keepdims=True)
    assert np.max(np.abs(outs[2] - outs[3]) / scale) < 2e-5
    with pytest.raises(Exception):
        _lib.check(lib.dbp_gram_mrc_parts(_lib.ptr(H), _lib.ptr(Y), n, b, u, u, t, c, offs, 1, 5, _lib.ptr(ref),
                                          _lib.stream_ptr()))
