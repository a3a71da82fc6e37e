"""On-device frame synthesis (dbp_synthesize, csrc/dbp_synth.cuh) against a
NumPy restatement of its documented counter mapping: Philox4x32-10 keyed by
the seed, counter (item, stream, block); Box-Muller per block.  Symbol
indices are bit-exact; Gaussian values agree to float32 rounding of
log/sin/cos.  Plus the model's statistics (H ~ CN(0, 1/B), uniform symbols,
y - H s ~ CN(0, N0)) and reproducibility of any item range on its own."""

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp

M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox(ctr, seed):
    """ctr: uint64 array [..., 4] of 32-bit words -> Philox4x32-10 output."""
    c = [ctr[..., i].astype(np.uint64) for i in range(4)]
    k0, k1 = np.uint64(seed & MASK), np.uint64((seed >> 32) & MASK)
    for _ in range(10):
        p0 = np.uint64(M0) * c[0]
        p1 = np.uint64(M1) * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK)
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + np.uint64(W0)) & np.uint64(MASK)
        k1 = (k1 + np.uint64(W1)) & np.uint64(MASK)
    return np.stack(c, -1)


def blocks(seed, items, stream, nblk):
    n = np.asarray(items, dtype=np.uint64)[:, None]
    j = np.arange(nblk, dtype=np.uint64)[None, :]
    ctr = np.stack(np.broadcast_arrays(n & np.uint64(MASK), n >> np.uint64(32),
                                       np.full_like(j, stream), j), -1)
    return philox(ctr, seed)  # [n][nblk][4]


def box_muller(x, s):
    k = np.float64(2.0 ** -32)
    u1a, u2a = (x[..., 0] + 1.0) * k, x[..., 1] * k
    u1b, u2b = (x[..., 2] + 1.0) * k, x[..., 3] * k
    ra, rb = s * np.sqrt(-2.0 * np.log(u1a)), s * np.sqrt(-2.0 * np.log(u1b))
    a = ra * np.cos(2 * np.pi * u2a) + 1j * ra * np.sin(2 * np.pi * u2a)
    b = rb * np.cos(2 * np.pi * u2b) + 1j * rb * np.sin(2 * np.pi * u2b)
    return np.stack([a, b], -1).reshape(x.shape[0], -1)  # entries 2j, 2j+1


def reference_synth(seed, items, b, u, t, const, n0):
    hs, ns = np.sqrt(0.5 / b), np.sqrt(0.5 * n0)
    H = box_muller(blocks(seed, items, 0, b * u // 2), hs).reshape(len(items), b, u)
    xs = blocks(seed, items, 1, (t * u + 3) // 4).reshape(len(items), -1)[:, :t * u]
    S = ((xs * np.uint64(const.size)) >> np.uint64(32)).astype(np.int64).reshape(len(items), t, u)
    noise = box_muller(blocks(seed, items, 2, t * b // 2), ns).reshape(len(items), t, b)
    Y = np.einsum("nbu,ntu->ntb", H, const.symbols[S]) + noise
    return H, Y, S


@pytest.mark.gpu
def test_counter_mapping_matches_numpy_restatement():
    const = dbp.make_constellation("qam16")
    seed, b, u, t, n0 = 0x1234_5678_9ABC, 64, 16, 14, 0.07
    H, Y, S = dbp.synth.synth_device(seed, 5, b, u, t, const, n0=n0, item0=7, return_symbols=True)
    Hr, Yr, Sr = reference_synth(seed, np.arange(7, 12), b, u, t, const, n0)
    np.testing.assert_array_equal(S.cpu().numpy(), Sr)
    np.testing.assert_allclose(H.cpu().numpy(), Hr, rtol=2e-5, atol=2e-7)
    np.testing.assert_allclose(Y.cpu().numpy(), Yr, rtol=2e-5, atol=2e-6)


@pytest.mark.gpu
def test_item_ranges_are_independent_and_reproducible():
    const = dbp.make_constellation("qam64")
    H1, Y1 = dbp.synth.synth_device(9, 40, 128, 16, 14, const, n0=0.01)
    H2, Y2 = dbp.synth.synth_device(9, 10, 128, 16, 14, const, n0=0.01, item0=25)
    assert np.array_equal(H1[25:35].cpu().numpy(), H2.cpu().numpy())
    assert np.array_equal(Y1[25:35].cpu().numpy(), Y2.cpu().numpy())
    H3, _ = dbp.synth.synth_device(10, 40, 128, 16, 14, const, n0=0.01)
    assert not np.array_equal(H1.cpu().numpy(), H3.cpu().numpy())


@pytest.mark.gpu
def test_model_statistics():
    const = dbp.make_constellation("qam16")
    n, b, u, t, n0 = 3000, 64, 8, 14, 0.25
    H, Y, S = dbp.synth.synth_device(3, n, b, u, t, const, n0=n0, return_symbols=True)
    h = H.cpu().numpy().astype(complex)
    s = S.cpu().numpy().astype(np.int64)
    y = Y.cpu().numpy().astype(complex)
    assert abs(np.mean(np.abs(h) ** 2) * b - 1.0) < 0.01
    assert abs(np.mean(h.real * h.imag)) < 0.01 / b
    counts = np.bincount(s.ravel(), minlength=16) / s.size
    assert np.all(np.abs(counts - 1 / 16) < 0.004)
    e = y - np.einsum("nbu,ntu->ntb", h, const.symbols[s])
    assert abs(np.mean(np.abs(e) ** 2) / n0 - 1.0) < 0.01


@pytest.mark.gpu
def test_detection_on_synthesized_frames_matches_oracle():
    """The detector on device-synthesized inputs equals the CPU oracle on the
    same (copied back) inputs."""
    from oracle import dbp_oracle as O
    from parity import XHAT_TOL, normwise_rel

    const = dbp.make_constellation("qam16")
    H, Y = dbp.synth.synth_device(5, 6, 128, 16, 14, const, n0=0.05)
    det = dbp.detect("pd", "lmmse", H, Y, 0.05, [32] * 4, const)
    ref = O.run_batch("pd", "lmmse", H.cpu().numpy().astype(complex), Y.cpu().numpy().astype(complex),
                      O.uniform_offsets(128, 4), 0.05, 1.0, const.symbols)
    assert normwise_rel(det.xhat.cpu().numpy(), ref["z"]) < XHAT_TOL
