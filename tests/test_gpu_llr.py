"""Gray-labelled bit LLRs (dbp_llr, soft.py) against the oracle's brute force
over all M symbols (oracle.dbp_oracle.bit_llr): max-log and exact
(log-sum-exp), per-UE and per-symbol variances, QPSK/16/64-QAM; the hard
decision implied by the LLR signs equals hard_detect's Gray label."""

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp
from oracle import dbp_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["qpsk", "qam16", "qam64"])
@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("per_symbol", [False, True])
def test_llr_matches_brute_force(name, exact, per_symbol):
    const = dbp.make_constellation(name)
    rng = np.random.default_rng(11)
    n, T, u = 7, 5, 6
    s = const.symbols[rng.integers(0, const.size, (n, T, u))]
    s2 = rng.uniform(0.02, 0.5, (n, T) if per_symbol else (n, u))
    noise = (rng.standard_normal((n, T, u)) + 1j * rng.standard_normal((n, T, u))) * 0.3
    x = (s + noise).astype(np.complex64)
    got = dbp.llr(x, s2.astype(np.float32), const, exact=exact)
    s2b = s2[:, :, None] if per_symbol else s2[:, None, :]
    ref = O.bit_llr(x, s2b, const.symbols, const.pam_levels, exact)
    scale = np.maximum(np.abs(ref), 1.0)
    assert np.max(np.abs(got - ref) / scale) < 1e-4


def test_llr_signs_give_the_hard_decision_labels():
    const = dbp.make_constellation("qam16")
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((50, 4, 8)) + 1j * rng.standard_normal((50, 4, 8))).astype(np.complex64)
    s2 = np.full((50, 8), 0.1, np.float32)
    bits = (dbp.llr(x, s2, const) < 0).astype(int)  # LLR < 0 -> bit 1
    nb = bits.shape[-1]
    label = (bits * (1 << np.arange(nb - 1, -1, -1))).sum(-1)
    idx = dbp.hard_detect_index(x.astype(complex), const)
    # exact ties (x on a midpoint) are measure-zero for continuous x
    assert np.array_equal(label, dbp.gray_labels(const)[idx])


@pytest.mark.parametrize("name", ["qpsk", "qam16", "qam64"])
def test_gray_bits_match_labels(name):
    """dbp_gray_bits of the detector's uint8 decisions and of int64 indices
    equal model.gray_labels unpacked MSB first."""
    const = dbp.make_constellation(name)
    rng = np.random.default_rng(3)
    idx = rng.integers(0, const.size, (9, 14, 5))
    nb = 2 * int(np.log2(len(const.pam_levels)))
    ref = (dbp.gray_labels(const)[idx][..., None] >> np.arange(nb - 1, -1, -1)) & 1
    assert np.array_equal(dbp.gray_bits(idx, const), ref)
    assert np.array_equal(dbp.gray_bits(idx.astype(np.uint8), const), ref)
    import torch
    dev = dbp.gray_bits(torch.as_tensor(idx.astype(np.uint8), device="cuda"), const)
    assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), ref)


def test_hard_bits_agree_with_llr_signs():
    """Detector decisions -> Gray bits equal the signs of the bit LLRs of the
    same x-hat (bit 1 <=> LLR < 0), end to end through pipeline.detect."""
    from oracle import dbp_oracle as O

    const = dbp.make_constellation("qam16")
    rng = np.random.default_rng(8)
    n, T, b, u = 40, 14, 64, 8
    H = (rng.standard_normal((n, b, u)) + 1j * rng.standard_normal((n, b, u))) / np.sqrt(2 * b)
    s = const.symbols[rng.integers(0, const.size, (n, T, u))]
    Y = np.einsum("nbu,ntu->ntb", H, s) + 0.1 * (rng.standard_normal((n, T, b)) + 1j * rng.standard_normal((n, T, b)))
    det = dbp.detect("pd", "lmmse", H, Y, 0.02, [32, 32], const)
    bits = dbp.gray_bits(det.decisions, const)
    llr = dbp.llr(det.xhat, det.sigma2, const)
    assert np.array_equal(np.asarray(bits), (np.asarray(llr) < 0).astype(np.uint8))
    assert O.gray_labels(const.symbols, const.pam_levels).shape == (const.size,)


def test_lama_soft_outputs_per_symbol_variance():
    """LAMA reports sigma2 per OFDM symbol ([n][T]); the LLRs of its x-hat with
    that variance equal the oracle's and their signs give the Gray bits of the
    detector's own decisions."""
    from oracle import dbp_oracle as O

    const = dbp.make_constellation("qam16")
    rng = np.random.default_rng(12)
    n, T, b, u = 30, 14, 64, 8
    H = (rng.standard_normal((n, b, u)) + 1j * rng.standard_normal((n, b, u))) / np.sqrt(2 * b)
    s = const.symbols[rng.integers(0, const.size, (n, T, u))]
    Y = np.einsum("nbu,ntu->ntb", H, s) + 0.15 * (rng.standard_normal((n, T, b)) + 1j * rng.standard_normal((n, T, b)))
    det = dbp.detect("pd", "lama", H, Y, 0.045, [32, 32], const, lama_params={"t_max": 6})
    s2 = np.asarray(det.sigma2)
    assert s2.shape == (n, T)
    x = np.asarray(det.xhat)
    got = dbp.llr(x, s2, const, exact=True)
    ref = O.bit_llr(x, s2[:, :, None], const.symbols, const.pam_levels, exact=True)
    assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)) < 1e-4
    bits = dbp.gray_bits(det.decisions, const)
    assert np.array_equal(np.asarray(bits), (dbp.llr(x, s2, const) < 0).astype(np.uint8))
