"""The oracle's bit-LLR restatement (oracle.dbp_oracle.bit_llr) against
closed forms: QPSK's per-dimension LLR 4 a v / s2 (exact = max-log), the
16-QAM max-log piecewise-linear form, Gray labels equal to the product's
model.gray_labels, and antisymmetry under x -> -x for the sign bits."""

import numpy as np

import paper_1808_04473_b200 as dbp
from oracle import dbp_oracle as O


def test_gray_labels_match_product():
    for name in ("qpsk", "qam16", "qam64"):
        c = dbp.make_constellation(name)
        assert np.array_equal(O.gray_labels(c.symbols, c.pam_levels), dbp.gray_labels(c))


def test_qpsk_closed_form():
    c = dbp.make_constellation("qpsk")
    a = c.pam_levels[1]  # levels (-a, a); level index 0 (-a) carries bit 0
    rng = np.random.default_rng(0)
    x = rng.standard_normal(200) + 1j * rng.standard_normal(200)
    s2 = rng.uniform(0.05, 2.0, 200)
    for exact in (False, True):
        got = O.bit_llr(x, s2, c.symbols, c.pam_levels, exact)
        np.testing.assert_allclose(got[:, 0], -4 * a * x.real / s2, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(got[:, 1], -4 * a * x.imag / s2, rtol=1e-12, atol=1e-12)


def test_qam16_maxlog_piecewise():
    c = dbp.make_constellation("qam16")
    lv = c.pam_levels  # (-3, -1, 1, 3) a; gray(i): 00 01 11 10
    a = lv[2]
    v = np.linspace(-5 * a, 5 * a, 101)
    got = O.bit_llr(v + 0j, 1.0, c.symbols, lv)
    # MSB: 0 for the negative half; LLR = max-log over the nearest of each half
    d = (v[:, None] - lv[None, :]) ** 2
    np.testing.assert_allclose(got[:, 0], d[:, 2:].min(1) - d[:, :2].min(1), atol=1e-12)
    # second bit: 1 on the inner levels
    np.testing.assert_allclose(got[:, 1], d[:, 1:3].min(1) - d[:, [0, 3]].min(1), atol=1e-12)


def test_exact_is_bounded_by_maxlog_gap_and_symmetric():
    c = dbp.make_constellation("qam64")
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(300) + 1j * rng.standard_normal(300)) * 0.8
    ml = O.bit_llr(x, 0.3, c.symbols, c.pam_levels)
    ex = O.bit_llr(x, 0.3, c.symbols, c.pam_levels, exact=True)
    # |exact - maxlog| <= log(number of symbols per bit class)
    assert np.max(np.abs(ex - ml)) <= np.log(c.size / 2) + 1e-12
    # the real / imaginary sign bits flip sign under x -> -x
    ex_neg = O.bit_llr(-x, 0.3, c.symbols, c.pam_levels, exact=True)
    np.testing.assert_allclose(ex_neg[:, [0, 3]], -ex[:, [0, 3]], atol=1e-9)
    np.testing.assert_allclose(ex_neg[:, [1, 2, 4, 5]], ex[:, [1, 2, 4, 5]], atol=1e-9)
