"""dbp_quadrature (paper_1808_04473_b200.asymptotics)
against the reference's own quadratures and analysis functions
(tests/golden/golden_quad.npz from tests/golden/make_golden_quad.py) and the
oracle restatement: fp64 on the GPU, agreement to ~1e-11 relative."""

import os

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp
from oracle import dbp_oracle as O
from paper_1808_04473_b200 import asymptotics as A

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_quad.npz"))


def close(a, b, rtol=1e-10, atol=1e-15):
    np.testing.assert_allclose(a, b, rtol=rtol, atol=atol)


@pytest.mark.parametrize("name", ["qpsk", "qam16", "qam64"])
def test_quadratures_match_reference(name):
    c = dbp.make_constellation(name)
    s2 = G["sigma2"]
    close(A.lama_mse_pam(s2, c.pam_levels), G[f"{name}_mse_pam"])  # one launch, 6 points
    close(A.lama_mse_pam(s2, c.pam_levels, 64), G[f"{name}_mse_pam_o64"])
    close(A.lama_mse(s2, c.symbols, 16), G[f"{name}_mse_2d_o16"])
    close(A.mi_awgn(c.es / G["sinr"][1:], c.symbols, 16), G[f"{name}_mi_o16"])
    close(A.awgn_mutual_information(c, G["sinr"], order=16), G[f"{name}_awgn_mi"])
    spec = A.MseSpec("lama", es=c.es, constellation=c)
    close(A.psi_mse(spec, s2), G[f"{name}_psi_lama"])
    close(A.se_trajectory(c, 0.05, 0.5, 8), G[f"{name}_se_traj"])
    # scalar calls keep the reference's scalar return type
    assert isinstance(A.lama_mse_pam(0.1, c.pam_levels), float)


def test_closed_form_psi_and_errors():
    for kind in ("mrc", "zf", "lmmse"):
        close(A.psi_mse(A.MseSpec(kind), G["sigma2"]), G[f"psi_{kind}"], rtol=1e-15)
    with pytest.raises(dbp.ConfigError):
        A.psi_mse(A.MseSpec("zf"), 0.0)
    with pytest.raises(dbp.ConfigError):
        A.MseSpec("lama")
    with pytest.raises(dbp.ConfigError):
        A.awgn_mutual_information(dbp.make_constellation("qpsk"), -1.0)


def test_sweep_matches_oracle_and_limits():
    """A 200-point MI sweep in one launch equals the oracle point by point on a
    sample; MI rises from 0 to log2 M."""
    c = dbp.make_constellation("qam16")
    sinr = np.geomspace(1e-3, 1e3, 200)
    mi = A.awgn_mutual_information(c, sinr, order=12)
    assert np.all(np.diff(mi) > -1e-12) and mi[0] < 0.01 and abs(mi[-1] - 4.0) < 1e-6  # saturates at log2 M
    for i in (0, 57, 133, 199):
        close(mi[i], O.mi_awgn(c.es / sinr[i], c.symbols, 12), rtol=1e-10)


@pytest.mark.parametrize("tag,beta,c", [("small", 8 / 64, 2), ("crit8", 16 / 256, 8)])
def test_message_passing_fixed_points_match_reference(tag, beta, c):
    """LAMA's state-evolution fixed points (PD / centralized) and per-cluster
    FD fixed points, iterated on the GPU (dbp_fixed_point), give the
    reference's SINRs; the Monte Carlo driver's ser_predicted follows."""
    q16 = dbp.make_constellation("qam16")
    w = np.full(c, 1.0 / c)
    for arch in ("pd", "fd", "centralized"):
        got = [A.asymptotic_sinr("lama", arch, q16, 10.0 ** (x / 10.0), beta, weights=w) for x in G[f"sinr_{tag}_snr"]]
        close(got, G[f"sinr_{tag}_lama_{arch}"], rtol=1e-9)
    if tag == "small":
        from paper_1808_04473_b200 import montecarlo as mc

        close([mc.ser_closed_form(q16, x) for x in G["sinr_small_lama_fd"]], G["ser_pred_q16"], rtol=1e-12)


def test_batched_fixed_points_one_launch():
    """A 3 SNR x 4 beta grid of LAMA fixed points in one dbp_fixed_point launch
    equals the points solved one by one, and satisfies the fixed-point
    equation w sigma2 = N0 + beta Psi(sigma2) on the GPU quadrature."""
    q16 = dbp.make_constellation("qam16")
    n0 = np.array([0.2, 0.05, 0.01])[:, None]
    beta = np.array([0.1, 0.25, 0.5, 0.8])[None, :]
    s2, it = A.fixed_points(q16, n0, beta)
    assert s2.shape == (3, 4) and np.all(it > 0)
    spec = A.MseSpec("lama", es=q16.es, constellation=q16)
    for i in range(3):
        for j in range(4):
            close(s2[i, j], A.solve_fixed_point(spec, float(n0[i, 0]), float(beta[0, j])).sigma2, rtol=1e-14)
    close(s2, n0 + beta * A.psi_mse(spec, s2), rtol=1e-10)


def test_fixed_point_multiplicity_matches_reference():
    q16 = dbp.make_constellation("qam16")
    spec = A.MseSpec("lama", es=q16.es, constellation=q16, order=32)
    for (n0, beta), want, mult in zip(((0.05, 0.5), (0.02, 1.4), (0.2, 2.0)), G["fpm_q16"], G["fpm_q16_multiple"]):
        m, hi, lo = A.fixed_point_multiplicity(spec, n0, beta)
        assert m == bool(mult)
        close([hi, lo], want, rtol=1e-8)
