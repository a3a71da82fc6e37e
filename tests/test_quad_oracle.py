"""The oracle's Gauss-Hermite quadratures (oracle.dbp_oracle: lama_mse_pam,
lama_mse, mi_awgn) against the reference's own
kernels (tests/golden/golden_quad.npz, tests/golden/make_golden_quad.py)."""

import os

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp
from oracle import dbp_oracle as O

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_quad.npz"))


def close(a, b, rtol=1e-11, atol=1e-15):
    np.testing.assert_allclose(a, b, rtol=rtol, atol=atol)


@pytest.mark.parametrize("name", ["qpsk", "qam16", "qam64"])
def test_oracle_quadratures_match_reference(name):
    c = dbp.make_constellation(name)
    close([O.lama_mse_pam(s, c.pam_levels) for s in G["sigma2"]], G[f"{name}_mse_pam"])
    close([O.lama_mse_pam(s, c.pam_levels, 64) for s in G["sigma2"]], G[f"{name}_mse_pam_o64"])
    close([O.lama_mse(s, c.symbols, 16) for s in G["sigma2"]], G[f"{name}_mse_2d_o16"])
    close([O.mi_awgn(c.es / s, c.symbols, 16) for s in G["sinr"][1:]], G[f"{name}_mi_o16"])
