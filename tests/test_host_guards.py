"""Host-side guards of the drop-in API that need no GPU.

``_check_sigma2`` mirrors the reference's variance guard
(/root/reference/pkg/src/dbp/equalize.py:115-120) and its own test
(/root/reference/pkg/tests/test_equalize.py:142-150); the device kernels report
the same condition as status ST_NEGVAR (tests/test_gpu_api.py)."""

import numpy as np
import pytest

import paper_1808_04473_b200 as dbp
from paper_1808_04473_b200.equalize import _check_sigma2


def test_negative_variance_guard():
    with pytest.raises(dbp.NegativeVarianceError):
        _check_sigma2(np.array([0.1, -0.5]), "zf")
    # rounding-level negatives are clamped, not fatal
    cleaned = _check_sigma2(np.array([0.1, -1e-14]), "zf")
    assert cleaned[1] == 0.0


def test_message_volume_matches_reference_formula():
    """model.message_volume (reference model.py:260-280): PD sends the Gram
    and the matched filter per subcarrier, FD the estimates, consensus
    sharing twice FD's volume.  The multi-GPU bench's NVLink algorithmic bytes
    are these volumes (distributed.nvlink_bytes)."""
    u, nsc, nsym, c = 16, 1200, 14, 4
    mv = dbp.message_volume(u, nsc, nsym, c)
    assert mv.pd_bytes == (u * u * nsc + u * nsc * nsym) * c * 8
    assert mv.fd_bytes == u * nsc * nsym * c * 8
    assert mv.cs_bytes == 2 * mv.fd_bytes
    assert dbp.message_volume(u, nsc, nsym, c, bytes_per_entry=4).pd_bytes == mv.pd_bytes // 2
    for bad in ((0, 1, 1, 1), (1, 1.5, 1, 1), (1, 1, 1, -2)):
        with pytest.raises(dbp.ConfigError):
            dbp.message_volume(*bad)
