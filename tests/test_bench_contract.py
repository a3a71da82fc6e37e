"""bench.py's JSON contract on the host (no GPU): both arms describe the
workload with the same config dict (the driver's same_config check), the
L2 note included, and every BASELINE config is a known workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_config_dict_carries_the_l2_note_for_both_arms():
    for name, wl in bench.WORKLOADS.items():
        cfg = bench.config_dict(name, wl)
        assert cfg["workload"] and cfg["items_per_step"] == wl["frames"] * bench.W
        step_bytes, sets = bench.input_sets(wl)
        assert step_bytes == wl["frames"] * bench.W * (wl["B"] * wl["U"] + bench.T * wl["B"]) * 8
        # below 4x the L2 two input sets alternate; above it every step streams from HBM anyway
        assert sets == (2 if step_bytes < 4 * bench.L2_BYTES else 1)
        assert cfg["l2"] == bench.l2_note(wl)
        assert f"{sets} input set(s)" in cfg["l2"]


def test_headline_workload_is_cfg2():
    wl = bench.WORKLOADS["cfg2"]
    assert (wl["arch"], wl["kind"], wl["B"], wl["C"], wl["U"], wl["frames"]) == ("pd", "lmmse", 128, 4, 16, 11)
