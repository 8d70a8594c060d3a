"""Checkpoint format (reference mesh/checkpoint.py, OMCK v1) and device diagnostics."""

import os

import pytest

from _cases import GOLD, bitwise_mismatch, case_tree, golden, state_of


def test_read_reference_checkpoint():
    from octomini_host.checkpoint import read_checkpoint

    t, hdr = read_checkpoint(os.path.join(GOLD, "amr_reflux_init.omck"))
    assert hdr["time"] == 0.25 and hdr["step"] == 7 and hdr["extra"] == {"gamma": 1.4}
    g = golden("amr_reflux")
    assert bitwise_mismatch(state_of(t), g["init"]) == 0


def test_corrupt_checkpoint_rejected(tmp_path):
    from octomini_host.checkpoint import read_checkpoint
    from paper_2107_10987_b200.io import CheckpointError

    raw = open(os.path.join(GOLD, "amr_reflux_init.omck"), "rb").read()
    p = tmp_path / "bad.omck"
    p.write_bytes(raw[:-10])
    with pytest.raises(CheckpointError):
        read_checkpoint(str(p))
    p.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(CheckpointError):
        read_checkpoint(str(p))


@pytest.mark.gpu
def test_device_checkpoint_bytes_match_reference(tmp_path):
    from paper_2107_10987_b200 import EosConfig, HydroMode
    from paper_2107_10987_b200.io import write_checkpoint
    from paper_2107_10987_b200.stepper import B200HydroStepper

    t, g = case_tree("amr_reflux")
    st = B200HydroStepper(t, EosConfig(gamma=1.4), HydroMode("new"))
    out = tmp_path / "dev.omck"
    write_checkpoint(st, str(out), time=0.25, step=7, extra={"gamma": 1.4})
    assert out.read_bytes() == open(os.path.join(GOLD, "amr_reflux_init.omck"), "rb").read()


@pytest.mark.gpu
def test_device_totals_match_conservation_totals():
    from paper_2107_10987_b200 import EosConfig, HydroMode
    from paper_2107_10987_b200.io import device_totals
    from octomini_host import conservation_totals
    from paper_2107_10987_b200.stepper import B200HydroStepper

    t, g = case_tree("sedov_c1")
    st = B200HydroStepper(t, EosConfig(gamma=1.4), HydroMode("new"))
    st.rk3_step(st.cfl_dt(0.4))
    dev = device_totals(st)
    ref = conservation_totals(t)
    for k in ("mass", "sx", "sy", "sz", "egas"):
        scale = max(abs(ref[k]), ref["mass"]) if k in ("sx", "sy", "sz") else abs(ref[k])
        assert abs(dev[k] - ref[k]) <= 1e-13 * scale, k
