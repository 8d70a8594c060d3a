"""The device pow (csrc/omb_pow.cuh: glibc's algorithm and tables, read off this
image's libm) compiled for the host and checked bitwise against libm's pow --
CPU only.  The reference's tau goes through glibc pow (reference.py:39,
hydro/eos.py:50-61), so this is what makes tau bitwise on the GPU."""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_host_compiled_pow_matches_libm(tmp_path):
    exe = tmp_path / "pow_check"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-o", str(exe),
                    os.path.join(HERE, "native", "pow_check.cpp"), "-lm"], check=True)
    res = subprocess.run([str(exe), str(1 << 24)], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout[-2000:]
    assert "0 mismatches" in res.stdout


def test_tables_are_this_libm():
    """omb_pow_tables.cuh regenerated from the image's libm is unchanged."""
    import sys

    csrc = os.path.join(os.path.dirname(HERE), "paper_2107_10987_b200", "csrc")
    path = os.path.join(csrc, "omb_pow_tables.cuh")
    before = open(path).read()
    subprocess.run([sys.executable, os.path.join(csrc, "gen_glibc_pow_tables.py")], check=True,
                   capture_output=True)
    assert open(path).read() == before
