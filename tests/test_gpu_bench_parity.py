"""Parity at the BENCHMARKED sizes (BASELINE.json configs c2-c5): the CUDA path
through ``B200HydroStepper`` against the C oracle (``OracleStepper``, the
restatement of the reference step pinned bitwise to the reference's goldens in
tests/test_oracle.py), on the same synthetic inputs bench.py times.

The reference path matched: ``pkg/src/octomini/hydro/step.py:81-144``
(cfl_dt + rk3_step); inputs are SURVEY.md §8(d)'s constructions.  Bar per cell
after one step: every field bitwise (tau too: the device pow is glibc's,
csrc/omb_pow.cuh), the north_star tolerance 1e-12 asserted as well; dt, amax and
fallback counts exactly equal.
"""

import os

import numpy as np
import pytest

from _cases import bitwise_mismatch, rel_close, state_of

pytestmark = pytest.mark.gpu

NTHR = os.cpu_count() or 1


def _sedov(level):
    from octomini_host import SedovConfig, build_uniform_tree, init_sedov
    from paper_2107_10987_b200 import EosConfig

    t = build_uniform_tree(level, 8, boundary="reflecting")
    init_sedov(SedovConfig(), t, EosConfig(gamma=1.4))
    return t


def _gpu(t, eos=None, mode=None, **kw):
    from paper_2107_10987_b200 import EosConfig, HydroMode
    from paper_2107_10987_b200.stepper import B200HydroStepper

    return B200HydroStepper(t, eos or EosConfig(gamma=1.4), mode or HydroMode("new"), **kw)


def _oracle(t, gamma=1.4, **kw):
    from oracle.step import OracleStepper

    return OracleStepper(t, gamma, nthreads=NTHR, **kw)


def _same(got, ref, where):
    assert bitwise_mismatch(got[:, :5], ref[:, :5]) == 0, f"{where}: rho/momenta/egas not bitwise"
    assert rel_close(got, ref, 1e-12) == 0, f"{where}: outside 1e-12"
    assert bitwise_mismatch(got, ref) == 0, f"{where}: tau not bitwise"


def _restore(t, arr):
    for lf, a in zip(t.sorted_leaves(), arr):
        lf.subgrid.interior[:] = a


def test_c2_one_step_vs_oracle():
    """c2: Sedov 128^3 = 4096 sub-grids of 8^3 (bench.py --config c2)."""
    t = _sedov(4)
    init = state_of(t).copy()
    g = _gpu(t)
    dt = g.cfl_dt(0.4)
    st = g.rk3_step(dt)
    got = state_of(t).copy()
    _restore(t, init)
    o = _oracle(t)
    assert o.cfl_dt(0.4) == dt
    o.rk3_step(dt)
    _same(got, state_of(t), "c2")
    assert st.amax == o.amax
    assert st.fallback_count == o.fallback


def test_c2_ten_steps_totals_vs_oracle():
    """c2 over 10 steps: every dt bitwise, the final state, and the conserved
    totals (problems/diagnostics.py:9-30) within 1e-12 of the oracle's."""
    from octomini_host import conservation_totals

    tg, tc = _sedov(4), _sedov(4)
    g = _gpu(tg, host_sync=False)
    o = _oracle(tc)
    for s in range(10):
        dt = g.cfl_dt(0.4)
        assert dt == o.cfl_dt(0.4), f"dt of step {s}"
        g.rk3_step(dt)
        o.rk3_step(dt)
    g.download()
    _same(state_of(tg), state_of(tc), "c2 after 10 steps")
    a = np.array(list(conservation_totals(tg).values()))
    b = np.array(list(conservation_totals(tc).values()))
    assert np.all(np.abs(a - b) <= 1e-12 * np.maximum(np.abs(b), 1e-30)), (a, b)


def test_c4_full_amr_one_step_vs_oracle():
    """c4: the full AMR Sedov tree (levels 3-6, 3,704 sub-grids)."""
    from octomini_host import amr_sedov_tree

    t = amr_sedov_tree()
    assert len(t.leaves()) == 3704
    init = state_of(t).copy()
    g = _gpu(t)
    dt = g.cfl_dt(0.4)
    st = g.rk3_step(dt)
    got = state_of(t).copy()
    _restore(t, init)
    o = _oracle(t)
    assert o.cfl_dt(0.4) == dt
    o.rk3_step(dt)
    _same(got, state_of(t), "c4")
    assert st.amax == o.amax
    assert st.fallback_count == o.fallback


def test_c4_run_lengths_bitwise():
    """The AMR run rule (leaves reading coarse/fine ghost regions join runs): the
    full c4 tree gives bitwise the same two steps with runs of 1 and of 4 leaves."""
    from octomini_host import amr_sedov_tree

    out = []
    for mr in (1, 4):
        t = amr_sedov_tree()
        g = _gpu(t, max_run=mr, host_sync=False)
        for _ in range(2):
            g.rk3_step(g.cfl_dt(0.4))
        g.download()
        out.append(state_of(t).copy())
    assert bitwise_mismatch(out[0], out[1]) == 0


def test_c5_standin_level4_vs_oracle():
    """c5 stand-in at 128^3 (rotating frame, fixed gravity, floors, outflow): one step."""
    from octomini_host import synthetic_star

    tg, eos, grav, om, fl = synthetic_star(level=4)
    tc, _, gravc, _, _ = synthetic_star(level=4)
    g = _gpu(tg, eos=eos, gravity=grav, omega=om, floors=fl)
    o = _oracle(tc, eos.gamma, omega=om, gravity=gravc, floors=(fl.rho, fl.tau, fl.vmax))
    dt = g.cfl_dt(0.4)
    assert dt == o.cfl_dt(0.4)
    st = g.rk3_step(dt)
    o.rk3_step(dt)
    a, b = state_of(tg), state_of(tc)
    assert rel_close(a, b, 1e-12) == 0
    assert bitwise_mismatch(a, b) == 0  # tau branch in the atmosphere: glibc pow on the device
    assert st.amax == o.amax
    assert st.fallback_count == o.fallback


def test_c3_morton_sample_vs_oracle():
    """c3: Sedov 256^3 (32,768 sub-grids) stepped on one GPU; the oracle advances a
    Morton sample of 512 leaves (the first level-2 octant).  Leaves whose 26
    neighbours are all in the sample (or off-domain) depend only on sample data
    for all three stages, so they must match exactly."""
    t = _sedov(5)
    init = state_of(t).copy()
    g = _gpu(t)
    dt = g.cfl_dt(0.4)
    g.rk3_step(dt)
    got = state_of(t).copy()
    _restore(t, init)
    leaves = t.sorted_leaves()
    sample = leaves[:512]
    inside = {lf.path for lf in sample}
    o = _oracle(t)
    assert o.cfl_dt(0.4) == dt
    o.rk3_step(dt, leaves=sample)
    ref = state_of(t)
    check = []
    for i, lf in enumerate(sample):
        ok = True
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    pos = t.neighbor_ipos(lf, (dx, dy, dz))
                    if pos is not None and t.leaf_at(lf.level, pos).path not in inside:
                        ok = False
        if ok:
            check.append(i)
    assert len(check) >= 200
    idx = np.array(check)
    _same(got[idx], ref[idx], "c3 sample")
