"""The fused stage kernel's logic (compiled for the host, tests/native) against
the golden fixtures made by the reference -- CPU only, no GPU needed."""

import numpy as np
import pytest

from _cases import bitwise_mismatch, case_tree, golden, sources_gravity, state_of
from emu import EmuStepper, lib


@pytest.mark.parametrize("name", ["smooth_periodic", "smooth_reflecting"])
@pytest.mark.parametrize("max_run,nthr", [(1, 512), (2, 512), (2, 256), (3, 384)])
def test_emulated_step_matches_golden(name, max_run, nthr):
    t, g = case_tree(name)
    dt = float(g["dts"][0])
    em = EmuStepper(t, 1.4, max_run=max_run, nthr=nthr)
    em.rk3_step(dt)
    got = state_of(t)
    assert bitwise_mismatch(got[:, :5], g["state1"][:, :5]) == 0
    assert bitwise_mismatch(got, g["state1"]) == 0
    assert em.amax == float(g["amax"][0])
    assert em.fallback == int(g["fallback"][0])


def test_emulated_old_scheme():
    t, g = case_tree("smooth_old")
    em = EmuStepper(t, 1.4, new_mode=False)
    em.rk3_step(float(g["dts"][0]))
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0
    assert em.amax == float(g["amax"][0])


def test_emulated_sedov_c1():
    t, g = case_tree("sedov_c1")
    em = EmuStepper(t, 1.4, max_run=4)
    em.rk3_step(float(g["dts"][0]))
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0
    assert em.amax == float(g["amax"][0])


def test_emulated_sources_and_floors():
    t, g = case_tree("sources")
    grav = sources_gravity(t, g)
    fl = tuple(float(x) for x in g["floors"])
    em = EmuStepper(t, float(g["gamma"]), omega=float(g["omega"]), grav=grav.fields, floors=fl)
    em.rk3_step(float(g["dts"][0]))
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0


def test_emulated_gather_matches_ghost_golden():
    import ctypes
    import octomini_host as mesh
    from paper_2107_10987_b200.batch import LeafBatch

    g = golden("ghosts")
    for bnd in ("periodic", "reflecting", "outflow"):
        t = mesh.build_uniform_tree(1, 8, boundary=bnd)
        for lf, u in zip(t.sorted_leaves(), g[bnd]):
            lf.subgrid.interior[:] = u[:, 3:11, 3:11, 3:11]
        b = LeafBatch(t)
        U = np.ascontiguousarray(b.pack())
        for i in range(b.L):
            out = np.empty((6, 14, 14, 14))
            lib().emu_gather(U.ctypes.data, b.fstride, b.info.ctypes.data, i, b.bc, out.ctypes.data)
            assert bitwise_mismatch(out, g[bnd][i]) == 0, (bnd, i)


def test_emulated_amr_reflux_two_steps():
    """Coarse/fine ghosts (virtual leaves) + flux export + reflux, vs the reference (2 steps)."""
    import hashlib

    t, g = case_tree("amr_reflux")
    em = EmuStepper(t, 1.4, max_run=2)
    assert em.b.nvirtual > 0 and len(em.b.reflux_leaf) > 0
    for s in range(2):
        em.rk3_step(float(g["dts"][s]))
        if s == 0:
            assert bitwise_mismatch(state_of(t), g["state1"]) == 0
        assert em.amax == float(g["amax"][s])
    assert hashlib.sha256(np.ascontiguousarray(state_of(t)).tobytes()).hexdigest() == str(g["final_sha"])


def test_emulated_amr_ghost_regions():
    """Gathered padded blocks (incl. prolonged / restricted regions) equal the reference ghost fill."""
    import ctypes
    import json

    import octomini_host as mesh
    from paper_2107_10987_b200._abi import OmbAmrDesc
    from paper_2107_10987_b200.batch import LeafBatch

    g = golden("ghosts")
    t = mesh.build_uniform_tree(1, 8, boundary="reflecting")
    t.split(t.leaf_at(1, (0, 0, 0)))
    t.reindex()
    assert [json.loads(p) for p in g["amr_paths"]] == [list(lf.path) for lf in t.sorted_leaves()]
    for lf, u in zip(t.sorted_leaves(), g["amr"]):
        lf.subgrid.interior[:] = u[:, 3:11, 3:11, 3:11]
    b = LeafBatch(t)
    U = np.ascontiguousarray(b.pack())
    tasks = np.ascontiguousarray(b.amr_tasks.reshape(-1))
    lib().emu_amr_ghosts(ctypes.byref(OmbAmrDesc(u=U.ctypes.data, fstride=b.fstride, tasks=tasks.ctypes.data,
                                                  ntasks=b.nvirtual)))
    for i in range(b.L):
        out = np.empty((6, 14, 14, 14))
        lib().emu_gather(U.ctypes.data, b.fstride, b.info.ctypes.data, i, b.bc, out.ctypes.data)
        assert bitwise_mismatch(out, g["amr"][i]) == 0, i


def test_emulated_amr_sedov_small():
    """Reduced config c4 (Sedov on a 3-level refined octree) vs the reference, one step."""
    t, g = case_tree("amr_sedov_small")
    em = EmuStepper(t, 1.4)
    em.rk3_step(float(g["dts"][0]))
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0
    assert em.amax == float(g["amax"][0])


@pytest.mark.parametrize("max_run", [1, 4])
def test_emulated_contact_detection(max_run):
    """contact_detection=True: the steepener inside the fused kernel's mono6 (P1/P3)."""
    t, g = case_tree("contact_step")
    em = EmuStepper(t, 1.4, contact=True, max_run=max_run)
    em.rk3_step(float(g["dts"][0]))
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0
    assert em.amax == float(g["amax"][0])
    assert em.fallback == int(g["fallback"][0])


@pytest.mark.parametrize("override", [True, False])
def test_emulated_override_equals_old(override):
    """new + quadrature_override and old: the reference's 10-step state bitwise
    (tests/test_hydro_step.py:151-164 pins old == new+override)."""
    t, g = case_tree("override_10")
    em = EmuStepper(t, 1.4, new_mode=override, override=override)  # override=False: the old scheme
    dt = float(g["dt"])
    for _ in range(10):
        em.rk3_step(dt)
    assert bitwise_mismatch(state_of(t), g["final"]) == 0


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("name", ["smooth_reflecting", "amr_sedov_small", "contact_step"])
def test_emulated_race_check(order, name):
    """Shared-memory race check of the fused kernel's phase code (compute-sanitizer
    is unavailable on the GPU pool): the simulated threads of every barrier
    interval run in descending / permuted order, and the cp.async staging lands
    only at the issuing thread's wait.  A read of data another thread writes in
    the same interval, or of a staged copy before its wait + barrier, changes the
    result; the golden step must come out bitwise regardless."""
    t, g = case_tree(name)
    lib().emu_set_order(order)
    try:
        em = EmuStepper(t, 1.4, contact=(name == "contact_step"), max_run=4)
        em.rk3_step(float(g["dts"][0]))
    finally:
        lib().emu_set_order(0)
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0
    assert em.amax == float(g["amax"][0])
    assert em.fallback == int(g["fallback"][0])


@pytest.mark.parametrize("name", ["sedov_c1", "amr_reflux"])
def test_emulated_scalar_tracks_rho(name):
    """The passive-scalar pass of the fused kernel (host emulation): X = rho stays
    bitwise rho, X = 2 rho stays 2 X (uniform and AMR with reflux)."""
    t, g = case_tree(name)
    em = EmuStepper(t, 1.4, max_run=4)
    rho = state_of(t)[:, 0]
    em.scalars = np.stack([rho, 2.0 * rho])
    em.rk3_step(float(g["dts"][0]))
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0
    assert np.array_equal(em.scalars[0], state_of(t)[:, 0])
    assert np.array_equal(em.scalars[1], 2.0 * em.scalars[0])


@pytest.mark.parametrize("name", ["sedov_n16", "sedov_n32", "smooth_n16", "fallback_n16"])
def test_emulated_subgrid_sizes(name):
    """16^3 and 32^3 sub-grids run as 8^3 blocks (paper_2107_10987_b200/blocks.py): the
    reference's step bitwise, and its per-leaf positivity-fallback count exactly."""
    t, g = case_tree(name)
    em = EmuStepper(t, 1.4)
    em.rk3_step(float(g["dts"][0]))
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0
    assert em.amax == float(g["amax"][0])
    assert em.fallback == int(g["fallback"][0])
