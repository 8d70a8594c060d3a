"""Device FMM gravity against the reference's own
FmmSolver (goldens made by tests/golden/make_golden.py fmm with the compiled
backend): the host preparation (entity table, dual-tree traversal, grouping)
must reproduce the reference's interaction groups exactly (CPU), and the
device solve must reproduce phi, g and dphi/dt bitwise (GPU)."""

import hashlib
import json

import numpy as np
import pytest

from _cases import golden
import octomini_host as mesh
from paper_2107_10987_b200 import gravity


def _fill(tree, g, name):
    assert [json.loads(p) for p in g[f"{name}_paths"]] == [list(lf.path) for lf in tree.sorted_leaves()]
    for lf, rho in zip(tree.sorted_leaves(), g[f"{name}_rho"]):
        lf.subgrid.interior[0] = rho
    return tree


def _tree(name):
    if name in ("u05", "u035", "u0"):
        return mesh.build_uniform_tree(1, 8)
    t = mesh.build_uniform_tree(1, 8)
    t.split(t.leaf_at(1, (0, 0, 0)))
    t.reindex()
    return t


@pytest.mark.parametrize("name", ["u05", "u035", "amr05"])
def test_interaction_groups_match_reference(name):
    from paper_2107_10987_b200 import _lib

    g = golden("fmm")
    t = _fill(_tree(name), g, name)
    table = gravity.EntityTable(t)
    pa, pb, pk = gravity.traverse(_lib.load(), table, float(g[f"{name}_theta"]))
    order, bounds, R, a_cell, b_cell = gravity.group_pairs(table, pa, pb, pk)
    assert [len(R), len(pa)] == list(g[f"{name}_stats"])
    assert np.array_equal(R, g[f"{name}_R"])
    h = hashlib.sha256()
    for k in range(len(R)):
        sel = order[bounds[k]:bounds[k + 1]]
        h.update(np.ascontiguousarray(pa[sel], dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(pb[sel], dtype=np.int64).tobytes())
        h.update(bytes([int(a_cell[k]), int(b_cell[k])]))
    assert h.hexdigest() == str(g[f"{name}_pairs_sha"])


def test_kernel_derivatives_formula():
    """D(R) of g = -1/|R|: D0 = -1/r, D1 = R/r^3 (multipole.py:173-191); at -R the odd ranks flip."""
    R = np.array([[0.3, -0.4, 1.2], [1.0, 2.0, -0.5]])
    D = gravity.derivative_table(R)
    for g in range(2):
        r = np.sqrt(R[g] @ R[g])
        assert D[g, 0, 0] == -1.0 / r
        assert np.allclose(D[g, 0, 1:4], R[g] / r ** 3, rtol=1e-15)
        assert np.array_equal(D[g, 1, 1:4], -D[g, 0, 1:4]) and np.array_equal(D[g, 1, 4:10], D[g, 0, 4:10])
        assert np.array_equal(D[g, 1, 10:], -D[g, 0, 10:])
    # trace-free rank 2 (the kernel is harmonic away from 0)
    assert abs(D[0, 0, 4] + D[0, 0, 7] + D[0, 0, 9]) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["u05", "u035", "amr05", "u0"])
def test_device_fmm_bitwise(name):
    """theta 0.5 / 0.35: the FMM; theta 0: the always-reject direct summation."""
    g = golden("fmm")
    t = _fill(_tree(name), g, name)
    solver = gravity.B200FmmSolver(float(g[f"{name}_theta"]))
    phi, gg = solver.solve_density(t)
    if f"{name}_stats" in g:
        assert solver.stats["pairs"] == int(g[f"{name}_stats"][1])
    for i, lf in enumerate(t.sorted_leaves()):
        assert np.array_equal(phi[lf.path], g[f"{name}_phi"][i]), (name, i, "phi")
        assert np.array_equal(gg[lf.path], g[f"{name}_g"][i]), (name, i, "g")


@pytest.mark.gpu
def test_device_fmm_full_solve_with_dphi_dt():
    g = golden("fmm")
    t = mesh.build_uniform_tree(1, 8, boundary="reflecting")
    assert [json.loads(p) for p in g["full_paths"]] == [list(lf.path) for lf in t.sorted_leaves()]
    for lf, u in zip(t.sorted_leaves(), g["full_u"]):
        lf.subgrid.u[...] = u  # interiors + the reference's filled ghosts
    field = gravity.B200FmmSolver(0.5).solve(t, need_derivative=True)
    for i, lf in enumerate(t.sorted_leaves()):
        for k in ("phi", "gx", "gy", "gz", "dphi_dt"):
            assert np.array_equal(field[lf.path][k], g[f"full_{k}"][i]), (i, k)


@pytest.mark.gpu
def test_self_gravitating_steps_match_reference():
    """HydroStepper + FmmSolver re-solved every stage (step.py:111-113) vs
    B200HydroStepper + B200FmmSolver solved on the device from the stage
    state: 2 RK3 steps, rotating frame, reflecting walls."""
    from _cases import EOS, case_tree, state_of

    from paper_2107_10987_b200 import HydroMode
    from paper_2107_10987_b200.stepper import B200HydroStepper

    t, g = case_tree("gravity_step")
    st = B200HydroStepper(t, EOS, HydroMode("new"), gravity=gravity.B200FmmSolver(0.5), omega=0.3)
    for s in range(2):
        dt = st.cfl_dt(0.4)
        assert dt == float(g["dts"][s])
        stats = st.rk3_step(dt)
        assert stats.amax == float(g["amax"][s])
        if s == 0:
            got, ref = state_of(t), g["state1"]
            assert np.count_nonzero(got != ref) == 0
    # after 2 steps: every field bitwise (tau too: the device pow is glibc's)
    got, ref = state_of(t), g["final"]
    assert np.count_nonzero(got != ref) == 0
    assert np.all(np.abs(got - ref) <= 1e-12 * np.abs(ref))
