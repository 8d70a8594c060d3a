"""The drop-in boundary driven by octomini's OWN objects (CPU, this container
only: /root/reference does not exist on the GPU box).  LeafBatch -- the
tree -> device-batch layer B200HydroStepper is built on -- from octomini's
trees equals the one from the host restatement (tests/octomini_host), and the
fused stage kernel's code (host emulation) steps octomini's trees to the
reference's goldens."""

import os
import sys

import numpy as np
import pytest

from _cases import EOS, bitwise_mismatch, golden, state_of

REF_SRC = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="octomini (the reference) not present")


@pytest.fixture(scope="module")
def om():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    os.environ.setdefault("OCTOMINI_BACKEND", "numpy")
    import octomini.mesh
    import octomini.problems

    return octomini


def _trees(om, kind):
    import octomini_host as host

    out = []
    for M in (om.mesh, host):
        if kind == "amr":
            t = M.build_uniform_tree(1, 8, boundary="periodic")
            t.split(t.leaf_at(1, (0, 0, 0)))
            t.reindex()
        else:
            t = M.build_uniform_tree(2, 8, boundary=kind)
        out.append(t)
    return out


@pytest.mark.parametrize("kind", ["reflecting", "periodic", "outflow", "amr"])
def test_leafbatch_from_octomini_trees(om, kind):
    from paper_2107_10987_b200.batch import LeafBatch

    t_ref, t_host = _trees(om, kind)
    assert [lf.path for lf in t_ref.sorted_leaves()] == [lf.path for lf in t_host.sorted_leaves()]
    rng = np.random.default_rng(5)
    for a, b in zip(t_ref.sorted_leaves(), t_host.sorted_leaves()):
        v = rng.uniform(0.5, 2.0, a.subgrid.interior.shape)
        a.subgrid.interior[:] = v
        b.subgrid.interior[:] = v
    A, B = LeafBatch(t_ref), LeafBatch(t_host)
    assert A.info.tobytes() == B.info.tobytes()
    for k in ("run_off", "run_leaf", "amr_tasks", "reflux_leaf", "reflux_off", "reflux_tasks", "dx"):
        assert np.array_equal(getattr(A, k), getattr(B, k)), k
    assert (A.bc, A.nvirtual, A.flux_slots, A.fstride) == (B.bc, B.nvirtual, B.flux_slots, B.fstride)
    assert bitwise_mismatch(A.pack(), B.pack()) == 0


def test_emulated_step_on_octomini_tree(om):
    """Sedov config c1 built by octomini itself (build_uniform_tree + init_sedov),
    stepped by the fused kernel's code: the reference's golden step, bitwise."""
    from emu import EmuStepper

    g = golden("sedov_c1")
    t = om.mesh.build_uniform_tree(2, 8, boundary="reflecting")
    om.problems.init_sedov(om.problems.SedovConfig(), t, om.hydro.EosConfig(gamma=1.4))
    assert bitwise_mismatch(state_of(t), g["init"]) == 0
    em = EmuStepper(t, 1.4)
    em.rk3_step(float(g["dts"][0]))
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0
    assert em.amax == float(g["amax"][0])


def test_stepper_accepts_octomini_types(om):
    """octomini's own EosConfig / HydroMode / FloorConfig carry what the stepper
    reads (duck-typed): gamma, dual_energy_eta, is_new, quadrature_override,
    contact_detection, rho / tau / vmax."""
    e = om.hydro.EosConfig(gamma=1.4)
    m = om.hydro.HydroMode("new", contact_detection=True)
    f = om.hydro.FloorConfig(rho=1e-4)
    assert (e.gamma, e.dual_energy_eta) == (EOS.gamma, EOS.dual_energy_eta)
    assert m.is_new and m.contact_detection and not m.quadrature_override
    assert (f.rho, f.tau, f.vmax) == (1e-4, 0.0, 0.0)
