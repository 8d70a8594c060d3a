"""Passive scalars (species) on the device: each follows tau's path through the
fused stage (PPM, KT flux with the hydro signal speeds, Simpson faces, reflux,
RK update; no sources, dual energy or floors).  The reference has no species
(SURVEY.md §0.2), so the checks are exact structural properties:
  * X = rho evolves BITWISE like rho (same reconstruction, same flux formula
    u * v_n, same update; rho gets no source term either) -- on a uniform
    Sedov tree, a reflecting smooth tree in the rotating frame with gravity,
    and an AMR tree with coarse/fine ghosts and reflux;
  * X = 2 rho stays exactly 2 X (every operation commutes with a power of two);
  * sum(X dV) is conserved on a periodic tree."""

import numpy as np
import pytest

from _cases import EOS, case_tree, sources_gravity, state_of

pytestmark = pytest.mark.gpu


def _stepper(t, **kw):
    from paper_2107_10987_b200 import HydroMode
    from paper_2107_10987_b200.stepper import B200HydroStepper

    eos = kw.pop("eos", EOS)
    return B200HydroStepper(t, eos, HydroMode("new"), host_sync=False, **kw)


@pytest.mark.parametrize("name,steps", [("sedov_c1", 3), ("smooth_reflecting", 2), ("amr_reflux", 2),
                                        ("amr_sedov_small", 1)])
def test_scalar_equal_to_rho_tracks_rho(name, steps):
    t, g = case_tree(name)
    st = _stepper(t, scalars=2)
    rho = state_of(t)[:, 0]
    st.set_scalars(np.stack([rho, 2.0 * rho]))
    for _ in range(steps):
        st.rk3_step(st.cfl_dt(0.4))
    st.download()
    X = st.get_scalars()
    rho = state_of(t)[:, 0]
    assert np.array_equal(X[0], rho)
    assert np.array_equal(X[1], 2.0 * X[0])


def test_scalar_with_sources_and_rotation():
    """Rotating frame + fixed gravity (outflow; no floors so rho is never clipped): rho has no
    source term, neither has X."""
    from paper_2107_10987_b200 import EosConfig

    t, g = case_tree("sources")
    grav = sources_gravity(t, g)
    st = _stepper(t, eos=EosConfig(gamma=float(g["gamma"])), gravity=grav, omega=float(g["omega"]), scalars=1)
    st.set_scalars(state_of(t)[None, :, 0])
    st.rk3_step(st.cfl_dt(0.4))
    st.download()
    assert np.array_equal(st.get_scalars()[0], state_of(t)[:, 0])


def test_scalar_total_conserved_periodic():
    t, g = case_tree("smooth_periodic")
    st = _stepper(t, scalars=1)
    rng = np.random.default_rng(3)
    X0 = rng.uniform(0.5, 1.5, (1, len(t.sorted_leaves()), 8, 8, 8))
    st.set_scalars(X0)
    for _ in range(3):
        st.rk3_step(st.cfl_dt(0.4))
    X = st.get_scalars()
    assert abs(X.sum() - X0.sum()) <= 1e-12 * X0.sum()
    assert not np.array_equal(X, X0)


def test_scalars_rejected_with_partition():
    from paper_2107_10987_b200.partition import Partition

    t, g = case_tree("sedov_c1")
    with pytest.raises(NotImplementedError):
        _stepper(t, scalars=1, partition=Partition(t, 2, 0))
