"""The scalar flux surface (reference hydro/flux.py:12-94) on the device:
kt_flux / physical_flux / face_flux against the reference's own outputs
(tests/golden/flux_points.npz, kernels.npz ``sod_flux``) bit for bit, and the
reference's flux tests (pkg/tests/test_hydro.py:180-279) restated."""

import numpy as np
import pytest

from _cases import EOS, bitwise_mismatch, golden

pytestmark = pytest.mark.gpu


class PState:
    """Point state with the reference PrimitiveState's fields (flux.py:12-30)."""

    def __init__(self, rho, v, p, eos=EOS, tau=None):
        self.rho, self.vx, self.vy, self.vz, self.p = rho, v[0], v[1], v[2], p
        self.eint = p / ((eos.gamma - 1.0) * rho)
        self.tau = (rho * self.eint) ** (1.0 / eos.gamma) if tau is None else tau


@pytest.fixture(scope="module")
def F():
    from paper_2107_10987_b200 import flux

    return flux


def test_sod_mass_flux_pinned(F):
    """test_hydro.py:195-207: F_rho = 0.5176569810216458 (and the reference's own value, bitwise)."""
    f = F.kt_flux(PState(1.0, (0, 0, 0), 1.0), PState(0.125, (0, 0, 0), 0.1), 0, EOS)
    assert f[0] == pytest.approx(0.5176569810216458, rel=1e-12)
    assert bitwise_mismatch(f, golden("kernels")["sod_flux"]) == 0


def test_kt_flux_matches_reference_points(F):
    g = golden("flux_points")
    S = g["states"]
    for ax in range(3):
        got = F.kt_flux_batch(S[0], S[1], ax, EOS.gamma)
        assert bitwise_mismatch(got, g[f"kt_{ax}"]) == 0
        phys = np.array([F.physical_flux(type("S", (), dict(zip(F.STATE_FIELDS, row)))(), ax) for row in S[0][:8]])
        assert bitwise_mismatch(phys, g[f"phys_{ax}"][:8]) == 0


def test_face_flux_matches_reference(F):
    g = golden("flux_points")
    assert bitwise_mismatch(F.face_flux_batch(g["face_pts"], True), g["face_new"]) == 0
    assert bitwise_mismatch(F.face_flux_batch(g["face_pts"], False), g["face_old"]) == 0
    assert bitwise_mismatch(F.face_flux(g["face_pts"][0]), g["face_pts"][0, 0]) == 0  # all equal: bitwise


def test_identical_states_and_upwind(F):
    """test_hydro.py:180-193: kt(s, s) = F(s); both states supersonic to -x: F(uR)."""
    s = PState(1.3, (0.2, -0.1, 0.4), 0.9)
    for ax in range(3):
        assert np.allclose(F.kt_flux(s, s, ax, EOS), F.physical_flux(s, ax), rtol=1e-14)
    l = PState(1.0, (-5.0, 0, 0), 0.5)
    r = PState(0.8, (-6.0, 0, 0), 0.4)
    assert np.allclose(F.kt_flux(l, r, 0, EOS), F.physical_flux(r, 0), rtol=1e-14)


def test_non_finite_rejected(F):
    from paper_2107_10987_b200 import NumericsError

    bad = PState(1.0, (np.nan, 0, 0), 1.0)
    ok = PState(1.0, (0, 0, 0), 1.0)
    with pytest.raises(NumericsError, match="non-finite state passed to kt_flux"):
        F.kt_flux(bad, ok, 0, EOS)


def test_swap_reflect_symmetry(F):
    """test_hydro.py:218-236."""
    rng = np.random.default_rng(1)
    for _ in range(10):
        rho = rng.uniform(0.1, 3.0, 2)
        p = rng.uniform(0.1, 3.0, 2)
        v = rng.normal(0, 1, (2, 3))
        f = F.kt_flux(PState(rho[0], v[0], p[0]), PState(rho[1], v[1], p[1]), 0, EOS)
        fm = F.kt_flux(PState(rho[1], (-v[1, 0], v[1, 1], v[1, 2]), p[1]),
                       PState(rho[0], (-v[0, 0], v[0, 1], v[0, 2]), p[0]), 0, EOS)
        assert fm[0] == pytest.approx(-f[0], rel=1e-12, abs=1e-14)
        assert fm[1] == pytest.approx(f[1], rel=1e-12, abs=1e-14)
        assert fm[2] == pytest.approx(-f[2], rel=1e-12, abs=1e-14)
        assert fm[4] == pytest.approx(-f[4], rel=1e-12, abs=1e-14)


def test_face_flux_shape_error(F):
    with pytest.raises(ValueError):
        F.face_flux(np.zeros((8, 6)))
