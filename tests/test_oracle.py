"""The CPU oracle against the golden fixtures the reference itself produced.

This pins the checker before it is trusted for the CUDA parity tests
(fixtures: tests/golden/make_golden.py, reference tests it mirrors:
pkg/tests/test_backends.py, test_hydro_step.py, test_mesh.py)."""

import hashlib

import numpy as np
import pytest

import oracle
from oracle.ghosts import exchange
from oracle.step import OracleStepper
import octomini_host as mesh

from _cases import bitwise_mismatch, case_tree, golden, sources_gravity, state_of

CORE = (slice(None), slice(None), slice(2, 12), slice(2, 12), slice(2, 12))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def K():
    return golden("kernels")


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_kernels_bitwise(K, seed):
    u = K[f"s{seed}_u"]
    prim = oracle.primitives(u, 1.4, 1e-3)
    assert sha(prim) == str(K[f"s{seed}_prim_sha"])
    for new in (True, False):
        for contact in (False, True):
            tag = f"s{seed}_{'new' if new else 'old'}_{'c' if contact else 'nc'}"
            lo, hi, fb = oracle.reconstruct(prim, 8, new, contact, 1.4)
            assert fb == int(K[tag + "_fallback"])
            assert sha(lo[CORE]) == str(K[tag + "_lo_sha"])
            assert sha(hi[CORE]) == str(K[tag + "_hi_sha"])
            if contact:
                continue
            for ov in ((False, True) if new else (False,)):
                t2 = tag + ("_ov" if ov else "")
                fx, fy, fz, am = oracle.fluxes(lo, hi, 8, 1.4, new, ov)
                for got, key in ((fx, "_fx"), (fy, "_fy"), (fz, "_fz")):
                    assert bitwise_mismatch(got, K[t2 + key]) == 0
                assert am == float(K[t2 + "_amax"])


@pytest.mark.parametrize("tag", ["fb", "fb2"])
def test_positivity_fallback_case(K, tag):
    prim = oracle.primitives(K[tag + "_u"], 1.4, 1e-3)
    lo, hi, fb = oracle.reconstruct(prim, 8, True, False, 1.4)
    assert fb == int(K[tag + "_fallback"])
    assert sha(lo[CORE]) == str(K[tag + "_lo_sha"]) and sha(hi[CORE]) == str(K[tag + "_hi_sha"])
    fx, fy, fz, am = oracle.fluxes(lo, hi, 8, 1.4, True, False)
    for got, key in ((fx, "_fx"), (fy, "_fy"), (fz, "_fz")):
        assert bitwise_mismatch(got, K[tag + key]) == 0
    assert am == float(K[tag + "_amax"])


@pytest.mark.parametrize("bnd", ["periodic", "reflecting", "outflow", "amr"])
def test_ghost_fill(bnd):
    g = golden("ghosts")
    if bnd == "amr":
        t = mesh.build_uniform_tree(1, 8, boundary="reflecting")
        t.split(t.leaf_at(1, (0, 0, 0)))
        t.reindex()
    else:
        t = mesh.build_uniform_tree(1, 8, boundary=bnd)
    for lf, u in zip(t.sorted_leaves(), g[bnd]):  # golden interiors as input
        lf.subgrid.interior[:] = u[:, 3:11, 3:11, 3:11]
    exchange(t)
    got = np.stack([lf.subgrid.u for lf in t.sorted_leaves()])
    assert bitwise_mismatch(got, g[bnd]) == 0


@pytest.mark.parametrize("name", ["smooth_periodic", "smooth_reflecting", "smooth_old", "amr_reflux",
                                  "amr_sedov_small"])
def test_step_cases_bitwise(name):
    t, g = case_tree(name)
    st = OracleStepper(t, 1.4, new_mode=(name != "smooth_old"))
    cfl = 0.3 if name == "smooth_old" else 0.4
    dts = []
    for s in range(len(g["dts"])):
        dt = st.cfl_dt(cfl)
        dts.append(dt)
        st.rk3_step(dt)
        if s == 0:
            assert bitwise_mismatch(state_of(t), g["state1"]) == 0
        assert st.amax == float(g["amax"][s])
        assert st.fallback == int(g["fallback"][s])
    assert dts == list(g["dts"])
    assert sha(state_of(t)) == str(g["final_sha"])


def test_sedov_c1_ten_steps():
    t, g = case_tree("sedov_c1")
    st = OracleStepper(t, 1.4)
    for s in range(10):
        dt = st.cfl_dt(0.4)
        assert dt == float(g["dts"][s])
        st.rk3_step(dt)
        if s == 0:
            assert bitwise_mismatch(state_of(t), g["state1"]) == 0
    assert sha(state_of(t)) == str(g["final_sha"])
    # SURVEY.md §8c regression values
    assert float(g["dts"][0]) == 0.006602767292665797
    assert float(g["dts"][9]) == 0.004866124696693348


def test_sources_and_floors():
    t, g = case_tree("sources")
    grav = sources_gravity(t, g)
    fl = tuple(float(x) for x in g["floors"])
    st = OracleStepper(t, float(g["gamma"]), omega=float(g["omega"]), gravity=grav, floors=fl)
    dt = st.cfl_dt(0.4)
    assert dt == float(g["dts"][0])
    st.rk3_step(dt)
    assert bitwise_mismatch(state_of(t), g["state1"]) == 0
