"""Generate the golden fixtures by running the REFERENCE (octomini) itself.

Run in the build container only (the reference does not travel):

    oracle/make_ref.sh                      # scratch build of octomini + Cython kernels
    NPY_DISABLE_CPU_FEATURES="AVX512F AVX512CD AVX512_SKX AVX512_CLX AVX512_CNL AVX512_ICL AVX512_SPR" \
    OCTOMINI_BACKEND=compiled PYTHONPATH=/tmp/omb_ref/src python tests/golden/make_golden.py

The numpy SIMD env makes numpy's float64 ``power`` call glibc ``pow`` (the
AVX-512 kernel differs from it in ~5% of inputs), so the
fixtures are reproducible by a libm-based restatement.  Every fixture records
the env it was made with.  Cases mirror the reference's own tests:
``tests/test_backends.py:19-72`` (random sub-grids), ``tests/test_hydro_step.py:21-149``
(uniform / smooth periodic / reflecting / AMR reflux), the Sedov benchmark
config c1, sources + floors, and the ghost-fill KATs of
``tests/test_mesh.py``.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from octomini import kernels  # noqa: E402
from octomini._kernels import _core as C  # noqa: E402
from octomini._kernels import reference as R  # noqa: E402
from octomini.hydro import (EosConfig, FloorConfig, HydroMode, HydroStepper,  # noqa: E402
                            conserved_from_primitive, kt_flux, PrimitiveState)
from octomini.mesh import build_uniform_tree, exchange_ghosts  # noqa: E402
from octomini.problems import SedovConfig, conservation_totals, init_sedov  # noqa: E402

assert kernels.BACKEND_NAME == "compiled", "set OCTOMINI_BACKEND=compiled"
ENV = {
    "NPY_DISABLE_CPU_FEATURES": os.environ.get("NPY_DISABLE_CPU_FEATURES", ""),
    "numpy": np.__version__,
    "backend": kernels.BACKEND_NAME,
}
if "AVX512F" not in ENV["NPY_DISABLE_CPU_FEATURES"]:
    print("warning: numpy AVX-512 power active; tau goldens will not match glibc pow", file=sys.stderr)

EOS = EosConfig(gamma=1.4)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def save(name, **arrays):
    arrays["env"] = np.array(json.dumps(ENV))
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, os.path.getsize(os.path.join(HERE, name + ".npz")), "bytes")


def random_subgrid(seed, n=8):
    """tests/test_backends.py:19-28"""
    rng = np.random.default_rng(seed)
    tree = build_uniform_tree(0, n, boundary="periodic")
    sg = tree.leaves()[0].subgrid
    rho = rng.uniform(0.2, 3.0, (n, n, n))
    p = rng.uniform(0.2, 3.0, (n, n, n))
    v = rng.normal(0, 1, (3, n, n, n))
    sg.interior[:] = conserved_from_primitive(rho, v, p, EOS)
    exchange_ghosts(tree)
    return sg


def kernel_cases():
    core = (slice(None), slice(None), slice(2, 12), slice(2, 12), slice(2, 12))
    out = {}
    for seed in (0, 1, 2, 3):
        sg = random_subgrid(seed)
        if seed == 3:  # a sharp contact so the steepener fires (test_backends.py:60-72)
            sg.interior[0, :4] *= 4.0
        prim = R.primitives(sg.u, EOS.gamma, EOS.dual_energy_eta)
        out[f"s{seed}_u"] = sg.u.copy()
        out[f"s{seed}_prim_sha"] = np.array(sha(prim))
        for new in (True, False):
            for contact in (False, True):
                lo, hi, fb = C.reconstruct(prim, 8, new, contact, EOS.gamma)
                tag = f"s{seed}_{'new' if new else 'old'}_{'c' if contact else 'nc'}"
                out[tag + "_lo_sha"] = np.array(sha(lo[core]))
                out[tag + "_hi_sha"] = np.array(sha(hi[core]))
                out[tag + "_fallback"] = np.array(fb)
                if contact:
                    continue
                for override in ((False, True) if new else (False,)):
                    fx, fy, fz, am = C.fluxes(lo, hi, 8, EOS.gamma, new, override)
                    t2 = tag + ("_ov" if override else "")
                    out[t2 + "_fx"], out[t2 + "_fy"], out[t2 + "_fz"] = fx, fy, fz
                    out[t2 + "_amax"] = np.array(am)
        # contact-on fluxes for the sharp-contact seed
        if seed == 3:
            lo, hi, _ = C.reconstruct(prim, 8, True, True, EOS.gamma)
            fx, fy, fz, am = C.fluxes(lo, hi, 8, EOS.gamma, True, False)
            out["s3_new_c_fx"], out["s3_new_c_fy"], out["s3_new_c_fz"] = fx, fy, fz
            out["s3_new_c_amax"] = np.array(am)
    # positivity fallback case (tests/test_hydro.py:152-170)
    tree = build_uniform_tree(0, 8, boundary="periodic")
    sg = tree.leaves()[0].subgrid
    rho = np.full((8, 8, 8), 1.0)
    rho[4, 4, 4] = 1e-12
    rho[5, 4, 4] = 1e3
    sg.interior[:] = conserved_from_primitive(rho, (0.0, 0.0, 0.0), 1.0, EOS)
    exchange_ghosts(tree)
    prim = R.primitives(sg.u, EOS.gamma, EOS.dual_energy_eta)
    lo, hi, fb = C.reconstruct(prim, 8, True, False, EOS.gamma)
    fx, fy, fz, am = C.fluxes(lo, hi, 8, EOS.gamma, True, False)
    out.update(fb_u=sg.u.copy(), fb_fallback=np.array(fb), fb_lo_sha=np.array(sha(lo[core])),
               fb_hi_sha=np.array(sha(hi[core])), fb_fx=fx, fb_fy=fy, fb_fz=fz, fb_amax=np.array(am))
    # zero-pressure cells (tau = 0 and egas < kinetic -> p = 0): fallback fires
    sg2 = random_subgrid(5)
    for c in ((3, 4, 5), (4, 4, 4), (6, 2, 7)):
        sg2.interior[5][c] = 0.0
        sg2.interior[4][c] = 0.0
    tree2 = build_uniform_tree(0, 8, boundary="periodic")
    tree2.leaves()[0].subgrid.interior[:] = sg2.interior
    exchange_ghosts(tree2)
    u2 = tree2.leaves()[0].subgrid.u
    prim = R.primitives(u2, EOS.gamma, EOS.dual_energy_eta)
    lo, hi, fb = C.reconstruct(prim, 8, True, False, EOS.gamma)
    assert fb > 0
    fx, fy, fz, am = C.fluxes(lo, hi, 8, EOS.gamma, True, False)
    out.update(fb2_u=u2.copy(), fb2_fallback=np.array(fb), fb2_lo_sha=np.array(sha(lo[core])),
               fb2_hi_sha=np.array(sha(hi[core])), fb2_fx=fx, fb2_fy=fy, fb2_fz=fz, fb2_amax=np.array(am))
    # KT scalar known answer (tests/test_hydro.py:195-207)
    l = PrimitiveState.from_fields(1.0, (0, 0, 0), 1.0, EOS)
    r = PrimitiveState.from_fields(0.125, (0, 0, 0), 0.1, EOS)
    out["sod_flux"] = kt_flux(l, r, 0, EOS)
    save("kernels", **out)


def state_of(tree):
    return np.stack([lf.subgrid.interior for lf in tree.sorted_leaves()])


def random_smooth(tree, seed=0, amp=0.2):
    """tests/test_hydro_step.py:37-49"""
    rng = np.random.default_rng(seed)
    for leaf in tree.leaves():
        sg = leaf.subgrid
        x = sg.cell_centers(0)[:, None, None]
        y = sg.cell_centers(1)[None, :, None]
        z = sg.cell_centers(2)[None, None, :]
        rho = 1.0 + amp * np.sin(np.pi * x) * np.cos(np.pi * y)
        p = 1.0 + amp * np.cos(np.pi * z)
        vx = amp * np.sin(np.pi * y)
        sg.interior[:] = conserved_from_primitive(
            rho, (vx, 0.05 * np.ones_like(rho), -0.02 * np.ones_like(rho)), p, EOS)
    del rng


def step_case(name, tree, steps=1, cfl=0.4, mode=HydroMode("new"), **kw):
    st = HydroStepper(tree, kw.pop("eos", EOS), mode, **kw)
    rec = dict(init=state_of(tree), paths=np.array([json.dumps(lf.path) for lf in tree.sorted_leaves()]))
    dts, amax, fb = [], [], []
    after = {}
    for s in range(steps):
        dt = st.cfl_dt(cfl)
        st.rk3_step(dt)
        dts.append(dt)
        amax.append(st.stats.amax)
        fb.append(st.stats.fallback_count)
        if s == 0:
            after["state1"] = state_of(tree)
    rec.update(after)
    rec.update(dts=np.array(dts), amax=np.array(amax), fallback=np.array(fb),
               final_sha=np.array(sha(state_of(tree))),
               totals=np.array([v for v in conservation_totals(tree).values()]))
    if steps > 1:
        rec["final"] = state_of(tree)
    save(name, **rec)


class FixedGravity:
    """Stub gravity returning one precomputed field set."""

    def __init__(self, fields):
        self.fields = fields

    def solve(self, tree, need_derivative=False):
        return self.fields


def sources_case():
    tree = build_uniform_tree(1, 8, boundary="outflow")
    random_smooth(tree, seed=4)
    # thin region to exercise the floors: scale density down in one leaf
    lf0 = tree.sorted_leaves()[0]
    lf0.subgrid.interior[0] *= 1e-3
    lf0.subgrid.interior[1:4] *= 1e-3
    fields = {}
    for lf in tree.sorted_leaves():
        sg = lf.subgrid
        x = sg.cell_centers(0)[:, None, None]
        y = sg.cell_centers(1)[None, :, None]
        z = sg.cell_centers(2)[None, None, :]
        r2 = x * x + y * y + z * z + 0.1
        f = dict(phi=-1.0 / np.sqrt(r2) + 0 * x, gx=-x / r2 ** 1.5 + 0 * y + 0 * z,
                 gy=-y / r2 ** 1.5 + 0 * x + 0 * z, gz=-z / r2 ** 1.5 + 0 * x + 0 * y,
                 dphi_dt=0.01 * np.cos(3 * x) * np.sin(2 * y) + 0 * z)
        fields[lf.path] = {k: np.ascontiguousarray(np.broadcast_to(v, (8, 8, 8))) for k, v in f.items()}
    grav = {f"g_{i}": np.stack([fields[lf.path][k] for k in ("gx", "gy", "gz", "dphi_dt")])
            for i, lf in enumerate(tree.sorted_leaves())}
    eos = EosConfig(gamma=5.0 / 3.0)
    st = HydroStepper(tree, eos, HydroMode("new"), gravity=FixedGravity(fields), omega=0.4,
                      floors=FloorConfig(rho=2e-3, tau=1e-4, vmax=0.05))
    init = state_of(tree)
    dt = st.cfl_dt(0.4)
    st.rk3_step(dt)
    save("sources", init=init, state1=state_of(tree), dts=np.array([dt]), amax=np.array([st.stats.amax]),
         fallback=np.array([st.stats.fallback_count]), omega=np.array(0.4), gamma=np.array(eos.gamma),
         floors=np.array([2e-3, 1e-4, 0.05]), **grav)


def ghost_cases():
    out = {}
    for bnd in ("periodic", "reflecting", "outflow"):
        tree = build_uniform_tree(1, 8, boundary=bnd)
        random_smooth(tree, seed=6)
        exchange_ghosts(tree)
        out[bnd] = np.stack([lf.subgrid.u for lf in tree.sorted_leaves()])
    tree = build_uniform_tree(1, 8, boundary="reflecting")
    tree.split(tree.leaf_at(1, (0, 0, 0)))
    tree.reindex()
    random_smooth(tree, seed=7)
    exchange_ghosts(tree)
    out["amr"] = np.stack([lf.subgrid.u for lf in tree.sorted_leaves()])
    out["amr_paths"] = np.array([json.dumps(lf.path) for lf in tree.sorted_leaves()])
    save("ghosts", **out)


def amr_sedov_case():
    """Reduced config c4: Sedov on a geometrically refined octree (SURVEY.md §8(d) construction)."""
    from octomini.mesh import refine_by_criterion

    radii = {2: 0.6, 3: 0.35}
    t = build_uniform_tree(2, 8, boundary="reflecting")

    def crit(leaf):
        sg = leaf.subgrid
        lo = sg.origin - 0.5 * sg.dx
        hi = lo + sg.dx * sg.n
        nearest = np.clip(0.0, lo, hi)
        return float(np.sqrt(np.sum(nearest * nearest))) <= radii.get(leaf.level, -1.0)

    refine_by_criterion(t, crit, 4)
    init_sedov(SedovConfig(), t, EOS)
    step_case("amr_sedov_small", t, steps=1)


def checkpoint_case():
    """A reference-written OMCK v1 checkpoint (mesh/checkpoint.py:34-55) of an AMR tree."""
    from octomini.mesh import checkpoint

    t = build_uniform_tree(1, 8, boundary="periodic")
    t.split(t.leaf_at(1, (0, 0, 0)))
    t.reindex()
    random_smooth(t, seed=5)
    checkpoint.write(t, os.path.join(HERE, "amr_reflux_init.omck"), time=0.25, step=7, extra={"gamma": 1.4})
    print("wrote amr_reflux_init.omck")


def fmm_case():
    """Gravity FMM (gravity/solver.py): solve_density on a uniform level-1 tree
    (theta 0.5 and 0.35) and on a corner-refined one, and the full solve with
    dphi/dt from -div(momentum) (test_gravity.py:31-35 random densities)."""
    from octomini.gravity import FmmSolver

    def fill(tree, seed, mom=False):
        rng = np.random.default_rng(seed)
        for leaf in tree.leaves():
            leaf.subgrid.interior[0] = rng.uniform(0.1, 2.0, (tree.n,) * 3)
            if mom:
                for c in (1, 2, 3):
                    leaf.subgrid.interior[c] = rng.uniform(-1.0, 1.0, (tree.n,) * 3)
        return tree

    out = {}
    cases = []
    t = fill(build_uniform_tree(1, 8), 5)
    cases += [("u05", t, 0.5), ("u035", t, 0.35), ("u0", t, 0.0)]
    t2 = build_uniform_tree(1, 8)
    t2.split(t2.leaf_at(1, (0, 0, 0)))
    t2.reindex()
    cases.append(("amr05", fill(t2, 6), 0.5))
    for name, tree, theta in cases:
        solver = FmmSolver(theta)
        phi, g = solver.solve_density(tree)
        leaves = tree.sorted_leaves()
        out[f"{name}_paths"] = np.array([json.dumps(list(lf.path)) for lf in leaves])
        out[f"{name}_rho"] = np.stack([lf.subgrid.interior[0] for lf in leaves])
        out[f"{name}_phi"] = np.stack([phi[lf.path] for lf in leaves])
        out[f"{name}_g"] = np.stack([g[lf.path] for lf in leaves])
        out[f"{name}_theta"] = np.array(theta)
        if theta == 0.0:  # direct traversal: no groups
            continue
        out[f"{name}_stats"] = np.array([solver.stats["groups"], solver.stats["pairs"]])
        grp = solver._groups
        out[f"{name}_R"] = np.array([gr[0] for gr in grp])
        h = hashlib.sha256()
        for gr in grp:
            h.update(np.ascontiguousarray(gr[1], dtype=np.int64).tobytes())
            h.update(np.ascontiguousarray(gr[2], dtype=np.int64).tobytes())
            h.update(bytes([int(gr[3]), int(gr[4])]))
        out[f"{name}_pairs_sha"] = np.array(h.hexdigest())
        out[f"{name}_theta"] = np.array(theta)
    # full solve: phi, g and dphi/dt (ghosts filled by the reference)
    t3 = fill(build_uniform_tree(1, 8, boundary="reflecting"), 7, mom=True)
    exchange_ghosts(t3)
    field = FmmSolver(0.5).solve(t3, need_derivative=True)
    leaves = t3.sorted_leaves()
    out["full_u"] = np.stack([lf.subgrid.u for lf in leaves])
    out["full_paths"] = np.array([json.dumps(list(lf.path)) for lf in leaves])
    for k in ("phi", "gx", "gy", "gz", "dphi_dt"):
        out[f"full_{k}"] = np.stack([field[lf.path][k] for lf in leaves])
    save("fmm", **out)


def gravity_step_case():
    """Self-gravitating hydro: HydroStepper with the FMM re-solved every stage
    (step.py:111-113), rotating frame, reflecting walls, 2 steps."""
    from octomini.gravity import FmmSolver

    tree = build_uniform_tree(1, 8, boundary="reflecting")
    random_smooth(tree, seed=9)
    step_case("gravity_step", tree, steps=2, gravity=FmmSolver(0.5), omega=0.3)


class DensityGravity:
    """State-dependent gravity stub (round-2 contract test): g from the centred
    density difference (reads the ghost cells the stage's fill produced), dphi/dt
    from the momentum, phi = -rho.  The reference calls solve() after the stage's
    ghost fill (hydro/step.py:106-113)."""

    def solve(self, tree, need_derivative=False):
        out = {}
        for lf in tree.leaves():
            u = lf.subgrid.u
            r = u[0]
            gx = -0.05 * (r[4:12, 3:11, 3:11] - r[2:10, 3:11, 3:11])
            gy = -0.05 * (r[3:11, 4:12, 3:11] - r[3:11, 2:10, 3:11])
            gz = -0.05 * (r[3:11, 3:11, 4:12] - r[3:11, 3:11, 2:10])
            dphi = 0.01 * (u[1, 4:12, 3:11, 3:11] - u[1, 2:10, 3:11, 3:11])
            out[lf.path] = dict(phi=-r[3:11, 3:11, 3:11].copy(), gx=gx, gy=gy, gz=gz, dphi_dt=dphi)
        return out


def density_gravity_cases():
    t = build_uniform_tree(1, 8, boundary="reflecting")
    random_smooth(t, seed=13)
    step_case("gravity_density", t, steps=2, gravity=DensityGravity(), omega=0.2)
    t = build_uniform_tree(1, 8, boundary="periodic")
    t.split(t.leaf_at(1, (0, 0, 0)))
    t.reindex()
    random_smooth(t, seed=14)
    step_case("gravity_density_amr", t, steps=1, gravity=DensityGravity())


def contact_tree(seed=12):
    """Level-1 periodic tree with a density jump x4 at x = 0 (pressure and velocity
    continuous: a contact) on the smooth field, so the steepener (_core.pyx:107-142) fires."""
    t = build_uniform_tree(1, 8, boundary="periodic")
    random_smooth(t, seed=seed)
    for lf in t.leaves():
        sg = lf.subgrid
        x = sg.cell_centers(0)[:, None, None] + 0.0 * sg.cell_centers(1)[None, :, None] + \
            0.0 * sg.cell_centers(2)[None, None, :]
        rho = (1.0 + 0.2 * np.sin(np.pi * x)) * np.where(x < 0.0, 4.0, 1.0)
        p = 1.0 + 0.1 * np.cos(np.pi * sg.cell_centers(2))[None, None, :] + 0.0 * x
        sg.interior[:] = conserved_from_primitive(rho, (0.3 + 0.0 * x, 0.1 + 0.0 * x, -0.05 + 0.0 * x), p, EOS)
    return t


def mode_cases():
    """HydroMode branches: contact steepening in a full step, and the
    quadrature_override hook -- new+override == old bitwise over 10 steps at a
    fixed dt (tests/test_hydro_step.py:151-164)."""
    step_case("contact_step", contact_tree(), steps=2, mode=HydroMode("new", contact_detection=True))
    # the same initial data without contact detection must differ (the branch is live)
    t = contact_tree()
    st = HydroStepper(t, EOS, HydroMode("new"))
    st.rk3_step(st.cfl_dt(0.4))
    off = state_of(t)
    g = np.load(os.path.join(HERE, "contact_step.npz"))
    assert not np.array_equal(off, g["state1"]), "contact steepening did not fire"

    def run(mode):
        tree = build_uniform_tree(1, 8, boundary="periodic")
        random_smooth(tree, seed=8)
        init = state_of(tree)
        st = HydroStepper(tree, EOS, mode)
        dt = st.cfl_dt(0.3)
        for _ in range(10):
            st.rk3_step(dt)
        return init, dt, state_of(tree), st.stats

    init, dt, old, _ = run(HydroMode("old"))
    _, dt2, new, stats = run(HydroMode("new", quadrature_override=True))
    assert dt == dt2 and np.array_equal(old, new), "reference: old != new+override"
    save("override_10", init=init, dt=np.array(dt), final=new, final_sha=np.array(sha(new)),
         amax_last=np.array(stats.amax), fallback_last=np.array(stats.fallback_count))


def flux_point_cases():
    """The scalar flux surface (hydro/flux.py): kt_flux on random point pairs for
    every axis, physical_flux, face_flux on random 9-point sets (both modes)."""
    from octomini.hydro.flux import face_flux, physical_flux

    rng = np.random.default_rng(21)
    n = 64
    rho = rng.uniform(0.1, 3.0, (2, n))
    p = rng.uniform(0.1, 3.0, (2, n))
    v = rng.normal(0, 1.5, (2, n, 3))
    v[:, :8] *= 8.0  # some supersonic pairs (one-sided upwinding)
    out = {}
    st = [[PrimitiveState.from_fields(float(rho[k, i]), tuple(float(x) for x in v[k, i]), float(p[k, i]), EOS)
           for i in range(n)] for k in range(2)]
    out["states"] = np.array([[[s.rho, s.vx, s.vy, s.vz, s.p, s.eint, s.tau] for s in st[k]] for k in range(2)])
    for ax in range(3):
        out[f"kt_{ax}"] = np.array([kt_flux(st[0][i], st[1][i], ax, EOS) for i in range(n)])
        out[f"phys_{ax}"] = np.array([physical_flux(st[0][i], ax) for i in range(n)])
    pts = rng.normal(0, 1, (32, 9, 6))
    pts[0] = pts[0, 0]  # all nine equal: returned bit for bit
    out["face_pts"] = pts
    out["face_new"] = np.array([face_flux(q, True) for q in pts])
    out["face_old"] = np.array([face_flux(q, False) for q in pts])
    save("flux_points", **out)


def subgrid_size_cases():
    """16^3 and 32^3 sub-grids (tree.py:13 VALID_N): Sedov at 32^3 cells as 8 leaves of 16^3 and as
    one leaf of 32^3 (reflecting, 2 steps), a smooth periodic 16^3 tree (1 step), and a 16^3 tree
    with density spikes so the positivity fallback fires (per-leaf counts)."""
    t = build_uniform_tree(1, 16, boundary="reflecting")
    init_sedov(SedovConfig(), t, EOS)
    step_case("sedov_n16", t, steps=2)
    t = build_uniform_tree(0, 32, boundary="reflecting")
    init_sedov(SedovConfig(), t, EOS)
    step_case("sedov_n32", t, steps=2)
    t = build_uniform_tree(1, 16, boundary="periodic")
    random_smooth(t, seed=15)
    step_case("smooth_n16", t, steps=1)
    t = build_uniform_tree(1, 16, boundary="periodic")
    random_smooth(t, seed=16)
    for lf in t.leaves():  # zero-pressure cells (egas = tau = 0, at rest): the fallback fires around them
        for c in ((7, 7, 7), (8, 3, 12), (0, 15, 3), (15, 0, 8), (3, 8, 0)):  # incl. cells on leaf / block edges
            lf.subgrid.interior[1:6][(slice(None),) + c] = 0.0
    step_case("fallback_n16", t, steps=1, cfl=0.1)


def main():
    if sys.argv[1:] == ["n16"]:
        subgrid_size_cases()
        return
    if sys.argv[1:] == ["modes"]:
        mode_cases()
        density_gravity_cases()
        flux_point_cases()
        return
    if sys.argv[1:] == ["fmm"]:
        fmm_case()
        gravity_step_case()
        return
    checkpoint_case()
    amr_sedov_case()
    kernel_cases()
    ghost_cases()
    # Sedov benchmark config c1 (32^3 = 64 leaves of 8^3, reflecting), 10 steps
    t = build_uniform_tree(2, 8, boundary="reflecting")
    init_sedov(SedovConfig(), t, EOS)
    step_case("sedov_c1", t, steps=10)
    # smooth periodic / reflecting level-1 trees, 1 step
    t = build_uniform_tree(1, 8, boundary="periodic")
    random_smooth(t, seed=3)
    step_case("smooth_periodic", t)
    t = build_uniform_tree(1, 8, boundary="reflecting")
    random_smooth(t, seed=11)
    step_case("smooth_reflecting", t)
    # old scheme, 2 steps (test_hydro_step.py:151-164 family)
    t = build_uniform_tree(1, 8, boundary="periodic")
    random_smooth(t, seed=8)
    step_case("smooth_old", t, steps=2, cfl=0.3, mode=HydroMode("old"))
    # AMR with reflux: level-1 tree, corner split (test_hydro_step.py:99-113)
    t = build_uniform_tree(1, 8, boundary="periodic")
    t.split(t.leaf_at(1, (0, 0, 0)))
    t.reindex()
    random_smooth(t, seed=5)
    step_case("amr_reflux", t, steps=2)
    sources_case()
    fmm_case()
    gravity_step_case()
    mode_cases()
    density_gravity_cases()
    flux_point_cases()
    subgrid_size_cases()


if __name__ == "__main__":
    main()
