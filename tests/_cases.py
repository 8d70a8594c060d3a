"""Shared test inputs: golden loading and tree builders (host mirror)."""

import json
import os

import numpy as np

import octomini_host as mesh
import octomini_host as problems
from paper_2107_10987_b200 import hydro

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EOS = hydro.EosConfig(gamma=1.4)


def golden(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def random_smooth(tree, seed=0, amp=0.2, eos=EOS):
    """Same field as the reference's tests/test_hydro_step.py:37-49."""
    for leaf in tree.leaves():
        sg = leaf.subgrid
        x = sg.cell_centers(0)[:, None, None]
        y = sg.cell_centers(1)[None, :, None]
        z = sg.cell_centers(2)[None, None, :]
        rho = 1.0 + amp * np.sin(np.pi * x) * np.cos(np.pi * y)
        p = 1.0 + amp * np.cos(np.pi * z)
        vx = amp * np.sin(np.pi * y)
        sg.interior[:] = mesh.conserved_from_primitive(
            rho, (vx, 0.05 * np.ones_like(rho), -0.02 * np.ones_like(rho)), p, eos)


def state_of(tree):
    return np.stack([lf.subgrid.interior for lf in tree.sorted_leaves()])


def set_state(tree, arr):
    for lf, a in zip(tree.sorted_leaves(), arr):
        lf.subgrid.interior[:] = a


def case_tree(name):
    """Rebuild the tree of a golden step case, with the golden initial state."""
    if name == "sedov_c1":
        t = mesh.build_uniform_tree(2, 8, boundary="reflecting")
        problems.init_sedov(problems.SedovConfig(), t, EOS)
    elif name == "smooth_periodic":
        t = mesh.build_uniform_tree(1, 8, boundary="periodic")
    elif name == "smooth_reflecting":
        t = mesh.build_uniform_tree(1, 8, boundary="reflecting")
    elif name == "smooth_old":
        t = mesh.build_uniform_tree(1, 8, boundary="periodic")
    elif name == "amr_reflux":
        t = mesh.build_uniform_tree(1, 8, boundary="periodic")
        t.split(t.leaf_at(1, (0, 0, 0)))
        t.reindex()
    elif name == "amr_sedov_small":
        t = problems.amr_sedov_tree(base_level=2, max_level=4, radii={2: 0.6, 3: 0.35}, eos=EOS)
    elif name == "gravity_step":
        t = mesh.build_uniform_tree(1, 8, boundary="reflecting")
    elif name == "sources":
        t = mesh.build_uniform_tree(1, 8, boundary="outflow")
    elif name in ("contact_step", "override_10", "gravity_density_amr"):
        t = mesh.build_uniform_tree(1, 8, boundary="periodic")
        if name == "gravity_density_amr":
            t.split(t.leaf_at(1, (0, 0, 0)))
            t.reindex()
    elif name == "gravity_density":
        t = mesh.build_uniform_tree(1, 8, boundary="reflecting")
    elif name == "sedov_n16":
        t = mesh.build_uniform_tree(1, 16, boundary="reflecting")
    elif name == "sedov_n32":
        t = mesh.build_uniform_tree(0, 32, boundary="reflecting")
    elif name in ("smooth_n16", "fallback_n16"):
        t = mesh.build_uniform_tree(1, 16, boundary="periodic")
    else:
        raise KeyError(name)
    g = golden(name)
    if "paths" in g:
        assert [json.loads(p) for p in g["paths"]] == [list(lf.path) for lf in t.sorted_leaves()]
    set_state(t, g["init"])
    return t, g


class FixedGravity:
    state_independent = True

    def __init__(self, fields):
        self.fields = fields

    def solve(self, tree, need_derivative=False):
        return self.fields


def sources_gravity(tree, g):
    fields = {}
    for i, lf in enumerate(tree.sorted_leaves()):
        a = g[f"g_{i}"]
        fields[lf.path] = dict(gx=a[0], gy=a[1], gz=a[2], dphi_dt=a[3], phi=np.zeros_like(a[0]))
    return FixedGravity(fields)


def bitwise_mismatch(a, b):
    """Number of entries that differ (NaN==NaN counts as equal; +-0 equal)."""
    a = np.asarray(a)
    b = np.asarray(b)
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    return int(np.size(same) - np.count_nonzero(same))


def rel_close(x, ref, rtol=1e-12):
    """Per-cell |x-ref| <= rtol*max(|ref|, field scale) (SURVEY.md §7 comparator)."""
    x = np.asarray(x)
    ref = np.asarray(ref)
    bad = 0
    for f in range(ref.shape[1]):
        xs, rs = x[:, f], ref[:, f]
        scale = max(float(np.max(np.abs(rs))), 1e-300)
        bad += int(np.count_nonzero(np.abs(xs - rs) > rtol * np.maximum(np.abs(rs), scale)))
    return bad


class DensityGravity:
    """The state-dependent gravity stub of tests/golden/make_golden.py (same
    expressions): g from centred density differences -- reads the ghost cells of
    the stage state -- dphi/dt from the momentum, phi = -rho."""

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
