"""Device FMM gravity: a drop-in for the reference's ``FmmSolver``
(pkg/src/octomini/gravity/solver.py:50-164), SURVEY.md §8(f) rank 4.

Host, once per tree topology (cached like ``FmmSolver.prepare``):
  * the entity table -- every octree node plus, below each leaf, the complete
    hierarchy of its sub-grid's blocks down to single cells (the numbering and
    centres of gravity/entities.py:15-139, built level by level over all leaves);
  * the dual-tree traversal in C++ (``omb_fmm_traverse``, the reference's
    stack discipline, opening criterion and lattice keys, _core.pyx:372-459);
  * the grouping by key (sorted keys, stable within a group, _core.pyx:476-494)
    and the per-target contribution lists in the reference's global M2L order
    (group by group, pair by pair, the b-side before the a-side,
    _core.pyx:563-608);
  * kernel derivatives for all groups at once, each component with the
    reference's operation order (multipole.py:173-199).
Device, per solve: cell masses -> upward translation per level -> M2L per
target -> downward translation per level -> phi, g per cell (``omb_fmm_*``).
Every floating-point operation keeps the reference's order, so phi and g are
bitwise those of the reference's compiled backend (tests/test_fmm.py).
"""

import os

import numpy as np

from . import _lib
from .device import ptr, stream_handle
from .geometry import GHOST, SX, SY, SZ

NCOMP = 20
S2 = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
S3 = [(0, 0, 0), (0, 0, 1), (0, 0, 2), (0, 1, 1), (0, 1, 2), (0, 2, 2), (1, 1, 1), (1, 1, 2), (1, 2, 2), (2, 2, 2)]


def derivative_table(R):
    """D0..D3 of the FMM kernel g(R) = -1/|R| for every interaction group at
    once (rows of R), evaluated with the reference's operation order per
    component (gravity/multipole.py:173-191) so they are bitwise its values:
    r2 as numpy's ``R @ R`` (a BLAS dot, not the naive sum), then
    D0 = -1/r, D1 = R/r^3, D2_ab = d_ab/r^3 - 3 R_a R_b / r^5,
    D3_abc = 15 R_a R_b R_c / r^7 - 3 (d_ab R_c + d_ac R_b + d_bc R_a) / r^5.
    Returns (G, 2, 20): [:, 0] at R, [:, 1] at -R (odd ranks negated,
    multipole.py:194-199)."""
    R = np.ascontiguousarray(R, dtype=np.float64)
    G = len(R)
    r2 = np.matmul(R[:, None, :], R[:, :, None])[:, 0, 0]
    head = min(G, 4096)  # the stacked product must be the reference's per-row dot; else take that
    if head and not np.array_equal(r2[:head], np.array([float(R[g] @ R[g]) for g in range(head)])):
        r2 = np.array([float(R[g] @ R[g]) for g in range(G)])
    r = np.sqrt(r2)
    r3 = r2 * r
    r5 = r3 * r2
    r7 = r5 * r2
    D = np.empty((G, 2, NCOMP))
    D[:, 0, 0] = -1.0 / r
    D[:, 0, 1:4] = R / r3[:, None]
    X = [R[:, 0], R[:, 1], R[:, 2]]
    for k, (a, b) in enumerate(S2):
        D[:, 0, 4 + k] = (1.0 if a == b else 0.0) / r3 - 3.0 * X[a] * X[b] / r5
    for k, (a, b, c) in enumerate(S3):
        dab, dac, dbc = (float(a == b), float(a == c), float(b == c))
        D[:, 0, 10 + k] = 15.0 * X[a] * X[b] * X[c] / r7 - 3.0 * (dab * X[c] + dac * X[b] + dbc * X[a]) / r5
    D[:, 1] = D[:, 0]
    D[:, 1, 1:4] *= -1.0
    D[:, 1, 10:] *= -1.0
    return D


class EntityTable:
    """The FMM entity table of a tree (the numbering and geometry of
    gravity/entities.py:15-139): ids in depth-first pre-order from the root,
    one per internal octree node; a leaf takes its sub-grid's whole block
    hierarchy, levels j = 0..log2(n) of 8^j blocks each (x-major), the last
    level being its cells.  Arrays: center (3), width, children (8, -1 for
    cells), is_cell, level; ``cell_base[i]`` = id of cell 0 of sorted leaf i.
    Built level by level over all leaves at once (numpy), with the reference's
    arithmetic for every centre: corner = lower + ipos * (width / 2^level),
    centre = corner + (b + 0.5) * w."""

    def __init__(self, tree):
        n = tree.n
        s = int(np.log2(n))
        assert 2 ** s == n
        per_leaf = (8 ** (s + 1) - 1) // 7
        # pre-order numbering (iterative DFS, children in octant order)
        inner, leaf_nodes, leaf_base, ident = [], [], [], {}
        cursor = 0
        stack = [tree.root]
        while stack:
            node = stack.pop()
            ident[id(node)] = cursor
            if node.is_leaf:
                leaf_nodes.append(node)
                leaf_base.append(cursor)
                cursor += per_leaf
            else:
                inner.append(node)
                cursor += 1
                stack.extend(reversed(node.children))
        total = cursor
        center = np.empty((total, 3))
        width = np.empty(total)
        children = np.full((total, 8), -1, dtype=np.int64)
        is_cell = np.zeros(total, dtype=bool)
        level = np.empty(total, dtype=np.int32)
        lower = np.asarray(tree.lower, dtype=np.float64)
        # internal nodes
        if inner:
            ids = np.array([ident[id(nd)] for nd in inner], dtype=np.int64)
            lv = np.array([nd.level for nd in inner])
            w = tree.width / (2 ** lv).astype(np.float64)
            corner = lower + np.array([nd.ipos for nd in inner]) * w[:, None]
            center[ids] = corner + 0.5 * w[:, None]
            width[ids] = w
            level[ids] = lv
            children[ids] = np.array([[ident[id(c)] for c in nd.children] for nd in inner], dtype=np.int64)
        # leaf block hierarchies, one level j at a time for every leaf
        base = np.array(leaf_base, dtype=np.int64)
        lv = np.array([nd.level for nd in leaf_nodes])
        ipos = np.array([nd.ipos for nd in leaf_nodes])
        corner = lower + ipos * (tree.width / (2 ** lv).astype(np.float64))[:, None]
        for j in range(s + 1):
            nb = 2 ** j
            first = base + (8 ** j - 1) // 7  # the leaf's level-j blocks follow levels 0..j-1
            ids = first[:, None] + np.arange(nb ** 3)[None, :]  # x-major: (bx*nb + by)*nb + bz
            w = tree.width / (2 ** (lv + j)).astype(np.float64)
            off = (np.arange(nb) + 0.5)[None, :] * w[:, None]  # (leaf, b)
            bx, by, bz = np.unravel_index(np.arange(nb ** 3), (nb, nb, nb))
            center[ids, 0] = corner[:, 0:1] + off[:, bx]
            center[ids, 1] = corner[:, 1:2] + off[:, by]
            center[ids, 2] = corner[:, 2:3] + off[:, bz]
            width[ids] = w[:, None]
            level[ids] = (lv + j)[:, None]
            if j < s:
                nxt = base + (8 ** (j + 1) - 1) // 7
                n2 = 2 * nb
                for k in range(8):
                    kx, ky, kz = k & 1, (k >> 1) & 1, (k >> 2) & 1
                    cidx = ((2 * bx + kx) * n2 + (2 * by + ky)) * n2 + (2 * bz + kz)
                    children[ids, k] = nxt[:, None] + cidx[None, :]
            else:
                is_cell[ids] = True
        cb = dict(zip((nd.path for nd in leaf_nodes), base + (8 ** s - 1) // 7))
        self.root = ident[id(tree.root)]
        self.center, self.width, self.children, self.is_cell, self.level = center, width, children, is_cell, level
        self.n = n
        self.nentities = total
        self.leaf_paths = [lf.path for lf in tree.sorted_leaves()]
        self.cell_base = np.array([cb[p] for p in self.leaf_paths], dtype=np.int64)


def _check_balance(tree):
    """The 2:1 check FmmSolver.prepare runs first (mesh/tree.py:180-183 via
    find_leaf_region, which raises StructureError on a violation)."""
    offs = [(i, j, k) for i in (-1, 0, 1) for j in (-1, 0, 1) for k in (-1, 0, 1) if (i, j, k) != (0, 0, 0)]
    for lf in tree.leaves():
        for off in offs:
            pos = tree.neighbor_ipos(lf, off)
            if pos is not None:
                tree.find_leaf_region(lf.level, pos)


def traverse(lib, table, theta):
    """Interaction pairs (a, b, key) in the reference's discovery order."""
    t = table
    center = np.ascontiguousarray(t.center)
    width = np.ascontiguousarray(t.width)
    children = np.ascontiguousarray(t.children)
    is_cell = np.ascontiguousarray(t.is_cell.astype(np.uint8))
    cap = max(1 << 16, 160 * t.nentities)
    while True:
        pa = np.empty(cap, dtype=np.int64)
        pb = np.empty(cap, dtype=np.int64)
        pk = np.empty(cap, dtype=np.int64)
        n = lib.omb_fmm_traverse(center.ctypes.data, width.ctypes.data, children.ctypes.data, is_cell.ctypes.data,
                                 t.nentities, t.root, float(theta), pa.ctypes.data, pb.ctypes.data, pk.ctypes.data,
                                 cap)
        if n >= 0:
            return pa[:n], pb[:n], pk[:n]
        cap = -n


def group_pairs(table, pa, pb, pk):
    """Groups in sorted-key order, pairs stable within a group (_core.pyx:476-494):
    returns (order, bounds, R per group, a_cell, b_cell per group)."""
    keys, first_idx, inverse = np.unique(pk, return_index=True, return_inverse=True)
    order = np.argsort(inverse, kind="stable")
    bounds = np.searchsorted(inverse[order], np.arange(len(keys) + 1))
    f = keys & 3
    R = table.center[pb[first_idx]] - table.center[pa[first_idx]]
    return order, bounds, R, (f & 2) != 0, (f & 1) != 0


class B200FmmSolver:
    """Order-3 FMM on the device; same API as the reference's ``FmmSolver``
    (``prepare``, ``solve_density``, ``solve``, ``stats``).  theta in [0, 1]; theta = 0 is the
    reference's always-reject direct summation (direct_traversal_eval, _core.pyx:611-690)."""

    def __init__(self, theta, device=None):
        if theta < 0.0 or theta > 1.0:
            raise ValueError("theta must lie in [0, 1]")
        import torch

        self.theta = float(theta)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.lib = _lib.load()
        self._signature = None
        self.stats = {}

    def _topology_signature(self, tree):
        return (tree.n, tree.width, tuple(leaf.path for leaf in tree.sorted_leaves()))

    def prepare(self, tree):
        sig = self._topology_signature(tree)
        if sig == self._signature:
            return
        import torch

        self._order_cache = {}
        _check_balance(tree)
        t = EntityTable(tree)
        self.table = t
        pa, pb, pk = traverse(self.lib, t, self.theta)
        if self.theta == 0.0:
            self._prepare_direct(tree, t, pa, pb)
            self._signature = sig
            return
        # groups (sorted keys) and per-target contribution lists in the global M2L order (C++, O(pairs))
        gcap = 1 << 22
        gfirst = np.empty(gcap, dtype=np.int64)
        gflags = np.empty(gcap, dtype=np.uint8)
        off = np.empty(t.nentities + 1, dtype=np.int64)
        contrib = np.empty(2 * len(pa), dtype=np.uint64)
        G = int(self.lib.omb_fmm_build(pa.ctypes.data, pb.ctypes.data, pk.ctypes.data, len(pa), t.nentities,
                                       gfirst.ctypes.data, gflags.ctypes.data, gcap, off.ctypes.data,
                                       contrib.ctypes.data))
        if G < 0:
            raise RuntimeError("FMM: too many interaction groups")
        R = t.center[pb[gfirst[:G]]] - t.center[pa[gfirst[:G]]]
        a_cell, b_cell = (gflags[:G] & 2) != 0, (gflags[:G] & 1) != 0
        self.stats["groups"] = G
        self.stats["pairs"] = int(len(pa))
        D = derivative_table(R)
        cnt = np.diff(off)
        targets = np.nonzero(cnt)[0].astype(np.int64)
        off = np.append(off[targets], off[-1]).astype(np.int64)  # CSR over the targets with contributions
        del pa, pb, pk
        dev = self.dev
        T = torch
        self._center = T.from_numpy(np.ascontiguousarray(t.center).reshape(-1)).to(dev)
        self._children = T.from_numpy(np.ascontiguousarray(t.children).reshape(-1)).to(dev)
        self._D = T.from_numpy(D.reshape(-1)).to(dev)
        self._cellcell = T.from_numpy((a_cell & b_cell).astype(np.uint8)).to(dev)
        self._off = T.from_numpy(off).to(dev)
        self._contrib = T.from_numpy(contrib.view(np.int64)).to(dev)
        del contrib
        # the L4..L19 pass needs no cell-cell contribution (90 % of them at theta 0.5): its
        # lists are the subsequence of the others, same order, CSR over the same targets
        g = (self._contrib >> 40) & 0x3FFFFF  # (bits 40..61; bit 62 flags the cell-cell words)
        keep = self._cellcell[g] == 0
        del g
        cs = T.cumsum(keep, 0)
        self._off1 = T.cat([T.zeros(1, dtype=T.int64, device=dev), cs])[self._off]
        del cs
        self._contrib1 = self._contrib[keep]
        del keep
        # M2L work per solve (bench roofline): cell-cell monopole contributions vs full order-3 ones
        self.stats["contrib_general"] = int(self._contrib1.numel())
        self.stats["contrib_cellcell"] = int(self._contrib.numel()) - self.stats["contrib_general"]
        self._targets = T.from_numpy(targets.astype(np.int64)).to(dev)
        self._cell_base = T.from_numpy(t.cell_base).to(dev)
        lv = t.level
        parents = {int(L): np.nonzero((lv == L) & ~t.is_cell)[0].astype(np.int64) for L in np.unique(lv)}
        self._up = [(L, T.from_numpy(parents[L]).to(dev)) for L in sorted(parents, reverse=True) if len(parents[L])]
        self._down = [(L, T.from_numpy(parents[L]).to(dev)) for L in sorted(parents) if len(parents[L])]
        self._dx3_dev = T.tensor([lf.subgrid.dx ** 3 for lf in tree.sorted_leaves()], dtype=T.float64, device=dev)
        self._M = T.zeros(t.nentities * NCOMP, dtype=T.float64, device=dev)
        self._M0c = T.zeros(t.nentities, dtype=T.float64, device=dev)  # compact monopoles (M2L pass 0)
        self._L = T.zeros_like(self._M)
        self._signature = sig

    def _prepare_direct(self, tree, t, pa, pb):
        """theta = 0: per-target cell-cell lists in the traversal's order."""
        import torch

        off = np.empty(t.nentities + 1, dtype=np.int64)
        contrib = np.empty(2 * len(pa), dtype=np.uint64)
        _lib.check(self.lib.omb_fmm_build_direct(pa.ctypes.data, pb.ctypes.data, len(pa), t.nentities,
                                                 off.ctypes.data, contrib.ctypes.data), "omb_fmm_build_direct")
        self.stats = {}  # the reference's direct path records no groups/pairs
        dev = self.dev
        self._center = torch.from_numpy(np.ascontiguousarray(t.center).reshape(-1)).to(dev)
        self._off = torch.from_numpy(off).to(dev)
        self._contrib = torch.from_numpy(contrib.view(np.int64)).to(dev)
        self._cell_base = torch.from_numpy(t.cell_base).to(dev)
        self._dx3_dev = torch.tensor([lf.subgrid.dx ** 3 for lf in tree.sorted_leaves()], dtype=torch.float64,
                                     device=dev)
        self._M = torch.zeros(t.nentities * NCOMP, dtype=torch.float64, device=dev)
        self._L = None
        self._up, self._down = [], []

    def _solve_into(self, rho_dev, dx3_dev, phi, gx, gy, gz, stream=None):
        """One solve of the density rho_dev ([L][512]) into phi, gx, gy, gz of the cells."""
        nleaf = len(self.table.leaf_paths)
        if self.theta == 0.0:
            lib, sh = self.lib, stream_handle(stream)
            self._M.zero_()
            _lib.check(lib.omb_fmm_masses(ptr(rho_dev), ptr(self._cell_base), nleaf, ptr(dx3_dev), ptr(self._M), sh),
                       "omb_fmm_masses")
            _lib.check(lib.omb_fmm_direct(ptr(self._off), ptr(self._contrib), ptr(self._center), ptr(self._M),
                                          ptr(self._cell_base), nleaf, ptr(phi), ptr(gx), ptr(gy), ptr(gz), sh),
                       "omb_fmm_direct")
            return
        self._run(rho_dev, dx3_dev, stream)
        _lib.check(self.lib.omb_fmm_fields(ptr(self._L), ptr(self._cell_base), nleaf, ptr(phi), ptr(gx), ptr(gy),
                                           ptr(gz), stream_handle(stream)), "omb_fmm_fields")

    # -- device passes ---------------------------------------------------------
    def _run(self, rho_dev, dx3_dev, stream=None):
        """rho_dev: [L][512] densities of sorted_leaves(); returns L (entities x 20)."""
        lib, sh = self.lib, stream_handle(stream)
        nleaf = len(self.table.leaf_paths)
        self._M.zero_()
        self._L.zero_()
        _lib.check(lib.omb_fmm_masses(ptr(rho_dev), ptr(self._cell_base), nleaf, ptr(dx3_dev), ptr(self._M), sh),
                   "omb_fmm_masses")
        for _, par in self._up:
            _lib.check(lib.omb_fmm_upward(ptr(par), int(par.numel()), ptr(self._children), ptr(self._center),
                                          ptr(self._M), sh), "omb_fmm_upward")
        sub = getattr(self, "_subset", None)  # partitioned: this rank's targets only
        nt = int(sub.numel()) if sub is not None else int(self._targets.numel())
        for part, off, contrib, cc in ((0, self._off, self._contrib, ptr(self._cellcell)),
                                       (1, self._off1, self._contrib1, None)):
            order = self._target_order(part, off, sub)
            _lib.check(lib.omb_fmm_m2l_part(part, ptr(off), ptr(contrib), ptr(self._D), cc, ptr(self._M),
                                            ptr(self._L), nt, ptr(self._targets), ptr(order), ptr(self._M0c),
                                            self.table.nentities, sh), "omb_fmm_m2l_part")
        for _, par in self._down:
            _lib.check(lib.omb_fmm_downward(ptr(par), int(par.numel()), ptr(self._children), ptr(self._center),
                                            ptr(self._L), sh), "omb_fmm_downward")
        return self._L

    def _target_order(self, part, off, sub):
        """The M2L threads take their targets longest contribution list first (cached per pass):
        a warp's 32 targets then have lists of about one length, instead of waiting for the longest
        of a mixed set.  Each target's own additions keep their order (bitwise the same).
        OMB_FMM_ORDER=0 keeps the entity order."""
        import os

        import torch

        if os.environ.get("OMB_FMM_ORDER", "1") == "0":
            return sub
        cache = self.__dict__.setdefault("_order_cache", {})
        key = (part, id(sub))
        if key not in cache:
            n = torch.diff(off)
            idx = sub if sub is not None else torch.arange(n.numel(), device=n.device)
            cache[key] = idx[torch.argsort(n[idx], descending=True, stable=True)].contiguous()
        return cache[key]

    def fields_device(self, rho_dev, dx3_dev, out4, stream=None):
        """phi, gx, gy, gz per cell into out4 ([4][L][512] device tensor)."""
        nleaf = len(self.table.leaf_paths)
        n = nleaf * 512
        o = out4.reshape(4, -1)
        self._solve_into(rho_dev, dx3_dev, o[0], o[1], o[2], o[3], stream)
        return o[:, :n]

    def launches_per_stage(self):
        """Kernels of one stage_fields call: 2 solves x (masses, upward levels, the
        monopole copy and the two M2L passes, downward levels, fields) + the
        -div(momentum) source."""
        per = 2 if self.theta == 0.0 else 5 + len(self._up) + len(self._down)
        paired = self.theta != 0.0 and os.environ.get("OMB_FMM_PAIR", "1") != "0"
        return 2 * per + 1 - (1 if paired else 0)  # (paired: one pass-0 launch for both solves)

    def stage_fields(self, U, fstride, info, bc, nleaf, grav, stream=None):
        """The stepper's per-stage solve (solver.py:134-153 on device data):
        gx, gy, gz of the density and dphi/dt (the potential of -div(momentum))
        of the [6][fstride] state U into grav ([4][fstride]: gx gy gz dphi_dt)."""
        import torch

        if not hasattr(self, "_dx3_dev") or self._dx3_dev.numel() != nleaf:
            raise RuntimeError("stage_fields before prepare() of the stepper's tree")
        lib, sh = self.lib, stream_handle(stream)
        n = nleaf * 512
        if getattr(self, "_scratch", None) is None or self._scratch.numel() < 2 * n:
            self._scratch = torch.empty(2 * n, dtype=torch.float64, device=self.dev)
        phi, rhodot = self._scratch[:n], self._scratch[n:2 * n]
        G = grav.reshape(4, -1)
        if self.theta != 0.0 and os.environ.get("OMB_FMM_PAIR", "1") != "0":
            # both solves at once (one pass over the interaction lists for the two mass sets)
            _lib.check(lib.omb_fmm_rhodot(ptr(U), fstride, ptr(info), bc, nleaf, None, 0, ptr(rhodot), sh),
                       "omb_fmm_rhodot")
            self._run_pair(U[:n], rhodot, self._dx3_dev, stream)
            _lib.check(lib.omb_fmm_fields(ptr(self._L), ptr(self._cell_base), nleaf, ptr(phi), ptr(G[0]),
                                          ptr(G[1]), ptr(G[2]), sh), "omb_fmm_fields")
            _lib.check(lib.omb_fmm_fields(ptr(self._L2), ptr(self._cell_base), nleaf, ptr(G[3]), ptr(phi),
                                          ptr(phi), ptr(phi), sh), "omb_fmm_fields")
            return
        self._solve_into(U[:n], self._dx3_dev, phi, G[0], G[1], G[2], stream)
        _lib.check(lib.omb_fmm_rhodot(ptr(U), fstride, ptr(info), bc, nleaf, None, 0, ptr(rhodot), sh),
                   "omb_fmm_rhodot")
        self._solve_into(rhodot, self._dx3_dev, G[3], phi, phi, phi, stream)

    def _run_pair(self, rho_a, rho_b, dx3_dev, stream=None):
        """Two solves (masses rho_a, rho_b) sharing the pass over the interaction lists:
        L of a in self._L, of b in self._L2.  Each solve bitwise as _run alone."""
        import torch

        lib, sh = self.lib, stream_handle(stream)
        nleaf = len(self.table.leaf_paths)
        if getattr(self, "_M2", None) is None:
            self._M2 = torch.zeros_like(self._M)
            self._L2 = torch.zeros_like(self._L)
            self._M0c2 = torch.zeros(2 * self._M0c.numel(), dtype=torch.float64, device=self.dev)  # (a, b) pairs
        for M, L in ((self._M, self._L), (self._M2, self._L2)):
            M.zero_()
            L.zero_()
        for rho, M in ((rho_a, self._M), (rho_b, self._M2)):
            _lib.check(lib.omb_fmm_masses(ptr(rho), ptr(self._cell_base), nleaf, ptr(dx3_dev), ptr(M), sh),
                       "omb_fmm_masses")
            for _, par in self._up:
                _lib.check(lib.omb_fmm_upward(ptr(par), int(par.numel()), ptr(self._children), ptr(self._center),
                                              ptr(M), sh), "omb_fmm_upward")
        sub = getattr(self, "_subset", None)
        nt = int(sub.numel()) if sub is not None else int(self._targets.numel())
        order = self._target_order(0, self._off, sub)
        _lib.check(lib.omb_fmm_m2l0_pair(ptr(self._off), ptr(self._contrib), ptr(self._D), ptr(self._cellcell),
                                         ptr(self._M), ptr(self._M2), ptr(self._L), ptr(self._L2), nt,
                                         ptr(self._targets), ptr(order), ptr(self._M0c2), None,
                                         self.table.nentities, sh), "omb_fmm_m2l0_pair")
        order = self._target_order(1, self._off1, sub)
        for M, L in ((self._M, self._L), (self._M2, self._L2)):
            _lib.check(lib.omb_fmm_m2l_part(1, ptr(self._off1), ptr(self._contrib1), ptr(self._D), None, ptr(M),
                                            ptr(L), nt, ptr(self._targets), ptr(order), None, self.table.nentities,
                                            sh), "omb_fmm_m2l_part")
        for L in (self._L, self._L2):
            for _, par in self._down:
                _lib.check(lib.omb_fmm_downward(ptr(par), int(par.numel()), ptr(self._children), ptr(self._center),
                                                ptr(L), sh), "omb_fmm_downward")

    # -- leaf-partitioned runs (one rank per GPU) -------------------------------
    def set_partition(self, part):
        """This rank solves M2L only for its own leaves' entities (blocks and
        cells) and the octree's internal nodes -- everything the downward pass
        to its cells reads; the masses come from all ranks (all_gather).
        Bitwise the single-GPU result for this rank's cells."""
        import torch

        self._order_cache = {}
        if self.theta == 0.0:
            raise NotImplementedError("theta = 0 with a partition")
        t = self.table
        b0, b1 = part.bounds[part.rank], part.bounds[part.rank + 1]
        # a leaf's entities (its block hierarchy, then its cells) are contiguous, ending at cell_base + n^3;
        # the octree's internal nodes belong to no leaf and every rank's downward pass needs them
        n3 = t.n ** 3
        per_leaf = (8 * n3 - 1) // 7
        in_leaf = np.zeros(t.nentities, dtype=bool)
        mine = np.zeros(t.nentities, dtype=bool)
        for i, cb in enumerate(t.cell_base):
            lo = cb + n3 - per_leaf
            in_leaf[lo:cb + n3] = True
            if b0 <= i < b1:
                mine[lo:cb + n3] = True
        tg = self._targets.cpu().numpy()
        keep = mine[tg] | ~in_leaf[tg]
        self._subset = torch.from_numpy(np.nonzero(keep)[0].astype(np.int64)).to(self.dev)
        self._part = part
        self._my_cell_base = torch.from_numpy(t.cell_base[b0:b1].copy()).to(self.dev)

    def stage_fields_partitioned(self, U, fstride, info, bc, grav, halo, dist, group, stream=None):
        """stage_fields for a rank of a leaf partition: rho and rho_dot of the owned
        leaves are all-gathered, the solves run on this rank's targets, and gx, gy,
        gz, dphi/dt of the owned leaves land in grav."""
        import torch

        p = self._part
        lib, sh = self.lib, stream_handle(stream)
        nown = p.nown
        G = len(self.table.leaf_paths)
        width = max(p.bounds[r + 1] - p.bounds[r] for r in range(p.world)) * 512
        if getattr(self, "_gather", None) is None:
            self._gather = torch.zeros(p.world * width * 2, dtype=torch.float64, device=self.dev)
            self._rho_all = torch.zeros(2 * G * 512, dtype=torch.float64, device=self.dev)
            self._sendb = torch.zeros(2 * width, dtype=torch.float64, device=self.dev)
            self._scr = torch.empty(nown * 512, dtype=torch.float64, device=self.dev)
        send = self._sendb
        send[:nown * 512].copy_(U[:nown * 512])  # owned densities
        _lib.check(lib.omb_fmm_rhodot(ptr(U), fstride, ptr(info), bc, nown, ptr(halo) if halo is not None else None,
                                      nown, ptr(send[width:]), sh), "omb_fmm_rhodot")
        dist.all_gather_into_tensor(self._gather, send, group=group)
        ga = self._gather.view(p.world, 2, width)
        for r in range(p.world):  # global leaf order: rank r owns [bounds[r], bounds[r+1])
            a, b = p.bounds[r] * 512, p.bounds[r + 1] * 512
            self._rho_all[a:b].copy_(ga[r, 0, :b - a])
            self._rho_all[G * 512 + a:G * 512 + b].copy_(ga[r, 1, :b - a])
        Gv = grav.reshape(4, -1)
        if os.environ.get("OMB_FMM_PAIR", "1") != "0":  # both solves in one pass over the lists
            self._run_pair(self._rho_all[:G * 512], self._rho_all[G * 512:], self._dx3_dev, stream)
            for L, outs in ((self._L, (self._scr, Gv[0], Gv[1], Gv[2])), (self._L2, (Gv[3], self._scr, self._scr,
                                                                                   self._scr))):
                _lib.check(lib.omb_fmm_fields(ptr(L), ptr(self._my_cell_base), nown, *[ptr(o) for o in outs], sh),
                           "omb_fmm_fields")
            return
        for k, (rho, outs) in enumerate(((self._rho_all[:G * 512], (self._scr, Gv[0], Gv[1], Gv[2])),
                                         (self._rho_all[G * 512:], (Gv[3], self._scr, self._scr, self._scr)))):
            self._run(rho, self._dx3_dev, stream)
            _lib.check(lib.omb_fmm_fields(ptr(self._L), ptr(self._my_cell_base), nown, *[ptr(o) for o in outs], sh),
                       "omb_fmm_fields")

    # -- the reference's host API ----------------------------------------------
    def solve_density(self, tree, per_leaf_density=None):
        """(phi, g) keyed by leaf path, from the current density (or a
        replacement per-leaf source), as solver.py:117-132."""
        import torch

        self.prepare(tree)
        leaves = tree.sorted_leaves()
        n = tree.n
        rho = np.empty((len(leaves), n ** 3))
        for i, lf in enumerate(leaves):
            src = lf.subgrid.interior[0] if per_leaf_density is None else per_leaf_density[lf.path]
            rho[i] = np.asarray(src, dtype=np.float64).reshape(-1)
        out = torch.empty(4 * len(leaves) * 512, dtype=torch.float64, device=self.dev)
        f = self.fields_device(torch.from_numpy(rho.reshape(-1)).to(self.dev), self._dx3_dev, out).cpu().numpy()
        f = f.reshape(4, len(leaves), n, n, n)
        out_phi, out_g = {}, {}
        for i, lf in enumerate(leaves):
            out_phi[lf.path] = f[0, i].copy()
            out_g[lf.path] = f[1:4, i].copy()
        return out_phi, out_g

    def solve(self, tree, need_derivative=True):
        """phi and g from rho, and dphi/dt from rho_dot = -div(momentum)
        (solver.py:134-153; the ghosts of the host sub-grids must be filled,
        as in the reference)."""
        self.prepare(tree)
        phi, g = self.solve_density(tree)
        dphi = None
        if need_derivative:
            rho_dot = {lf.path: momentum_divergence_source(lf.subgrid) for lf in tree.sorted_leaves()}
            dphi, _ = self.solve_density(tree, per_leaf_density=rho_dot)
        field = GravityField()
        for path in phi:
            gx, gy, gz = g[path]
            field.add_leaf(path, phi[path], gx, gy, gz, dphi[path] if dphi is not None else None)
        return field


class GravityField:
    """Per-leaf potential, acceleration and potential time derivative
    (gravity/solver.py:33-47); what a gravity solver's ``solve`` returns."""

    def __init__(self):
        self.per_leaf = {}

    def __getitem__(self, path):
        return self.per_leaf[path]

    def add_leaf(self, path, phi, gx, gy, gz, dphi_dt=None):
        self.per_leaf[path] = {"phi": phi, "gx": gx, "gy": gy, "gz": gz,
                               "dphi_dt": dphi_dt if dphi_dt is not None else np.zeros_like(phi)}


def momentum_divergence_source(subgrid):
    """rho_dot = -div(s) by second-order central differences over the filled
    ghosts (gravity/solver.py:156-168), same numpy expression."""
    g = GHOST
    n = subgrid.n
    u = subgrid.u
    inv2dx = 1.0 / (2.0 * subgrid.dx)
    sl = slice(g, g + n)
    return -(
        (u[SX, g + 1: g + n + 1, sl, sl] - u[SX, g - 1: g + n - 1, sl, sl])
        + (u[SY, sl, g + 1: g + n + 1, sl] - u[SY, sl, g - 1: g + n - 1, sl])
        + (u[SZ, sl, sl, g + 1: g + n + 1] - u[SZ, sl, sl, g - 1: g + n - 1])
    ) * inv2dx
