"""Tree -> device batch: leaf order, SoA state layout, neighbour tables, runs.

The B200 layout: the state of record on the device is
``U[6][fstride]`` with leaf ``i`` (in ``tree.sorted_leaves()`` order, the
reference's canonical order, tree.py:148-150) owning the 512 doubles at
``i*512`` of every field, x-major / z-fastest like ``SubGrid.interior``.
Ghost cells are never materialised: the stage kernel gathers halos straight
from neighbour interiors through ``info[i].nbr`` (same-level neighbour per
26-offset, from ``Octree.neighbor_ipos``/``find_leaf_region``,
tree.py:161-195) and ``offmask`` (physical walls).

Leaves are grouped into RUNS: chains of same-level leaves adjacent along +x
that one CTA streams through as a single x-pencil, so the halo planes
between them are computed once.  Runs are capped at ``max_run`` leaves to
keep >= a few waves of CTAs on 148 SMs.
"""

import operator

import numpy as np

from ._abi import AMR_TASK_INTS, BC_CODES, LEAF_INFO_DTYPE
from .geometry import NFIELDS

_SU = operator.attrgetter("subgrid._u")

OFFS = [(i, j, k) for i in (-1, 0, 1) for j in (-1, 0, 1) for k in (-1, 0, 1)]


class UnsupportedTree(NotImplementedError):
    pass


AMR = -2  # neighbor_table code: region covered by a coarser or finer leaf


def neighbor_table(tree, leaves, allow_amr=False):
    """(len(leaves), 27) global indices (into `leaves`) of the same-level
    neighbour at each offset (OFFS order; centre = self), -1 where the
    offset leaves the domain (non-periodic).  Uses Octree.neighbor_ipos /
    find_leaf_region semantics (tree.py:161-195); raises UnsupportedTree for
    coarse/fine neighbours.  Uniform trees take a vectorised lattice path."""
    G = len(leaves)
    levels = {lf.level for lf in leaves}
    index = {lf.path: i for i, lf in enumerate(leaves)}
    out = np.full((G, 27), -1, dtype=np.int64)
    if len(levels) == 1 and len(tree.leaves()) == G and G == 8 ** next(iter(levels)):
        lev = next(iter(levels))
        span = 2 ** lev
        ip = np.array([lf.ipos for lf in leaves], dtype=np.int64)
        lut = np.empty((span, span, span), dtype=np.int64)
        lut[ip[:, 0], ip[:, 1], ip[:, 2]] = np.arange(G)
        for q, o in enumerate(OFFS):
            pos = ip + np.array(o)
            if tree.boundary == "periodic":
                pos %= span
                out[:, q] = lut[pos[:, 0], pos[:, 1], pos[:, 2]]
            else:
                ok = np.all((pos >= 0) & (pos < span), axis=1)
                pc = np.clip(pos, 0, span - 1)
                out[:, q] = np.where(ok, lut[pc[:, 0], pc[:, 1], pc[:, 2]], -1)
        return out
    for i, lf in enumerate(leaves):
        for q, o in enumerate(OFFS):
            if o == (0, 0, 0):
                out[i, q] = i
                continue
            pos = tree.neighbor_ipos(lf, o)
            if pos is None:
                continue
            cover = tree.find_leaf_region(lf.level, pos)
            if cover[0][1] != "same":
                if not allow_amr:
                    raise UnsupportedTree("coarse/fine neighbours need the AMR path (single GPU)")
                out[i, q] = AMR
                continue
            j = index.get(cover[0][0].path)
            if j is None:
                raise UnsupportedTree("neighbour outside the leaf set")
            out[i, q] = j
    return out


MAX_RUN = 4  # leaves per run: the stage kernel's shared-memory LeafInfo slots (omb_stage.cuh Smem::LINFO)


class LeafBatch:
    """Device batch of leaves.  The first ``ncompute`` leaves are advanced by
    the stage kernel; the rest (multi-GPU halo leaves owned by other ranks)
    only provide ghost data.  ``gnbr`` optionally supplies the neighbour
    table in global indices with ``gids`` the global index of each leaf."""

    def __init__(self, tree, max_run=4, leaves=None, ncompute=None, gnbr=None, gids=None, extra_exporters=()):
        if not 1 <= max_run <= MAX_RUN:
            raise ValueError(f"max_run must be in [1, {MAX_RUN}] (the stage kernel stages at most "
                             f"{MAX_RUN} leaf descriptors per run), got {max_run}")
        self.blocks = None
        if tree.n != 8:  # 16^3 / 32^3 leaves run as 8^3 blocks (blocks.py)
            if tree.n not in (16, 32) or leaves is not None or gnbr is not None:
                raise UnsupportedTree(f"{tree.n}^3 sub-grids: uniform single-GPU trees of n = 16 or 32 only")
            from .blocks import BlockTree

            try:
                tree = self.blocks = BlockTree(tree)
            except NotImplementedError as e:
                raise UnsupportedTree(str(e)) from None
        self.tree = tree
        self.n = tree.n
        # padded edge of the host arrays the host transfers read / write (blocks: their leaf's)
        self.host_m = 8 * self.blocks.nb + 6 if self.blocks is not None else 14
        if tree.boundary not in BC_CODES:
            raise ValueError(f"unknown boundary {tree.boundary!r}")
        self.bc = BC_CODES[tree.boundary]
        self.leaves = leaves if leaves is not None else tree.sorted_leaves()
        self.L = len(self.leaves)
        self.ncompute = self.L if ncompute is None else ncompute
        if gnbr is None:
            gnbr = neighbor_table(tree, self.leaves, allow_amr=True)
            gids = np.arange(self.L)
        local = {int(g): i for i, g in enumerate(gids)}
        self.amr = bool(np.any(gnbr == AMR))
        self.info = np.zeros(self.L, dtype=LEAF_INFO_DTYPE)
        self.dx = np.empty(self.L)
        for i, lf in enumerate(self.leaves):
            sg = lf.subgrid
            rec = self.info[i]
            span = 2 ** lf.level
            off = 0
            if tree.boundary != "periodic":
                for a in range(3):
                    if lf.ipos[a] - 1 < 0:
                        off |= 1 << (2 * a)
                    if lf.ipos[a] + 1 >= span:
                        off |= 1 << (2 * a + 1)
            rec["offmask"] = off
            if i < self.ncompute:
                row = gnbr[int(gids[i])]
                rec["nbr"] = [local[int(g)] if g >= 0 else g for g in row]
            else:
                rec["nbr"] = -1
            # cell centres origin + dx * i (blocks: the leaf's origin, offsets in flags)
            rec["ox"], rec["oy"], rec["oz"] = (float(x) for x in getattr(sg, "leaf_origin", sg.origin))
            if self.blocks is not None:
                from .blocks import block_flags

                rec["flags"] |= block_flags(lf.b, self.blocks.nb)
            rec["dx"] = sg.dx
            rec["inv_dx"] = 1.0 / sg.dx
            self.dx[i] = sg.dx
        self.nvirtual = 0
        self.amr_tasks = np.zeros((0, AMR_TASK_INTS), dtype=np.int32)
        self.flux_slots = 0
        self.reflux_off = np.zeros(1, dtype=np.int32)
        self.reflux_leaf = np.zeros(0, dtype=np.int32)
        self.reflux_tasks = np.zeros((0, 6), dtype=np.int32)
        self.solo = np.zeros(self.L, dtype=bool)
        self.slot_of = {}
        if self.amr:
            self._build_amr(extra_exporters)
        self.fstride = (self.L + self.nvirtual) * 512
        self._build_runs(max_run)

    # -- AMR: virtual neighbour leaves, flux export, reflux --------------------
    def _build_amr(self, extra_exporters=()):
        """Coarse/fine neighbour regions become VIRTUAL leaves (indices L..):
        before each stage omb_amr_ghosts fills, in a virtual leaf's interior,
        exactly the cells the stage kernel's gather reads for that region,
        with the reference's prolongation / restriction (mesh/ghosts.py:62-112,
        mesh/transfer.py:13-64).  Leaves on a coarse/fine face export their
        face fluxes; coarse ones defer their update to omb_reflux_update,
        which first applies the reflux substitution (hydro/step.py:206-241)."""
        tree, n, L = self.tree, self.n, self.L
        index = {lf.path: i for i, lf in enumerate(self.leaves)}
        tasks = []
        g = 3
        for i, lf in enumerate(self.leaves[:self.ncompute]):
            nbr = self.info[i]["nbr"]
            for q, o in enumerate(OFFS):
                if nbr[q] != AMR:
                    continue
                pos = tree.neighbor_ipos(lf, o)
                cover = tree.find_leaf_region(lf.level, pos)
                role = cover[0][1]
                t = np.zeros(AMR_TASK_INTS, dtype=np.int32)
                t[1:4] = o
                t[4] = L + len(tasks)
                if role == "coarse":
                    t[0] = 0
                    t[5] = index[cover[0][0].path]
                    for a in range(3):
                        c = o[a]
                        fr = (0, g) if c == 1 else ((n - g, n) if c == -1 else (0, n))
                        octa = int(pos[a]) & 1
                        c0 = octa * (n // 2) + fr[0] // 2
                        c1 = octa * (n // 2) + (fr[1] - 1) // 2 + 1
                        # the reference prolongs the coarse sub-block clipped to [c0-1, c1+1) (ghosts.py:62-85);
                        # its one-sided edge slopes (transfer.py _edge_padded) then fall on the margin
                        # rows, never on the cells the region samples.  That invariant is also what lets a
                        # leaf reading virtual regions join a run: inside a run, A's +x diagonal ghosts come
                        # from B's face region instead of A's own -- the same coarse cells with the same
                        # interior-slope values (c4 tree: runs of 1 and 4 bitwise equal,
                        # tests/test_gpu_bench_parity.py::test_c4_run_lengths_bitwise)
                        m0, m1 = max(c0 - 1, 0), min(c1 + 1, n)
                        t[6 + a], t[9 + a], t[12 + a] = m0, m1, fr[0] + octa * n - 2 * m0
                else:
                    t[0] = 1
                    for k, (child, _) in enumerate(cover):
                        t[5 + k] = index[child.path]
                tasks.append(t)
                nbr[q] = t[4]
            self.info[i]["nbr"] = nbr
            # a leaf whose ghost regions come from virtual leaves still joins a run: the gather
            # reads them through its own LeafInfo (only flux exporters run alone, below)
        self.nvirtual = len(tasks)
        self.amr_tasks = np.array(tasks, dtype=np.int32).reshape(-1, AMR_TASK_INTS)
        # reflux relations across faces (the reference's _reflux loop order)
        faces = [(ax, side) for ax in range(3) for side in (-1, 1)]
        slot = {}
        rtasks = {}

        def get_slot(j):
            if j not in slot:
                slot[j] = len(slot)
            return slot[j]

        for i, lf in enumerate(self.leaves[:self.ncompute]):
            for ax, side in faces:
                off = [0, 0, 0]
                off[ax] = side
                pos = tree.neighbor_ipos(lf, off)
                if pos is None:
                    continue
                cover = tree.find_leaf_region(lf.level, pos)
                if cover[0][1] != "fine":
                    continue
                t1, t2 = [x for x in range(3) if x != ax]
                for child, _ in cover:
                    k = [int(child.ipos[x]) & 1 for x in range(3)]
                    if k[ax] != (0 if side > 0 else 1):
                        continue
                    rtasks.setdefault(i, []).append((ax, side, index[child.path], k[t1], k[t2]))
        for i in sorted(rtasks):
            get_slot(i)
            for (_, _, j, _, _) in rtasks[i]:
                get_slot(j)
        for j in extra_exporters:  # owned fine leaves whose fluxes other ranks' reflux reads
            get_slot(int(j))
        self.flux_slots = len(slot)
        self.slot_of = dict(slot)
        for j, sl in slot.items():
            self.info[j]["flags"] |= 1  # export face fluxes (halo leaves: received instead)
            self.info[j]["slot"] = sl
            self.solo[j] = True
        self.reflux_leaf = np.array(sorted(rtasks), dtype=np.int32)
        off = [0]
        rows = []
        for i in self.reflux_leaf:
            self.info[i]["flags"] |= 2  # update deferred to the reflux kernel
            for (ax, side, j, k1, k2) in rtasks[int(i)]:
                rows.append((ax, side, slot[j], k1, k2, 0))
            off.append(len(rows))
        self.reflux_off = np.array(off, dtype=np.int32)
        self.reflux_tasks = np.array(rows, dtype=np.int32).reshape(-1, 6)

    def _build_runs(self, max_run):
        xp = OFFS.index((1, 0, 0))
        xm = OFFS.index((-1, 0, 0))
        runs = []
        for i, lf in enumerate(self.leaves[:self.ncompute]):
            prev = self.info[i]["nbr"][xm]
            # a run starts where there is no computed same-level -x neighbour inside the domain
            if prev >= 0 and prev < self.ncompute and lf.ipos[0] > 0 and not self.solo[i] and not self.solo[prev]:
                continue
            chain = [i]
            while not self.solo[i]:
                cur = chain[-1]
                nxt = self.info[cur]["nbr"][xp]
                if nxt < 0 or nxt >= self.ncompute or self.solo[nxt] or \
                        self.leaves[cur].ipos[0] + 1 >= 2 ** self.leaves[cur].level:
                    break
                chain.append(int(nxt))
            # balanced split into pieces of <= max_run
            k = -(-len(chain) // max_run)
            base, extra = divmod(len(chain), k)
            s = 0
            for p in range(k):
                w = base + (1 if p < extra else 0)
                runs.append(chain[s:s + w])
                s += w
        assert sum(len(r) for r in runs) == self.ncompute
        self.runs = runs
        self.run_off = np.zeros(len(runs) + 1, dtype=np.int32)
        self.run_off[1:] = np.cumsum([len(r) for r in runs])
        self.run_leaf = np.array([i for r in runs for i in r], dtype=np.int32)
        self.nruns = len(runs)

    def split_tail(self, counts):
        """Shorten the CTAs of the stage kernel's last wave.  The runs are ordered
        longest first (one CTA each, dispatched in order); then, for each k in
        ``counts``, the last k runs of >= 2 leaves are split in halves and moved to
        the end.  The final wave then holds short CTAs, so the SMs run out of work
        closer together.  A k that is not below the run count (a batch of at most one
        wave) is skipped.  Results are bitwise the same for any run layout."""
        runs = list(self.runs)
        for k in counts:
            if k <= 0 or k >= len(runs):
                continue
            runs.sort(key=len, reverse=True)
            head, tail = runs[:-k], runs[-k:]
            short = []
            for r in tail:
                if len(r) >= 2:
                    h = len(r) // 2
                    short += [r[:h], r[h:]]
                else:
                    short.append(r)
            runs = head + sorted(short, key=len, reverse=True)
        assert sorted(i for r in runs for i in r) == list(range(self.ncompute))
        self.runs = runs
        self.run_off = np.zeros(len(runs) + 1, dtype=np.int32)
        self.run_off[1:] = np.cumsum([len(r) for r in runs])
        self.run_leaf = np.array([i for r in runs for i in r], dtype=np.int32)
        self.nruns = len(runs)

    def tail_parts(self, part_runs):
        """Launch parts of a stage whose output is downloaded while it still runs:
        the runs sorted by their last leaf, cut every ``part_runs`` runs.  Returns
        (run_off, run_leaf, cuts, bounds): part k is runs [cuts[k], cuts[k+1]) of
        the sorted table, and once parts 0..k are done every leaf below
        bounds[k+1] is final (no later run writes it)."""
        runs = self.runs
        order = sorted(range(len(runs)), key=lambda r: max(runs[r]))
        cuts = list(range(0, len(order), max(1, part_runs))) + [len(order)]
        srt = [runs[r] for r in order]
        run_off = np.zeros(len(srt) + 1, dtype=np.int32)
        run_off[1:] = np.cumsum([len(r) for r in srt])
        run_leaf = np.array([i for r in srt for i in r], dtype=np.int32)
        # suffix minimum of the runs' first leaves
        first = [min(r) for r in srt] + [self.ncompute]
        suf = list(first)
        for k in range(len(srt) - 1, -1, -1):
            suf[k] = min(suf[k], suf[k + 1])
        bounds = [0] + [suf[c] for c in cuts[1:]]
        return run_off, run_leaf, cuts, bounds

    # -- host <-> packed state --------------------------------------------------
    def _leaf_ptrs(self, count):
        """Data pointers of the first ``count`` leaves' padded host arrays
        (SubGrid.u), or None if one is not a C-contiguous float64 (6, 14, 14, 14)
        array.  Cached: rebuilt only when a leaf's array object changed (the
        cache holds the arrays, so their memory cannot be reused meanwhile)."""
        if self.blocks is not None:
            return self._block_ptrs(count)
        cache = getattr(self, "_ptr_cache", {}).get(count)
        if cache is not None:  # fast identity check (C-level loops; 32768 leaves ~1 ms)
            try:
                if all(map(operator.is_, map(_SU, cache[2]), cache[0])):
                    return cache[1]
            except AttributeError:  # subgrids without the reference's _u slot
                pass
        arrs = [lf.subgrid.u for lf in self.leaves[:count]]
        if any(u is None for u in arrs):  # 16^3 / 32^3 blocks: interior views only
            return None
        ptrs = np.empty(count, dtype=np.uintp)
        for i, u in enumerate(arrs):
            if not (u.flags.c_contiguous and u.dtype == np.float64 and u.shape == (NFIELDS, 14, 14, 14)):
                return None
            ptrs[i] = u.__array_interface__["data"][0]
        if not hasattr(self, "_ptr_cache"):
            self._ptr_cache = {}
        self._ptr_cache[count] = (arrs, ptrs, self.leaves[:count])
        return ptrs

    def _block_ptrs(self, count):
        """The same for 8^3 blocks of 16^3 / 32^3 leaves: each block's corner inside
        its leaf's padded (6, m, m, m) array (m = host_m), so the host transfers copy
        the block's interior straight out of / into the leaf's array.  Cached;
        revalidated by the identity of the leaves' arrays."""
        cache = getattr(self, "_ptr_cache", {}).get(count)
        if cache is not None:
            try:
                if all(map(operator.is_, map(_SU, cache[2]), cache[0])):
                    return cache[1]
            except AttributeError:
                pass
        m = self.host_m
        blocks = self.leaves[:count]
        parents, where = [], {}
        for bk in blocks:
            if id(bk.leaf) not in where:
                where[id(bk.leaf)] = len(parents)
                parents.append(bk.leaf)
        arrs = [lf.subgrid.u for lf in parents]
        base = np.empty(len(parents), dtype=np.uintp)
        for k, u in enumerate(arrs):
            if u is None or not (u.flags.c_contiguous and u.dtype == np.float64 and u.shape == (NFIELDS, m, m, m)):
                return None
            base[k] = u.__array_interface__["data"][0]
        ptrs = np.empty(count, dtype=np.uintp)
        for i, bk in enumerate(blocks):
            bx, by, bz = bk.b
            ptrs[i] = int(base[where[id(bk.leaf)]]) + 8 * ((8 * bx * m + 8 * by) * m + 8 * bz)
        if not hasattr(self, "_ptr_cache"):
            self._ptr_cache = {}
        self._ptr_cache[count] = (arrs, ptrs, parents)
        return ptrs

    def pack(self, out=None, lib=None):
        """Interiors of all batch leaves into ``out`` ([6][L+nvirtual][8][8][8]);
        virtual (AMR ghost) leaves are left as they are."""
        U = out if out is not None else np.zeros((NFIELDS, self.L + self.nvirtual, 8, 8, 8))
        ptrs = self._leaf_ptrs(self.L) if lib is not None else None
        if ptrs is not None and U.flags.c_contiguous:
            lib.omb_host_pack(ptrs.ctypes.data, self.L, 8, self.host_m, self.fstride, U.ctypes.data)
            return U
        for i, lf in enumerate(self.leaves):
            U[:, i] = lf.subgrid.interior
        return U

    def unpack(self, U, lib=None):
        """Write the computed leaves back (halo leaves belong to other ranks)."""
        ptrs = self._leaf_ptrs(self.ncompute) if lib is not None else None
        if ptrs is not None and U.flags.c_contiguous and self.ncompute == self.L:
            lib.omb_host_unpack(U.ctypes.data, self.L, 8, self.host_m, self.fstride, ptrs.ctypes.data)
            return
        for i, lf in enumerate(self.leaves[:self.ncompute]):
            lf.subgrid.interior[:] = U[:, i]

    def pack_gravity(self, fields):
        G = np.zeros((4, self.L + self.nvirtual, 8, 8, 8))
        for i, lf in enumerate(self.leaves):
            if self.blocks is None:
                f, sl = fields[lf.path], (slice(None),) * 3
            else:  # a block of a 16^3 / 32^3 leaf: its part of the leaf's fields
                f = fields[lf.leaf.path]
                sl = tuple(slice(8 * b, 8 * b + 8) for b in lf.b)
            n = self.blocks.nb * 8 if self.blocks is not None else 8
            for k, name in enumerate(("gx", "gy", "gz", "dphi_dt")):
                G[k, i] = np.broadcast_to(f[name], (n, n, n))[sl]
        return G
