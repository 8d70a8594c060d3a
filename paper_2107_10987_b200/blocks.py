"""16^3 and 32^3 sub-grids on the 8^3 stage kernel (octomini accepts n in
(8, 16, 32), ``pkg/src/octomini/mesh/tree.py:13``; the paper compares the three
sub-grid sizes).

A uniform tree of n^3 leaves at level L covers exactly the cells of a uniform
tree of 8^3 leaves at level L + log2(n/8), and the reference's step computes
every cell from its 3-wide stencil alone -- same-level ghost cells are copies
of the neighbour's interior -- so each n^3 leaf is run as (n/8)^3 BLOCKS of
8^3: ``BlockTree`` is a view of the caller's tree whose leaves are those
blocks, each block's ``subgrid.interior`` a numpy view into its leaf's
current interior (writes land in the caller's arrays).  What depends on the leaf size
is restored per block through its LeafInfo flags (``blocks.block_flags``):

* the positivity-fallback count: the reference counts every position of
  [2, n+4)^3 of each LEAF (_core.pyx:143-155); a block counts the part of that
  range it owns -- one cell beyond the leaf on its outer faces, none on faces
  shared with sibling blocks -- so every position is counted once per leaf;
* cell centres (rotating-frame sources): origin + dx * (8 b + i) from the
  leaf's origin, as SubGrid.cell_centers forms them, not from a block origin.

Adaptive trees with n > 8 are not supported (their coarse/fine ghost regions
are cut at n^3 leaf boundaries); ``LeafBatch`` raises UnsupportedTree.
"""

import numpy as np


def block_flags(b, nb):
    """LeafInfo.flags bits of block index b (per axis, 0..nb-1) of a leaf split in nb^3:
    bits 2+2a / 3+2a: the fallback count starts at 3 / ends at 10 on axis a (not 2 / 11);
    bits 8+5a: the block's cell offset 8*b_a inside its leaf."""
    f = 0
    for a in range(3):
        if b[a] > 0:
            f |= 1 << (2 + 2 * a)
        if b[a] < nb - 1:
            f |= 1 << (3 + 2 * a)
        f |= (8 * int(b[a])) << (8 + 5 * a)
    return f


class BlockSubGrid:
    __slots__ = ("n", "level", "origin", "dx", "leaf_origin", "offset", "_parent", "_sl")

    def __init__(self, parent, b, level):
        self.n = 8
        self.level = level
        self.dx = parent.dx
        self.leaf_origin = parent.origin
        self.offset = 8 * np.asarray(b)
        # cell centres as the leaf forms them: origin + dx * (8 b + i)
        self.origin = parent.origin + parent.dx * self.offset.astype(np.float64)
        self._parent = parent
        self._sl = (slice(None),) + tuple(slice(8 * int(x), 8 * int(x) + 8) for x in b)

    @property
    def interior(self):  # a view into the leaf's CURRENT array (a user may replace SubGrid.u)
        return self._parent.interior[self._sl]

    @property
    def u(self):  # no padded array of its own: host transfers go through the interior views
        return None                       # (numpy; a leaf-at-once fancy-index gather was slower)


class Block:
    __slots__ = ("leaf", "b", "level", "path", "ipos", "subgrid")

    def __init__(self, leaf, b, extra_levels):
        self.leaf = leaf
        self.b = tuple(int(x) for x in b)
        self.level = leaf.level + extra_levels
        nb = 2 ** extra_levels
        self.ipos = np.asarray(leaf.ipos, dtype=np.int64) * nb + np.asarray(b, dtype=np.int64)
        # Morton path below the leaf: one octant per extra level (tree.py _octant: x = bit 0)
        p = []
        for k in range(extra_levels - 1, -1, -1):
            p.append(((b[0] >> k) & 1) | (((b[1] >> k) & 1) << 1) | (((b[2] >> k) & 1) << 2))
        self.path = tuple(leaf.path) + tuple(p)
        self.subgrid = BlockSubGrid(leaf.subgrid, b, self.level)


class BlockTree:
    """The 8^3-block view of a uniform tree of n^3 leaves (n = 16 or 32): the
    subset of the Octree interface LeafBatch uses."""

    def __init__(self, tree):
        levels = {lf.level for lf in tree.leaves()}
        if len(levels) != 1:
            raise NotImplementedError("16^3 / 32^3 sub-grids: uniform trees only")
        self.parent = tree
        self.n = 8
        self.nb = tree.n // 8
        self.extra = int(np.log2(self.nb))
        self.boundary = tree.boundary
        self.width = tree.width
        self.lower = tree.lower
        bs = [(x, y, z) for x in range(self.nb) for y in range(self.nb) for z in range(self.nb)]
        self._blocks = []
        for lf in tree.sorted_leaves():
            blk = sorted((Block(lf, b, self.extra) for b in bs), key=lambda k: k.path)
            self._blocks += blk
        self._at = {(bk.level, *map(int, bk.ipos)): bk for bk in self._blocks}

    def leaves(self):
        return list(self._blocks)

    def sorted_leaves(self):
        return list(self._blocks)  # leaf order, then Morton order inside each leaf = path order

    def leaf_at(self, level, ipos):
        return self._at.get((level, int(ipos[0]), int(ipos[1]), int(ipos[2])))

    def find_leaf_region(self, level, ipos):
        return [(self.leaf_at(level, ipos), "same")]

    def neighbor_ipos(self, leaf, offset):
        span = 2 ** leaf.level
        pos = leaf.ipos + np.asarray(offset, dtype=np.int64)
        if self.boundary == "periodic":
            return pos % span
        if np.any(pos < 0) or np.any(pos >= span):
            return None
        return pos

