"""Leaf partition across ranks (one process per GPU) and the halo exchange.

SURVEY.md §8(e): the path shards by octree leaf.  Rank r owns a contiguous
chunk of ``tree.sorted_leaves()`` (Morton order, reference tree.py:148-150)
balanced by leaf count -- for the 256^3 config on 8 GPUs exactly one
level-1 octant each.  Every RK stage needs one exchange: the current-stage
interiors of the same-level neighbour leaves owned by other ranks (the
reference reads them through ``fill_leaf_ghosts``, mesh/ghosts.py:115-150).
Whole 8^3 neighbour leaves are exchanged (all_to_all over NCCL/NVLink); the
stage kernel then gathers their 3-wide halo exactly as for local leaves, so
results are bitwise independent of the number of ranks.

The CFL reduction is an all-reduce(MIN) of (worst, dt) and, for the
reference's non-finite check, of the first bad global leaf index; the
per-stage signal-speed maxima and fallback counts are reduced after the step.
"""

import numpy as np

from .batch import LeafBatch


def amr_sources(tree, leaves, gnbr):
    """Per leaf: global indices of the leaves its coarse/fine ghost regions read
    (the coarse neighbour, or the 8 finer children), from find_leaf_region."""
    from .batch import AMR, OFFS

    index = {lf.path: i for i, lf in enumerate(leaves)}
    src = [[] for _ in leaves]
    for i, lf in enumerate(leaves):
        for q in np.nonzero(gnbr[i] == AMR)[0]:
            pos = tree.neighbor_ipos(lf, OFFS[q])
            for nb, _ in tree.find_leaf_region(lf.level, pos):
                src[i].append(index[nb.path])
    return src


def reflux_pairs(tree, leaves):
    """(coarse leaf, fine child) global index pairs of the reference's reflux
    (hydro/step.py:206-241): the coarse leaf needs the child's face fluxes."""
    index = {lf.path: i for i, lf in enumerate(leaves)}
    out = []
    for i, lf in enumerate(leaves):
        for ax in range(3):
            for side in (-1, 1):
                off = [0, 0, 0]
                off[ax] = side
                pos = tree.neighbor_ipos(lf, off)
                if pos is None:
                    continue
                cover = tree.find_leaf_region(lf.level, pos)
                if cover[0][1] != "fine":
                    continue
                for child, _ in cover:
                    k = int(child.ipos[ax]) & 1
                    if k == (0 if side > 0 else 1):
                        out.append((i, index[child.path]))
    return out


class Partition:
    def __init__(self, tree, world, rank):
        from .batch import AMR, neighbor_table

        self.world, self.rank = world, rank
        leaves = tree.sorted_leaves()
        G = len(leaves)
        self.G = G
        self.bounds = [G * r // world for r in range(world + 1)]
        owner = np.searchsorted(np.array(self.bounds[1:]), np.arange(G), side="right")
        self.owner = owner
        gnbr = neighbor_table(tree, leaves, allow_amr=True)
        self.gnbr = gnbr
        self.amr = bool(np.any(gnbr == AMR))
        # dependency edges (reader -> source): same-level neighbours, AMR ghost sources
        src = np.repeat(np.arange(G), 27)
        dst = gnbr.reshape(-1)
        keep = dst >= 0
        e_src, e_dst = [src[keep]], [dst[keep]]
        if self.amr:
            srcs = amr_sources(tree, leaves, gnbr)
            a = [(i, j) for i, lst in enumerate(srcs) for j in lst]
            if a:
                a = np.array(a, dtype=np.int64)
                e_src.append(a[:, 0])
                e_dst.append(a[:, 1])
        es, ed = np.concatenate(e_src), np.concatenate(e_dst)
        cross = owner[es] != owner[ed]
        pairs = np.unique(np.stack([owner[es[cross]], ed[cross]], axis=1), axis=0) if np.any(cross) else \
            np.zeros((0, 2), dtype=np.int64)
        halo_of = [pairs[pairs[:, 0] == r, 1] for r in range(world)]
        b0, b1 = self.bounds[rank], self.bounds[rank + 1]
        mine = halo_of[rank]
        self.halo = mine[np.lexsort((mine, owner[mine]))]  # by (owner, index)
        self.recv_counts = [int(np.count_nonzero(owner[self.halo] == s)) for s in range(world)]
        self.send = []
        for s in range(world):
            h = halo_of[s]
            self.send.append(np.sort(h[owner[h] == rank]) if s != rank else np.zeros(0, dtype=np.int64))
        self.send_counts = [len(x) for x in self.send]
        self.nown = b1 - b0
        self.gids = np.concatenate([np.arange(b0, b1), self.halo]).astype(np.int64)
        self.leaves = [leaves[int(g)] for g in self.gids]
        self.send_local = np.concatenate([x - b0 for x in self.send]).astype(np.int32) if world > 1 else \
            np.zeros(0, dtype=np.int32)
        # second exchange (AMR only): fine children's exported face fluxes for remote coarse leaves
        self.flux_send = [np.zeros(0, dtype=np.int64) for _ in range(world)]
        self.flux_recv = [np.zeros(0, dtype=np.int64) for _ in range(world)]
        if self.amr:
            rp = reflux_pairs(tree, leaves)
            for s in range(world):
                if s == rank:
                    continue
                self.flux_send[s] = np.array(sorted({j for i, j in rp if owner[i] == s and owner[j] == rank}),
                                             dtype=np.int64)
                self.flux_recv[s] = np.array(sorted({j for i, j in rp if owner[i] == rank and owner[j] == s}),
                                             dtype=np.int64)
        self.flux_send_counts = [len(x) for x in self.flux_send]
        self.flux_recv_counts = [len(x) for x in self.flux_recv]

    def batch(self, tree, max_run=4):
        b0 = self.bounds[self.rank]
        extra = sorted({int(j) - b0 for lst in self.flux_send for j in lst})
        b = LeafBatch(tree, max_run=max_run, leaves=self.leaves, ncompute=self.nown, gnbr=self.gnbr,
                      gids=self.gids, extra_exporters=extra)
        # flux-slot lists of the second exchange (batch slots, per peer, in global-index order)
        local = {int(g): i for i, g in enumerate(self.gids)}
        self.flux_send_slots = np.array([b.slot_of[local[int(j)]] for lst in self.flux_send for j in lst],
                                        dtype=np.int32)
        self.flux_recv_slots = np.array([b.slot_of[local[int(j)]] for lst in self.flux_recv for j in lst],
                                        dtype=np.int32)
        return b


def exchange(dist, group, state, send_idx, send_counts, recv_counts, nown, pack, unpack, sendbuf, recvbuf):
    """One halo exchange of ``state`` ([6][fstride]): pack the owned leaves
    other ranks need, all_to_all, unpack into the halo slots (local indices
    nown.. in (owner, index) order)."""
    per = 6 * 512
    if sum(send_counts):
        pack(state, send_idx, sendbuf)
    dist.all_to_all_single(recvbuf[:sum(recv_counts) * per], sendbuf[:sum(send_counts) * per], [c * per for c in recv_counts], [c * per for c in send_counts],
                           group=group)
    if sum(recv_counts):
        unpack(recvbuf, state, nown)
