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

from .batch import LeafBatch, neighbor_table


class Partition:
    def __init__(self, tree, world, rank):
        self.world, self.rank = world, rank
        leaves = tree.sorted_leaves()
        G = len(leaves)
        self.G = G
        self.bounds = [G * r // world for r in range(world + 1)]
        owner = np.searchsorted(np.array(self.bounds[1:]), np.arange(G), side="right")
        self.owner = owner
        gnbr = neighbor_table(tree, leaves)
        self.gnbr = gnbr
        # halo of every rank: neighbours of its leaves owned elsewhere
        src = np.repeat(np.arange(G), 27)
        dst = gnbr.reshape(-1)
        keep = (dst >= 0) & (owner[np.maximum(dst, 0)] != owner[src])
        pairs = np.unique(np.stack([owner[src[keep]], dst[keep]], axis=1), axis=0)  # (rank, global leaf)
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
        # local index of each leaf to send (owned leaves are local 0..nown-1)
        self.send_local = np.concatenate([x - b0 for x in self.send]).astype(np.int32) if world > 1 else \
            np.zeros(0, dtype=np.int32)

    def batch(self, tree, max_run=4):
        return LeafBatch(tree, max_run=max_run, leaves=self.leaves, ncompute=self.nown, gnbr=self.gnbr,
                         gids=self.gids)


def exchange(dist, group, state, send_idx, send_counts, recv_counts, nown, pack, unpack, sendbuf, recvbuf):
    """One halo exchange of ``state`` ([6][fstride]): pack the owned leaves
    other ranks need, all_to_all, unpack into the halo slots (local indices
    nown.. in (owner, index) order)."""
    per = 6 * 512
    if sum(send_counts):
        pack(state, send_idx, sendbuf)
    dist.all_to_all_single(recvbuf, sendbuf, [c * per for c in recv_counts], [c * per for c in send_counts],
                           group=group)
    if sum(recv_counts):
        unpack(recvbuf, state, nown)
