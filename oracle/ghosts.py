"""Oracle restatement of the ghost exchange -- TEST INFRASTRUCTURE ONLY.

Follows reference ``pkg/src/octomini/mesh/ghosts.py:22-157`` (26 boxes per
leaf: same-level copy, coarse prolongation, fine restriction, physical
boundary mirror/clamp composed per axis) and ``mesh/transfer.py:13-64``
(minmod prolongation with one-sided edge slopes; pairwise restriction).
"""

import numpy as np

G = 3
SX = 1
OFFSETS = [(i, j, k) for i in (-1, 0, 1) for j in (-1, 0, 1) for k in (-1, 0, 1) if (i, j, k) != (0, 0, 0)]


def _minmod(a, b):
    return np.where(a * b > 0.0, np.where(np.abs(a) < np.abs(b), a, b), 0.0)


def _limited_slope(blk, ax):
    n = blk.shape[ax]
    if n == 1:
        return np.zeros_like(blk)
    lo = 2 * np.take(blk, [0], axis=ax) - np.take(blk, [1], axis=ax)
    hi = 2 * np.take(blk, [-1], axis=ax) - np.take(blk, [-2], axis=ax)
    pad = np.concatenate([lo, blk, hi], axis=ax)
    fwd = np.take(pad, range(2, n + 2), axis=ax) - np.take(pad, range(1, n + 1), axis=ax)
    bwd = np.take(pad, range(1, n + 1), axis=ax) - np.take(pad, range(0, n), axis=ax)
    return _minmod(fwd, bwd)


def prolong(blk):
    blk = np.asarray(blk)
    sl = [_limited_slope(blk, ax) for ax in (1, 2, 3)]
    f, a, b, c = blk.shape
    out = np.empty((f, 2 * a, 2 * b, 2 * c))
    for i in (0, 1):
        for j in (0, 1):
            for k in (0, 1):
                out[:, i::2, j::2, k::2] = (blk + sl[0] * (0.25 if i else -0.25)
                                            + sl[1] * (0.25 if j else -0.25) + sl[2] * (0.25 if k else -0.25))
    return out


def restrict(fine):
    f = np.asarray(fine)
    p = lambda i, j, k: f[:, i::2, j::2, k::2]  # noqa: E731
    return 0.125 * (((p(0, 0, 0) + p(1, 0, 0)) + (p(0, 1, 0) + p(1, 1, 0)))
                    + ((p(0, 0, 1) + p(1, 0, 1)) + (p(0, 1, 1) + p(1, 1, 1))))


def _source(tree, leaf, rd):
    n = leaf.subgrid.n
    if not any(rd):
        return leaf.subgrid.interior
    pos = tree.neighbor_ipos(leaf, rd)
    cover = tree.find_leaf_region(leaf.level, pos)
    role = cover[0][1]
    if role == "same":
        sl = tuple(slice(G, 2 * G) if c == 1 else (slice(n, n + G) if c == -1 else slice(G, G + n)) for c in rd)
        return cover[0][0].subgrid.u[(slice(None),) + sl]
    want = [(0, G) if c == 1 else ((n - G, n) if c == -1 else (0, n)) for c in rd]
    if role == "coarse":
        nb = cover[0][0]
        octant = [int(pos[a]) & 1 for a in range(3)]
        csl, off = [], []
        for a in range(3):
            c0 = octant[a] * (n // 2) + want[a][0] // 2
            c1 = octant[a] * (n // 2) + (want[a][1] - 1) // 2 + 1
            m0, m1 = max(c0 - 1, 0), min(c1 + 1, n)
            csl.append(slice(m0, m1))
            off.append(want[a][0] + octant[a] * n - 2 * m0)
        fine = prolong(nb.subgrid.interior[:, csl[0], csl[1], csl[2]])
        return fine[:, off[0]:off[0] + want[0][1] - want[0][0], off[1]:off[1] + want[1][1] - want[1][0],
                    off[2]:off[2] + want[2][1] - want[2][0]]
    out = np.empty((leaf.subgrid.u.shape[0],) + tuple(G if c else n for c in rd))
    for child, _ in cover:
        k = [int(child.ipos[a]) & 1 for a in range(3)]
        src, dst = [], []
        for a in range(3):
            c0 = max(want[a][0], k[a] * (n // 2))
            c1 = min(want[a][1], (k[a] + 1) * (n // 2))
            if c0 >= c1:
                break
            src.append(slice(G + 2 * c0 - k[a] * n, G + 2 * c1 - k[a] * n))
            dst.append(slice(c0 - want[a][0], c1 - want[a][0]))
        else:
            out[:, dst[0], dst[1], dst[2]] = restrict(child.subgrid.u[:, src[0], src[1], src[2]])
    return out


def fill_leaf(tree, leaf):
    n = leaf.subgrid.n
    u = leaf.subgrid.u
    span = 2 ** leaf.level
    for r in OFFSETS:
        off = {}
        rd = list(r)
        if tree.boundary != "periodic":
            for a in range(3):
                p = leaf.ipos[a] + r[a]
                if p < 0 or p >= span:
                    off[a] = r[a]
                    rd[a] = 0
        blk = _source(tree, leaf, tuple(rd))
        idx, flips = [], []
        for a in range(3):
            w = blk.shape[1 + a]
            if a in off:
                t = np.arange(G)
                if tree.boundary == "reflecting":
                    idx.append(w - 1 - t if off[a] == 1 else G - 1 - t)
                    flips.append(a)
                else:
                    idx.append(np.full(G, w - 1 if off[a] == 1 else 0))
            else:
                idx.append(np.arange(w))
        piece = blk[:, idx[0][:, None, None], idx[1][None, :, None], idx[2][None, None, :]]
        if flips:
            piece = piece.copy()
            for a in flips:
                piece[SX + a] = -piece[SX + a]
        tgt = [(0, G) if c == -1 else ((G, G + n) if c == 0 else (G + n, 2 * G + n)) for c in r]
        u[:, tgt[0][0]:tgt[0][1], tgt[1][0]:tgt[1][1], tgt[2][0]:tgt[2][1]] = piece


def exchange(tree, leaves=None):
    for lf in (leaves if leaves is not None else tree.leaves()):
        fill_leaf(tree, lf)
