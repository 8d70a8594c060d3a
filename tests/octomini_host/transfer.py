"""Inter-level transfer on the host (tree construction / split only).

Restates ``octomini.mesh.transfer`` (reference ``pkg/src/octomini/mesh/transfer.py:13-64``):
minmod-limited linear prolongation whose slopes become one-sided at the block
edge (linear extrapolation pad), and the pairwise 8-cell restriction average.
Arithmetic order is kept so refined initial data is bit-identical.
"""

import numpy as np


def minmod(a, b):
    pick = np.where(np.abs(a) < np.abs(b), a, b)
    return np.where(a * b > 0.0, pick, 0.0)


def _slopes(block, axis):
    nax = block.shape[axis]
    if nax == 1:
        return np.zeros_like(block)
    first = np.take(block, [0], axis=axis)
    second = np.take(block, [1], axis=axis)
    last = np.take(block, [-1], axis=axis)
    before_last = np.take(block, [-2], axis=axis)
    pad = np.concatenate([2 * first - second, block, 2 * last - before_last], axis=axis)
    up = np.take(pad, range(2, nax + 2), axis=axis) - np.take(pad, range(1, nax + 1), axis=axis)
    down = np.take(pad, range(1, nax + 1), axis=axis) - np.take(pad, range(0, nax), axis=axis)
    return minmod(up, down)


def prolong_block(block):
    block = np.asarray(block)
    s = [_slopes(block, ax) for ax in (1, 2, 3)]
    f, nx, ny, nz = block.shape
    out = np.empty((f, 2 * nx, 2 * ny, 2 * nz), dtype=block.dtype)
    for cx in (0, 1):
        for cy in (0, 1):
            for cz in (0, 1):
                q = (0.25 if cx else -0.25, 0.25 if cy else -0.25, 0.25 if cz else -0.25)
                out[:, cx::2, cy::2, cz::2] = block + s[0] * q[0] + s[1] * q[1] + s[2] * q[2]
    return out


def restrict_block(fine):
    f = np.asarray(fine)
    e = lambda i, j, k: f[:, i::2, j::2, k::2]  # noqa: E731
    return 0.125 * (((e(0, 0, 0) + e(1, 0, 0)) + (e(0, 1, 0) + e(1, 1, 0)))
                    + ((e(0, 0, 1) + e(1, 0, 1)) + (e(0, 1, 1) + e(1, 1, 1))))
