"""Grid geometry shared by the host mirror, the C-ABI tables and the tests.

Restates the integer facts of ``octomini.geometry`` (reference
``pkg/src/octomini/geometry.py:16-123``): field numbering, ghost width, the
13 reconstruction line directions and, per face-normal axis, the 9 face
quadrature points with the (line, dP, flip) rows behind each of them.  The
point and row ORDER is normative: it fixes the floating-point summation
order of the face quadrature (reference ``_core.pyx:282-346``).
"""

import numpy as np

RHO, SX, SY, SZ, EGAS, TAU = range(6)
NFIELDS = 6
PRHO, PVX, PVY, PVZ, PP, PTAU = range(6)

GHOST = 3

# 13 lines through the cell centre, first non-zero component positive
# (reference geometry.py:24-41).  Index = line id used everywhere below.
LINE_DIRS = np.array(
    [(1, 0, 0), (0, 1, 0), (0, 0, 1),
     (1, 1, 0), (1, -1, 0), (1, 0, 1), (1, 0, -1), (0, 1, 1), (0, 1, -1),
     (1, 1, 1), (1, 1, -1), (1, -1, 1), (1, -1, -1)],
    dtype=np.int64,
)
NLINES = 13

W_CENTER = 16.0 / 36.0
W_EDGE = 4.0 / 36.0
W_VERTEX = 1.0 / 36.0

KIND_CENTER, KIND_EDGE, KIND_VERTEX = 0, 1, 2
_KIND_NAMES = ("center", "edge", "vertex")

# transverse offsets of the 9 points in the reference's enumeration order
# (tb outer, tc inner over (0, -1/2, +1/2)), then stable-sorted by kind
_HALF = (0.0, -0.5, 0.5)


def _points_for_axis(a):
    b, c = [ax for ax in range(3) if ax != a]
    pts = []
    for tb in _HALF:
        for tc in _HALF:
            halves = int(tb != 0.0) + int(tc != 0.0)
            rows = []
            for line in range(NLINES):
                d = LINE_DIRS[line]
                if d[a] == 0:
                    continue
                if (d[b] != 0) != (tb != 0.0) or (d[c] != 0) != (tc != 0.0):
                    continue
                # the point sits at lower + (1/2 along a, tb, tc); the line's
                # interface through it joins P = point - d/2 and P + d
                off = np.zeros(3)
                off[a], off[b], off[c] = 0.5, tb, tc
                p = off - 0.5 * d
                rows.append((line, tuple(int(round(x)) for x in p), bool(d[a] < 0)))
            assert len(rows) == 1 << halves
            pts.append((halves, (tb, tc), rows))
    pts.sort(key=lambda t: t[0])  # stable: keeps the enumeration order per kind
    return [(_KIND_NAMES[k], rows) for k, _, rows in pts]


FACE_TABLES = [_points_for_axis(a) for a in range(3)]


def flat_face_table(axis):
    """(kind(9,), nrows(9,), line(25,), dp(25,3), flip(25,)) int32 arrays."""
    kinds, nrows, lines, dps, flips = [], [], [], [], []
    for kind, rows in FACE_TABLES[axis]:
        kinds.append(_KIND_NAMES.index(kind))
        nrows.append(len(rows))
        for line, dp, flip in rows:
            lines.append(line)
            dps.append(dp)
            flips.append(int(flip))
    return (np.array(kinds, np.int32), np.array(nrows, np.int32),
            np.array(lines, np.int32), np.array(dps, np.int32).reshape(-1, 3),
            np.array(flips, np.int32))
