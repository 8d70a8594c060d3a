"""Independent restatement of the face-quadrature table generator
(reference ``pkg/src/octomini/geometry.py:51-123``) for the oracle.

Kept separate from the product's geometry module so the checker does not
share code with the thing it checks."""

import numpy as np

LINE_DIRS = np.array([(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, -1, 0), (1, 0, 1), (1, 0, -1),
                      (0, 1, 1), (0, 1, -1), (1, 1, 1), (1, 1, -1), (1, -1, 1), (1, -1, -1)])


def flat_face_table(axis):
    b, c = [x for x in range(3) if x != axis]
    entries = []
    for tb in (0.0, -0.5, 0.5):
        for tc in (0.0, -0.5, 0.5):
            kind = (tb != 0) + (tc != 0)
            rows = []
            for line, d in enumerate(LINE_DIRS):
                if abs(d[axis]) != 1 or (abs(d[b]) == 1) != (tb != 0) or (abs(d[c]) == 1) != (tc != 0):
                    continue
                pt = np.zeros(3)
                pt[axis], pt[b], pt[c] = 0.5, tb, tc
                rows.append((line, np.round(pt - d / 2.0).astype(int), int(d[axis] < 0)))
            entries.append((kind, rows))
    entries.sort(key=lambda e: e[0])
    kinds = np.array([k for k, _ in entries], np.int32)
    nrows = np.array([len(r) for _, r in entries], np.int32)
    lines = np.array([x[0] for _, r in entries for x in r], np.int32)
    dps = np.array([x[1] for _, r in entries for x in r], np.int32)
    flips = np.array([x[2] for _, r in entries for x in r], np.int32)
    return kinds, nrows, lines, dps, flips
