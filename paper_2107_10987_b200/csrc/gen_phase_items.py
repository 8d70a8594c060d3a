"""Generate omb_items.cuh: the item tables of the stage kernel's reconstruction
phases (omb_stage.cuh: boundary_lines = P1A/P1B, inplane_lines = P3).  An item
is one (line, position) of a plane: position pos10 = (y-2)*10 + (z-2) in [2,12)^2.
Entry bits: 0-6 pos10, 7-10 the line's index in the phase, 11 FULL (its lo/hi
feed a flux: all six fields are reconstructed; otherwise rho and p only, for
the reference's positivity-fallback count), 12 KT (P1 only: the interface
from the previous plane into this position feeds a face, i.e. its flux is
computed here).

Order, the point of the tables:
  1. by cost: KT items with 3 axes, 2 axes, 1 axis, then FULL-only, then
     rho/p-only -- so warps are uniformly heavy or light and the heavy ones spread
     over fewer warps (the barrier after P1 held 60 % of the kernel's barrier
     stalls with the per-line order: every warp carried a heavy lane);
  2. within a class, each line's 8 x 8 block first as half-warps of (8 z of
     row y, the same z of row y + 4): the 8-byte shared-memory accesses then hit
     distinct banks through both pitches the items use (prim ring rows: 14
     doubles; lo/hi and point-flux slots: 10 -- both put rows 4 apart 8 doubles
     apart mod 16); the rest greedily, then a local search (swaps inside a class)
     on the exact per-half-warp bank cost of every access site.

    python paper_2107_10987_b200/csrc/gen_phase_items.py
"""

import os
import random

DIRS = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, -1, 0), (1, 0, 1), (1, 0, -1), (0, 1, 1), (0, 1, -1),
        (1, 1, 1), (1, 1, -1), (1, -1, 1), (1, -1, -1)]  # geometry.py:24-41
ALL = [(y, z) for y in range(2, 12) for z in range(2, 12)]
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "omb_items.cuh")


def needed(l):
    if l == 0:
        return {(y, z) for y in range(3, 11) for z in range(3, 11)}
    if l in (1, 3, 4):
        return {(y, z) for y in range(2, 12) for z in range(3, 11)}
    if l in (2, 5, 6):
        return {(y, z) for y in range(3, 11) for z in range(2, 12)}
    return set(ALL)


def used_range(l):  # omb_stage.cuh used_range: P ranges of interfaces that feed faces of interior cells
    ylo = 2 if l in (3, 9, 10) else 3
    yhi = 11 if l in (4, 11, 12) else 10
    zlo = 2 if l in (5, 9, 11) else 3
    zhi = 11 if l in (6, 10, 12) else 10
    return ylo, yhi, zlo, zhi


def kt_set(l):
    ylo, yhi, zlo, zhi = used_range(l)
    d = DIRS[l]
    return {(y, z) for (y, z) in ALL if ylo <= y - d[1] <= yhi and zlo <= z - d[2] <= zhi}


def nax(l):
    return 1 if l == 0 else (3 if l >= 9 else 2)


def banks(p):
    return (p[0] * 14 + p[1]) % 16, (p[0] * 10 + p[1]) % 16


def paired_rows(cells):
    """Up to 64 cells of a rectangle in half-warps of (8 z of row y, the same z of row y + 4): both
    pitches (14, 10) put rows y and y + 4 eight doubles apart mod 16, so each half-warp hits 16
    distinct bank pairs.  Returns (ordered, leftover)."""
    have = set(cells)
    for y0 in sorted({y for y, _ in cells}):
        for z0 in sorted({z for _, z in cells}):
            out = []
            for q in range(4):
                for h in (0, 4):
                    out += [(y0 + q + h, z0 + j) for j in range(8)]
            if set(out) <= have:  # the first 8 x 8 square inside the set
                return out, [c for c in cells if c not in set(out)]
    return [], list(cells)


def table(lines, with_kt, seed):
    rng = random.Random(seed)
    groups = []  # (class rank, line index, positions)
    for k, l in enumerate(lines):
        full, kt = needed(l), (kt_set(l) if with_kt else set())
        cls = {}
        for p in ALL:
            c = (3 - nax(l)) if p in kt else (3 if p in full else 4)
            cls.setdefault(c, []).append(p)
        for c, ps in cls.items():
            rng.shuffle(ps)
            groups.append((c, k, ps))
    groups.sort(key=lambda g: (g[0], g[1]))
    # KT classes: each line's paired-row block of 64 (aligned half-warps, conflict-free), the rest after
    items = []
    for c in sorted({g[0] for g in groups}):
        if c <= 3:  # KT with 3, 2, 1 axes; reconstruction only
            rest = []
            for cc, k, ps in groups:
                if cc != c:
                    continue
                blk, left = paired_rows(ps)
                l = lines[k]
                items += [(k, p, p in needed(l), with_kt and p in kt_set(l)) for p in blk]
                rest.append((cc, k, left))
            todo = rest
        else:
            todo = [g for g in groups if g[0] == c]
        for _, k, ps in todo:
            pool = list(ps)
            while pool:
                w = len(items) // 16
                used = [banks(ip) for (kk, ip, _, _) in items[16 * w:] if kk == k]
                u14, u10 = {b[0] for b in used}, {b[1] for b in used}
                j = min(range(len(pool)), key=lambda i: (banks(pool[i])[0] in u14) + (banks(pool[i])[1] in u10))
                p = pool.pop(j)
                l = lines[k]
                items.append((k, p, p in needed(l), with_kt and p in kt_set(l)))
    return items



PL, NP, RING = 196, 100, 6 * 196  # omb_stage.cuh: ring plane pitch, lo/hi slots per line, ring slot stride


def accesses(item, phase_kt):
    """The shared-memory double addresses one item touches, per access site (site -> address):
    the 5 stencil loads of mono6 (ring rows of pitch 14; planes k for lines with d.x = 1), the
    hi store / lo-hi stores (slots of pitch 10), and for P1 KT items the previous-plane hi load
    and the point-flux store at P = pos - d."""
    k_line, (y, z), full, kt, l = item
    d = DIRS[l]
    c0, dd = y * 14 + z, d[1] * 14 + d[2]
    out = {}
    for k in range(5):
        out[("ring", k)] = ((k if d[0] else 2) * RING) + c0 + (k - 2) * dd
    pos = (y - 2) * 10 + (z - 2)
    out["slot"] = k_line * 6 * NP + pos
    if kt:
        out["hp"] = k_line * 6 * NP + pos - 10 * d[1] - d[2]
        out["raw"] = (l % 4) * 6 * NP + pos - 10 * d[1] - d[2]
    return out


def window_cost(items, phase_kt):
    """Excess wavefronts of one half-warp: per access site, max lanes on one bank pair minus 1."""
    sites = {}
    for it in items:
        for key, a in accesses(it, phase_kt).items():
            sites.setdefault(key, {}).setdefault(a % 16, set()).add(a)
    return sum(max(len(v) for v in banks.values()) - 1 for banks in sites.values())


def anneal(items, lines, phase_kt, iters, seed):
    """Swap items of the same cost class (the class order stays) while the half-warp bank
    cost does not grow."""
    rng = random.Random(seed)
    full = [(k, p, f, t, lines[k]) for (k, p, f, t) in items]
    cls = [(3 - nax(lines[k])) if t else (3 if f else 4) for (k, p, f, t) in items]
    by_cls = {}
    for i, c in enumerate(cls):
        by_cls.setdefault(c, []).append(i)
    win = lambda i: i // 16
    cost = {w: window_cost(full[16 * w:16 * w + 16], phase_kt) for w in range((len(full) + 15) // 16)}
    for _ in range(iters):
        c = rng.choice(list(by_cls))
        a, b = rng.sample(by_cls[c], 2) if len(by_cls[c]) > 1 else (None, None)
        if a is None or win(a) == win(b):
            continue
        wa, wb = win(a), win(b)
        before = cost[wa] + cost[wb]
        full[a], full[b] = full[b], full[a]
        ca = window_cost(full[16 * wa:16 * wa + 16], phase_kt)
        cb = window_cost(full[16 * wb:16 * wb + 16], phase_kt)
        if ca + cb <= before:
            cost[wa], cost[wb] = ca, cb
        else:
            full[a], full[b] = full[b], full[a]
    return [(k, p, f, t) for (k, p, f, t, _) in full], sum(cost.values())


def excess(items):
    tot = 0
    for w in range(0, len(items), 16):
        hw = items[w:w + 16]
        for k in {it[0] for it in hw}:
            for b in (0, 1):
                bs = [banks(it[1])[b] for it in hw if it[0] == k]
                tot += len(bs) - len(set(bs))
    return tot


def encode(items):
    out = []
    for k, (y, z), full, kt in items:
        out.append(((y - 2) * 10 + (z - 2)) | (k << 7) | (int(full) << 11) | (int(kt) << 12))
    return out


PHASES = [("P1A_NEW", [0, 3, 4, 5, 6], True), ("P1B_NEW", [9, 10, 11, 12], True), ("P1A_OLD", [0], True),
          ("P3_NEW", [1, 2, 7, 8], False), ("P3_OLD", [1, 2], False)]


def main():
    L = ["// GENERATED by gen_phase_items.py -- do not edit.",
         "// Item tables of the stage kernel's reconstruction phases (see omb_stage.cuh, boundary_lines / inplane_lines).",
         "// entry: bits 0-6 pos10, 7-10 line index in the phase, 11 FULL, 12 KT.", "#pragma once", ""]
    allv, off = [], 0
    for name, lines, kt in PHASES:
        best = min((table(lines, kt, s) for s in range(40)), key=excess)
        best, cost = anneal(best, lines, kt, 60000, 7)
        print(name, "half-warp bank cost", cost)
        assert sorted((k, p) for k, p, _, _ in best) == sorted((k, p) for k in range(len(lines)) for p in ALL)
        enc = encode(best)
        L.append(f"// {name}: lines {lines}, {len(enc)} items, excess wavefronts per plane {cost}")
        L.append(f"#define OMB_ITEMS_{name}_OFF {off}")
        L.append(f"#define OMB_ITEMS_{name}_N {len(enc)}")
        allv += enc
        off += len(enc)
    L.append(f"#define OMB_ITEMS_TOTAL {off}")
    L.append("#define OMB_ITEMS_ALL {" + ", ".join(map(str, allv)) + "}")
    L.append("")
    open(OUT, "w").write("\n".join(L))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
