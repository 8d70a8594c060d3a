"""Attribute ncu per-SASS-instruction samples to source lines via nvdisasm -g.

usage: python sass_lines.py <sass.csv from ncu --page source --print-source=sass --csv> <nvdisasm -g output> <kernel mangled name>
(profiling helper; the product does not use it)"""
import collections
import csv
import re
import sys


def main(sass_csv, dis_txt, kname, top=40):
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) > 3]
    iA, iW, iE = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    base = int(data[0][iA], 16)
    lines = open(dis_txt).read().split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith("//---") and kname in l)
    cur = ("?", 0)
    off2src = {}
    for l in lines[start + 1:]:
        if l.startswith("//---"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            off2src[int(m.group(1), 16)] = cur
    samp = collections.Counter()
    exe = collections.Counter()
    tot = 0
    for r in data:
        off = int(r[iA], 16) - base
        src = off2src.get(off, ("?", 0))
        w = float(r[iW] or 0)
        samp[src] += w
        exe[src] += float(r[iE] or 0)
        tot += w
    for src, w in samp.most_common(top):
        print(f"{100 * w / tot:5.1f}%  {src[0]}:{src[1]}  exec={exe[src]:.3g}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
