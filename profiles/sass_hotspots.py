"""Join an ncu source-page capture (per-SASS-instruction metrics) with the
line table of the same build (nvdisasm -g) and aggregate by source line and by
opcode.  Usage (here, no GPU):

    python profiles/sass_hotspots.py REPORT.ncu-rep [libomb200.so] [top]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(so, func):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True, check=True)
    cub = [f for f in os.listdir(d) if f.startswith("omb_kernels") and f.endswith(".cubin") and "fmm" not in f][0]
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    cur, inside, table = None, False, {}
    for ln in out.splitlines():
        if ln.startswith(".text.") or ln.startswith("//----"):
            inside = func in ln
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            table[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return table


def main(rep, so="paper_2107_10987_b200/libomb200.so", top=40):
    so = os.path.abspath(so)
    func = "_Z7k_stageILi512ELi0EEvN3omb9StageArgsE"
    raw = subprocess.run(["ncu", "-i", os.path.abspath(rep), "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True, cwd="/tmp").stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ia, isamp, iexe = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index(
        "Instructions Executed")
    iconf = hdr.index("L1 Wavefronts Shared Excessive")
    data = rows[2:]
    base = int(data[0][ia], 16)
    table = sass_lines(so, func)
    by_line = collections.defaultdict(lambda: [0, 0, 0])
    by_op = collections.defaultdict(lambda: [0, 0])
    tot_s = tot_e = 0
    for r in data:
        off = int(r[ia], 16) - base
        src, ins = table.get(off, (None, r[1].strip()))
        s, e, c = int(r[isamp] or 0), int(r[iexe] or 0), int(r[iconf] or 0)
        tot_s += s
        tot_e += e
        by_line[src][0] += s
        by_line[src][1] += e
        by_line[src][2] += c
        op = ins.split()[0] if not ins.startswith("@") else ins.split()[1]
        by_op[op.split(".")[0]][0] += e
        by_op[op.split(".")[0]][1] += s
    print(f"total stall samples {tot_s}, warp instructions {tot_e}")
    print("\n-- by source line (samples %, instr %, excess shared wavefronts)")
    for k, (s, e, c) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:int(top)]:
        print(f"{str(k):42s} {100 * s / tot_s:6.2f} {100 * e / tot_e:6.2f} {c:10d}")
    print("\n-- by opcode (instr %, samples %)")
    for k, (e, s) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:30]:
        print(f"{k:12s} {100 * e / tot_e:6.2f} {100 * s / tot_s:6.2f}")


if __name__ == "__main__":
    main(*sys.argv[1:])


def opcode_lines(rep, so, opcode, top=25):
    """Source lines executing the most instructions of one opcode (prefix match)."""
    so = os.path.abspath(so)
    func = "_Z7k_stageILi512ELi0EEvN3omb9StageArgsE"
    raw = subprocess.run(["ncu", "-i", os.path.abspath(rep), "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True, cwd="/tmp").stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ia, iexe = hdr.index("Address"), hdr.index("Instructions Executed")
    data = rows[2:]
    base = int(data[0][ia], 16)
    table = sass_lines(so, func)
    agg = collections.Counter()
    full = collections.Counter()
    for r in data:
        src, ins = table.get(int(r[ia], 16) - base, (None, r[1].strip()))
        op = ins.split()[1] if ins.startswith("@") else ins.split()[0]
        if op.startswith(opcode):
            agg[src] += int(r[iexe] or 0)
            full[op] += int(r[iexe] or 0)
    tot = sum(agg.values())
    print(f"{opcode}: {tot} warp instructions; variants {full.most_common(6)}")
    for k, v in agg.most_common(top):
        print(f"  {str(k):42s} {100 * v / tot:6.2f}")


def stall_lines(rep, so, reasons=("stall_barrier", "stall_wait", "stall_short_sb", "stall_branch_resolving",
                                  "stall_no_inst", "stall_math"), top=12):
    """Per stall reason: the source lines holding most of its samples."""
    so = os.path.abspath(so)
    func = "_Z7k_stageILi512ELi0EEvN3omb9StageArgsE"
    raw = subprocess.run(["ncu", "-i", os.path.abspath(rep), "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True, cwd="/tmp").stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ia = hdr.index("Address")
    data = rows[2:]
    base = int(data[0][ia], 16)
    table = sass_lines(so, func)
    for rs in reasons:
        j = hdr.index(rs)
        agg = collections.Counter()
        for r in data:
            src, _ = table.get(int(r[ia], 16) - base, (None, ""))
            agg[src] += int(r[j] or 0)
        tot = sum(agg.values())
        print(f"{rs}: {tot} samples")
        for k, v in agg.most_common(top):
            print(f"  {str(k):42s} {100 * v / max(tot, 1):6.2f}")


def calls(rep, so):
    """Executed CALL instructions (out-of-line subroutines: IEEE division/sqrt slow paths) per source line."""
    so = os.path.abspath(so)
    func = "_Z7k_stageILi512ELi0EEvN3omb9StageArgsE"
    raw = subprocess.run(["ncu", "-i", os.path.abspath(rep), "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True, cwd="/tmp").stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ia, iexe, ithr = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
    data = rows[2:]
    base = int(data[0][ia], 16)
    table = sass_lines(so, func)
    for r in data:
        off = int(r[ia], 16) - base
        src, ins = table.get(off, (None, r[1].strip()))
        if "CALL" in ins and int(r[iexe] or 0):
            print(f"{off:6x} {str(src):36s} {ins[:40]:40s} warp {r[iexe]:>10s} thread {r[ithr]:>12s}")
