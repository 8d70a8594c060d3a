"""One-file summary of an ncu --set full capture of k_stage (the metrics DESIGN/README cite):
    python profiles/ncu_summary.py REPORT.ncu-rep OUT.txt "title"
"""
import csv
import io
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__inst_executed.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__average_warp_latency_per_inst_issued.ratio",
        "smsp__inst_executed.sum"]


def main(rep, out, title):
    raw = subprocess.run(["ncu", "-i", os.path.abspath(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         cwd="/tmp").stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    lines = [f"# {title}", "# ncu --set full --import-source on --clock-control none -k regex:k_stage -s 9 -c 1 "
             "python bench.py --config c2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline", ""]
    lines += [f"{k} = {v[h.index(k)]} {u[h.index(k)]}" for k in KEYS if k in h]
    lines += ["", "# stall reasons (warps per issue-active cycle)"]
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            lines.append(f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]} = {v[h.index(k)]}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
