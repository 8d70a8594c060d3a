"""Device FMM timing (not part of the product): host preparation once per
topology, then the per-stage device solve (density + dphi/dt solves).

    python profiles/fmm_bench.py [level] [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main(level=3, reps=5):
    import torch

    from paper_2107_10987_b200.batch import LeafBatch
    from paper_2107_10987_b200.gravity import B200FmmSolver
    from octomini_host import synthetic_star

    tree, eos, _, om, fl = synthetic_star(level=level)
    s = B200FmmSolver(0.5)
    t0 = time.perf_counter()
    s.prepare(tree)
    t1 = time.perf_counter()
    b = LeafBatch(tree)
    U = torch.from_numpy(b.pack().reshape(-1)).cuda()
    info = torch.from_numpy(b.info.view("u1").copy()).cuda()
    G = torch.zeros(4 * b.fstride, dtype=torch.float64, device="cuda")
    s.stage_fields(U, b.fstride, info, b.bc, b.L, G)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        s.stage_fields(U, b.fstride, info, b.bc, b.L, G)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    cells = b.L * 512
    print(f"L{level}: {b.L} leaves, {s.table.nentities} entities, {s.stats['groups']} groups, "
          f"{s.stats['pairs']} pairs; prepare {t1 - t0:.1f} s (host); per-stage device solve "
          f"(density + dphi/dt) {ms:.2f} ms = {2 * s.stats['pairs'] / (ms / 2 * 1e-3) / 1e9:.2f} G interactions/s "
          f"per solve; {cells} cells")


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:3]])
