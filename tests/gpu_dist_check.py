"""Multi-GPU parity check, run under torchrun (one rank per GPU):

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tests/gpu_dist_check.py

Each rank advances its leaf partition of the Sedov c1 tree (and of the
smooth periodic case, two AMR trees, whose coarse/fine ghost sources and
reflux face fluxes cross ranks, and a self-gravitating tree with the device FMM
split over the ranks) with the halo reads / exchanges and compares its leaves
with the single-process golden state bitwise; dt must equal the golden dt.
Exit code 0 = parity."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))  # (HERE also provides octomini_host, the input trees)


def main():
    import torch
    import torch.distributed as dist

    from _cases import EOS, case_tree, state_of
    from paper_2107_10987_b200 import HydroMode
    from paper_2107_10987_b200.partition import Partition
    from paper_2107_10987_b200.stepper import B200HydroStepper

    lr = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    rank, world = dist.get_rank(), dist.get_world_size()
    bad = 0
    from paper_2107_10987_b200.gravity import B200FmmSolver

    for name, steps in (("sedov_c1", 3), ("smooth_periodic", 1), ("amr_reflux", 2), ("amr_sedov_small", 1),
                        ("gravity_step", 2)):
        t, g = case_tree(name)
        part = Partition(t, world, rank)
        kw = dict(gravity=B200FmmSolver(0.5), omega=0.3) if name == "gravity_step" else {}
        st = B200HydroStepper(t, EOS, HydroMode("new"), partition=part, max_run=2, **kw)
        for s in range(steps):
            dt = st.cfl_dt(0.4)
            if dt != float(g["dts"][s]):
                print(f"rank {rank} {name}: dt {dt!r} != golden {float(g['dts'][s])!r}", flush=True)
                bad += 1
            stats = st.rk3_step(dt)
            if s == 0:
                b0, b1 = part.bounds[rank], part.bounds[rank + 1]
                mine = state_of(t)[b0:b1]
                ref = g["state1"][b0:b1]
                nb = int(np.count_nonzero(mine[:, :5] != ref[:, :5]))
                ntau = int(np.count_nonzero(mine[:, 5] != ref[:, 5]))  # tau bitwise too (glibc pow on device)
                if nb or ntau:
                    print(f"rank {rank} {name}: {nb} rho/s/E mismatches, {ntau} tau mismatches", flush=True)
                    bad += 1
                if stats.amax != float(g["amax"][0]):
                    print(f"rank {rank} {name}: amax {stats.amax!r} != {float(g['amax'][0])!r}", flush=True)
                    bad += 1
    # config c2 (Sedov 128^3, 4096 leaves), 2 steps: the partitioned result equals the same
    # steps on this rank's GPU alone, bitwise (results must not depend on the GPU count)
    from octomini_host import SedovConfig, build_uniform_tree, init_sedov

    def c2():
        tr = build_uniform_tree(4, 8, boundary="reflecting")
        init_sedov(SedovConfig(), tr, EOS)
        return tr

    ts, tp = c2(), c2()
    single = B200HydroStepper(ts, EOS, HydroMode("new"), host_sync=False)
    part = Partition(tp, world, rank)
    multi = B200HydroStepper(tp, EOS, HydroMode("new"), partition=part)
    for s in range(2):
        d1, d2 = single.cfl_dt(0.4), multi.cfl_dt(0.4)
        if d1 != d2:
            print(f"rank {rank} c2: dt {d2!r} != single-GPU {d1!r}", flush=True)
            bad += 1
        single.rk3_step(d1)
        multi.rk3_step(d2)
    single.download()
    b0, b1 = part.bounds[rank], part.bounds[rank + 1]
    nmis = int(np.count_nonzero(state_of(tp)[b0:b1] != state_of(ts)[b0:b1]))
    if nmis:
        print(f"rank {rank} c2: {nmis} values differ from the single-GPU steps", flush=True)
        bad += 1
    t = torch.tensor([bad], device="cuda")
    dist.all_reduce(t)
    if rank == 0:
        print(f"multi-GPU parity on {world} ranks: {'OK' if int(t.item()) == 0 else 'FAIL'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(t.item()) == 0 else 1)


if __name__ == "__main__":
    main()
