"""Benchmark of the B200 FP64 hydro step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One "step" is what the reference driver does per timestep
(``om/driver.py:165-168``): ``cfl_dt(0.4)`` then one SSP-RK3 ``rk3_step`` --
here the CFL reduction kernels plus three launches of the fused stage kernel,
dt kept on the device.  Workload (N=1): config c2 of BASELINE.json, Sedov-Taylor
blast wave on a uniform 128^3 grid = 4096 sub-grids of 8^3 (level-4 octree,
reflecting walls), synthetic initial data from ``init_sedov`` (no RNG).
``value`` = cells x steps / device time (state resident in HBM); ``e2e`` = the
same metric through the public drop-in API (``B200HydroStepper.cfl_dt`` +
``rk3_step`` with host_sync) including the H2D upload and D2H download of the
whole state every step.

``--impl reference`` times the CPU oracle (C restatement of the reference's
compiled kernels + its numpy orchestration, all host threads) on a bounded
sample of the same workload, rank 0 only.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))  # octomini_host: synthetic inputs (octomini's tree API)

METRIC = "hydro cell-updates/sec (FP64) per GPU & at 1/2/4/8 B200; % of roofline"
UNIT = "cell-updates/s"
# algorithmic FP64 flops per cell per RK stage (non-redundant count)
FLOPS_PER_CELL_STAGE = 4115.0
FLOPS_PER_CELL_UPDATE = 12362.0
# algorithmic HBM bytes per cell per stage: read cur + write next (48+48) + u0 on 2 of 3 stages
BYTES_PER_CELL_STAGE = 48.0 + 48.0 + 48.0 * 2.0 / 3.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=60)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--level", type=int, default=None, help="octree level of the uniform tree (default: c2 = 4)")
    p.add_argument("--max-run", type=int, default=4)
    p.add_argument("--e2e-steps", type=int, default=8)
    p.add_argument("--cpu-leaves", type=int, default=512)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--subgrid", type=int, default=8, choices=[8, 16, 32],
                   help="sub-grid edge of the uniform Sedov trees (16/32: single GPU; run as 8^3 blocks)")
    p.add_argument("--efficiency-steps", type=int, default=10,
                   help="N>1: steps of the whole workload on rank 0's GPU alone (0 = skip)")
    p.add_argument("--config", default=None, choices=["c2", "c3", "c4", "c5", "c5g"],
                   help="c2: uniform 128^3; c3: uniform 256^3 (default at every N); c4: AMR Sedov, "
                        "levels 3-6; c5: rotating polytrope stand-in, fixed gravity, 128^3; c5g: the same star "
                        "self-gravitating (device FMM re-solved every stage, theta 0.5; --level sets the tree, "
                        "default 4 = 128^3)")
    return p.parse_args()


SUBGRID_N = 8  # --subgrid: sub-grid edge of the uniform Sedov trees (8, 16 or 32; same cells)


def sedov_tree(level):
    from octomini_host import SedovConfig, build_uniform_tree, init_sedov
    from paper_2107_10987_b200 import EosConfig

    if level == "c4":
        from octomini_host import amr_sedov_tree

        return amr_sedov_tree()
    # the same 8*2^level cells per edge as SUBGRID_N^3 leaves (c2 may also read 512 x 16^3)
    t = build_uniform_tree(level - {8: 0, 16: 1, 32: 2}[SUBGRID_N], SUBGRID_N, boundary="reflecting")
    init_sedov(SedovConfig(), t, EosConfig(gamma=1.4))
    return t


def resolve_level(args, world):
    if args.config in ("c4", "c5", "c5g"):
        return args.config
    if args.config == "c3":
        return 5
    if args.config == "c2":
        return 4
    # every N runs the same workload (strong scaling): config c3, 256^3, fits one B200
    return args.level if args.level is not None else 5


def workload_name(level, nleaves):
    if level == "c5":
        return ("star_uniform_L4_n8 (config c5 stand-in: closed-form n=1 polytrope, rotating frame, fixed "
                "self-gravity, rho floor 1e-4, outflow, gamma 5/3)")
    if level == "c5g":
        return ("star_uniform_n8 self-gravitating (config c5: closed-form rotating n=1 polytrope, floors, outflow, "
                "gamma 5/3; gravity = device FMM theta 0.5 re-solved every stage from the stage state, phi/g and "
                "dphi/dt, as HydroStepper + FmmSolver)")
    if level == "c4":
        return f"sedov_amr_L3-6_n8 (config c4): {nleaves} sub-grids of 8^3 on levels 3-6 (SURVEY.md 8d construction)"
    tag = {4: " (config c2: 128^3)", 5: " (config c3: 256^3)"}.get(level, "")
    lv = level - {8: 0, 16: 1, 32: 2}[SUBGRID_N]
    return f"sedov_uniform_L{lv}_n{SUBGRID_N}{tag}"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return {}


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi every 50 ms from before the warm-up on; stop(t0, t1) keeps the
    samples taken inside the timed wall-clock window [t0, t1] (the nearest ones
    when the window is shorter than the sampling period)."""

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
                                      bufsize=1)
            import threading

            self.rows = []
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.p = None

    def _read(self):
        for line in self.p.stdout:  # stamp each sample with the host wall clock
            self.rows.append((time.time(), line.strip().split(",")))

    def stop(self, t0=None, t1=None):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.p.terminate()
        self.p.wait()
        self.t.join(timeout=1.0)
        os.unlink(self.f.name)
        rows = [(ts, r) for ts, r in self.rows if len(r) >= 9]
        if t0 is not None and rows:
            inside = [(ts, r) for ts, r in rows if t0 <= ts <= t1]
            if not inside:  # window shorter than the period: the samples around it
                inside = sorted(rows, key=lambda x: min(abs(x[0] - t0), abs(x[0] - t1)))[:2]
            rows = inside
        rows = [r for _, r in rows]
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, nm in enumerate(names):
                if r[5 + k].strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU side: the oracle (test infrastructure) timed on the host cores
# ---------------------------------------------------------------------------
def cpu_run(level, nleaves, steps, warmup):
    """Time OracleStepper on a contiguous (Morton) sample of leaves; returns
    (cell-updates/s, threads, sample description)."""
    import oracle
    from oracle.step import OracleStepper

    kw = {}
    gamma = 1.4
    if level == "c5":
        from octomini_host import synthetic_star

        tree, eos, grav, om, fl = synthetic_star(level=4)
        kw = dict(omega=om, gravity=grav, floors=(fl.rho, fl.tau, fl.vmax))
        gamma = eos.gamma
    else:
        tree = sedov_tree(level)
    leaves = tree.sorted_leaves()[:nleaves]
    # the reference's reflux reads the fine face-neighbours' fluxes: close the sample under that relation
    chosen = {lf.path for lf in leaves}
    grew = True
    while grew:
        grew = False
        for lf in list(leaves):
            for ax in range(3):
                for side in (-1, 1):
                    off = [0, 0, 0]
                    off[ax] = side
                    pos = tree.neighbor_ipos(lf, off)
                    if pos is None:
                        continue
                    cover = tree.find_leaf_region(lf.level, pos)
                    if cover[0][1] == "fine":
                        for child, _ in cover:
                            if child.path not in chosen:
                                chosen.add(child.path)
                                leaves.append(child)
                                grew = True
    nthr = os.cpu_count() or 1
    st = OracleStepper(tree, gamma, nthreads=nthr, **kw)
    oracle.lib()
    times = []
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        dt = st.cfl_dt(0.4)  # full-tree CFL, as the reference's step does
        st.rk3_step(dt, leaves=leaves)
        t1 = time.perf_counter()
        if k >= warmup:
            times.append(t1 - t0)
    tot = sum(times)
    value = len(leaves) * 512 * len(times) / tot
    sample = (f"{len(times)} x (cfl_dt over all {len(tree.leaves())} leaves + one RK3 step of the first "
              f"{len(leaves)} Morton-ordered leaves = {len(leaves) * 512} cells), C oracle (omb_oracle.c) "
              f"with {nthr} pthreads + numpy ghost exchange")
    return value, nthr, sample, tot / len(times)


def reference_arm(args, rank, world):
    if rank != 0:
        return
    level = resolve_level(args, world)
    # size the per-step sample so the whole run stays within ~3 minutes
    probe_v, nthr, _, _ = cpu_run(level, 8, 1, 0)
    budget = 150.0 / max(1, args.steps + args.warmup)
    nleaves = int(max(8, min(args.cpu_leaves, budget * probe_v / 512)))
    v, nthr, sample, per = cpu_run(level, nleaves, args.steps, args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (init_sedov, no RNG)",
            "config": {"workload": f"{workload_name(level, None)}, reflecting, cfl 0.4; CPU sample per step"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthr, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def fp64_peak(lib, torch):
    import ctypes

    s = torch.cuda.current_stream()
    h = ctypes.c_void_p(s.cuda_stream)
    scratch = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks = 148 * 8
    iters = 4096
    for _ in range(2):
        lib.omb_fp64_peak(scratch.data_ptr(), blocks, iters, h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        lib.omb_fp64_peak(scratch.data_ptr(), blocks, iters, h)
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    flops = reps * blocks * 256 * 8 * iters * 2.0
    return flops / sec / 1e12


def _transfer_label(st):
    if st._mapped is None:
        return "threads (host packing + DMA)"
    if st._gather_frac is None:
        return "mapped (GPU reads/writes the pinned host leaves)"
    return (f"hybrid (upload: GPU reads {st._gather_frac[0]:.0%} of the leaves from the pinned host slab, "
            "host threads pack the rest + DMA; download: DMA + host threads)")


def gpu_arm(args, rank, world):
    import gc

    import torch

    from paper_2107_10987_b200 import EosConfig, HydroMode, _lib
    from paper_2107_10987_b200.stepper import B200HydroStepper

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist = None
    if world > 1:
        import torch.distributed as dist

    # N=1: config c2 (128^3, level 4); N>1: config c3 (256^3, level 5) partitioned by leaf
    level = resolve_level(args, world)
    extra = {}
    if level == "c5":
        from octomini_host import synthetic_star

        tree, eos, grav, om, fl = synthetic_star(level=4)
        extra = dict(gravity=grav, omega=om, floors=fl)
    elif level == "c5g":
        from paper_2107_10987_b200.gravity import B200FmmSolver
        from octomini_host import synthetic_star

        tree, eos, _, om, fl = synthetic_star(level=args.level or 4)
        extra = dict(gravity=B200FmmSolver(0.5), omega=om, floors=fl)
    else:
        tree = sedov_tree(level)
        eos = EosConfig(gamma=1.4)
    part = None
    from paper_2107_10987_b200.partition import Partition

    if world > 1:
        part = Partition(tree, world, rank)
    t_prep = time.perf_counter()
    st = B200HydroStepper(tree, eos, HydroMode("new"), host_sync=False, max_run=args.max_run, partition=part,
                          **extra)
    t_prep = time.perf_counter() - t_prep
    lib = _lib.load()
    cells = st.nglobal * 512  # whole job
    local_cells = st.batch.ncompute * 512
    peak64 = fp64_peak(lib, torch)

    # warm-up (the clock sampler runs from here on)
    clk = ClockSampler(torch.cuda.current_device())
    for _ in range(args.warmup):
        st._cfl_launch(0.4)
        st.launch_step(None)
    torch.cuda.synchronize()

    K = args.steps
    acc_h = torch.empty((K, 6), dtype=torch.int64).pin_memory()
    dt_h = torch.empty((K, 1), dtype=torch.float64).pin_memory()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
          for _ in range(K)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    w_start = time.time()
    t_start.record()
    for k in range(K):
        st._cfl_launch(0.4)
        st.launch_step(None, events=ev[k])
        acc_h[k].copy_(st._acc, non_blocking=True)
        dt_h[k].copy_(st._dt, non_blocking=True)
    t_end.record()
    torch.cuda.synchronize()
    w_end = time.time()
    clocks = clk.stop(w_start, w_end)
    if dist is not None:
        dist.barrier()
    ms = t_start.elapsed_time(t_end)
    stage_ms = [a.elapsed_time(b) for row in ev for (a, b) in row]
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # the reference's mid-step CFL guard (step.py:132-139) on every timed step
    amax = acc_h[:, :3].numpy().view(np.float64)
    ratio = dt_h.numpy() * amax / st.dx_min
    aborted = bool(np.any(ratio > 1.0))
    info = {"nglobal": st.nglobal, "nruns": st.batch.nruns, "L": st.batch.L, "ncompute": st.batch.ncompute,
            "run_lengths": {int(k): int(v) for k, v in zip(*np.unique(np.diff(st.batch.run_off), return_counts=True))},
            "launches": st.native_launches_per_step()}
    fmm = None
    if level == "c5g":  # the per-stage FMM solve on its own (density + dphi/dt), CUDA events
        fs = st.gravity
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(3):
            if world > 1:  # this rank's targets; masses all-gathered
                fs.stage_fields_partitioned(st._buf[st._state], st.batch.fstride, st._info, st.batch.bc, st._grav,
                                            st._halo_tab[st._state] if st._p2p else None, dist, None)
            else:
                fs.stage_fields(st._buf[st._state], st.batch.fstride, st._info, st.batch.bc, st.batch.L, st._grav)
        f1.record()
        torch.cuda.synchronize()
        fmm_ms = f0.elapsed_time(f1) / 3
        fmm = {"stage_ms": fmm_ms, "solves_per_stage": 2, "pairs": fs.stats["pairs"], "groups": fs.stats["groups"],
               "entities": int(fs.table.nentities), "theta": fs.theta,
               "interactions_per_s": 2 * 2 * fs.stats["pairs"] / (fmm_ms / 1e3),
               "prepare_s_host": t_prep, "share_of_step": 3 * fmm_ms / (ms / K)}
        # roofline of the M2L passes (k_fmm_m2l, omb_fmm.cu): algorithmic FP64 flops per contribution
        # = 8 for a cell-cell monopole (L0..L3 += m D), 202 for a full order-3 one (L0 56, L1 78,
        # L2 48, L3 20), each pair contributing to both ends; 2 solves per stage
        if "contrib_general" in fs.stats:
            fl = 2 * (8.0 * fs.stats["contrib_cellcell"] + 202.0 * fs.stats["contrib_general"])
            fmm["roofline"] = {"bound": "fp64", "kernel": "k_fmm_m2l (+ upward/downward passes in the time)",
                               "flops_per_stage": fl, "achieved": fl / (fmm_ms / 1e3) / 1e12, "peak": peak64,
                               "unit": "TFLOP/s", "frac": fl / (fmm_ms / 1e3) / 1e12 / peak64,
                               "contrib_cellcell": fs.stats["contrib_cellcell"],
                               "contrib_general": fs.stats["contrib_general"]}
    # same-box single-GPU reference for the parallel efficiency: rank 0 steps the WHOLE
    # workload alone (same warm-up and step count, same initial state -- the host tree is
    # untouched by the host_sync=False run), the other ranks wait
    single = None
    if world > 1 and args.efficiency_steps != 0 and level in (4, 5, "c4", "c5"):
        del st
        gc.collect()
        torch.cuda.empty_cache()
        dist.barrier()
        if rank == 0:
            st1 = B200HydroStepper(tree, eos, HydroMode("new"), host_sync=False, max_run=args.max_run, **extra)
            for _ in range(args.warmup):
                st1._cfl_launch(0.4)
                st1.launch_step(None)
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            for _ in range(K):
                st1._cfl_launch(0.4)
                st1.launch_step(None)
            s1.record()
            torch.cuda.synchronize()
            ms1 = s0.elapsed_time(s1)
            single = {"value": cells * K / (ms1 / 1e3), "ms_per_step": ms1 / K, "steps": K, "warmup": args.warmup,
                      "what": "the same workload and step sequence on rank 0's GPU alone, same run"}
            del st1
            gc.collect()
            torch.cuda.empty_cache()
        dist.barrier()
        st = None
    # free the host tree and device buffers before the e2e / non-flat trees (c3 at 8 ranks:
    # 4.3 GB of host leaves per rank per tree)
    del st, tree, part
    gc.collect()
    torch.cuda.empty_cache()

    # end-to-end through the public drop-in API (host state of record, H2D + D2H every step)
    e2e = None
    if args.e2e_steps > 0:
        extra2 = {}
        if level == "c5":
            t2, _, g2, om2, fl2 = synthetic_star(level=4)
            extra2 = dict(gravity=g2, omega=om2, floors=fl2)
        elif level == "c5g":  # same topology: the FMM preparation is reused
            t2, _, _, om2, fl2 = synthetic_star(level=args.level or 4)
            extra2 = dict(gravity=extra["gravity"], omega=om2, floors=fl2)
        else:
            t2 = sedov_tree(level)
        p2 = Partition(t2, world, rank) if world > 1 else None
        st2 = B200HydroStepper(t2, eos, HydroMode("new"), host_sync=True, max_run=args.max_run, partition=p2,
                               **extra2)
        for _ in range(2):
            st2.rk3_step(st2.cfl_dt(0.4))
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            dt = st2.cfl_dt(0.4)
            st2.rk3_step(dt)
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        wall = w1 - w0
        if dist is not None:
            t = torch.tensor([wall], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall = float(t.item())
        up = 6 * st2.batch.ncompute * 512 * 8  # the owned leaves' interiors (halo leaves come from peers)
        down = 6 * st2.batch.ncompute * 512 * 8  # the owned leaves back into the host tree
        e2e = {"value": cells * args.e2e_steps / wall, "unit": UNIT,
               "h2d_bytes_per_step": up, "d2h_bytes_per_step": down + 2 * 8 + 4 + 6 * 8,
               "steps": args.e2e_steps, "api": "B200HydroStepper.cfl_dt + rk3_step (host_sync=True)",
               "transfer": _transfer_label(st2)}
        del st2, t2, p2
        gc.collect()
        torch.cuda.empty_cache()

    # the same step on a NON-FLAT state (every cell off the limiter's flat shortcut), same tree
    nontrivial = None
    if level in (4, 5) and args.e2e_steps >= 0:
        from octomini_host import smooth_state

        t3 = smooth_state(sedov_tree(level))
        p3 = Partition(t3, world, rank) if world > 1 else None
        st3 = B200HydroStepper(t3, eos, HydroMode("new"), host_sync=False, max_run=args.max_run, partition=p3)
        for _ in range(2):
            st3._cfl_launch(0.4)
            st3.launch_step(None)
        K3 = max(3, min(10, K))
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K3):
            st3._cfl_launch(0.4)
            st3.launch_step(None)
        e1.record()
        torch.cuda.synchronize()
        ms3 = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms3], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms3 = float(t.item())
        nontrivial = {"value": cells * K3 / (ms3 / 1e3), "unit": UNIT, "ms_per_step": ms3 / K3, "steps": K3,
                      "state": "smooth sinusoidal field of the reference tests (test_hydro_step.py:37-49) on the "
                               "same tree: no flat cells"}

    if rank != 0:
        return
    value = cells * K / (ms / 1e3)
    mean_stage = sum(stage_ms) / len(stage_ms)
    achieved_tf = FLOPS_PER_CELL_STAGE * local_cells / (mean_stage / 1e3) / 1e12
    pk = peaks()
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    achieved_gbs = BYTES_PER_CELL_STAGE * local_cells / (mean_stage / 1e3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "stage_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            traffic = json.load(f).get("bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong",
        "per_gpu": value / world,
        "parallel_efficiency": (value / (world * single["value"])) if single else (1.0 if world == 1 else None),
        "single_gpu": single,
        "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (init_sedov Sedov-Taylor, no RNG)",
        "config": {"workload": f"{workload_name(level, info['nglobal'])}: " + (
                       f"{info['nglobal']} sub-grids of 8^3" if SUBGRID_N == 8 else
                       f"{info['nglobal'] // (SUBGRID_N // 8) ** 3} sub-grids of {SUBGRID_N}^3 (run as "
                       f"{info['nglobal']} 8^3 blocks)") + f" = {cells} cells, "
                               "reflecting, cfl 0.4, scheme new",
                   "step": "cfl_dt + 3 fused RK stages, dt on device",
                   "l2": "working set (3 x 6 x cells x 8 B = %.0f MB) > 126 MB L2; no flush" % (3 * 48 * cells / 1e6),
                   "runs": info["nruns"], "max_run": args.max_run, "run_lengths": info["run_lengths"],
                   "parallelism": f"leaf-partitioned x{world}",
                   "halo_leaves_per_rank": int(info["L"] - info["ncompute"])},
        "roofline": {"bound": "fp64", "achieved": achieved_tf, "peak": peak64, "unit": "TFLOP/s",
                     "frac": achieved_tf / peak64, "traffic": traffic,
                     "kernel": "k_stage (fused RK stage)", "stage_ms": mean_stage,
                     "flops_per_launch": FLOPS_PER_CELL_STAGE * local_cells,
                     "peak_source": "in-run DFMA probe (omb_fp64_peak); MEASURED_PEAKS.json has no FP64 entry",
                     "hbm": {"achieved_gbs": achieved_gbs, "peak_gbs": hbm_peak, "frac": achieved_gbs / hbm_peak,
                             "algorithmic_bytes_per_launch": BYTES_PER_CELL_STAGE * local_cells}},
        "clocks": clocks,
        "e2e": e2e,
        "nontrivial_state": nontrivial,
        "gpu_launches": K * info["launches"],
        "fmm": fmm,
        "cfl_abort_in_timed_steps": aborted,
    }
    if not args.no_cpu_baseline and world == 1 and level != "c5g":
        v, nthr, sample, _ = cpu_run(level, min(args.cpu_leaves, info["L"]), 1, 0)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": nthr, "kind": "port", "sample": sample}
    emit(line)


_JSON_OUT = None


def emit(line):
    """Print the one JSON result line on the real stdout (fd 1 is pointed at stderr
    while the job runs, so NCCL's "NCCL version" banner cannot land on stdout)."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # NCCL writes its version banner to fd 1 from C; keep stdout for the single JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse()
    global SUBGRID_N
    SUBGRID_N = args.subgrid
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":  # CPU only, rank 0 alone; no collectives needed
        reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    gpu_arm(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
