"""B200HydroStepper -- drop-in for ``octomini.hydro.HydroStepper``.

Same constructor (``pkg/src/octomini/hydro/step.py:52-77``), same
``cfl_dt(cfl) -> float`` (:81-92), ``rk3_step(dt) -> StepStats`` (:94-102)
and ``stats`` contract, same ``NumericsError`` messages.  The step runs on
the GPU: the octree's leaves are batched once (``batch.LeafBatch``), state
lives in HBM as ``[6][L*512]`` float64, and each RK stage is ONE launch of
the fused kernel (ghost gather + primitives + reconstruction + fluxes +
quadrature + update, ``csrc/omb_stage.cuh``).

Host synchronisation follows the reference's ownership model: the host
``leaf.subgrid.interior`` arrays are the state of record.  With
``host_sync=True`` (default) ``rk3_step`` uploads the host state (unless
``cfl_dt`` just did), runs three stages and writes the result back into the
leaves, exactly where the reference leaves it.  With ``host_sync=False`` the
state stays resident on the device between calls (``download()`` /
``upload()`` move it explicitly) -- the mode benchmarks use.

The CFL-abort test of step.py:132-139 is evaluated after the three stages
from the per-stage signal speeds the kernel accumulates; on abort the state
is rolled back to the output of the last stage that passed, as the
reference leaves it when it raises.
"""

import ctypes
import operator
import os
import sys

import numpy as np

from . import _lib
from ._abi import FLUX_SLOT_DOUBLES, OmbAmrDesc, OmbCflDesc, OmbRefluxDesc, OmbStageDesc
from .batch import LeafBatch
from .device import ptr, require_cuda, stream_handle, torch
from .errors import NumericsError
from .hydro import SSP_RK3_STAGES, FloorConfig, StepStats


_SU = operator.attrgetter("subgrid._u")


class _DeviceArray:
    """A float64 device array by pointer, for torch.as_tensor (__cuda_array_interface__)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


def _on_device(fn):
    """Run a stepper method with its device current, so streams (stream_handle) and
    the library's per-device setup resolve to ``self.dev`` even when the caller's
    current device is another one."""
    import functools

    @functools.wraps(fn)
    def wrapped(self, *a, **kw):
        with torch.cuda.device(self.dev):
            return fn(self, *a, **kw)

    return wrapped


class B200HydroStepper:
    def __init__(self, tree, eos, mode, executor=None, gravity=None, omega=0.0, floors=None, abort_courant=1.0,
                 buffers=None, profiler=None, lane_pool=None, *, host_sync=True, max_run=4, device=None,
                 leaves=None, partition=None, group=None, scalars=0):
        if scalars and partition is not None:
            raise NotImplementedError("passive scalars on a partitioned tree")
        dev = require_cuda(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        with torch.cuda.device(dev):  # allocations, library setup and streams on `device`
            self._setup(tree, eos, mode, executor, gravity, omega, floors, abort_courant, buffers, profiler,
                        lane_pool, host_sync, max_run, leaves, partition, group)
            self._setup_scalars(int(scalars))

    def _setup(self, tree, eos, mode, executor, gravity, omega, floors, abort_courant, buffers, profiler, lane_pool,
               host_sync, max_run, leaves, partition, group):
        self.tree = tree
        self.eos = eos
        self.mode = mode
        self.executor = executor  # accepted for signature parity; the GPU needs no task executor
        self.gravity = gravity
        self.omega = omega
        self.floors = floors or FloorConfig()
        self.abort_courant = abort_courant
        self.buffers = buffers
        self.profiler = profiler
        self.lane_pool = lane_pool
        self.stats = StepStats()
        self.host_sync = host_sync
        self.lib = _lib.load()
        self.part = partition
        self.group = group
        if partition is not None:
            import torch.distributed as dist

            self.dist = dist
            # ranks on one host share its cores for the host-side packing
            per_host = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
            if per_host > 1:
                self.lib.omb_set_host_threads(max(1, (os.cpu_count() or 1) // per_host))
            self.batch = partition.batch(tree, max_run=max_run)
        else:
            self.dist = None
            self.batch = LeafBatch(tree, max_run=max_run, leaves=leaves)
        b = self.batch
        # the stage kernel's last CTAs made of shorter runs (half an SM count of runs split in
        # halves, twice: 4 -> 2 -> 1 leaves), so the SMs run dry closer together.  c2 Sedov:
        # 4.56 -> 4.35 ms per stage; c5 star (about uniform cost per run): +0.9 %
        # (profiles/r01_split_tail_ab.jsonl).  OMB_SPLIT_TAIL=k[,k2...] overrides, 0 = off.
        split = os.environ.get("OMB_SPLIT_TAIL")
        half = torch.cuda.get_device_properties(self.dev).multi_processor_count // 2
        b.split_tail([int(v) for v in split.split(",")] if split else [half, half])
        T = torch
        dev = self.dev
        # multi-GPU halo: uniform partitions read neighbour leaves straight from their owners'
        # buffers over NVLink (CUDA IPC, OmbStageDesc.halo); AMR partitions exchange with NCCL
        self._p2p = (partition is not None and not partition.amr
                     and os.environ.get("OMB_HALO", "p2p") == "p2p")
        if self._p2p:
            fs = T.tensor([b.fstride], dtype=T.int64, device=dev)
            self.dist.all_reduce(fs, op=self.dist.ReduceOp.MAX, group=group)
            b.fstride = int(fs.item())  # one field stride on every rank: peer addressing
        self._info = T.from_numpy(b.info.view(np.uint8).copy()).to(dev)
        self._run_off = T.from_numpy(b.run_off.copy()).to(dev)
        self._run_leaf = T.from_numpy(b.run_leaf.copy()).to(dev)
        self._dx = T.from_numpy(b.dx.copy()).to(dev)
        n = 6 * b.fstride
        # A: state / u0, B, C: stage 1, 2 outputs, D: stage 3 output
        if self._p2p:  # own allocations, shareable with the peer ranks (CUDA IPC)
            self._buf, self._ipc = [], []
            for _ in range(4):
                p_ = ctypes.c_void_p()
                h = ctypes.create_string_buffer(64)
                _lib.check(self.lib.omb_ipc_alloc(8 * n, ctypes.byref(p_), h), "omb_ipc_alloc")
                self._ipc.append(h.raw)
                self._buf.append(T.as_tensor(_DeviceArray(p_.value, n), device=dev))
        else:
            self._buf = [T.empty(n, dtype=T.float64, device=dev) for _ in range(4)]
        self._state = 0
        self._dt = T.zeros(1, dtype=T.float64, device=dev)
        self._acc = T.zeros(6, dtype=T.int64, device=dev)  # amax bits x3, fallback x3
        self._cfl_ratio = T.empty(b.L, dtype=T.float64, device=dev)
        self._cfl_bad = T.empty(b.L, dtype=T.int32, device=dev)
        self._cfl_out = T.empty(2, dtype=T.float64, device=dev)
        self._cfl_badleaf = T.empty(1, dtype=T.int32, device=dev)
        self._pinned = None  # staging buffer of the host-thread transfer path (allocated on first use)
        # AMR (coarse/fine neighbours): virtual-leaf ghost tasks, flux export slots, reflux lists
        self._amr_tasks = T.from_numpy(b.amr_tasks.reshape(-1).copy()).to(dev) if b.nvirtual else None
        self._flux = T.empty(max(1, b.flux_slots) * FLUX_SLOT_DOUBLES, dtype=T.float64, device=dev) \
            if b.flux_slots else None
        self._rleaf = T.from_numpy(b.reflux_leaf.copy()).to(dev) if len(b.reflux_leaf) else None
        self._roff = T.from_numpy(b.reflux_off.copy()).to(dev) if len(b.reflux_leaf) else None
        self._rtasks = T.from_numpy(b.reflux_tasks.reshape(-1).copy()).to(dev) if len(b.reflux_leaf) else None
        self._grav = None
        from .gravity import B200FmmSolver

        # a device FMM (gravity.B200FmmSolver) is solved on the device every stage, in place
        self._dev_gravity = isinstance(gravity, B200FmmSolver)
        if b.blocks is not None and (self._dev_gravity or (gravity is not None and
                                                            not getattr(gravity, "state_independent", False))):
            raise NotImplementedError("16^3 / 32^3 sub-grids with a state-dependent gravity solver")
        if self._dev_gravity:
            gravity.prepare(tree)
            if partition is not None:
                gravity.set_partition(partition)
            self._grav = T.zeros(4 * b.fstride, dtype=T.float64, device=dev)
        self._fresh = False  # device state was just uploaded from the host by cfl_dt
        # host_sync transfers.  "mapped": the owned leaves' arrays move into mapped pinned
        # memory that the GPU reads / writes directly (omb_host_gather/scatter) -- no host
        # thread touches the data, which pays when several ranks share the host's memory
        # bandwidth (4 ranks: 2x faster than the threads path).  "threads": the arrays stay
        # in place and host threads pack them around DMA copies.  "hybrid" (1 rank): the
        # arrays move into the mapped slab (aligned rows: host unpacking is faster there
        # too), the GPU gathers the last OMB_GATHER_FRAC of the leaves on a side stream
        # while host threads pack the rest; downloads go through the host threads.
        # OMB_HOST_XFER=mapped|threads|hybrid overrides the choice.
        self._mapped = None
        self._gather_frac = None
        xfer = os.environ.get("OMB_HOST_XFER", "auto")
        if xfer == "auto":
            xfer = "mapped" if int(os.environ.get("LOCAL_WORLD_SIZE", "1")) > 1 else "hybrid"
        if host_sync and xfer == "mapped":
            self._rehome(b.ncompute)
        elif host_sync and xfer == "hybrid":
            frac = min(1.0, max(0.0, float(os.environ.get("OMB_GATHER_FRAC", "0.1"))))
            k = b.ncompute - int(round(b.ncompute * frac))  # leaves [0, k): host threads; [k, nc): GPU
            self._rehome(b.ncompute - k)  # (the gather's stash: written, read by no scatter)
            if self._mapped is not None:
                self._gather_frac = (frac, k)
                self._xfer_stream = torch.cuda.Stream(dev)
                self._scatter_tail = os.environ.get("OMB_SCATTER_TAIL", "1") == "1"
        # the last stage is launched in parts of OMB_TAIL_WAVES waves of runs (runs sorted by
        # leaf), and each part's leaves are copied back while the next part computes: by the
        # copy engine + host threads (omb_host_download_after), or, mapped, by a scatter kernel
        # on a side stream (OMB_MAPPED_TAIL=0: one scatter after the stage); 0 = one launch
        self._tail = None
        waves = int(os.environ.get("OMB_TAIL_WAVES", "1"))
        mapped_tail = os.environ.get("OMB_MAPPED_TAIL", "1") == "1"
        if (host_sync and (self._mapped is None or mapped_tail) and waves > 0 and b.nvirtual == 0
                and self._rleaf is None and self._flux is None and not self._dev_gravity):
            part_runs = (int(os.environ.get("OMB_TAIL_RUNS", "0"))  # (tests: small parts)
                         or waves * torch.cuda.get_device_properties(dev).multi_processor_count)
            if b.nruns > part_runs:
                ro, rl, cuts, bounds = b.tail_parts(part_runs)
                self._tail = {"run_off": T.from_numpy(ro).to(dev), "run_leaf": T.from_numpy(rl).to(dev),
                              "cuts": cuts, "bounds": np.array(bounds, dtype=np.int32),
                              "events": [torch.cuda.Event() for _ in range(len(cuts) - 1)],
                              "stream": torch.cuda.Stream(dev)}
        self.dx_min = float(min(lf.subgrid.dx for lf in tree.leaves()))
        self.nglobal = partition.G if partition is not None else b.L
        if partition is not None:
            self._send_idx = T.from_numpy(partition.send_local.copy()).to(dev)
            self._sendbuf = T.empty(max(1, sum(partition.send_counts)) * 3072, dtype=T.float64, device=dev)
            self._recvbuf = T.empty(max(1, sum(partition.recv_counts)) * 3072, dtype=T.float64, device=dev)
            self._gids = partition.gids
            if self._p2p:
                ok = 1
                try:
                    self._setup_p2p()
                except Exception as e:  # noqa: BLE001 -- e.g. no peer access between the devices
                    ok = 0
                    sys.stderr.write(f"NVLink halo reads unavailable ({e}); exchanging with NCCL\n")
                flag = torch.tensor([ok], dtype=torch.int64, device=dev)
                self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=group)
                self._p2p = bool(flag.item())  # every rank takes the same path
            if partition.amr and (sum(partition.flux_send_counts) or sum(partition.flux_recv_counts)):
                self._fsend = T.from_numpy(partition.flux_send_slots.copy()).to(dev)
                self._frecv = T.from_numpy(partition.flux_recv_slots.copy()).to(dev)
                self._fsendbuf = T.empty(max(1, sum(partition.flux_send_counts)) * FLUX_SLOT_DOUBLES,
                                         dtype=T.float64, device=dev)
                self._frecvbuf = T.empty(max(1, sum(partition.flux_recv_counts)) * FLUX_SLOT_DOUBLES,
                                         dtype=T.float64, device=dev)
        self.upload()

    # -- passive scalars (species) ------------------------------------------------------
    def _setup_scalars(self, ns):
        """``scalars=NS`` passive scalars X_k (species densities; north_star / SURVEY.md §0.2):
        each follows tau's path -- PPM reconstruction, the KT flux with the hydro state's
        signal speeds, the Simpson faces, reflux, the RK update -- with no source, dual-energy
        resync or floor.  One extra pass of the fused stage kernel per scalar and stage
        (k_stage<.., 1>, on (rho, s, p, X) from omb_scalar_input).  The reference has no
        species, so the check is structural: X = rho evolves bitwise like rho
        (tests/test_gpu_scalars.py).  Device-resident: set_scalars / get_scalars."""
        self.nscalars = ns
        if ns == 0:
            return
        b = self.batch
        if b.blocks is not None:
            raise NotImplementedError("passive scalars with 16^3 / 32^3 sub-grids")
        self._sbuf = [[torch.zeros(b.fstride, dtype=torch.float64, device=self.dev) for _ in range(4)]
                      for _ in range(ns)]
        self._sin = torch.empty(6 * b.fstride, dtype=torch.float64, device=self.dev)
        self._sacc = torch.zeros(2, dtype=torch.int64, device=self.dev)  # the scalar passes' amax / fallback: unused

    @_on_device
    def set_scalars(self, values):
        """values: (NS, L, n, n, n) in sorted_leaves() order, or {leaf.path: (NS, n, n, n)}."""
        b = self.batch
        if isinstance(values, dict):
            values = np.stack([np.asarray(values[lf.path]) for lf in b.leaves[:b.L]], axis=1)
        values = np.ascontiguousarray(values, dtype=np.float64)
        if values.shape != (self.nscalars, b.L, 8, 8, 8):
            raise ValueError(f"scalars must have shape {(self.nscalars, b.L, 8, 8, 8)}")
        for k in range(self.nscalars):
            self._sbuf[k][self._state][:b.L * 512].copy_(torch.from_numpy(values[k].reshape(-1)))

    @_on_device
    def get_scalars(self):
        b = self.batch
        return np.stack([self._sbuf[k][self._state][:b.L * 512].cpu().numpy().reshape(b.L, 8, 8, 8)
                         for k in range(self.nscalars)])

    def _scalar_passes(self, d, cur, nxt, stream=None):
        """After the hydro stage described by ``d`` (input buffer index cur): every scalar's
        stage cur -> nxt, with the same stage weights, dt and signal speeds."""
        b = self.batch
        sh = stream_handle(stream)
        g = self.eos.gamma
        n_all = b.L + b.nvirtual
        for k in range(self.nscalars):
            X = self._sbuf[k]
            _lib.check(self.lib.omb_scalar_input(ptr(self._buf[cur]), b.fstride, n_all, ptr(X[cur]), b.L, g, g - 1.0,
                                                 self.eos.dual_energy_eta, ptr(self._sin), sh), "omb_scalar_input")
            if self._amr_tasks is not None:  # X's coarse/fine ghost regions; fields 0-4 redone from the state's
                ad = OmbAmrDesc(u=ptr(self._sin), fstride=b.fstride, tasks=ptr(self._amr_tasks), ntasks=b.nvirtual)
                _lib.check(self.lib.omb_amr_ghosts(ctypes.byref(ad), sh), "omb_amr_ghosts")
                _lib.check(self.lib.omb_scalar_input(ptr(self._buf[cur]), b.fstride, n_all, None, 0, g, g - 1.0,
                                                     self.eos.dual_energy_eta, ptr(self._sin), sh), "omb_scalar_input")
            ds = OmbStageDesc.from_buffer_copy(d)
            ds.run_off, ds.run_leaf, ds.nruns = ptr(self._run_off), ptr(self._run_leaf), b.nruns  # (not a tail part)
            ds.ucur = ptr(self._sin)
            ds.scalar = 1
            ds.s_u0 = ptr(X[self._state])
            ds.s_next = ptr(X[nxt])
            ds.amax_bits = self._sacc.data_ptr()
            ds.fallback = self._sacc.data_ptr() + 8
            ds.halo = None
            _lib.check(self.lib.omb_stage(ctypes.byref(ds), sh), "omb_stage (scalar)")
            if self._rleaf is not None:
                rd = OmbRefluxDesc(stage=ds, leaf=ptr(self._rleaf), off=ptr(self._roff), tasks=ptr(self._rtasks),
                                   nleaves=len(b.reflux_leaf))
                _lib.check(self.lib.omb_reflux_update(ctypes.byref(rd), sh), "omb_reflux_update (scalar)")

    # -- host <-> device -------------------------------------------------------------
    TRANSFER_CHUNKS = 8

    SPAN_STASH = 48 * 56  # ghost z + line-edge doubles per leaf of the zero-copy spans (omb_host_gather)

    def _rehome(self, stash_leaves):
        """Move the owned leaves' padded arrays (SubGrid.u) into one pinned host slab,
        mapped into the device address space, and point each SubGrid at its slot
        (values copied; the leaf's arrays stay ordinary C-contiguous float64 numpy
        arrays).  Skipped for subgrid types without the reference's ``_u`` slot.
        ``stash_leaves``: how many leaves the zero-copy kernels move per call."""
        b = self.batch
        nc = b.ncompute
        sgs = [lf.subgrid for lf in b.leaves[:nc]]
        if nc == 0 or not all(hasattr(sg, "_u") and sg.n == 8 for sg in sgs):
            return
        slab = torch.empty((nc, 6, 14, 14, 14), dtype=torch.float64, pin_memory=True)
        arr = slab.numpy()
        views = []
        for k, sg in enumerate(sgs):
            arr[k] = sg.u
            sg._u = arr[k]
            views.append(sg._u)
        base = slab.data_ptr()
        ptrs = torch.arange(nc, dtype=torch.int64) * (6 * 14 ** 3 * 8) + base
        self._mapped = {"slab": slab, "views": views, "leaves": b.leaves[:nc], "ptrs": ptrs.to(self.dev),
                        "hptrs": ptrs.numpy().astype(np.uintp),  # (fixed: _mapped_check keeps the views)
                        "stash": torch.empty(max(1, stash_leaves) * self.SPAN_STASH, dtype=torch.float64,
                                             device=self.dev)}

    def _mapped_check(self):
        """Leaves whose array was replaced since the re-homing (a user assigned a new
        SubGrid.u) are copied into their slab slot again."""
        m = self._mapped
        if all(map(operator.is_, map(_SU, m["leaves"]), m["views"])):  # (C-level loops: 32768 leaves ~2 ms)
            return
        for lf, v in zip(m["leaves"], m["views"]):
            sg = lf.subgrid
            if sg._u is not v:
                if sg._u is not None:
                    v[...] = sg._u
                sg._u = v

    @_on_device
    def upload(self):
        """Copy the host leaves' interiors into the device state.  Mapped slab: one
        kernel reads them over PCIe.  Threads: pipelined, host threads pack chunk c
        while chunk c-1 is on the copy engine.  Hybrid: both at once on disjoint
        leaf ranges.  Only owned leaves: halo leaves come from their owners every stage."""
        b = self.batch
        if self._mapped is not None:
            self._mapped_check()
            m = self._mapped
            if self._gather_frac is None:
                _lib.check(self.lib.omb_host_gather(ptr(m["ptrs"]), b.ncompute, b.fstride,
                                                    ptr(self._buf[self._state]), ptr(m["stash"]), stream_handle(None)),
                           "omb_host_gather")
                return
            k = self._gather_frac[1]
            if k < b.ncompute:  # hybrid: the GPU reads leaves [k, nc) while host threads pack [0, k)
                side, main = self._xfer_stream, torch.cuda.current_stream(self.dev)
                side.wait_stream(main)
                _lib.check(self.lib.omb_host_gather(ptr(m["ptrs"]) + 8 * k, b.ncompute - k, b.fstride,
                                                    ptr(self._buf[self._state]) + 8 * 512 * k, ptr(m["stash"]),
                                                    ctypes.c_void_p(side.cuda_stream)), "omb_host_gather")
                self._upload_threads(k)
                main.wait_stream(side)
                return
        self._upload_threads(b.ncompute)

    def _host_ptrs(self):
        """The owned leaves' host array addresses: the slab's (after _mapped_check) or
        the batch's cached table (None: not all standard arrays)."""
        if self._mapped is not None:
            return self._mapped["hptrs"]
        return self.batch._leaf_ptrs(self.batch.ncompute)

    def _upload_threads(self, count):
        b = self.batch
        if count == 0:
            return
        if self._pinned is None:
            self._pinned = torch.zeros(6 * b.fstride, dtype=torch.float64).pin_memory()
        if getattr(self, "_up_ev", None) is not None:
            self._up_ev.synchronize()  # the previous upload's copies still read the pinned buffer
        self._up_ev = torch.cuda.Event()
        ptrs = self._host_ptrs()
        if ptrs is not None:
            _lib.check(self.lib.omb_host_upload(ptrs.ctypes.data, count, 8, b.host_m, b.fstride, ptr(self._pinned),
                                                ptr(self._buf[self._state]), self.TRANSFER_CHUNKS,
                                                stream_handle(None)), "omb_host_upload")
        else:  # (not hybrid: its leaves are slab views)
            host = self._pinned.numpy().reshape(6, b.L + b.nvirtual, 8, 8, 8)
            b.pack(out=host)
            self._buf[self._state].copy_(self._pinned, non_blocking=True)
        self._up_ev.record()

    @_on_device
    def download(self, checked=False):
        """Copy the device state back into the host leaves (the owned ones).  Mapped
        slab: one kernel writes them over PCIe, then the stream is synchronised.
        Otherwise pipelined: chunk c is unpacked while chunk c+1 is in flight.
        checked: the slab views were revalidated since the last user code ran."""
        b = self.batch
        if self._mapped is not None and not checked:
            self._mapped_check()
        if self._mapped is not None and self._gather_frac is None:
            m = self._mapped
            _lib.check(self.lib.omb_host_scatter(ptr(self._buf[self._state]), ptr(m["stash"]), b.ncompute,
                                                 b.fstride, ptr(m["ptrs"]), stream_handle(None)), "omb_host_scatter")
            torch.cuda.current_stream(self.dev).synchronize()
            return
        if self._pinned is None:
            self._pinned = torch.zeros(6 * b.fstride, dtype=torch.float64).pin_memory()
        ptrs = self._host_ptrs()
        if ptrs is not None:
            _lib.check(self.lib.omb_host_download(ptr(self._buf[self._state]), ptr(self._pinned), b.ncompute, 8,
                                                  b.host_m, b.fstride, ptrs.ctypes.data, self.TRANSFER_CHUNKS,
                                                  stream_handle(None)), "omb_host_download")
            return
        self._pinned.copy_(self._buf[self._state])
        b.unpack(self._pinned.numpy().reshape(6, b.L + b.nvirtual, 8, 8, 8))

    def _download_tail(self, checked=False):
        b = self.batch
        t = self._tail
        if self._mapped is not None and self._gather_frac is None:
            # each part's final leaves are written to the mapped host slab as soon as the
            # part is done (its event), on the side stream, while later parts compute
            m = self._mapped
            side = t["stream"]
            cur = self._buf[self._state]
            st = self.SPAN_STASH
            bnd = t["bounds"]
            for k, ev in enumerate(t["events"]):
                lo, hi = int(bnd[k]), int(bnd[k + 1])
                if hi <= lo:
                    continue
                side.wait_event(ev)
                _lib.check(self.lib.omb_host_scatter(ptr(cur) + 8 * 512 * lo, ptr(m["stash"]) + 8 * st * lo, hi - lo,
                                                     b.fstride, ptr(m["ptrs"]) + 8 * lo,
                                                     ctypes.c_void_p(side.cuda_stream)), "omb_host_scatter")
            side.synchronize()
            torch.cuda.current_stream(self.dev).synchronize()
            return
        if self._mapped is not None and not checked:
            self._mapped_check()
        ptrs = self._host_ptrs()
        if ptrs is None:
            self.download(checked=True)
            return
        if self._pinned is None:
            self._pinned = torch.zeros(6 * b.fstride, dtype=torch.float64).pin_memory()
        bnd, nparts = t["bounds"], len(t["events"])
        side = None
        if self._gather_frac is not None and self._scatter_tail:
            # hybrid: the leaves the upload gathered ([k, nc), the last parts) are written back
            # by the GPU on a side stream (their stash holds this step's host ghost doubles)
            m, k, st = self._mapped, self._gather_frac[1], self.SPAN_STASH
            side = self._xfer_stream
            cur = ptr(self._buf[self._state])
            for c in range(nparts):
                lo, hi = max(int(bnd[c]), k), int(bnd[c + 1])
                if hi <= lo:
                    continue
                side.wait_event(t["events"][c])
                _lib.check(self.lib.omb_host_scatter(cur + 8 * 512 * lo, ptr(m["stash"]) + 8 * st * (lo - k), hi - lo,
                                                     b.fstride, ptr(m["ptrs"]) + 8 * lo,
                                                     ctypes.c_void_p(side.cuda_stream)), "omb_host_scatter")
            nparts = int(np.searchsorted(bnd, k, side="left"))  # parts starting below k
            bnd = np.minimum(bnd[:nparts + 1], k).astype(np.int32)
        if nparts > 0:
            ev = (ctypes.c_void_p * nparts)(*[e.cuda_event for e in t["events"][:nparts]])
            _lib.check(self.lib.omb_host_download_after(ptr(self._buf[self._state]), ptr(self._pinned), 8, b.host_m,
                                                        b.fstride, ptrs.ctypes.data, nparts, bnd.ctypes.data,
                                                        ev, ctypes.c_void_p(t["stream"].cuda_stream)),
                       "omb_host_download_after")
        if side is not None:
            side.synchronize()

    def state_tensor(self):
        return self._buf[self._state]

    # -- multi-GPU halo: NVLink peer reads ---------------------------------------------
    def _setup_p2p(self):
        """Open every rank's 4 state buffers (CUDA IPC through torch's storage sharing)
        and build, per buffer index, the table of halo-leaf addresses in their owners'
        buffers (the stage kernel reads them directly; no halo exchange)."""
        p = self.part
        world = p.world
        allh = [None] * world
        self.dist.all_gather_object(allh, self._ipc, group=self.group)
        base = [[0] * 4 for _ in range(world)]
        for r in range(world):
            for i in range(4):
                if r == p.rank:
                    base[r][i] = self._buf[i].data_ptr()
                else:
                    q = ctypes.c_void_p()
                    _lib.check(self.lib.omb_ipc_open(ctypes.create_string_buffer(allh[r][i], 64), ctypes.byref(q)),
                               "omb_ipc_open")
                    base[r][i] = q.value
        halo = np.asarray(p.halo, dtype=np.int64)
        owner = p.owner[halo]
        local = halo - np.asarray(p.bounds, dtype=np.int64)[owner]  # the owner's leaf index
        tab = np.zeros((4, max(1, len(halo))), dtype=np.uint64)
        for i in range(4):
            b_i = np.array([base[r][i] for r in range(world)], dtype=np.uint64)
            tab[i, :len(halo)] = b_i[owner] + (local * 512 * 8).astype(np.uint64)
        self._halo_tab = torch.from_numpy(tab.view(np.int64)).to(self.dev)
        self._bar = torch.zeros(1, dtype=torch.float64, device=self.dev)

    # -- multi-GPU halo exchange ------------------------------------------------------
    def _exchange(self, buf_index, stream=None):
        if self.part is None:
            return
        from .partition import exchange

        L = self.lib
        sh = stream_handle(stream)
        fs = self.batch.fstride

        def pack(state, idx, out):
            _lib.check(L.omb_pack_leaves(ptr(state), fs, ptr(idx), int(idx.numel()), ptr(out), sh), "omb_pack_leaves")

        def unpack(inp, state, first):
            n = sum(self.part.recv_counts)
            _lib.check(L.omb_unpack_leaves(ptr(inp), n, ptr(state), fs, first, sh), "omb_unpack_leaves")

        p = self.part
        exchange(self.dist, self.group, self._buf[buf_index], self._send_idx, p.send_counts, p.recv_counts, p.nown,
                 pack, unpack, self._sendbuf, self._recvbuf)

    def _exchange_fluxes(self, stream=None):
        """Second exchange of AMR multi-GPU runs: exported face fluxes of fine leaves
        whose coarse face-neighbour lives on another rank (reflux, step.py:206-241)."""
        p = self.part
        sh = stream_handle(stream)
        row = FLUX_SLOT_DOUBLES
        ns, nr = sum(p.flux_send_counts), sum(p.flux_recv_counts)
        if ns:
            _lib.check(self.lib.omb_gather_rows(ptr(self._flux), row, ptr(self._fsend), ns, ptr(self._fsendbuf), sh),
                       "omb_gather_rows")
        self.dist.all_to_all_single(self._frecvbuf[:nr * row], self._fsendbuf[:ns * row], [c * row for c in p.flux_recv_counts],
                                    [c * row for c in p.flux_send_counts], group=self.group)
        if nr:
            _lib.check(self.lib.omb_scatter_rows(ptr(self._frecvbuf), row, ptr(self._frecv), nr, ptr(self._flux), sh),
                       "omb_scatter_rows")

    # -- timestep ---------------------------------------------------------------------
    @_on_device
    def _cfl_launch(self, cfl, stream=None):
        b = self.batch
        g = self.eos.gamma
        d = OmbCflDesc(u=ptr(self._buf[self._state]), fstride=b.fstride, nleaves=b.ncompute, dx=ptr(self._dx),
                       gamma=g, gm1=g - 1.0, eta=self.eos.dual_energy_eta, cfl=float(cfl),
                       ratio=ptr(self._cfl_ratio), bad=ptr(self._cfl_bad), out=ptr(self._cfl_out),
                       bad_leaf=ptr(self._cfl_badleaf), dt_dev=ptr(self._dt))
        _lib.check(self.lib.omb_cfl(ctypes.byref(d), stream_handle(stream)), "omb_cfl")
        if self.part is not None:
            # min over ranks of (worst, cfl*worst): RN(cfl*w) is monotone in w, so this is exact
            self.dist.all_reduce(self._cfl_out, op=self.dist.ReduceOp.MIN, group=self.group)
            self._dt.copy_(self._cfl_out[1:2])

    @_on_device
    def cfl_dt(self, cfl):
        """dt = cfl * min over leaves of dx / max(max_axis|v| + c)  (step.py:81-92)."""
        if self.host_sync:
            self.upload()
            self._fresh = True
        self._cfl_launch(cfl)
        out = self._cfl_out.cpu().numpy()
        bad = int(self._cfl_badleaf.cpu().item())
        if self.part is not None:
            big = 1 << 62
            gb = torch.tensor([int(self._gids[bad]) if bad >= 0 else big], dtype=torch.int64, device=self.dev)
            self.dist.all_reduce(gb, op=self.dist.ReduceOp.MIN, group=self.group)
            g = int(gb.item())
            if g < big:
                raise NumericsError(f"non-finite wave speed on leaf {self.tree.sorted_leaves()[g].path}")
        elif bad >= 0:
            lf = self.batch.leaves[bad]
            raise NumericsError(f"non-finite wave speed on leaf {getattr(lf, 'leaf', lf).path}")
        return cfl * float(out[0])

    # -- one step -----------------------------------------------------------------------
    def _stage_desc(self, cur, nxt, s, a, bw):
        b = self.batch
        g = self.eos.gamma
        fl = self.floors
        acc = self._acc
        return OmbStageDesc(
            ucur=ptr(self._buf[cur]), u0=ptr(self._buf[self._state]), unext=ptr(self._buf[nxt]),
            grav=ptr(self._grav), fstride=b.fstride, info=ptr(self._info), run_off=ptr(self._run_off),
            run_leaf=ptr(self._run_leaf), nruns=b.nruns, dt=ptr(self._dt), a=a, b=bw, gamma=g, gm1=g - 1.0,
            eta=self.eos.dual_energy_eta, inv_gamma=1.0 / g, omega=float(self.omega),
            floor_rho=float(fl.rho), floor_tau=float(fl.tau), floor_vmax=float(fl.vmax), bc=b.bc,
            new_mode=int(self.mode.is_new), override_center=int(self.mode.quadrature_override),
            contact=int(self.mode.contact_detection), amax_bits=acc.data_ptr() + 8 * s,
            fallback=acc.data_ptr() + 8 * (3 + s), flux=ptr(self._flux))

    @_on_device
    def launch_step(self, dt=None, stream=None, events=None, tail=False):
        """Enqueue the three stages (no host sync) and advance the device state.
        dt=None uses the device dt written by the last cfl launch; tail=True
        launches the last stage in the parts of ``self._tail`` (an event after
        each).  Returns (buffer of the step-start state, [buffer of each stage's
        output])."""
        if dt is not None:
            self._dt.fill_(float(dt))
        self._acc.zero_()
        outs = []
        cur = self._state
        others = [i for i in range(4) if i != self._state]
        for s, (a, bw) in enumerate(SSP_RK3_STAGES):
            nxt = others[s]
            if self._p2p:
                # every rank has finished the previous stage (its output = this stage's input)
                # before anyone reads it; also no rank writes a buffer a peer still reads
                self.dist.all_reduce(self._bar, group=self.group)
            else:
                self._exchange(cur, stream)
            sh = stream_handle(stream)
            if self._amr_tasks is not None:
                ad = OmbAmrDesc(u=ptr(self._buf[cur]), fstride=self.batch.fstride, tasks=ptr(self._amr_tasks),
                                ntasks=self.batch.nvirtual)
                _lib.check(self.lib.omb_amr_ghosts(ctypes.byref(ad), sh), "omb_amr_ghosts")
            if self.gravity is not None and not self._dev_gravity:
                self._host_gravity(cur, stream)
            if self._dev_gravity:
                # device FMM on this stage's state (the reference's order: ghost fill, then
                # gravity, then reconstruction -- step.py:106-113)
                if self.part is not None:
                    self.gravity.stage_fields_partitioned(
                        self._buf[cur], self.batch.fstride, self._info, self.batch.bc, self._grav,
                        self._halo_tab[cur] if self._p2p else None, self.dist, self.group, stream)
                else:
                    self.gravity.stage_fields(self._buf[cur], self.batch.fstride, self._info, self.batch.bc,
                                              self.batch.L, self._grav, stream)
            d = self._stage_desc(cur, nxt, s, a, bw)
            if self._p2p:
                d.halo = self._halo_tab[cur].data_ptr()
                d.nown = self.batch.ncompute
            if events is not None:
                events[s][0].record()
            if tail and s == 2:
                t = self._tail
                cuts = t["cuts"]
                for k in range(len(cuts) - 1):
                    d.run_off = ptr(t["run_off"]) + 4 * cuts[k]
                    d.run_leaf = ptr(t["run_leaf"])
                    d.nruns = cuts[k + 1] - cuts[k]
                    _lib.check(self.lib.omb_stage(ctypes.byref(d), sh), "omb_stage")
                    t["events"][k].record(stream)
            else:
                _lib.check(self.lib.omb_stage(ctypes.byref(d), sh), "omb_stage")
            if events is not None:
                events[s][1].record()
            if getattr(self, "_fsend", None) is not None:
                self._exchange_fluxes(stream)
            if self._rleaf is not None:
                rd = OmbRefluxDesc(stage=d, leaf=ptr(self._rleaf), off=ptr(self._roff), tasks=ptr(self._rtasks),
                                   nleaves=len(self.batch.reflux_leaf))
                _lib.check(self.lib.omb_reflux_update(ctypes.byref(rd), sh), "omb_reflux_update")
            if self.nscalars:
                self._scalar_passes(d, cur, nxt, stream)
            outs.append(nxt)
            cur = nxt
        start = self._state
        self._state = outs[2]
        return start, outs

    def _host_gravity(self, cur, stream=None):
        """A host gravity object, re-solved every stage like the reference (step.py:106-113):
        the stage state with its ghosts filled (omb_gather_leaves -- the reference's
        exchange_ghosts, AMR regions included) is written into every leaf's padded
        ``SubGrid.u`` first, so solvers that read the state (e.g. octomini's FmmSolver:
        density, and rho_dot from the momentum ghosts, gravity/solver.py:134-171) see
        exactly what the reference hands them.  Objects marked ``state_independent``
        (fixed fields) skip the copy.  A field set returned again (same object) is
        uploaded only once."""
        if not getattr(self.gravity, "state_independent", False):
            if self.part is not None:
                raise NotImplementedError("a state-dependent host gravity solver needs the whole tree on one rank; "
                                          "use gravity.B200FmmSolver with a partition")
            b = self.batch
            sh = stream_handle(stream)
            n = b.L
            padded = torch.empty((n, 6, 14, 14, 14), dtype=torch.float64, device=self.dev)
            for first in range(0, n, 65535):
                k = min(65535, n - first)
                _lib.check(self.lib.omb_gather_leaves(ptr(self._buf[cur]), b.fstride, ptr(self._info), first, k,
                                                      b.bc, padded.data_ptr() + 8 * first * 6 * 14 ** 3, sh),
                           "omb_gather_leaves")
            host = padded.cpu().numpy()
            for k, lf in enumerate(b.leaves[:n]):
                lf.subgrid.u[...] = host[k]
        fields = self.gravity.solve(self.tree, need_derivative=True)
        if fields is not getattr(self, "_grav_src", None):
            self._grav = torch.from_numpy(self.batch.pack_gravity(fields).reshape(-1)).to(self.dev)
            self._grav_src = fields

    def native_launches_per_step(self):
        """Kernels of libomb200 one cfl launch + launch_step enqueue (k_cfl_leaf/reduce,
        then per stage: halo pack/unpack, AMR ghosts, k_stage, flux rows, reflux)."""
        per = 1
        p = self.part
        if p is not None:
            if not self._p2p:  # (NVLink peer reads: no pack / unpack)
                per += int(sum(p.send_counts) > 0) + int(sum(p.recv_counts) > 0)
            if getattr(self, "_fsend", None) is not None:
                per += int(sum(p.flux_send_counts) > 0) + int(sum(p.flux_recv_counts) > 0)
        per += int(self._amr_tasks is not None) + int(self._rleaf is not None)
        if self._dev_gravity:
            per += self.gravity.launches_per_stage()
        return 2 + 3 * per

    def _reduce_stats(self):
        if self.part is not None:
            self.dist.all_reduce(self._acc[:3], op=self.dist.ReduceOp.MAX, group=self.group)
            self.dist.all_reduce(self._acc[3:], op=self.dist.ReduceOp.SUM, group=self.group)

    @_on_device
    def rk3_step(self, dt):
        """One SSP-RK3 step (step.py:94-102) on the device."""
        if self.host_sync and not self._fresh:
            self.upload()  # (revalidates the slab views)
        elif self.host_sync and self._mapped is not None:
            self._mapped_check()  # leaf arrays a user replaced since cfl_dt's upload
        self._fresh = False
        tail = self.host_sync and self._tail is not None
        start, outs = self.launch_step(dt, tail=tail)
        if tail:
            self._download_tail(checked=True)  # the result, copied back while its last stage runs
        self._reduce_stats()
        acc = self._acc.cpu().numpy()
        amax = acc[:3].view(np.float64)
        fb = acc[3:]
        # the reference's logical count is per leaf of ITS tree (16^3 / 32^3 leaves run as 8^3 blocks)
        L = len(self.tree.leaves()) if self.batch.blocks is not None else self.nglobal
        stats = StepStats()
        u_prev = start
        for s in range(3):
            stats.kernel_launches += 2 * L  # the reference's logical count (step.py:128)
            stats.fallback_count += int(fb[s])
            stats.amax = max(stats.amax, float(amax[s]))
            if dt * float(amax[s]) / self.dx_min > self.abort_courant:
                self.stats = stats
                self._state = u_prev
                if self.host_sync:
                    self.download()
                raise NumericsError(
                    f"CFL violation mid-step: dt*amax/dx = {dt * float(amax[s]) / self.dx_min:.3f} "
                    f"exceeds {self.abort_courant}")
            u_prev = outs[s]
        self.stats = stats
        if self.host_sync and not tail:
            self.download(checked=True)
        return stats
