"""Host emulation of the fused CUDA stage (tests/native/emu_stage.cpp) --
runs the kernel's exact phase code under g++ to check its bookkeeping
against the oracle on machines without a GPU.  Test harness only."""

import ctypes
import os
import subprocess

import numpy as np

from paper_2107_10987_b200._abi import FLUX_SLOT_DOUBLES, OmbAmrDesc, OmbRefluxDesc, OmbStageDesc
from paper_2107_10987_b200.batch import LeafBatch
from paper_2107_10987_b200.hydro import SSP_RK3_STAGES

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.environ.get("OMB_EMU_SO") or os.path.join(HERE, "native", "_build", "libomb_emu.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        srcs = [os.path.join(HERE, "native", "emu_stage.cpp"),
                os.path.join(ROOT, "paper_2107_10987_b200", "csrc", "omb_stage.cuh"),
                os.path.join(ROOT, "paper_2107_10987_b200", "csrc", "omb_math.cuh"),
                os.path.join(ROOT, "paper_2107_10987_b200", "csrc", "omb_items.cuh"),
                os.path.join(ROOT, "paper_2107_10987_b200", "csrc", "omb_pow.cuh")]
        if not os.path.exists(SO) or os.path.getmtime(SO) < max(os.path.getmtime(s) for s in srcs):
            os.makedirs(os.path.dirname(SO), exist_ok=True)
            subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=c++17", "-o", SO, srcs[0]],
                           check=True)
        _lib = ctypes.CDLL(SO)
        _lib.emu_stage.argtypes = [ctypes.POINTER(OmbStageDesc), ctypes.c_int]
        _lib.emu_set_order.argtypes = [ctypes.c_int]
        _lib.emu_scalar_input.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_void_p]
        _lib.emu_gather.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_void_p]
        _lib.emu_amr_ghosts.argtypes = [ctypes.POINTER(OmbAmrDesc)]
        _lib.emu_reflux_update.argtypes = [ctypes.POINTER(OmbRefluxDesc)]
    return _lib


def ptr(a):
    return a.ctypes.data if a is not None else None


class EmuStepper:
    """rk3_step on packed host arrays through the emulated stage kernel."""

    def __init__(self, tree, gamma, eta=1e-3, new_mode=True, override=False, contact=False, omega=0.0,
                 grav=None, floors=(0.0, 0.0, 0.0), max_run=4, nthr=512):
        self.b = LeafBatch(tree, max_run=max_run)
        self.tree, self.gamma, self.eta = tree, gamma, eta
        self.flags = (int(new_mode), int(override), int(contact))
        self.omega, self.grav, self.floors, self.nthr = omega, grav, floors, nthr
        self.run_off = np.ascontiguousarray(self.b.run_off)
        self.run_leaf = np.ascontiguousarray(self.b.run_leaf)
        self.amax = 0.0
        self.fallback = 0

    scalars = None  # (NS, L*512): passive scalars, stepped by the scalar pass after each stage

    def rk3_step(self, dt):
        b = self.b
        U0 = np.ascontiguousarray(b.pack())
        X = None if self.scalars is None else [[np.ascontiguousarray(x.reshape(-1).copy()), np.zeros(b.fstride),
                                                np.zeros(b.fstride), np.zeros(b.fstride)] for x in self.scalars]
        if X is not None:
            for xs in X:  # stage buffers sized like a field (virtual leaves included)
                xs[0] = np.concatenate([xs[0], np.zeros(b.fstride - xs[0].size)])
        bufs = [U0, np.empty_like(U0), np.empty_like(U0), np.empty_like(U0)]
        dtv = np.array([dt])
        G = None if self.grav is None else np.ascontiguousarray(b.pack_gravity(self.grav))
        self.amax, self.fallback = 0.0, 0
        flux = np.zeros(max(1, b.flux_slots) * FLUX_SLOT_DOUBLES)
        tasks = np.ascontiguousarray(b.amr_tasks.reshape(-1))
        rleaf, roff = np.ascontiguousarray(b.reflux_leaf), np.ascontiguousarray(b.reflux_off)
        rtasks = np.ascontiguousarray(b.reflux_tasks.reshape(-1))
        cur = 0
        for s, (a, bb) in enumerate(SSP_RK3_STAGES):
            am = np.zeros(1, dtype=np.uint64)
            fb = np.zeros(1, dtype=np.uint64)
            nxt = s + 1
            if b.nvirtual:
                lib().emu_amr_ghosts(ctypes.byref(OmbAmrDesc(u=ptr(bufs[cur]), fstride=b.fstride, tasks=ptr(tasks),
                                                              ntasks=b.nvirtual)))
            d = OmbStageDesc(ucur=ptr(bufs[cur]), u0=ptr(U0), unext=ptr(bufs[nxt]), grav=ptr(G),
                             fstride=b.fstride, info=ptr(b.info), run_off=ptr(self.run_off),
                             run_leaf=ptr(self.run_leaf), nruns=b.nruns, dt=ptr(dtv), a=a, b=bb,
                             gamma=self.gamma, gm1=self.gamma - 1.0, eta=self.eta, inv_gamma=1.0 / self.gamma,
                             omega=self.omega, floor_rho=self.floors[0], floor_tau=self.floors[1],
                             floor_vmax=self.floors[2], bc=b.bc, new_mode=self.flags[0],
                             override_center=self.flags[1], contact=self.flags[2], amax_bits=ptr(am),
                             fallback=ptr(fb), flux=ptr(flux))
            rc = lib().emu_stage(ctypes.byref(d), self.nthr)
            if rc != 0:
                raise RuntimeError(f"emu_stage failed ({rc})")
            if len(rleaf):
                lib().emu_reflux_update(ctypes.byref(OmbRefluxDesc(stage=d, leaf=ptr(rleaf), off=ptr(roff),
                                                                   tasks=ptr(rtasks), nleaves=len(rleaf))))
            for xs in X or []:  # the scalar pass, as B200HydroStepper._scalar_passes
                sin = np.zeros(6 * b.fstride)
                args = (ptr(bufs[cur]), b.fstride, b.L + b.nvirtual)
                lib().emu_scalar_input(*args, ptr(xs[cur]), b.L, self.gamma, self.gamma - 1.0, self.eta, ptr(sin))
                if b.nvirtual:
                    lib().emu_amr_ghosts(ctypes.byref(OmbAmrDesc(u=ptr(sin), fstride=b.fstride, tasks=ptr(tasks),
                                                                  ntasks=b.nvirtual)))
                    lib().emu_scalar_input(*args, None, 0, self.gamma, self.gamma - 1.0, self.eta, ptr(sin))
                ds = OmbStageDesc.from_buffer_copy(d)
                dummy = np.zeros(2, dtype=np.uint64)
                ds.ucur, ds.scalar, ds.s_u0, ds.s_next = ptr(sin), 1, ptr(xs[0]), ptr(xs[nxt])
                ds.amax_bits, ds.fallback = ptr(dummy), ptr(dummy[1:])
                rc = lib().emu_stage(ctypes.byref(ds), self.nthr)
                if rc != 0:
                    raise RuntimeError(f"emu_stage (scalar) failed ({rc})")
                if len(rleaf):
                    lib().emu_reflux_update(ctypes.byref(OmbRefluxDesc(stage=ds, leaf=ptr(rleaf), off=ptr(roff),
                                                                       tasks=ptr(rtasks), nleaves=len(rleaf))))
            self.amax = max(self.amax, float(am.view(np.float64)[0]))
            self.fallback += int(fb[0])
            cur = nxt
        b.unpack(bufs[cur])
        if X is not None:
            self.scalars = np.stack([xs[cur][:b.L * 512].reshape(b.L, 8, 8, 8) for xs in X])


class EmuDistStepper:
    """Multi-rank (torch.distributed, gloo on CPU) version of EmuStepper: the
    rank's Partition batch, halo exchange with all_to_all_single between
    stages, the emulated stage kernel on the owned leaves."""

    def __init__(self, tree, gamma, world, rank, max_run=4, nthr=512):
        import torch.distributed as dist

        from paper_2107_10987_b200.partition import Partition

        self.dist = dist
        self.part = Partition(tree, world, rank)
        self.b = self.part.batch(tree, max_run=max_run)
        self.gamma = gamma
        self.nthr = nthr
        self.run_off = np.ascontiguousarray(self.b.run_off)
        self.run_leaf = np.ascontiguousarray(self.b.run_leaf)

    def _exchange(self, U):
        import torch

        from paper_2107_10987_b200.partition import exchange

        p = self.part
        per = 6 * 512
        send = np.zeros(max(1, sum(p.send_counts)) * per)
        recv = np.zeros(max(1, sum(p.recv_counts)) * per)

        def pack(state, idx, out):
            out[:len(idx) * per] = state.reshape(6, -1, 512)[:, idx].transpose(1, 0, 2).reshape(-1)

        def unpack(inp, state, first):
            n = sum(p.recv_counts)
            state.reshape(6, -1, 512)[:, first:first + n] = inp[:n * per].reshape(n, 6, 512).transpose(1, 0, 2)

        pack(U, p.send_local, send)
        st, rt = torch.from_numpy(send), torch.from_numpy(recv)
        self.dist.all_to_all_single(rt, st, [c * per for c in p.recv_counts], [c * per for c in p.send_counts])
        unpack(recv, U, p.nown)
        _ = exchange  # the product's helper is exercised on the GPU path

    def _exchange_fluxes(self, flux):
        import torch

        p = self.part
        row = FLUX_SLOT_DOUBLES
        ns, nr = sum(p.flux_send_counts), sum(p.flux_recv_counts)
        send = np.zeros(max(1, ns) * row)
        recv = np.zeros(max(1, nr) * row)
        fl = flux.reshape(-1, row)
        send[:ns * row] = fl[p.flux_send_slots].reshape(-1)
        self.dist.all_to_all_single(torch.from_numpy(recv[:nr * row]), torch.from_numpy(send[:ns * row]),
                                    [c * row for c in p.flux_recv_counts], [c * row for c in p.flux_send_counts])
        fl[p.flux_recv_slots] = recv[:nr * row].reshape(nr, row)

    scalars = None  # (NS, L*512): passive scalars, stepped by the scalar pass after each stage

    def rk3_step(self, dt):
        b = self.b
        U0 = np.ascontiguousarray(b.pack())
        X = None if self.scalars is None else [[np.ascontiguousarray(x.reshape(-1).copy()), np.zeros(b.fstride),
                                                np.zeros(b.fstride), np.zeros(b.fstride)] for x in self.scalars]
        if X is not None:
            for xs in X:  # stage buffers sized like a field (virtual leaves included)
                xs[0] = np.concatenate([xs[0], np.zeros(b.fstride - xs[0].size)])
        bufs = [U0, np.empty_like(U0), np.empty_like(U0), np.empty_like(U0)]
        dtv = np.array([dt])
        flux = np.zeros(max(1, b.flux_slots) * FLUX_SLOT_DOUBLES)
        tasks = np.ascontiguousarray(b.amr_tasks.reshape(-1))
        rleaf, roff = np.ascontiguousarray(b.reflux_leaf), np.ascontiguousarray(b.reflux_off)
        rtasks = np.ascontiguousarray(b.reflux_tasks.reshape(-1))
        self.amax = 0.0
        cur = 0
        for s, (a, bb) in enumerate(SSP_RK3_STAGES):
            self._exchange(bufs[cur])
            if b.nvirtual:
                lib().emu_amr_ghosts(ctypes.byref(OmbAmrDesc(u=ptr(bufs[cur]), fstride=b.fstride, tasks=ptr(tasks),
                                                              ntasks=b.nvirtual)))
            am = np.zeros(1, dtype=np.uint64)
            fb = np.zeros(1, dtype=np.uint64)
            nxt = s + 1
            d = OmbStageDesc(ucur=ptr(bufs[cur]), u0=ptr(U0), unext=ptr(bufs[nxt]), grav=None,
                             fstride=b.fstride, info=ptr(b.info), run_off=ptr(self.run_off),
                             run_leaf=ptr(self.run_leaf), nruns=b.nruns, dt=ptr(dtv), a=a, b=bb,
                             gamma=self.gamma, gm1=self.gamma - 1.0, eta=1e-3, inv_gamma=1.0 / self.gamma,
                             omega=0.0, floor_rho=0.0, floor_tau=0.0, floor_vmax=0.0, bc=b.bc, new_mode=1,
                             override_center=0, contact=0, amax_bits=ptr(am), fallback=ptr(fb), flux=ptr(flux))
            rc = lib().emu_stage(ctypes.byref(d), self.nthr)
            if rc != 0:
                raise RuntimeError(f"emu_stage failed ({rc})")
            if self.part.amr:
                self._exchange_fluxes(flux)
            if len(rleaf):
                lib().emu_reflux_update(ctypes.byref(OmbRefluxDesc(stage=d, leaf=ptr(rleaf), off=ptr(roff),
                                                                   tasks=ptr(rtasks), nleaves=len(rleaf))))
            for xs in X or []:  # the scalar pass, as B200HydroStepper._scalar_passes
                sin = np.zeros(6 * b.fstride)
                args = (ptr(bufs[cur]), b.fstride, b.L + b.nvirtual)
                lib().emu_scalar_input(*args, ptr(xs[cur]), b.L, self.gamma, self.gamma - 1.0, self.eta, ptr(sin))
                if b.nvirtual:
                    lib().emu_amr_ghosts(ctypes.byref(OmbAmrDesc(u=ptr(sin), fstride=b.fstride, tasks=ptr(tasks),
                                                                  ntasks=b.nvirtual)))
                    lib().emu_scalar_input(*args, None, 0, self.gamma, self.gamma - 1.0, self.eta, ptr(sin))
                ds = OmbStageDesc.from_buffer_copy(d)
                dummy = np.zeros(2, dtype=np.uint64)
                ds.ucur, ds.scalar, ds.s_u0, ds.s_next = ptr(sin), 1, ptr(xs[0]), ptr(xs[nxt])
                ds.amax_bits, ds.fallback = ptr(dummy), ptr(dummy[1:])
                rc = lib().emu_stage(ctypes.byref(ds), self.nthr)
                if rc != 0:
                    raise RuntimeError(f"emu_stage (scalar) failed ({rc})")
                if len(rleaf):
                    lib().emu_reflux_update(ctypes.byref(OmbRefluxDesc(stage=ds, leaf=ptr(rleaf), off=ptr(roff),
                                                                       tasks=ptr(rtasks), nleaves=len(rleaf))))
            self.amax = max(self.amax, float(am.view(np.float64)[0]))
            cur = nxt
        b.unpack(bufs[cur])
