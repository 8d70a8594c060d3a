"""Oracle restatement of the tree-level SSP-RK3 step -- TEST INFRASTRUCTURE ONLY.

Follows reference ``pkg/src/octomini/hydro/step.py:20-288``: per stage ghost
exchange -> (primitives, reconstruct, fluxes per leaf) -> reflux -> CFL
abort check -> update (+ sources, dual-energy resync, floors).  The per-leaf
kernels are the C restatement in ``omb_oracle.c`` (pthreads over leaves);
this file is the orchestration, operating on the host tree in place like
the reference does.
"""

import ctypes

import numpy as np

from . import _p, leaf_speed, lib
from .ghosts import exchange

RK3 = ((0.0, 1.0), (0.75, 0.25), (1.0 / 3.0, 2.0 / 3.0))


class OracleNumericsError(Exception):
    pass


class OracleStepper:
    def __init__(self, tree, gamma, eta=1e-3, new_mode=True, contact=False, override=False,
                 omega=0.0, gravity=None, floors=(0.0, 0.0, 0.0), abort_courant=1.0, nthreads=0,
                 error_cls=OracleNumericsError):
        self.tree, self.gamma, self.eta = tree, gamma, eta
        self.new_mode, self.contact, self.override = new_mode, contact, override
        self.omega, self.gravity, self.floors = omega, gravity, floors
        self.abort_courant, self.nthreads = abort_courant, nthreads
        self.error_cls = error_cls
        self.amax = 0.0
        self.fallback = 0
        self.kernel_launches = 0

    # step.py:81-92
    def cfl_dt(self, cfl):
        worst = np.inf
        for lf in self.tree.sorted_leaves():
            s = leaf_speed(lf.subgrid.interior, self.gamma, self.eta)
            if not np.isfinite(s):
                raise self.error_cls(f"non-finite wave speed on leaf {lf.path}")
            worst = min(worst, lf.subgrid.dx / s)
        return cfl * worst

    def rk3_step(self, dt, leaves=None):
        """One step.  ``leaves`` restricts the work to a subset (bench sampling:
        the other leaves only provide ghost data and are not advanced)."""
        self.amax, self.fallback, self.kernel_launches = 0.0, 0, 0
        work = leaves if leaves is not None else self.tree.sorted_leaves()
        u0 = {lf.path: lf.subgrid.interior.copy() for lf in work}
        for a, b in RK3:
            self._stage(work, u0, dt, a, b)

    def _stage(self, leaves, u0, dt, a, b):
        exchange(self.tree, leaves)
        fields = self.gravity.solve(self.tree, need_derivative=True) if self.gravity is not None else None
        L = len(leaves)
        n = self.tree.n
        m = n + 6
        U = np.empty((L, 6, m, m, m))
        for i, lf in enumerate(leaves):
            U[i] = lf.subgrid.u
        FX = np.empty((L, 6, n + 1, n, n))
        FY = np.empty((L, 6, n, n + 1, n))
        FZ = np.empty((L, 6, n, n, n + 1))
        am = np.empty(L)
        fb = np.empty(L, dtype=np.int64)
        rc = lib().orc_stage_fluxes(L, n, _p(U), self.gamma, self.eta, int(self.new_mode), int(self.contact),
                                    int(self.override), _p(FX), _p(FY), _p(FZ), _p(am),
                                    fb.ctypes.data_as(ctypes.POINTER(ctypes.c_long)), self.nthreads)
        if rc != 0:
            raise RuntimeError(f"oracle stage failed: {rc}")
        self.kernel_launches += 2 * L
        self.fallback += int(fb.sum())
        store = {lf.path: [FX[i], FY[i], FZ[i]] for i, lf in enumerate(leaves)}
        self._reflux(leaves, store)
        amax = float(np.max(am)) if L else 0.0
        self.amax = max(self.amax, amax)
        dxmin = min(lf.subgrid.dx for lf in leaves)
        if dt * amax / dxmin > self.abort_courant:
            raise self.error_cls(f"CFL violation mid-step: dt*amax/dx = {dt * amax / dxmin:.3f} "
                                 f"exceeds {self.abort_courant}")
        fr, ft, fv = self.floors
        for i, lf in enumerate(leaves):
            sg = lf.subgrid
            cur = np.ascontiguousarray(sg.interior)
            out = np.empty_like(cur)
            g = None
            if fields is not None:
                f = fields[lf.path]
                g = np.ascontiguousarray(np.stack([f["gx"], f["gy"], f["gz"], f["dphi_dt"]]), dtype=np.float64)
            fx, fy, fz = (np.ascontiguousarray(x) for x in store[lf.path])
            lib().orc_update(_p(cur), _p(np.ascontiguousarray(u0[lf.path])), _p(fx), _p(fy), _p(fz), n,
                             dt, a, b, 1.0 / sg.dx, self.gamma, self.eta, self.omega,
                             float(sg.origin[0]), float(sg.origin[1]), sg.dx,
                             _p(g) if g is not None else None, fr, ft, fv, _p(out))
            sg.interior[:] = out

    # step.py:206-241
    def _reflux(self, leaves, store):
        tree = self.tree
        n = tree.n
        inset = {lf.path for lf in leaves}
        for lf in leaves:
            for ax in range(3):
                for side in (-1, 1):
                    off = [0, 0, 0]
                    off[ax] = side
                    pos = tree.neighbor_ipos(lf, off)
                    if pos is None:
                        continue
                    cover = tree.find_leaf_region(lf.level, pos)
                    if cover[0][1] != "fine":
                        continue
                    F = store[lf.path][ax]
                    t1, t2 = [x for x in range(3) if x != ax]
                    for child, _ in cover:
                        k = [int(child.ipos[x]) & 1 for x in range(3)]
                        if k[ax] != (0 if side > 0 else 1):
                            continue
                        if child.path not in inset:
                            raise RuntimeError("reflux needs every fine neighbour in the working set")
                        cf = store[child.path][ax]
                        sl = [slice(None)] * 4
                        sl[1 + ax] = 0 if side > 0 else n
                        fine = cf[tuple(sl)]
                        red = 0.25 * ((fine[:, 0::2, 0::2] + fine[:, 1::2, 0::2])
                                      + (fine[:, 0::2, 1::2] + fine[:, 1::2, 1::2]))
                        dst = [slice(None)] * 4
                        dst[1 + ax] = n if side > 0 else 0
                        dst[1 + t1] = slice(k[t1] * n // 2, (k[t1] + 1) * n // 2)
                        dst[1 + t2] = slice(k[t2] * n // 2, (k[t2] + 1) * n // 2)
                        F[tuple(dst)] = red
