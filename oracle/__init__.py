"""CPU oracle for the B200 hydro step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / the reference arm.  The product package never imports
it.  ``omb_oracle.c`` restates the reference's compiled kernels
(``pkg/src/octomini/_kernels/_core.pyx``); ``ghosts.py`` and ``step.py``
restate the numpy orchestration (``mesh/ghosts.py``, ``mesh/transfer.py``,
``hydro/step.py``).  Pinned bit-for-bit against goldens made by the
reference itself (``tests/golden/make_golden.py``).
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libomb_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_lp = ctypes.POINTER(ctypes.c_long)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        build()
    L = ctypes.CDLL(_SO)
    L.orc_set_face_table.argtypes = [ctypes.c_int, _ip, _ip, _ip, _ip, _ip]
    L.orc_primitives.argtypes = [_dp, ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp]
    L.orc_reconstruct.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, _dp, _dp]
    L.orc_reconstruct.restype = ctypes.c_long
    L.orc_fluxes.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp]
    L.orc_fluxes.restype = ctypes.c_double
    L.orc_leaf_speed.argtypes = [_dp, ctypes.c_int, ctypes.c_double, ctypes.c_double]
    L.orc_leaf_speed.restype = ctypes.c_double
    L.orc_update.argtypes = ([_dp] * 5 + [ctypes.c_int] + [ctypes.c_double] * 10 + [_dp]
                             + [ctypes.c_double] * 3 + [_dp])
    L.orc_stage_fluxes.argtypes = ([ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, _dp, _lp,
                                    ctypes.c_int])
    L.orc_stage_fluxes.restype = ctypes.c_int
    L.orc_max_threads.restype = ctypes.c_int
    L.orc_pow_batch.argtypes = [_dp, _dp, ctypes.c_long, _dp]
    # the face tables come from the geometry generator (reference geometry.py:51-123 semantics)
    from ._tables import flat_face_table

    for a in range(3):
        t = [np.ascontiguousarray(x, dtype=np.int32) for x in flat_face_table(a)]
        L.orc_set_face_table(a, *[x.ctypes.data_as(_ip) for x in t])
    _lib = L
    return L


def _p(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


# -- per-sub-grid kernel API (the reference's `kernels` module surface) -------

BACKEND_NAME = "oracle"


def primitives(u, gamma, eta):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    lib().orc_primitives(_p(u), u.shape[-1], gamma, eta, _p(out))
    return out


def reconstruct(prim, n, new_mode, contact_on, gamma, out_lo=None, out_hi=None):
    prim = np.ascontiguousarray(prim, dtype=np.float64)
    m = prim.shape[-1]
    lo = out_lo if out_lo is not None else np.zeros((13, 6, m, m, m))
    hi = out_hi if out_hi is not None else np.zeros((13, 6, m, m, m))
    fb = lib().orc_reconstruct(_p(prim), m, int(new_mode), int(contact_on), gamma, _p(lo), _p(hi))
    return lo, hi, int(fb)


def fluxes(lo, hi, n, gamma, new_mode, override_center):
    lo = np.ascontiguousarray(lo)
    hi = np.ascontiguousarray(hi)
    fx = np.empty((6, n + 1, n, n))
    fy = np.empty((6, n, n + 1, n))
    fz = np.empty((6, n, n, n + 1))
    amax = lib().orc_fluxes(_p(lo), _p(hi), n, gamma, int(new_mode), int(override_center), _p(fx), _p(fy), _p(fz))
    return fx, fy, fz, float(amax)


def leaf_speed(interior, gamma, eta):
    u = np.ascontiguousarray(interior, dtype=np.float64)
    return float(lib().orc_leaf_speed(_p(u), u.shape[-1], gamma, eta))


def max_threads():
    return int(lib().orc_max_threads())


def pow_batch(x, y):
    """libm pow element-wise (the host reference of the device pow self-check)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty_like(x)
    lib().orc_pow_batch(_p(x), _p(y), x.size, _p(out))
    return out
