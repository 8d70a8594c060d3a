"""ctypes mirror of include/omb200.h (structs only; no library loading).

Shared by the product loader (_lib.py) and the test harnesses so the struct
layouts live in one place.
"""

import ctypes

import numpy as np

c_dp = ctypes.POINTER(ctypes.c_double)
c_ip = ctypes.POINTER(ctypes.c_int)
c_u64p = ctypes.POINTER(ctypes.c_uint64)

LEAF_INFO_DTYPE = np.dtype([("nbr", "<i4", (27,)), ("offmask", "<i4"), ("ox", "<f8"), ("oy", "<f8"),
                            ("oz", "<f8"), ("dx", "<f8"), ("inv_dx", "<f8"), ("flags", "<i4"), ("slot", "<i4")],
                           align=True)
assert LEAF_INFO_DTYPE.itemsize == 160
AMR_TASK_INTS = 16
FLUX_SLOT_DOUBLES = 3 * 6 * 9 * 8 * 8  # FX, FY, FZ of one 8^3 leaf (reference flux layouts)


class OmbStageDesc(ctypes.Structure):
    _fields_ = [
        ("ucur", ctypes.c_void_p), ("u0", ctypes.c_void_p), ("unext", ctypes.c_void_p),
        ("grav", ctypes.c_void_p), ("fstride", ctypes.c_longlong), ("info", ctypes.c_void_p),
        ("run_off", ctypes.c_void_p), ("run_leaf", ctypes.c_void_p), ("nruns", ctypes.c_int),
        ("dt", ctypes.c_void_p), ("a", ctypes.c_double), ("b", ctypes.c_double),
        ("gamma", ctypes.c_double), ("gm1", ctypes.c_double), ("eta", ctypes.c_double),
        ("inv_gamma", ctypes.c_double), ("omega", ctypes.c_double),
        ("floor_rho", ctypes.c_double), ("floor_tau", ctypes.c_double), ("floor_vmax", ctypes.c_double),
        ("bc", ctypes.c_int), ("new_mode", ctypes.c_int), ("override_center", ctypes.c_int),
        ("contact", ctypes.c_int), ("amax_bits", ctypes.c_void_p), ("fallback", ctypes.c_void_p),
        ("flux", ctypes.c_void_p), ("halo", ctypes.c_void_p), ("nown", ctypes.c_int),
        ("scalar", ctypes.c_int), ("s_u0", ctypes.c_void_p), ("s_next", ctypes.c_void_p),
    ]


class OmbAmrDesc(ctypes.Structure):
    _fields_ = [
        ("u", ctypes.c_void_p), ("fstride", ctypes.c_longlong), ("tasks", ctypes.c_void_p), ("ntasks", ctypes.c_int),
    ]


class OmbRefluxDesc(ctypes.Structure):
    _fields_ = [
        ("stage", OmbStageDesc), ("leaf", ctypes.c_void_p), ("off", ctypes.c_void_p), ("tasks", ctypes.c_void_p),
        ("nleaves", ctypes.c_int),
    ]


class OmbCflDesc(ctypes.Structure):
    _fields_ = [
        ("u", ctypes.c_void_p), ("fstride", ctypes.c_longlong), ("nleaves", ctypes.c_int),
        ("dx", ctypes.c_void_p), ("gamma", ctypes.c_double), ("gm1", ctypes.c_double),
        ("eta", ctypes.c_double), ("cfl", ctypes.c_double), ("ratio", ctypes.c_void_p),
        ("bad", ctypes.c_void_p), ("out", ctypes.c_void_p), ("bad_leaf", ctypes.c_void_p),
        ("dt_dev", ctypes.c_void_p),
    ]


BC_CODES = {"outflow": 0, "reflecting": 1, "periodic": 2}
