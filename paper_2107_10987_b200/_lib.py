"""Loader of the in-tree CUDA library libomb200.so (include/omb200.h).

There is no fallback: if the library (or a CUDA device) is missing, every
entry point raises NativeError.  The product never imports the oracle.
"""

import ctypes
import os

from ._abi import OmbAmrDesc, OmbCflDesc, OmbRefluxDesc, OmbStageDesc
from .errors import NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("OMB_LIB_PATH") or os.path.join(_HERE, "libomb200.so")  # override: A/B experiments
ABI_VERSION = 7
_lib = None

EXPORTS = ("omb_abi_version", "omb_last_error", "omb_stage_smem_bytes", "omb_primitives", "omb_reconstruct",
           "omb_fluxes", "omb_stage", "omb_cfl", "omb_gather", "omb_gather_leaves", "omb_fp64_peak", "omb_pack_leaves", "omb_unpack_leaves", "omb_selftest_div", "omb_selftest_pow", "omb_kt_flux", "omb_physical_flux", "omb_face_flux", "omb_scalar_input", "omb_host_pack", "omb_host_unpack", "omb_host_upload", "omb_host_download", "omb_host_download_after", "omb_host_gather", "omb_host_scatter", "omb_set_host_threads", "omb_amr_ghosts",
           "omb_reflux_update", "omb_leaf_sums", "omb_disk_order",
           "omb_gather_rows", "omb_scatter_rows", "omb_enable_peer_access", "omb_ipc_alloc", "omb_ipc_open",
           "omb_fmm_traverse", "omb_fmm_build", "omb_fmm_build_direct", "omb_fmm_direct", "omb_fmm_masses", "omb_fmm_upward", "omb_fmm_m2l", "omb_fmm_m2l_part", "omb_fmm_m2l0_pair", "omb_fmm_downward",
           "omb_fmm_fields", "omb_fmm_rhodot", "omb_fmm_last_error")


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise NativeError(f"{SO_PATH} is not built (run paper_2107_10987_b200/build.py or __graft_entry__.build())")
    L = ctypes.CDLL(SO_PATH)
    vp, i, d, ll = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong
    L.omb_abi_version.restype = i
    L.omb_last_error.restype = ctypes.c_char_p
    L.omb_stage_smem_bytes.restype = i
    L.omb_primitives.argtypes = [vp, i, d, d, vp, vp]
    L.omb_reconstruct.argtypes = [vp, i, i, i, d, vp, vp, vp, vp]
    L.omb_fluxes.argtypes = [vp, vp, i, d, i, i, vp, vp, vp, vp, vp]
    L.omb_stage.argtypes = [ctypes.POINTER(OmbStageDesc), vp]
    L.omb_cfl.argtypes = [ctypes.POINTER(OmbCflDesc), vp]
    L.omb_gather.argtypes = [vp, ll, vp, i, i, vp, vp]
    L.omb_gather_leaves.argtypes = [vp, ll, vp, i, i, i, vp, vp]
    L.omb_fp64_peak.argtypes = [vp, i, i, vp]
    L.omb_pack_leaves.argtypes = [vp, ll, vp, i, vp, vp]
    L.omb_unpack_leaves.argtypes = [vp, i, vp, ll, i, vp]
    L.omb_selftest_div.argtypes = [ctypes.c_ulonglong, ll, vp, vp]
    L.omb_selftest_pow.argtypes = [vp, vp, ll, vp, vp]
    L.omb_kt_flux.argtypes = [vp, vp, i, i, d, vp, vp, vp]
    L.omb_face_flux.argtypes = [vp, i, i, vp, vp]
    L.omb_physical_flux.argtypes = [vp, i, i, vp, vp]
    L.omb_scalar_input.argtypes = [vp, ll, i, vp, i, d, d, d, vp, vp]
    L.omb_host_pack.argtypes = [vp, i, i, i, ll, vp]
    L.omb_host_unpack.argtypes = [vp, i, i, i, ll, vp]
    L.omb_host_upload.argtypes = [vp, i, i, i, ll, vp, vp, i, vp]
    L.omb_host_download.argtypes = [vp, vp, i, i, i, ll, vp, i, vp]
    L.omb_host_download_after.argtypes = [vp, vp, i, i, ll, vp, i, vp, vp, vp]
    L.omb_host_gather.argtypes = [vp, i, ll, vp, vp, vp]
    L.omb_host_scatter.argtypes = [vp, vp, i, ll, vp, vp]
    L.omb_set_host_threads.argtypes = [i]
    L.omb_amr_ghosts.argtypes = [ctypes.POINTER(OmbAmrDesc), vp]
    L.omb_leaf_sums.argtypes = [vp, ll, i, vp, vp]
    L.omb_disk_order.argtypes = [vp, ll, i, vp, vp]
    L.omb_gather_rows.argtypes = [vp, ll, vp, i, vp, vp]
    L.omb_scatter_rows.argtypes = [vp, ll, vp, i, vp, vp]
    L.omb_enable_peer_access.argtypes = [i]
    L.omb_ipc_alloc.argtypes = [ll, vp, vp]
    L.omb_ipc_open.argtypes = [vp, vp]
    L.omb_fmm_traverse.argtypes = [vp, vp, vp, vp, ll, ll, ctypes.c_double, vp, vp, vp, ll]
    L.omb_fmm_build.argtypes = [vp, vp, vp, ll, ll, vp, vp, ll, vp, vp]
    L.omb_fmm_masses.argtypes = [vp, vp, i, vp, vp, vp]
    L.omb_fmm_build_direct.argtypes = [vp, vp, ll, ll, vp, vp]
    L.omb_fmm_direct.argtypes = [vp, vp, vp, vp, vp, i, vp, vp, vp, vp, vp]
    L.omb_fmm_upward.argtypes = [vp, i, vp, vp, vp, vp]
    L.omb_fmm_m2l.argtypes = [vp, vp, vp, vp, vp, vp, ll, vp, vp, vp]
    L.omb_fmm_m2l_part.argtypes = [i, vp, vp, vp, vp, vp, vp, ll, vp, vp, vp, ll, vp]
    L.omb_fmm_m2l0_pair.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, ll, vp, vp, vp, vp, ll, vp]
    L.omb_fmm_downward.argtypes = [vp, i, vp, vp, vp, vp]
    L.omb_fmm_fields.argtypes = [vp, vp, i, vp, vp, vp, vp, vp]
    L.omb_fmm_rhodot.argtypes = [vp, ll, vp, i, i, vp, i, vp, vp]
    L.omb_reflux_update.argtypes = [ctypes.POINTER(OmbRefluxDesc), vp]
    for fn in EXPORTS[3:]:
        getattr(L, fn).restype = i
    L.omb_fmm_traverse.restype = ll
    L.omb_fmm_build.restype = ll
    L.omb_fmm_last_error.restype = ctypes.c_char_p
    if L.omb_abi_version() != ABI_VERSION:
        raise NativeError(f"libomb200.so ABI {L.omb_abi_version()} != {ABI_VERSION}")
    _lib = L
    return L


def check(rc, what):
    if rc != 0:
        L = load()
        # the FMM passes (omb_fmm.cu) keep their own thread-local message
        raw = L.omb_fmm_last_error() if what.startswith("omb_fmm") else L.omb_last_error()
        msg = (raw or b"").decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")
