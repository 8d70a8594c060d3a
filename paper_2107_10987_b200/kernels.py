"""Per-sub-grid kernel module: the reference's ``octomini.kernels`` surface
(``pkg/src/octomini/kernels.py:33-42``) served by the CUDA library.

``primitives``, ``reconstruct`` and ``fluxes`` take and return numpy arrays
with the reference's shapes and semantics (``_kernels/_core.pyx:41-347``,
``_kernels/reference.py:30-45``) so existing callers -- and the reference's
own backend-parity tests (``tests/test_backends.py``) -- can point
``compiled`` at this module.  Arrays are copied host->device, the sm_100a
kernel runs, results are copied back.  No CPU fallback: without the library
or a GPU every call raises NativeError.
"""

import numpy as np

from . import _lib
from .device import ptr, require_cuda, stream_handle, to_device, torch

BACKEND_NAME = "b200"


def _dev():
    return require_cuda()


def primitives(u, gamma, eta):
    dev = _dev()
    u = np.asarray(u, dtype=np.float64)
    m = u.shape[-1]
    du = to_device(u, dev)
    out = torch.empty_like(du)
    _lib.check(_lib.load().omb_primitives(ptr(du), m, float(gamma), float(eta), ptr(out), stream_handle()),
               "omb_primitives")
    return out.cpu().numpy()


def reconstruct(prim, n, new_mode, contact_on, gamma, out_lo=None, out_hi=None):
    dev = _dev()
    prim = np.asarray(prim, dtype=np.float64)
    m = prim.shape[-1]
    dp = to_device(prim, dev)
    shape = (13, 6, m, m, m)
    # fresh outputs are zero outside the written core, like the reference's np.zeros
    lo = torch.zeros(shape, dtype=torch.float64, device=dev) if out_lo is None else to_device(out_lo, dev)
    hi = torch.zeros(shape, dtype=torch.float64, device=dev) if out_hi is None else to_device(out_hi, dev)
    fb = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().omb_reconstruct(ptr(dp), m, int(bool(new_mode)), int(bool(contact_on)), float(gamma),
                                           ptr(lo), ptr(hi), ptr(fb), stream_handle()), "omb_reconstruct")
    lo_h, hi_h = lo.cpu().numpy(), hi.cpu().numpy()
    if out_lo is not None:
        out_lo[...] = lo_h
        lo_h = out_lo
    if out_hi is not None:
        out_hi[...] = hi_h
        hi_h = out_hi
    return lo_h, hi_h, int(fb.item())


def fluxes(lo, hi, n, gamma, new_mode, override_center):
    dev = _dev()
    dlo = to_device(lo, dev)
    dhi = to_device(hi, dev)
    fx = torch.empty((6, n + 1, n, n), dtype=torch.float64, device=dev)
    fy = torch.empty((6, n, n + 1, n), dtype=torch.float64, device=dev)
    fz = torch.empty((6, n, n, n + 1), dtype=torch.float64, device=dev)
    am = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().omb_fluxes(ptr(dlo), ptr(dhi), int(n), float(gamma), int(bool(new_mode)),
                                      int(bool(override_center)), ptr(fx), ptr(fy), ptr(fz), ptr(am),
                                      stream_handle()), "omb_fluxes")
    amax = float(am.cpu().numpy().view(np.float64)[0])
    return fx.cpu().numpy(), fy.cpu().numpy(), fz.cpu().numpy(), amax
