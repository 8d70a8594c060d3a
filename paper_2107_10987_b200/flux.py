"""Point-flux surface of ``octomini.hydro.flux`` on the device.

``kt_flux(left, right, axis, eos)`` and ``physical_flux(state, axis)``
(``pkg/src/octomini/hydro/flux.py:40-67``) take point states with the
reference's ``PrimitiveState`` attributes (``rho, vx, vy, vz, p, eint, tau``;
any object that has them), and ``face_flux(point_fluxes, new_mode)``
(``flux.py:70-91``) the 9 quadrature-point fluxes of a face.  Each call runs
the sm_100a kernels behind ``omb_kt_flux`` / ``omb_face_flux``; the batched
forms ``kt_flux_batch`` / ``face_flux_batch`` take arrays of many points.
Same arithmetic as the reference (bitwise), same ``NumericsError`` on a
non-finite state.  No CPU fallback.
"""

import numpy as np

from . import _lib
from .device import ptr, require_cuda, stream_handle, torch
from .errors import NumericsError

STATE_FIELDS = ("rho", "vx", "vy", "vz", "p", "eint", "tau")


def _pack(states):
    return np.array([[float(getattr(s, k)) for k in STATE_FIELDS] for s in states], dtype=np.float64)


def kt_flux_batch(left, right, axis, gamma):
    """left, right: (n, 7) arrays of (rho, vx, vy, vz, p, eint, tau) -> (n, 6) fluxes."""
    dev = require_cuda()
    L = torch.from_numpy(np.ascontiguousarray(left, dtype=np.float64)).to(dev)
    R = torch.from_numpy(np.ascontiguousarray(right, dtype=np.float64)).to(dev)
    n = L.shape[0]
    out = torch.empty((n, 6), dtype=torch.float64, device=dev)
    bad = torch.full((1,), n, dtype=torch.int32, device=dev)
    _lib.check(_lib.load().omb_kt_flux(ptr(L), ptr(R), n, int(axis), float(gamma), ptr(out), ptr(bad),
                                       stream_handle()), "omb_kt_flux")
    if int(bad.item()) < n:
        raise NumericsError("non-finite state passed to kt_flux")
    return out.cpu().numpy()


def kt_flux(left, right, axis, eos):
    """flux.py:50-67 for one pair of point states."""
    return kt_flux_batch(_pack([left]), _pack([right]), axis, eos.gamma)[0]


def physical_flux(state, axis):
    """flux.py:40-47: the exact Euler flux of one point state along ``axis``."""
    dev = require_cuda()
    S = torch.from_numpy(_pack([state])).to(dev)
    out = torch.empty((1, 6), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().omb_physical_flux(ptr(S), 1, int(axis), ptr(out), stream_handle()), "omb_physical_flux")
    return out.cpu().numpy()[0]


def face_flux_batch(points, new_mode=True):
    """points: (n, 9, 6) -> (n, 6), flux.py:70-91 for each face."""
    dev = require_cuda()
    P = torch.from_numpy(np.ascontiguousarray(points, dtype=np.float64)).to(dev)
    if P.ndim != 3 or P.shape[1] != 9 or P.shape[2] != 6:
        raise ValueError("face_flux expects 9 point fluxes")
    n = P.shape[0]
    out = torch.empty((n, 6), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().omb_face_flux(ptr(P), n, int(bool(new_mode)), ptr(out), stream_handle()),
               "omb_face_flux")
    return out.cpu().numpy()


def face_flux(point_fluxes, new_mode=True):
    pf = np.asarray(point_fluxes, dtype=np.float64)
    if pf.shape[0] != 9:
        raise ValueError("face_flux expects 9 point fluxes")
    return face_flux_batch(pf[None], new_mode)[0]
