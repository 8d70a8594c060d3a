"""EOS helpers of octomini (pkg/src/octomini/hydro/eos.py:28-77), restated for
building synthetic inputs when octomini itself is not importable (the GPU box).
Test / bench infrastructure: the product never imports this."""

import numpy as np

from paper_2107_10987_b200.geometry import EGAS, RHO, SX, SY, SZ, TAU


def kinetic_energy(u):
    return 0.5 * (u[SX] ** 2 + u[SY] ** 2 + u[SZ] ** 2) / u[RHO]


def internal_energy(u, eos):
    e1 = u[EGAS] - kinetic_energy(u)
    return np.where(e1 >= eos.dual_energy_eta * u[EGAS], e1, u[TAU] ** eos.gamma)


def pressure(u, eos):
    return (eos.gamma - 1.0) * internal_energy(u, eos)


def sound_speed(u, eos):
    return np.sqrt(eos.gamma * pressure(u, eos) / u[RHO])


def conserved_from_primitive(rho, v, p, eos):
    parts = [np.asarray(x, dtype=np.float64) for x in (rho, v[0], v[1], v[2], p)]
    shape = np.broadcast_shapes(*(x.shape for x in parts))
    rho, vx, vy, vz, p = (np.broadcast_to(x, shape) for x in parts)
    eint = p / (eos.gamma - 1.0)
    u = np.empty((6,) + shape)
    u[RHO] = rho
    u[SX] = rho * vx
    u[SY] = rho * vy
    u[SZ] = rho * vz
    u[EGAS] = eint + 0.5 * rho * (vx ** 2 + vy ** 2 + vz ** 2)
    u[TAU] = eint ** (1.0 / eos.gamma)
    return u
