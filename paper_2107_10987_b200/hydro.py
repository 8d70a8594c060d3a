"""Configuration types and host-side EOS helpers of the hydro step.

Mirrors the reference's public types so callers can swap steppers:
``EosConfig`` / ``conserved_from_primitive`` / ``kinetic_energy`` ...
(``pkg/src/octomini/hydro/eos.py:17-77``), ``HydroMode``
(``hydro/reconstruct.py:13-25``), ``FloorConfig`` / ``StepStats`` /
``SSP_RK3_STAGES`` (``hydro/step.py:20,36-46``).  These run on the host only
(initial data, diagnostics); the step itself runs in the CUDA kernels.
"""

from dataclasses import dataclass

import numpy as np

from .geometry import EGAS, RHO, SX, SY, SZ, TAU

SSP_RK3_STAGES = ((0.0, 1.0), (0.75, 0.25), (1.0 / 3.0, 2.0 / 3.0))


@dataclass(frozen=True)
class EosConfig:
    gamma: float = 5.0 / 3.0
    dual_energy_eta: float = 1.0e-3

    def __post_init__(self):
        if not self.gamma > 1.0:
            raise ValueError("gamma must exceed 1")
        if not 0.0 < self.dual_energy_eta < 1.0:
            raise ValueError("dual_energy_eta must lie in (0, 1)")


@dataclass(frozen=True)
class HydroMode:
    scheme: str = "new"
    contact_detection: bool = False
    quadrature_override: bool = False

    def __post_init__(self):
        if self.scheme not in ("old", "new"):
            raise ValueError("scheme must be 'old' or 'new'")

    @property
    def is_new(self):
        return self.scheme == "new"


@dataclass
class FloorConfig:
    rho: float = 0.0
    tau: float = 0.0
    vmax: float = 0.0


@dataclass
class StepStats:
    amax: float = 0.0
    fallback_count: int = 0
    kernel_launches: int = 0


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


class GravityField:
    """Per-leaf potential, acceleration and potential time derivative
    (gravity/solver.py:33-47); what a gravity solver's ``solve`` returns."""

    def __init__(self):
        self.per_leaf = {}

    def __getitem__(self, path):
        return self.per_leaf[path]

    def add_leaf(self, path, phi, gx, gy, gz, dphi_dt=None):
        self.per_leaf[path] = {"phi": phi, "gx": gx, "gy": gy, "gz": gz,
                               "dphi_dt": dphi_dt if dphi_dt is not None else np.zeros_like(phi)}


def momentum_divergence_source(subgrid):
    """rho_dot = -div(s) by second-order central differences over the filled
    ghosts (gravity/solver.py:156-168), same numpy expression."""
    from .geometry import GHOST

    g = GHOST
    n = subgrid.n
    u = subgrid.u
    inv2dx = 1.0 / (2.0 * subgrid.dx)
    sl = slice(g, g + n)
    return -(
        (u[SX, g + 1: g + n + 1, sl, sl] - u[SX, g - 1: g + n - 1, sl, sl])
        + (u[SY, sl, g + 1: g + n + 1, sl] - u[SY, sl, g - 1: g + n - 1, sl])
        + (u[SZ, sl, sl, g + 1: g + n + 1] - u[SZ, sl, sl, g - 1: g + n - 1])
    ) * inv2dx
