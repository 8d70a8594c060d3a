"""Configuration and statistics types of the hydro step (the schema the
drop-in shares with the reference): ``EosConfig`` (``pkg/src/octomini/hydro/eos.py:17-25``),
``HydroMode`` (``hydro/reconstruct.py:13-25``), ``FloorConfig`` / ``StepStats`` /
``SSP_RK3_STAGES`` (``hydro/step.py:20,36-46``).  The reference's own objects
work as well (duck-typed: ``gamma``, ``dual_energy_eta``, ``is_new`` ...).
"""

from dataclasses import dataclass

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
