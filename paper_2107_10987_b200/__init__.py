"""B200-native FP64 hydro step (reconstruct -> KT flux -> RK3 update -> CFL dt)
of octomini / Octo-Tiger's hydro module (arXiv 2107.10987), behind the
reference's HydroStepper and per-sub-grid kernel API.

Host side is Python; the compute runs in hand-written sm_100a CUDA kernels
(libomb200.so, C ABI in include/omb200.h).  PyTorch provides device memory
and streams only.  The octree, its initial data and checkpoint reader are the
caller's (octomini's own ``mesh`` / ``problems``): the stepper consumes any
tree with octomini's interface.
"""

from .errors import NativeError, NumericsError, StructureError  # noqa: F401
from .hydro import SSP_RK3_STAGES, EosConfig, FloorConfig, HydroMode, StepStats  # noqa: F401

__version__ = "0.1.0"


def HydroStepper(*args, **kwargs):  # noqa: N802 - mirrors the reference's class name
    """Construct the B200 stepper (same signature as octomini's HydroStepper)."""
    from .stepper import B200HydroStepper

    return B200HydroStepper(*args, **kwargs)
