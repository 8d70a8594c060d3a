"""Exception types of the hydro path (reference ``pkg/src/octomini/errors.py``).

When the reference package is importable the classes derive from its own, so
``except octomini.errors.NumericsError`` in an existing caller still catches
errors raised by the B200 stepper.
"""

try:  # pragma: no cover - depends on the host having octomini installed
    from octomini import errors as _ref
except Exception:  # noqa: BLE001
    _ref = None


def _base(name, fallback):
    return getattr(_ref, name) if _ref is not None else fallback


class _OmbError(Exception):
    pass


OctominiError = _base("OctominiError", _OmbError)


class StructureError(_base("StructureError", OctominiError)):
    """Octree invariant violated (2:1 balance, uncovered region)."""


class NumericsError(_base("NumericsError", OctominiError)):
    """A numerical guard tripped: CFL abort, non-finite wave speed."""


class CapacityError(_base("CapacityError", OctominiError)):
    """Requested tree exceeds the memory budget."""


class NativeError(RuntimeError):
    """The CUDA C-ABI library returned an error code (or is missing)."""
