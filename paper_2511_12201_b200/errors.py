"""Exception hierarchy of the operator API.

Mirrors the reference's ``slimattn/errors.py:4-37`` class-for-class so callers
catching reference exceptions keep working. The C-ABI returns integer status
codes (``include/omnisparse.h``: ``OMNI_E_*``); :func:`raise_for_status` maps
them 1:1 onto these classes.
"""

from __future__ import annotations


class SlimAttnError(Exception):
    """Base class for all package errors (reference errors.py:4)."""


class ShapeError(SlimAttnError):
    """Operand shapes are incompatible (errors.py:8)."""


class ParameterError(SlimAttnError):
    """A scalar parameter is outside its valid range (errors.py:12)."""


class DegenerateRowError(SlimAttnError):
    """A softmax row has no unmasked cells (errors.py:16)."""


class IntegrityError(SlimAttnError):
    """Input data violates a structural contract (errors.py:20)."""


class LayoutError(SlimAttnError):
    """A token layout is inconsistent or unusable (errors.py:24)."""


class DegenerateContextError(SlimAttnError):
    """A decode step has an empty fetched KV set (errors.py:28)."""


class TensorFileError(SlimAttnError):
    """A tensor file is malformed or cannot be read (errors.py:32)."""


class WorkloadError(SlimAttnError):
    """A synthetic workload spec is infeasible (errors.py:36)."""


class CudaError(SlimAttnError):
    """The CUDA runtime reported an error inside the native library."""


# Status codes returned by every ``omni_*`` entry point (include/omnisparse.h).
STATUS_OK = 0
_STATUS_TO_EXC = {
    1: ShapeError,
    2: ParameterError,
    3: DegenerateRowError,
    4: IntegrityError,
    5: LayoutError,
    6: DegenerateContextError,
    7: CudaError,
}


def raise_for_status(code: int, what: str, detail: str = "") -> None:
    """Raise the exception class that C-ABI status ``code`` maps to."""
    if code == STATUS_OK:
        return
    exc = _STATUS_TO_EXC.get(code, SlimAttnError)
    msg = f"{what} failed with status {code}"
    if detail:
        msg += f": {detail}"
    raise exc(msg)
