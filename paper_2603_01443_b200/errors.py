"""Error contract of the drop-in boundary.

Same hierarchy and meaning as the reference package
(`/root/reference/pkg/src/cutbench/errors.py:4-25`), plus two device-side
classes that the reference cannot raise because it never touches a GPU:
``DeviceError`` (a CUDA/NCCL call failed inside the native library) and
``NativeUnavailableError`` (the sm_100a library or a CUDA device is missing —
there is deliberately no CPU fallback, so this is raised instead).
"""


class CutbenchError(Exception):
    """Root of every error raised by this package."""


class ValidationError(CutbenchError):
    """An argument or invariant check failed; the message names the constraint."""


class UnsupportedTopologyError(ValidationError):
    """A two-qubit gate spans two segments that are not neighbours."""


class CapacityError(CutbenchError):
    """A state vector would exceed the qubit guard or the device memory."""


class DegenerateFitError(CutbenchError):
    """Kept for API parity with the reference (boundary fitting is out of scope)."""


class BudgetExceededError(CutbenchError):
    """A cooperative deadline expired between kernel launches."""


class DeviceError(CutbenchError):
    """A CUDA or NCCL call inside the native library reported an error."""


class NativeUnavailableError(CutbenchError):
    """The sm_100a library could not be loaded or no CUDA device is visible."""
