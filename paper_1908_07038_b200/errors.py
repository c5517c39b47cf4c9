"""Exception tree of the drop-in (class names, bases and messages of the reference's
``spheregrid.errors``, /root/reference/pkg/src/spheregrid/errors.py:8-100).

The native library reports domain errors as ``"<ClassName>: <message>"``; ``raise_native``
maps that prefix back onto these classes so callers catch exactly what the reference
raises (SURVEY.md §8(b) "Semantics the wrappers must preserve").
"""

from __future__ import annotations


class SpheregridError(Exception):
    """Root of every library error (errors.py:8)."""


class UnknownGridName(SpheregridError):
    def __init__(self, name):
        super().__init__(f"unknown grid name: {name!r}")
        self.name = name


class NotLocated(SpheregridError):
    """A target point lies in no local source element (errors.py:92-95)."""

    def __init__(self, message, target_global_index=None):
        super().__init__(message)
        self.target_global_index = target_global_index


def _plain(name: str) -> type:
    return type(name, (SpheregridError,), {"__module__": __name__})


# grid / geometry
InvalidSpec = _plain("InvalidSpec")
IndexOutOfRange = _plain("IndexOutOfRange")
NotOnUnitSphere = _plain("NotOnUnitSphere")
# partition
InvalidDistribution = _plain("InvalidDistribution")
TooManyParts = _plain("TooManyParts")
# parallel
InvalidRank = _plain("InvalidRank")
DeadlockDetected = _plain("DeadlockDetected")
UnconsumedMessages = _plain("UnconsumedMessages")
# field
DuplicateName = _plain("DuplicateName")
AlreadyAllocated = _plain("AlreadyAllocated")
NoDevice = _plain("NoDevice")
StaleHost = _plain("StaleHost")
StaleDevice = _plain("StaleDevice")
ShapeMismatch = _plain("ShapeMismatch")
# function space
InconsistentMesh = _plain("InconsistentMesh")
PlanMismatch = _plain("PlanMismatch")
# interpolation
DegenerateTriangle = _plain("DegenerateTriangle")
# runtime
DoubleInitialise = _plain("DoubleInitialise")
# native-only failures (no reference counterpart): CUDA / NCCL errors surface as these
CudaError = _plain("CudaError")
NcclError = _plain("NcclError")

_BY_NAME = {
    cls.__name__: cls
    for cls in list(globals().values())
    if isinstance(cls, type) and issubclass(cls, SpheregridError)
}


def error_class(name: str) -> type:
    return _BY_NAME.get(name, SpheregridError)
