"""Executor error types, rooted in the reference's ``CollschedError``.

The reference raises for broken preconditions and returns validation
violations as data (pkg/src/collsched/errors.py:1-11).  The executor keeps
that convention: misuse (shape/dtype/size mismatches, unregistered buffers,
a schedule that fails ``validate_schedule``) raises a subclass of
``CollschedError``; device failures surface as ``DeviceError``.

When the reference package is importable its ``CollschedError`` is the base
class, so ``except collsched.CollschedError`` catches executor errors too.
"""

from __future__ import annotations

from ._refpath import import_collsched

_cs = import_collsched()
if _cs is not None:
    CollschedError = _cs.CollschedError
else:  # reference not on this machine: same name, same role

    class CollschedError(Exception):  # type: ignore[no-redef]
        """Base class for all errors raised by collsched (stand-in)."""


class ExecutorError(CollschedError):
    """Base class for errors raised by the B200 executor."""


class InvalidArgument(ExecutorError):
    """Shape, dtype, size or device mismatch on a collective call."""


class PlanError(ExecutorError):
    """A schedule could not be lowered to executor tables (malformed forest,
    or a schedule that failed ``validate_schedule``)."""

    def __init__(self, message, violations=()):
        super().__init__(message)
        self.violations = tuple(violations)


class NotRegistered(ExecutorError):
    """An output buffer was not mapped to the peers (registration missing)."""


class Unsupported(ExecutorError):
    """dtype / reduction op / topology size the executor does not handle."""


class DeviceError(ExecutorError):
    """CUDA runtime failure or a device-side flag wait that timed out."""


class NativeLibraryMissing(ExecutorError):
    """The compiled sm_100a library is absent: the executor has no fallback."""


class ReferenceMissing(ExecutorError):
    """The reference package (``collsched``) is not importable: schedules are
    parsed, generated and validated only by the reference itself."""


FC_CODES = {
    1: InvalidArgument,
    2: DeviceError,
    3: Unsupported,
    4: NotRegistered,
    5: PlanError,
    6: DeviceError,
}
