"""Exception hierarchy of the round-attention hot path.

Same classes and the same parent/child relations as the reference
(`pkg/src/roundkv/errors.py:8-41`), so callers that catch the reference's
exceptions keep working.  The C-ABI (`include/roundkv_b200.h`) reports
failures as integer status codes; `from_status` maps them onto these
classes (see `RK_ERR_*` in the header).
"""

from __future__ import annotations


class RoundKVError(Exception):
    """Base class for all errors raised by this package (errors.py:8)."""


class InputError(RoundKVError):
    """Invalid user-supplied input (errors.py:12)."""


class ParseError(InputError):
    """Malformed conversation document (errors.py:16)."""


class TraceError(InputError):
    """Malformed attention trace (errors.py:20)."""


class ConfigError(InputError):
    """Invalid run configuration (errors.py:24)."""


class DomainError(InputError):
    """Numeric or shape argument outside its documented domain (errors.py:28)."""


class CapacityError(RoundKVError):
    """Device tier capacity exceeded (errors.py:32)."""


class ConsistencyError(RoundKVError):
    """Tiered-store misuse: duplicate block, fetch of a dropped block (errors.py:36)."""


class InvariantError(RoundKVError):
    """An internal invariant failed to hold (errors.py:40)."""


class DeviceError(RoundKVError):
    """A CUDA runtime call failed inside the native library (no reference
    counterpart: the reference never touches a device)."""


# status codes returned by every rk_* entry point (include/roundkv_b200.h)
RK_OK = 0
RK_ERR_DOMAIN = -1
RK_ERR_CAPACITY = -2
RK_ERR_CONSISTENCY = -3
RK_ERR_INVARIANT = -4
RK_ERR_CUDA = -5
RK_ERR_UNSUPPORTED = -6

_STATUS_CLASSES = {
    RK_ERR_DOMAIN: DomainError,
    RK_ERR_CAPACITY: CapacityError,
    RK_ERR_CONSISTENCY: ConsistencyError,
    RK_ERR_INVARIANT: InvariantError,
    RK_ERR_CUDA: DeviceError,
    RK_ERR_UNSUPPORTED: DomainError,
}


def from_status(status: int, message: str) -> RoundKVError:
    """Exception instance for a negative C-ABI status."""
    return _STATUS_CLASSES.get(status, RoundKVError)(message)
