"""Error types and wire error codes of the reference
(/root/reference/pkg/src/swarmlm/errors.py:1-56), restated so the product has
no dependency on the reference package. Codes travel in ERROR frames as u16.
"""

from __future__ import annotations

ERR_GENERIC = 1
ERR_BUSY = 2
ERR_DESYNC = 3
ERR_UNKNOWN_SESSION = 4
ERR_UNKNOWN_TAPE = 5
ERR_BAD_REQUEST = 6
ERR_CAPACITY = 7


class SwarmError(Exception):
    """Base class (errors.py:4-5)."""


class InputError(SwarmError):
    """Malformed or out-of-contract input (errors.py:8-9)."""


class CapacityError(SwarmError):
    """A resource limit was exceeded (errors.py:12-13)."""


class ProtocolError(SwarmError):
    """Malformed bytes on the wire (errors.py:16-17)."""


class TransportError(SwarmError):
    """Connection-level failure (errors.py:20-21)."""


class TimeoutError_(SwarmError):
    """An RPC deadline elapsed (errors.py:24-25)."""


class RemoteError(SwarmError):
    """A peer replied with an ERROR frame (errors.py:28-34)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"remote error {code}: {message}")
        self.code = code
        self.message = message


class DeviceError(SwarmError):
    """The CUDA library reported a failure (ERR_GENERIC from the C-ABI)."""


def raise_for(code: int, message: str) -> None:
    """Map a C-ABI return code to the reference's exception vocabulary."""
    if code == ERR_BAD_REQUEST:
        raise InputError(message)
    if code == ERR_CAPACITY:
        raise CapacityError(message)
    if code in (ERR_BUSY, ERR_DESYNC, ERR_UNKNOWN_SESSION, ERR_UNKNOWN_TAPE):
        raise RemoteError(code, message)
    raise DeviceError(f"libpetals_b200 error {code}: {message}")
