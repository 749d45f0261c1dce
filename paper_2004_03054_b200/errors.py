"""Exception tree of the drop-in, mirroring the reference's ``luda.errors``.

Reference: ``pkg/src/luda/errors.py:4-46``. Class names, the inheritance shape
(``CorruptionError`` is a ``FormatError``; ``CapacityError`` is a
``DeviceError``) and ``CorruptionError.offset`` are kept so that callers written
against the reference catch the same things from the B200 backend.

Native status codes returned through the C ABI (``include/luda_b200.h``) map
onto these classes in :func:`from_status`.
"""


class LudaError(Exception):
    """Base class for every error raised by the compaction path."""


class FormatError(LudaError):
    """Malformed or truncated on-disk structure (footer, filter, index, block)."""


class CorruptionError(FormatError):
    """Checksum mismatch; ``offset`` is the damaged block's offset in its file."""

    def __init__(self, message, offset=None):
        if offset is not None:
            message = f"{message} (block offset {offset})"
        super().__init__(message)
        self.offset = offset


class OrderingError(LudaError):
    """Keys violate the internal-key order (unsorted input run)."""


class SizeOverflowError(LudaError):
    """Payload exceeds a configured size limit; the caller must split."""


class StoreClosedError(LudaError):
    """Operation on a closed store (kept for interface parity)."""


class WriteStalled(LudaError):
    """Level-0 backlog stall (kept for interface parity)."""


class DeviceError(LudaError):
    """Failure inside the offload device backend."""


class CapacityError(DeviceError):
    """Device region allocation exceeded the configured capacity."""


class UnsupportedInputError(DeviceError):
    """Input is valid for the reference but outside this backend's fast-path
    envelope (e.g. user keys of differing lengths inside one job)."""


# Status codes of the C ABI (include/luda_b200.h: enum luda_status).
STATUS_OK = 0
STATUS_CORRUPT = 1
STATUS_FORMAT = 2
STATUS_CAPACITY = 3
STATUS_ORDERING = 4
STATUS_DEVICE = 5
STATUS_UNSUPPORTED = 6


def from_status(status: int, message: str, offset=None) -> LudaError:
    """Map a native status code to the reference exception class."""
    if status == STATUS_CORRUPT:
        return CorruptionError(message, offset=offset)
    if status == STATUS_FORMAT:
        return FormatError(message)
    if status == STATUS_CAPACITY:
        return CapacityError(message)
    if status == STATUS_ORDERING:
        return OrderingError(message)
    if status == STATUS_UNSUPPORTED:
        return UnsupportedInputError(message)
    return DeviceError(message)
