"""Exceptions raised by the B200 NAR path.

Class names match the reference hierarchy (pkg/src/nar/errors.py:4-29) so
``except ConfigurationError`` written against the reference keeps working.
Status codes coming back through the C ABI are translated by
``_lib.check``: NAR_ERR_CONFIG -> ConfigurationError, NAR_ERR_INVALID ->
ValueError, NAR_ERR_NOMEM -> MemoryError, NAR_ERR_CUDA -> RuntimeError.
"""


class NarError(Exception):
    """Root of every toolkit-specific exception."""


class FormatError(NarError):
    """Container magic / version / layout not recognised."""


class CorruptError(NarError):
    """Container payload truncated or failing its checksum."""


class CapacityError(NarError):
    """A hard limit (streams, channels) would be exceeded."""


class InsufficientPointsError(NarError):
    """Too few points for the requested operation."""


class ConfigurationError(NarError):
    """Selection, channel map or network shape is inconsistent."""


class CheckpointError(NarError):
    """Weights are unreadable or do not fit the network configuration."""
