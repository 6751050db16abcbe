"""Error taxonomy mirroring R/errors.py (exit codes 2/3/4 in the reference CLI)."""


class SplatSlamError(Exception):
    """Base class of the package's errors."""


class DataError(SplatSlamError):
    """Malformed or insufficient input data (empty map, workspace too small ...)."""


class ConfigError(SplatSlamError):
    """Invalid configuration."""


class NumericalError(SplatSlamError):
    """A device-side failure (CUDA error) or a non-finite result."""


class DomainError(SplatSlamError):
    """Arguments outside the supported domain (bad dimensions, null pointers)."""
