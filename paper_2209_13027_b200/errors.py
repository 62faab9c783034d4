"""Exception hierarchy of the drop-in API.

Names and subclass relations mirror the reference package (errors.py:4-37)
so callers that catch ``ShapeError`` / ``ConfigError`` / ``NumericalError``
keep working. Device-side failures reach Python as C-ABI return codes
(include/ddcca.h) and are re-raised here by ``_native.check``:
DDCCA_ESHAPE -> ShapeError, DDCCA_ECONFIG -> ConfigError,
DDCCA_ENUMERICAL -> NumericalError, DDCCA_ECUDA -> _native.DeviceError.
"""

__all__ = [
    "DdccanetError", "ParseError", "IoError", "ShapeError", "EmptyDatasetError",
    "ConfigError", "RecipeError", "NumericalError", "CorruptModelError",
]


class DdccanetError(Exception):
    """Root of every error this package raises."""


class ParseError(DdccanetError):
    """Input text or file content could not be parsed."""


class IoError(DdccanetError):
    """A file could not be found or read."""


class ShapeError(DdccanetError):
    """Array shapes / dimensions do not fit the operation (also: labels out of range)."""


class EmptyDatasetError(DdccanetError):
    """No samples were provided."""


class ConfigError(DdccanetError):
    """A configuration value is invalid or inconsistent."""


class RecipeError(DdccanetError):
    """Second-view construction does not match the raw planes."""


class NumericalError(DdccanetError):
    """Numerical breakdown: empty statistics, indefinite matrix, Jacobi non-convergence."""


class CorruptModelError(DdccanetError):
    """A stored model failed validation."""
