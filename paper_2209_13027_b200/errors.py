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


def _derive(name: str, doc: str) -> type:
    """A direct DdccanetError subclass, defined in this module (picklable, catchable by name)."""
    return type(name, (DdccanetError,), {"__doc__": doc, "__module__": __name__, "__qualname__": name})


# (name, meaning) of every concrete error, in the reference's order
ParseError = _derive("ParseError", "Input text or file content could not be parsed.")
IoError = _derive("IoError", "A file could not be found or read.")
ShapeError = _derive("ShapeError", "Array shapes / dimensions do not fit the operation (also: labels out of range).")
EmptyDatasetError = _derive("EmptyDatasetError", "No samples were provided.")
ConfigError = _derive("ConfigError", "A configuration value is invalid or inconsistent.")
RecipeError = _derive("RecipeError", "Second-view construction does not match the raw planes.")
NumericalError = _derive("NumericalError",
                         "Numerical breakdown: empty statistics, indefinite matrix, Jacobi non-convergence.")
CorruptModelError = _derive("CorruptModelError", "A stored model failed validation.")
