"""CPU-side checks of the C-ABI boundary: the library loads and exports every declared symbol."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ddcca.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"DDCCA_API\s+[\w\s\*]+?\b(ddcca_\w+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for need in ("ddcca_moments_partial", "ddcca_moments_tree", "ddcca_solve", "ddcca_conv", "ddcca_conv_hash",
                 "ddcca_block_hist", "ddcca_iq_expand", "ddcca_last_error"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    from paper_2209_13027_b200 import _build, _native

    lib_path = _build.build()
    lib = ctypes.CDLL(str(lib_path))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(_native.EXPORTED) == set(declared_symbols())
    h = _native.load()
    assert h.ddcca_version() >= 1
    # pure host-side queries work without a GPU
    assert h.ddcca_payload_len(25, 40) == 2 * 625 + 2 * 25 * 40 + 2 * 25 + 1 + 40
    g = _native.geom(112, 92, 5, 5)
    assert h.ddcca_moments_workspace(ctypes.byref(g), 4, 1024, 40) > 0
    assert h.ddcca_solve_workspace(49) >= 49 * 49 * 8


def test_argument_validation_maps_to_reference_errors():
    from paper_2209_13027_b200 import ConfigError, ShapeError, _native

    h = _native.load()
    with pytest.raises(ConfigError):
        _native.check(h.ddcca_block_hist(None, 1, 1, 8, 8, 17, 4, 4, 4, 4, None, 0, 1, 0, 0, None), "hist")
    with pytest.raises(ShapeError):
        _native.check(h.ddcca_block_hist(None, 1, 1, 3, 3, 4, 4, 4, 4, 4, None, 0, 1, 0, 0, None), "hist")
    g = _native.geom(3, 3, 4, 2, 1, "none")
    with pytest.raises(ShapeError):
        _native.check(h.ddcca_conv(None, 1, ctypes.byref(g), None, 1, 1, None, None), "conv")
    g = _native.geom(8, 8, 3, 3)
    with pytest.raises(ConfigError):
        _native.check(h.ddcca_conv(None, 1, ctypes.byref(g), None, 10, 1, None, None), "conv")
