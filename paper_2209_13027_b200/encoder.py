"""Binary hashing and information-quality (IQ) block-histogram features.

API mirror of encoder.py:21-144 of the reference. On the transform path the
hash is fused into the last layer's conv (ddcca_conv_hash) and histograms
are built by ddcca_block_hist; the functions below expose the same device
kernels for callers that already hold final-layer maps.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from . import engine as E
from .errors import ConfigError, ShapeError

ZERO_BIN_POLICIES = ("zero", "floor")


@dataclass(frozen=True)
class EncoderConfig:
    """Block size, overlap, empty-bin policy (encoder.py:21-47)."""

    block_h: int
    block_w: int
    overlap: float = 0.0
    zero_bin_policy: str = "zero"

    def __post_init__(self):
        if self.block_h < 1 or self.block_w < 1:
            raise ConfigError(f"block size {self.block_h}x{self.block_w} must be >= 1x1")
        if not 0.0 <= self.overlap < 1.0:
            raise ConfigError(f"overlap ratio {self.overlap} outside [0, 1)")
        if self.zero_bin_policy not in ZERO_BIN_POLICIES:
            raise ConfigError(f"zero bin policy {self.zero_bin_policy!r} not one of {ZERO_BIN_POLICIES}")

    def block_starts(self, p: int, q: int) -> list[tuple[int, int]]:
        """Top-left block corners, row-major, partial blocks dropped (Python banker's round)."""
        sh = max(1, int(round((1.0 - self.overlap) * self.block_h)))
        sw = max(1, int(round((1.0 - self.overlap) * self.block_w)))
        return [(i, j) for i in range(0, p - self.block_h + 1, sh) for j in range(0, q - self.block_w + 1, sw)]

    def block_count(self, p: int, q: int) -> int:
        return len(self.block_starts(p, q))


@dataclass(frozen=True)
class FeatureVector:
    """Two-view feature with the view boundary (encoder.py:102-115)."""

    values: np.ndarray
    view_boundary: int

    @property
    def view1(self) -> np.ndarray:
        return self.values[: self.view_boundary]

    @property
    def view2(self) -> np.ndarray:
        return self.values[self.view_boundary:]


def _ex(executor):
    from .execution import Executor

    return executor if executor is not None and hasattr(executor, "stream") else Executor()


def _hash_dev(ex, maps_dev, n_bits: int):
    """(G*n_bits, p, q) float32 device -> (G, p, q) codes."""
    import torch

    lib = _native.load()
    n, p, q = maps_dev.shape
    groups = n // n_bits
    codes = torch.empty((groups, p, q), dtype=torch.uint8 if n_bits <= 8 else torch.int16, device=ex.device)
    _native.check(lib.ddcca_sign_hash(_native.ptr(maps_dev), groups, n_bits, p * q, _native.ptr(codes),
                                      _native.stream_ptr(ex.stream)), "hash_combine")
    return codes


def binarize(plane, executor=None) -> np.ndarray:
    """1 where strictly positive, else 0 (encoder.py:50-52); device sign kernel."""
    a = np.asarray(plane)
    flat = a.reshape(1, 1, -1) if a.ndim else a.reshape(1, 1, 1)
    return hash_combine(flat, executor).reshape(a.shape).astype(np.int64)


def hash_combine(bitmaps, executor=None) -> np.ndarray:
    """sum_l 2^l * (map_l > 0), first map = LSB (encoder.py:55-68); device kernel.

    Inputs are sign maps or raw responses (only their sign matters, exactly
    as hash_combine(binarize(...)) in the reference).
    """
    import torch

    st = np.asarray(bitmaps)
    if st.ndim != 3:
        raise ShapeError(f"expected a list of 2-D bit maps, got shape {st.shape}")
    nb = st.shape[0]
    if not 1 <= nb <= 30:
        raise ConfigError(f"can combine 1..30 bit maps, got {nb}")
    if nb > 16:
        raise ConfigError(f"device hashing supports up to 16 bit maps, got {nb}")
    ex = _ex(executor)
    with torch.cuda.stream(ex.stream):
        dev = torch.from_numpy(np.ascontiguousarray(st.astype(np.float32))).to(ex.device)
        codes = _hash_dev(ex, dev, nb)
        out = codes.cpu().numpy()
    if out.dtype == np.int16:
        out = out.view(np.uint16)
    return out[0].astype(np.int64)


def _encode_dev(ex, maps_dev, n_bits: int, cfg: EncoderConfig):
    """(n_maps, p, q) device responses of one view -> float64 features on device."""
    import torch

    lib = _native.load()
    n, p, q = maps_dev.shape
    if n % n_bits:
        raise ShapeError(f"{n} maps not divisible into groups of {n_bits}")
    plan = E.block_plan(cfg, p, q, n_bits)
    groups = n // n_bits
    codes = _hash_dev(ex, maps_dev, n_bits)
    kind = E.count_kind(plan.bpc)
    counts = torch.empty(groups * plan.blocks * plan.bins, dtype=torch.int16 if kind == 2 else torch.uint8,
                         device=ex.device)
    _native.check(lib.ddcca_block_hist(_native.ptr(codes), codes.element_size(), groups, p, q, n_bits, plan.bh,
                                       plan.bw, plan.sh, plan.sw, _native.ptr(counts), kind, 1,
                                       plan.blocks * plan.bins, 0, _native.stream_ptr(ex.stream)), "block_hist")
    return E.Engine(ex).expand(counts, plan, cfg)


def iq_block_features(q_map, cfg: EncoderConfig, n_bits: int, executor=None) -> np.ndarray:
    """Per-block -log p features of one code map (encoder.py:71-99)."""
    import torch

    qm = np.asarray(q_map)
    if qm.ndim != 2:
        raise ShapeError(f"expected a 2-D code map, got shape {qm.shape}")
    p, q = qm.shape
    if not cfg.block_starts(p, q):
        raise ShapeError(f"{cfg.block_h}x{cfg.block_w} blocks do not fit a {p}x{q} map")
    if qm.size and (qm.min() < 0 or qm.max() >= (1 << n_bits)):
        raise ShapeError(f"code {int(qm.max())} exceeds {n_bits}-bit range")
    # decompose codes into sign planes and reuse the device hash + histogram path
    planes = ((qm[None, :, :] >> np.arange(n_bits)[:, None, None]) & 1).astype(np.float32)
    ex = _ex(executor)
    with torch.cuda.stream(ex.stream):
        out = _encode_dev(ex, torch.from_numpy(np.ascontiguousarray(planes)).to(ex.device), n_bits, cfg)
        return out.cpu().numpy()


def encode_view(maps, n_bits: int, cfg: EncoderConfig, executor=None) -> np.ndarray:
    """Hash-pool groups of n_bits maps and encode each (encoder.py:118-131)."""
    import torch

    a = np.asarray(maps)
    if a.ndim != 3:
        raise ShapeError(f"expected (n_maps, p, q) maps, got shape {a.shape}")
    if a.shape[0] % n_bits:
        raise ShapeError(f"{a.shape[0]} maps not divisible into groups of {n_bits}")
    if not 1 <= n_bits <= 16:
        raise ConfigError(f"device hashing supports 1..16 bit maps, got {n_bits}")
    ex = _ex(executor)
    with torch.cuda.stream(ex.stream):
        dev = torch.from_numpy(np.ascontiguousarray(a.astype(np.float32))).to(ex.device)
        return _encode_dev(ex, dev, n_bits, cfg).cpu().numpy()


def encode_sample(maps1, maps2, n_bits: int, cfg: EncoderConfig, executor=None) -> FeatureVector:
    """View 1 then view 2 (encoder.py:134-138)."""
    o1 = encode_view(maps1, n_bits, cfg, executor)
    o2 = encode_view(maps2, n_bits, cfg, executor)
    return FeatureVector(values=np.concatenate([o1, o2]), view_boundary=o1.size)


def feature_length(map_shape, maps_per_view: int, n_bits: int, cfg: EncoderConfig) -> int:
    """2 views x groups x blocks x 2^n_bits (encoder.py:141-144)."""
    return 2 * (maps_per_view // n_bits) * cfg.block_count(*map_shape) * (1 << n_bits)
