"""DDCCA second-order statistics: accumulator type and its operations.

API mirror of moments.py:26-193 of the reference. The accumulator keeps the
reference's host fields (numpy, float64) so existing callers and the model
writer keep working; every operation runs on the device through the C ABI:

  accumulate_batch  -> ddcca_accumulate_columns (explicit patch columns)
  merge / pairwise_merge / parallel_accumulate -> ddcca_moments_tree
  finalize          -> ddcca_finalize

On the fit path (cascade.train_network) the accumulators never leave the
device: they are the rows of the per-batch payload matrix produced by
ddcca_moments_partial (csrc/moments.cu) straight from the image maps.
The payload layout is [c11 | c22 | s1 | s2 | g1 | g2 | n | n_per_class]
(include/ddcca.h).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _native
from .errors import ConfigError, ShapeError
from .patches import PatchMatrix


@dataclass
class MomentAccumulator:
    """Running Grams, class / global sums and counts (moments.py:26-60)."""

    c11: np.ndarray
    c22: np.ndarray
    class_sum1: np.ndarray
    class_sum2: np.ndarray
    global_sum1: np.ndarray
    global_sum2: np.ndarray
    patch_count: int
    per_class_patch_count: np.ndarray

    @classmethod
    def zeros(cls, dim: int, class_count: int) -> "MomentAccumulator":
        if dim < 1 or class_count < 1:
            raise ConfigError(f"invalid accumulator shape dim={dim} classes={class_count}")
        z = np.zeros
        return cls(z((dim, dim)), z((dim, dim)), z((dim, class_count)), z((dim, class_count)), z(dim), z(dim), 0,
                   np.zeros(class_count, dtype=np.int64))

    @property
    def dim(self) -> int:
        return self.c11.shape[0]

    @property
    def class_count(self) -> int:
        return self.class_sum1.shape[1]

    # -- payload conversion (device <-> host) ------------------------------------
    def to_payload(self) -> np.ndarray:
        return np.concatenate([
            self.c11.ravel(), self.c22.ravel(), self.class_sum1.ravel(), self.class_sum2.ravel(),
            self.global_sum1, self.global_sum2, [float(self.patch_count)],
            self.per_class_patch_count.astype(np.float64),
        ])

    @classmethod
    def from_payload(cls, payload, dim: int, class_count: int) -> "MomentAccumulator":
        p = np.asarray(payload, dtype=np.float64)
        d, c = dim, class_count
        o = 0

        def take(n, shape=None):
            nonlocal o
            v = p[o:o + n].copy()
            o += n
            return v.reshape(shape) if shape else v

        c11 = take(d * d, (d, d))
        c22 = take(d * d, (d, d))
        s1 = take(d * c, (d, c))
        s2 = take(d * c, (d, c))
        g1 = take(d)
        g2 = take(d)
        n = int(round(take(1)[0]))
        ncls = np.rint(take(c)).astype(np.int64)
        return cls(c11, c22, s1, s2, g1, g2, n, ncls)


@dataclass(frozen=True)
class DiscriminantMoments:
    """Finalized statistics for the solver (moments.py:63-76)."""

    c11: np.ndarray
    c22: np.ndarray
    cw: np.ndarray
    cb: np.ndarray
    ctilde: np.ndarray
    patch_count: int

    @property
    def dim(self) -> int:
        return self.c11.shape[0]


def _columns(patches) -> np.ndarray:
    vals = patches.values if isinstance(patches, PatchMatrix) else np.asarray(patches, dtype=np.float64)
    if vals.ndim != 2:
        raise ShapeError(f"patch matrix must be 2-D, got shape {vals.shape}")
    return vals


def _executor(executor=None):
    from .execution import Executor

    return executor or Executor()


def accumulate_batch(acc: MomentAccumulator, p1, p2, labels, executor=None) -> MomentAccumulator:
    """Fold paired patch columns into ``acc`` in place (moments.py:86-110), on the device."""
    import torch

    x = _columns(p1)
    y = _columns(p2)
    lab = np.asarray(labels, dtype=np.int64)
    if x.shape != y.shape:
        raise ShapeError(f"view patch matrices differ: {x.shape} vs {y.shape}")
    if x.shape[0] != acc.dim:
        raise ShapeError(f"patch dim {x.shape[0]} does not match accumulator dim {acc.dim}")
    if lab.shape != (x.shape[1],):
        raise ShapeError(f"need one label per column: {lab.shape} vs {x.shape[1]} columns")
    if lab.size and (lab.min() < 0 or lab.max() >= acc.class_count):
        raise ShapeError(f"label outside [0, {acc.class_count})")
    ex = _executor(executor)
    lib = _native.load()
    with torch.cuda.stream(ex.stream):
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(ex.device)
        pay = dev(acc.to_payload())
        xd, yd, ld = dev(x), dev(y), dev(lab)
        _native.check(lib.ddcca_accumulate_columns(_native.ptr(xd), _native.ptr(yd), _native.ptr(ld), x.shape[1],
                                                   acc.dim, acc.class_count, _native.ptr(pay),
                                                   _native.stream_ptr(ex.stream)), "accumulate_batch")
        out = MomentAccumulator.from_payload(pay.cpu().numpy(), acc.dim, acc.class_count)
    acc.c11, acc.c22 = out.c11, out.c22
    acc.class_sum1, acc.class_sum2 = out.class_sum1, out.class_sum2
    acc.global_sum1, acc.global_sum2 = out.global_sum1, out.global_sum2
    acc.patch_count, acc.per_class_patch_count = out.patch_count, out.per_class_patch_count
    return acc


def _check_same(accs: Sequence[MomentAccumulator]) -> None:
    a = accs[0]
    for b in accs[1:]:
        if a.dim != b.dim or a.class_count != b.class_count:
            raise ShapeError(
                f"cannot merge accumulators of shape (dim={a.dim}, classes={a.class_count}) "
                f"and (dim={b.dim}, classes={b.class_count})"
            )


def pairwise_merge(accs: Sequence[MomentAccumulator], executor=None) -> MomentAccumulator:
    """Fixed left-to-right binary tree over the list (moments.py:132-144), on the device."""
    import torch

    if not accs:
        raise ConfigError("nothing to merge")
    accs = list(accs)
    _check_same(accs)
    if len(accs) == 1:
        return accs[0]
    ex = _executor(executor)
    from .engine import tree_merge

    with torch.cuda.stream(ex.stream):
        parts = torch.from_numpy(np.stack([a.to_payload() for a in accs])).to(ex.device)
        out = tree_merge(ex, parts).cpu().numpy()
    return MomentAccumulator.from_payload(out, accs[0].dim, accs[0].class_count)


def merge(a: MomentAccumulator, b: MomentAccumulator, executor=None) -> MomentAccumulator:
    """Componentwise sum, non-mutating (moments.py:113-129)."""
    return pairwise_merge([a, b], executor)


def parallel_accumulate(batch_jobs: Sequence[Callable[[], MomentAccumulator]], executor) -> MomentAccumulator:
    """Run per-batch jobs and reduce them (moments.py:147-165).

    The jobs are host callables (each typically launches device work); their
    accumulators are always merged through the fixed tree, which satisfies
    both the deterministic and the fast-mode contract of the reference.
    """
    if not batch_jobs:
        raise ConfigError("no batches to accumulate")
    parts = executor.map_ordered(lambda job: job(), batch_jobs)
    return pairwise_merge(parts, executor if hasattr(executor, "stream") else None)


def finalize(acc: MomentAccumulator, epsilon: float = 1e-4, executor=None) -> DiscriminantMoments:
    """Cw, Cb, Ctilde and the relative ridge (moments.py:168-193), on the device."""
    import torch

    if epsilon < 0:
        raise ConfigError(f"ridge coefficient {epsilon} must be >= 0")
    if acc.patch_count < 1:
        from .errors import NumericalError

        raise NumericalError("cannot finalize an empty accumulator")
    ex = _executor(executor)
    lib = _native.load()
    d = acc.dim
    with torch.cuda.stream(ex.stream):
        pay = torch.from_numpy(acc.to_payload()).to(ex.device)
        fin = torch.empty((5, d, d), dtype=torch.float64, device=ex.device)
        st = torch.zeros(1, dtype=torch.int32, device=ex.device)
        _native.check(lib.ddcca_finalize(_native.ptr(pay), d, acc.class_count, float(epsilon), _native.ptr(fin),
                                         _native.ptr(st), _native.stream_ptr(ex.stream)), "finalize")
        _native.status_error(int(st.item()), "finalize")
        f = fin.cpu().numpy()
    return DiscriminantMoments(c11=f[0], c22=f[1], cw=f[2], cb=f[3], ctilde=f[4], patch_count=acc.patch_count)
