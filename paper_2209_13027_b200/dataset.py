"""Labelled two-view datasets (the container the fit/transform API consumes).

Mirrors ViewPairSample / ViewPairDataset (dataset.py:20-59 of the
reference). File ingestion (PGM/CSV manifests) is outside this build's
scope; ``ViewPairDataset.from_arrays`` builds a
dataset from stacked arrays without per-sample Python objects, which is how
the benchmark and large runs feed the device path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ParseError, ShapeError


@dataclass(frozen=True)
class ViewPairSample:
    view1: np.ndarray
    view2: np.ndarray
    label: int

    def __post_init__(self):
        if self.view1.shape != self.view2.shape:
            raise ShapeError(f"views differ in size: {self.view1.shape} vs {self.view2.shape}")
        if self.label < 0:
            raise ParseError(f"negative class label {self.label}")


def _is_tensor(a) -> bool:
    t = type(a)
    return t.__module__.startswith("torch") and t.__name__ == "Tensor"


@dataclass
class ViewPairDataset:
    """Ordered labelled view pairs with contiguous class ids."""

    samples: list
    class_count: int
    label_map: dict = field(default_factory=dict)
    _stacks: tuple | None = field(default=None, repr=False)

    @classmethod
    def from_arrays(cls, view1, view2, labels, class_count: int | None = None, label_map=None):
        # pinned torch tensors are kept as they are: train_network then uploads them
        # asynchronously, chunk by chunk, overlapped with the first layer's moments
        v1 = view1 if _is_tensor(view1) else np.asarray(view1)
        v2 = view2 if _is_tensor(view2) else np.asarray(view2)
        lab = np.asarray(labels, dtype=np.int64)
        if v1.ndim != 3 or v1.shape != v2.shape:
            raise ShapeError(f"need two equal (M, p, q) stacks, got {v1.shape} and {v2.shape}")
        if lab.shape != (v1.shape[0],):
            raise ShapeError("one label per sample required")
        if lab.size and lab.min() < 0:
            raise ParseError("negative class label")
        cc = int(lab.max()) + 1 if class_count is None else int(class_count)
        ds = cls(samples=[], class_count=cc, label_map=dict(label_map or {}))
        ds._stacks = (v1, v2, lab)
        return ds

    def __len__(self) -> int:
        return self._stacks[2].shape[0] if self._stacks is not None else len(self.samples)

    @property
    def labels(self) -> np.ndarray:
        if self._stacks is not None:
            return self._stacks[2].copy()
        return np.array([s.label for s in self.samples], dtype=np.int64)

    @property
    def image_shape(self) -> tuple[int, int]:
        if self._stacks is not None:
            return tuple(self._stacks[0].shape[1:])
        return self.samples[0].view1.shape

    def view_stack(self, view: int) -> np.ndarray:
        """(M, p, q) array of one view (a copy, like dataset.py:56-59)."""
        if self._stacks is not None:
            return np.array(self._stacks[0 if view == 1 else 1], copy=True)
        attr = "view1" if view == 1 else "view2"
        return np.stack([getattr(s, attr) for s in self.samples])

    def stacks_view(self):
        """(view1, view2, labels) without copying when built from arrays."""
        if self._stacks is not None:
            return self._stacks
        return self.view_stack(1), self.view_stack(2), self.labels
