"""Labelled two-view datasets (the container the fit/transform API consumes).

Mirrors ViewPairSample / ViewPairDataset (dataset.py:20-59 of the
reference) and its ingestion (dataset.py:60-230: load_pgm, write_pgm,
load_matrix_csv, load_dataset). ``ViewPairDataset.from_arrays`` builds a
dataset from stacked arrays without per-sample Python objects, which is how
the benchmark and large runs feed the device path. ``load_dataset`` decodes
the manifest's PGM files with the native parallel loader
(``ddcca_pgm_load_many``) straight into pinned float32 stacks (so
train_network uploads them chunk by chunk) and builds the LBP second view
of the ``lbp_plus_gray`` recipe on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

import ctypes as C
import math
from pathlib import Path

from .errors import EmptyDatasetError, IoError, ParseError, ShapeError


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
    # multi-GPU: the stacks hold rows [row_offset, row_offset + n) of a dataset of total_rows
    # samples (ViewPairDataset.shard); train_network / compute_features only read their rank's rows
    row_offset: int = 0
    total_rows: int | None = None

    @classmethod
    def shard(cls, view1, view2, labels, first_row: int, total_rows: int, class_count: int, label_map=None):
        """This rank's rows of a larger dataset (no host copy of the other ranks' samples): the fit and
        the transform see a dataset of ``total_rows`` samples, batched and sharded as usual, and read
        only rows [first_row, first_row + len(labels)), which must cover the rank's batch shard."""
        ds = cls.from_arrays(view1, view2, labels, class_count=class_count, label_map=label_map)
        if first_row < 0 or first_row + len(ds) > total_rows:
            raise ShapeError(f"rows [{first_row}, {first_row + len(ds)}) outside a dataset of {total_rows}")
        ds.row_offset = int(first_row)
        ds.total_rows = int(total_rows)
        return ds

    @property
    def global_len(self) -> int:
        """Samples of the whole (possibly sharded) dataset."""
        return self.total_rows if self.total_rows is not None else len(self)

    def local_rows(self, s0: int, s1: int):
        """(view1, view2, labels) rows [s0, s1) of the whole dataset, from this object's stacks."""
        v1, v2, lab = self.stacks_view()
        a, b = s0 - self.row_offset, s1 - self.row_offset
        if a < 0 or b > len(lab):
            raise ShapeError(f"rows [{s0}, {s1}) are not in this shard [{self.row_offset}, "
                             f"{self.row_offset + len(lab)})")
        return v1[a:b], v2[a:b], lab[a:b]

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


# ----------------------------------------------------------------------------
# ingestion (dataset.py:60-230)
# ----------------------------------------------------------------------------

def _native_err(rc: int, what: str):
    from . import _native

    msg = _native.load().ddcca_last_error().decode(errors="replace")
    if msg.startswith("cannot read"):
        return IoError(msg)
    return ParseError(msg if msg else what)


def load_pgm(path) -> np.ndarray:
    """Binary PGM (P5) -> [0, 1] float64 plane (dataset.py:68-118).

    The header is parsed by the native loader (``ddcca_pgm_info``); the samples
    (8-bit, or big-endian 16-bit when maxval > 255) are divided by maxval in
    float64, so the plane equals the reference's bit for bit.
    """
    from . import _native

    lib = _native.load()
    w, h, mv, off = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
    if lib.ddcca_pgm_info(str(path).encode(), C.byref(w), C.byref(h), C.byref(mv), C.byref(off)):
        raise _native_err(1, str(path))
    raw = Path(path).read_bytes()
    item = 2 if mv.value > 255 else 1
    n = w.value * h.value * item
    payload = raw[off.value:off.value + n]
    if len(payload) < n:
        raise ParseError(f"{path}: truncated PGM payload ({len(payload)}/{n} bytes)")
    vals = np.frombuffer(payload, dtype=">u2" if item == 2 else np.uint8).astype(np.float64)
    return vals.reshape(h.value, w.value) / mv.value


def write_pgm(path, plane: np.ndarray, maxval: int = 255) -> None:
    """Quantize a [0, 1] plane to a binary PGM file, round-to-nearest (dataset.py:121-129)."""
    if not 1 <= maxval <= 65535:
        raise ParseError(f"PGM maxval must be in [1, 65535], got {maxval}")
    levels = np.clip(np.rint(np.asarray(plane, dtype=np.float64) * maxval), 0, maxval)
    rows, cols = levels.shape
    samples = levels.astype(">u2" if maxval > 255 else np.uint8).tobytes()
    Path(path).write_bytes(b"P5\n%d %d\n%d\n" % (cols, rows, maxval) + samples)


def load_matrix_csv(path) -> np.ndarray:
    """Rectangular numeric CSV -> float plane, values verbatim (dataset.py:132-158)."""
    path = Path(path)
    try:
        text = path.read_text(encoding="ascii")
    except OSError as e:
        raise IoError(f"cannot read {path}: {e}") from e
    rows = []
    for lineno, line in enumerate(text.splitlines(), start=1):
        if not line.strip():
            continue
        try:
            row = [float(c) for c in line.split(",")]
        except ValueError as e:
            raise ParseError(f"{path}:{lineno}: non-numeric cell") from e
        if not all(math.isfinite(v) for v in row):
            raise ParseError(f"{path}:{lineno}: non-finite cell")
        if rows and len(row) != len(rows[0]):
            raise ParseError(f"{path}:{lineno}: ragged row ({len(row)} cells, expected {len(rows[0])})")
        rows.append(row)
    if not rows:
        raise ParseError(f"{path}: empty CSV matrix")
    return np.array(rows, dtype=np.float64)


def _manifest(manifest: Path):
    try:
        text = manifest.read_text(encoding="utf-8")
    except OSError as e:
        raise IoError(f"cannot read manifest {manifest}: {e}") from e
    base = manifest.parent
    lines = []
    for lineno, line in enumerate(text.splitlines(), start=1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        fields = [f.strip() for f in line.split(",")]
        if len(fields) < 2:
            raise ParseError(f"{manifest}:{lineno}: expected 'path[,path...],label'")
        try:
            raw_label = int(fields[-1])
        except ValueError as e:
            raise ParseError(f"{manifest}:{lineno}: label {fields[-1]!r} is not an integer") from e
        if raw_label < 0:
            raise ParseError(f"{manifest}:{lineno}: negative label {raw_label}")
        lines.append((lineno, [(base / p).resolve() for p in fields[:-1]], raw_label))
    return lines


def load_dataset(manifest, recipe=None, threads: int = 16, executor=None) -> ViewPairDataset:
    """Manifest of "path[,path...],label" lines -> dataset (dataset.py:175-230).

    Relative paths resolve against the manifest's directory; class ids are
    re-indexed in first-appearance order (``label_map`` keeps the originals);
    with ``recipe`` None two paths form an external pair and one path is
    duplicated. All-PGM manifests are decoded in parallel by the native loader
    into pinned float32 stacks; ``lbp_plus_gray`` computes view 2 on the device.
    """
    import torch

    from . import _native
    from .views import ViewRecipe, apply_recipe, lbp_stack

    manifest = Path(manifest)
    lines = _manifest(manifest)
    if not lines:
        raise EmptyDatasetError(f"{manifest}: no samples")
    label_map: dict[int, int] = {}
    labels = []
    for _, _, raw in lines:
        if raw not in label_map:
            label_map[raw] = len(label_map)
        labels.append(label_map[raw])
    labels = np.asarray(labels, dtype=np.int64)
    kinds = {len(paths) for _, paths, _ in lines}
    all_pgm = all(p.suffix.lower() == ".pgm" for _, paths, _ in lines for p in paths)
    rec = recipe
    fast = all_pgm and len(kinds) == 1 and (
        rec is None or rec.kind in ("lbp_plus_gray", "external_pair", "identity_pair", "channel_split"))
    if not fast:
        # mixed / CSV manifests: per-line planes through the reference recipe semantics
        samples, shape = [], None
        for lineno, paths, _ in lines:
            planes = [_load_plane(p) for p in paths]
            r = rec if rec is not None else ViewRecipe("external_pair" if len(planes) >= 2 else "identity_pair")
            v1, v2 = apply_recipe(planes, r, executor)
            if shape is None:
                shape = v1.shape
            elif v1.shape != shape:
                raise ShapeError(f"{manifest}:{lineno}: sample size {v1.shape} differs from {shape}")
            samples.append((v1, v2))
        v1 = np.stack([a for a, _ in samples]).astype(np.float32)
        v2 = np.stack([b for _, b in samples]).astype(np.float32)
        return ViewPairDataset.from_arrays(v1, v2, labels, class_count=len(label_map), label_map=label_map)
    npl = kinds.pop()
    r = rec if rec is not None else ViewRecipe("external_pair" if npl >= 2 else "identity_pair")
    if r.kind == "lbp_plus_gray" and npl != 1:
        from .errors import RecipeError

        raise RecipeError("lbp_plus_gray expects a single gray plane")
    lib = _native.load()
    w, h, mv = C.c_int(), C.c_int(), C.c_int()
    first = str(lines[0][1][0]).encode()
    if lib.ddcca_pgm_info(first, C.byref(w), C.byref(h), C.byref(mv), None):
        raise _native_err(1, str(lines[0][1][0]))
    p_, q_ = h.value, w.value
    m = len(lines)
    planes = []
    for k in range(npl):
        buf = torch.empty((m, p_, q_), dtype=torch.float32).pin_memory()
        paths = (C.c_char_p * m)(*[str(ps[k]).encode() for _, ps, _ in lines])
        if lib.ddcca_pgm_load_many(paths, m, p_, q_, C.c_void_p(buf.data_ptr()), int(threads)):
            err = _native_err(1, str(manifest))
            if "differs" in str(err):
                raise ShapeError(str(err))
            raise err
        planes.append(buf)
    if r.kind == "lbp_plus_gray":
        dev = lbp_stack(planes[0].cuda(non_blocking=True), executor)
        v2 = torch.empty_like(planes[0]).pin_memory()
        v2.copy_(dev)
        v1 = planes[0]
    elif r.kind == "channel_split":
        from .errors import RecipeError

        if max(r.c1, r.c2) >= npl:
            raise RecipeError(f"channel_split({r.c1},{r.c2}) needs {max(r.c1, r.c2) + 1} channel planes, "
                              f"manifest line has {npl}")
        v1, v2 = planes[r.c1], planes[r.c2]
    elif r.kind == "external_pair":
        if npl < 2:
            from .errors import RecipeError

            raise RecipeError("external_pair expects two planes per manifest line")
        v1, v2 = planes[0], planes[1]
    else:  # identity_pair
        if npl != 1:
            from .errors import RecipeError

            raise RecipeError("identity_pair expects a single plane")
        v1, v2 = planes[0], planes[0]
    return ViewPairDataset.from_arrays(v1, v2, labels, class_count=len(label_map), label_map=label_map)


def _load_plane(path: Path) -> np.ndarray:
    suffix = path.suffix.lower()
    if suffix == ".pgm":
        return load_pgm(path)
    if suffix == ".csv":
        return load_matrix_csv(path)
    raise ParseError(f"{path}: unsupported file type {suffix!r} (expected .pgm or .csv)")
