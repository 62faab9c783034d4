"""Downstream classifier on the device (classify.py of the reference).

Same names, fields and errors as the reference module: ``fit`` /
``predict_many`` / ``predict`` / ``evaluate``, ``ClassifierModel``,
``EvalReport``, ``CLASSIFIER_KINDS``, ``NN_METRICS``. The nearest-neighbour
classifier (the reference default, config.py:39-41) runs as one fused CUDA
kernel (``ddcca_nn_classify``): a float64 GEMM of queries against the training
rows with the distance and the lowest-label tie rule (classify.py:136-138) in
the epilogue, so the distance matrix never exists. Rows are float64 features
(numpy or device tensors) or, without ever expanding them, the integer block
counts ``compute_feature_counts`` leaves in HBM (``CountFeatures``), expanded
through the IQ LUT inside the kernel's tile staging.

``ridge_one_vs_all`` (classify.py:86-106): the Gram of the bias-augmented rows
x = [f, 1] (dual X X' when n <= d + 1, else primal X' X) plus the ridge, its
eigen-decomposition with the same device Jacobi the filter solve uses
(``sym_eig``: the reference's round-robin schedule and ordering rules), and
the one-vs-all targets y = +-1 solved through V diag(1/w) V'; the GEMMs are
float64 cuBLAS calls on the device (plain library GEMMs, off the hot path).
The eigen-solve is a single-CTA Jacobi, so the solved dimension (min(n, d + 1))
is capped at ``RIDGE_MAX_DIM``. Prediction runs through the tiled GEMM
(``ddcca_linear_classify``: largest [x, 1] . w_c, lowest class on ties).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigError, ShapeError

CLASSIFIER_KINDS = ("nearest_neighbor", "ridge_one_vs_all")
NN_METRICS = ("euclidean", "cosine")
RIDGE_MAX_DIM = 1024  # largest eigen-solve (min(n, d + 1)) the single-CTA Jacobi takes in reasonable time


@dataclass
class CountFeatures:
    """Device block counts (m, featlen) + their BlockPlan and EncoderConfig (the lossless feature form)."""

    counts: object
    plan: object
    encoder: object

    @property
    def shape(self):
        return tuple(self.counts.shape)


@dataclass
class ClassifierModel:
    kind: str
    class_count: int
    metric: str = "euclidean"
    lam: float = 0.0
    train_features: object | None = None  # device rows (float64 / u8 / u16), host float64 rows, or CountFeatures
    train_labels: np.ndarray | None = None
    weights: np.ndarray | None = None
    row_kind: int = 3
    lut: object | None = None  # device LUT for count rows
    count_source: object | None = None  # the CountFeatures the rows came from (model files write their values)

    @property
    def feature_dim(self) -> int:
        return int(self.train_features.shape[1])


@dataclass
class EvalReport:
    accuracy: float
    per_class_accuracy: np.ndarray
    confusion: np.ndarray
    stage_seconds: dict[str, float] = field(default_factory=dict)
    threads: int = 1
    deterministic: bool = True

    @property
    def total(self) -> int:
        return int(self.confusion.sum())


def _executor(executor):
    from .cascade import _executor as ex

    return ex(executor)


def _rows(ex, features):
    """-> (device rows, row_kind, device lut or None)."""
    import torch

    from . import engine as E

    if isinstance(features, CountFeatures):
        c = features.counts
        kind = E.count_kind(features.plan.bpc)
        lut = torch.from_numpy(E.iq_lut(features.encoder)).to(ex.device)
        if kind == 1:  # saturating u8 -> exact u16
            out = torch.empty(c.shape, dtype=torch.int16, device=ex.device)
            nblk = c.numel() // features.plan.bins
            with torch.cuda.stream(ex.stream):
                _native.check(_native.load().ddcca_counts_to_u16(
                    _native.ptr(c), nblk, features.plan.bins, features.plan.bpc, _native.ptr(out),
                    _native.stream_ptr(ex.stream)), "counts_to_u16")
            return out, 2, lut
        return c.contiguous(), kind, lut
    if isinstance(features, torch.Tensor):
        t = features.to(ex.device, dtype=torch.float64).contiguous()
    else:
        a = np.ascontiguousarray(np.asarray(features, dtype=np.float64))
        if a.ndim != 2:
            raise ShapeError(f"features must be 2-D, got shape {a.shape}")
        t = torch.from_numpy(a).to(ex.device)
    return t, 3, None


def _check_training_set(n_rows: int, labels: np.ndarray) -> int:
    if n_rows != labels.shape[0]:
        raise ShapeError(f"features ({n_rows} rows) do not pair with {labels.shape[0]} labels")
    if labels.size == 0 or labels.min() < 0:
        raise ConfigError("labels must be non-negative and non-empty")
    class_count = int(labels.max()) + 1
    present = np.bincount(labels, minlength=class_count)
    if np.any(present == 0):
        raise ConfigError("every class id in [0, max] needs at least one training sample")
    return class_count


def fit(features, labels, kind: str = "nearest_neighbor", metric: str = "euclidean", lam: float | None = None,
        executor=None) -> ClassifierModel:
    """Train a classifier on row-wise feature vectors (classify.py:69-106)."""
    labels = np.asarray(labels, dtype=np.int64)
    n_rows = features.shape[0]
    if len(getattr(features, "shape", ())) != 2:
        raise ShapeError(f"features must be 2-D, got shape {getattr(features, 'shape', None)}")
    class_count = _check_training_set(n_rows, labels)
    if kind not in CLASSIFIER_KINDS:
        raise ConfigError(f"classifier kind {kind!r} not one of {CLASSIFIER_KINDS}")
    if kind == "ridge_one_vs_all":
        return _fit_ridge(_executor(executor), features, labels, class_count, lam)
    if metric not in NN_METRICS:
        raise ConfigError(f"metric {metric!r} not one of {NN_METRICS}")
    ex = _executor(executor)
    rows, row_kind, lut = _rows(ex, features)
    return ClassifierModel(kind=kind, class_count=class_count, metric=metric, train_features=rows,
                           train_labels=labels.copy(), row_kind=row_kind, lut=lut,
                           count_source=features if isinstance(features, CountFeatures) else None)


def _fit_ridge(ex, features, labels: np.ndarray, class_count: int, lam) -> ClassifierModel:
    """One-vs-all ridge regression on [x, 1] (classify.py:86-106), on the device."""
    import torch

    from . import engine as E
    from .solver import sym_eig

    with torch.cuda.stream(ex.stream):
        if isinstance(features, CountFeatures):
            f = E.Engine(ex).expand(features.counts, features.plan, features.encoder)
        else:
            f, _, _ = _rows(ex, features)
        n, d = f.shape
        x = torch.cat([f, torch.ones((n, 1), dtype=torch.float64, device=ex.device)], dim=1)
        if lam is None:
            lam = 1e-3 * float(torch.sum(x * x).item()) / x.shape[1]
        if lam <= 0:
            raise ConfigError(f"ridge lambda {lam} must be > 0")
        m = min(n, d + 1)
        if m > RIDGE_MAX_DIM:
            raise ConfigError(f"ridge fit solves a {m} x {m} eigenproblem; the device Jacobi takes at most "
                              f"{RIDGE_MAX_DIM} (fewer training rows or features)")
        lab = torch.from_numpy(labels).to(ex.device)
        y = torch.where(lab[:, None] == torch.arange(class_count, device=ex.device)[None, :], 1.0, -1.0).to(
            torch.float64)
        eye = torch.eye(m, dtype=torch.float64, device=ex.device)
        g = (x @ x.T if n <= d + 1 else x.T @ x) + lam * eye
        w_eig, v = sym_eig((0.5 * (g + g.T)).cpu().numpy(), ex)
        vd = torch.from_numpy(v).to(ex.device)
        inv = torch.from_numpy(1.0 / w_eig).to(ex.device)
        if n <= d + 1:
            # dual form: w = X'(XX' + lam I)^-1 Y
            solved = (vd * inv) @ (vd.T @ y)
            weights = (x.T @ solved).T
        else:
            weights = ((vd * inv) @ (vd.T @ (x.T @ y))).T
        out = weights.contiguous().cpu().numpy()
    return ClassifierModel(kind="ridge_one_vs_all", class_count=class_count, lam=float(lam), weights=out)


def predict_many(model: ClassifierModel, features, executor=None) -> np.ndarray:
    """Predicted class ids for row-wise feature vectors (classify.py:123-143)."""
    import torch

    ex = _executor(executor)
    if model.kind != "nearest_neighbor":
        return _predict_linear(ex, model, features)
    if not hasattr(model.train_features, "data_ptr"):  # e.g. a loaded model: float64 rows on the host
        rows, model.row_kind, model.lut = _rows(ex, model.train_features)
        model.train_features = rows
    q, q_kind, _ = _rows(ex, features)
    if q.ndim != 2 or q.shape[1] != model.feature_dim:
        raise ShapeError(f"feature dim {q.shape[-1] if q.ndim else '?'} does not match model dim {model.feature_dim}")
    if q_kind != model.row_kind:
        raise ShapeError("query rows and training rows must use the same feature form (float64 or counts)")
    lib = _native.load()
    nq, nt, dim = q.shape[0], model.train_features.shape[0], q.shape[1]
    with torch.cuda.stream(ex.stream):
        labels = torch.from_numpy(model.train_labels).to(ex.device)
        pred = torch.empty(nq, dtype=torch.int64, device=ex.device)
        ws_bytes = lib.ddcca_nn_workspace(nq, nt)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=ex.device)
        lut = model.lut
        _native.check(lib.ddcca_nn_classify(
            _native.ptr(q), nq, _native.ptr(model.train_features), nt, dim, model.row_kind,
            _native.ptr(lut) if lut is not None else None, int(lut.numel()) if lut is not None else 0,
            _native.ptr(labels), 0 if model.metric == "euclidean" else 1, _native.ptr(pred), _native.ptr(ws),
            ws_bytes, _native.stream_ptr(ex.stream)), "nn_classify")
        out = pred.cpu().numpy()
    return out


def _predict_linear(ex, model: ClassifierModel, features) -> np.ndarray:
    """Ridge one-vs-all scores [x, 1] . w_c, argmax with the lowest class on ties (classify.py:140-142)."""
    import torch

    from . import engine as E

    w = np.asarray(model.weights, dtype=np.float64)
    if isinstance(features, CountFeatures):
        with torch.cuda.stream(ex.stream):
            q = E.Engine(ex).expand(features.counts, features.plan, features.encoder)
    else:
        q, _, _ = _rows(ex, features)
    if q.ndim != 2 or q.shape[1] != w.shape[1] - 1:
        raise ShapeError(f"feature dim {q.shape[-1]} does not match model dim {w.shape[1] - 1}")
    lib = _native.load()
    nq, nc, dim = q.shape[0], w.shape[0], w.shape[1] - 1
    with torch.cuda.stream(ex.stream):
        wd = torch.from_numpy(np.ascontiguousarray(w[:, :dim])).to(ex.device)
        bd = torch.from_numpy(np.ascontiguousarray(w[:, dim])).to(ex.device)
        ids = torch.arange(nc, dtype=torch.int64, device=ex.device)
        pred = torch.empty(nq, dtype=torch.int64, device=ex.device)
        ws_bytes = lib.ddcca_nn_workspace(nq, nc)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=ex.device)
        _native.check(lib.ddcca_linear_classify(_native.ptr(q), nq, _native.ptr(wd), nc, dim, _native.ptr(bd),
                                                _native.ptr(ids), _native.ptr(pred), _native.ptr(ws), ws_bytes,
                                                _native.stream_ptr(ex.stream)), "linear_classify")
        return pred.cpu().numpy()


def predict(model: ClassifierModel, feature, executor=None) -> int:
    f = feature
    if not isinstance(f, CountFeatures):
        f = np.asarray(feature, dtype=np.float64)[None, :]
    return int(predict_many(model, f, executor)[0])


def evaluate(model: ClassifierModel, features, labels, stage_seconds: dict[str, float] | None = None,
             threads: int = 1, deterministic: bool = True, executor=None) -> EvalReport:
    """Confusion counts, overall and per-class accuracy (classify.py:150-176)."""
    truth = np.asarray(labels, dtype=np.int64)
    if truth.size == 0:
        raise ConfigError("evaluation needs at least one labelled sample")
    guess = predict_many(model, features, executor)
    k = model.class_count
    confusion = np.bincount(truth * k + guess, minlength=k * k).reshape(k, k).astype(np.int64)
    support = confusion.sum(axis=1)
    hits = np.diagonal(confusion).astype(np.float64)
    per_class = np.full(k, np.nan)
    per_class[support > 0] = hits[support > 0] / support[support > 0]
    return EvalReport(accuracy=float(hits.sum() / truth.size), per_class_accuracy=per_class, confusion=confusion,
                      stage_seconds=dict(stage_seconds or {}), threads=threads, deterministic=deterministic)
