"""Layer-wise training and application of the two-view filter cascade.

API mirror of cascade.py:26-259 of the reference, backed by the device
engine (engine.py). ``train_network`` is the fit entry point and
``pipeline.compute_features`` the transform entry point; everything between
the host arrays and the returned FilterBank / features runs as sm_100a
kernels. Maps are stored as float32 on the device (the reference keeps
float64 on the host); statistics and the solve are float64.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine as E
from .errors import ConfigError, ShapeError
from .patches import BatchSpec, PatchGeometry, batch_partition
from .solver import FilterBank, FilterLayer

CHUNK_COLS = 1 << 17  # reference chunking constant (cascade.py:26); the device path needs no chunks


@dataclass(frozen=True)
class LayerConfig:
    """Filter count, window geometry, centering (cascade.py:29-41)."""

    filters: int
    geom: PatchGeometry
    center: bool = True

    def __post_init__(self):
        if self.filters < 1:
            raise ConfigError(f"filter count {self.filters} must be >= 1")
        if self.filters > self.geom.dim:
            raise ConfigError(f"filter count {self.filters} exceeds patch dimension {self.geom.dim}")


@dataclass(frozen=True)
class NetworkConfig:
    """Layers, sample batching, ridge (cascade.py:44-52)."""

    layers: tuple
    batch: BatchSpec = BatchSpec()
    epsilon: float = 1e-4

    def __post_init__(self):
        if not self.layers:
            raise ConfigError("network needs at least one layer")


@dataclass
class LayerOutput:
    """Maps of both views for a set of samples plus lineage (cascade.py:55-80)."""

    maps1: np.ndarray
    maps2: np.ndarray
    labels: np.ndarray
    lineage: tuple

    def __post_init__(self):
        if self.maps1.shape != self.maps2.shape:
            raise ShapeError(f"view map stacks differ: {self.maps1.shape} vs {self.maps2.shape}")
        if len(self.lineage) != self.maps1.shape[1]:
            raise ShapeError("one lineage entry per map required")

    @property
    def n_samples(self) -> int:
        return self.maps1.shape[0]

    @property
    def n_maps(self) -> int:
        return self.maps1.shape[1]

    @property
    def map_shape(self) -> tuple[int, int]:
        return self.maps1.shape[2], self.maps1.shape[3]


def _child_lineage(lineage, count: int):
    return tuple(parent + (g,) for parent in lineage for g in range(count))


def layer_input(ds) -> LayerOutput:
    """Dataset as first-layer input: one map per view (cascade.py:83-90)."""
    v1, v2, lab = ds.stacks_view()
    return LayerOutput(maps1=np.asarray(v1)[:, None], maps2=np.asarray(v2)[:, None], labels=np.asarray(lab),
                       lineage=((),))


def _executor(executor):
    from .execution import Executor

    return executor if executor is not None and hasattr(executor, "stream") else Executor()


def _to_dev32(ex, a):
    """Host array (numpy or pinned torch tensor) -> float32 device tensor on the executor's stream."""
    import torch

    if isinstance(a, torch.Tensor):
        t = a if a.dtype == torch.float32 else a.float()
        t = t.contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32)))
    return t.to(ex.device, non_blocking=t.is_pinned())


def _labels_dev(ex, labels):
    import torch

    return torch.from_numpy(np.ascontiguousarray(np.asarray(labels, dtype=np.int32))).to(ex.device)


def device_layers(bank: FilterBank, ex) -> list:
    """DeviceLayers for a bank (cached on the bank per device)."""
    cache = getattr(bank, "_device_cache", None)
    if cache is not None and cache[0] == str(ex.device):
        return cache[1]
    layers = [E.layer_from_filters(ex, l.filters1, l.filters2, l.geom, l.center) for l in bank.layers]
    object.__setattr__(bank, "_device_cache", (str(ex.device), layers))
    return layers


def _bank_from_device(layers: list) -> FilterBank:
    out = []
    for lay in layers:
        w1 = lay.w1.cpu().numpy()
        w2 = lay.w2.cpu().numpy()
        L, g = lay.count, lay.geom
        out.append(FilterLayer(filters1=np.ascontiguousarray(w1.T).reshape(L, g.l1, g.l2).copy(),
                               filters2=np.ascontiguousarray(w2.T).reshape(L, g.l1, g.l2).copy(),
                               geom=g, center=lay.center))
    return FilterBank(layers=tuple(out))


def conv2d(plane, kernel, padding: str = "zero_same", center: bool = False, executor=None) -> np.ndarray:
    """Cross-correlate one map with one kernel (cascade.py:93-100)."""
    kernel = np.asarray(kernel, dtype=np.float64)
    if kernel.ndim != 2:
        raise ShapeError(f"kernel must be 2-D, got shape {kernel.shape}")
    geom = PatchGeometry(kernel.shape[0], kernel.shape[1], 1, padding)
    layer = FilterLayer(kernel[None], kernel[None], geom, center)
    return apply_filters(np.asarray(plane, dtype=np.float64)[None], layer, 1, executor)[0, 0]


def apply_filters(stack, layer: FilterLayer, view: int, executor=None) -> np.ndarray:
    """(N, p, q) -> (N, L, p', q') filter-minor (cascade.py:108-126), float32 device conv."""
    import torch

    stack = np.asarray(stack)
    if stack.ndim != 3:
        raise ShapeError(f"expected (N, p, q) maps, got shape {stack.shape}")
    ex = _executor(executor)
    with torch.cuda.stream(ex.stream):
        dl = E.layer_from_filters(ex, layer.filters1, layer.filters2, layer.geom, layer.center)
        out = E.conv(ex, _to_dev32(ex, stack), dl, view)
        return out.cpu().numpy().astype(np.float64)


def apply_layer(inputs: LayerOutput, layer: FilterLayer, executor, batch: BatchSpec) -> LayerOutput:
    """Run one trained layer over all samples (cascade.py:133-152)."""
    n, m = inputs.n_samples, inputs.n_maps
    p, q = inputs.map_shape
    o1 = apply_filters(inputs.maps1.reshape(-1, p, q), layer, 1, executor)
    o2 = apply_filters(inputs.maps2.reshape(-1, p, q), layer, 2, executor)
    oh, ow = o1.shape[2:]
    return LayerOutput(maps1=o1.reshape(n, m * layer.count, oh, ow), maps2=o2.reshape(n, m * layer.count, oh, ow),
                       labels=inputs.labels, lineage=_child_lineage(inputs.lineage, layer.count))


def accumulate_layer_moments(inputs: LayerOutput, geom: PatchGeometry, center: bool, class_count: int,
                             batch: BatchSpec, executor):
    """Per-batch moments of a layer's input maps merged by the fixed tree (cascade.py:155-189)."""
    import torch

    from .moments import MomentAccumulator

    ex = _executor(executor)
    n, m = inputs.n_samples, inputs.n_maps
    p, q = inputs.map_shape
    lab = np.asarray(inputs.labels)
    if lab.size and (lab.min() < 0 or lab.max() >= class_count):
        raise ShapeError(f"label outside [0, {class_count})")
    ranges = batch_partition(n, batch)
    with torch.cuda.stream(ex.stream):
        m1 = _to_dev32(ex, inputs.maps1.reshape(-1, p, q))
        m2 = _to_dev32(ex, inputs.maps2.reshape(-1, p, q))
        mlab = _labels_dev(ex, np.repeat(lab, m))
        offs = np.array([0] + [r.stop * m for r in ranges], dtype=np.int64)
        parts = E.moments_partials(ex, m1, m2, mlab, offs, geom, center, class_count)
        merged = E.tree_merge(ex, parts).cpu().numpy()
    return MomentAccumulator.from_payload(merged, geom.dim, class_count)


def train_layer(inputs: LayerOutput, cfg: LayerConfig, class_count: int, batch: BatchSpec, executor,
                epsilon: float = 1e-4) -> FilterLayer:
    """One layer's filters from its input maps (cascade.py:192-204)."""
    import torch

    ex = _executor(executor)
    n, m = inputs.n_samples, inputs.n_maps
    p, q = inputs.map_shape
    lab = np.asarray(inputs.labels)
    if lab.size and (lab.min() < 0 or lab.max() >= class_count):
        raise ShapeError(f"label outside [0, {class_count})")  # accumulate_batch, moments.py:91-98
    ranges = batch_partition(n, batch)
    with torch.cuda.stream(ex.stream):
        m1 = _to_dev32(ex, inputs.maps1.reshape(-1, p, q))
        m2 = _to_dev32(ex, inputs.maps2.reshape(-1, p, q))
        mlab = _labels_dev(ex, np.repeat(lab, m))
        offs = np.array([0] + [r.stop * m for r in ranges], dtype=np.int64)
        parts = E.moments_partials(ex, m1, m2, mlab, offs, cfg.geom, cfg.center, class_count)
        merged = E.tree_merge(ex, parts)
        lay = E.solve_layer(ex, merged, cfg.geom, cfg.filters, cfg.center, class_count, epsilon)
        return _bank_from_device([lay]).layers[0]


def train_network(ds, cfg: NetworkConfig, executor, stage_hook=None) -> FilterBank:
    """Fit: train all layers bottom-up on the device (cascade.py:207-223).

    Intermediate layers are not materialized for the whole training set:
    each layer's input maps are recomputed per super-batch from the images
    (the conv is cheaper than writing and re-reading them), so memory stays
    bounded for any corpus size. With a torch.distributed process group the
    samples are sharded by whole batches over the ranks and the per-layer
    partial moments are reduced with NCCL before the solve.
    """
    import torch

    ex = _executor(executor)
    n = ds.global_len
    bs = cfg.batch.batch_size
    gb = batch_partition(n, cfg.batch)
    mine = ex.shard(len(gb))
    s0 = gb[mine.start].start if len(mine) else ds.row_offset
    s1 = gb[mine.stop - 1].stop if len(mine) else ds.row_offset
    h1, h2, lab = ds.local_rows(s0, s1)
    lab = np.asarray(lab)
    if lab.size and (lab.min() < 0 or lab.max() >= ds.class_count):
        raise ShapeError(f"label outside [0, {ds.class_count})")
    eng = E.Engine(ex)
    with torch.cuda.stream(ex.stream):
        if _pinned(h1) and _pinned(h2):
            # pinned host views: upload in chunks on a copy stream; the first layer's
            # moments start on each chunk as it lands (Engine.uploader)
            eng.uploader = ChunkedUpload(ex, h1, h2, lab, UPLOAD_CHUNK_BATCHES * bs)
            i1, i2, ld = eng.uploader.d1, eng.uploader.d2, eng.uploader.labels
        else:
            i1 = _to_dev32(ex, h1)
            i2 = _to_dev32(ex, h2)
            ld = _labels_dev(ex, lab)
        res = eng.fit(i1, i2, ld, ds.class_count, list(cfg.layers), bs, cfg.epsilon, n_global=n, first_sample=s0,
                      stage_hook=stage_hook)
        bank = _bank_from_device(res.layers)  # reads on the executor's stream
    object.__setattr__(bank, "_device_cache", (str(ex.device), res.layers))
    # the transform of the same samples reuses the uploaded images and the retained
    # last-hidden-layer maps (pipeline.compute_feature_counts)
    ds._device_state = {"device": str(ex.device), "rows": (s0, s1), "images": (i1, i2), "engine": eng,
                        "bank": id(bank)}
    return bank


UPLOAD_CHUNK_BATCHES = 16  # sample batches per image upload chunk


def _pinned(a) -> bool:
    import torch

    return isinstance(a, torch.Tensor) and a.dtype == torch.float32 and a.is_pinned() and a.is_contiguous()


class ChunkedUpload:
    """Pinned (m, p, q) float32 views (+ labels) -> device tensors, chunk by chunk on the
    executor's persistent upload stream, submitted lazily.

    A chunk's copies are enqueued only when the fit reaches rows ``lookahead`` chunks before
    it (``event_for``): host->device copies share the copy engine in submission order, so
    submitting the whole image upload up front would queue every small copy the fit issues
    on the compute stream (plan tables, label slices) behind all of it -- the first layer's
    moments could then not start before the last chunk landed. The labels go first (pinned,
    asynchronous) and the compute stream waits for them.
    """

    def __init__(self, ex, h1, h2, labels, rows_per_chunk: int, lookahead: int = 2):
        import torch

        m = h1.shape[0]
        up = getattr(ex, "upload_stream", None)
        if up is None:
            up = ex.upload_stream = torch.cuda.Stream(device=ex.device)
        self.ex, self.up, self.h1, self.h2 = ex, up, h1, h2
        self.lookahead = max(0, int(lookahead))
        step = max(1, rows_per_chunk)
        self.ends = [min(m, r0 + step) for r0 in range(0, m, step)]
        self.events = []
        # Buffers are allocated on the upload stream and marked as used by the compute stream:
        # the caching allocator then never hands this upload a block that earlier compute work
        # may still read, so the upload need not wait for the compute stream -- the next fit's
        # images stream in while the previous transform still runs.
        self._lab_host = torch.from_numpy(np.ascontiguousarray(np.asarray(labels, dtype=np.int32))).pin_memory()
        with torch.cuda.stream(up):
            self.d1 = torch.empty(h1.shape, dtype=torch.float32, device=ex.device)
            self.d2 = torch.empty(h2.shape, dtype=torch.float32, device=ex.device)
            self.labels = self._lab_host.to(ex.device, non_blocking=True)
            lab_ev = torch.cuda.Event()
            lab_ev.record(up)
        for t in (self.d1, self.d2, self.labels):
            t.record_stream(ex.stream)
        ex.stream.wait_event(lab_ev)

    def _submit(self, upto: int):
        import torch

        upto = min(upto, len(self.ends) - 1)
        with torch.cuda.stream(self.up):
            while len(self.events) <= upto:
                i = len(self.events)
                r0 = self.ends[i - 1] if i else 0
                r1 = self.ends[i]
                self.d1[r0:r1].copy_(self.h1[r0:r1], non_blocking=True)
                self.d2[r0:r1].copy_(self.h2[r0:r1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.up)
                self.events.append(ev)

    def event_for(self, row_end: int):
        """Event after which rows [0, row_end) are on the device (submits chunks as needed)."""
        i = next((k for k, e in enumerate(self.ends) if e >= row_end), len(self.ends) - 1)
        self._submit(i + self.lookahead)
        return self.events[i]

    def finish(self):
        """Submit every remaining chunk; the event of the last one."""
        self._submit(len(self.ends) - 1)
        return self.events[-1] if self.events else None


def _rows(a, s0: int, s1: int):
    """Row slice of a numpy array or (pinned) torch tensor, without a host copy."""
    return a[s0:s1]


def forward_stacks(view1, view2, bank: FilterBank, executor=None):
    """(B, p, q) views through every layer -> (B, n_maps, p', q') each (cascade.py:226-235)."""
    import torch

    ex = _executor(executor)
    v1 = np.asarray(view1)
    b = v1.shape[0]
    with torch.cuda.stream(ex.stream):
        layers = device_layers(bank, ex)
        m1 = E.forward_maps(ex, _to_dev32(ex, v1), layers, 1)
        m2 = E.forward_maps(ex, _to_dev32(ex, view2), layers, 2)
        r1 = m1.reshape(b, -1, m1.shape[1], m1.shape[2]).cpu().numpy().astype(np.float64)
        r2 = m2.reshape(b, -1, m2.shape[1], m2.shape[2]).cpu().numpy().astype(np.float64)
    return r1, r2


def forward(ds, bank: FilterBank, executor, batch: BatchSpec) -> LayerOutput:
    """Final-layer maps for the whole dataset (cascade.py:238-259)."""
    v1, v2, lab = ds.stacks_view()
    parts = [forward_stacks(np.asarray(v1)[r.start:r.stop], np.asarray(v2)[r.start:r.stop], bank, executor)
             for r in batch_partition(len(ds), batch)]
    lineage = ((),)
    for layer in bank.layers:
        lineage = _child_lineage(lineage, layer.count)
    return LayerOutput(maps1=np.concatenate([a for a, _ in parts]), maps2=np.concatenate([b for _, b in parts]),
                       labels=np.asarray(lab), lineage=lineage)
