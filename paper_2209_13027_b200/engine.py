"""Device-resident DDCCANet fit/transform engine (the hot path).

Everything between the host inputs and the outputs runs as sm_100a kernels
from libddcca (csrc/*.cu) on the executor's stream; torch supplies device
memory, streams and torch.distributed (NCCL) for the one exchange per layer.

Fit (cascade.train_network, cascade.py:207-223) per layer i:
  for each super-batch of whole sample batches on this rank:
    maps_i = forward through layers < i            (ddcca_conv, recomputed)
    partials[b] = moments of batch b               (ddcca_moments_partial)
  merged = fixed tree over all batches             (ddcca_moments_tree; NCCL
                                                    all_gather or all_reduce)
  layer_i = finalize + solve                       (ddcca_solve, 1 CTA FP64)
Transform (pipeline.compute_features, pipeline.py:61-86):
  for each super-batch: maps = forward through layers < S; last layer conv
  fused with sign-hash (ddcca_conv_hash) -> block histograms
  (ddcca_block_hist) written straight into the (M, featlen) count matrix;
  optional LUT expansion to the reference's float64 features
  (ddcca_iq_expand).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigError, ShapeError
from .patches import PatchGeometry

MAP_BUDGET_BYTES = 6 << 30  # per view, per super-batch (deepest layer input)
KEEP_MAPS_BYTES = 48 << 30  # fit keeps the last layer's input maps (both views) for the transform if they fit
MOMENTS_F32_BLOCKS = 1  # ddcca.h DDCCA_MOMENTS_F32_BLOCKS
MOMENTS_FINE_SPLITS = 2  # ddcca.h DDCCA_MOMENTS_FINE_SPLITS
FINE_ALL_MAPS = 8192  # fits with fewer maps per view at a layer use 32-map splits there too
HOST_CHUNK_BATCHES = 4  # sample batches per streamed device->host count copy



def _torch():
    import torch

    return torch


@dataclass
class DeviceLayer:
    """A trained layer kept on the device (float64 vectors + float32 conv packs)."""

    geom: PatchGeometry
    center: bool
    count: int
    w1: object  # torch float64 (d, count)
    w2: object
    rho: object  # torch float64 (count,)
    pack1: object  # torch float32 (d * count) tap-major
    pack2: object
    fin: object = None  # torch float64 (5, d, d): c11, c22, cw, cb, ctilde
    host1: object = None  # numpy float32 copies of the packs (constant-bank kernels)
    host2: object = None

    def pack(self, view: int):
        return self.pack1 if view == 1 else self.pack2

    def host_pack(self, view: int):
        return self.host1 if view == 1 else self.host2


# ----------------------------------------------------------------------------
# thin op wrappers (one C-ABI call each)
# ----------------------------------------------------------------------------

def payload_len(dim: int, classes: int) -> int:
    return int(_native.load().ddcca_payload_len(dim, classes))


def moments_partials(ex, maps1, maps2, map_labels, batch_offsets: np.ndarray, geom: PatchGeometry, center: bool,
                     classes: int, out=None, flags: int = 0):
    """Per-batch partial accumulators (n_batches, payload_len) float64 on device."""
    torch = _torch()
    lib = _native.load()
    n, p, q = maps1.shape
    if maps2.shape != maps1.shape:
        raise ShapeError(f"view map stacks differ: {tuple(maps1.shape)} vs {tuple(maps2.shape)}")
    offs = np.ascontiguousarray(batch_offsets, dtype=np.int64)
    nb = len(offs) - 1
    g = geom.native(p, q)
    max_maps = int(np.max(np.diff(offs)))
    ws_bytes = int(lib.ddcca_moments_workspace(C.byref(g), nb, max_maps, classes))
    plen = payload_len(geom.dim, classes)
    if out is None:
        out = torch.empty((nb, plen), dtype=torch.float64, device=ex.device)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=ex.device)
    rc = lib.ddcca_moments_partial_ex(_native.ptr(maps1), _native.ptr(maps2), _native.ptr(map_labels),
                                      offs.ctypes.data_as(C.POINTER(C.c_int64)), nb, C.byref(g), int(bool(center)),
                                      classes, _native.ptr(out), _native.ptr(ws), ws_bytes, int(flags),
                                      _native.stream_ptr(ex.stream))
    _native.check(rc, "moments")
    return out


def tree_merge(ex, parts):
    """Left-to-right pairwise tree over the rows of ``parts`` (moments.py:132-144); clobbers ``parts``."""
    torch = _torch()
    lib = _native.load()
    n, plen = parts.shape
    out = torch.empty(plen, dtype=torch.float64, device=ex.device)
    _native.check(lib.ddcca_moments_tree(_native.ptr(parts), n, plen, _native.ptr(out),
                                         _native.stream_ptr(ex.stream)), "pairwise_merge")
    return out


def solve_layer(ex, payload, geom: PatchGeometry, count: int, center: bool, classes: int, eps: float,
                check: bool = True) -> DeviceLayer:
    torch = _torch()
    lib = _native.load()
    d = geom.dim
    dev = ex.device
    fin = torch.empty((5, d, d), dtype=torch.float64, device=dev)
    w1 = torch.empty((d, count), dtype=torch.float64, device=dev)
    w2 = torch.empty((d, count), dtype=torch.float64, device=dev)
    rho = torch.empty(count, dtype=torch.float64, device=dev)
    pack1 = torch.empty(d * count, dtype=torch.float32, device=dev)
    pack2 = torch.empty(d * count, dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    ws_bytes = int(lib.ddcca_solve_workspace(d))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    rc = lib.ddcca_solve(_native.ptr(payload), d, classes, float(eps), count, _native.ptr(fin), _native.ptr(w1),
                         _native.ptr(w2), _native.ptr(rho), _native.ptr(pack1), _native.ptr(pack2),
                         _native.ptr(status), _native.ptr(ws), ws_bytes, _native.stream_ptr(ex.stream))
    _native.check(rc, "solve_dcca")
    layer = DeviceLayer(geom, bool(center), count, w1, w2, rho, pack1, pack2, fin)
    layer._status = status
    if check:
        check_layer(layer)
    return layer


def fetch_host_packs(layer: DeviceLayer) -> None:
    """Host copies of the float32 taps (tiny). The conv kernels read the device packs
    (ddcca_conv_dev / ddcca_conv_hist_dev); kept for callers of the host-pack entry points."""
    layer.host1 = np.ascontiguousarray(layer.pack1.cpu().numpy())
    layer.host2 = np.ascontiguousarray(layer.pack2.cpu().numpy())


def check_layer(layer: DeviceLayer) -> None:
    st = getattr(layer, "_status", None)
    if st is not None:
        _native.status_error(int(st.item()), "solve_dcca")


def check_layers(layers: list) -> None:
    """Solve statuses of all layers with one device->host read (the end of a fit)."""
    torch = _torch()
    sts = [lay._status for lay in layers if getattr(lay, "_status", None) is not None]
    if not sts:
        return
    for code in torch.cat(sts).cpu().tolist():
        _native.status_error(int(code), "solve_dcca")


def layer_from_filters(ex, filters1, filters2, geom: PatchGeometry, center: bool) -> DeviceLayer:
    """Upload host filter banks (L, l1, l2) as a DeviceLayer (for injected / loaded banks)."""
    torch = _torch()
    f1 = np.asarray(filters1, dtype=np.float64)
    f2 = np.asarray(filters2, dtype=np.float64)
    count = f1.shape[0]
    if f1.shape != f2.shape or f1.shape[1:] != (geom.l1, geom.l2):
        raise ShapeError(f"filter banks {f1.shape} / {f2.shape} do not match {geom.l1}x{geom.l2}")
    w1 = torch.from_numpy(np.ascontiguousarray(f1.reshape(count, -1).T)).to(ex.device)
    w2 = torch.from_numpy(np.ascontiguousarray(f2.reshape(count, -1).T)).to(ex.device)
    lib = _native.load()
    packs = []
    for w in (w1, w2):
        pk = torch.empty(geom.dim * count, dtype=torch.float32, device=ex.device)
        _native.check(lib.ddcca_pack_filters(_native.ptr(w), count, geom.dim, _native.ptr(pk),
                                             _native.stream_ptr(ex.stream)), "pack_filters")
        packs.append(pk)
    lay = DeviceLayer(geom, bool(center), count, w1, w2, None, packs[0], packs[1])
    lay.host1 = np.ascontiguousarray(f1.reshape(count, -1).T.astype(np.float32))
    lay.host2 = np.ascontiguousarray(f2.reshape(count, -1).T.astype(np.float32))
    return lay


def conv(ex, maps, layer: DeviceLayer, view: int, out=None):
    """(n, p, q) float32 -> (n, L, oh, ow) float32 filter-minor (apply_filters, cascade.py:108-126)."""
    torch = _torch()
    lib = _native.load()
    n, p, q = maps.shape
    oh, ow = layer.geom.out_shape(p, q)
    if out is None:
        out = torch.empty((n, layer.count, oh, ow), dtype=torch.float32, device=ex.device)
    g = layer.geom.native(p, q)
    # constant-bank kernel fed from the device pack (no host copy of the solve's taps)
    rc = lib.ddcca_conv_dev(_native.ptr(maps), n, C.byref(g), _native.ptr(layer.pack(view)), layer.count,
                            int(layer.center), _native.ptr(out), _native.stream_ptr(ex.stream))
    if rc == _native.OK:
        return out
    if rc != _native.ECONFIG:
        _native.check(rc, "conv")
    _native.check(lib.ddcca_conv(_native.ptr(maps), n, C.byref(g), _native.ptr(layer.pack(view)), layer.count,
                                 int(layer.center), _native.ptr(out), _native.stream_ptr(ex.stream)), "conv")
    return out


CONV_RESPONSES = 2  # include/ddcca.h DDCCA_CONV_RESPONSES


def conv_hist(ex, maps, layer: DeviceLayer, view: int, plan, counts_base, kind: int, groups_per_row: int,
              row_stride: int, group_stride: int, responses: bool = False) -> bool:
    """Fused last-layer conv + sign hash + block histograms; False if the shape is not covered."""
    lib = _native.load()
    if plan.sh != plan.bh or plan.sw != plan.bw:
        return False
    n, p, q = maps.shape
    g = layer.geom.native(p, q)
    rc = lib.ddcca_conv_hist_dev(_native.ptr(maps), n, C.byref(g), _native.ptr(layer.pack(view)), layer.count,
                                int(layer.center) | (CONV_RESPONSES if responses else 0), plan.bh, plan.bw,
                                _native.ptr(counts_base), kind, groups_per_row,
                                row_stride, group_stride, _native.stream_ptr(ex.stream))
    if rc == _native.ECONFIG:
        return False
    _native.check(rc, "conv_hist")
    return True


def conv_hash(ex, maps, layer: DeviceLayer, view: int, out=None):
    """Last-layer conv fused with sign-hash: (n, p, q) -> codes (n, oh, ow) u8/u16."""
    torch = _torch()
    lib = _native.load()
    n, p, q = maps.shape
    oh, ow = layer.geom.out_shape(p, q)
    dt = torch.uint8 if layer.count <= 8 else torch.int16
    if out is None:
        out = torch.empty((n, oh, ow), dtype=dt, device=ex.device)
    g = layer.geom.native(p, q)
    _native.check(lib.ddcca_conv_hash(_native.ptr(maps), n, C.byref(g), _native.ptr(layer.pack(view)), layer.count,
                                      int(layer.center), _native.ptr(out), _native.stream_ptr(ex.stream)),
                  "conv_hash")
    return out


def count_kind(bpc: int) -> int:
    """0: u8, 1: saturating u8 (decoded with the block sum), 2: u16."""
    if bpc <= 255:
        return 0
    if bpc <= 510:
        return 1
    return 2


def forward_maps(ex, images, layers: list, view: int):
    """forward_stacks for one view (cascade.py:226-235): (b, p, q) -> (b * n_maps, p', q')."""
    cur = images
    for layer in layers:
        n, p, q = cur.shape
        out = conv(ex, cur, layer, view)
        cur = out.view(n * layer.count, out.shape[2], out.shape[3])
    return cur


# ----------------------------------------------------------------------------
# encoder geometry
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class BlockPlan:
    bh: int
    bw: int
    sh: int
    sw: int
    nby: int
    nbx: int
    n_bits: int

    @property
    def blocks(self) -> int:
        return self.nby * self.nbx

    @property
    def bins(self) -> int:
        return 1 << self.n_bits

    @property
    def bpc(self) -> int:
        return self.bh * self.bw


def block_plan(enc, p: int, q: int, n_bits: int) -> BlockPlan:
    """EncoderConfig.block_starts (encoder.py:38-44) as a regular grid; Python round() = banker's."""
    sh = max(1, int(round((1.0 - enc.overlap) * enc.block_h)))
    sw = max(1, int(round((1.0 - enc.overlap) * enc.block_w)))
    if p < enc.block_h or q < enc.block_w:
        raise ShapeError(f"{enc.block_h}x{enc.block_w} blocks do not fit a {p}x{q} map")
    nby = len(range(0, p - enc.block_h + 1, sh))
    nbx = len(range(0, q - enc.block_w + 1, sw))
    return BlockPlan(enc.block_h, enc.block_w, sh, sw, nby, nbx, n_bits)


def iq_lut(enc) -> np.ndarray:
    """Feature value for each count 0..bpc, bitwise equal to encoder.py:87-97 (same numpy log)."""
    bpc = enc.block_h * enc.block_w
    lut = np.empty(bpc + 1)
    lut[0] = 0.0 if enc.zero_bin_policy == "zero" else float(np.log(2.0 * bpc))
    lut[1:] = -np.log(np.arange(1, bpc + 1) / bpc)
    return lut


# ----------------------------------------------------------------------------
# Engine
# ----------------------------------------------------------------------------

@dataclass
class FitResult:
    layers: list
    stats: list = field(default_factory=list)  # per layer: merged payload (device)


class Engine:
    """Fit + transform on device for one executor (one GPU, one sample shard)."""

    def __init__(self, executor, map_budget_bytes: int = MAP_BUDGET_BYTES, keep_maps_bytes: int = KEEP_MAPS_BYTES):
        self.ex = executor
        self.budget = map_budget_bytes
        self.uploader = None  # cascade.ChunkedUpload of an in-flight chunked image upload
        self.n_global_fit = None  # global sample count of the fit in progress (moments_flags)
        self.keep_maps_bytes = keep_maps_bytes
        self.maps_cache = None  # last hidden layer's maps of the fitted shard, reused by the transform
        self.profile = None   # dict name -> [(start_event, end_event)] when profiling
        self.work = {}        # name -> algorithmic work of one call (for the roofline)
        self.launches = 0     # kernels launched by this engine
        self.host_copy_done = None  # event of the last streamed device->host count copy

    def _timed(self, name: str, kernels: int, work: dict | None, fn, *a, **k):
        torch = _torch()
        torch.cuda.nvtx.range_push(name)  # stage ranges for nsys / ncu --nvtx (no-ops otherwise)
        try:
            return self._timed_body(name, kernels, work, fn, *a, **k)
        finally:
            torch.cuda.nvtx.range_pop()

    def _timed_body(self, name: str, kernels: int, work: dict | None, fn, *a, **k):
        self.launches += kernels
        if work is not None and self.profile is not None:
            acc = self.work.setdefault(name, {"kind": work.get("kind"), "flops": 0.0, "bytes": 0.0, "calls": 0})
            acc["flops"] += work.get("flops", 0.0)
            acc["bytes"] += work.get("bytes", 0.0)
            if "gram_flops" in work:
                acc["gram_flops"] = acc.get("gram_flops", 0.0) + work["gram_flops"]
            acc["calls"] += 1
        if self.profile is None:
            return fn(*a, **k)
        torch = _torch()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(self.ex.stream)
        out = fn(*a, **k)
        e.record(self.ex.stream)
        self.profile.setdefault(name, []).append((s, e))
        return out

    def _forward(self, images, layers: list, view: int, out=None):
        """Maps after ``layers`` (filter-minor); ``out`` receives the last layer's output."""
        cur = images
        for li, layer in enumerate(layers):
            n, p, q = cur.shape
            oh, ow = layer.geom.out_shape(p, q)
            fl = 2.0 * n * oh * ow * layer.count * layer.geom.dim
            by = 4.0 * n * (p * q + layer.count * oh * ow)
            dst = out.view(n, layer.count, oh, ow) if (out is not None and li == len(layers) - 1) else None
            name = f"conv_l{li + 1}"
            res = self._timed(name, 1, {"kind": "fma", "flops": fl, "bytes": by}, conv, self.ex, cur,
                              layer, view, dst)
            if self.profile is not None and _native.load().ddcca_conv_last_path() == 1:
                # tcgen05 responses kernel (convtc.cu): HBM-bound (responses written back);
                # executed tensor work as the conv-histogram's: 3 MMAs M128 N64 K16 per tap row
                # and 8-column block, 128-row tiles
                acc = self.work[name]
                acc["kind"] = "hbm"
                acc["tensor_flops"] = acc.get("tensor_flops", 0.0) + (
                    2.0 * 128 * 64 * 16 * 3 * layer.geom.l1 * (-(-q // 8)) * (-(-p // 128)) * n)
            cur = res.view(n * layer.count, oh, ow)
        return cur

    def _cache_key(self, images1, layers: list):
        return (images1.data_ptr(), tuple(images1.shape), tuple(id(l) for l in layers))

    def cached_maps(self, images1, layers: list):
        c = self.maps_cache
        if c is not None and c["key"] == self._cache_key(images1, layers):
            return c
        return None

    # -- helpers -------------------------------------------------------------
    def _superbatches(self, batch_ranges: list, bytes_per_sample: int):
        """Group consecutive sample batches so one group's deepest maps fit the budget."""
        groups, cur, cur_n = [], [], 0
        for r in batch_ranges:
            n = len(r)
            if cur and (cur_n + n) * bytes_per_sample > self.budget:
                groups.append(cur)
                cur, cur_n = [], 0
            cur.append(r)
            cur_n += n
        if cur:
            groups.append(cur)
        return groups

    @staticmethod
    def _split_at(groups: list, ends: list, first_sample: int) -> list:
        """Split batch groups so no group crosses an upload-chunk boundary (local row ``ends``)."""
        out = []
        for g in groups:
            cur, cur_chunk = [], None
            for r in g:
                chunk = next(i for i, e in enumerate(ends) if e >= r.stop - first_sample)
                if cur and chunk != cur_chunk:
                    out.append(cur)
                    cur = []
                cur.append(r)
                cur_chunk = chunk
            if cur:
                out.append(cur)
        return out

    @staticmethod
    def _maps_per_sample(layers: list) -> int:
        return int(np.prod([lay.count for lay in layers])) if layers else 1

    def _shape_after(self, p: int, q: int, layers: list):
        for lay in layers:
            p, q = lay.geom.out_shape(p, q)
        return p, q

    # -- fit -------------------------------------------------------------------
    def layer_partials(self, images1, images2, labels, layers: list, geom: PatchGeometry, center: bool,
                       classes: int, batch_ranges: list, first_sample: int = 0, keep: bool = False):
        """Per-batch partial moments for the given (local) batches; returns (n_batches, plen).

        ``keep``: also retain this layer's input maps for the whole shard (when they fit
        ``keep_maps_bytes``) so the transform does not recompute them.
        """
        torch = _torch()
        ex = self.ex
        m_local, p0, q0 = images1.shape
        p, q = self._shape_after(p0, q0, layers)
        n_in = self._maps_per_sample(layers)
        plen = payload_len(geom.dim, classes)
        parts = torch.empty((len(batch_ranges), plen), dtype=torch.float64, device=ex.device)
        keep_buf = None
        if keep and layers and 2 * m_local * n_in * p * q * 4 <= self.keep_maps_bytes:
            self.maps_cache = None
            keep_buf = (torch.empty((m_local * n_in, p, q), dtype=torch.float32, device=ex.device),
                        torch.empty((m_local * n_in, p, q), dtype=torch.float32, device=ex.device))
        row = 0
        groups = self._superbatches(batch_ranges, n_in * p * q * 4)
        up = self.uploader if not layers else None
        if up is not None:
            # images still arriving (train_network's chunked upload): one group per upload
            # chunk, each waiting only for its own rows, so the copies overlap the moments
            groups = self._split_at(groups, up.ends, first_sample)
        for group in groups:
            s0, s1 = group[0].start - first_sample, group[-1].stop - first_sample
            if up is not None:
                ex.stream.wait_event(up.event_for(s1))
            if keep_buf is not None:
                m1 = self._forward(images1[s0:s1], layers, 1, out=keep_buf[0][s0 * n_in:s1 * n_in])
                m2 = self._forward(images2[s0:s1], layers, 2, out=keep_buf[1][s0 * n_in:s1 * n_in])
            else:
                m1 = self._forward(images1[s0:s1], layers, 1)
                m2 = self._forward(images2[s0:s1], layers, 2)
            mlab = labels[s0:s1].repeat_interleave(n_in) if n_in > 1 else labels[s0:s1]
            offs = np.cumsum([0] + [len(r) * n_in for r in group], dtype=np.int64)
            nmaps = int(offs[-1])
            # algorithmic work: one DFMA per (own pixel, canonical lag), both views; the
            # full-GEMM convention of the same statistics (2 d^2 per patch) as "gram_flops"
            lags = geom.l1 * (2 * geom.l2 - 1) - (geom.l2 - 1)
            fl = 2.0 * 2 * nmaps * p * q * lags
            oh, ow = geom.out_shape(p, q)
            gfl = 2.0 * 2 * nmaps * oh * ow * geom.dim * geom.dim
            # the blocked form (layers >= 2 by default) runs the lag products as FP32 FMAs
            kind = "fma" if self.moments_flags(layers) & MOMENTS_F32_BLOCKS else "fp64"
            self._timed(f"moments_l{len(layers) + 1}", 5, {"kind": kind, "flops": fl, "gram_flops": gfl,
                                                          "bytes": 8.0 * nmaps * p * q},
                        moments_partials, ex, m1, m2, mlab, offs, geom, center, classes,
                        out=parts[row:row + len(group)], flags=self.moments_flags(layers))
            row += len(group)
        if keep_buf is not None:
            self.maps_cache = {"key": self._cache_key(images1, layers), "m1": keep_buf[0], "m2": keep_buf[1],
                               "n_in": n_in}
        return parts

    def moments_flags(self, layers: list) -> int:
        """Float32-blocked lag products for layers fed by filter responses (ExecSettings.moments);
        32-map splits (4x the CTAs) for the first layer (one map per sample) and for every layer
        of a small fit (fewer than FINE_ALL_MAPS maps per view at the layer, all ranks together:
        their lag grids would not fill the GPU). Both depend only on the layer and the global
        sample count, never on how batches are grouped into calls or ranks, so the partials stay
        bitwise independent of the GPU count."""
        mode = getattr(self.ex.settings, "moments", "blocked")
        flags = MOMENTS_F32_BLOCKS if (layers and mode == "blocked") else 0
        n = self.n_global_fit
        if not layers or (n is not None and n * self._maps_per_sample(layers) < FINE_ALL_MAPS):
            flags |= MOMENTS_FINE_SPLITS
        return flags

    def reduce_partials(self, parts, n_global_batches: int, local_batches: range):
        """Merged accumulator over all ranks' batches (fixed tree or sum-allreduce)."""
        torch = _torch()
        ex = self.ex
        levels = max(1, int(math.ceil(math.log2(max(parts.shape[0], 1))))) if parts.shape[0] > 1 else 0
        if ex.world_size == 1:
            return self._timed("tree", levels, None, tree_merge, ex, parts)
        if ex.deterministic:
            # every rank's per-batch partials in global batch order, same tree everywhere:
            # bitwise identical to the single-GPU result for any GPU count
            from .execution import gather_batch_partials

            with torch.cuda.stream(ex.stream):
                allp = gather_batch_partials(parts, n_global_batches, ex.world_size, ex.group)
            return tree_merge(ex, allp)
        from .execution import allreduce_partials

        with torch.cuda.stream(ex.stream):
            return allreduce_partials(parts, lambda t: tree_merge(ex, t), ex.group)

    def fit(self, images1, images2, labels, classes: int, layer_cfgs: list, batch_size: int, eps: float,
            n_global: int | None = None, first_sample: int = 0, keep_stats: bool = False,
            stage_hook=None) -> FitResult:
        """Train all layers. images*: (m_local, p, q) float32 device; labels: (m_local,) int32 device.

        ``n_global`` / ``first_sample`` describe the global sample set when this
        rank holds only its shard (samples [first_sample, first_sample + m_local)).
        """
        torch = _torch()
        ex = self.ex
        m_local = images1.shape[0]
        n_global = m_local if n_global is None else n_global
        self.n_global_fit = n_global  # fixes the split policy of every layer (moments_flags)
        gb = [range(s, min(s + batch_size, n_global)) for s in range(0, n_global, batch_size)]
        mine = ex.shard(len(gb))
        local = [gb[b] for b in mine]
        if local and (local[0].start != first_sample or local[-1].stop - first_sample != m_local):
            raise ShapeError("local images do not match this rank's batch shard")
        layers, stats = [], []
        with torch.cuda.stream(ex.stream):
            for i, cfg in enumerate(layer_cfgs):
                if stage_hook:
                    stage_hook(f"layer {i + 1}: accumulating moments over {len(gb)} batches")
                last = i == len(layer_cfgs) - 1
                parts = self.layer_partials(images1, images2, labels, layers, cfg.geom, cfg.center, classes, local,
                                            first_sample, keep=last and self.keep_maps_bytes > 0)
                merged = self.reduce_partials(parts, len(gb), mine)
                # no host round trip between layers: the next layer's convs read this
                # layer's taps from the device pack, statuses are checked once below
                layer = self._timed(f"solve_l{i + 1}", 3, None, solve_layer, ex, merged, cfg.geom, cfg.filters,
                                    cfg.center, classes, eps, check=False)
                layers.append(layer)
                if keep_stats:
                    stats.append(merged)
            check_layers(layers)
        if self.uploader is not None:
            ev = self.uploader.finish()  # (every chunk was reached by the first layer)
            if ev is not None:
                ex.stream.wait_event(ev)
            self.uploader = None
        return FitResult(layers, stats)

    # -- transform ---------------------------------------------------------
    def feature_geometry(self, p0: int, q0: int, layers: list, enc):
        p, q = self._shape_after(p0, q0, layers)
        n_bits = layers[-1].count
        if not 1 <= n_bits <= 16:
            raise ConfigError(f"device hashing supports 1..16 bit maps, got {n_bits}")
        plan = block_plan(enc, p, q, n_bits)
        groups = self._maps_per_sample(layers[:-1])
        featlen = 2 * groups * plan.blocks * plan.bins
        return plan, groups, featlen

    def transform_counts(self, images1, images2, layers: list, enc, batch_size: int, out=None, host_out=None,
                         sink=None):
        """(m, p, q) x2 -> per-sample block counts (m, featlen) u8/u16 on device.

        ``host_out`` (pinned host tensor of the same shape): each super-batch's counts
        are copied out on a side stream while the next super-batch is computed. The
        executor's stream does NOT wait for those copies (the next fit can start while the
        counts still stream out over PCIe); ``self.host_copy_done`` is the event that
        completes with the last copy (pipeline.compute_feature_counts hands it to the
        caller's stream).
        ``sink(s0, s1, counts)``: streaming consumer; the device buffer then holds
        one super-batch only (for outputs larger than HBM, e.g. the 3-stage config)
        and the returned tensor is that rolling buffer.
        """
        torch = _torch()
        ex = self.ex
        lib = _native.load()
        m, p0, q0 = images1.shape
        plan, groups, featlen = self.feature_geometry(p0, q0, layers, enc)
        kind = count_kind(plan.bpc)
        dt = torch.int16 if kind == 2 else torch.uint8
        ranges = [range(s, min(s + batch_size, m)) for s in range(0, m, batch_size)]
        pm, qm = self._shape_after(p0, q0, layers[:-1])
        per_view = groups * plan.blocks * plan.bins
        per_sample = max(groups * pm * qm * 4, featlen * (2 if kind == 2 else 1) if sink is not None else 0)
        supers = self._superbatches(ranges, per_sample)
        if host_out is not None:
            # small groups so each group's device->host copy overlaps the next group's kernels
            supers = [g[i:i + HOST_CHUNK_BATCHES] for g in supers for i in range(0, len(g), HOST_CHUNK_BATCHES)]
        if out is None:
            rows = max(g[-1].stop - g[0].start for g in supers) if sink is not None else m
            out = torch.empty((rows, featlen), dtype=dt, device=ex.device)
        cache = self.cached_maps(images1, layers[:-1])
        copy_stream = torch.cuda.Stream(device=ex.device) if host_out is not None else None
        with torch.cuda.stream(ex.stream):
            for group in supers:
                s0, s1 = group[0].start, group[-1].stop
                o0 = 0 if sink is not None else s0  # row offset inside `out`
                for view, imgs in ((1, images1), (2, images2)):
                    if cache is not None:
                        src = cache["m1"] if view == 1 else cache["m2"]
                        maps = src[s0 * groups:s1 * groups]
                    else:
                        maps = self._forward(imgs[s0:s1], layers[:-1], view)
                    last = layers[-1]
                    n, pp, qq = maps.shape
                    oh, ow = last.geom.out_shape(pp, qq)
                    fl = 2.0 * n * oh * ow * last.count * last.geom.dim
                    by = 4.0 * n * pp * qq + n * oh * ow * (1 if last.count <= 8 else 2)
                    base = out[o0:o0 + (s1 - s0)].view(-1)[(view - 1) * per_view:]
                    nb_cols = plan.nbx * plan.bw
                    fl_f = 2.0 * n * plan.nby * plan.bh * nb_cols * last.count * last.geom.dim
                    by_f = 4.0 * n * pp * qq + n * plan.blocks * plan.bins * out.element_size()
                    wk = {"kind": "fma", "flops": fl_f, "bytes": by_f}
                    if self._timed("conv_hist", 1, wk, conv_hist, ex, maps, last, view, plan, base, kind, groups,
                                   featlen, plan.blocks * plan.bins, len(layers) > 1):
                        if lib.ddcca_conv_hist_last_path() == 1 and self.profile is not None:
                            # tcgen05 f16 kernel (convtc.cu): 3 MMAs M128 x N(8 filters x 8 columns) x K16
                            # per tap row and 8-output-column block, 128-row tiles
                            blocks = -(-nb_cols // 8)
                            tiles = -(-pp // 128)
                            ex_fl = 2.0 * 128 * 64 * 16 * 3 * last.geom.l1 * blocks * tiles * n
                            acc = self.work["conv_hist"]
                            acc["kind"] = "tensor"
                            acc["tensor_flops"] = acc.get("tensor_flops", 0.0) + ex_fl
                        continue
                    codes = self._timed("conv_hash", 1, {"kind": "fma", "flops": fl, "bytes": by}, conv_hash, ex,
                                        maps, last, view)
                    hb = codes.numel() * codes.element_size() + n * plan.blocks * plan.bins * out.element_size()
                    self._timed("block_hist", 1, {"kind": "hbm", "bytes": float(hb)}, lambda: _native.check(
                        lib.ddcca_block_hist(
                            _native.ptr(codes), codes.element_size(), codes.shape[0], codes.shape[1],
                            codes.shape[2], plan.n_bits, plan.bh, plan.bw, plan.sh, plan.sw, _native.ptr(base),
                            kind, groups, featlen, plan.blocks * plan.bins, _native.stream_ptr(ex.stream)),
                        "block_hist"))
                if copy_stream is not None:
                    ev = torch.cuda.Event()
                    ev.record(ex.stream)
                    copy_stream.wait_event(ev)
                    with torch.cuda.stream(copy_stream):
                        host_out[s0:s1].copy_(out[o0:o0 + (s1 - s0)], non_blocking=True)
                if sink is not None:
                    sink(s0, s1, out[:s1 - s0])
            if copy_stream is not None:
                # the device buffer stays allocated until the copy stream is done with it
                out.record_stream(copy_stream)
                self.host_copy_done = torch.cuda.Event()
                self.host_copy_done.record(copy_stream)
        return out, plan

    def expand(self, counts, plan: BlockPlan, enc):
        """Counts -> float64 IQ features (iq_block_features values) on device."""
        torch = _torch()
        ex = self.ex
        lib = _native.load()
        lut = torch.from_numpy(iq_lut(enc)).to(ex.device)
        out = torch.empty(counts.shape, dtype=torch.float64, device=ex.device)
        nblk = counts.numel() // plan.bins
        _native.check(lib.ddcca_iq_expand(_native.ptr(counts), count_kind(plan.bpc), nblk, plan.n_bits, plan.bpc,
                                          _native.ptr(lut), _native.ptr(out), _native.stream_ptr(ex.stream)),
                      "iq_expand")
        return out


def decode_counts(counts: np.ndarray, plan: BlockPlan) -> np.ndarray:
    """Host-side view of device counts as exact integers (undo the saturating u8 form)."""
    c = np.asarray(counts)
    if c.dtype == np.int16:
        return c.view(np.uint16).astype(np.int64)
    c = c.astype(np.int64)
    if count_kind(plan.bpc) == 1:
        blk = c.reshape(-1, plan.bins)
        extra = plan.bpc - blk.sum(axis=1)
        sat = blk == 255
        blk[sat] += np.repeat(extra, sat.sum(axis=1))
        c = blk.reshape(c.shape)
    return c
