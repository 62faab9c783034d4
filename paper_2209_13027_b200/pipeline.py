"""Transform entry point and stage timing.

``compute_features`` restates pipeline.py:61-86 of the reference: forward +
encode every sample, batch by batch, returning an (M, featlen) float64
matrix. Here the whole transform is device work (engine.Engine); the
float64 matrix is produced on the device by a LUT expansion of the integer
block counts and copied out once. ``compute_feature_counts`` returns the
lossless integer form (u8 / saturating u8 / u16 block counts) and is what
large runs and the benchmark keep in HBM or stream to the host.
"""

from __future__ import annotations

import sys
import time
from contextlib import contextmanager

import numpy as np

from . import engine as E
from .cascade import _executor, _to_dev32, device_layers


def log(stage: str, message: str) -> None:
    print(f"[{stage}] {message}", file=sys.stderr)


class StageTimer:
    """perf_counter stage timing with stage-tagged failure logs (pipeline.py:44-58)."""

    def __init__(self):
        self.seconds: dict[str, float] = {}

    @contextmanager
    def stage(self, name: str):
        t0 = time.perf_counter()
        try:
            yield
        except BaseException as e:
            log(name, f"failed after {time.perf_counter() - t0:.3f} s: {e}")
            raise
        self.seconds[name] = self.seconds.get(name, 0.0) + time.perf_counter() - t0
        log(name, f"done in {self.seconds[name]:.3f} s")


def _encoder_and_batch(config):
    enc = config.encoder
    batch = config.net.batch.batch_size if hasattr(config, "net") else 128
    return enc, batch


def compute_feature_counts(ds, bank, config, executor=None, host_out=None):
    """Device block counts plus the BlockPlan for this rank's samples.

    World size 1: all samples. With a process group, the rank's batch shard
    (the same contiguous shard train_network used), rows [s0, s1) of the
    dataset. ``host_out``: optional pinned host tensor; counts are streamed into
    it super-batch by super-batch while the transform proceeds. The caller's
    current stream is ordered after those copies (synchronize it, or the device,
    before reading ``host_out``); the executor's stream is not, so a following fit
    overlaps the tail of the copies (PCIe is full duplex: the next upload and
    this download share no direction).
    """
    import torch

    from .patches import batch_partition

    ex = _executor(executor)
    enc, bs = _encoder_and_batch(config)
    n = ds.global_len
    gb = batch_partition(n, config.net.batch) if hasattr(config, "net") else [range(0, n)]
    mine = ex.shard(len(gb))
    s0 = gb[mine.start].start if len(mine) else ds.row_offset
    s1 = gb[mine.stop - 1].stop if len(mine) else ds.row_offset
    st = getattr(ds, "_device_state", None)
    with torch.cuda.stream(ex.stream):
        layers = device_layers(bank, ex)
        if st is not None and st["device"] == str(ex.device) and st["rows"] == (s0, s1) and st["bank"] == id(bank):
            eng = st["engine"]
            i1, i2 = st["images"]
        else:
            eng = E.Engine(ex)
            r1, r2, _ = ds.local_rows(s0, s1)
            i1 = _to_dev32(ex, r1)
            i2 = _to_dev32(ex, r2)
        counts, plan = eng.transform_counts(i1, i2, layers, enc, bs, host_out=host_out)
    handoff(ex, counts)
    if host_out is not None and eng.host_copy_done is not None:
        torch.cuda.current_stream(ex.device).wait_event(eng.host_copy_done)
    return counts, plan


def handoff(ex, *tensors) -> None:
    """Stream-ordered handoff of device results to the caller's current stream.

    The executor's stream is a non-blocking stream: without this, a caller that reads
    a returned tensor on its own stream (e.g. ``.cpu()`` on the default stream) could
    read it before the kernels writing it have finished.
    """
    import torch

    cur = torch.cuda.current_stream(ex.device)
    if cur != ex.stream:
        cur.wait_stream(ex.stream)
        for t in tensors:
            t.record_stream(cur)


def feature_rows(ds, config, executor=None) -> range:
    """Dataset rows whose features this rank's ``compute_features`` returns.

    ``range(0, M)`` without a process group; with one, the rank's contiguous
    batch shard (the samples train_network accumulated on this rank).
    """
    from .patches import batch_partition

    ex = _executor(executor)
    n = ds.global_len
    gb = batch_partition(n, config.net.batch) if hasattr(config, "net") else [range(0, n)]
    mine = ex.shard(len(gb))
    if not len(mine):
        return range(0, 0)
    return range(gb[mine.start].start, gb[mine.stop - 1].stop)


def compute_features(ds, bank, config, executor=None) -> np.ndarray:
    """Transform: (M, featlen) float64 IQ features, identical layout to the reference.

    Without a process group this is the reference's full (M, featlen) matrix
    (pipeline.py:61-86). Under a process group (world > 1) the transform is
    sharded like the fit: each rank returns only the rows of its batch shard,
    ``feature_rows(ds, config, executor)``, in dataset order — pair them with
    ``ds.labels[feature_rows(...)]``, or gather them yourself.
    """
    import torch

    ex = _executor(executor)
    enc, _ = _encoder_and_batch(config)
    counts, plan = compute_feature_counts(ds, bank, config, ex)
    with torch.cuda.stream(ex.stream):
        feats = E.Engine(ex).expand(counts, plan, enc)
        out = feats.cpu().numpy()
    return out


def write_feature_csv(path, counts, plan, enc, first_index: int = 0, threads: int = 16) -> None:
    """Feature CSV of run_extract (pipeline.py:143-166) from block counts, without float64 features.

    One line per sample: ``index,v0,v1,...`` with every value as Python's
    ``format(v, ".17g")`` of the IQ feature; the 17-digit strings of the
    bpc + 1 LUT values are formatted here once and the native writer
    (``ddcca_write_feature_csv``) copies them per count with ``threads``
    workers. ``counts``: (m, featlen) host array / tensor (u8, saturating u8
    or u16 as ``compute_feature_counts`` returns them).
    """
    import ctypes as C

    from . import _native

    c = counts.cpu().numpy() if hasattr(counts, "cpu") else np.asarray(counts)
    c = np.ascontiguousarray(c)
    kind = E.count_kind(plan.bpc)
    if kind == 2:
        c = c.view(np.uint16)
    lut = E.iq_lut(enc)
    strs = [format(float(v), ".17g").encode("ascii") for v in lut]
    arr = (C.c_char_p * len(strs))(*strs)
    lens = (C.c_int * len(strs))(*[len(x) for x in strs])
    rows, cols = c.shape
    _native.check(_native.load().ddcca_write_feature_csv(c.ctypes.data_as(C.c_void_p), kind, rows, cols, plan.bins,
                                                         plan.bpc, arr, lens, int(first_index), str(path).encode(),
                                                         int(threads)), "write_feature_csv")
