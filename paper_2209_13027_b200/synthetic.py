"""Seeded synthetic two-view corpora for tests and the benchmark.

Generalizes the reference generator (synthetic.py:20-71: Gaussian blobs,
class k mod C, amplitude U(0.75, 1), round bumps for even classes and
elongated diagonal ones for odd classes, optional clipped Gaussian noise) to
rectangular p x q images, vectorized over samples. Second views follow
BASELINE.md: LBP of view 1 (ORL, views.py:41-58), an independently rendered
second channel (ETH-80), or a correlated plane (Caltech / 3-stage). Values
are float32 in [0, 1] — the device path's storage type; the CPU oracle is
fed the same float32 values.
"""

from __future__ import annotations

import numpy as np

_LBP_OFFSETS = ((-1, -1), (-1, 0), (-1, 1), (0, 1), (1, 1), (1, 0), (1, -1), (0, -1))


def blob_images(n: int, p: int, q: int, classes: int, seed: int = 0, noise: float = 0.02, chunk: int = 2048):
    """(n, p, q) float32 blob images and int64 labels k mod classes."""
    rng = np.random.default_rng(seed)
    ang = 2.0 * np.pi * np.arange(classes) / classes + np.pi / 4.0
    cy0 = p / 2.0 + (p / 4.0) * np.sin(ang)
    cx0 = q / 2.0 + (q / 4.0) * np.cos(ang)
    s = float(min(p, q))
    labels = np.arange(n) % classes
    # per-sample parameters drawn up front (deterministic for any chunking)
    jy = rng.normal(0.0, p / 32.0, n)
    jx = rng.normal(0.0, q / 32.0, n)
    amp = rng.uniform(0.75, 1.0, n)
    f1 = rng.uniform(0.9, 1.1, n)
    f2 = rng.uniform(0.9, 1.1, n)
    even = labels % 2 == 0
    su = np.where(even, s / 6.0 * f1, s / 4.0 * f1)
    sv = np.where(even, s / 6.0 * f1, s / 10.0 * f2)
    cy = cy0[labels] + jy
    cx = cx0[labels] + jx
    yy = np.arange(p, dtype=np.float64)[None, :, None]
    xx = np.arange(q, dtype=np.float64)[None, None, :]
    out = np.empty((n, p, q), dtype=np.float32)
    nrng = np.random.default_rng(seed + 0x9E3779B9)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        dy = yy - cy[a:b, None, None]
        dx = xx - cx[a:b, None, None]
        ev = even[a:b, None, None]
        r2 = np.sqrt(0.5)
        u = np.where(ev, dy, (dy + dx) * r2)
        v = np.where(ev, dx, (dy - dx) * r2)
        img = amp[a:b, None, None] * np.exp(-(u * u) / (2.0 * su[a:b, None, None] ** 2)
                                            - (v * v) / (2.0 * sv[a:b, None, None] ** 2))
        img = np.clip(img, 0.0, 1.0)
        if noise > 0:
            img = np.clip(img + nrng.normal(0.0, noise, img.shape), 0.0, 1.0)
        out[a:b] = img.astype(np.float32)
    return out, labels.astype(np.int64)


def blob_images_device(n: int, p: int, q: int, classes: int, seed: int = 0, noise: float = 0.02, device="cuda",
                       start: int = 0, stop: int | None = None, chunk: int = 4096):
    """Same blob model rendered with torch on ``device`` (benchmark-scale corpora).

    Per-sample parameters come from the same numpy stream as blob_images;
    noise comes from a torch generator, so pixel values differ from the
    numpy renderer (both are valid draws of the model). ``start``/``stop``
    render only a sample range (a rank's shard) with identical parameters.
    Returns (float32 tensor (stop-start, p, q) on device, int64 numpy labels).
    """
    import torch

    stop = n if stop is None else stop
    rng = np.random.default_rng(seed)
    ang = 2.0 * np.pi * np.arange(classes) / classes + np.pi / 4.0
    cy0 = p / 2.0 + (p / 4.0) * np.sin(ang)
    cx0 = q / 2.0 + (q / 4.0) * np.cos(ang)
    s = float(min(p, q))
    labels = np.arange(n) % classes
    jy = rng.normal(0.0, p / 32.0, n)
    jx = rng.normal(0.0, q / 32.0, n)
    amp = rng.uniform(0.75, 1.0, n)
    f1 = rng.uniform(0.9, 1.1, n)
    f2 = rng.uniform(0.9, 1.1, n)
    even = labels % 2 == 0
    su = np.where(even, s / 6.0 * f1, s / 4.0 * f1)
    sv = np.where(even, s / 6.0 * f1, s / 10.0 * f2)
    cy = cy0[labels] + jy
    cx = cx0[labels] + jx
    dev = torch.device(device)
    par = {k: torch.from_numpy(v[start:stop].astype(np.float32)).to(dev)
           for k, v in dict(cy=cy, cx=cx, amp=amp, su=su, sv=sv, even=even.astype(np.float32)).items()}
    yy = torch.arange(p, dtype=torch.float32, device=dev)[None, :, None]
    xx = torch.arange(q, dtype=torch.float32, device=dev)[None, None, :]
    out = torch.empty((stop - start, p, q), dtype=torch.float32, device=dev)
    r2 = float(np.sqrt(0.5))
    for a in range(0, stop - start, chunk):
        b = min(stop - start, a + chunk)
        P = {k: v[a:b, None, None] for k, v in par.items()}
        dy, dx = yy - P["cy"], xx - P["cx"]
        u = torch.where(P["even"] > 0, dy, (dy + dx) * r2)
        v = torch.where(P["even"] > 0, dx, (dy - dx) * r2)
        img = (P["amp"] * torch.exp(-(u * u) / (2 * P["su"] ** 2) - (v * v) / (2 * P["sv"] ** 2))).clamp_(0, 1)
        if noise > 0:
            g = torch.Generator(device=dev)
            g.manual_seed(seed * 1000003 + (start + a))
            img = (img + noise * torch.randn(img.shape, generator=g, device=dev)).clamp_(0, 1)
        out[a:b] = img
    return out, labels[start:stop].astype(np.int64)


def second_view_device(view1, kind: str, seed: int = 1, noise: float = 0.02, executor=None):
    """Torch version of second_view for 'pair' and 'lbp' (device tensors)."""
    import torch

    if kind == "lbp":
        from .execution import Executor
        from .views import lbp_stack

        ex = executor if executor is not None else Executor(device=view1.device)
        return lbp_stack(view1, ex)  # the ddcca_lbp kernel (views.py:41-58), on view1's device
    if kind in ("pair", "channel"):
        sm = view1.clone()
        sm[:, 1:-1, 1:-1] = (view1[:, :-2, 1:-1] + view1[:, 2:, 1:-1] + view1[:, 1:-1, :-2] + view1[:, 1:-1, 2:]
                             + view1[:, 1:-1, 1:-1]) / 5.0
        g = torch.Generator(device=view1.device)
        g.manual_seed(seed)
        return (0.8 * sm ** 1.5 + noise * torch.randn(view1.shape, generator=g, device=view1.device)).clamp_(0, 1)
    raise ValueError(f"unknown second-view kind {kind!r}")


def lbp_maps(imgs: np.ndarray) -> np.ndarray:
    """8-neighbour LBP / 255 of each image (views.py:41-58): strict >, clockwise from top-left, zero pad."""
    x = np.asarray(imgs, dtype=np.float64)
    n, p, q = x.shape
    pad = np.zeros((n, p + 2, q + 2))
    pad[:, 1:-1, 1:-1] = x
    code = np.zeros((n, p, q))
    for bit, (dy, dx) in enumerate(_LBP_OFFSETS):
        code += float(1 << bit) * (pad[:, 1 + dy:1 + dy + p, 1 + dx:1 + dx + q] > x)
    return (code / 255.0).astype(np.float32)


def second_view(view1: np.ndarray, labels: np.ndarray, kind: str, classes: int, seed: int = 1,
                noise: float = 0.02) -> np.ndarray:
    """Second view by config: 'lbp' (ORL), 'channel' (ETH-80), 'pair' (Caltech / 3-stage)."""
    n, p, q = view1.shape
    if kind == "lbp":
        return lbp_maps(view1)
    rng = np.random.default_rng(seed)
    if kind == "channel":
        other, _ = blob_images(n, p, q, classes, seed=seed + 17, noise=noise)
        return np.clip(0.6 * view1 + 0.4 * other, 0.0, 1.0).astype(np.float32)
    if kind == "pair":
        # correlated plane: smoothed, rescaled copy of view 1 plus independent noise
        sm = view1.astype(np.float64).copy()
        sm[:, 1:-1, 1:-1] = (view1[:, :-2, 1:-1] + view1[:, 2:, 1:-1] + view1[:, 1:-1, :-2] + view1[:, 1:-1, 2:]
                             + view1[:, 1:-1, 1:-1]) / 5.0
        out = np.empty_like(view1)
        for a in range(0, n, 2048):
            b = min(n, a + 2048)
            out[a:b] = np.clip(0.8 * sm[a:b] ** 1.5 + rng.normal(0.0, noise, (b - a, p, q)), 0.0, 1.0)
        return out.astype(np.float32)
    raise ValueError(f"unknown second-view kind {kind!r}")


# Benchmark configurations (BASELINE.json `configs`, unstated parameters pinned in SURVEY.md §8(d)).
CONFIGS = {
    "orl": dict(m=400, p=112, q=92, classes=40, layers=((8, 5, 5), (8, 5, 5)), block=(7, 7), view2="lbp"),
    "eth80": dict(m=3280, p=128, q=128, classes=8, layers=((8, 7, 7), (8, 7, 7)), block=(16, 16), view2="channel"),
    "caltech256": dict(m=30607, p=128, q=128, classes=257, layers=((8, 7, 7), (8, 7, 7)), block=(16, 16),
                       view2="pair"),
    "caltech256x10": dict(m=306070, p=128, q=128, classes=257, layers=((8, 7, 7), (8, 7, 7)), block=(16, 16),
                          view2="pair"),
    "three_stage": dict(m=2048, p=256, q=256, classes=257, layers=((12, 9, 9), (12, 9, 9), (12, 9, 9)),
                        block=(32, 32), view2="pair"),
}


def make_corpus(name: str, m: int | None = None, seed: int = 0):
    """(view1, view2, labels, cfg) for a named configuration (optionally the first m samples)."""
    cfg = dict(CONFIGS[name])
    n = cfg["m"] if m is None else m
    v1, lab = blob_images(n, cfg["p"], cfg["q"], cfg["classes"], seed=seed)
    v2 = second_view(v1, lab, cfg["view2"], cfg["classes"], seed=seed + 1)
    return v1, v2, lab, cfg
