"""Numpy restatement of the ddccanet fit/transform path (TEST INFRASTRUCTURE ONLY).

See ``oracle/__init__.py`` for who may import this. Citations are to
/root/reference/pkg/src/ddccanet/<file>:<line>. The restatement keeps the
reference's arithmetic order where it matters for bit-level agreement
(float64 everywhere, BLAS Grams, per-class masked sums, Jacobi rotation
order) so that, on the same machine, most outputs agree bitwise with the
reference; the golden tests only require the tolerances in tests/.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

__all__ = [
    "OracleError", "OracleShapeError", "OracleConfigError", "OracleNumericalError",
    "Geometry", "im2col", "batch_ranges",
    "Acc", "acc_zeros", "acc_add_columns", "acc_merge", "acc_tree", "acc_finalize",
    "Finalized", "eig_sym", "inv_sqrt", "dcca_solve", "Pairs", "Layer", "to_layer",
    "conv_stack", "conv_plane", "layer_stats", "train", "forward_maps",
    "EncodeCfg", "block_origins", "sign_bits", "combine_bits", "block_iq",
    "encode_maps", "encode_pair", "feature_len", "features", "Pool",
    "iq_lut", "block_counts", "nn_predict", "nn_accuracy", "lbp",
]


class OracleError(Exception):
    """Base class for oracle-side validation failures."""


class OracleShapeError(OracleError):
    pass


class OracleConfigError(OracleError):
    pass


class OracleNumericalError(OracleError):
    pass


# --------------------------------------------------------------------------
# Patch geometry and im2col                                  (patches.py)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Geometry:
    """Window geometry; restates PatchGeometry (patches.py:22-65)."""

    l1: int
    l2: int
    stride: int = 1
    padding: str = "zero_same"

    def __post_init__(self):
        if self.l1 < 1 or self.l2 < 1 or self.stride < 1:
            raise OracleConfigError("bad geometry")
        if self.padding not in ("none", "zero_same"):
            raise OracleConfigError(f"padding {self.padding!r}")

    @property
    def dim(self) -> int:
        return self.l1 * self.l2

    def grid(self, p: int, q: int) -> tuple[int, int]:
        """Output grid; patches.py:41-52 (ceil division for zero_same)."""
        s = self.stride
        if self.padding == "zero_same":
            return (p + s - 1) // s, (q + s - 1) // s
        if p < self.l1 or q < self.l2:
            raise OracleShapeError("window larger than map without padding")
        return (p - self.l1) // s + 1, (q - self.l2) // s + 1

    def pads(self, p: int, q: int) -> tuple[int, int, int, int]:
        """(top, bottom, left, right); patches.py:54-65."""
        if self.padding == "none":
            return 0, 0, 0, 0
        oh, ow = self.grid(p, q)
        t = (self.l1 - 1) // 2
        lf = (self.l2 - 1) // 2
        b = max(0, (oh - 1) * self.stride + self.l1 - p - t)
        r = max(0, (ow - 1) * self.stride + self.l2 - q - lf)
        return t, b, lf, r


def im2col(maps: np.ndarray, geom: Geometry, center: bool) -> np.ndarray:
    """(N, p, q) maps -> (dim, N*oh*ow) patch columns; patches.py:97-125.

    Column order: map-major, then row-major window positions; row order is
    the row-major scan of the window. ``center`` subtracts each column's own
    mean, which counts the zero padding (padding precedes windowing).
    """
    maps = np.asarray(maps, dtype=np.float64)
    if maps.ndim == 2:
        maps = maps[None]
    if maps.ndim != 3:
        raise OracleShapeError(f"need (N, p, q), got {maps.shape}")
    n, p, q = maps.shape
    oh, ow = geom.grid(p, q)
    t, b, lf, r = geom.pads(p, q)
    if t or b or lf or r:
        src = np.zeros((n, p + t + b, q + lf + r))
        src[:, t:t + p, lf:lf + q] = maps
    else:
        src = maps
    win = sliding_window_view(src, (geom.l1, geom.l2), axis=(1, 2))[:, ::geom.stride, ::geom.stride]
    rows = win.reshape(n * oh * ow, geom.dim)
    rows = rows - rows.mean(axis=1, keepdims=True) if center else np.ascontiguousarray(rows)
    return rows.T


def batch_ranges(m: int, batch: int) -> list[range]:
    """Contiguous manifest-order batches; patches.py:148-157."""
    if m < 1:
        raise OracleConfigError("empty sample list")
    if batch < 1:
        raise OracleConfigError("batch size must be >= 1")
    return [range(s, min(s + batch, m)) for s in range(0, m, batch)]


# --------------------------------------------------------------------------
# Moments                                                    (moments.py)
# --------------------------------------------------------------------------

@dataclass
class Acc:
    """Streaming statistics; restates MomentAccumulator (moments.py:26-60)."""

    c11: np.ndarray
    c22: np.ndarray
    s1: np.ndarray  # (dim, classes)
    s2: np.ndarray
    g1: np.ndarray  # (dim,)
    g2: np.ndarray
    n: int
    n_class: np.ndarray  # (classes,) int64


def acc_zeros(dim: int, classes: int) -> Acc:
    """moments.py:34-48."""
    if dim < 1 or classes < 1:
        raise OracleConfigError("bad accumulator shape")
    z = np.zeros
    return Acc(z((dim, dim)), z((dim, dim)), z((dim, classes)), z((dim, classes)),
               z(dim), z(dim), 0, np.zeros(classes, dtype=np.int64))


def acc_add_columns(acc: Acc, x, y, labels) -> Acc:
    """Fold paired patch columns into ``acc`` in place; moments.py:86-110."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    lab = np.asarray(labels, dtype=np.int64)
    dim, classes = acc.c11.shape[0], acc.s1.shape[1]
    if x.ndim != 2 or y.ndim != 2 or x.shape != y.shape:
        raise OracleShapeError("view patch matrices differ")
    if x.shape[0] != dim:
        raise OracleShapeError("patch dim mismatch")
    if lab.shape != (x.shape[1],):
        raise OracleShapeError("one label per column")
    if lab.size and (lab.min() < 0 or lab.max() >= classes):
        raise OracleShapeError("label out of range")
    acc.c11 += x @ x.T
    acc.c22 += y @ y.T
    for c in np.unique(lab):
        sel = lab == c
        acc.s1[:, c] += x[:, sel].sum(axis=1)
        acc.s2[:, c] += y[:, sel].sum(axis=1)
        acc.n_class[c] += int(sel.sum())
    acc.g1 += x.sum(axis=1)
    acc.g2 += y.sum(axis=1)
    acc.n += x.shape[1]
    return acc


def acc_merge(a: Acc, b: Acc) -> Acc:
    """Non-mutating componentwise sum; moments.py:113-129."""
    if a.c11.shape != b.c11.shape or a.s1.shape != b.s1.shape:
        raise OracleShapeError("accumulator shapes differ")
    return Acc(a.c11 + b.c11, a.c22 + b.c22, a.s1 + b.s1, a.s2 + b.s2,
               a.g1 + b.g1, a.g2 + b.g2, a.n + b.n, a.n_class + b.n_class)


def acc_tree(parts) -> Acc:
    """Left-to-right pairwise tree fixed by list order; moments.py:132-144."""
    level = list(parts)
    if not level:
        raise OracleConfigError("nothing to merge")
    while len(level) > 1:
        paired = [acc_merge(level[i], level[i + 1]) for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            paired.append(level[-1])
        level = paired
    return level[0]


@dataclass(frozen=True)
class Finalized:
    """DiscriminantMoments (moments.py:63-76)."""

    c11: np.ndarray
    c22: np.ndarray
    cw: np.ndarray
    cb: np.ndarray
    ctilde: np.ndarray
    n: int


def acc_finalize(acc: Acc, eps: float = 1e-4) -> Finalized:
    """Cw = S1 S2', Cb = g1 g2' - Cw, Ct = Cw - Cb, ridge; moments.py:168-193."""
    if eps < 0:
        raise OracleConfigError("negative ridge")
    if acc.n < 1:
        raise OracleNumericalError("empty accumulator")
    cw = acc.s1 @ acc.s2.T
    cb = np.outer(acc.g1, acc.g2) - cw
    ct = cw - cb
    dim = acc.c11.shape[0]
    eye = np.eye(dim)
    a = 0.5 * (acc.c11 + acc.c11.T)
    b = 0.5 * (acc.c22 + acc.c22.T)
    a = a + eps * (np.trace(a) / dim) * eye
    b = b + eps * (np.trace(b) / dim) * eye
    return Finalized(a, b, cw, cb, ct, acc.n)


# --------------------------------------------------------------------------
# Solver                                                      (solver.py)
# --------------------------------------------------------------------------

_TOL = 1e-12
_SWEEPS = 100
_SCHEDULES: dict[int, list] = {}


def rr_schedule(n: int) -> list:
    """Round-robin tournament of disjoint pairs; solver.py:32-46."""
    if n in _SCHEDULES:
        return _SCHEDULES[n]
    m = n + (n % 2)
    seats = list(range(m))
    rounds = []
    for _ in range(m - 1):
        ps, qs = [], []
        for i in range(m // 2):
            u, v = seats[i], seats[m - 1 - i]
            if u < n and v < n:
                ps.append(min(u, v))
                qs.append(max(u, v))
        rounds.append((np.array(ps, dtype=np.intp), np.array(qs, dtype=np.intp)))
        seats = [seats[0], seats[-1]] + seats[1:-1]
    _SCHEDULES[n] = rounds
    return rounds


def col_signs(v: np.ndarray) -> np.ndarray:
    """Sign making each column's largest-|.| entry (first on ties) positive; solver.py:49-57."""
    pick = np.argmax(np.abs(v), axis=0)
    s = np.sign(v[pick, np.arange(v.shape[1])])
    s[s == 0] = 1.0
    return s


def order_runs(w: np.ndarray, v: np.ndarray):
    """Lexicographic order inside near-equal eigenvalue runs; solver.py:60-79.

    A run extends while |w[k] - w[run_start]| <= 1e-10 * max|w|.
    """
    n = len(w)
    tol = 1e-10 * (float(np.abs(w).max()) if n else 0.0)
    perm = np.arange(n)
    start = 0
    for k in range(1, n + 1):
        if k < n and abs(w[k] - w[start]) <= tol:
            continue
        if k - start > 1:
            idx = perm[start:k]
            keys = [tuple(v[:, j]) for j in idx]
            perm[start:k] = idx[np.array(sorted(range(len(idx)), key=keys.__getitem__))]
        start = k
    return w[perm], v[:, perm]


def offdiag(a: np.ndarray) -> float:
    """Frobenius norm of the off-diagonal part; solver.py:82-87."""
    b = a.copy()
    np.fill_diagonal(b, 0.0)
    return float(np.linalg.norm(b))


def eig_sym(s: np.ndarray):
    """Cyclic round-robin Jacobi, descending, sign- and run-normalized; solver.py:90-158."""
    s = np.asarray(s, dtype=np.float64)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise OracleShapeError("need a square matrix")
    n = s.shape[0]
    mx = float(np.abs(s).max())
    unit = s / mx if mx > 0.0 else s
    fro = mx * float(np.linalg.norm(unit)) if mx > 0.0 else 0.0
    if mx > 0.0 and np.linalg.norm(unit - unit.T) > 1e-10 * np.linalg.norm(unit):
        raise OracleShapeError("matrix is not symmetric")
    vec = np.eye(n)
    if n == 1 or mx == 0.0:
        d = np.diag(s).copy()
        o = np.argsort(-d, kind="stable")
        return d[o], vec[:, o]
    a = 0.5 * (unit + unit.T) * (mx / fro)
    done = False
    for _ in range(_SWEEPS):
        if offdiag(a) <= _TOL:
            done = True
            break
        for ps, qs in rr_schedule(n):
            apq = a[ps, qs]
            live = apq != 0.0
            if not live.any():
                continue
            theta = np.zeros_like(apq)
            np.divide(a[qs, qs] - a[ps, ps], 2.0 * apq, out=theta, where=live)
            with np.errstate(over="ignore"):
                t = np.where(theta >= 0.0, 1.0, -1.0) / (np.abs(theta) + np.sqrt(theta * theta + 1.0))
            c = 1.0 / np.sqrt(t * t + 1.0)
            sn = t * c
            c = np.where(live, c, 1.0)
            sn = np.where(live, sn, 0.0)
            rot = np.eye(n)
            rot[ps, ps] = c
            rot[qs, qs] = c
            rot[ps, qs] = sn
            rot[qs, ps] = -sn
            a = rot.T @ a @ rot
            vec = vec @ rot
        a = 0.5 * (a + a.T)
    if not done and offdiag(a) > _TOL:
        raise OracleNumericalError("Jacobi did not converge")
    d = np.diag(a).copy() * fro
    o = np.argsort(-d, kind="stable")
    d, vec = d[o], vec[:, o]
    vec = vec * col_signs(vec)
    return order_runs(d, vec)


def inv_sqrt(c: np.ndarray) -> np.ndarray:
    """V diag(w^-1/2) V', symmetrized; solver.py:161-170."""
    w, v = eig_sym(c)
    if w[-1] <= 0.0:
        raise OracleNumericalError("matrix is not positive definite")
    r = (v * (w ** -0.5)) @ v.T
    return 0.5 * (r + r.T)


@dataclass(frozen=True)
class Pairs:
    """CanonicalPairs (solver.py:173-183)."""

    w1: np.ndarray
    w2: np.ndarray
    rho: np.ndarray


def dcca_solve(m: Finalized, count: int) -> Pairs:
    """Whitened SVD via eig(TT'), sign rule, null completion; solver.py:216-257."""
    dim = m.c11.shape[0]
    if not 1 <= count <= dim:
        raise OracleConfigError("filter count out of range")
    r1 = inv_sqrt(m.c11)
    r2 = inv_sqrt(m.c22)
    t = r1 @ m.ctilde @ r2
    g = t @ t.T
    lam, u = eig_sym(0.5 * (g + g.T))
    sig = np.sqrt(np.clip(lam, 0.0, None))
    v = np.zeros((dim, count))
    nb = None
    nxt = dim - 1
    for k in range(count):
        if sig[k] > 1e-12 * max(sig[0], 1e-300):
            v[:, k] = (t.T @ u[:, k]) / sig[k]
        else:
            sig[k] = 0.0
            if nb is None:
                h = t.T @ t
                _, nb = eig_sym(0.5 * (h + h.T))
            v[:, k] = nb[:, nxt]
            nxt -= 1
    w1 = r1 @ u[:, :count]
    w2 = r2 @ v
    f = col_signs(w1)
    w1 = w1 * f
    w2 = w2 * f
    z = sig[:count] == 0.0
    if z.any():
        w2[:, z] = w2[:, z] * col_signs(w2[:, z])
    return Pairs(w1, w2, sig[:count].copy())


@dataclass(frozen=True)
class Layer:
    """FilterLayer (solver.py:186-197): (L, l1, l2) kernels per view."""

    f1: np.ndarray
    f2: np.ndarray
    geom: Geometry
    center: bool

    @property
    def count(self) -> int:
        return self.f1.shape[0]


def to_layer(pairs: Pairs, geom: Geometry, center: bool = True) -> Layer:
    """Row-major unflatten of each canonical vector; solver.py:260-272."""
    if pairs.w1.shape[0] != geom.dim:
        raise OracleShapeError("vector length does not match kernel size")
    L = pairs.w1.shape[1]
    return Layer(pairs.w1.T.reshape(L, geom.l1, geom.l2).copy(),
                 pairs.w2.T.reshape(L, geom.l1, geom.l2).copy(), geom, center)


# --------------------------------------------------------------------------
# Cascade                                                     (cascade.py)
# --------------------------------------------------------------------------

CHUNK = 1 << 17  # cascade.py:26


def _chunks(n: int, per_map: int) -> list[range]:
    """cascade.py:103-105."""
    k = max(1, CHUNK // max(per_map, 1))
    return [range(i, min(i + k, n)) for i in range(0, n, k)]


def conv_stack(stack: np.ndarray, layer: Layer, view: int) -> np.ndarray:
    """(N, p, q) -> (N, L, oh, ow), filter-minor; cascade.py:108-126."""
    stack = np.asarray(stack, dtype=np.float64)
    n, p, q = stack.shape
    oh, ow = layer.geom.grid(p, q)
    bank = (layer.f1 if view == 1 else layer.f2).reshape(layer.count, layer.geom.dim)
    out = np.empty((n, layer.count, oh, ow))
    for ch in _chunks(n, oh * ow):
        resp = bank @ im2col(stack[ch.start:ch.stop], layer.geom, layer.center)
        out[ch.start:ch.stop] = resp.reshape(layer.count, len(ch), oh, ow).transpose(1, 0, 2, 3)
    return out


def conv_plane(plane, kernel, padding="zero_same", center=False) -> np.ndarray:
    """Single-plane cross-correlation; cascade.py:93-100."""
    kernel = np.asarray(kernel, dtype=np.float64)
    g = Geometry(kernel.shape[0], kernel.shape[1], 1, padding)
    cols = im2col(np.asarray(plane, dtype=np.float64)[None], g, center)
    return (kernel.reshape(-1) @ cols).reshape(g.grid(*np.asarray(plane).shape))


class Pool:
    """Executor restatement (execution.py:26-68): ordered map on a thread pool."""

    def __init__(self, threads: int = 1, deterministic: bool = True):
        self.threads = threads
        self.deterministic = deterministic
        self._ex = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None

    def map(self, fn, items) -> list:
        if self._ex is None:
            return [fn(i) for i in items]
        return list(self._ex.map(fn, items))

    def close(self):
        if self._ex is not None:
            self._ex.shutdown(wait=True)
            self._ex = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def layer_stats(maps1, maps2, labels, geom: Geometry, center: bool, classes: int,
                batch: int, pool: Pool) -> Acc:
    """accumulate_layer_moments + _batch_accumulator_job; cascade.py:155-189.

    maps*: (M, n_maps, p, q); labels: (M,). One accumulator per sample batch,
    fixed chunk boundaries inside it, reduced through the fixed tree.
    """
    m_all, nm, p, q = maps1.shape
    oh, ow = geom.grid(p, q)

    def job(r: range) -> Acc:
        f1 = maps1[r.start:r.stop].reshape(-1, p, q)
        f2 = maps2[r.start:r.stop].reshape(-1, p, q)
        ml = np.repeat(np.asarray(labels)[r.start:r.stop], nm)
        acc = acc_zeros(geom.dim, classes)
        for ch in _chunks(f1.shape[0], oh * ow):
            acc_add_columns(acc, im2col(f1[ch.start:ch.stop], geom, center),
                            im2col(f2[ch.start:ch.stop], geom, center),
                            np.repeat(ml[ch.start:ch.stop], oh * ow))
        return acc

    parts = pool.map(job, batch_ranges(m_all, batch))
    if pool.deterministic:
        return acc_tree(parts)
    total = parts[0]
    for a in parts[1:]:
        total = acc_merge(total, a)
    return total


def _apply(maps1, maps2, layer: Layer, batch: int, pool: Pool):
    """apply_layer (cascade.py:133-152): materialize the next layer's maps."""
    m_all, nm, p, q = maps1.shape
    oh, ow = layer.geom.grid(p, q)

    def run(r: range):
        b = len(r)
        o1 = conv_stack(maps1[r.start:r.stop].reshape(-1, p, q), layer, 1)
        o2 = conv_stack(maps2[r.start:r.stop].reshape(-1, p, q), layer, 2)
        return o1.reshape(b, nm * layer.count, oh, ow), o2.reshape(b, nm * layer.count, oh, ow)

    parts = pool.map(run, batch_ranges(m_all, batch))
    return np.concatenate([a for a, _ in parts]), np.concatenate([b for _, b in parts])


def train(view1, view2, labels, classes: int, layers, batch: int = 128, eps: float = 1e-4,
          pool: Pool | None = None, return_stats: bool = False):
    """train_network / train_layer; cascade.py:192-223.

    ``layers`` is a sequence of (filters, Geometry, center). Returns a list of
    Layer (and, with ``return_stats``, the per-layer Acc and Finalized).
    """
    pool = pool or Pool()
    cur1 = np.asarray(view1, dtype=np.float64)[:, None]
    cur2 = np.asarray(view2, dtype=np.float64)[:, None]
    out, stats = [], []
    for i, (count, geom, center) in enumerate(layers):
        if count < 1 or count > geom.dim:
            raise OracleConfigError("filter count out of range")
        acc = layer_stats(cur1, cur2, labels, geom, center, classes, batch, pool)
        fin = acc_finalize(acc, eps)
        lay = to_layer(dcca_solve(fin, count), geom, center)
        out.append(lay)
        stats.append((acc, fin))
        if i + 1 < len(layers):
            cur1, cur2 = _apply(cur1, cur2, lay, batch, pool)
    return (out, stats) if return_stats else out


def forward_maps(view1, view2, layers):
    """forward_stacks (cascade.py:226-235): (B, p, q) -> (B, prod L, p', q') per view."""
    m1 = np.asarray(view1, dtype=np.float64)[:, None]
    m2 = np.asarray(view2, dtype=np.float64)[:, None]
    for lay in layers:
        b, n_in, p, q = m1.shape
        oh, ow = lay.geom.grid(p, q)
        m1 = conv_stack(m1.reshape(-1, p, q), lay, 1).reshape(b, n_in * lay.count, oh, ow)
        m2 = conv_stack(m2.reshape(-1, p, q), lay, 2).reshape(b, n_in * lay.count, oh, ow)
    return m1, m2


# --------------------------------------------------------------------------
# Encoder                                                     (encoder.py)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class EncodeCfg:
    """EncoderConfig (encoder.py:21-47)."""

    block_h: int
    block_w: int
    overlap: float = 0.0
    zero_bin_policy: str = "zero"

    def __post_init__(self):
        if self.block_h < 1 or self.block_w < 1:
            raise OracleConfigError("block must be >= 1x1")
        if not 0.0 <= self.overlap < 1.0:
            raise OracleConfigError("overlap outside [0, 1)")
        if self.zero_bin_policy not in ("zero", "floor"):
            raise OracleConfigError("bad zero-bin policy")


def block_origins(cfg: EncodeCfg, p: int, q: int) -> list[tuple[int, int]]:
    """Row-major block corners, partial blocks dropped; encoder.py:38-44 (banker's round)."""
    sh = max(1, int(round((1.0 - cfg.overlap) * cfg.block_h)))
    sw = max(1, int(round((1.0 - cfg.overlap) * cfg.block_w)))
    return [(i, j) for i in range(0, p - cfg.block_h + 1, sh) for j in range(0, q - cfg.block_w + 1, sw)]


def sign_bits(plane) -> np.ndarray:
    """Strict > 0; encoder.py:50-52."""
    return (np.asarray(plane) > 0).astype(np.int64)


def combine_bits(bits) -> np.ndarray:
    """LSB-first 2^l weights over the leading axis; encoder.py:55-68."""
    st = np.asarray(bits)
    if st.ndim != 3:
        raise OracleShapeError("need (L, p, q) bit maps")
    L = st.shape[0]
    if not 1 <= L <= 30:
        raise OracleConfigError("1..30 bit maps")
    w = 1 << np.arange(L, dtype=np.int64)
    return np.tensordot(w, st.astype(np.int64), axes=([0], [0]))


def iq_lut(cfg: EncodeCfg) -> np.ndarray:
    """Feature value per count 0..bpc, restating encoder.py:87-97 elementwise.

    lut[0] is the zero-bin value; lut[k] = -log(k / bpc). Bitwise equal to
    the reference's vectorized ``-np.log(counts / bpc)`` (same numpy ufuncs).
    """
    bpc = cfg.block_h * cfg.block_w
    z = 0.0 if cfg.zero_bin_policy == "zero" else float(np.log(2.0 * bpc))
    k = np.arange(bpc + 1)
    lut = np.empty(bpc + 1)
    lut[0] = z
    lut[1:] = -np.log(k[1:] / bpc)
    return lut


def block_counts(code: np.ndarray, cfg: EncodeCfg, n_bits: int) -> np.ndarray:
    """Per-block bincounts (A, 2^n_bits) in block-scan order; encoder.py:90-94."""
    code = np.asarray(code)
    p, q = code.shape
    starts = block_origins(cfg, p, q)
    if not starts:
        raise OracleShapeError("blocks do not fit the map")
    bins = 1 << n_bits
    out = np.empty((len(starts), bins), dtype=np.int64)
    for k, (i, j) in enumerate(starts):
        cnt = np.bincount(code[i:i + cfg.block_h, j:j + cfg.block_w].ravel(), minlength=bins)
        if cnt.size > bins:
            raise OracleShapeError("code exceeds bit range")
        out[k] = cnt
    return out


def block_iq(code: np.ndarray, cfg: EncodeCfg, n_bits: int) -> np.ndarray:
    """iq_block_features (encoder.py:71-99): -log p per bin, zero-bin policy."""
    cnt = block_counts(code, cfg, n_bits)
    bpc = cfg.block_h * cfg.block_w
    z = 0.0 if cfg.zero_bin_policy == "zero" else float(np.log(2.0 * bpc))
    out = np.full(cnt.shape, z)
    occ = cnt > 0
    out[occ] = -np.log(cnt[occ] / bpc)
    return out.reshape(-1)


def encode_maps(maps: np.ndarray, n_bits: int, cfg: EncodeCfg) -> np.ndarray:
    """encode_view (encoder.py:118-131): groups of n_bits consecutive maps."""
    maps = np.asarray(maps)
    if maps.ndim != 3:
        raise OracleShapeError("need (n_maps, p, q)")
    if maps.shape[0] % n_bits:
        raise OracleShapeError("maps not divisible into groups")
    return np.concatenate([
        block_iq(combine_bits(sign_bits(maps[g * n_bits:(g + 1) * n_bits])), cfg, n_bits)
        for g in range(maps.shape[0] // n_bits)
    ])


def encode_pair(maps1, maps2, n_bits: int, cfg: EncodeCfg) -> tuple[np.ndarray, int]:
    """encode_sample (encoder.py:134-138): view 1 then view 2; returns (values, boundary)."""
    a = encode_maps(maps1, n_bits, cfg)
    b = encode_maps(maps2, n_bits, cfg)
    return np.concatenate([a, b]), a.size


def feature_len(map_shape, maps_per_view: int, n_bits: int, cfg: EncodeCfg) -> int:
    """encoder.py:141-144."""
    return 2 * (maps_per_view // n_bits) * len(block_origins(cfg, *map_shape)) * (1 << n_bits)


def features(view1, view2, layers, cfg: EncodeCfg, batch: int = 128, pool: Pool | None = None) -> np.ndarray:
    """compute_features (pipeline.py:61-86): forward + encode per batch, stacked."""
    pool = pool or Pool()
    v1 = np.asarray(view1, dtype=np.float64)
    v2 = np.asarray(view2, dtype=np.float64)
    n_bits = layers[-1].count

    def run(r: range) -> np.ndarray:
        m1, m2 = forward_maps(v1[r.start:r.stop], v2[r.start:r.stop], layers)
        return np.stack([encode_pair(m1[i], m2[i], n_bits, cfg)[0] for i in range(m1.shape[0])])

    return np.vstack(pool.map(run, batch_ranges(v1.shape[0], batch)))


# ---------------------------------------------------------------------------
# downstream nearest-neighbour classifier (classify.py:109-143)
# ---------------------------------------------------------------------------

def nn_predict(train: np.ndarray, labels: np.ndarray, queries: np.ndarray, metric: str = "euclidean",
               chunk: int = 256) -> np.ndarray:
    """Nearest training row per query; ties -> lowest label (classify.py:136-138).

    euclidean: q2 + t2 - 2 q.t (classify.py:113-115); cosine: 1 - q.t / (|q||t|)
    with similarity 0 where a norm is 0 (classify.py:116-120).
    """
    train = np.asarray(train, dtype=np.float64)
    queries = np.asarray(queries, dtype=np.float64)
    labels = np.asarray(labels, dtype=np.int64)
    out = np.empty(queries.shape[0], dtype=np.int64)
    for s in range(0, queries.shape[0], chunk):
        q = queries[s:s + chunk]
        dot = q @ train.T
        if metric == "euclidean":
            d = np.sum(q * q, axis=1)[:, None] + np.sum(train * train, axis=1)[None, :] - 2.0 * dot
        else:
            den = np.linalg.norm(q, axis=1)[:, None] * np.linalg.norm(train, axis=1)[None, :]
            sim = np.divide(dot, den, out=np.zeros_like(dot), where=den > 0)
            d = 1.0 - sim
        for i, row in enumerate(d):
            out[s + i] = labels[row == row.min()].min()
    return out


def nn_accuracy(pred: np.ndarray, labels: np.ndarray) -> float:
    """evaluate (classify.py:150-176): trace(confusion) / n."""
    return float(np.mean(np.asarray(pred) == np.asarray(labels)))


# ---------------------------------------------------------------------------
# second view (views.py:41-58)
# ---------------------------------------------------------------------------

_LBP_NEIGHBOURS = ((-1, -1), (-1, 0), (-1, 1), (0, 1), (1, 1), (1, 0), (1, -1), (0, -1))


def lbp(img: np.ndarray) -> np.ndarray:
    """8-neighbour LBP / 255: strict neighbour > centre, clockwise from the top-left, zero padding."""
    x = np.asarray(img, dtype=np.float64)
    if x.ndim != 2 or x.shape[0] < 3 or x.shape[1] < 3:
        raise OracleShapeError(f"lbp needs at least a 3x3 image, got {x.shape}")
    p, q = x.shape
    pad = np.zeros((p + 2, q + 2))
    pad[1:-1, 1:-1] = x
    code = np.zeros((p, q))
    for bit, (dy, dx) in enumerate(_LBP_NEIGHBOURS):
        code += float(1 << bit) * (pad[1 + dy:1 + dy + p, 1 + dx:1 + dx + q] > x)
    return code / 255.0
