"""Filter solve: canonical pairs, filter layers/banks, device eigensolver.

API mirror of solver.py:90-272 of the reference. ``sym_eig``, ``inv_sqrt``
and ``solve_dcca`` run the single-CTA float64 Jacobi kernel
(csrc/solve.cu), which restates the reference's rotation schedule, stopping
rule, sign rule and degenerate-run ordering. ``reshape_filters`` is a pure
row-major relayout.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigError, ShapeError
from .moments import DiscriminantMoments
from .patches import PatchGeometry


@dataclass(frozen=True)
class CanonicalPairs:
    """Projection pairs: columns of w1 / w2 and their correlations (solver.py:173-183)."""

    w1: np.ndarray
    w2: np.ndarray
    rho: np.ndarray

    @property
    def count(self) -> int:
        return self.w1.shape[1]


@dataclass(frozen=True)
class FilterLayer:
    """One layer's (L, l1, l2) kernels for view 1 and view 2 (solver.py:186-197)."""

    filters1: np.ndarray
    filters2: np.ndarray
    geom: PatchGeometry
    center: bool

    @property
    def count(self) -> int:
        return self.filters1.shape[0]


@dataclass(frozen=True)
class FilterBank:
    """The trained cascade (solver.py:200-213)."""

    layers: tuple

    @property
    def depth(self) -> int:
        return len(self.layers)

    @property
    def maps_per_view(self) -> int:
        n = 1
        for layer in self.layers:
            n *= layer.count
        return n


def _ex(executor):
    from .execution import Executor

    return executor or Executor()


def _eig_call(s: np.ndarray, mode: int, executor=None):
    import torch

    s = np.asarray(s, dtype=np.float64)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise ShapeError(f"expected a square matrix, got shape {s.shape}")
    n = s.shape[0]
    ex = _ex(executor)
    lib = _native.load()
    with torch.cuda.stream(ex.stream):
        sd = torch.from_numpy(np.ascontiguousarray(s)).to(ex.device)
        w = torch.empty(n, dtype=torch.float64, device=ex.device)
        v = torch.empty((n, n), dtype=torch.float64, device=ex.device)
        st = torch.zeros(1, dtype=torch.int32, device=ex.device)
        nb = int(lib.ddcca_solve_workspace(n))
        ws = torch.empty(nb, dtype=torch.uint8, device=ex.device)
        _native.check(lib.ddcca_sym_eig(_native.ptr(sd), n, mode, _native.ptr(w), _native.ptr(v), _native.ptr(st),
                                        _native.ptr(ws), nb, _native.stream_ptr(ex.stream)), "sym_eig")
        code = int(st.item())
        if code == _native.ESHAPE:
            raise ShapeError("matrix is not symmetric")
        if code == _native.ENUMERICAL and mode == 1:
            from .errors import NumericalError

            raise NumericalError("matrix is not positive definite; is the ridge term missing?")
        _native.status_error(code, "sym_eig")
        return w.cpu().numpy(), v.cpu().numpy()


def sym_eig(s: np.ndarray, executor=None):
    """Eigenvalues (descending) and sign-normalized eigenvectors (solver.py:90-158)."""
    return _eig_call(s, 0, executor)


def inv_sqrt(c: np.ndarray, executor=None) -> np.ndarray:
    """Symmetrized V diag(w^-1/2) V^T of an SPD matrix (solver.py:161-170)."""
    return _eig_call(c, 1, executor)[1]


def solve_dcca(m: DiscriminantMoments, count: int, executor=None) -> CanonicalPairs:
    """Leading canonical pairs of the discriminant problem (solver.py:216-257), on the device."""
    import torch

    dim = m.dim
    if not 1 <= count <= dim:
        raise ConfigError(f"filter count {count} outside [1, {dim}]")
    ex = _ex(executor)
    lib = _native.load()
    with torch.cuda.stream(ex.stream):
        fin = torch.from_numpy(np.stack([m.c11, m.c22, m.cw, m.cb, m.ctilde]).astype(np.float64)).to(ex.device)
        w1 = torch.empty((dim, count), dtype=torch.float64, device=ex.device)
        w2 = torch.empty((dim, count), dtype=torch.float64, device=ex.device)
        rho = torch.empty(count, dtype=torch.float64, device=ex.device)
        st = torch.zeros(1, dtype=torch.int32, device=ex.device)
        nb = int(lib.ddcca_solve_workspace(dim))
        ws = torch.empty(nb, dtype=torch.uint8, device=ex.device)
        _native.check(lib.ddcca_solve(None, dim, 1, 0.0, count, _native.ptr(fin), _native.ptr(w1), _native.ptr(w2),
                                      _native.ptr(rho), None, None, _native.ptr(st), _native.ptr(ws), nb,
                                      _native.stream_ptr(ex.stream)), "solve_dcca")
        _native.status_error(int(st.item()), "solve_dcca")
        return CanonicalPairs(w1=w1.cpu().numpy(), w2=w2.cpu().numpy(), rho=rho.cpu().numpy())


def reshape_filters(pairs: CanonicalPairs, geom: PatchGeometry, center: bool = True) -> FilterLayer:
    """Column g -> row-major l1 x l2 kernel g (solver.py:260-272)."""
    if pairs.w1.shape[0] != geom.dim:
        raise ShapeError(f"vector length {pairs.w1.shape[0]} does not match {geom.l1}x{geom.l2} kernels")
    L = pairs.count
    return FilterLayer(filters1=np.ascontiguousarray(pairs.w1.T).reshape(L, geom.l1, geom.l2).copy(),
                       filters2=np.ascontiguousarray(pairs.w2.T).reshape(L, geom.l1, geom.l2).copy(),
                       geom=geom, center=center)
