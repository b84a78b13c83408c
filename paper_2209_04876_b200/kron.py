"""Implicit Kronecker multiplies on the device.

Drop-in for pkg/src/kronsolve/kron.py: the same names and signatures, with every multiply
executed by the CUDA kernels of libkronsolve_b200.so.  The sketched operator is organised
once per sparse diagonal into a (left group, right group) view -- the reference redoes its
np.unique/argsort bookkeeping on every call (kron.py:284-297, :338-346) -- and cached on the
SparseDiagonal object."""

from __future__ import annotations

import ctypes
import functools
import itertools
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _state
from . import _device as D
from . import _lib
from .errors import InvalidInputError
from .tensor import as_matrix

SPARSE_FALLBACK_FRACTION = 0.5
BALANCED_PARTITION_MAX_ORDER = 30


def check_factors(factors: Sequence) -> list[torch.Tensor]:
    """Validated device copies of the factors (kron.py:31-34)."""
    if len(factors) == 0:
        raise InvalidInputError("need at least one factor")
    return [as_matrix(a, f"factor {n}") for n, a in enumerate(factors)]


def kron_operator_shape(factors) -> tuple[int, int]:
    return (math.prod(int(a.shape[0]) for a in factors), math.prod(int(a.shape[1]) for a in factors))


def _kron_apply_dev(facs: list[torch.Tensor], b: torch.Tensor) -> torch.Tensor:
    """(F_0 kron ... kron F_{N-1}) b for a 2-d device b (rows = prod cols)."""
    rows = [int(a.shape[0]) for a in facs]
    cols = [int(a.shape[1]) for a in facs]
    w = int(b.shape[1])
    outt = D.empty(math.prod(rows), w)
    if outt.numel() == 0:
        return outt.zero_()
    if b.numel() == 0:
        return outt.zero_()
    fptr = _lib.ptr_array(ctypes.c_void_p, [a.data_ptr() for a in facs])
    _lib.call("ks_kron_mat_mul", len(facs), fptr, _lib.ptr_array(ctypes.c_int64, rows),
              _lib.ptr_array(ctypes.c_int64, cols), D.p(b), w, D.p(outt), D.stream())
    return outt


def kron_mat_mul(factors: Sequence, b):
    """``(A1 kron ... kron AN) @ b`` without forming the product (kron.py:44-77)."""
    host = not D.on_device(b)
    facs = check_factors(factors)
    bt = D.to_dev(b)
    squeeze = bt.ndim == 1
    if squeeze:
        bt = bt[:, None]
    if bt.ndim != 2:
        raise InvalidInputError("b must be a vector or a matrix")
    _, cols = kron_operator_shape(facs)
    if bt.shape[0] != cols:
        raise InvalidInputError(f"b has {bt.shape[0]} rows but the operator has {cols} columns")
    res = _kron_apply_dev(facs, bt.contiguous())
    return D.out(res[:, 0] if squeeze else res, host)


def kron_vec_square(factors: Sequence, c):
    """Square-factor Kronecker times vector (kron.py:80-100)."""
    host = not D.on_device(c)
    facs = check_factors(factors)
    for n, a in enumerate(facs):
        if a.shape[0] != a.shape[1]:
            raise InvalidInputError(f"factor {n} is {tuple(a.shape)}, expected square")
    ct = D.to_dev(c).reshape(-1)
    size = math.prod(int(a.shape[0]) for a in facs)
    if ct.numel() != size:
        raise InvalidInputError(f"vector length {ct.numel()} != operator size {size}")
    return D.out(_kron_apply_dev(facs, ct[:, None].contiguous())[:, 0], host)


@dataclass(frozen=True)
class FactorPartition:
    """Split of factor positions minimising the larger column product (kron.py:103-114)."""

    left: tuple[int, ...]
    right: tuple[int, ...]
    left_product: int
    right_product: int

    @property
    def objective(self) -> int:
        return max(self.left_product, self.right_product)


def balanced_partition(col_dims: Sequence[int]) -> FactorPartition:
    """Exhaustive min-max split; ties -> smaller left product, then lexicographic left tuple
    (kron.py:117-144).  Host-side integer logic."""
    dims = [int(d) for d in col_dims]
    if not dims:
        raise InvalidInputError("need at least one column dimension")
    if len(dims) > BALANCED_PARTITION_MAX_ORDER:
        raise InvalidInputError(
            f"exhaustive partition search supports at most {BALANCED_PARTITION_MAX_ORDER} "
            f"factors, got {len(dims)}")
    if min(dims) < 1:
        raise InvalidInputError("column dimensions must be positive")
    return _partition_of(tuple(dims))


@functools.lru_cache(maxsize=256)
def _partition_of(dims: tuple) -> FactorPartition:
    total = math.prod(dims)
    key_best, left_best = None, None
    for size in range(len(dims) + 1):
        for subset in itertools.combinations(range(len(dims)), size):
            lp = math.prod(dims[i] for i in subset)
            key = (max(lp, total // lp), lp, subset)
            if key_best is None or key < key_best:
                key_best, left_best = key, subset
    lp = key_best[1]
    right = tuple(i for i in range(len(dims)) if i not in left_best)
    return FactorPartition(left=left_best, right=right, left_product=lp, right_product=total // lp)


@dataclass(frozen=True)
class SparseDiagonal:
    """Sparse diagonal over the Kronecker rows: strictly increasing flat indices + values
    (kron.py:147-170).  ``_views`` caches device groupings per factor list."""

    indices: object
    values: object
    _views: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if isinstance(self.indices, torch.Tensor) or isinstance(self.values, torch.Tensor):
            idx = D.to_dev(self.indices, D.I64).reshape(-1)
            val = D.to_dev(self.values).reshape(-1)
            if idx.numel() != val.numel():
                raise InvalidInputError("indices and values must have equal length")
            if idx.numel():
                bad_order = bool((idx[1:] <= idx[:-1]).any().item()) if idx.numel() > 1 else False
                if bad_order:
                    raise InvalidInputError("indices must be strictly increasing")
                if int(idx[0].item()) < 0:
                    raise InvalidInputError("indices must be nonnegative")
                D.check_flags(D.finite_flags(val), "values")
        else:
            idx = np.asarray(self.indices, dtype=np.int64).reshape(-1)
            val = np.asarray(self.values, dtype=np.float64).reshape(-1)
            if idx.size != val.size:
                raise InvalidInputError("indices and values must have equal length")
            if idx.size and np.any(np.diff(idx) <= 0):
                raise InvalidInputError("indices must be strictly increasing")
            if idx.size and idx[0] < 0:
                raise InvalidInputError("indices must be nonnegative")
            if not np.all(np.isfinite(val)):
                raise InvalidInputError("values must be finite")
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "values", val)

    @classmethod
    def _trusted(cls, indices, values) -> "SparseDiagonal":
        """Construct without the validation passes (device syncs) for diagonals built by
        sparse_diagonal_from_sketch, which are sorted, unique and finite by construction."""
        obj = object.__new__(cls)
        object.__setattr__(obj, "indices", indices)
        object.__setattr__(obj, "values", values)
        object.__setattr__(obj, "_views", {})
        return obj

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])

    def last_index(self) -> int:
        return int(self.indices[-1].item() if isinstance(self.indices, torch.Tensor) else self.indices[-1])


def sparse_diagonal_from_sketch(sketch, row_shape: Sequence[int]) -> SparseDiagonal:
    """sqrt(S^T S) on the sampled rows (kron.py:173-190), sorted/deduplicated on the device
    with NumPy's exact reduceat summation order."""
    host = not D.on_device(sketch.indices)
    idx = D.to_dev(sketch.indices, D.I64)
    w = D.to_dev(sketch.weights).reshape(-1)
    if idx.ndim == 2:
        nf = int(idx.shape[1])
        shape = [int(r) for r in row_shape]
    else:
        nf = 1
        shape = [math.prod(int(r) for r in row_shape)]
        idx = idx.reshape(-1, 1)
    s = int(idx.shape[0])
    sd_idx = D.empty(max(s, 1), dtype=D.I64)
    sd_val = D.empty(max(s, 1))
    nnz = ctypes.c_int64(0)
    _lib.call("ks_sketch_diag", nf, D.p(idx.contiguous()), _lib.ptr_array(ctypes.c_int64, shape), D.p(w), s,
              D.p(sd_idx), D.p(sd_val), ctypes.byref(nnz), D.stream())
    k = nnz.value
    if host:
        return SparseDiagonal(indices=D.out(sd_idx[:k], host), values=D.out(sd_val[:k], host))
    return SparseDiagonal._trusted(sd_idx[:k], sd_val[:k])


def kron_rows(factors: Sequence, multi_indices) -> torch.Tensor:
    """Rows of the Kronecker product at the given multi-indices (kron.py:193-205)."""
    host = not D.on_device(multi_indices)
    mi = D.to_dev(multi_indices, D.I64)
    if mi.ndim == 1:
        mi = mi[None, :]
    if factors and mi.numel():
        # NumPy fancy-indexing rules (negative indices wrap, anything else out of range raises
        # IndexError) checked before the gather, so a bad index never becomes a device fault.
        rows = torch.tensor([int(a.shape[0]) for a in factors], dtype=D.I64, device=mi.device)
        cols = mi[:, :len(factors)]
        if mi.shape[1] < len(factors) or bool(((cols < -rows) | (cols >= rows)).any()):
            raise IndexError("multi-index out of range for the Kronecker factors")
    acc = D.zeros(mi.shape[0], 1) + 1.0
    for n, a in enumerate(factors):
        at = D.to_dev(a)
        part = at[mi[:, n], :]
        acc = (acc[:, :, None] * part[:, None, :]).reshape(mi.shape[0], -1)
    return D.out(acc, host)


class _View:
    """Device grouping of a sparse diagonal for one factor list (kept alive with its buffers)."""

    def __init__(self, facs, sd: SparseDiagonal):
        self.facs = facs
        rows = [int(a.shape[0]) for a in facs]
        cols = [int(a.shape[1]) for a in facs]
        self.part = balanced_partition(cols)
        left, right = self.part.left, self.part.right
        self.dL = math.prod(cols[i] for i in left)
        self.dR = math.prod(cols[i] for i in right)
        nnz = sd.nnz
        self.nnz = nnz
        self.sd_idx = D.to_dev(sd.indices, D.I64)
        self.sd_val = D.to_dev(sd.values)
        self.seg = D.empty(nnz + 1, dtype=D.I64)
        self.lrow = D.empty(nnz, dtype=D.I64)
        self.rrow = D.empty(nnz, dtype=D.I64)
        self.v = D.empty(nnz)
        self.perm = D.empty(nnz, dtype=D.I64)
        self.Lbuf = D.empty(nnz, self.dL) if len(left) != 1 else None
        self.Rbuf = D.empty(nnz, self.dR) if len(right) != 1 else None
        u_left = ctypes.c_int64(0)
        fptr = _lib.ptr_array(ctypes.c_void_p, [a.data_ptr() for a in facs])
        _lib.call("ks_sketch_group", len(facs), fptr, _lib.ptr_array(ctypes.c_int64, rows),
                  _lib.ptr_array(ctypes.c_int64, cols), len(left),
                  _lib.ptr_array(ctypes.c_int32, list(left) or [0]), len(right),
                  _lib.ptr_array(ctypes.c_int32, list(right) or [0]), D.p(self.sd_idx),
                  D.p(self.sd_val), nnz, D.p(self.seg), D.p(self.lrow), D.p(self.rrow), D.p(self.v),
                  D.p(self.perm), D.p(self.Lbuf), D.p(self.Rbuf), ctypes.byref(u_left), D.stream())
        self.u_left = u_left.value
        self.prefix = tuple(left) == tuple(range(len(left)))
        Lmat = self.Lbuf if self.Lbuf is not None else facs[left[0]]
        Rmat = self.Rbuf if self.Rbuf is not None else facs[right[0]]
        self.Lmat, self.Rmat = Lmat, Rmat
        self.struct = _lib.SketchView(
            Lmat.data_ptr(), int(Lmat.shape[1]), self.dL, Rmat.data_ptr(), int(Rmat.shape[1]), self.dR,
            self.u_left, nnz, self.seg.data_ptr(), self.lrow.data_ptr(), self.rrow.data_ptr(),
            self.v.data_ptr())
        self.col_shape = tuple(cols)
        self.order = tuple(left) + tuple(right)

    @classmethod
    def from_parts(cls, facs, sd: SparseDiagonal, seg, lrow, rrow, u_left: int):
        """Two-factor view already built by ks_sketch_diag_grouped2 (left {0}, right {1}; grouped
        order == sparse-diagonal order)."""
        v = object.__new__(cls)
        v.facs = facs
        rows = [int(a.shape[0]) for a in facs]
        cols = [int(a.shape[1]) for a in facs]
        v.part = balanced_partition(cols)
        v.dL, v.dR = cols[0], cols[1]
        v.nnz = sd.nnz
        v.sd_idx, v.sd_val = sd.indices, sd.values
        v.seg, v.lrow, v.rrow = seg, lrow, rrow
        v.v = sd.values
        v.perm = None
        v.Lbuf = v.Rbuf = None
        v.u_left = int(u_left)
        v.prefix = True
        v.Lmat, v.Rmat = facs[0], facs[1]
        v.struct = _lib.SketchView(facs[0].data_ptr(), cols[0], v.dL, facs[1].data_ptr(), cols[1], v.dR, v.u_left,
                                   v.nnz, seg.data_ptr(), lrow.data_ptr(), rrow.data_ptr(), sd.values.data_ptr())
        v.col_shape = tuple(cols)
        v.order = (0, 1)
        del rows
        return v

    def perm_arg(self):
        # grouped order == sparse-diagonal order when the left group is a prefix
        return None if self.prefix else self.perm

    def to_groups(self, c: torch.Tensor) -> torch.Tensor:
        """kron.py:252-255: natural flat order -> (left, right) grouped (dL x dR)."""
        if self.order == tuple(range(len(self.order))):
            return c.reshape(self.dL, self.dR)
        return c.reshape(self.col_shape).permute(self.order).reshape(self.dL, self.dR).contiguous()

    def from_groups(self, g: torch.Tensor) -> torch.Tensor:
        """kron.py:243-249: grouped -> natural flat order."""
        if self.order == tuple(range(len(self.order))):
            return g.reshape(-1)
        inv = tuple(int(i) for i in np.argsort(np.asarray(self.order)))
        shape = tuple(self.col_shape[i] for i in self.order)
        return g.reshape(shape).permute(inv).reshape(-1).contiguous()


def grouped2_eligible(facs) -> bool:
    """Two factors whose balanced partition is (left {0}, right {1})."""
    if len(facs) != 2:
        return False
    part = balanced_partition([int(a.shape[1]) for a in facs])
    return part.left == (0,) and part.right == (1,)


def sketch_diag_grouped2_launch(facs, sketch_indices: torch.Tensor, sketch_weights: torch.Tensor,
                                first_raw: torch.Tensor | None = None):
    """Launch-only half of sketch_diag_and_view2 (graph-capturable): returns the device buffers
    (sd_idx, sd_val, seg, lrow, rrow, counts_dev); ``first_raw`` (optional, s int64) receives each
    entry's first draw index."""
    rows = [int(a.shape[0]) for a in facs]
    s = int(sketch_indices.shape[0])
    bufs = (D.empty(max(s, 1), dtype=D.I64), D.empty(max(s, 1)), D.empty(s + 1, dtype=D.I64),
            D.empty(max(s, 1), dtype=D.I64), D.empty(max(s, 1), dtype=D.I64), D.empty(2, dtype=D.I64))
    sd_idx, sd_val, seg, lrow, rrow, cdev = bufs
    _lib.call("ks_sketch_diag_grouped2_ex", D.p(sketch_indices.contiguous()), _lib.ptr_array(ctypes.c_int64, rows),
              D.p(sketch_weights.contiguous()), s, D.p(sd_idx), D.p(sd_val), D.p(seg), D.p(lrow), D.p(rrow), None,
              D.p(cdev), D.p(first_raw), D.stream())
    return bufs


def sketch_diag_grouped2_finish(facs, bufs):
    """Read (nnz, u_left) and wrap the buffers as a SparseDiagonal and its cached view."""
    sd_idx, sd_val, seg, lrow, rrow, cdev = bufs
    nnz, ul = (int(v) for v in cdev.cpu().tolist())
    sd = SparseDiagonal._trusted(sd_idx[:nnz], sd_val[:nnz])
    view = _View.from_parts(facs, sd, seg, lrow, rrow, ul)
    sd._views[tuple((a.data_ptr(), tuple(a.shape)) for a in facs)] = view
    return sd, view


def sketch_diag_and_view2(facs, sketch_indices: torch.Tensor, sketch_weights: torch.Tensor):
    """Sparse diagonal of a two-factor row sketch together with its grouped view (one fused
    device pass, one host round trip); None when the factors' balanced partition is not
    (left {0}, right {1})."""
    if not grouped2_eligible(facs):
        return None
    return sketch_diag_grouped2_finish(facs, sketch_diag_grouped2_launch(facs, sketch_indices, sketch_weights))


def _view_for(facs, sd: SparseDiagonal) -> _View:
    key = tuple((a.data_ptr(), tuple(a.shape)) for a in facs)
    v = sd._views.get(key)
    if v is None:
        v = _View(facs, sd)
        sd._views.clear()
        sd._views[key] = v
    return v


def _check_sd(sd: SparseDiagonal, rows: int):
    if sd.nnz and sd.last_index() >= rows:
        raise InvalidInputError("sparse diagonal index out of range")


def sketched_kron_apply(factors: Sequence, s_diag: SparseDiagonal, c):
    """Entries of ``S K c`` at the nonzero rows of ``S`` (kron.py:258-300)."""
    host = not D.on_device(c)
    facs = check_factors(factors)
    rows, cols = kron_operator_shape(facs)
    ct = D.to_dev(c).reshape(-1)
    if ct.numel() != cols:
        raise InvalidInputError(f"vector length {ct.numel()} != operator columns {cols}")
    if s_diag.nnz == 0:
        return D.out(D.empty(0), host)
    _check_sd(s_diag, rows)
    if s_diag.nnz > rows * SPARSE_FALLBACK_FRACTION:
        full = _kron_apply_dev(facs, ct[:, None].contiguous())[:, 0]
        idx = D.to_dev(s_diag.indices, D.I64)
        return D.out(D.to_dev(s_diag.values) * full[idx], host)
    view = _view_for(facs, s_diag)
    X = view.to_groups(ct).contiguous()
    vals = D.empty(view.nnz)
    _lib.call("ks_sketched_apply", ctypes.byref(view.struct), D.p(X), D.p(view.perm_arg()), D.p(vals),
              D.stream())
    return D.out(vals, host)


def sketched_kron_transpose_apply(factors: Sequence, s_diag: SparseDiagonal, b_values):
    """``K^T S b`` from the entries of b on the sketched rows (kron.py:312-354)."""
    host = not D.on_device(b_values)
    facs = check_factors(factors)
    rows, cols = kron_operator_shape(facs)
    bv = D.to_dev(b_values).reshape(-1)
    if bv.numel() != s_diag.nnz:
        raise InvalidInputError("b_values must align with the sparse diagonal")
    if s_diag.nnz == 0:
        return D.out(D.zeros(cols), host)
    _check_sd(s_diag, rows)
    if s_diag.nnz > rows * SPARSE_FALLBACK_FRACTION:
        full = D.zeros(rows)
        idx = D.to_dev(s_diag.indices, D.I64)
        full[idx] = D.to_dev(s_diag.values) * bv
        return D.out(_kron_apply_dev([a.T.contiguous() for a in facs], full[:, None])[:, 0], host)
    view = _view_for(facs, s_diag)
    G = D.empty(view.dL, view.dR)
    _lib.call("ks_sketched_transpose_apply", ctypes.byref(view.struct), D.p(bv.contiguous()),
              D.p(view.perm_arg()), D.p(G), D.stream())
    return D.out(view.from_groups(G), host)


def sketch_rows_of_kron(factors: Sequence, sketch):
    """Materialise the sketched matrix ``S K``: one rescaled row per draw (kron.py:208-222)."""
    host = not D.on_device(sketch.weights)
    facs = check_factors(factors)
    rows, _ = kron_operator_shape(facs)
    idx = D.to_dev(sketch.indices, D.I64).contiguous()
    w = D.to_dev(sketch.weights).reshape(-1).contiguous()
    flat = idx.ndim == 1
    if idx.numel():
        if flat:
            lo, hi = int(idx.min()), int(idx.max())
            if lo < 0 or hi >= rows:
                raise InvalidInputError("sketch index out of range")
        else:
            mn, mx = idx.min(dim=0).values.tolist(), idx.max(dim=0).values.tolist()
            for n, a in enumerate(facs):
                if mn[n] < 0 or mx[n] >= int(a.shape[0]):
                    raise InvalidInputError(f"sketch index out of range in mode {n}")
    s = int(w.numel())
    ncols = math.prod(int(a.shape[1]) for a in facs)
    out = D.empty(s, ncols)
    _lib.call("ks_sketch_rows", len(facs), _lib.ptr_array(ctypes.c_void_p, [a.data_ptr() for a in facs]),
              _lib.ptr_array(ctypes.c_int64, [int(a.shape[0]) for a in facs]),
              _lib.ptr_array(ctypes.c_int32, [int(a.shape[1]) for a in facs]), D.p(idx), int(flat), D.p(w), s,
              D.p(out), D.stream())
    return D.out(out, host)


# Public entry points are gated (capture vs. concurrent solves, see _state.py).
_state.gate_names(globals(), [
    "balanced_partition",
    "check_factors",
    "kron_mat_mul",
    "kron_operator_shape",
    "kron_rows",
    "kron_vec_square",
    "sketch_rows_of_kron",
    "sketched_kron_apply",
    "sketched_kron_transpose_apply",
    "sparse_diagonal_from_sketch",
])
