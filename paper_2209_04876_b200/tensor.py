"""Dense primitives on the device: validation and the thin SVD.

Mirrors pkg/src/kronsolve/tensor.py for the functions on the FastKroneckerRegression path:
``as_matrix`` / ``as_tensor`` (tensor.py:35-52), ``CompactSvd`` / ``compact_svd``
(tensor.py:55-107), ``vectorize`` / ``devectorize`` (tensor.py:118-130).  The SVD runs on the
GPU (Householder TSQR + one-sided Jacobi, csrc/ks_small.cu); LAPACK is not used."""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _state
from . import _device as D
from . import _lib
from .errors import InvalidInputError

DEFAULT_RANK_TOL = 1e-10


def as_matrix(a, name: str = "matrix") -> torch.Tensor:
    """Validated 2-d float64 CUDA tensor (InvalidInputError on ndim != 2 or non-finite)."""
    t = D.to_dev(a)
    if t.ndim != 2:
        raise InvalidInputError(f"{name} must be 2-dimensional, got ndim={t.ndim}")
    if t.numel():
        D.check_flags(D.finite_flags(t), name)
    return t


def as_tensor(x, name: str = "tensor") -> torch.Tensor:
    t = D.to_dev(x)
    if t.ndim < 1:
        t = t.reshape(1)
    if t.numel():
        D.check_flags(D.finite_flags(t), name)
    return t


@dataclass(frozen=True)
class CompactSvd:
    """``a = u @ diag(sigma) @ v.T`` with positive, non-increasing singular values."""

    u: object
    sigma: object
    v: object
    rank_tol: float = DEFAULT_RANK_TOL

    @property
    def rank(self) -> int:
        return int(self.sigma.shape[0])

    def reconstruct(self):
        if isinstance(self.u, torch.Tensor):
            return (self.u * self.sigma) @ self.v.T
        return (self.u * self.sigma) @ self.v.T


def _compact_svd_dev(t: torch.Tensor, rank_tol: float):
    return _compact_svds_dev([t], rank_tol)[0]


def _compact_svds_dev(ts, rank_tol: float):
    """Thin SVDs of several matrices with ONE synchronisation: every ks_compact_svd runs without
    its own rank read-back, then all singular values come back in one copy and the ranks
    (sigma_j > rank_tol * sigma_0, tensor.py:76-107) are counted here."""
    outs, sig = [], []
    for t in ts:
        n, d = t.shape
        k = min(n, d)
        if k == 0:
            outs.append((t.new_zeros((n, 0)), t.new_zeros((0,)), t.new_zeros((d, 0))))
            continue
        if k > 128:
            from .errors import SizeGuardError
            raise SizeGuardError(f"compact_svd on the device supports min(n, d) <= 128, got {k}")
        u, s, v = D.empty(n, k), D.empty(k), D.empty(d, k)
        _lib.call("ks_compact_svd", D.p(t), n, d, float(rank_tol), D.p(u), D.p(s), D.p(v), None, D.stream())
        outs.append((u, s, v))
        sig.append(s)
    hs = torch.cat(sig).cpu().tolist() if sig else []
    res, off = [], 0
    for u, s, v in outs:
        k = int(s.numel())
        if k == 0:
            res.append((u, s, v))
            continue
        h = hs[off:off + k]
        off += k
        r = sum(1 for x in h if x > rank_tol * h[0]) if h[0] > 0.0 else 0
        res.append((u[:, :r].contiguous(), s[:r].contiguous(), v[:, :r].contiguous()))
    return res


def compact_svd(a, rank_tol: float = DEFAULT_RANK_TOL) -> CompactSvd:
    """Thin SVD with singular values <= rank_tol * sigma_max dropped (tensor.py:76-107)."""
    host = not D.on_device(a)
    t = as_matrix(a)
    if not 0.0 <= rank_tol < 1.0:
        raise InvalidInputError(f"rank_tol must be in [0, 1), got {rank_tol}")
    u, s, v = _compact_svd_dev(t, rank_tol)
    return CompactSvd(u=D.out(u, host), sigma=D.out(s, host), v=D.out(v, host), rank_tol=rank_tol)


def vectorize(x):
    """Row-major flatten (tensor.py:118-120)."""
    host = not D.on_device(x)
    return D.out(as_tensor(x).reshape(-1), host)


def devectorize(v, shape: Sequence[int]):
    """Inverse of vectorize (tensor.py:123-130)."""
    size = math.prod(shape)
    if isinstance(v, torch.Tensor):
        t = v.reshape(-1)
        if t.numel() != size:
            raise InvalidInputError(f"vector of length {t.numel()} cannot fill shape {tuple(shape)}")
        return t.reshape(tuple(shape))
    a = np.asarray(v, dtype=np.float64).reshape(-1)
    if a.size != size:
        raise InvalidInputError(f"vector of length {a.size} cannot fill shape {tuple(shape)}")
    return a.reshape(tuple(shape))


# ---------------------------------------------------------------------------
# Unfoldings and mode products (tensor.py:110-183) -- used by the Tucker factor updates
# ---------------------------------------------------------------------------

def unfold(x, mode: int):
    """Mode-``mode`` unfolding: (I_mode, prod of the other dims), other indices lexicographic
    (tensor.py:133-143).  A layout copy on the device."""
    host = not D.on_device(x)
    t = as_tensor(x)
    if not 0 <= mode < t.ndim:
        raise InvalidInputError(f"mode {mode} out of range for order-{t.ndim} tensor")
    return D.out(t.movedim(mode, 0).reshape(int(t.shape[mode]), -1).contiguous(), host)


def fold(m, shape: Sequence[int], mode: int):
    """Inverse of :func:`unfold` (tensor.py:146-156)."""
    host = not D.on_device(m)
    t = D.to_dev(m)
    shape = tuple(int(s) for s in shape)
    if not 0 <= mode < len(shape):
        raise InvalidInputError(f"mode {mode} out of range for shape {shape}")
    rest = shape[:mode] + shape[mode + 1:]
    if tuple(t.shape) != (shape[mode], math.prod(rest)):
        raise InvalidInputError(f"matrix of shape {tuple(t.shape)} does not unfold to {shape} at mode {mode}")
    return D.out(t.reshape((shape[mode],) + rest).movedim(0, mode).contiguous(), host)


def _mode_mul_dev(x: torch.Tensor, a: torch.Tensor, mode: int, transpose: bool = False) -> torch.Tensor:
    """x x_mode A (A: J x I_mode) or, with ``transpose``, x x_mode A^T (A: I_mode x J), as one
    batched strided ks_gemm over the fibres of ``mode``."""
    shape = tuple(int(s) for s in x.shape)
    k = shape[mode]
    j = int(a.shape[1] if transpose else a.shape[0])
    p = math.prod(shape[:mode])
    q = math.prod(shape[mode + 1:])
    out = D.empty(*(shape[:mode] + (j,) + shape[mode + 1:]))
    if out.numel() == 0:
        return out.zero_()
    a_rs, a_cs = (1, j) if transpose else (k, 1)  # element (row i of the output fibre, k)
    if q == 1:
        # last mode: out (p x j) = x (p x k) . op(A)^T in one GEMM
        _lib.call("ks_gemm", p, j, k, 1.0, D.p(x), k, 1, 0, D.p(a), a_cs, a_rs, 0, 0.0, D.p(out), j, 1, 0, 1,
                  D.stream())
    else:
        _lib.call("ks_gemm", j, q, k, 1.0, D.p(a), a_rs, a_cs, 0, D.p(x), q, 1, k * q, 0.0, D.p(out), q, 1, j * q,
                  p, D.stream())
    return out


def n_mode_product(x, a, mode: int):
    """Multiply every mode-``mode`` fibre of ``x`` by ``a`` (tensor.py:159-172)."""
    host = not D.on_device(x)
    t = as_tensor(x)
    m = as_matrix(a)
    if not 0 <= mode < t.ndim:
        raise InvalidInputError(f"mode {mode} out of range for order-{t.ndim} tensor")
    if int(m.shape[1]) != int(t.shape[mode]):
        raise InvalidInputError(f"matrix with {int(m.shape[1])} columns cannot multiply mode {mode} of size "
                                f"{int(t.shape[mode])}")
    return D.out(_mode_mul_dev(t.contiguous(), m, mode), host)


def multi_mode_product(x, factors: Sequence):
    """``x x_1 A1 x_2 ... x_N AN`` (tensor.py:175-183)."""
    host = not D.on_device(x)
    t = as_tensor(x)
    if len(factors) != t.ndim:
        raise InvalidInputError(f"need {t.ndim} factors for an order-{t.ndim} tensor, got {len(factors)}")
    for mode, a in enumerate(factors):
        m = as_matrix(a)
        if int(m.shape[1]) != int(t.shape[mode]):
            raise InvalidInputError(f"factor {mode} does not match mode size {int(t.shape[mode])}")
        t = _mode_mul_dev(t, m, mode)
    return D.out(t, host)


def _pinv_dev(t: torch.Tensor, rank_tol: float) -> torch.Tensor:
    """(V / sigma) U^T from the compact SVD, zero matrix at rank 0 (tensor.py:110-115)."""
    n, d = int(t.shape[0]), int(t.shape[1])
    u, s, v = _compact_svd_dev(t, rank_tol)
    k = int(s.numel())
    out = D.zeros(d, n)
    if k:
        _lib.call("ks_pinv_compose", D.p(u.contiguous()), n, D.p(s), D.p(v.contiguous()), d, k, D.p(out),
                  D.stream())
    return out


def pseudo_inverse(a, rank_tol: float = DEFAULT_RANK_TOL):
    """Moore-Penrose inverse via the compact SVD (tensor.py:110-115)."""
    host = not D.on_device(a)
    return D.out(_pinv_dev(as_matrix(a), rank_tol), host)


EXPLICIT_KRON_MAX_ENTRIES = 10 ** 7


def explicit_kron(factors: Sequence, max_entries: int = EXPLICIT_KRON_MAX_ENTRIES):
    """Dense ``A1 kron ... kron AN`` (tensor.py:186-198): the reference's test-oracle path, kept
    size-guarded; built on the device by successive outer products."""
    if len(factors) == 0:
        raise InvalidInputError("need at least one factor")
    from .errors import SizeGuardError
    host = not any(D.on_device(a) for a in factors)
    mats = [as_matrix(a, f"factor {n}") for n, a in enumerate(factors)]
    rows = math.prod(int(a.shape[0]) for a in mats)
    cols = math.prod(int(a.shape[1]) for a in mats)
    if rows * cols > max_entries:
        raise SizeGuardError(f"explicit Kronecker product would hold {rows}x{cols} entries "
                             f"(guard: {max_entries})")
    from .solvers import _kron_dev
    return D.out(_kron_dev([D.to_dev(a) for a in mats]), host)


def stack_columns(m):
    """Column-major flatten for the vec-trick identities (tensor.py:201-203)."""
    if isinstance(m, torch.Tensor):
        return m.to(torch.float64).T.reshape(-1)
    return np.asarray(m, dtype=np.float64).reshape(-1, order="F")


def unstack_columns(v, shape):
    """Inverse of :func:`stack_columns` for a (rows, cols) shape (tensor.py:206-213)."""
    rows, cols = shape
    if isinstance(v, torch.Tensor):
        t = v.to(torch.float64).reshape(-1)
        if t.numel() != rows * cols:
            raise InvalidInputError(f"vector of length {t.numel()} cannot fill a {rows}x{cols} matrix")
        return t.reshape(cols, rows).T
    a = np.asarray(v, dtype=np.float64).reshape(-1)
    if a.size != rows * cols:
        raise InvalidInputError(f"vector of length {a.size} cannot fill a {rows}x{cols} matrix")
    return a.reshape((rows, cols), order="F")


# Public entry points are gated (capture vs. concurrent solves, see _state.py).
_state.gate_names(globals(), [
    "as_matrix",
    "as_tensor",
    "compact_svd",
    "devectorize",
    "explicit_kron",
    "fold",
    "multi_mode_product",
    "n_mode_product",
    "pseudo_inverse",
    "stack_columns",
    "unfold",
    "unstack_columns",
    "vectorize",
])
