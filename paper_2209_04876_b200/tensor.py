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
    n, d = t.shape
    k = min(n, d)
    if k == 0:
        return t.new_zeros((n, 0)), t.new_zeros((0,)), t.new_zeros((d, 0))
    if k > 128:
        from .errors import SizeGuardError
        raise SizeGuardError(f"compact_svd on the device supports min(n, d) <= 128, got {k}")
    u = D.empty(n, k)
    s = D.empty(k)
    v = D.empty(d, k)
    rank = ctypes.c_int32(0)
    _lib.call("ks_compact_svd", D.p(t), n, d, float(rank_tol), D.p(u), D.p(s), D.p(v),
              ctypes.byref(rank), D.stream())
    r = rank.value
    return u[:, :r].contiguous(), s[:r].contiguous(), v[:, :r].contiguous()


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
