"""Kronecker ridge regression solvers on the device.

Drop-in for the north-star functions of pkg/src/kronsolve/solvers.py:
``RegressionConfig`` (:61-112), ``SolveReport`` (:115-123), ``factor_gram`` / ``FactorGram``
(:126-150), ``FactorCache`` / ``build_factor_cache`` (:153-163), ``KronPreconditioner`` /
``pseudo_reciprocal`` / ``build_kron_preconditioner`` (:166-198), ``richardson_solve``
(:201-248), ``ridge_loss`` (:251-262), ``kronmatmul_svd_solve`` (:302-320),
``exact_factor_scores`` (:323-331) and ``fast_kronecker_regression`` (:372-462).

Inside ``fast_kronecker_regression`` every step -- Gaussian/uniform streams, Gram and JL
products, sampler tables, inverse-CDF draws, sketch deduplication, the sketched operator and
all Richardson iterations -- runs on the GPU; the host only spawns seeds, evaluates the
sample-count formulas and reads back the iteration count and residual history once."""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, replace
from functools import reduce
from typing import Callable, Sequence

import numpy as np
import torch

from . import _device as D
from . import _lib
from . import _state
from ._state import CACHE_LOCK, CAPTURE_MODE, GATE, TLSlot
from .errors import InvalidInputError, NumericalFailureError, SizeGuardError
from .kron import (SparseDiagonal, _kron_apply_dev, _view_for, check_factors, grouped2_eligible,
                   kron_operator_shape, sketch_diag_grouped2_finish, sketch_diag_grouped2_launch,
                   kron_vec_square, sparse_diagonal_from_sketch)
from .leverage import (JL_LOG_FACTOR, REGRESSION_SAMPLE_CONSTANT, LeverageScores, ProductSampler,
                       RowSketch, _inverse_small, _jl_scores_dev, _spectral_rows_dev,
                       ridge_leverage_scores, spectral_sample_count)
from ._numpy_rng import pcg64_state
from .tensor import CompactSvd, _compact_svd_dev, _compact_svds_dev, as_matrix, compact_svd

DEFAULT_DENSE_GUARD = 10 ** 8
_DIVERGENCE_WINDOW = 5
_DIVERGENCE_GROWTH = 10.0


@dataclass(frozen=True)
class RegressionConfig:
    """Solver knobs (solvers.py:61-112): same fields, defaults and validation."""

    eps: float = 0.25
    delta: float = 0.05
    lam: float = 0.0
    alpha: float = 1.0
    mode: str = "practical"
    max_richardson_iters: int | None = None
    residual_tol: float = 1e-9
    seed: int = 0
    damping: float | None = None
    jl_log_factor: float = JL_LOG_FACTOR
    share_row_sketch: bool = False

    def __post_init__(self):
        if not 0.0 < self.eps < 1.0:
            raise InvalidInputError(f"eps must be in (0, 1), got {self.eps}")
        if not 0.0 < self.delta < 1.0:
            raise InvalidInputError(f"delta must be in (0, 1), got {self.delta}")
        if self.lam < 0.0:
            raise InvalidInputError(f"lambda must be >= 0, got {self.lam}")
        if not 0.0 < self.alpha <= 1.0:
            raise InvalidInputError(f"alpha must be in (0, 1], got {self.alpha}")
        if self.mode not in ("theoretical", "practical"):
            raise InvalidInputError(f"unknown mode {self.mode!r}")
        if self.residual_tol <= 0.0:
            raise InvalidInputError("residual_tol must be positive")

    @property
    def effective_alpha(self) -> float:
        return 1.0 if self.mode == "theoretical" else self.alpha

    @property
    def effective_damping(self) -> float:
        return (1.0 - math.sqrt(self.eps)) if self.damping is None else self.damping

    @property
    def effective_max_iters(self) -> int:
        if self.max_richardson_iters is not None:
            return self.max_richardson_iters
        return 8 * max(1, math.ceil(math.log(1.0 / self.eps)))

    def with_lam(self, lam: float) -> "RegressionConfig":
        return replace(self, lam=lam)


@dataclass(frozen=True)
class SolveReport:
    solution: object
    loss: float
    iterations: int
    sample_count: int
    wall_time: float


@dataclass(frozen=True)
class FactorGram:
    """``A^T A = v diag(eigenvalues) v^T``; eigenvalues descending, clipped at 0."""

    v: object
    eigenvalues: object
    matrix: object

    @property
    def dim(self) -> int:
        return int(self.v.shape[0])


def _gram_dev(a: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    n, d = int(a.shape[0]), int(a.shape[1])
    g = D.empty(d, d) if out is None else out
    if d <= 128:
        _lib.call("ks_gemm_tn_tall", d, d, n, 1.0, D.p(a), d, 1, D.p(a), d, 1, D.p(g), D.stream())
    else:
        _lib.call("ks_gemm", d, d, n, 1.0, D.p(a), 1, d, 0, D.p(a), d, 1, 0, 0.0, D.p(g), d, 1, 0, 1, D.stream())
    return g


def _factor_gram_dev(g: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Symmetrise and eigendecompose a PSD Gram on the device (one-sided Jacobi)."""
    d = int(g.shape[0])
    gs = (0.5 * (g + g.T)).contiguous()
    if d > 128:
        from .errors import SizeGuardError
        raise SizeGuardError(f"device eigensolver supports d <= 128, got {d}")
    w = D.empty(d)
    v = D.empty(d, d)
    _lib.call("ks_svd_small", D.p(gs), d, D.p(w), D.p(v), D.stream())
    return v, w, gs


def factor_gram(a, assume_gram: bool = False) -> FactorGram:
    """Eigendecomposition of ``a.T @ a`` (or of ``a`` if it is a Gram) -- solvers.py:143-150."""
    host = not D.on_device(a)
    at = as_matrix(a)
    g = at if assume_gram else _gram_dev(at)
    v, w, gs = _factor_gram_dev(g)
    return FactorGram(v=D.out(v, host), eigenvalues=D.out(w, host), matrix=D.out(gs, host))


@dataclass(frozen=True)
class FactorCache:
    svd: CompactSvd
    gram: FactorGram


def build_factor_cache(a) -> FactorCache:
    host = not D.on_device(a)
    at = as_matrix(a)
    u, s, v = _compact_svd_dev(at, 1e-10)
    gv, gw, gs = _factor_gram_dev(_gram_dev(at))
    o = lambda t: D.out(t, host)  # noqa: E731
    return FactorCache(svd=CompactSvd(u=o(u), sigma=o(s), v=o(v)), gram=FactorGram(v=o(gv), eigenvalues=o(gw),
                                                                                 matrix=o(gs)))


def pseudo_reciprocal(d):
    """Entrywise 1/d with zeros kept at zero (solvers.py:186-191)."""
    if isinstance(d, torch.Tensor):
        return torch.where(d > 0, 1.0 / torch.where(d > 0, d, torch.ones_like(d)), torch.zeros_like(d))
    d = np.asarray(d, dtype=np.float64)
    out = np.zeros_like(d)
    nz = d > 0
    out[nz] = 1.0 / d[nz]
    return out


@dataclass(frozen=True)
class KronPreconditioner:
    """``(V kron ...) D (V kron ...)^T`` (solvers.py:166-183)."""

    v_factors: tuple
    d_diag: object
    lam: float

    def apply(self, x):
        host = not D.on_device(x)
        vs = [D.to_dev(v) for v in self.v_factors]
        dd = D.to_dev(self.d_diag)
        xt = D.to_dev(x).reshape(-1)
        if len(vs) == 2:
            d1, d2 = int(vs[0].shape[0]), int(vs[1].shape[0])
            if d1 <= 128 and d2 <= 128:
                y = D.empty(d1 * d2)
                _lib.call("ks_kron_precond_apply", D.p(vs[0]), D.p(vs[1]), d1, d2, D.p(dd), D.p(xt.contiguous()),
                          D.p(y), D.stream())
                return D.out(y, host)
        t = _kron_apply_dev([v.T.contiguous() for v in vs], xt[:, None].contiguous())[:, 0] * dd
        return D.out(_kron_apply_dev(vs, t[:, None].contiguous())[:, 0], host)


def build_kron_preconditioner(grams: Sequence[FactorGram], lam: float) -> KronPreconditioner:
    host = not D.on_device(grams[0].eigenvalues)
    eig = reduce(torch.kron, [D.to_dev(g.eigenvalues) for g in grams])
    dd = pseudo_reciprocal(eig + lam)
    return KronPreconditioner(v_factors=tuple(g.v for g in grams), d_diag=D.out(dd, host), lam=lam)


def _norm(x) -> float:
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            out = D.empty(1)
            xt = x.reshape(-1).to(D.F64).contiguous()
            _lib.call("ks_sumsq_diff", D.p(xt), D.p(None), xt.numel(), D.p(out), D.stream())
            return math.sqrt(float(out.item()))
        return float(torch.linalg.norm(x.reshape(-1).to(torch.float64)))
    return float(np.linalg.norm(np.asarray(x, dtype=np.float64)))


def richardson_solve(apply_normal: Callable, apply_precond: Callable, rhs, damping: float,
                     config: RegressionConfig, x0=None, callback: Callable | None = None):
    """Damped preconditioned Richardson iteration with user callables (solvers.py:201-248).

    Works on NumPy arrays or CUDA tensors (whatever the callables consume).  The fused
    device loop used by ``fast_kronecker_regression`` is ``ks_richardson_sketched``."""
    if isinstance(rhs, torch.Tensor):
        rhs = rhs.reshape(-1).to(torch.float64)
        x = torch.zeros_like(rhs) if x0 is None else torch.as_tensor(x0, dtype=torch.float64,
                                                                      device=rhs.device).clone()
    else:
        rhs = np.asarray(rhs, dtype=np.float64).reshape(-1)
        x = np.zeros_like(rhs) if x0 is None else np.array(x0, dtype=np.float64)
    if tuple(x.shape) != tuple(rhs.shape):
        raise InvalidInputError("x0 must match the right-hand side length")
    scale = _norm(apply_precond(rhs))
    tol = config.residual_tol * max(scale, np.finfo(float).tiny)
    history: list[float] = []
    iterations = 0
    for _ in range(config.effective_max_iters):
        step = apply_precond(apply_normal(x) - rhs)
        norm = _norm(step)
        history.append(norm)
        if norm <= tol:
            break
        if len(history) > _DIVERGENCE_WINDOW:
            window = history[-(_DIVERGENCE_WINDOW + 1):]
            if (all(window[i + 1] > window[i] for i in range(_DIVERGENCE_WINDOW))
                    and window[-1] > _DIVERGENCE_GROWTH * window[0]):
                raise NumericalFailureError("Richardson iteration diverged", iterations=iterations,
                                            diagnostics={"residual_history": history})
        x = x - damping * step
        iterations += 1
        if callback is not None:
            callback(x)
    return x, iterations


def _kron_dev(mats):
    """A_1 kron ... kron A_k (row-major, on the device) by successive ks_kron_explicit2 launches."""
    acc = mats[0].contiguous()
    for a in mats[1:]:
        a = a.contiguous()
        m, p = int(acc.shape[0]), int(acc.shape[1])
        k, q = int(a.shape[0]), int(a.shape[1])
        if m * k * p * q == 0:
            acc = D.zeros(m * k, p * q)
            continue
        out = D.empty(m * k, p * q)
        _lib.call("ks_kron_explicit2", D.p(acc), m, p, D.p(a), k, q, D.p(out), D.stream())
        acc = out
    return acc


def _split_first(facs):
    """(A_0, kron(A_1..)) with the right group materialised when N > 2."""
    if len(facs) == 2:
        return facs[0], facs[1]
    return facs[0], _kron_dev(facs[1:])


def _ridge_loss_dev(facs: list[torch.Tensor], x: torch.Tensor, b: torch.Tensor, lam: float) -> float:
    r2, x2 = _ridge_loss_parts(facs, x, b).cpu().tolist()
    return float(r2 + lam * x2)


def _ridge_loss_parts(facs: list[torch.Tensor], x: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """[||K x - b||^2, ||x||^2] on the device (no host round trip)."""
    out = D.empty(2)
    rows = [int(a.shape[0]) for a in facs]
    cols = [int(a.shape[1]) for a in facs]
    rest_entries = math.prod(rows[1:]) * math.prod(cols[1:])
    if len(facs) >= 2 and cols[0] <= 128 and math.prod(cols[1:]) <= 128 and rest_entries <= (1 << 25):
        L, R = _split_first(facs)
        X = x.reshape(cols[0], -1).contiguous()
        B = b.reshape(rows[0], -1)
        _lib.call("ks_kron2_residual_sumsq", D.p(L), D.p(X), D.p(R), D.p(B), int(B.shape[1]), rows[0],
                  int(B.shape[1]), cols[0], int(X.shape[1]), D.p(out[0:1]), D.stream())
    else:
        kx = _kron_apply_dev(facs, x.reshape(-1, 1).contiguous())[:, 0]
        _lib.call("ks_sumsq_diff", D.p(kx), D.p(b), kx.numel(), D.p(out[0:1]), D.stream())
    _lib.call("ks_sumsq_diff", D.p(x), D.p(None), x.numel(), D.p(out[1:2]), D.stream())
    return out


def ridge_loss(factors: Sequence, x, b, lam: float) -> float:
    """``||K x - b||^2 + lam ||x||^2`` without materialising K x (solvers.py:251-262)."""
    facs = check_factors(factors)
    rows, cols = kron_operator_shape(facs)
    xt = D.to_dev(x).reshape(-1).contiguous()
    bt = D.to_dev(b).reshape(-1).contiguous()
    if xt.numel() != cols or bt.numel() != rows:
        raise InvalidInputError(f"x/b of lengths {xt.numel()}/{bt.numel()} do not match operator {rows}x{cols}")
    return _ridge_loss_dev(facs, xt, bt, lam)


def _validated_problem(factors, b):
    """solvers.py:265-274: validated device factors; b is kept where it lives."""
    facs = [D.to_dev(a) for a in factors]
    if len(facs) == 0:
        raise InvalidInputError("need at least one factor")
    flags = torch.zeros(len(facs), 2, dtype=torch.int32, device=D.dev())
    for n, a in enumerate(facs):
        if a.ndim != 2:
            raise InvalidInputError(f"factor {n} must be 2-dimensional, got ndim={a.ndim}")
        if a.numel():
            _lib.call("ks_check_finite_nonzero", D.p(a), a.numel(), D.p(flags[n]), D.stream())
    fl = flags.cpu().tolist()
    for n, (bad, nz) in enumerate(fl):
        if bad:
            raise InvalidInputError(f"factor {n} contains non-finite entries")
    rows, cols = kron_operator_shape(facs)
    blen = int(b.numel()) if isinstance(b, torch.Tensor) else int(np.asarray(b).size)
    if blen != rows:
        raise InvalidInputError(f"b has length {blen}, operator has {rows} rows")
    for n, (bad, nz) in enumerate(fl):
        if not nz:
            raise InvalidInputError(f"factor {n} is identically zero")
    return facs, rows, cols


def _exact_solve_dev(facs: list[torch.Tensor], bt: torch.Tensor, lam: float) -> torch.Tensor:
    return _exact_solve_svds(facs, bt, lam, _compact_svds_dev(facs, 1e-10))


def _exact_solve_svds(facs: list[torch.Tensor], bt: torch.Tensor, lam: float, svds, loss_identity: list | None = None
                      ) -> torch.Tensor:
    """The exact solve after the factors' compact SVDs (solvers.py:312-318): no host round trip.

    ``loss_identity`` (a list, optional): when the K1 / K13 pass runs, ||b||^2 comes out of
    the same pass and [ridge loss, ||b||^2] by the exact-solution identity
    ||K x - b||^2 + lam ||x||^2 = ||b||^2 - sum_k s_k^2 t_k^2 / (s_k^2 + lam)   (t = U^T b, s = kron of
    the singular values) is appended as one device tensor -- no second pass over b.  The caller
    checks the cancellation before trusting it."""
    us = [s[0] for s in svds]
    ranks = [int(s[1].numel()) for s in svds]
    if min(ranks) == 0:
        return D.zeros(math.prod(int(a.shape[1]) for a in facs))
    bsq = None
    rest_rows = math.prod(int(a.shape[0]) for a in facs[1:])
    rest_rank = math.prod(ranks[1:])
    nk = [int(a.shape[0]) for a in facs]
    if len(facs) == 3 and _lib.load().ks_kron3_supported(nk[0], nk[1], nk[2], *ranks) == 1:
        # K13: one streaming pass over b in the reference's rightmost-first order (ks_kron3.cu)
        T = D.empty(ranks[0], ranks[1] * ranks[2])
        us3 = [u.contiguous() for u in us]
        if loss_identity is not None:
            bsq = D.empty(1)
            _lib.call("ks_kron3_contract_sumsq", D.p(us3[0]), D.p(us3[1]), D.p(us3[2]), D.p(bt), nk[0], nk[1],
                      nk[2], *ranks, D.p(T), D.p(bsq), D.stream())
        else:
            _lib.call("ks_kron3_contract", D.p(us3[0]), D.p(us3[1]), D.p(us3[2]), D.p(bt), nk[0], nk[1], nk[2],
                      *ranks, D.p(T), D.stream())
        t = T.reshape(-1)
    elif len(facs) >= 2 and ranks[0] <= 128 and rest_rank <= 128 and rest_rows * rest_rank <= (1 << 25):
        # the n^2 pass on the FP64 tensor pipe (TMA + DMMA K1 kernel): t = U_0^T B U_rest with
        # B the n_0 x prod(n_rest) reshape of b and, for N >= 3, the right group's U's
        # materialised as one Kronecker product (the Tucker core's K13: 512 x 32768 B at c5)
        n1 = int(facs[0].shape[0])
        U0, Ur = _split_first(us)
        T = D.empty(ranks[0], rest_rank)
        if loss_identity is not None:
            bsq = D.empty(1)
            _lib.call("ks_kron2_contract_sumsq", D.p(U0), D.p(bt), rest_rows, D.p(Ur.contiguous()), n1, rest_rows,
                      ranks[0], rest_rank, D.p(T), D.p(bsq), D.stream())
        else:
            _lib.call("ks_kron2_contract", D.p(U0), D.p(bt), rest_rows, D.p(Ur.contiguous()), n1, rest_rows,
                      ranks[0], rest_rank, D.p(T), D.stream())
        t = T.reshape(-1)
    else:
        t = _kron_apply_dev([u.T.contiguous() for u in us], bt.reshape(-1, 1).contiguous())[:, 0]
    sigma = reduce(torch.kron, [s[1] for s in svds])
    if bsq is not None:
        s2 = sigma * sigma
        loss_identity.append(torch.cat([bsq - torch.sum(t * t * s2 / (s2 + lam)).reshape(1), bsq]))
    t = t * (sigma / (sigma * sigma + lam))
    return _kron_apply_dev([s[2] for s in svds], t.reshape(-1, 1).contiguous())[:, 0]


def kronmatmul_svd_solve(factors: Sequence, b, lam: float, *, with_loss: bool = True) -> SolveReport:
    """Exact ridge solution from factor SVDs and implicit Kronecker products (solvers.py:302-320).
    ``with_loss=False`` (an extension, as for fast_kronecker_regression) skips the loss: nan."""
    host = not D.on_device(b)
    if not host and lam >= 0:
        got = _exact_solve_graph(factors, b, lam, with_loss)
        if got is not None:
            x, loss, wall = got
            return SolveReport(solution=x, loss=loss, iterations=0, sample_count=0, wall_time=wall)
    facs, rows, cols = _validated_problem(factors, b)
    if lam < 0:
        raise InvalidInputError(f"lambda must be >= 0, got {lam}")
    bt = D.to_dev(b).reshape(-1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = _exact_solve_dev(facs, bt, lam)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    loss = _ridge_loss_dev(facs, x, bt, lam) if with_loss else float("nan")
    return SolveReport(solution=D.out(x, host), loss=loss, iterations=0, sample_count=0, wall_time=wall)


class _ExactGraph:
    """Captured exact solve (compact SVDs, the n-pass, scaling, back-transform, loss) for one key:
    the factors are copied into the entry's own buffers before every replay (the Tucker ALS passes
    new factor tensors on every sweep), b is read in place (keyed by its address)."""

    def __init__(self, ranks):
        self.ranks = ranks
        self.identity = False
        self.disabled = False
        self.graph = None
        self.facs = None
        self.out = None


_EXACT_GRAPHS: dict = {}


def _exact_graph_key(facs, bt, lam, with_loss=True):
    if not (_USE_GRAPHS[0] and bt.is_cuda and bt.dtype == torch.float64 and bt.is_contiguous()):
        return None
    if any(a.dtype != torch.float64 for a in facs) or min(min(int(x) for x in a.shape) for a in facs) == 0:
        return None
    return (_state.thread_key(), torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream,
            tuple(tuple(a.shape) for a in facs), (bt.data_ptr(), bt.numel()), float(lam), bool(with_loss))


def _exact_solve_graph(factors, b, lam, with_loss=True):
    """(x, loss, wall) of the exact solve from a replayed graph, or None: the eager path then runs
    (first sight of the key -- it records the factors' ranks --, a rank that moved, a declined
    CholeskyQR2, or any input the eager validation has to reject in the reference's order).  The
    factors' finite / nonzero validation is a graph node; its flags lead the one read-back and raise
    the reference's errors (solvers.py:265-274) before any result is returned."""
    if not all(isinstance(a, torch.Tensor) and a.is_cuda for a in factors) or len(factors) == 0:
        return None
    facs = list(factors)
    if any(a.ndim != 2 for a in facs):
        return None
    rows, _ = kron_operator_shape(facs)
    if int(b.numel()) != rows:
        return None
    bt = b.reshape(-1)
    key = _exact_graph_key(facs, bt, lam, with_loss)
    if key is None:
        return None
    entry = _state.cache_get(_EXACT_GRAPHS, key)
    if entry is not None and entry.disabled:
        return None
    if entry is None:
        svds = _compact_svds_dev([a.contiguous() for a in facs], 1e-10)
        _state.cache_put(_EXACT_GRAPHS, key, _ExactGraph([int(sv[1].numel()) for sv in svds]), _GRAPH_CAP)
        return None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if entry.graph is None:
        entry.facs = [torch.empty(tuple(a.shape), dtype=a.dtype, device=a.device) for a in facs]  # row-major
        for dst, a in zip(entry.facs, facs):
            dst.copy_(a)
        g = torch.cuda.CUDAGraph()
        with GATE.capture() as ok:
            if not ok:
                return None
            try:
                with torch.cuda.graph(g, capture_error_mode=CAPTURE_MODE):
                    flags = torch.zeros(len(facs), 2, dtype=torch.int32, device=D.dev())
                    for n, a in enumerate(entry.facs):
                        _lib.call("ks_check_finite_nonzero", D.p(a), a.numel(), D.p(flags[n]), D.stream())
                    svds = []
                    info = torch.zeros(2 * len(facs), dtype=torch.int32, device=D.dev())
                    for i, (a, r) in enumerate(zip(entry.facs, entry.ranks)):
                        n, d = int(a.shape[0]), int(a.shape[1])
                        k = min(n, d)
                        u, sg, v = D.empty(n, k), D.empty(k), D.empty(d, k)
                        _lib.call("ks_compact_svd_async", D.p(a), n, d, 1e-10, D.p(u), D.p(sg), D.p(v),
                                  D.p(info[2 * i:2 * i + 2]), D.stream())
                        svds.append((u[:, :r].contiguous(), sg[:r].contiguous(), v[:, :r].contiguous(), sg))
                    ident = [] if with_loss else None
                    x = _exact_solve_svds(entry.facs, bt, lam, svds, loss_identity=ident)
                    # the loss: [identity value, ||b||^2] when the K1 / K13 pass gave ||b||^2 (no second
                    # pass over b), else the direct pass [||K x - b||^2, ||x||^2]
                    entry.identity = bool(ident)
                    if not with_loss:
                        parts = torch.zeros(2, dtype=torch.float64, device=D.dev())
                    else:
                        parts = ident[0] if ident else _ridge_loss_parts(entry.facs, x, bt)
                    # one read-back: the loss parts, the QR status words, every factor's singular
                    # values (the ranks check)
                    entry.out = {"x": x, "back": torch.cat([flags.reshape(-1).to(torch.float64), parts,
                                                            info.to(torch.float64)] + [sv[3] for sv in svds])}
            except Exception:
                _state.cache_drop(_EXACT_GRAPHS, key)
                raise
        entry.graph = g
    else:
        for dst, a in zip(entry.facs, facs):
            dst.copy_(a)
    entry.graph.replay()
    x = entry.out["x"].clone()
    back = entry.out["back"].cpu().tolist()
    wall = time.perf_counter() - t0
    nf = len(facs)
    fl = back[:2 * nf]
    for n in range(nf):
        if fl[2 * n]:
            raise InvalidInputError(f"factor {n} contains non-finite entries")
    for n in range(nf):
        if not fl[2 * n + 1]:
            raise InvalidInputError(f"factor {n} is identically zero")
    back = back[2 * nf:]
    if any(v != 0.0 for v in back[2:2 + 2 * nf]):  # a CholeskyQR2 declined: Householder, eagerly
        entry.disabled = True  # and from now on for this key (the factorisation would decline again)
        return None
    off = 2 + 2 * nf
    for a, r in zip(facs, entry.ranks):
        k = min(int(a.shape[0]), int(a.shape[1]))
        h = back[off:off + k]
        off += k
        if (sum(1 for v in h if v > 1e-10 * h[0]) if h[0] > 0.0 else 0) != r:
            _state.cache_drop(_EXACT_GRAPHS, key)  # the numerical rank moved: recompute eagerly
            return None
    if not with_loss:
        return x, float("nan"), wall
    if not entry.identity:
        return x, float(back[0] + lam * back[1]), wall
    loss, bsq = back[0], back[1]
    if not loss >= _IDENTITY_MIN_FRAC * bsq:
        # more than three digits of ||b||^2 cancel (a near-exact fit): the direct pass instead
        r2, x2 = _ridge_loss_parts(entry.facs, x, bt).cpu().tolist()  # the row-major copies
        loss = r2 + lam * x2
    return x, float(loss), wall


# the exact solve's loss comes from ||b||^2 - sum s^2 t^2 / (s^2 + lam) only while the loss keeps at
# least this fraction of ||b||^2 (relative error <= ~1e-13 / fraction); below it, the direct pass
_IDENTITY_MIN_FRAC = 1e-3


def exact_factor_scores(factors: Sequence, caches: Sequence[FactorCache] | None = None) -> list[LeverageScores]:
    out = []
    for n, a in enumerate(factors):
        svd = caches[n].svd if caches is not None else compact_svd(a)
        out.append(ridge_leverage_scores(svd, 0.0))
    return out


def _regression_sample_count(cols: int, config: RegressionConfig) -> int:
    return max(1, math.ceil(config.effective_alpha * REGRESSION_SAMPLE_CONSTANT * cols
                            * math.log(40 * cols) * math.log(1.0 / config.delta) / config.eps))


_SIDE = {}


def _side_stream(k: int = 0) -> torch.cuda.Stream:
    """k-th auxiliary stream of the current stream (0: eigensolves, 1..: per-factor JL work).
    Keyed by the current stream, so concurrent solves on their own streams (and a capture, which
    runs on its own capture stream) never share a side stream."""
    key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream, k)
    s = _SIDE.get(key)
    if s is None:
        with CACHE_LOCK:
            s = _SIDE.get(key)
            if s is None:
                s = torch.cuda.Stream(device=key[0])
                _SIDE[key] = s
    return s


def _factor_grams_async(gts: list[torch.Tensor]):
    """Launch the Gram eigendecompositions on a side stream; returns a handle for _join_grams."""
    main = torch.cuda.current_stream()
    side = _side_stream()
    side.wait_stream(main)
    outs = []
    same = len({int(g.shape[0]) for g in gts}) == 1
    with torch.cuda.stream(side):
        if same and 1 < len(gts) <= 8:
            # one launch, one CTA per Gram, symmetrised on load
            d = int(gts[0].shape[0])
            w = D.empty(len(gts), d)
            v = D.empty(len(gts), d, d)
            _lib.call("ks_sym_eig_batched", len(gts), _lib.ptr_array(ctypes.c_void_p, [g.data_ptr() for g in gts]),
                      d, D.p(w), D.p(v), D.stream())
            outs = [(v[i], w[i]) for i in range(len(gts))]
            keep = [w, v]
        else:
            keep = []
            for g in gts:
                d = int(g.shape[0])
                if d <= 128:  # the same symmetric eigensolver as the batched / graph paths
                    w = D.empty(1, d)
                    v = D.empty(1, d, d)
                    _lib.call("ks_sym_eig_batched", 1, _lib.ptr_array(ctypes.c_void_p, [g.data_ptr()]), d, D.p(w),
                              D.p(v), D.stream())
                    outs.append((v[0], w[0]))
                    keep += [w, v]
                else:
                    vv, ww, gs = _factor_gram_dev(g)
                    outs.append((vv, ww))
    if not torch.cuda.is_current_stream_capturing():
        for g in gts:
            g.record_stream(side)
    ev = torch.cuda.Event()
    ev.record(side)
    return (outs, ev, keep)


def _join_grams(handle):
    if isinstance(handle, list):
        return handle
    if handle[0] == "per-factor":
        _, outs, evs = handle
        for ev in evs:
            torch.cuda.current_stream().wait_event(ev)
        return outs
    outs, ev, keep = handle
    torch.cuda.current_stream().wait_event(ev)
    if not torch.cuda.is_current_stream_capturing():
        for t in keep:
            t.record_stream(torch.cuda.current_stream())
    return outs


class _CholeskyFailed(Exception):
    """A JL Gram was not numerically positive definite; the solve is redone with LU inverses."""


def _chol_status(v):
    if v[0]:
        raise _CholeskyFailed()


def _jl_factor(gram: torch.Tensor) -> torch.Tensor:
    """Device factorisation of a JL Gram (first half of ks_jl_projection) into a workspace."""
    from .leverage import check_later
    d = int(gram.shape[0])
    ws = D.empty(d * (d + 1) + d)
    info = torch.zeros(1, dtype=torch.int32, device=gram.device)
    _lib.call("ks_jl_cholesky", D.p(gram), d, D.p(ws), D.p(info), D.stream())
    check_later(info, _chol_status)
    return ws


def _jl_scores_chol(a: torch.Tensor, a_tilde: torch.Tensor, gram: torch.Tensor, eps: float, seed,
                    log_factor: float, use_chol: bool = True, factor: torch.Tensor | None = None,
                    factor_stream=None, pre_g=None) -> torch.Tensor:
    """JL scores with (1+eps/4) (G a_tilde) gram^-1 from a device Cholesky solve (leverage.py:114-129).
    The positive-definiteness flag is checked with the solve's other deferred flags; on failure
    the solve is repeated with ``use_chol=False`` (LU inverse, as the reference's np.linalg.inv).
    ``factor``: a workspace from _jl_factor (made on ``factor_stream``)."""
    from .leverage import _jl_ga, _jl_scores_from_q, check_later
    d = int(a.shape[1])
    tl = _TL_CUR[0]
    if pre_g is not None and tl is not None:
        torch.cuda.current_stream().wait_event(pre_g[1])
        _tl_event(tl, f"jl g ready ({int(a.shape[0])})")
    ga, r = _jl_ga(a, a_tilde, seed, log_factor, pre_g)
    _tl_event(tl, "jl ga")
    q = D.empty(r, d)
    if use_chol and factor is not None:
        if factor_stream is not None:
            torch.cuda.current_stream().wait_stream(factor_stream)
            _tl_event(tl, "jl factor ready")
        _lib.call("ks_jl_solve", D.p(factor), d, D.p(ga), r, 1.0 + eps / 4.0, D.p(q), D.stream())
        _tl_event(tl, "jl solve")
    elif use_chol:
        info = torch.zeros(1, dtype=torch.int32, device=a.device)
        _lib.call("ks_jl_projection", D.p(gram), d, D.p(ga), r, 1.0 + eps / 4.0, D.p(q), D.p(info), D.stream())
        check_later(info, _chol_status)
    else:
        gi = _inverse_small(gram)
        _lib.call("ks_gemm", r, d, d, 1.0 + eps / 4.0, D.p(ga), d, 1, 0, D.p(gi), d, 1, 0, 0.0, D.p(q), d, 1, 0, 1,
                  D.stream())
    return _jl_scores_from_q(a, q, r, eps)


def _inverse_from_eig(v: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    d = int(w.numel())
    if float(w.min().item()) <= 0.0:
        raise NumericalFailureError("approximate Gram matrix is singular; cannot estimate leverage scores",
                                    diagnostics={"shape": (d, d)})
    vs = (v / w[None, :]).contiguous()
    out = D.empty(d, d)
    _lib.call("ks_gemm", d, d, d, 1.0, D.p(vs), d, 1, 0, D.p(v), 1, d, 0, 0.0, D.p(out), d, 1, 0, 1, D.stream())
    return out


class FastSolveTrace:
    """Device intermediates of one fast solve (parity tests compare them with the oracle)."""

    def __init__(self):
        self.__dict__.update(scores=[], eig=[], sampler=None, sketch=None, sdiag=None, rhs=None, history=[],
                             a_tilde_rows=[])


# ---------------------------------------------------------------------------------------------
# Whole-solve CUDA graph (two factors, single-factor groups, device or page-locked b): Grams,
# eigensolves (side stream), JL estimates, sampler, draws, sparse diagonal + view, the b gather
# and the fused right-hand-side + Richardson launch are one graph; a replay costs one launch and
# one small device->host read of the loop state, the history and the validation flags.
# ---------------------------------------------------------------------------------------------


class _SolveGraph:
    def __init__(self):
        self.graph = None
        self.out = None
        self.checks = []


_SOLVE_GRAPHS: dict = {}
_LAST_LOOP_EVENTS = TLSlot()  # this thread's (stage start, end, kernel start) events of its last replayed loop
_LAST_HISTORY = TLSlot()  # this thread's last fast solve: the Richardson step-norm history
_SOLVE_STATS = {"eager": 0, "capture": 0, "replay": 0}
_GRAPH_CAP = 16  # cached whole-solve graphs (keys are per thread and per stream)


def last_solve_history() -> list:
    """Step norms of the calling thread's last fast solve (graph or eager path): the history the
    reference's richardson_solve appends (solvers.py:226-230)."""
    h = _LAST_HISTORY[0]
    return list(h) if h is not None else []


_USE_SOLVE_GRAPH = [True]


def _solve_graph_key(facs, b, config: RegressionConfig):
    if not (_USE_SOLVE_GRAPH[0] and _USE_GRAPHS[0] and _USE_FUSED[0]) or len(facs) != 2 \
            or not grouped2_eligible(facs):
        return None
    d0, d1 = int(facs[0].shape[1]), int(facs[1].shape[1])
    if d0 not in (16, 32, 64) or d1 not in (16, 32, 64) or config.effective_max_iters > 1024:
        return None
    if not isinstance(b, torch.Tensor) or b.dtype != torch.float64 or not b.is_contiguous():
        return None
    if not (b.is_cuda or b.is_pinned()):
        return None
    try:
        key = (_state.thread_key(), torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream,
               tuple((a.data_ptr(), tuple(a.shape), tuple(a.stride())) for a in facs),
               (b.data_ptr(), b.numel(), b.is_cuda), config, _switches())
        hash(key)
    except TypeError:
        return None
    return key


def _switches():
    """The process-wide path switches a captured graph bakes in (part of every graph key)."""
    return (_NO_PREDRAW[0], _TIMELINE[0], _GATHER_BESIDE[0], _USE_FUSED[0])


def _eig_on(stream, g, tl=None, name=""):
    d = int(g.shape[0])
    w = D.empty(1, d)
    v = D.empty(1, d, d)
    _tl_event(tl, name + " start", stream)
    with torch.cuda.stream(stream):
        _lib.call("ks_sym_eig_batched", 1, _lib.ptr_array(ctypes.c_void_p, [g.data_ptr()]), d, D.p(w), D.p(v),
                  D.stream())
    _tl_event(tl, name, stream)
    ev = torch.cuda.Event()
    ev.record(stream)
    return (v[0], w[0]), ev


# diagnostic switches, read once at import and part of every graph key
_NO_PREDRAW = [bool(os.environ.get("KS_NO_PREDRAW"))]
_TIMELINE = [bool(os.environ.get("KS_GRAPH_TIMELINE"))]  # external events at the solve graph's joins
_GATHER_BESIDE = [os.environ.get("KS_GATHER_BESIDE_SKETCH") == "1"]  # sampled-b gather beside the sketch
_TL_CUR = TLSlot()  # the timeline this thread is capturing


def _tl_event(tl, name, stream=None):
    if tl is None:
        return
    ev = torch.cuda.Event(enable_timing=True, external=True)
    ev.record(stream if stream is not None else torch.cuda.current_stream())
    tl.append((name, ev))


def _tilde_rows(facs, config: RegressionConfig):
    """Rows of each factor's JL input: s_n spectral rows when row sampling applies (solvers.py:421-436),
    else all n rows."""
    nf = len(facs)
    eps_one = math.log1p(config.eps / 4.0) / nf
    eps_two = eps_one / (2.0 + eps_one)
    delta_n = config.delta / (2.0 * nf)
    out = []
    for a in facs:
        s_n = math.ceil(config.effective_alpha * spectral_sample_count(int(a.shape[1]), eps_two, delta_n))
        out.append(s_n if s_n < int(a.shape[0]) else int(a.shape[0]))
    return out, eps_two, delta_n


def _predraw_jl_sketches(facs, config: RegressionConfig, seeds):
    """The JL Gaussian sketches (leverage.py:124-126) depend only on the seeds and the shapes: draw
    them first, each on its own stream (off the Gram / upload critical path).  Returns per factor
    (g, event)."""
    from .leverage import device_standard_normal, jl_projection_rows
    main = torch.cuda.current_stream()
    nts, _, _ = _tilde_rows(facs, config)
    out = []
    for n, a in enumerate(facs):
        r = jl_projection_rows(int(a.shape[0]), config.jl_log_factor)
        st = _side_stream(12 + n)
        st.wait_stream(main)
        with torch.cuda.stream(st):
            g = device_standard_normal(seeds[2 * n + 1], r * nts[n], divisor=math.sqrt(r))
        ev = torch.cuda.Event()
        ev.record(st)
        out.append((g, ev))
    return out


def _solve_graph_body(facs, b, config: RegressionConfig, s: int, factor1_stream=None, pre_g=None):
    """Launch-only device pipeline of the fused two-factor solve (captured once per key).

    ``factor1_stream``: the stream on which facs[1] becomes ready (its upload, when the graph also
    holds the host-to-device copies); then factor 1's Gram, eigensolve and JL chain start as soon
    as it lands, while factor 0's already run (per-factor eigensolve launches instead of the batched
    one)."""
    seeds = _spawned_seeds(config.seed, 5)
    eps_jl = 4.0 * math.log1p(config.eps / 4.0) / 2
    d0, d1 = int(facs[0].shape[1]), int(facs[1].shape[1])
    main = torch.cuda.current_stream()
    tl = [] if _TIMELINE[0] else None
    _TL_CUR[0] = tl
    _tl_event(tl, "start")
    if pre_g is None and not _NO_PREDRAW[0]:
        pre_g = _predraw_jl_sketches(facs, config, seeds)
    # per factor, on its own stream as soon as the factor exists: the spectral row sample when it
    # applies (leverage.py:235-252), the Gram of the JL input, then its eigendecomposition
    nts, eps_two, delta_n = _tilde_rows(facs, config)
    f1s = factor1_stream if factor1_stream is not None else _side_stream(8)
    if factor1_stream is None:
        f1s.wait_stream(main)
    tildes, gts, evs = [], [], []
    for n, a in enumerate(facs):
        with torch.cuda.stream(main if n == 0 else f1s):
            if nts[n] < int(a.shape[0]):
                at = _spectral_rows_dev(a, eps_two, delta_n, seeds[2 * n], config.effective_alpha,
                                        divisor=math.sqrt(1.0 - eps_two))
            else:
                at = a
            gts.append(_gram_dev(at))
            tildes.append(at)
            ev = torch.cuda.Event()
            ev.record()
            evs.append(ev)
    e0s, e1s = _side_stream(0), _side_stream(10)
    e0s.wait_event(evs[0])
    e1s.wait_event(evs[1])
    _tl_event(tl, "gram0", e0s)
    _tl_event(tl, "gram1", e1s)
    r0, ev_e0 = _eig_on(e0s, gts[0], tl, "eig0")
    r1, ev_e1 = _eig_on(e1s, gts[1], tl, "eig1")
    grams_h = ("per-factor", [r0, r1], [ev_e0, ev_e1])
    ready = [None, evs[1]]
    b_raw = D.empty(max(s, 1))
    gst = _side_stream(11)
    _, _, _, _, _, g2 = _jl_and_sampling(facs, tildes, gts, eps_jl, config, True, seeds, s, ready,
                                         (b, b_raw, gst), pre_g)
    sd_idx, sd_val, seg, lrow, rrow, cdev, first_raw = g2
    _tl_event(tl, "sketch")
    struct = _lib.SketchView(facs[0].data_ptr(), d0, d0, facs[1].data_ptr(), d1, d1, s, s, seg.data_ptr(),
                             lrow.data_ptr(), rrow.data_ptr(), sd_val.data_ptr())
    # the loop's work plan needs only the sketch: built while the eigensolves and the b gather
    # still run
    plan_ws = torch.empty(int(_lib.load().ks_richardson_plan_bytes(s, s)), dtype=torch.uint8, device=D.dev())
    _lib.call("ks_richardson_plan_async", ctypes.byref(struct), D.p(cdev), D.p(plan_ws), D.stream())
    _tl_event(tl, "plan")
    main.wait_stream(gst)
    _tl_event(tl, "b gathered")
    b_at = D.empty(s)  # b at the sparse-diagonal rows = b_raw at each entry's first draw
    _lib.call("ks_gather_count", D.p(b_raw), D.p(first_raw), D.p(cdev), s, D.p(b_at), D.stream())
    (VL, wL), (VR, wR) = _join_grams(grams_h)
    max_iters = config.effective_max_iters
    x = D.empty(d0, d1)
    hist = D.zeros(max(1, max_iters))
    rhs = D.empty(d0, d1)
    state = torch.zeros(4, dtype=torch.int32, device=D.dev())
    # external events around the loop launch: readable after every replay (bench.py's roofline)
    ev0 = torch.cuda.Event(enable_timing=True, external=True)
    evk = torch.cuda.Event(enable_timing=True, external=True)  # recorded by the C entry before the kernel
    ev1 = torch.cuda.Event(enable_timing=True, external=True)
    ev0.record()
    evk.record()  # creates the event; the C entry records it again right before the persistent launch
    _lib.load().ks_debug_loop_kernel_event(ctypes.c_void_p(evk.cuda_event))
    try:
        _lib.call("ks_richardson_fused_async", ctypes.byref(struct), D.p(cdev), None, D.p(b_at), D.p(VL), D.p(wL),
                  D.p(VR), D.p(wR), None, float(config.lam), float(config.effective_damping), int(max_iters),
                  float(config.residual_tol), D.p(x), D.p(hist), D.p(rhs), D.p(state), D.p(plan_ws), D.stream())
    finally:
        _lib.load().ks_debug_loop_kernel_event(None)
    ev1.record()
    _tl_event(tl, "loop end")
    _TL_CUR[0] = None
    return dict(x=x, hist=hist, state=state, loop_events=(ev0, ev1, evk), timeline=tl,
                keep=(gts, tildes, b_at, b_raw, first_raw, sd_idx, sd_val, seg, lrow, rrow, cdev, rhs, plan_ws,
                      pre_g))


class _PackedChecks:
    """Every deferred flag word and the loop state of a solve graph, packed inside the graph into one
    int32 buffer: one device-to-host copy per replay (into a page-locked buffer allocated once)
    instead of one copy per flag.  Handlers run in registration order, as DeferredChecks does."""

    def __init__(self, checks, state, hist):
        self.slices = []
        parts, off = [], 0
        for f, h in checks:
            n = int(f.numel())
            parts.append(f.reshape(-1).to(torch.int32))
            self.slices.append((off, n, h))
            off += n
        self.state_off = off
        parts.append(state.reshape(-1).to(torch.int32))
        self.buf = torch.cat(parts)  # a graph node: refreshed by every replay
        self.host = torch.empty(int(self.buf.numel()), dtype=torch.int32).pin_memory()
        self.hist = hist
        self.hist_host = torch.empty(int(hist.numel()), dtype=torch.float64).pin_memory()

    def fetch(self):
        self.host.copy_(self.buf, non_blocking=True)
        self.hist_host.copy_(self.hist, non_blocking=True)

    def run(self):
        """After a synchronisation: run the handlers; returns (status, iterations, hist_len, history)."""
        v = self.host.tolist()
        for off, n, h in self.slices:
            h(v[off:off + n])
        status, iters, hlen = v[self.state_off:self.state_off + 3]
        return status, iters, hlen, self.hist_host[:hlen].tolist()


def _fast_solve_graph(facs, b, config: RegressionConfig, key=None):
    """(x natural order, iterations, s) from the whole-solve graph, or None when this call has to
    run eagerly (ineligible input, or the first sight of a key: the eager pass warms every lazy
    initialisation before capture)."""
    from . import leverage as _lev
    if key is None:
        key = _solve_graph_key(facs, b, config)
    if key is None:
        return None
    entry = _state.cache_get(_SOLVE_GRAPHS, key)
    if entry is None:
        _state.cache_put(_SOLVE_GRAPHS, key, _SolveGraph(), _GRAPH_CAP)
        _SOLVE_STATS["eager"] += 1
        return None
    s = _regression_sample_count(math.prod(int(a.shape[1]) for a in facs), config)
    if entry.graph is None:
        g = torch.cuda.CUDAGraph()
        cap = _lev.DeferredChecks()
        outer = _lev._DEFERRED[0]
        _lev._DEFERRED[0] = cap
        gate = GATE.capture()
        try:
            if not gate.__enter__():
                return None  # other solves in flight: eager this time, captured on a later call
            with torch.cuda.graph(g, capture_error_mode=CAPTURE_MODE):
                # the factors' finite / nonzero validation rides in the graph on a side stream (off
                # the critical path); its flags lead the packed read-back, so a replay on new
                # contents at the same addresses raises the reference's error before any result
                main = torch.cuda.current_stream()
                flags = torch.zeros(len(facs), 2, dtype=torch.int32, device=D.dev())
                vst = _side_stream(24)
                vst.wait_stream(main)
                with torch.cuda.stream(vst):
                    flags.zero_()
                    for n, a in enumerate(facs):
                        _lib.call("ks_check_finite_nonzero", D.p(a), a.numel(), D.p(flags[n]), D.stream())
                entry.out = _solve_graph_body(facs, b.reshape(-1), config, s)
                main.wait_stream(vst)
                entry.packed = _PackedChecks([(flags.reshape(-1), _validation_handler(len(facs)))] + cap.items,
                                             entry.out["state"], entry.out["hist"])
                if _FETCH_IN_GRAPH[0]:
                    entry.packed.fetch()  # the read-back copies as graph nodes
        except Exception:
            _state.cache_drop(_SOLVE_GRAPHS, key)
            raise
        finally:
            gate.__exit__(None, None, None)
            _lev._DEFERRED[0] = outer
        entry.graph, entry.checks = g, cap.items
        _SOLVE_STATS["capture"] += 1
        _LAST_LOOP_EVENTS[0] = entry.out["loop_events"]
    else:
        _SOLVE_STATS["replay"] += 1
    _mark("graph launch")
    _LAST_LOOP_EVENTS[0] = entry.out["loop_events"]
    entry.graph.replay()
    out = entry.out
    if not _FETCH_IN_GRAPH[0]:
        entry.packed.fetch()
    x = out["x"].reshape(-1).clone()
    torch.cuda.current_stream().synchronize()
    _mark("richardson")
    try:
        status, iters, hlen, history = entry.packed.run()
    except (_CholeskyFailed, _lev.ScoresFallback):
        return None  # the eager path retries (LU inverses / compact-SVD scores)
    _LAST_HISTORY[0] = history
    if status == 2:
        raise NumericalFailureError("Richardson iteration diverged", iterations=iters,
                                    diagnostics={"residual_history": history})
    return x, iters, s


class _HostFacsGraph:
    """Whole-solve graph for page-locked HOST factors: the factor uploads and their validation are
    graph nodes too, so the upload of factor 1 overlaps factor 0's Gram / eigensolve / JL chain."""

    def __init__(self):
        self.graph = None
        self.dev = None
        self.flags = None
        self.out = None
        self.checks = []


_HOST_GRAPHS: dict = {}
# the whole-solve graphs' read-back copies (flags, loop state, history, x) captured as graph nodes
_FETCH_IN_GRAPH = [os.environ.get("KS_FETCH_OUTSIDE", "0") != "1"]


def _host_graph_key(factors, b, config: RegressionConfig):
    if not (_USE_SOLVE_GRAPH[0] and _USE_GRAPHS[0] and _USE_FUSED[0]) or len(factors) != 2:
        return None
    for a in factors:
        if not (isinstance(a, torch.Tensor) and not a.is_cuda and a.dtype == torch.float64 and a.ndim == 2
                and a.is_contiguous() and a.is_pinned()):
            return None
    if not (isinstance(b, torch.Tensor) and b.dtype == torch.float64 and b.is_contiguous()
            and (b.is_cuda or b.is_pinned())):
        return None
    rows = math.prod(int(a.shape[0]) for a in factors)
    if int(b.numel()) != rows:
        return None  # the regular path raises the reference's error
    for a in factors:
        n, d = int(a.shape[0]), int(a.shape[1])
        if d not in (16, 32, 64) or n < 16:
            return None
    if config.effective_max_iters > 1024:
        return None
    s = _regression_sample_count(math.prod(int(a.shape[1]) for a in factors), config)
    if s >= rows:
        return None
    try:
        key = ("host", _state.thread_key(), torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream,
               tuple((a.data_ptr(), tuple(a.shape)) for a in factors), (b.data_ptr(), b.numel(), b.is_cuda), config,
               _switches())
        hash(key)
    except TypeError:
        return None
    return key


def _validation_handler(nf: int):
    def handler(v):
        for n in range(nf):
            if v[2 * n]:
                raise InvalidInputError(f"factor {n} contains non-finite entries")
        for n in range(nf):
            if not v[2 * n + 1]:
                raise InvalidInputError(f"factor {n} is identically zero")
    return handler


def _fast_solve_host_graph(factors, b, config: RegressionConfig, with_loss: bool):
    """fast_kronecker_regression for page-locked host factors from one graph replay (uploads,
    validation, the whole solve), or None (first sight of the key / ineligible / LU retry needed)."""
    from . import leverage as _lev
    if not 0.0 < config.eps <= 0.25:
        return None
    key = _host_graph_key(factors, b, config)
    if key is None:
        return None
    entry = _state.cache_get(_HOST_GRAPHS, key)
    if entry is None:
        _state.cache_put(_HOST_GRAPHS, key, _HostFacsGraph(), _GRAPH_CAP)
        return None
    s = _regression_sample_count(math.prod(int(a.shape[1]) for a in factors), config)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _mark("t0")
    if entry.graph is None:
        entry.dev = [D.empty(*a.shape) for a in factors]
        entry.flags = torch.zeros(len(factors), 2, dtype=torch.int32, device=D.dev())
        g = torch.cuda.CUDAGraph()
        cap = _lev.DeferredChecks()
        outer = _lev._DEFERRED[0]
        _lev._DEFERRED[0] = cap
        gate = GATE.capture()
        try:
            if not gate.__enter__():
                entry.dev = None
                return None  # other solves in flight: the regular path this time
            with torch.cuda.graph(g, capture_error_mode=CAPTURE_MODE):
                main = torch.cuda.current_stream()
                # the JL sketches need no input data: drawn while the factors upload
                pre_g = None if _NO_PREDRAW[0] else _predraw_jl_sketches(entry.dev, config, _spawned_seeds(config.seed, 5))
                side = _side_stream(9)
                entry.dev[0].copy_(factors[0], non_blocking=True)
                side.wait_stream(main)  # after factor 0's upload: the PCIe link serves one copy at a time
                with torch.cuda.stream(side):
                    entry.dev[1].copy_(factors[1], non_blocking=True)
                    _lib.call("ks_check_finite_nonzero", D.p(entry.dev[1]), entry.dev[1].numel(),
                              D.p(entry.flags[1]), D.stream())
                _lib.call("ks_check_finite_nonzero", D.p(entry.dev[0]), entry.dev[0].numel(), D.p(entry.flags[0]),
                          D.stream())
                entry.out = _solve_graph_body(entry.dev, b.reshape(-1), config, s, factor1_stream=side, pre_g=pre_g)
                main.wait_stream(side)
                # the factor validation flags first: the reference validates before solving
                entry.packed = _PackedChecks([(entry.flags.reshape(-1), _validation_handler(len(factors)))]
                                             + cap.items, entry.out["state"], entry.out["hist"])
                entry.x_host = torch.empty(int(entry.out["x"].numel()), dtype=torch.float64).pin_memory()
                if _FETCH_IN_GRAPH[0]:
                    entry.packed.fetch()
                    entry.x_host.copy_(entry.out["x"].reshape(-1), non_blocking=True)
        except Exception:
            _state.cache_drop(_HOST_GRAPHS, key)
            raise
        finally:
            gate.__exit__(None, None, None)
            _lev._DEFERRED[0] = outer
        entry.graph, entry.checks = g, cap.items
    _mark("graph launch")
    _LAST_LOOP_EVENTS[0] = entry.out["loop_events"]
    entry.graph.replay()
    out = entry.out
    if not _FETCH_IN_GRAPH[0]:
        entry.packed.fetch()
        entry.x_host.copy_(out["x"].reshape(-1), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    _mark("richardson")
    try:
        status, iters, hlen, history = entry.packed.run()
    except (_CholeskyFailed, _lev.ScoresFallback):
        return None  # the regular path retries (LU inverses / compact-SVD scores)
    _LAST_HISTORY[0] = history
    x_h = entry.x_host
    if status == 2:
        raise NumericalFailureError("Richardson iteration diverged", iterations=iters,
                                    diagnostics={"residual_history": history})
    _mark("solve_end")
    wall = time.perf_counter() - t0
    if with_loss:
        x = out["x"].reshape(-1).clone()
        loss = _ridge_loss_dev(entry.dev, x, D.to_dev(b).reshape(-1), config.lam)
    else:
        loss = float("nan")
    return SolveReport(solution=x_h.numpy().copy(), loss=loss, iterations=iters, sample_count=s, wall_time=wall)


def _fast_sketch_dev(facs, config: RegressionConfig, caches=None):
    """The sketch and the preconditioner's factor eigendecompositions of fast_kronecker_regression
    (solvers.py:404-452) without the solve: (sparse diagonal, [(V_n, w_n)], s).  Deterministic: every
    rank of a row-sharded solve computes the same sketch."""
    from . import leverage as _lev
    use_chol, fast_scores = True, True
    for _attempt in range(3):
        deferred = _lev.DeferredChecks()
        _lev._DEFERRED[0] = deferred
        try:
            return _fast_solve_pass(facs, None, config, caches, None, use_chol, deferred, fast_scores,
                                    sketch_only=True)
        except _CholeskyFailed:
            use_chol = False
        except _lev.ScoresFallback:
            fast_scores = False
        finally:
            _lev._DEFERRED[0] = None
    raise AssertionError("unreachable")


def _fast_solve_dev(facs, b, config: RegressionConfig, caches, trace: FastSolveTrace | None = None):
    """The device pipeline of solvers.py:404-459; returns (x natural order, iterations, s)."""
    from . import leverage as _lev
    if caches is None and trace is None:
        got = _fast_solve_graph(facs, b, config)
        if got is not None:
            return got
    use_chol, fast_scores = True, True
    for _attempt in range(3):
        deferred = _lev.DeferredChecks()
        _lev._DEFERRED[0] = deferred
        failure = None
        try:
            return _fast_solve_pass(facs, b, config, caches, trace, use_chol, deferred, fast_scores)
        except (_CholeskyFailed, _lev.ScoresFallback) as exc:
            failure = exc
        except Exception:
            # a pending device flag (invalid scores, generator failure) explains a later error
            # better: raise the reference's exception for it first
            _lev._DEFERRED[0] = None
            try:
                deferred.run()
            except (_CholeskyFailed, _lev.ScoresFallback) as exc:
                failure = exc
            if failure is None:
                raise
        finally:
            _lev._DEFERRED[0] = None
        if isinstance(failure, _CholeskyFailed):
            assert use_chol
            use_chol = False
        else:
            assert fast_scores
            fast_scores = False
    raise AssertionError("unreachable")


_SEEDS: dict = {}


def _spawned_seeds(seed, count: int):
    """SeedSequence(seed).spawn(count) (solvers.py:415-416), memoised for integer seeds: the
    children are a pure function of (seed, count) and spawning costs ~60 us of host time."""
    if isinstance(seed, (int, np.integer)) and not isinstance(seed, bool):
        key = (int(seed), count)
        got = _SEEDS.get(key)
        if got is None:
            if len(_SEEDS) > 256:
                _SEEDS.clear()
            got = _SEEDS[key] = tuple(np.random.SeedSequence(int(seed)).spawn(count))
        return got
    return np.random.SeedSequence(seed).spawn(count)


def _jl_and_sampling(facs, tildes, gts, eps_jl: float, config: RegressionConfig, use_chol: bool, seeds, s: int,
                     ready=None, raw_b=None, pre_g=None):
    """JL leverage estimates of every factor (leverage.py:85-130), the product sampler's tables
    and the s draws with their weights (solvers.py:430-452).  Launch-only: no host round trips,
    so the whole stage can be captured in a CUDA graph."""
    scores, afs = [], []
    main = torch.cuda.current_stream()
    capturing = torch.cuda.is_current_stream_capturing()
    # the per-factor JL estimates are independent: factor n > 0 runs on its own stream, and every
    # Gram factorisation (needs only the Gram) runs on its own stream while the Gaussian sketch is
    # drawn (all streams fork here, before any work is enqueued)
    nf = len(facs)
    chol_st = [_side_stream(16 + n) for n in range(nf)] if use_chol else []

    def fork(st, n):  # ready[n]: event after which factor n's inputs exist (else: main's progress)
        if ready is not None and ready[n] is not None:
            st.wait_event(ready[n])
        else:
            st.wait_stream(main)

    for n in range(1, nf):
        fork(_side_stream(n), n)
    for n, cs in enumerate(chol_st):
        fork(cs, n)
    factors = []
    for n in range(nf):
        if use_chol:
            with torch.cuda.stream(chol_st[n]):
                factors.append(_jl_factor(gts[n]))
    for n, a in enumerate(facs):
        st = main if n == 0 else _side_stream(n)
        with torch.cuda.stream(st):
            scores.append(_jl_scores_chol(a, tildes[n], gts[n], eps_jl, seeds[2 * n + 1], config.jl_log_factor,
                                          use_chol, factors[n] if use_chol else None,
                                          chol_st[n] if use_chol else None,
                                          pre_g[n] if pre_g is not None else None))
        afs.append(1.0 + eps_jl / 2.0)
    for n in range(1, nf):
        main.wait_stream(_side_stream(n))
        if not capturing:
            scores[n].record_stream(main)
    for cs in chol_st:
        main.wait_stream(cs)
    _tl_event(_TL_CUR[0], "jl scores")
    sampler = ProductSampler([LeverageScores(sc, 0.0, af) for sc, af in zip(scores, afs)])
    _tl_event(_TL_CUR[0], "sampler tables")
    state, inc = pcg64_state(seeds[-1])
    draws = sampler._sample_dev(s, state, inc)
    w = sampler._weights_dev(draws, s)
    _tl_event(_TL_CUR[0], "draws")
    # two factors: the sparse diagonal and its grouped view are built here too (launch-only)
    if raw_b is not None and _USE_FUSED[0] and grouped2_eligible(facs):
        # raw_b = (b, out): b read at the raw draws on a side stream while the sketch is sorted and
        # deduplicated (the read may cross PCIe: page-locked host b); joined by the caller
        b, b_raw, gst = raw_b
        # the gather is issued after the sketch kernels: run beside them, the scattered reads (one
        # PCIe request each when b is page-locked host memory) slow both down, and the sum is the
        # same (tools/graph_timeline.py --host); the loop plan then overlaps the gather
        after = not _GATHER_BESIDE[0]
        if not after:
            gst.wait_stream(main)
            with torch.cuda.stream(gst):
                _lib.call("ks_gather_draws2", D.p(b), D.p(draws), int(facs[1].shape[0]), s, D.p(b_raw), D.stream())
        first_raw = D.empty(max(s, 1), dtype=D.I64)
        g2 = sketch_diag_grouped2_launch(facs, draws, w, first_raw) + (first_raw,)
        if after:
            gst.wait_stream(main)
            with torch.cuda.stream(gst):
                _lib.call("ks_gather_draws2", D.p(b), D.p(draws), int(facs[1].shape[0]), s, D.p(b_raw), D.stream())
        return scores, afs, sampler, draws, w, g2
    g2 = sketch_diag_grouped2_launch(facs, draws, w) if _USE_FUSED[0] and grouped2_eligible(facs) else None
    return scores, afs, sampler, draws, w, g2


class _PrefixGraph:
    """CUDA graph of _jl_and_sampling for one (factor buffers, shapes, config) key.  The Grams
    are written into ``gts`` (static inputs) eagerly before every replay; outputs and deferred
    flag tensors are static graph-pool tensors."""

    def __init__(self):
        self.graph = None
        self.gts = None
        self.out = None
        self.checks = []


_PREFIX_GRAPHS: dict = {}
_USE_FUSED = [True]  # fused right-hand side + loop kernel for single-factor groups
_PREFIX_STATS = {"eager": 0, "capture": 0, "replay": 0}
_USE_GRAPHS = [True]


def _prefix_key(facs, tildes, config: RegressionConfig, use_chol: bool):
    if not _USE_GRAPHS[0] or not use_chol or any(t is not a for t, a in zip(tildes, facs)):
        return None
    try:
        key = (_state.thread_key(), torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream,
               tuple((a.data_ptr(), tuple(a.shape), tuple(a.stride())) for a in facs), config, _switches())
        hash(key)
    except TypeError:
        return None
    return key


def _prefix_graph_run(key, entry, gts, run, deferred):
    """First sight of a key: eager (warms every lazy initialisation).  Second: capture, then
    replay.  Afterwards: replay only."""
    from . import leverage as _lev
    if entry is None:
        _PREFIX_STATS["eager"] += 1
        _state.cache_put(_PREFIX_GRAPHS, key, _PrefixGraph(), _GRAPH_CAP)
        return run()
    if entry.graph is None:
        with GATE.capture() as ok:
            if not ok:
                return run()  # other solves in flight: eager this time
            _PREFIX_STATS["capture"] += 1
            entry.gts = gts
            g = torch.cuda.CUDAGraph()
            cap = _lev.DeferredChecks()
            outer = _lev._DEFERRED[0]
            _lev._DEFERRED[0] = cap
            try:
                with torch.cuda.graph(g, capture_error_mode=CAPTURE_MODE):
                    entry.out = run()
            except Exception:
                _state.cache_drop(_PREFIX_GRAPHS, key)
                raise
            finally:
                _lev._DEFERRED[0] = outer
        entry.graph = g
        entry.checks = cap.items
    _PREFIX_STATS["replay"] += 1
    entry.graph.replay()
    for flags, handler in entry.checks:
        deferred.add(flags, handler)
    return entry.out


# Phase marks for tools/profile_fast.py --phases and bench.py: (name, host time, CUDA event),
# collected per thread while enabled (``_PHASES[0] = []``; ``_PHASES[0] = None`` disables).
_PHASES = TLSlot()


def _mark(name: str):
    ph = _PHASES[0]
    if ph is not None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        ph.append((name, time.perf_counter(), ev))


def _fast_solve_pass(facs, b, config: RegressionConfig, caches, trace, use_chol: bool, deferred,
                     fast_scores: bool = True, sketch_only: bool = False):
    from . import leverage as _lev
    _mark("start")
    n_factors = len(facs)
    rows = [int(a.shape[0]) for a in facs]
    cols_l = [int(a.shape[1]) for a in facs]
    cols = math.prod(cols_l)
    lam = config.lam
    alpha = config.effective_alpha
    s = _regression_sample_count(cols, config)
    seeds = _spawned_seeds(config.seed, 2 * n_factors + 1)
    grams, scores, afs = [], [], []
    if caches is not None:
        for cache in caches:
            g = cache.gram
            grams.append((D.to_dev(g.v), D.to_dev(g.eigenvalues)))
            sv = cache.svd
            scores.append(D.to_dev(ridge_leverage_scores(CompactSvd(D.to_dev(sv.u), D.to_dev(sv.sigma),
                                                                    D.to_dev(sv.v)), 0.0).scores))
            afs.append(1.0)
    else:
        eps_one = math.log1p(config.eps / 4.0) / n_factors
        eps_two = eps_one / (2.0 + eps_one)
        delta_n = config.delta / (2.0 * n_factors)
        eps_jl = 4.0 * math.log1p(config.eps / 4.0) / n_factors
        tildes = []
        # per-factor spectral row sampling (leverage.py:235-252) is independent across factors:
        # factor n > 0 runs on its own stream (no host round trip inside; joined below)
        main = torch.cuda.current_stream()
        spectral = [math.ceil(alpha * spectral_sample_count(int(a.shape[1]), eps_two, delta_n)) < int(a.shape[0])
                    for a in facs]
        for n in range(1, n_factors):
            if spectral[n]:
                _side_stream(n).wait_stream(main)
        for n, a in enumerate(facs):
            if not spectral[n]:
                a_tilde = a
            else:
                with torch.cuda.stream(main if n == 0 else _side_stream(n)):
                    a_tilde = _spectral_rows_dev(a, eps_two, delta_n, seeds[2 * n], alpha, fast_scores,
                                                 divisor=math.sqrt(1.0 - eps_two))
                if n > 0:
                    a_tilde.record_stream(main)
            if trace is not None:
                trace.a_tilde_rows.append(int(a_tilde.shape[0]))
            tildes.append(a_tilde)
        for n in range(1, n_factors):
            if spectral[n]:
                main.wait_stream(_side_stream(n))
        key = _prefix_key(facs, tildes, config, use_chol) if trace is None else None
        entry = _state.cache_get(_PREFIX_GRAPHS, key) if key is not None else None
        gts = [_gram_dev(t, out=entry.gts[n] if entry is not None and entry.gts is not None else None)
               for n, t in enumerate(tildes)]
        # The preconditioner's eigendecompositions (solvers.py:440, 446) run on a side stream,
        # overlapped with the JL estimates, sampling and sketch construction; joined before the
        # Richardson loop.
        _mark("factor grams")
        grams = _factor_grams_async(gts)
        run = lambda: _jl_and_sampling(facs, tildes, gts, eps_jl, config, use_chol, seeds, s)  # noqa: E731
        if key is None:
            scores, afs, sampler, draws, w, g2 = run()
        else:
            scores, afs, sampler, draws, w, g2 = _prefix_graph_run(key, entry, gts, run, deferred)
        _mark("jl scores+sampling")
    if caches is not None:
        sampler = ProductSampler([LeverageScores(sc, 0.0, af) for sc, af in zip(scores, afs)])
        state, inc = pcg64_state(seeds[-1])
        draws = sampler._sample_dev(s, state, inc)
        w = sampler._weights_dev(draws, s)
        g2 = sketch_diag_grouped2_launch(facs, draws, w) if _USE_FUSED[0] and grouped2_eligible(facs) else None
    _mark("draws+weights")
    if g2 is not None:
        sdiag, _ = sketch_diag_grouped2_finish(facs, g2)
    else:
        sdiag = sparse_diagonal_from_sketch(RowSketch(draws, w), rows)
    _mark("sparse diagonal")
    if sketch_only:  # the replicated front half of a row-sharded solve (distributed.py)
        grams = _join_grams(grams)
        _lev._DEFERRED[0] = None
        deferred.run()
        return sdiag, grams, s
    idx = sdiag.indices
    if isinstance(b, torch.Tensor) and b.is_cuda:
        b_at = D.empty(sdiag.nnz)
        _lib.call("ks_gather", D.p(b), D.p(idx), sdiag.nnz, D.p(b_at), D.stream())
    else:
        # host-resident b: only the sampled entries cross PCIe (the solve never reads the rest)
        bh = b.reshape(-1) if isinstance(b, torch.Tensor) else np.asarray(b, dtype=np.float64).reshape(-1)
        ih = idx.cpu().numpy()
        b_at = D.to_dev(np.asarray(bh[ih], dtype=np.float64))
    _mark("gather b")
    view = _view_for(facs, sdiag)
    _mark("sketch view")
    left, right = view.part.left, view.part.right
    max_iters = config.effective_max_iters
    x = D.empty(view.dL, view.dR)
    hist = D.zeros(max(1, max_iters))
    rhs = D.empty(view.dL, view.dR)
    iters = ctypes.c_int32(0)
    hlen = ctypes.c_int32(0)
    lib = _lib.load()
    fused = (_USE_FUSED[0] and len(left) >= 1 and len(right) >= 1 and view.dL in (16, 32, 64)
             and view.dR in (16, 32, 64) and view.nnz > 0 and max_iters <= 1024)
    dg = VL = VR = None
    if fused:
        # right-hand side, preconditioner diagonal and the loop in one persistent launch; a group
        # of several factors (the Tucker core's right group) has the Kronecker products of their
        # eigenbases and eigenvalues, in the group's column order (as the preconditioner below)
        grams = _join_grams(grams)
        def group(idx):
            if len(idx) == 1:
                return grams[idx[0]]
            V = _kron_dev([grams[i][0] for i in idx])
            w = _kron_dev([grams[i][1].reshape(-1, 1) for i in idx]).reshape(-1)
            return V, w
        VL, wL = group(left)
        VR, wR = group(right)
        VL, wL, VR, wR = (t.contiguous() for t in (VL, wL, VR, wR))
        _mark("precond")
        deferred.stage()  # flag copies complete with the loop launch's own synchronisation
        _LAST_LOOP_EVENTS[0] = None
        rc = lib.ks_richardson_fused(ctypes.byref(view.struct), D.p(view.perm_arg()), D.p(b_at.contiguous()),
                                     D.p(VL), D.p(wL), D.p(VR), D.p(wR), None, float(lam),
                                     float(config.effective_damping), int(max_iters), float(config.residual_tol),
                                     D.p(x), D.p(hist), D.p(rhs), ctypes.byref(iters), ctypes.byref(hlen),
                                     D.stream())
        if trace is not None:
            dg = view.to_groups(pseudo_reciprocal(torch.kron(wL, wR) + lam)).contiguous()
    else:
        bv = (sdiag.values * b_at).contiguous()
        _lib.call("ks_sketched_transpose_apply", ctypes.byref(view.struct), D.p(bv), D.p(view.perm_arg()),
                  D.p(rhs), D.stream())
        _mark("rhs")
        # preconditioner in grouped (left | right) order
        grams = _join_grams(grams)
        eig = reduce(torch.kron, [w for _, w in grams])
        dinv = pseudo_reciprocal(eig + lam)
        VL = reduce(torch.kron, [grams[i][0] for i in left]) if left else torch.ones(1, 1, dtype=D.F64,
                                                                                     device=D.dev())
        VR = reduce(torch.kron, [grams[i][0] for i in right])
        VL = VL.contiguous()
        VR = VR.contiguous()
        dg = view.to_groups(dinv).contiguous()
        _mark("precond")
        deferred.stage()  # flag copies complete with the loop launch's own synchronisation
        rc = lib.ks_richardson_sketched(ctypes.byref(view.struct), D.p(VL), D.p(VR), D.p(dg), D.p(rhs),
                                        float(lam), float(config.effective_damping), int(max_iters),
                                        float(config.residual_tol), D.p(x), D.p(hist), ctypes.byref(iters),
                                        ctypes.byref(hlen), D.stream())
    _mark("richardson")
    _lev._DEFERRED[0] = None
    deferred.run(synced=True)  # generator / Cholesky / sampler-table flags, copied with the loop launch
    history = hist[: hlen.value].cpu().tolist()
    _LAST_HISTORY[0] = history
    if rc == _lib.KS_EDIVERGED:
        raise NumericalFailureError("Richardson iteration diverged", iterations=iters.value,
                                    diagnostics={"residual_history": history})
    _lib.check(rc, "ks_richardson_sketched")
    if trace is not None:
        trace.loop_inputs = dict(view=view, VL=VL, VR=VR, dinv=dg, rhs=rhs, lam=float(lam), b_at=b_at,
                                 wL=grams[left[0]][1] if len(left) == 1 else None,
                                 wR=grams[right[0]][1] if len(right) == 1 else None,
                                 damping=float(config.effective_damping), max_iters=int(max_iters),
                                 tol=float(config.residual_tol))
        trace.scores = scores
        trace.eig = [w for _, w in grams]
        trace.sampler = sampler
        trace.sketch = RowSketch(draws, w)
        trace.sdiag = sdiag
        trace.rhs = view.from_groups(rhs)
        trace.history = history
    return view.from_groups(x), iters.value, s


def fast_kronecker_regression(factors: Sequence, b, config: RegressionConfig,
                              caches: Sequence[FactorCache] | None = None, _trace: FastSolveTrace | None = None,
                              *, with_loss: bool = True) -> SolveReport:
    """(1+eps)-approximate Kronecker ridge regression (solvers.py:372-462), all on the GPU.

    ``wall_time`` covers the solve (as in the reference); the reported loss is evaluated
    exactly afterwards (``with_loss=False`` skips it: loss = nan; an extension for timing).  With host-resident ``b`` only its sampled entries are transferred
    for the solve; the loss pass then uploads it."""
    host = not D.on_device(b)
    if caches is None and _trace is None:
        got = (_fast_solve_host_graph if host else _fast_solve_dev_replay)(factors, b, config, with_loss)
        if got is not None:
            return got
    facs, rows, cols = _validated_problem(factors, b)
    if not 0.0 < config.eps <= 0.25:
        raise InvalidInputError(f"fast regression requires eps in (0, 1/4], got {config.eps}")
    if caches is not None and len(caches) != len(facs):
        raise InvalidInputError("need one cache entry per factor")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _mark("t0")
    s = _regression_sample_count(cols, config)
    if s >= rows:
        bt = D.to_dev(b).reshape(-1)
        x = _exact_solve_dev(facs, bt, config.lam)
        torch.cuda.synchronize()
        _mark("solve_end")
        wall = time.perf_counter() - t0
        loss = _ridge_loss_dev(facs, x, bt, config.lam) if with_loss else float("nan")
        return SolveReport(solution=D.out(x, host), loss=loss, iterations=0, sample_count=0, wall_time=wall)
    bsrc = b if D.on_device(b) else (b if isinstance(b, torch.Tensor) else np.asarray(b, dtype=np.float64))
    if D.on_device(bsrc):
        bsrc = bsrc.reshape(-1).to(torch.float64).contiguous()
    x, iters, s = _fast_solve_dev(facs, bsrc, config, caches, _trace)
    torch.cuda.synchronize()
    _mark("solve_end")
    wall = time.perf_counter() - t0
    if with_loss:
        bt = D.to_dev(b).reshape(-1)
        loss = _ridge_loss_dev(facs, x, bt, config.lam)
    else:
        loss = float("nan")
    return SolveReport(solution=D.out(x, host), loss=loss, iterations=iters, sample_count=s, wall_time=wall)


def _fast_solve_dev_replay(factors, b, config: RegressionConfig, with_loss: bool):
    """fast_kronecker_regression for device-resident inputs whose whole-solve graph is already
    captured: host-side shape checks only, then one replay (the factor validation is a graph node,
    its flags read back with the results), so no synchronising validation round trip precedes the
    solve.  None: not eligible / not captured yet (the regular path validates eagerly)."""
    if not 0.0 < config.eps <= 0.25 or len(factors) != 2:
        return None
    for a in factors:
        if not (isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == torch.float64 and a.ndim == 2
                and a.is_contiguous()):
            return None
    if not (isinstance(b, torch.Tensor) and b.is_cuda and b.dtype == torch.float64 and b.is_contiguous()):
        return None
    facs = list(factors)
    rows, cols = kron_operator_shape(facs)
    if int(b.numel()) != rows or _regression_sample_count(cols, config) >= rows:
        return None
    bsrc = b.reshape(-1)
    key = _solve_graph_key(facs, bsrc, config)
    entry = _state.cache_get(_SOLVE_GRAPHS, key) if key is not None else None
    if entry is None or entry.graph is None:
        return None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _mark("t0")
    got = _fast_solve_graph(facs, bsrc, config, key)
    if got is None:
        return None
    x, iters, s = got
    _mark("solve_end")
    wall = time.perf_counter() - t0
    loss = _ridge_loss_dev(facs, x, bsrc, config.lam) if with_loss else float("nan")
    return SolveReport(solution=x, loss=loss, iterations=iters, sample_count=s, wall_time=wall)


def _pinv_sym_dev(m: torch.Tensor) -> torch.Tensor:
    """np.linalg.pinv (rcond 1e-15) of a symmetric matrix on the device: the one-sided Jacobi SVD
    for n <= 128; above that the dense eigensolver of the CUDA math library (cuSOLVER syevd via
    torch.linalg.eigh) -- used only by the dense comparison baseline sketch_and_solve_ridge."""
    n = int(m.shape[0])
    if n <= 128:
        from .tensor import _pinv_dev
        return _pinv_dev(m.contiguous(), 1e-15)
    w, v = torch.linalg.eigh(0.5 * (m + m.T))
    a = w.abs()
    keep = a > 1e-15 * a.max()
    inv = torch.where(keep, 1.0 / torch.where(keep, w, torch.ones_like(w)), torch.zeros_like(w))
    return ((v * inv) @ v.T).contiguous()


def naive_normal_solve(factors: Sequence, b, lam: float,
                       max_dense_entries: int | None = DEFAULT_DENSE_GUARD) -> SolveReport:
    """Exact ridge solution of the normal equations (solvers.py:277-299).

    The reference densifies ``K^T K = kron(A_n^T A_n)`` and pseudo-inverts it.  Its pseudo-inverse
    (singular values above 1e-15 of the largest) is exactly ``(kron V_n) diag(pinv(kron w_n + lam))
    (kron V_n)^T`` from the factor Gram eigendecompositions, which is how it is applied here:
    O(sum d_n^3) instead of O(prod d_n^3), same result to rounding.  The size guard is kept."""
    host = not D.on_device(b)
    facs, rows, cols = _validated_problem(factors, b)
    if lam < 0:
        raise InvalidInputError(f"lambda must be >= 0, got {lam}")
    if max_dense_entries is not None and cols * cols > max_dense_entries:
        raise SizeGuardError(f"normal matrix would hold {cols}x{cols} entries (guard: {max_dense_entries})")
    bt = D.to_dev(b).reshape(-1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eig = [_factor_gram_dev(_gram_dev(a)) for a in facs]
    ktb = _kron_apply_dev([a.T.contiguous() for a in facs], bt[:, None].contiguous())
    w = reduce(torch.kron, [e[1] for e in eig]) + lam
    a = w.abs()
    keep = a > 1e-15 * a.max()
    dinv = torch.where(keep, 1.0 / torch.where(keep, w, torch.ones_like(w)), torch.zeros_like(w))
    t = _kron_apply_dev([e[0].T.contiguous() for e in eig], ktb) * dinv[:, None]
    x = _kron_apply_dev([e[0] for e in eig], t.contiguous())[:, 0].contiguous()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return SolveReport(solution=D.out(x, host), loss=_ridge_loss_dev(facs, x, bt, lam), iterations=0,
                       sample_count=0, wall_time=wall)


def sketch_and_solve_ridge(factors: Sequence, b, config: RegressionConfig, sketch=None,
                           max_dense_entries: int | None = DEFAULT_DENSE_GUARD) -> SolveReport:
    """Sketch-and-solve baseline (DJSSW19, solvers.py:334-369): draw rows from the exact
    leverage-score product distribution, materialise S K (ks_sketch_rows), solve
    ``((SK)^T SK + lam I)^+ (SK)^T S b``."""
    from .kron import sketch_rows_of_kron
    from .leverage import RowSketch, build_product_sampler, regression_sample_count, sample_rows
    host = not D.on_device(b)
    facs, rows, cols = _validated_problem(factors, b)
    bt = D.to_dev(b).reshape(-1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if sketch is None:
        sampler = build_product_sampler(exact_factor_scores(facs))
        s = max(1, math.ceil(config.effective_alpha * regression_sample_count(cols, config.eps)))
        sketch = sample_rows(sampler, s, config.seed)
    s = sketch.sample_count
    if max_dense_entries is not None and max(s * cols, cols * cols) > max_dense_entries:
        raise SizeGuardError(f"sketched matrix would hold {s}x{cols} entries (guard: {max_dense_entries})")
    idx = D.to_dev(sketch.indices, D.I64)
    sw = D.to_dev(sketch.weights).reshape(-1)
    sk = sketch_rows_of_kron(facs, RowSketch(indices=idx, weights=sw))
    if idx.ndim == 2:
        strides = torch.tensor([math.prod(int(a.shape[0]) for a in facs[n + 1:]) for n in range(len(facs))],
                               dtype=torch.int64, device=idx.device)
        flat = (idx * strides).sum(dim=1).contiguous()
    else:
        flat = idx.contiguous()
    bat = D.empty(s)
    _lib.call("ks_gather", D.p(bt), D.p(flat), s, D.p(bat), D.stream())
    sb = (sw * bat).contiguous()
    m = D.empty(cols, cols)
    _lib.call("ks_gemm", cols, cols, s, 1.0, D.p(sk), 1, cols, 0, D.p(sk), cols, 1, 0, 0.0, D.p(m), cols, 1, 0, 1,
              D.stream())
    m += config.lam * torch.eye(cols, dtype=D.F64, device=m.device)
    r = D.empty(cols, 1)
    _lib.call("ks_gemm", cols, 1, s, 1.0, D.p(sk), 1, cols, 0, D.p(sb), 1, 1, 0, 0.0, D.p(r), 1, 1, 0, 1, D.stream())
    p = _pinv_sym_dev(m)
    x = D.empty(cols, 1)
    _lib.call("ks_gemm", cols, 1, cols, 1.0, D.p(p), cols, 1, 0, D.p(r), 1, 1, 0, 0.0, D.p(x), 1, 1, 0, 1, D.stream())
    x = x[:, 0].contiguous()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return SolveReport(solution=D.out(x, host), loss=_ridge_loss_dev(facs, x, bt, config.lam), iterations=0,
                       sample_count=s, wall_time=wall)


# Public entry points are gated (capture vs. concurrent solves, see _state.py).
_state.gate_names(globals(), [
    "build_factor_cache",
    "build_kron_preconditioner",
    "exact_factor_scores",
    "factor_gram",
    "fast_kronecker_regression",
    "kronmatmul_svd_solve",
    "naive_normal_solve",
    "pseudo_reciprocal",
    "richardson_solve",
    "ridge_loss",
    "sketch_and_solve_ridge",
])
KronPreconditioner.apply = _state.gated(KronPreconditioner.apply)
