"""Leverage scores, row sketches and the Kronecker product sampler on the device.

Drop-in for pkg/src/kronsolve/leverage.py.  All arithmetic runs in CUDA kernels; the NumPy
random streams the reference draws on the host (``default_rng(seed).random`` /
``.standard_normal`` / ``.choice``) are regenerated bit-exactly on the GPU from the same
PCG64 state (csrc/ks_rng.cu), so sampled indices match the reference for the same seed."""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _device as D
from . import _lib
from . import _state
from ._numpy_rng import pcg64_state, split128, ziggurat_tables
from .errors import InvalidInputError, NumericalFailureError
from .tensor import CompactSvd, as_matrix, compact_svd

SPECTRAL_SAMPLE_CONSTANT = 144
REGRESSION_SAMPLE_CONSTANT = 1680
JL_LOG_FACTOR = 8.0


@dataclass(frozen=True)
class LeverageScores:
    """Per-row (ridge) leverage scores plus their approximation factor (leverage.py:32-48)."""

    scores: object
    lam: float
    approx_factor: float = 1.0

    def normalized(self):
        host = not D.on_device(self.scores)
        probs, _ = _tables(D.to_dev(self.scores).reshape(-1), renorm=False, want_cdf=False,
                           what="score vector")
        return D.out(probs, host)


def ridge_leverage_scores(svd: CompactSvd, lam: float) -> LeverageScores:
    """l_i = sum_k s_k^2/(s_k^2+lam) u_ik^2 (leverage.py:51-64)."""
    if lam < 0:
        raise InvalidInputError(f"lambda must be >= 0, got {lam}")
    host = not D.on_device(svd.u)
    u = D.to_dev(svd.u)
    n = int(u.shape[0])
    if svd.rank == 0:
        return LeverageScores(D.out(D.zeros(n), host), lam, 1.0)
    s = D.to_dev(svd.sigma)
    s2 = s * s
    wts = (s2 / (s2 + lam)).contiguous()
    scores = D.empty(n)
    _lib.call("ks_row_weighted_sumsq", D.p(u), n, int(u.shape[1]), D.p(wts), D.p(scores), D.stream())
    return LeverageScores(D.out(scores, host), lam, 1.0)


def statistical_leverage_scores(a) -> LeverageScores:
    return ridge_leverage_scores(compact_svd(a), 0.0)


def spectral_sample_count(d: int, eps: float, delta: float, beta: float = 1.0) -> int:
    """leverage.py:72-76."""
    return math.ceil(SPECTRAL_SAMPLE_CONSTANT * d * math.log(2 * d / delta) / (beta * eps ** 2))


def regression_sample_count(d: int, eps: float, beta: float = 1.0) -> int:
    """leverage.py:79-82."""
    return math.ceil(REGRESSION_SAMPLE_CONSTANT * d * math.log(40 * d) / (beta * eps))


_TABLES = {}


class DeferredChecks:
    """Device validation flags read in one host round trip at the end of a fast solve (instead
    of a stream synchronisation after every kernel that can fail).  Handlers run in order and
    raise the reference's exception for the first failure."""

    def __init__(self):
        self.items = []
        self._host = None

    def add(self, flags: torch.Tensor, handler):
        self.items.append((flags, handler))

    def stage(self):
        """Queue the device->host copies of every flag on the current stream (no wait); a later
        stream synchronisation (e.g. the Richardson launch's own) completes them."""
        self._host = [(f.to("cpu", non_blocking=True), h) for f, h in self.items]
        self.items = []

    def run(self, synced: bool = False):
        """Evaluate the handlers.  ``synced``: the stream was synchronised after stage()."""
        if self._host is None:
            self.stage()
            synced = False
        if not synced:
            torch.cuda.current_stream().synchronize()
        staged, self._host = self._host, None
        for f, handler in staged:
            handler(f.reshape(-1).tolist())


_DEFERRED = _state.TLSlot()  # this thread's enclosing fast solve's DeferredChecks (or None)


def check_later(flags: torch.Tensor, handler):
    """Run ``handler(flags as a list)`` now, or at the end of the enclosing fast solve."""
    d = _DEFERRED[0]
    if d is None:
        handler(flags.cpu().tolist())
    else:
        d.add(flags, handler)


def _zig_status(v):
    if v[0]:
        raise NumericalFailureError(f"device normal generator: ziggurat chain resolution failed (code {v[0]})")


def _zig_tables_dev():
    dev = D.dev()
    t = _TABLES.get(dev)
    if t is None:
        ki, wi, fi = ziggurat_tables()
        t = (torch.from_numpy(ki.view(np.int64)).to(dev), torch.from_numpy(wi).to(dev),
             torch.from_numpy(fi).to(dev))
        _TABLES[dev] = t
    return t


def device_standard_normal(seed, count: int, divisor: float = 1.0) -> torch.Tensor:
    """``default_rng(seed).standard_normal(count) / divisor`` generated on the GPU."""
    state, inc = pcg64_state(seed)
    sh, sl = split128(state)
    ih, il = split128(inc)
    ki, wi, fi = _zig_tables_dev()
    out = D.empty(count)
    if count:
        status = torch.zeros(1, dtype=torch.int32, device=D.dev())
        _lib.call("ks_pcg64_standard_normal", sh, sl, ih, il, count, float(divisor), D.p(ki), D.p(wi),
                  D.p(fi), D.p(out), D.p(status), D.stream())
        check_later(status, _zig_status)
    return out


def device_uniforms(state: int, inc: int, count: int, skip: int = 0) -> torch.Tensor:
    """``Generator.random(count)`` of a PCG64 stream (after ``skip`` draws) on the GPU."""
    sh, sl = split128(state)
    ih, il = split128(inc)
    out = D.empty(count)
    if count:
        _lib.call("ks_pcg64_random", sh, sl, ih, il, skip, count, D.p(out), D.stream())
    return out


def _inverse_small(m: torch.Tensor) -> torch.Tensor:
    d = int(m.shape[0])
    x = D.empty(d, d)
    info = torch.zeros(2, dtype=torch.int32, device=m.device)
    _lib.call("ks_inverse_small", D.p(m), d, D.p(x), D.p(info), D.stream())
    inf = info.cpu().tolist()
    if inf[0] != 0:
        raise NumericalFailureError("approximate Gram matrix is singular; cannot estimate leverage scores",
                                    diagnostics={"shape": tuple(m.shape)})
    if inf[1] != 0:
        raise NumericalFailureError("approximate Gram matrix is numerically singular",
                                    diagnostics={"shape": tuple(m.shape)})
    return x


def jl_projection_rows(n: int, log_factor: float = JL_LOG_FACTOR) -> int:
    """Gaussian projection height (leverage.py:125)."""
    return max(1, math.ceil(log_factor * math.log(max(n, 2))))


def _jl_ga(a: torch.Tensor, a_tilde: torch.Tensor, seed, log_factor: float, pre=None):
    """GA = g @ a_tilde with g = default_rng(seed).standard_normal((r, n_tilde)) / sqrt(r) drawn
    on the device (leverage.py:124-127).  Returns (GA (r x d), r).  ``pre``: (g, event) drawn
    earlier (the sketch depends only on the seed), waited for here."""
    n, d = int(a.shape[0]), int(a.shape[1])
    nt = int(a_tilde.shape[0])
    r = jl_projection_rows(n, log_factor)
    if pre is not None:
        g, ev = pre
        torch.cuda.current_stream().wait_event(ev)
    else:
        g = device_standard_normal(seed, r * nt, divisor=math.sqrt(r))
    ga = D.empty(r, d)
    if r <= 128 and d <= 128:
        _lib.call("ks_gemm_tn_tall", r, d, nt, 1.0, D.p(g), 1, nt, D.p(a_tilde), d, 1, D.p(ga), D.stream())
    else:
        _lib.call("ks_gemm", r, d, nt, 1.0, D.p(g), nt, 1, 0, D.p(a_tilde), d, 1, 0, 0.0, D.p(ga), d, 1, 0, 1,
                  D.stream())
    return ga, r


def _jl_scores_dev(a: torch.Tensor, a_tilde: torch.Tensor, gram_inv: torch.Tensor, eps: float, seed,
                   log_factor: float) -> torch.Tensor:
    d = int(a.shape[1])
    ga, r = _jl_ga(a, a_tilde, seed, log_factor)
    # Q = (1 + eps/4) GA gram^-1
    q = D.empty(r, d)
    _lib.call("ks_gemm", r, d, d, 1.0 + eps / 4.0, D.p(ga), d, 1, 0, D.p(gram_inv), d, 1, 0, 0.0, D.p(q), d, 1,
              0, 1, D.stream())
    return _jl_scores_from_q(a, q, r, eps)


def _jl_scores_from_q(a: torch.Tensor, q: torch.Tensor, r: int, eps: float) -> torch.Tensor:
    """scores_i = ||Q a_i||^2 / ((1+eps/4)(1-eps/20)) (leverage.py:127-129)."""
    n, d = int(a.shape[0]), int(a.shape[1])
    denom = (1.0 + eps / 4.0) * (1.0 - eps / 20.0)
    scores = D.empty(n)
    if r <= 256:
        _lib.call("ks_jl_scores", D.p(a), n, d, D.p(q), r, denom, D.p(scores), D.stream())
    else:
        proj = D.empty(n, r)
        _lib.call("ks_gemm", n, r, d, 1.0, D.p(a), d, 1, 0, D.p(q), 1, d, 0, 0.0, D.p(proj), r, 1, 0, 1,
                  D.stream())
        w = torch.full((r,), 1.0 / denom, dtype=D.F64, device=a.device)
        _lib.call("ks_row_weighted_sumsq", D.p(proj), n, r, D.p(w), D.p(scores), D.stream())
    return scores


def approx_leverage_scores_jl(a, a_tilde, gram_tilde, eps: float, seed,
                              log_factor: float = JL_LOG_FACTOR) -> LeverageScores:
    """JL estimate ||G a_tilde M a_i||^2 / ((1+eps/4)(1-eps/20)) (leverage.py:85-130)."""
    host = not D.on_device(a)
    at = as_matrix(a, "a")
    att = as_matrix(a_tilde, "a_tilde")
    gt = as_matrix(gram_tilde, "gram_tilde")
    if not 0.0 < eps <= 0.25:
        raise InvalidInputError(f"eps must be in (0, 1/4], got {eps}")
    gi = _inverse_small(gt)
    scores = _jl_scores_dev(at, att, gi, eps, seed, log_factor)
    return LeverageScores(D.out(scores, host), 0.0, 1.0 + eps / 2.0)


@dataclass(frozen=True)
class RowSketch:
    """``s`` i.i.d. draws (indices (s, N) or (s,)) with weights 1/sqrt(p s) (leverage.py:133-147)."""

    indices: object
    weights: object

    @property
    def sample_count(self) -> int:
        return int(self.weights.shape[0])


def _tables(scores: torch.Tensor, renorm: bool, want_cdf: bool = True, what: str = "score vector"):
    n = int(scores.numel())
    if n == 0:
        raise InvalidInputError(f"{what} must be a nonempty vector")
    probs = D.empty(n)
    cdf = D.empty(n) if want_cdf else None
    flags = torch.zeros(1, dtype=torch.int32, device=scores.device)
    _lib.call("ks_sampler_tables", D.p(scores), n, 1 if renorm else 0, D.p(probs), D.p(cdf), D.p(flags),
              D.stream())

    def handler(v):
        if v[0] & 1:
            raise InvalidInputError(f"{what} must be nonnegative finite")
        if v[0] & 2:
            raise InvalidInputError(f"{what} sums to zero")

    check_later(flags, handler)  # immediate outside a fast solve, deferred inside one
    return probs, cdf


class ProductSampler:
    """Row sampler for a Kronecker product, one categorical draw per factor (leverage.py:150-201).

    ``per_factor_probabilities`` / ``per_factor_cdf`` are device tensors built with NumPy's
    exact pairwise sum and sequential cumsum, so draws match the reference bit for bit."""

    def __init__(self, per_factor_scores: Sequence[LeverageScores]):
        if len(per_factor_scores) == 0:
            raise InvalidInputError("need at least one score vector")
        self._host = not D.on_device(per_factor_scores[0].scores)
        scs = []
        for n, ls in enumerate(per_factor_scores):
            sc = D.to_dev(ls.scores)
            if sc.ndim != 1 or sc.numel() == 0:
                raise InvalidInputError(f"score vector {n} must be a nonempty vector")
            scs.append(sc.contiguous())
        if len(scs) <= 8:
            # one launch for every factor's pairwise total / probabilities / exact cdf
            probs = [D.empty(int(sc.numel())) for sc in scs]
            cdfs = [D.empty(int(sc.numel())) for sc in scs]
            flags = torch.zeros(len(scs), dtype=torch.int32, device=D.dev())
            _lib.call("ks_sampler_tables_batched", len(scs),
                      _lib.ptr_array(ctypes.c_void_p, [s.data_ptr() for s in scs]),
                      _lib.ptr_array(ctypes.c_int64, [int(s.numel()) for s in scs]), 0,
                      _lib.ptr_array(ctypes.c_void_p, [p.data_ptr() for p in probs]),
                      _lib.ptr_array(ctypes.c_void_p, [c.data_ptr() for c in cdfs]), D.p(flags), D.stream())
            check_later(flags, self._check_flags)
        else:
            probs, cdfs = [], []
            for n, sc in enumerate(scs):
                p, c = _tables(sc, renorm=False, what=f"score vector {n}")
                probs.append(p)
                cdfs.append(c)
        self._probs = probs
        self._cdfs = cdfs
        self.beta = float(np.prod([1.0 / ls.approx_factor for ls in per_factor_scores]))

    @staticmethod
    def _check_flags(flags):
        """Raise the reference's InvalidInputError for invalid score vectors (leverage.py:163-171)."""
        for n, f in enumerate(flags):
            if f & 1:
                raise InvalidInputError(f"score vector {n} must be nonnegative finite")
            if f & 2:
                raise InvalidInputError(f"score vector {n} sums to zero")

    @property
    def per_factor_probabilities(self):
        return [D.out(p, self._host) for p in self._probs]

    @property
    def per_factor_cdf(self):
        return [D.out(c, self._host) for c in self._cdfs]

    @property
    def order(self) -> int:
        return len(self._probs)

    @property
    def row_shape(self) -> tuple[int, ...]:
        return tuple(int(p.numel()) for p in self._probs)

    def _probabilities_dev(self, idx: torch.Tensor, s: int) -> torch.Tensor:
        w = D.empty(s)
        pptr = _lib.ptr_array(ctypes.c_void_p, [p.data_ptr() for p in self._probs])
        # weights kernel computes 1/sqrt(prob*s); recover prob directly instead
        out = torch.ones(s, dtype=D.F64, device=idx.device)
        for n, p in enumerate(self._probs):
            out = out * p[idx[:, n]]
        del w, pptr
        return out

    def probabilities(self, indices):
        host = not D.on_device(indices)
        idx = D.to_dev(indices, D.I64)
        if idx.ndim == 1:
            idx = idx[None, :]
        return D.out(self._probabilities_dev(idx, int(idx.shape[0])), host)

    def _sample_dev(self, s: int, state: int, inc: int, skip: int = 0) -> torch.Tensor:
        draws = D.empty(s, self.order, dtype=D.I64)
        for n, cdf in enumerate(self._cdfs):
            u = device_uniforms(state, inc, s, skip + n * s)
            _lib.call("ks_searchsorted_right", D.p(cdf), int(cdf.numel()), D.p(u), s, D.p(draws), self.order, n,
                      D.stream())
        return draws

    def sample(self, s: int, rng: np.random.Generator):
        """Draw ``s`` multi-indices; consumes ``order * s`` draws of ``rng`` like the reference."""
        state, inc = pcg64_state(rng)
        draws = self._sample_dev(s, state, inc)
        rng.bit_generator.advance(self.order * s)
        return D.out(draws, self._host)

    def _weights_dev(self, draws: torch.Tensor, s: int) -> torch.Tensor:
        w = D.empty(s)
        pptr = _lib.ptr_array(ctypes.c_void_p, [p.data_ptr() for p in self._probs])
        _lib.call("ks_sketch_weights", self.order, pptr, D.p(draws), s, D.p(w), D.stream())
        return w


def build_product_sampler(per_factor_scores: Sequence[LeverageScores]) -> ProductSampler:
    return ProductSampler(per_factor_scores)


def sample_rows(sampler, s: int, seed) -> RowSketch:
    """``s`` i.i.d. draws with weights 1/sqrt(p_j s) (leverage.py:208-232)."""
    if s < 1:
        raise InvalidInputError(f"sample count must be >= 1, got {s}")
    state, inc = pcg64_state(seed)
    if isinstance(sampler, ProductSampler):
        draws = sampler._sample_dev(s, state, inc)
        w = sampler._weights_dev(draws, s)
        return RowSketch(indices=D.out(draws, sampler._host), weights=D.out(w, sampler._host))
    host = not D.on_device(sampler)
    pin = D.to_dev(sampler).reshape(-1)
    probs, cdf = _tables(pin, renorm=True, what="probability vector")
    u = device_uniforms(state, inc, s)
    idx = D.empty(s, dtype=D.I64)
    _lib.call("ks_searchsorted_right", D.p(cdf), int(cdf.numel()), D.p(u), s, D.p(idx), 1, 0, D.stream())
    w = D.empty(s)
    pptr = _lib.ptr_array(ctypes.c_void_p, [probs.data_ptr()])
    _lib.call("ks_sketch_weights", 1, pptr, D.p(idx), s, D.p(w), D.stream())
    return RowSketch(indices=D.out(idx, host), weights=D.out(w, host))


class ScoresFallback(Exception):
    """CholeskyQR2 declined (ill-conditioned factor): redo the solve with the compact-SVD scores."""


def _scores_status(v):
    if v[0] or v[1]:
        raise ScoresFallback()


def _statistical_scores_dev(a: torch.Tensor, fast: bool = True) -> torch.Tensor:
    """ridge_leverage_scores(compact_svd(a), 0).scores: for a tall, numerically full-rank a the
    squared row norms of a R^-1 (CholeskyQR2 R, one fused pass); otherwise the compact SVD.
    Inside a fast solve (deferred checks active) the CholeskyQR2 path is asynchronous and a
    declined factorisation raises ScoresFallback at the end of the solve (which is then redone with
    fast=False)."""
    n, d = int(a.shape[0]), int(a.shape[1])
    if fast and n >= 4 * d and d <= 128:
        sc = D.empty(n)
        if _DEFERRED[0] is not None:
            info = torch.zeros(2, dtype=torch.int32, device=a.device)
            _lib.call("ks_leverage_scores_tall_async", D.p(a.contiguous()), n, d, D.p(sc), D.p(info), D.stream())
            check_later(info, _scores_status)
            return sc
        ok = ctypes.c_int32(0)
        _lib.call("ks_leverage_scores_tall", D.p(a.contiguous()), n, d, D.p(sc), ctypes.byref(ok), D.stream())
        if ok.value:
            return sc
    return ridge_leverage_scores(compact_svd(a), 0.0).scores


def _spectral_rows_dev(a: torch.Tensor, eps: float, delta: float, seed, alpha: float,
                       fast_scores: bool = True, divisor: float = 1.0) -> torch.Tensor:
    """w[:, None] * a[idx, :] of leverage.py:249-252 (divided by ``divisor`` afterwards, as the
    caller solvers.py:424-427 does), in one gather kernel."""
    from .solvers import _TL_CUR, _tl_event
    tl = _TL_CUR[0]
    sc = _statistical_scores_dev(a, fast_scores)
    _tl_event(tl, f"spectral scores ({int(a.shape[0])})")
    p1, _ = _tables(D.to_dev(sc), renorm=False, want_cdf=False, what="score vector")
    _tl_event(tl, "spectral tables")
    s = max(1, math.ceil(alpha * spectral_sample_count(int(a.shape[1]), eps, delta)))
    sk = sample_rows(p1, s, seed)
    _tl_event(tl, "spectral draws")
    idx = D.to_dev(sk.indices, D.I64)
    w = D.to_dev(sk.weights)
    a = a.contiguous()
    out = D.empty(int(idx.shape[0]), int(a.shape[1]))
    _lib.call("ks_scaled_row_gather", D.p(a), int(a.shape[0]), int(a.shape[1]), D.p(idx), D.p(w),
              int(idx.shape[0]), float(divisor), D.p(out), D.stream())
    return out


def spectral_approx_rows(a, eps: float, delta: float, seed, alpha: float = 1.0):
    """Leverage-sampled spectral approximation ``S a`` (leverage.py:235-252)."""
    host = not D.on_device(a)
    at = as_matrix(a)
    if not 0.0 < eps < 1.0:
        raise InvalidInputError(f"eps must be in (0, 1), got {eps}")
    if not 0.0 < delta < 1.0:
        raise InvalidInputError(f"delta must be in (0, 1), got {delta}")
    return D.out(_spectral_rows_dev(at, eps, delta, seed, alpha), host)


# Public entry points are gated (capture vs. concurrent solves, see _state.py).
_state.gate_names(globals(), [
    "approx_leverage_scores_jl",
    "build_product_sampler",
    "ridge_leverage_scores",
    "sample_rows",
    "spectral_approx_rows",
    "statistical_leverage_scores",
])
ProductSampler.sample = _state.gated(ProductSampler.sample)
ProductSampler.probabilities = _state.gated(ProductSampler.probabilities)
