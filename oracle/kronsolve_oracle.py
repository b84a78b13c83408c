"""CPU oracle for the FastKroneckerRegression hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference package ``kronsolve``
(arXiv 2209.04876, mounted read-only at /root/reference/pkg/src/kronsolve) for
the functions on the north-star path.  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import it.  The product package
``paper_2209_04876_b200`` never imports or calls anything in ``oracle/``.

Parity pinning: ``tests/test_oracle.py`` checks the functions here against the
real reference (when /root/reference is present, i.e. in the build container)
and against the committed fixtures in ``tests/golden/`` that were produced by
running the reference itself (``tests/golden/make_golden.py`` for c1-c3/c5,
``tests/golden/make_golden_c4.py`` for c4); ``tests/test_rng_oracle.py`` pins
the PCG64 / ziggurat restatement in ``rng_oracle.py`` against NumPy.

Each function cites the reference file:line it restates.  The floating-point
operation order follows the reference (same NumPy calls in the same order) so
that oracle and reference agree bit-for-bit where NumPy is deterministic.

Third-party arithmetic on this path lives in NumPy 2.3.5 / OpenBLAS 0.3.30
(the only dependency, ``pkg/pyproject.toml:10``): PCG64 + ziggurat random
streams, pairwise summation, LAPACK gesdd/syevd/gesv.  The oracle calls the
same NumPy entry points the reference calls.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass
from functools import reduce

import numpy as np

# constants: leverage.py:24-29, kron.py:26-28, solvers.py:53-58, tensor.py:281
SPECTRAL_C = 144
REGRESSION_C = 1680
JL_LOG_FACTOR = 8.0
SPARSE_FALLBACK_FRACTION = 0.5
RANK_TOL = 1e-10
DIVERGENCE_WINDOW = 5
DIVERGENCE_GROWTH = 10.0


class OracleError(Exception):
    """Raised where the reference raises (InvalidInput / SizeGuard / NumericalFailure)."""

    def __init__(self, kind, message, iterations=None, history=None):
        super().__init__(message)
        self.kind = kind
        self.iterations = iterations
        self.history = history


# ---------------------------------------------------------------------------
# Kronecker multiplies (kron.py)
# ---------------------------------------------------------------------------

def kron_mat_mul(factors, b):
    """(A1 (x) ... (x) AN) b, rightmost factor first -- kron.py:44-77."""
    mats = [np.asarray(a, dtype=np.float64) for a in factors]
    b = np.asarray(b, dtype=np.float64)
    vec = b.ndim == 1
    cur = b[:, None] if vec else b
    if cur.shape[0] != math.prod(a.shape[1] for a in mats):
        raise OracleError("invalid", "b does not match the operator columns")
    cur = _peel(mats, cur)
    return cur[:, 0] if vec else cur


def _peel(mats, cur):
    # kron.py:66-77: tensordot over the rightmost factor's column index, then
    # move the new row index next to the block index and recurse.
    if len(mats) == 1:
        return mats[0] @ cur
    last = mats[-1]
    rows_last, cols_last = last.shape
    blocks = cur.shape[0] // cols_last
    width = cur.shape[1]
    z = np.tensordot(cur.reshape(blocks, cols_last, width), last, axes=([1], [1]))
    z = z.transpose(0, 2, 1).reshape(blocks, rows_last * width)
    out = _peel(mats[:-1], z)
    return out.reshape(out.shape[0] * rows_last, width)


def kron_vec_square(factors, c):
    """Square-factor Kronecker times vector by cyclic reshapes -- kron.py:80-100."""
    v = np.asarray(c, dtype=np.float64).reshape(-1)
    for a in factors[::-1]:
        a = np.asarray(a, dtype=np.float64)
        v = np.ascontiguousarray((v.reshape(-1, a.shape[0]) @ a.T).T).reshape(-1)
    return v


def balanced_partition(col_dims):
    """Exhaustive min-max split of factor positions -- kron.py:117-144.

    Returns (left, right, left_product, right_product)."""
    dims = [int(x) for x in col_dims]
    total = math.prod(dims)
    best = None
    for k in range(len(dims) + 1):
        for subset in itertools.combinations(range(len(dims)), k):
            lp = math.prod(dims[i] for i in subset)
            key = (max(lp, total // lp), lp, subset)
            if best is None or key < best:
                best = key
    _, lp, left = best
    right = tuple(i for i in range(len(dims)) if i not in left)
    return left, right, lp, total // lp


def sparse_diagonal_from_sketch(indices, weights, row_shape):
    """sqrt(S^T S) on the sampled rows -- kron.py:173-190.

    Returns (sorted unique flat indices, values)."""
    idx = np.asarray(indices)
    flat = np.ravel_multi_index(tuple(idx.T), tuple(row_shape)) if idx.ndim == 2 else idx
    perm = np.argsort(flat, kind="stable")
    flat_sorted = flat[perm]
    sq = np.asarray(weights)[perm] ** 2
    uniq, first = np.unique(flat_sorted, return_index=True)
    return uniq.astype(np.int64), np.sqrt(np.add.reduceat(sq, first))


def _rows_of(factors, multi):
    # kron.py:193-205 (kron_rows): row-wise Kronecker of the selected rows
    multi = np.atleast_2d(np.asarray(multi, dtype=np.intp))
    acc = np.ones((multi.shape[0], 1))
    for n, a in enumerate(factors):
        sel = a[multi[:, n], :]
        acc = (acc[:, :, None] * sel[:, None, :]).reshape(multi.shape[0], -1)
    return acc


def _groups(flat, row_shape, left, right):
    # kron.py:225-240 (_split_indices)
    multi = np.stack(np.unravel_index(flat, row_shape), axis=1)

    def one(pos):
        if not pos:
            return np.zeros(multi.shape[0], dtype=np.int64), np.zeros((multi.shape[0], 0), dtype=np.intp)
        sub = multi[:, list(pos)]
        return np.ravel_multi_index(tuple(sub.T), tuple(row_shape[i] for i in pos)), sub

    return one(left) + one(right)


def _first_multi(multi, flat, uniq):
    # kron.py:303-309 (_first_occurrences)
    perm = np.argsort(flat, kind="stable")
    return multi[perm[np.searchsorted(flat[perm], uniq)]]


def sketched_kron_apply(factors, sd_indices, sd_values, c):
    """Entries of S K c on the sketched rows -- kron.py:258-300."""
    mats = [np.asarray(a, dtype=np.float64) for a in factors]
    rows = math.prod(a.shape[0] for a in mats)
    col_shape = tuple(a.shape[1] for a in mats)
    row_shape = tuple(a.shape[0] for a in mats)
    c = np.asarray(c, dtype=np.float64).reshape(-1)
    if sd_indices.size == 0:
        return np.zeros(0)
    if sd_indices.size > rows * SPARSE_FALLBACK_FRACTION:
        return sd_values * kron_mat_mul(mats, c)[sd_indices]
    left, right, lp, _ = balanced_partition(col_shape)
    li, mleft, ri, mright = _groups(sd_indices, row_shape, left, right)
    order = left + right
    cmat = c.reshape(col_shape).transpose(order).reshape(-1).reshape(lp, -1).T
    uri, rpos = np.unique(ri, return_inverse=True)
    y = _rows_of([mats[i] for i in right], _first_multi(mright, ri, uri)) @ cmat
    uli, lpos = np.unique(li, return_inverse=True)
    lrows = _rows_of([mats[i] for i in left], _first_multi(mleft, li, uli))
    return sd_values * np.einsum("tj,tj->t", y[rpos], lrows[lpos])


def sketched_kron_transpose_apply(factors, sd_indices, sd_values, b_values):
    """K^T S b from the entries of b on the sketched rows -- kron.py:312-354."""
    mats = [np.asarray(a, dtype=np.float64) for a in factors]
    rows = math.prod(a.shape[0] for a in mats)
    col_shape = tuple(a.shape[1] for a in mats)
    row_shape = tuple(a.shape[0] for a in mats)
    b_values = np.asarray(b_values, dtype=np.float64).reshape(-1)
    if sd_indices.size == 0:
        return np.zeros(math.prod(col_shape))
    if sd_indices.size > rows * SPARSE_FALLBACK_FRACTION:
        dense = np.zeros(rows)
        dense[sd_indices] = sd_values * b_values
        return kron_mat_mul([a.T for a in mats], dense)
    left, right, _, rp = balanced_partition(col_shape)
    li, mleft, ri, mright = _groups(sd_indices, row_shape, left, right)
    scaled = sd_values * b_values
    rrows = _rows_of([mats[i] for i in right], mright)
    uli, lpos = np.unique(li, return_inverse=True)
    lrows = _rows_of([mats[i] for i in left], _first_multi(mleft, li, uli))
    acc = np.zeros((uli.size, rp))
    np.add.at(acc, lpos, scaled[:, None] * rrows)
    grouped = (acc.T @ lrows).T.reshape(-1)
    order = left + right
    inv = np.argsort(np.asarray(order))
    return grouped.reshape(tuple(col_shape[i] for i in order)).transpose(tuple(inv)).reshape(-1)


# ---------------------------------------------------------------------------
# SVD, leverage scores, sampling (tensor.py, leverage.py)
# ---------------------------------------------------------------------------

@dataclass
class Svd:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray


def compact_svd(a, rank_tol=RANK_TOL):
    """Truncated thin SVD -- tensor.py:76-107."""
    a = np.asarray(a, dtype=np.float64)
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    r = 0 if (s.size == 0 or s[0] <= 0.0) else int(np.count_nonzero(s > rank_tol * s[0]))
    return Svd(u[:, :r].copy(), s[:r].copy(), vt[:r].T.copy())


def ridge_scores(svd, lam):
    """l_i = sum_k s_k^2/(s_k^2+lam) u_ik^2 -- leverage.py:51-64."""
    if svd.sigma.size == 0:
        return np.zeros(svd.u.shape[0])
    s2 = svd.sigma ** 2
    return (svd.u ** 2) @ (s2 / (s2 + lam))


def spectral_sample_count(d, eps, delta, beta=1.0):
    """leverage.py:72-76."""
    return math.ceil(SPECTRAL_C * d * math.log(2 * d / delta) / (beta * eps ** 2))


def regression_sample_count(d, eps, beta=1.0):
    """leverage.py:79-82."""
    return math.ceil(REGRESSION_C * d * math.log(40 * d) / (beta * eps))


def jl_rows(n, log_factor=JL_LOG_FACTOR):
    """Gaussian projection height -- leverage.py:125."""
    return max(1, math.ceil(log_factor * math.log(max(n, 2))))


def jl_scores(a, a_tilde, gram_tilde, eps, seed, log_factor=JL_LOG_FACTOR):
    """JL leverage-score estimates -- leverage.py:85-130.  Returns (scores, approx_factor)."""
    a = np.asarray(a, dtype=np.float64)
    a_tilde = np.asarray(a_tilde, dtype=np.float64)
    gram_tilde = np.asarray(gram_tilde, dtype=np.float64)
    if not 0.0 < eps <= 0.25:
        raise OracleError("invalid", "eps out of (0, 1/4]")
    try:
        pm = (1.0 + eps / 4.0) * np.linalg.solve(gram_tilde, a.T)
    except np.linalg.LinAlgError as exc:
        raise OracleError("numerical", "singular approximate Gram") from exc
    if not np.all(np.isfinite(pm)):
        raise OracleError("numerical", "numerically singular approximate Gram")
    gen = np.random.default_rng(seed)
    r = jl_rows(a.shape[0], log_factor)
    g = gen.standard_normal((r, a_tilde.shape[0])) / math.sqrt(r)
    proj = (g @ a_tilde) @ pm
    scores = np.einsum("ri,ri->i", proj, proj)
    scores /= (1.0 + eps / 4.0) * (1.0 - eps / 20.0)
    return scores, 1.0 + eps / 2.0


class Sampler:
    """Product-distribution row sampler -- leverage.py:150-201."""

    def __init__(self, score_list, approx_factors=None):
        self.probs = []
        for sc in score_list:
            sc = np.asarray(sc, dtype=np.float64)
            if sc.ndim != 1 or sc.size == 0 or np.any(sc < 0) or not np.all(np.isfinite(sc)):
                raise OracleError("invalid", "bad score vector")
            tot = sc.sum()
            if tot <= 0.0:
                raise OracleError("invalid", "score vector sums to zero")
            self.probs.append(sc / tot)
        self.cdfs = [np.cumsum(p) for p in self.probs]
        af = approx_factors or [1.0] * len(score_list)
        self.beta = float(np.prod([1.0 / f for f in af]))

    @property
    def row_shape(self):
        return tuple(p.size for p in self.probs)

    def joint(self, idx):
        idx = np.atleast_2d(np.asarray(idx, dtype=np.intp))
        out = np.ones(idx.shape[0])
        for n, p in enumerate(self.probs):
            out *= p[idx[:, n]]
        return out

    def draw(self, s, gen):
        out = np.empty((s, len(self.cdfs)), dtype=np.intp)
        for n, cdf in enumerate(self.cdfs):
            u = gen.random(s)
            out[:, n] = np.searchsorted(cdf, u, side="right")
            np.clip(out[:, n], 0, cdf.size - 1, out=out[:, n])
        return out


def sample_rows(sampler, s, seed):
    """Draws + weights 1/sqrt(p s) -- leverage.py:208-232."""
    if s < 1:
        raise OracleError("invalid", "sample count must be >= 1")
    gen = np.random.default_rng(seed)
    if isinstance(sampler, Sampler):
        idx = sampler.draw(s, gen)
        pr = sampler.joint(idx)
    else:
        p = np.asarray(sampler, dtype=np.float64).reshape(-1)
        if np.any(p < 0) or not np.all(np.isfinite(p)):
            raise OracleError("invalid", "probabilities must be nonnegative finite")
        tot = p.sum()
        if tot <= 0.0:
            raise OracleError("invalid", "probability vector sums to zero")
        p = p / tot
        idx = gen.choice(p.size, size=s, replace=True, p=p)
        pr = p[idx]
    return idx, 1.0 / np.sqrt(pr * s)


def spectral_approx_rows(a, eps, delta, seed, alpha=1.0):
    """Leverage-sampled spectral approximation S a -- leverage.py:235-252."""
    a = np.asarray(a, dtype=np.float64)
    sc = ridge_scores(compact_svd(a), 0.0)
    tot = float(sc.sum())
    if tot <= 0.0:
        raise OracleError("invalid", "all-zero scores")
    s = max(1, math.ceil(alpha * spectral_sample_count(a.shape[1], eps, delta)))
    idx, w = sample_rows(sc / tot, s, seed)
    return w[:, None] * a[idx, :]


# ---------------------------------------------------------------------------
# Solvers (solvers.py)
# ---------------------------------------------------------------------------

def factor_gram(a, assume_gram=False):
    """Descending clipped eigendecomposition of A^T A -- solvers.py:143-150.

    Returns (v, eigenvalues, symmetrised matrix)."""
    a = np.asarray(a, dtype=np.float64)
    g = a if assume_gram else a.T @ a
    g = 0.5 * (g + g.T)
    w, v = np.linalg.eigh(g)
    return np.ascontiguousarray(v[:, ::-1]), np.clip(w[::-1], 0.0, None), g


def pseudo_reciprocal(d):
    """solvers.py:186-191."""
    out = np.zeros_like(d)
    nz = d > 0
    out[nz] = 1.0 / d[nz]
    return out


class Preconditioner:
    """(V (x) ...) D (V (x) ...)^T -- solvers.py:166-198."""

    def __init__(self, grams, lam):
        self.vs = [g[0] for g in grams]
        self.d = pseudo_reciprocal(reduce(np.kron, [g[1] for g in grams]) + lam)

    def apply(self, x):
        t = kron_vec_square([v.T for v in self.vs], x) * self.d
        return kron_vec_square(self.vs, t)


def effective_max_iters(eps, max_iters=None):
    """solvers.py:105-109."""
    return max_iters if max_iters is not None else 8 * max(1, math.ceil(math.log(1.0 / eps)))


def richardson(apply_normal, apply_precond, rhs, damping, max_iters, residual_tol=1e-9, x0=None,
               callback=None):
    """Damped preconditioned Richardson -- solvers.py:201-248.

    Returns (x, iterations, history)."""
    rhs = np.asarray(rhs, dtype=np.float64).reshape(-1)
    x = np.zeros_like(rhs) if x0 is None else np.array(x0, dtype=np.float64)
    scale = float(np.linalg.norm(apply_precond(rhs)))
    tol = residual_tol * max(scale, np.finfo(float).tiny)
    hist = []
    done = 0
    for _ in range(max_iters):
        step = apply_precond(apply_normal(x) - rhs)
        nrm = float(np.linalg.norm(step))
        hist.append(nrm)
        if nrm <= tol:
            break
        if len(hist) > DIVERGENCE_WINDOW:
            win = hist[-(DIVERGENCE_WINDOW + 1):]
            if all(win[i + 1] > win[i] for i in range(DIVERGENCE_WINDOW)) and \
                    win[-1] > DIVERGENCE_GROWTH * win[0]:
                raise OracleError("numerical", "Richardson iteration diverged", done, hist)
        x = x - damping * step
        done += 1
        if callback is not None:
            callback(x)
    return x, done, hist


def ridge_loss(factors, x, b, lam):
    """||K x - b||^2 + lam ||x||^2 -- solvers.py:251-262."""
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    r = kron_mat_mul(factors, x) - b
    return float(r @ r + lam * (x @ x))


@dataclass
class Report:
    solution: np.ndarray
    loss: float
    iterations: int
    sample_count: int
    wall_time: float
    trace: dict


def kronmatmul_svd_solve(factors, b, lam, with_loss=True):
    """Exact SVD-composed ridge solve -- solvers.py:302-320."""
    import time
    mats = [np.asarray(a, dtype=np.float64) for a in factors]
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    t0 = time.perf_counter()
    svds = [compact_svd(a) for a in mats]
    t = kron_mat_mul([s.u.T for s in svds], b)
    sig = reduce(np.kron, [s.sigma for s in svds])
    t = t * (sig / (sig ** 2 + lam))
    x = kron_mat_mul([s.v for s in svds], t)
    wall = time.perf_counter() - t0
    loss = ridge_loss(mats, x, b, lam) if with_loss else float("nan")
    return Report(x, loss, 0, 0, wall, {})


def sample_count(cols, eps, delta, alpha):
    """solvers.py:405-407."""
    return max(1, math.ceil(alpha * REGRESSION_C * cols * math.log(40 * cols) * math.log(1.0 / delta) / eps))


def fast_kronecker_regression(factors, b, eps=0.25, delta=0.05, lam=0.0, alpha=1.0, seed=0,
                              max_iters=None, residual_tol=1e-9, damping=None,
                              jl_log_factor=JL_LOG_FACTOR, caches=None, with_loss=True, b_at=None):
    """Algorithm 1 -- solvers.py:372-462.

    ``caches`` is a list of (svd, (v, eigenvalues, gram)) tuples (FactorCache).
    ``b_at``: optional callable idx -> b[idx] replacing the read of b at the sparse-diagonal
    rows (solvers.py:448), for right-hand sides too large to hold (BASELINE c4: 34 GB); then
    ``b`` may be None and ``with_loss`` must be False.
    ``trace`` holds every intermediate the GPU path is compared on."""
    import time
    mats = [np.asarray(a, dtype=np.float64) for a in factors]
    if b_at is None:
        b = np.asarray(b, dtype=np.float64).reshape(-1)
        b_at = b.__getitem__
    elif with_loss:
        raise OracleError("invalid", "b_at needs with_loss=False")
    nf = len(mats)
    rows = math.prod(a.shape[0] for a in mats)
    cols = math.prod(a.shape[1] for a in mats)
    for a in mats:
        if not np.any(a):
            raise OracleError("invalid", "factor identically zero")
    if not 0.0 < eps <= 0.25:
        raise OracleError("invalid", "fast regression requires eps in (0, 1/4]")
    t0 = time.perf_counter()
    s = sample_count(cols, eps, delta, alpha)
    if s >= rows:
        ex = kronmatmul_svd_solve(mats, b, lam, with_loss=with_loss)
        return Report(ex.solution, ex.loss, 0, 0, time.perf_counter() - t0, {"exact": True})
    seeds = np.random.SeedSequence(seed).spawn(2 * nf + 1)
    trace = {"s": s, "scores": [], "eig": [], "v": [], "a_tilde_rows": []}
    grams, score_list, afs = [], [], []
    if caches is not None:
        for sv, gr in caches:
            grams.append(gr)
            score_list.append(ridge_scores(sv, 0.0))
            afs.append(1.0)
    else:
        eps_one = math.log1p(eps / 4.0) / nf
        eps_two = eps_one / (2.0 + eps_one)
        delta_n = delta / (2.0 * nf)
        eps_jl = 4.0 * math.log1p(eps / 4.0) / nf
        for n, a in enumerate(mats):
            s_n = math.ceil(alpha * spectral_sample_count(a.shape[1], eps_two, delta_n))
            if s_n >= a.shape[0]:
                at = a
            else:
                at = spectral_approx_rows(a, eps_two, delta_n, seeds[2 * n], alpha=alpha) / math.sqrt(1.0 - eps_two)
            trace["a_tilde_rows"].append(at.shape[0])
            gt = at.T @ at
            grams.append(factor_gram(gt, assume_gram=True))
            sc, af = jl_scores(a, at, gt, eps_jl, seeds[2 * n + 1], jl_log_factor)
            score_list.append(sc)
            afs.append(af)
    for g, sc in zip(grams, score_list):
        trace["eig"].append(g[1])
        trace["v"].append(g[0])
        trace["scores"].append(sc)
    sampler = Sampler(score_list, afs)
    pre = Preconditioner(grams, lam)
    idx, w = sample_rows(sampler, s, seeds[-1])
    row_shape = tuple(a.shape[0] for a in mats)
    sd_idx, sd_val = sparse_diagonal_from_sketch(idx, w, row_shape)
    rhs = sketched_kron_transpose_apply(mats, sd_idx, sd_val, sd_val * np.asarray(b_at(sd_idx), dtype=np.float64))

    def normal(x):
        return sketched_kron_transpose_apply(mats, sd_idx, sd_val,
                                             sketched_kron_apply(mats, sd_idx, sd_val, x)) + lam * x

    damp = (1.0 - math.sqrt(eps)) if damping is None else damping
    x, iters, hist = richardson(normal, pre.apply, rhs, damp, effective_max_iters(eps, max_iters),
                                residual_tol)
    wall = time.perf_counter() - t0
    trace.update(probs=sampler.probs, cdfs=sampler.cdfs, beta=sampler.beta, indices=idx, weights=w,
                 sd_indices=sd_idx, sd_values=sd_val, rhs=rhs, history=hist, d_diag=pre.d)
    loss = ridge_loss(mats, x, b, lam) if with_loss else float("nan")
    return Report(x, loss, iters, s, wall, trace)


# ---------------------------------------------------------------------------
# Tucker core update (tucker.py:108-127) and the data generators
# ---------------------------------------------------------------------------

def core_update_exact(factors, x_tensor, lam):
    """tucker.py:119-120: exact core solve of the Kronecker regression."""
    rep = kronmatmul_svd_solve(factors, np.asarray(x_tensor, dtype=np.float64).reshape(-1), lam,
                               with_loss=False)
    return rep.solution.reshape(tuple(a.shape[1] for a in factors))


def core_update_fast(factors, x_tensor, lam, caches, **cfg):
    """tucker.py:121-124: fast core solve with cached per-factor SVD + Gram."""
    rep = fast_kronecker_regression(factors, np.asarray(x_tensor, dtype=np.float64).reshape(-1),
                                    lam=lam, caches=caches, with_loss=False, **cfg)
    return rep.solution.reshape(tuple(a.shape[1] for a in factors)), rep


def factor_cache(a):
    """solvers.py:161-163: (compact_svd(a), factor_gram(a))."""
    return compact_svd(a), factor_gram(a)


def synth_regression(n, d, order=2, seed=0):
    """experiments.py:106-115: N(1, var 1e-3) factors, all-ones target."""
    gen = np.random.default_rng(seed)
    facs = [gen.normal(1.0, math.sqrt(0.001), (n, d)) for _ in range(order)]
    return facs, np.ones(n ** order)


def synth_tucker(shape, rank, noise_std, seed=0, relative=False):
    """experiments.py:118-131 consumption order.  Absolute noise N(0, noise_std^2) by default
    (BASELINE.json config 5); ``relative=True`` is generate_synth_tucker's own scaling,
    noise * ||x|| / sqrt(x.size) (experiments.py:128-130)."""
    gen = np.random.default_rng(seed)
    core = gen.standard_normal(tuple(rank))
    facs = []
    for i_n, r_n in zip(shape, rank):
        q, _ = np.linalg.qr(gen.standard_normal((i_n, r_n)))
        facs.append(q)
    x = core
    for mode, a in enumerate(facs):
        x = np.moveaxis(np.tensordot(a, x, axes=(1, mode)), 0, mode)
    if noise_std > 0:
        scale = noise_std * float(np.linalg.norm(x)) / math.sqrt(x.size) if relative else noise_std
        x = x + gen.standard_normal(x.shape) * scale
    return x


def initial_tucker_factors(shape, core_shape, seed):
    """tucker.py:400-409: orthonormal Q factors of N(0,1) matrices."""
    gen = np.random.default_rng(seed)
    out = []
    for i_n, r_n in zip(shape, core_shape):
        q, _ = np.linalg.qr(gen.standard_normal((i_n, r_n)))
        out.append(q)
    return out


# ---------------------------------------------------------------------------
# Dense comparison baselines (solvers.py:277-299, :334-369) -- SURVEY.md 8(f) row 3
# ---------------------------------------------------------------------------

def naive_normal_solve(factors, b, lam):
    """Densified normal equations: pinv(kron(A^T A) + lam I) K^T b -- solvers.py:277-299."""
    mats = [np.asarray(a, dtype=np.float64) for a in factors]
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    cols = math.prod(a.shape[1] for a in mats)
    gram = reduce(np.kron, [a.T @ a for a in mats])
    ktb = kron_mat_mul([a.T for a in mats], b)
    x = np.linalg.pinv(gram + lam * np.eye(cols)) @ ktb
    return Report(x, ridge_loss(mats, x, b, lam), 0, 0, 0.0, {})


def sketch_and_solve_ridge(factors, b, eps=0.25, lam=0.0, alpha=1.0, seed=0, sketch=None):
    """Sketch-and-solve with exact leverage-score product sampling -- solvers.py:334-369.

    ``sketch`` = (indices, weights) overrides the draw."""
    mats = [np.asarray(a, dtype=np.float64) for a in factors]
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    cols = math.prod(a.shape[1] for a in mats)
    if sketch is None:
        sampler = Sampler([ridge_scores(compact_svd(a), 0.0) for a in mats])
        s = max(1, math.ceil(alpha * regression_sample_count(cols, eps)))
        idx, w = sample_rows(sampler, s, seed)
    else:
        idx, w = sketch
    s = w.size
    idx = np.asarray(idx)
    multi = idx if idx.ndim == 2 else np.stack(np.unravel_index(idx, tuple(a.shape[0] for a in mats)), axis=1)
    sk = w[:, None] * _rows_of(mats, multi)
    flat = np.ravel_multi_index(tuple(multi.T), tuple(a.shape[0] for a in mats))
    sb = w * b[flat]
    x = np.linalg.pinv(sk.T @ sk + lam * np.eye(cols)) @ (sk.T @ sb)
    return Report(x, ridge_loss(mats, x, b, lam), 0, s, 0.0, {"indices": idx, "weights": w})
