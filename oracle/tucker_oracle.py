"""CPU oracle for the Tucker-ALS factor-matrix updates -- TEST INFRASTRUCTURE ONLY.

NumPy restatement of the SURVEY.md 8(f) rows 1-2 of the reference ``kronsolve``
(pkg/src/kronsolve/tucker.py): ``naive_factor_update``, ``build_factor_workspace`` with its
Woodbury-corrected preconditioner, ``_power_iteration``, ``fast_factor_matrix_update`` and the
``tucker_als`` driver with its loss bookkeeping.  Like ``kronsolve_oracle`` it is the checker: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` may import it; the product package never
does.  Pinned against the live reference by ``tests/test_tucker_oracle.py`` (build container) and
against the committed fixture ``tests/golden/tucker_units.npz`` produced by running the reference
(``tests/golden/make_golden.py tucker``).

The floating-point operation order follows the reference (same NumPy calls in the same order).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from functools import reduce

import numpy as np

from . import kronsolve_oracle as K

POWER_MAX = 100          # tucker.py:40
POWER_TOL = 1e-6         # tucker.py:41
SAFETY = 1.05            # tucker.py:42
DENSE_GUARD = 10 ** 8  # solvers.py:53 DEFAULT_DENSE_GUARD


@dataclass(frozen=True)
class Cfg:
    """The RegressionConfig fields the factor updates read (solvers.py:60-112)."""

    eps: float = 0.25
    delta: float = 0.05
    lam: float = 0.0
    alpha: float = 1.0
    max_iters: int | None = None
    residual_tol: float = 1e-9
    seed: int = 0
    damping: float | None = None
    share_row_sketch: bool = False

    @property
    def damp(self):
        return (1.0 - math.sqrt(self.eps)) if self.damping is None else self.damping

    @property
    def iters(self):
        return K.effective_max_iters(self.eps, self.max_iters)


def unfold(x, n):
    """tensor.py:133-143: mode-n fibres become columns, other indices lexicographic."""
    x = np.asarray(x, dtype=np.float64)
    return np.moveaxis(x, n, 0).reshape(x.shape[n], -1)


def pseudo_inverse(a):
    """tensor.py:110-115: V diag(1/sigma) U^T from the compact SVD."""
    sv = K.compact_svd(a)
    if sv.sigma.size == 0:
        return np.zeros((np.asarray(a).shape[1], np.asarray(a).shape[0]))
    return (sv.v / sv.sigma) @ sv.u.T


def reconstruct(core, factors):
    """tucker.py:80-82 (multi_mode_product, tensor.py:159-183)."""
    x = np.asarray(core, dtype=np.float64)
    for mode, a in enumerate(factors):
        x = np.moveaxis(np.tensordot(np.asarray(a), x, axes=(1, mode)), 0, mode)
    return x


def regularized_loss(core, factors, lam, x):
    """tucker.py:96-101."""
    err = float(np.sum((reconstruct(core, factors) - x) ** 2))
    reg = float(np.sum(np.asarray(core) ** 2)) + sum(float(np.sum(a ** 2)) for a in factors)
    return err + lam * reg


def naive_factor_update(core, factors, lam, x, n, guard=DENSE_GUARD):
    """tucker.py:130-159: per-row normal equations through the Gram Kronecker identity."""
    others = [a for k, a in enumerate(factors) if k != n]
    g_n = unfold(core, n)
    r_rest = g_n.shape[1]
    if guard is not None and r_rest * r_rest > guard:
        raise K.OracleError("size", "Gram Kronecker product too large")
    gram_rest = reduce(np.kron, [a.T @ a for a in others], np.ones((1, 1)))
    kkt = g_n @ gram_rest @ g_n.T
    b = unfold(x, n)
    kbt = g_n @ (K.kron_mat_mul([a.T for a in others], b.T) if others else b.T)
    y = np.linalg.pinv(kkt + lam * np.eye(g_n.shape[0])) @ kbt
    return y.T


def power_iteration(op, dim, seed=0):
    """tucker.py:283-313: best Rayleigh quotient of at most 100 normalised power steps."""
    gen = np.random.default_rng(seed)
    v = gen.standard_normal(dim)
    v /= np.linalg.norm(v)
    est = 0.0
    best = 0.0
    for _ in range(POWER_MAX):
        u = op(v)
        if not np.all(np.isfinite(u)):
            raise K.OracleError("numerical", "power iteration produced non-finite values")
        nrm = float(np.linalg.norm(u))
        if nrm <= 1e-300:
            return 0.0
        new = float(v @ u)
        best = max(best, new)
        v = u / nrm
        if abs(new - est) <= POWER_TOL * max(1e-30, abs(new)):
            break
        est = new
    return best


@dataclass
class Workspace:
    """tucker.py:162-214 (FactorUpdateWorkspace)."""

    g_n: np.ndarray
    gn_pinv: np.ndarray
    gnt_pinv: np.ndarray
    w: float
    vs: list
    base_diag: np.ndarray
    right: np.ndarray
    mid: np.ndarray
    grams: list
    norm_sq: float = 0.0

    def apply_base(self, z):
        t = K.kron_vec_square([v.T for v in self.vs], z) * self.base_diag
        return K.kron_vec_square(self.vs, t)

    def apply(self, z):
        base = self.apply_base(z)
        corr = self.gn_pinv @ (self.mid @ (self.right @ base))
        return base - self.apply_base(corr)

    def project_feasible(self, z):
        return self.g_n.T @ (self.gnt_pinv @ z)

    def constraint_projector(self):
        return np.eye(self.gn_pinv.shape[0]) - self.g_n.T @ self.gnt_pinv


def build_factor_workspace(core, factors, n, eps, lam, grams=None):
    """tucker.py:217-280.  ``grams``: per-factor (v, eigenvalues, matrix) of ALL factors, or None."""
    core = np.asarray(core, dtype=np.float64)
    if core.ndim < 2:
        raise K.OracleError("invalid", "factor updates need an order >= 2 model")
    if not 0.0 < eps < 1.0 / 3.0:
        raise K.OracleError("invalid", "eps must be in (0, 1/3)")
    g_n = unfold(core, n)
    if not np.any(g_n):
        raise K.OracleError("invalid", "core unfolding is identically zero")
    gn_pinv = pseudo_inverse(g_n)
    gnt_pinv = gn_pinv.T
    if grams is None:
        grams = [K.factor_gram(a) for a in factors]
    og = [g for k, g in enumerate(grams) if k != n]
    mats = [g[2] for g in og]
    r_rest = g_n.shape[1]

    def op(v):
        u = v - g_n.T @ (gnt_pinv @ v)
        t = K.kron_mat_mul(mats, u)
        t = t + lam * (gn_pinv @ (gn_pinv.T @ u))
        return t - g_n.T @ (gnt_pinv @ t)

    norm_sq = power_iteration(op, r_rest)
    w = (1.0 + 12.0 / eps) * norm_sq * SAFETY
    eig = reduce(np.kron, [g[1] for g in og])
    base_diag = K.pseudo_reciprocal(eig + w)
    vs = [g[0] for g in og]
    right = lam * gnt_pinv - w * g_n
    t = K.kron_mat_mul([v.T for v in vs], gn_pinv)
    p0 = K.kron_mat_mul(vs, base_diag[:, None] * t)
    cm = np.eye(g_n.shape[0]) + right @ p0
    try:
        mid = np.linalg.solve(cm, np.eye(g_n.shape[0]))
    except np.linalg.LinAlgError as exc:
        raise K.OracleError("numerical", "Woodbury core matrix is singular") from exc
    return Workspace(g_n, gn_pinv, gnt_pinv, w, vs, base_diag, right, mid, mats, norm_sq)


def factor_sample_count(r_rest, i_n, cfg: Cfg):
    """tucker.py:336-338."""
    return max(1, math.ceil(cfg.alpha * K.REGRESSION_C * r_rest * math.log(40 * r_rest)
                            * math.log(i_n / cfg.delta) / cfg.eps))


def fast_factor_matrix_update(core, factors, lam, x, n, cfg: Cfg, caches=None, trace=None):
    """tucker.py:316-379.  ``caches``: per-factor (svd, (v, eig, gram)) of ALL factors, or None."""
    x = np.asarray(x, dtype=np.float64)
    if not 0.0 < cfg.eps < 1.0 / 3.0:
        raise K.OracleError("invalid", "factor updates require eps in (0, 1/3)")
    others = [a for k, a in enumerate(factors) if k != n]
    i_n = factors[n].shape[0]
    r_rest = math.prod(a.shape[1] for a in others)
    i_rest = math.prod(a.shape[0] for a in others)
    s = factor_sample_count(r_rest, i_n, cfg)
    if s >= i_rest:
        return naive_factor_update(core, factors, lam, x, n)
    grams = [c[1] for c in caches] if caches is not None else None
    ws = build_factor_workspace(core, factors, n, cfg.eps, lam, grams)
    svds = [c[0] for k, c in enumerate(caches) if k != n] if caches is not None else \
        [K.compact_svd(a) for a in others]
    sampler = K.Sampler([K.ridge_scores(sv, 0.0) for sv in svds])
    b = unfold(x, n)
    row_shape = tuple(a.shape[0] for a in others)
    w = ws.w
    seeds = np.random.SeedSequence(cfg.seed).spawn(i_n)
    out = np.empty((i_n, core.shape[n]))
    shared = K.sample_rows(sampler, s, seeds[0]) if cfg.share_row_sketch else None
    if trace is not None:
        trace.update(s=s, w=w, norm_sq=ws.norm_sq, rows=[])
    for i in range(i_n):
        idx, wt = shared if shared is not None else K.sample_rows(sampler, s, seeds[i])
        sd_idx, sd_val = K.sparse_diagonal_from_sketch(idx, wt, row_shape)
        rhs = K.sketched_kron_transpose_apply(others, sd_idx, sd_val, sd_val * b[i, sd_idx])

        def normal(z):
            t = K.sketched_kron_transpose_apply(others, sd_idx, sd_val,
                                                K.sketched_kron_apply(others, sd_idx, sd_val, z))
            t = t + w * z
            t = t + lam * (ws.gn_pinv @ (ws.gnt_pinv @ z))
            return t - w * (ws.gn_pinv @ (ws.g_n @ z))

        z, iters, hist = K.richardson(normal, ws.apply, rhs, cfg.damp, cfg.iters, cfg.residual_tol)
        z = ws.project_feasible(z)
        out[i, :] = ws.gnt_pinv @ z
        if trace is not None:
            trace["rows"].append(dict(iters=iters, hist=hist, sd_indices=sd_idx, sd_values=sd_val))
    return out


def initial_model(shape, core_shape, seed):
    """tucker.py:400-409: orthonormal Q of N(0,1) matrices, zero core."""
    return np.zeros(tuple(core_shape)), K.initial_tucker_factors(shape, core_shape, seed)


@dataclass
class AlsReport:
    """tucker.py:382-397."""

    step_labels: list = field(default_factory=list)
    step_losses: list = field(default_factory=list)
    step_errors: list = field(default_factory=list)
    sweep_losses: list = field(default_factory=list)
    sweep_rres: list = field(default_factory=list)
    rre: float = math.nan


def _reseed(cfg: Cfg, seq):
    """tucker.py:496-498."""
    return replace(cfg, seed=int(seq.generate_state(1)[0]))


def tucker_als(x, core_shape, lam=0.0, sweeps=5, mode="exact", cfg: Cfg | None = None,
               loss_change_tol=None):
    """tucker.py:412-493.  Returns (core, factors, AlsReport)."""
    x = np.asarray(x, dtype=np.float64)
    core_shape = tuple(int(r) for r in core_shape)
    cfg = replace(cfg or Cfg(), lam=lam)
    core, factors = initial_model(x.shape, core_shape, cfg.seed)
    caches = [K.factor_cache(a) for a in factors]
    rep = AlsReport()
    xsq = float(np.sum(x ** 2))

    def record(label):
        err = float(np.sum((reconstruct(core, factors) - x) ** 2))
        reg = float(np.sum(core ** 2)) + sum(float(np.sum(a ** 2)) for a in factors)
        rep.step_labels.append(label)
        rep.step_losses.append(err + lam * reg)
        rep.step_errors.append(err)

    core = K.core_update_exact(factors, x, lam)
    record("init-core")
    root = np.random.SeedSequence(cfg.seed)
    prev = rep.step_losses[-1]
    for sweep in range(sweeps):
        seeds = root.spawn(x.ndim + 1)
        for n in range(x.ndim):
            if mode == "exact":
                factors[n] = naive_factor_update(core, factors, lam, x, n)
            else:
                factors[n] = fast_factor_matrix_update(core, factors, lam, x, n,
                                                       _reseed(cfg, seeds[n]), caches=caches)
            caches[n] = K.factor_cache(factors[n])
            record(f"sweep{sweep}-factor{n}")
        if mode == "exact":
            core = K.core_update_exact(factors, x, lam)
        else:
            c = _reseed(cfg, seeds[-1])
            core, _ = K.core_update_fast(factors, x, lam, caches, eps=c.eps, delta=c.delta, alpha=c.alpha,
                                         seed=c.seed, max_iters=c.max_iters, residual_tol=c.residual_tol,
                                         damping=c.damping)
        record(f"sweep{sweep}-core")
        rep.sweep_losses.append(rep.step_losses[-1])
        rep.sweep_rres.append(rep.step_errors[-1] / xsq if xsq > 0 else 0.0)
        loss = rep.sweep_losses[-1]
        if loss_change_tol is not None and abs(prev - loss) <= loss_change_tol * max(1.0, abs(prev)):
            break
        prev = loss
    num = float(np.sum((reconstruct(core, factors) - x) ** 2))
    rep.rre = (0.0 if num == 0.0 else math.inf) if xsq == 0.0 else num / xsq
    return core, factors, rep
