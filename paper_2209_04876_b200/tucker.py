"""Tucker ALS on the device: core update, factor-matrix updates and the ALS driver.

Drop-in for pkg/src/kronsolve/tucker.py:
  * ``TuckerModel`` (:45-77), ``reconstruct`` / ``relative_error`` / ``regularized_loss`` (:80-101)
  * ``core_update`` (:108-127) -- exact (kronmatmul_svd_solve) or sketched (fast_kronecker_regression)
  * ``naive_factor_update`` (:130-159) -- per-row normal equations through the Gram Kronecker
    identity: mode-product chain (ks_gemm), kron of Grams, R_n x R_n pseudo-inverse (Jacobi SVD)
  * ``FactorUpdateWorkspace`` / ``build_factor_workspace`` (:162-280) with ``_power_iteration``
    (:283-313) fused into one CTA (ks_factor_workspace) and the Woodbury core inverse
    (ks_inverse_small)
  * ``fast_factor_matrix_update`` (:316-379) -- every row's random stream, product-sampler draws,
    sparse diagonal (one composite-key sort for all rows) and then ONE launch that solves all rows'
    penalised constrained Richardson problems, one CTA per row (ks_factor_rows_richardson)
  * ``AlsReport`` / ``initial_model`` / ``tucker_als`` (:382-493) -- Householder QR with LAPACK's
    sign convention for the orthonormal start (ks_qr_explicit).

Inputs may be NumPy arrays (results come back as NumPy) or CUDA tensors (results stay on the
device).  Host work is orchestration: seeds, sample counts, shape checks, loop control."""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np
import torch

from . import _state
from . import _device as D
from . import _lib
from ._numpy_rng import pcg64_state, seedseq_children_seed_words, split128
from .errors import InvalidInputError, NumericalFailureError, SizeGuardError
from .kron import _kron_apply_dev
from .leverage import REGRESSION_SAMPLE_CONSTANT, ProductSampler, device_standard_normal, ridge_leverage_scores
from .solvers import (DEFAULT_DENSE_GUARD, FactorCache, FactorGram, RegressionConfig, _factor_gram_dev, _gram_dev,
                      build_factor_cache, fast_kronecker_regression, kronmatmul_svd_solve)
from .tensor import (CompactSvd, _compact_svd_dev, _mode_mul_dev, _pinv_dev, as_matrix, as_tensor, devectorize,
                     vectorize)

POWER_ITERATION_MAX = 100
POWER_ITERATION_TOL = 1e-6
PENALTY_SAFETY_MARGIN = 1.05


@dataclass
class TuckerModel:
    """Core tensor plus one loading matrix per mode (tucker.py:45-77)."""

    core: object
    factors: list
    lam: float = 0.0

    def __post_init__(self):
        host = not D.on_device(self.core)
        core = as_tensor(self.core, "core")
        self.core = D.out(core, host)
        if len(self.factors) != core.ndim:
            raise InvalidInputError(
                f"core has order {core.ndim} but got {len(self.factors)} factors")
        facs = []
        for n, a in enumerate(self.factors):
            a = a if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
            if a.ndim != 2 or a.shape[1] != core.shape[n]:
                raise InvalidInputError(
                    f"factor {n} of shape {tuple(a.shape)} does not match core dim {core.shape[n]}")
            if a.shape[0] < a.shape[1]:
                raise InvalidInputError(
                    f"factor {n} is {tuple(a.shape)}; ranks above the dimension are not supported")
            facs.append(a)
        self.factors = facs
        if self.lam < 0:
            raise InvalidInputError(f"lambda must be >= 0, got {self.lam}")

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(int(a.shape[0]) for a in self.factors)

    @property
    def core_shape(self) -> tuple[int, ...]:
        return tuple(int(s) for s in self.core.shape)


def _dev_model(model: TuckerModel):
    return D.to_dev(model.core), [D.to_dev(a) for a in model.factors]


def _reconstruct_dev(core: torch.Tensor, facs: list[torch.Tensor]) -> torch.Tensor:
    t = core.contiguous()
    for mode, a in enumerate(facs):
        t = _mode_mul_dev(t, a, mode)
    return t


def _sumsq(a: torch.Tensor, b: torch.Tensor | None = None) -> torch.Tensor:
    out = D.empty(1)
    a = a.reshape(-1).contiguous()
    _lib.call("ks_sumsq_diff", D.p(a), D.p(None if b is None else b.reshape(-1).contiguous()), a.numel(),
              D.p(out), D.stream())
    return out


def reconstruct(model: TuckerModel):
    """Core multiplied by every factor along its mode (tucker.py:80-82)."""
    host = not D.on_device(model.core)
    core, facs = _dev_model(model)
    return D.out(_reconstruct_dev(core, facs), host)


def relative_error(model: TuckerModel, x) -> float:
    """``||Xhat - X||_F^2 / ||X||_F^2`` (tucker.py:85-93)."""
    xt = as_tensor(x)
    core, facs = _dev_model(model)
    num = float(_sumsq(_reconstruct_dev(core, facs), xt).item())
    den = float(_sumsq(xt).item())
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / den


def _losses_dev(core, facs, xt):
    err = _sumsq(_reconstruct_dev(core, facs), xt)
    reg = _sumsq(core)
    for a in facs:
        reg = reg + _sumsq(a)
    return err, reg


def regularized_loss(model: TuckerModel, x) -> float:
    """Squared reconstruction error plus lam times all squared Frobenius norms (tucker.py:96-101)."""
    xt = as_tensor(x)
    core, facs = _dev_model(model)
    err, reg = _losses_dev(core, facs, xt)
    return float(err.item()) + model.lam * float(reg.item())


def core_update(model: TuckerModel, x, mode: str = "exact", config: RegressionConfig | None = None,
                caches: Sequence[FactorCache] | None = None):
    """Solve the core regression at fixed factors; returns the new core (tucker.py:108-127)."""
    xs = tuple(int(s) for s in x.shape) if hasattr(x, "shape") else np.asarray(x).shape
    if tuple(xs) != model.shape:
        raise InvalidInputError(f"tensor shape {tuple(xs)} != model shape {model.shape}")
    # the reference's SolveReport.loss is discarded here (only the core is returned): not computed
    if mode == "exact":
        report = kronmatmul_svd_solve(model.factors, vectorize(x), model.lam, with_loss=False)
    elif mode == "fast":
        cfg = (config or RegressionConfig()).with_lam(model.lam)
        report = fast_kronecker_regression(model.factors, vectorize(x), cfg, caches=caches, with_loss=False)
    else:
        raise InvalidInputError(f"unknown core update mode {mode!r}")
    return devectorize(report.solution, model.core_shape)


# ---------------------------------------------------------------------------
# small dense helpers (device)
# ---------------------------------------------------------------------------

def _mm(a: torch.Tensor, b: torch.Tensor, ta: bool = False, tb: bool = False) -> torch.Tensor:
    """op(a) @ op(b) with ks_gemm (op = transpose when flagged)."""
    m = int(a.shape[1] if ta else a.shape[0])
    k = int(a.shape[0] if ta else a.shape[1])
    n = int(b.shape[0] if tb else b.shape[1])
    out = D.empty(m, n)
    if out.numel() == 0:
        return out
    if k == 0:
        return out.zero_()
    lda, ldb = int(a.shape[1]), int(b.shape[1])
    a_rs, a_cs = (1, lda) if ta else (lda, 1)
    b_rs, b_cs = (1, ldb) if tb else (ldb, 1)
    _lib.call("ks_gemm", m, n, k, 1.0, D.p(a), a_rs, a_cs, 0, D.p(b), b_rs, b_cs, 0, 0.0, D.p(out), n, 1, 0, 1,
              D.stream())
    return out


def _unfold_dev(t: torch.Tensor, n: int) -> torch.Tensor:
    return t.movedim(n, 0).reshape(int(t.shape[n]), -1).contiguous()


def _ptrs(ts):
    return _lib.ptr_array(ctypes.c_void_p, [0 if t is None else t.data_ptr() for t in ts])


# ---------------------------------------------------------------------------
# exact factor update
# ---------------------------------------------------------------------------

def naive_factor_update(model: TuckerModel, x, n: int, max_dense_entries: int | None = DEFAULT_DENSE_GUARD):
    """Exact ridge update of factor ``n``: every row solved via ``(KK^T + lam I)^+ K b_i^T`` with
    ``K = G_(n) (kron of others)^T`` (tucker.py:130-159)."""
    host = not D.on_device(x)
    xt = as_tensor(x)
    if tuple(int(s) for s in xt.shape) != model.shape:
        raise InvalidInputError(f"tensor shape {tuple(xt.shape)} != model shape {model.shape}")
    if not 0 <= n < len(model.factors):
        raise InvalidInputError(f"mode {n} out of range")
    core, facs = _dev_model(model)
    return D.out(_naive_factor_update_dev(core, facs, model.lam, xt, n, max_dense_entries), host)


def _naive_factor_update_dev(core, facs, lam, xt, n, max_dense_entries=DEFAULT_DENSE_GUARD):
    others = [(m, a) for m, a in enumerate(facs) if m != n]
    g_n = _unfold_dev(core, n)
    rn, r_rest = int(g_n.shape[0]), int(g_n.shape[1])
    if max_dense_entries is not None and r_rest * r_rest > max_dense_entries:
        raise SizeGuardError(
            f"Gram Kronecker product would hold {r_rest}x{r_rest} entries (guard: {max_dense_entries})")
    # K K^T = G (kron of Grams) G^T
    if others:
        grams = [_gram_dev(a) for _, a in others]
        w = _kron_apply_dev(grams, g_n.T.contiguous())
    else:
        w = g_n.T.contiguous()
    kkt = _mm(g_n, w)
    # (kron of others)^T B^T as the mode-product chain x x_m A_m^T (cheapest reduction first)
    y = xt.contiguous()
    order = sorted(others, key=lambda ma: int(ma[1].shape[1]) / max(1, int(ma[1].shape[0])))
    for m, a in order:
        y = _mode_mul_dev(y, a, m, transpose=True)
    yu = _unfold_dev(y, n)                        # I_n x R_rest  (= (K B^T)^T before G)
    mat = kkt + lam * torch.eye(rn, dtype=D.F64, device=kkt.device)
    pinv = _pinv_dev(mat.contiguous(), 1e-15)     # np.linalg.pinv's default rcond
    p = _mm(pinv, g_n)                            # (KK^T + lam I)^+ G   (R_n x R_rest)
    return _mm(yu, p, tb=True)                    # rows: ((KK^T + lam I)^+ G (kron)^T b_i^T)^T


# ---------------------------------------------------------------------------
# constrained-update workspace (Woodbury preconditioner)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class FactorUpdateWorkspace:
    """Preassembled operators for the constrained factor-row solves (tucker.py:162-214)."""

    g_n: object
    gn_pinv: object
    gnt_pinv: object
    penalty_weight: float
    v_factors: tuple
    base_diag: object
    correction_left: object
    correction_mid: object
    correction_right: object
    gram_matrices: tuple
    _dev: dict = field(default=None, repr=False, compare=False)

    @property
    def woodbury_core_inverse(self):
        return self.correction_mid

    def _apply(self, z, which: int):
        host = not D.on_device(z)
        d = self._dev
        zt = D.to_dev(z).reshape(-1).contiguous()
        if zt.numel() != d["r_rest"]:
            raise InvalidInputError(f"vector of length {zt.numel()} does not match {d['r_rest']}")
        out = D.empty(d["r_rest"])
        _lib.call("ks_factor_ws_apply", d["M"], _lib.ptr_array(ctypes.c_int32, d["R"]), _ptrs(d["V"]),
                  _ptrs(d["G"]), d["rn"], D.p(d["gn"]), D.p(d["gnp"]), D.p(d["mid"]), D.p(d["right"]),
                  D.p(d["bdiag"]), D.p(d["w"]), float(d["lam"]), D.p(zt), which, D.p(out), D.stream())
        return D.out(out, host)

    def constraint_projector(self):
        """Dense ``N = I - G^T (G^T)^+`` (orthogonal projector, test aid)."""
        d = self._dev
        nm = torch.eye(d["r_rest"], dtype=D.F64, device=d["gn"].device) - _mm(d["gn"], d["gnp"], ta=True, tb=True)
        return D.out(nm, d["host"])

    def project_feasible(self, z):
        """``G^T (G^T)^+ z`` (tucker.py:189-191)."""
        host = not D.on_device(z)
        d = self._dev
        zt = D.to_dev(z).reshape(-1, 1).contiguous()
        p = _mm(d["gnp"], zt, ta=True)
        return D.out(_mm(d["gn"], p, ta=True).reshape(-1), host)

    def apply_base(self, z):
        """``(K^T K + w I)^+ z`` through the factor eigendecompositions (tucker.py:189-193)."""
        return self._apply(z, 1)

    def apply(self, z):
        """Woodbury-corrected inverse of the penalised normal matrix (tucker.py:194-200)."""
        return self._apply(z, 0)

    def apply_penalized_normal(self, z):
        """Exact ``(K^T K + w I + G^+ (lam (G^T)^+ - w G)) z`` (tucker.py:202-206)."""
        return self._apply(z, 2)


def _other_grams(model_facs, n, caches):
    if caches is not None:
        grams = []
        for k, c in enumerate(caches):
            if k == n:
                continue
            g = c.gram
            grams.append((D.to_dev(g.v), D.to_dev(g.eigenvalues), D.to_dev(g.matrix)))
        return grams
    out = []
    for k, a in enumerate(model_facs):
        if k == n:
            continue
        v, w, gs = _factor_gram_dev(_gram_dev(a))
        out.append((v, w, gs))
    return out


def _build_workspace_dev(core, facs, n, eps, lam, caches, host=False):
    if core.ndim < 2:
        raise InvalidInputError("factor updates need an order >= 2 model")
    if not 0.0 < eps < 1.0 / 3.0:
        raise InvalidInputError(f"eps must be in (0, 1/3), got {eps}")
    g_n = _unfold_dev(core, n)
    fl = D.finite_flags(g_n)
    if not int(fl[1].item()):
        raise InvalidInputError("core unfolding is identically zero")
    rn, r_rest = int(g_n.shape[0]), int(g_n.shape[1])
    gnp = _pinv_dev(g_n, 1e-10)                   # R_rest x R_n
    grams = _other_grams(facs, n, caches)
    M = len(grams)
    R = [int(v.shape[0]) for v, _, _ in grams]
    v0 = device_standard_normal(0, r_rest)        # _power_iteration's default_rng(0) start
    wout = D.zeros(2)
    bdiag = D.empty(r_rest)
    right = D.empty(rn, r_rest)
    cm = D.empty(rn, rn)
    flags = torch.zeros(1, dtype=torch.int32, device=D.dev())
    _lib.call("ks_factor_workspace", M, _lib.ptr_array(ctypes.c_int32, R), _ptrs([g[0] for g in grams]),
              _ptrs([g[2] for g in grams]), _ptrs([g[1] for g in grams]), rn, D.p(g_n), D.p(gnp), float(lam),
              float(eps), D.p(v0), D.p(wout), D.p(bdiag), D.p(right), D.p(cm), D.p(flags), D.stream())
    mid = D.empty(rn, rn)
    info = torch.zeros(2, dtype=torch.int32, device=D.dev())
    _lib.call("ks_inverse_small", D.p(cm), rn, D.p(mid), D.p(info), D.stream())
    host_vals = torch.cat([wout, flags.to(D.F64), info.to(D.F64)]).cpu().tolist()
    w, est, bad, sing = host_vals[0], host_vals[1], host_vals[2], host_vals[3]
    if bad:
        raise NumericalFailureError("power iteration produced non-finite values", diagnostics={"estimate": est})
    if sing:
        raise NumericalFailureError("Woodbury core matrix is singular", diagnostics={"w": w, "mode": n})
    o = lambda t: D.out(t, host)  # noqa: E731
    dev = dict(M=M, R=R, V=[g[0] for g in grams], G=[g[2] for g in grams], rn=rn, r_rest=r_rest, gn=g_n, gnp=gnp,
               mid=mid, right=right, bdiag=bdiag, w=wout, lam=lam, host=host, estimate=est)
    return FactorUpdateWorkspace(
        g_n=o(g_n), gn_pinv=o(gnp), gnt_pinv=o(gnp.T), penalty_weight=w,
        v_factors=tuple(o(g[0]) for g in grams), base_diag=o(bdiag), correction_left=o(gnp),
        correction_mid=o(mid), correction_right=o(right), gram_matrices=tuple(o(g[2]) for g in grams), _dev=dev)


def build_factor_workspace(model: TuckerModel, n: int, eps: float, lam: float,
                           caches: Sequence[FactorCache] | None = None) -> FactorUpdateWorkspace:
    """Assemble the constrained-update preconditioner for factor ``n`` (tucker.py:217-280)."""
    host = not D.on_device(model.core)
    core, facs = _dev_model(model)
    return _build_workspace_dev(core, facs, n, eps, lam, caches, host)


def _power_iteration(operator, dim: int, seed: int = 0) -> float:
    """Largest-eigenvalue lower bound of a PSD operator (tucker.py:283-313), for user operators on
    CUDA tensors; ``build_factor_workspace`` runs the same loop fused in one CTA."""
    v = device_standard_normal(seed, dim)
    v = v / math.sqrt(float(_sumsq(v).item()))
    estimate = 0.0
    best = 0.0
    for _ in range(POWER_ITERATION_MAX):
        u = D.to_dev(operator(v)).reshape(-1)
        if not bool(torch.isfinite(u).all()):
            raise NumericalFailureError("power iteration produced non-finite values",
                                        diagnostics={"estimate": estimate})
        norm = math.sqrt(float(_sumsq(u).item()))
        if norm <= 1e-300:
            return 0.0
        new_estimate = float(_mm(v.reshape(1, -1), u.reshape(-1, 1)).item())
        best = max(best, new_estimate)
        v = u / norm
        if abs(new_estimate - estimate) <= POWER_ITERATION_TOL * max(1e-30, abs(new_estimate)):
            break
        estimate = new_estimate
    return best


# ---------------------------------------------------------------------------
# sketched factor update
# ---------------------------------------------------------------------------

def _factor_sample_count(config: RegressionConfig, r_rest: int, i_n: int) -> int:
    return max(1, math.ceil(config.effective_alpha * REGRESSION_SAMPLE_CONSTANT * r_rest * math.log(40 * r_rest)
                            * math.log(i_n / config.delta) / config.eps))


def _row_states(seed, rows: int, share: bool):
    """Seeding words of SeedSequence(seed).spawn(rows) (only the first child when shared) and
    whether they are pcg64_set_seed inputs (1) or final PCG64 states (0)."""
    use = 1 if share else rows
    if isinstance(seed, (int, np.integer)) and int(seed) >= 0:
        words = seedseq_children_seed_words(int(seed), use)
        return torch.from_numpy(words.view(np.int64)).to(D.dev()), 1
    seeds = np.random.SeedSequence(seed).spawn(rows)[:use]
    words = np.empty((use, 4), dtype=np.uint64)
    for i, ss in enumerate(seeds):
        st, inc = pcg64_state(ss)
        words[i] = (*split128(st), *split128(inc))
    return torch.from_numpy(words.view(np.int64)).to(D.dev()), 0


def fast_factor_matrix_update(model: TuckerModel, x, n: int, config: RegressionConfig,
                              caches: Sequence[FactorCache] | None = None):
    """Sketched update of factor ``n``; each row is solved independently (tucker.py:316-379).

    All rows run in one launch (one CTA per row); the sampled rows, weights and iterations are
    the reference's (same per-row SeedSequence children, same stopping rules)."""
    host = not D.on_device(x)
    xt = as_tensor(x)
    if tuple(int(s) for s in xt.shape) != model.shape:
        raise InvalidInputError(f"tensor shape {tuple(xt.shape)} != model shape {model.shape}")
    if not 0 <= n < len(model.factors):
        raise InvalidInputError(f"mode {n} out of range")
    if not 0.0 < config.eps < 1.0 / 3.0:
        raise InvalidInputError(f"factor updates require eps in (0, 1/3), got {config.eps}")
    core, facs = _dev_model(model)
    out, _ = _fast_factor_update_dev(core, facs, model.lam, xt, n, config, caches)
    return D.out(out, host)


def _fast_factor_update_dev(core, facs, lam, xt, n, config, caches, trace=None):
    others = [(m, a) for m, a in enumerate(facs) if m != n]
    i_n = int(facs[n].shape[0])
    r_rest = math.prod(int(a.shape[1]) for _, a in others)
    i_rest = math.prod(int(a.shape[0]) for _, a in others)
    s = _factor_sample_count(config, r_rest, i_n)
    if s >= i_rest:
        return _naive_factor_update_dev(core, facs, lam, xt, n), None
    ws = _build_workspace_dev(core, facs, n, config.eps, lam, caches)
    d = ws._dev
    if caches is not None:
        svds = [caches[m].svd for m, _ in others]
    else:
        svds = []
        for _, a in others:
            u, sg, v = _compact_svd_dev(a, 1e-10)
            svds.append(CompactSvd(u=u, sigma=sg, v=v))
    sampler = ProductSampler([ridge_leverage_scores(sv, 0.0) for sv in svds])
    M = len(others)
    share = bool(config.share_row_sketch)
    nstreams = 1 if share else i_n
    states, seeded = _row_states(config.seed, i_n, share)
    u = D.empty(M * nstreams * s)
    _lib.call("ks_pcg64_random_streams", D.p(states), seeded, nstreams, M, s, D.p(u), D.stream())
    idx = D.empty(nstreams * s, M + 1, dtype=D.I64)
    w = D.empty(nstreams * s)
    _lib.call("ks_factor_draws_rows", M, _ptrs(sampler._cdfs), _ptrs(sampler._probs),
              _lib.ptr_array(ctypes.c_int64, [int(c.numel()) for c in sampler._cdfs]), D.p(u), nstreams, s,
              D.p(idx), D.p(w), D.stream())
    # one sort dedups every row's sketch: key = row * I_rest + ravel(draw) (kron.py:173-190 per row)
    row_shape = [nstreams] + [int(a.shape[0]) for _, a in others]
    sd_idx = D.empty(nstreams * s, dtype=D.I64)
    sd_val = D.empty(nstreams * s)
    nnz = ctypes.c_int64(0)
    _lib.call("ks_sketch_diag", M + 1, D.p(idx), _lib.ptr_array(ctypes.c_int64, row_shape), D.p(w), nstreams * s,
              D.p(sd_idx), D.p(sd_val), ctypes.byref(nnz), D.stream())
    kr = None
    if M >= 3:
        kr = D.empty(max(1, nnz.value) * math.prod(int(a.shape[1]) for _, a in others[1:]))
    strides = [int(st) for st in xt.stride()]
    max_iters = int(config.effective_max_iters)
    rn = d["rn"]
    out = D.empty(i_n, rn)
    iters = torch.zeros(i_n, dtype=torch.int32, device=D.dev())
    flags = torch.zeros(i_n, dtype=torch.int32, device=D.dev())
    hist = D.zeros(i_n, max(1, max_iters))
    _lib.call("ks_factor_rows_richardson", M, _ptrs([a for _, a in others]),
              _lib.ptr_array(ctypes.c_int64, [int(a.shape[0]) for _, a in others]),
              _lib.ptr_array(ctypes.c_int32, d["R"]), _ptrs(d["V"]), rn, D.p(d["gn"]), D.p(d["gnp"]),
              D.p(d["mid"]), D.p(d["right"]), D.p(d["bdiag"]), D.p(d["w"]), float(lam), D.p(sd_idx), D.p(sd_val),
              nnz.value, int(share), i_n, D.p(xt), strides[n],
              _lib.ptr_array(ctypes.c_int64, [strides[m] for m, _ in others]), D.p(kr),
              float(config.effective_damping), max_iters, float(config.residual_tol), s, D.p(out), D.p(iters),
              D.p(flags), D.p(hist), D.stream())
    fl = flags.cpu()
    if bool((fl == 2).any()):
        raise SizeGuardError("a factor row holds more samples than the launch was sized for")
    bad = torch.nonzero(fl == 1).reshape(-1)
    if bad.numel():
        r = int(bad[0])
        it = int(iters[r].item())
        h = hist[r, :it + 1].cpu().tolist()
        raise NumericalFailureError("Richardson iteration diverged", iterations=it,
                                    diagnostics={"residual_history": h, "row": r})
    if trace is not None:
        trace.update(s=s, w=ws.penalty_weight, iters=iters, hist=hist, sd_idx=sd_idx[:nnz.value],
                     sd_val=sd_val[:nnz.value], idx=idx, weights=w)
    return out, ws


# ---------------------------------------------------------------------------
# ALS driver
# ---------------------------------------------------------------------------

@dataclass
class AlsReport:
    """Loss/time trace of one alternating-least-squares run (tucker.py:382-397)."""

    step_labels: list = field(default_factory=list)
    step_losses: list = field(default_factory=list)
    step_errors: list = field(default_factory=list)
    step_seconds: list = field(default_factory=list)
    sweep_losses: list = field(default_factory=list)
    sweep_rres: list = field(default_factory=list)
    sweep_seconds: list = field(default_factory=list)
    rre: float = math.nan

    @property
    def mean_sweep_seconds(self) -> float:
        return float(np.mean(self.sweep_seconds)) if self.sweep_seconds else math.nan


def _initial_factors_dev(shape, core_shape, seed):
    total = sum(int(i) * int(r) for i, r in zip(shape, core_shape))
    g = device_standard_normal(seed, total)
    facs, off = [], 0
    for i_n, r_n in zip(shape, core_shape):
        a = g[off:off + i_n * r_n].reshape(i_n, r_n).contiguous()
        off += i_n * r_n
        q = D.empty(i_n, r_n)
        _lib.call("ks_qr_explicit", D.p(a), i_n, r_n, D.p(q), D.stream())
        facs.append(q)
    return facs


def initial_model(x, core_shape: Sequence[int], lam: float, seed) -> TuckerModel:
    """Random orthonormal factors, zero core (tucker.py:400-409)."""
    host = not D.on_device(x)
    shape = tuple(int(s) for s in x.shape)
    facs = _initial_factors_dev(shape, tuple(int(r) for r in core_shape), seed)
    core = D.zeros(*tuple(int(r) for r in core_shape))
    return TuckerModel(core=D.out(core, host), factors=[D.out(a, host) for a in facs], lam=lam)


def _reseed(config: RegressionConfig, seed_seq: np.random.SeedSequence) -> RegressionConfig:
    return replace(config, seed=int(seed_seq.generate_state(1)[0]))


def tucker_als(x, core_shape: Sequence[int], lam: float = 0.0, sweeps: int = 5, solver_mode: str = "exact",
               config: RegressionConfig | None = None, loss_change_tol: float | None = None):
    """Alternating least squares for the regularised Tucker objective (tucker.py:412-493).

    Returns ``(model, AlsReport)``; the model holds NumPy arrays for host input and CUDA tensors
    for device input."""
    host = not D.on_device(x)
    xt = as_tensor(x)
    core_shape = tuple(int(r) for r in core_shape)
    shape = tuple(int(s) for s in xt.shape)
    if len(core_shape) != xt.ndim:
        raise InvalidInputError(f"core shape {core_shape} does not match tensor order {xt.ndim}")
    if any(r < 1 or r > i for r, i in zip(core_shape, shape)):
        raise InvalidInputError(f"core shape {core_shape} must be componentwise in [1, {shape}]")
    if sweeps < 1:
        raise InvalidInputError(f"sweeps must be >= 1, got {sweeps}")
    if solver_mode not in ("exact", "fast"):
        raise InvalidInputError(f"unknown solver mode {solver_mode!r}")
    config = (config or RegressionConfig()).with_lam(lam)

    facs = _initial_factors_dev(shape, core_shape, config.seed)
    core = D.zeros(*core_shape)
    caches = [build_factor_cache(a) for a in facs]
    report = AlsReport()
    x_norm_sq = float(_sumsq(xt).item())

    def record(label: str, seconds: float):
        err, reg = _losses_dev(core, facs, xt)
        e, r = torch.cat([err, reg]).cpu().tolist()
        report.step_labels.append(label)
        report.step_losses.append(e + lam * r)
        report.step_errors.append(e)
        report.step_seconds.append(seconds)

    def timed():
        torch.cuda.synchronize()
        return time.perf_counter()

    def model_now():
        return TuckerModel(core=core, factors=list(facs), lam=lam)

    t0 = timed()
    core = D.to_dev(core_update(model_now(), xt, mode="exact")).reshape(core_shape).contiguous()
    record("init-core", timed() - t0)
    seed_root = np.random.SeedSequence(config.seed)
    prev_sweep_loss = report.step_losses[-1]
    for sweep in range(sweeps):
        sweep_start = timed()
        sweep_seeds = seed_root.spawn(xt.ndim + 1)
        for n in range(xt.ndim):
            t0 = timed()
            if solver_mode == "exact":
                facs[n] = _naive_factor_update_dev(core, facs, lam, xt, n)
            else:
                step_cfg = _reseed(config, sweep_seeds[n])
                if not 0.0 < step_cfg.eps < 1.0 / 3.0:
                    raise InvalidInputError(f"factor updates require eps in (0, 1/3), got {step_cfg.eps}")
                facs[n], _ = _fast_factor_update_dev(core, facs, lam, xt, n, step_cfg, caches)
            caches[n] = build_factor_cache(facs[n])
            record(f"sweep{sweep}-factor{n}", timed() - t0)
        t0 = timed()
        if solver_mode == "exact":
            core = D.to_dev(core_update(model_now(), xt, mode="exact"))
        else:
            step_cfg = _reseed(config, sweep_seeds[-1])
            core = D.to_dev(core_update(model_now(), xt, mode="fast", config=step_cfg, caches=caches))
        core = core.reshape(core_shape).contiguous()
        record(f"sweep{sweep}-core", timed() - t0)
        report.sweep_losses.append(report.step_losses[-1])
        report.sweep_rres.append(report.step_errors[-1] / x_norm_sq if x_norm_sq > 0 else 0.0)
        report.sweep_seconds.append(timed() - sweep_start)
        loss = report.sweep_losses[-1]
        if (loss_change_tol is not None
                and abs(prev_sweep_loss - loss) <= loss_change_tol * max(1.0, abs(prev_sweep_loss))):
            break
        prev_sweep_loss = loss
    num = float(_sumsq(_reconstruct_dev(core, facs), xt).item())
    report.rre = (0.0 if num == 0.0 else math.inf) if x_norm_sq == 0.0 else num / x_norm_sq
    model = TuckerModel(core=D.out(core, host), factors=[D.out(a, host) for a in facs], lam=lam)
    return model, report


# Public entry points are gated (capture vs. concurrent solves, see _state.py).
_state.gate_names(globals(), [
    "build_factor_workspace",
    "core_update",
    "fast_factor_matrix_update",
    "initial_model",
    "naive_factor_update",
    "reconstruct",
    "regularized_loss",
    "relative_error",
    "tucker_als",
])
FactorUpdateWorkspace.apply = _state.gated(FactorUpdateWorkspace.apply)
