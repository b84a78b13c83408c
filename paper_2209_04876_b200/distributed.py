"""Row-sharded multi-GPU execution of the FastKroneckerRegression path.

The n1 x n2 reshape of b (factor 0 = slow index) and every sampled row shard by contiguous
ranges of factor-0 rows, one rank per GPU:

* exact KronMatMul  t = U1^T B U2 : each rank contracts its row block, one d1*d2 all-reduce;
* loss              ||A1 X A2^T - B||^2 : per-rank partial over its rows, one scalar all-reduce;
* fast solve        preprocessing is replicated (identical NumPy-exact streams on every rank, so
                    every rank draws the same sketch); each rank keeps the samples whose factor-0
                    row it owns, and the Richardson loop all-reduces the d1*d2 Gram partial
                    H_local x once per iteration (the only exchange in the loop); the
                    preconditioner and the update are replicated.

Collectives go through ``torch.distributed`` (NCCL on GPUs, gloo on CPU for the tests); the local
compute is supplied by an ops object so the same plan runs the device kernels in production and
NumPy stand-ins in the CPU tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _state


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous balanced split of the n0 factor-0 rows over `world` ranks."""

    world: int
    rank: int
    n0: int

    def __post_init__(self):
        if not (1 <= self.world and 0 <= self.rank < self.world and self.n0 >= 1):
            raise ValueError(f"bad shard plan {self}")

    def range_of(self, r: int) -> tuple[int, int]:
        base, extra = divmod(self.n0, self.world)
        start = r * base + min(r, extra)
        return start, start + base + (1 if r < extra else 0)

    @property
    def rows(self) -> tuple[int, int]:
        return self.range_of(self.rank)

    def owner_of_row(self, i0):
        """Rank owning factor-0 row(s) i0 (vectorised)."""
        i0 = np.asarray(i0)
        base, extra = divmod(self.n0, self.world)
        cut = extra * (base + 1)
        return np.where(i0 < cut, i0 // (base + 1), extra + (i0 - cut) // max(base, 1))

    def owned_mask(self, flat, n_rest: int):
        """Mask of flat Kronecker row indices whose factor-0 row this rank owns."""
        lo, hi = self.rows
        i0 = np.asarray(flat) // n_rest
        return (i0 >= lo) & (i0 < hi)


def allreduce_sum(t, dist=None):
    """Sum a tensor over all ranks in place (no-op for a single process)."""
    if dist is None:
        import torch.distributed as dist  # noqa: F811
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
    return t


class ShardedKron2:
    """Two-factor n^2 passes on a row block [lo, hi) of B, combined across ranks.

    ``ops`` provides ``contract(L_rows, B_rows, R) -> T`` (p x q partial) and
    ``resid(L_rows, X, R, B_rows) -> float`` (partial sum of squares) for the local block.
    """

    def __init__(self, plan: ShardPlan, ops, torch_mod):
        self.plan, self.ops, self.torch = plan, ops, torch_mod

    def contract(self, L, B_rows, R):
        lo, hi = self.plan.rows
        T = self.ops.contract(L[lo:hi], B_rows, R)
        return allreduce_sum(T)

    def residual_sumsq(self, L, X, R, B_rows):
        lo, hi = self.plan.rows
        s = self.ops.resid(L[lo:hi], X, R, B_rows)
        t = self.torch.tensor([s], dtype=self.torch.float64, device=self.ops.device)
        return float(allreduce_sum(t).item())


def shard_sparse_diagonal(plan: ShardPlan, indices, values, n_rest: int):
    """Samples of the (replicated) sparse diagonal whose factor-0 row this rank owns."""
    idx = np.asarray(indices)
    mask = plan.owned_mask(idx, n_rest)
    return idx[mask], np.asarray(values)[mask]


def sharded_richardson(apply_normal_local, apply_precond, rhs_local, damping: float, max_iters: int,
                       residual_tol: float, torch_mod, lam: float):
    """Richardson loop of solvers.py:201-248 with the normal operator summed across ranks.

    ``apply_normal_local(x)`` returns this rank's part of (SK)^T S (SK) x; the right-hand side
    partials are all-reduced once up front.  Stopping and divergence rules match the
    reference; every rank takes identical decisions because it sees identical norms."""
    rhs = allreduce_sum(rhs_local.clone())
    x = torch_mod.zeros_like(rhs)
    scale = float(torch_mod.linalg.norm(apply_precond(rhs)))
    tol = residual_tol * max(scale, np.finfo(float).tiny)
    hist, iters = [], 0
    for _ in range(max_iters):
        hx = allreduce_sum(apply_normal_local(x)) + lam * x
        step = apply_precond(hx - rhs)
        nrm = float(torch_mod.linalg.norm(step))
        hist.append(nrm)
        if nrm <= tol:
            break
        if len(hist) > 5:
            win = hist[-6:]
            if all(win[i + 1] > win[i] for i in range(5)) and win[-1] > 10.0 * win[0]:
                from .errors import NumericalFailureError
                raise NumericalFailureError("Richardson iteration diverged", iterations=iters,
                                            diagnostics={"residual_history": hist})
        x = x - damping * step
        iters += 1
    return x, iters, hist


def row_block_of_b(b, plan: ShardPlan, n_rest: int):
    """The rank's contiguous slice of vec(b) (rows [lo, hi) of the n0 x n_rest reshape)."""
    lo, hi = plan.rows
    return b[lo * n_rest: hi * n_rest]


def split_counts(n: int, world: int) -> list[int]:
    base, extra = divmod(n, world)
    return [base + (1 if r < extra else 0) for r in range(world)]


def expected_allreduce_bytes(d1: int, d2: int, iterations: int) -> int:
    """Bytes each rank contributes to collectives in one sharded fast solve (rhs + one Gram partial
    per iteration), for reporting."""
    return 8 * d1 * d2 * (iterations + 1) + 8 * math.prod((1,))


# ---------------------------------------------------------------------------
# Device execution (NCCL): the exact solve and the loss on row-sharded b
# ---------------------------------------------------------------------------

class DeviceKron2Ops:
    """Local compute of ShardedKron2 on the GPU: the K1 contraction (ks_kron2_contract) and the K2
    residual pass (ks_kron2_residual_sumsq) on this rank's row block."""

    def __init__(self):
        import torch
        from . import _device as D
        self.torch, self.D = torch, D
        self.device = D.dev()

    def contract(self, L_rows, B_rows, R):
        from . import _lib
        D = self.D
        m, p = int(L_rows.shape[0]), int(L_rows.shape[1])
        k, q = int(R.shape[0]), int(R.shape[1])
        T = D.empty(p, q)
        if m == 0:
            return T.zero_()
        _lib.call("ks_kron2_contract", D.p(L_rows.contiguous()), D.p(B_rows), int(B_rows.stride(0)), D.p(R), m, k, p,
                  q, D.p(T), D.stream())
        return T

    def resid(self, L_rows, X, R, B_rows):
        from . import _lib
        D = self.D
        out = D.zeros(1)
        m = int(L_rows.shape[0])
        if m:
            _lib.call("ks_kron2_residual_sumsq", D.p(L_rows.contiguous()), D.p(X.contiguous()), D.p(R), D.p(B_rows),
                      int(B_rows.stride(0)), m, int(R.shape[0]), int(L_rows.shape[1]), int(R.shape[1]), D.p(out),
                      D.stream())
        return float(out.item())


def sharded_kronmatmul_svd_solve(factors, b_rows, lam: float, plan: ShardPlan, dist=None):
    """kronmatmul_svd_solve (solvers.py:302-320) with b row-sharded over the ranks:
    every rank holds both (small) factors and its rows [lo, hi) of the n1 x n2 reshape of b
    (``b_rows``, device, (hi - lo) x n2).  The compact SVDs are replicated, the n^2 contraction
    U1[lo:hi]^T B_rows U2 runs locally on the FP64 tensor pipe, one d1*d2 all-reduce combines it,
    and x = (V1 (x) V2) (sigma / (sigma^2 + lam)) t is replicated.  Returns (x, loss): the loss is
    the sharded K2 pass plus one scalar all-reduce."""
    import torch
    from functools import reduce as _reduce
    from . import _device as D
    from .kron import _kron_apply_dev
    from .tensor import _compact_svd_dev
    facs = [D.to_dev(a) for a in factors]
    if len(facs) != 2:
        raise ValueError("the row-sharded exact solve covers the two-factor problem")
    lo, hi = plan.rows
    svds = [_compact_svd_dev(a, 1e-10) for a in facs]
    ops = DeviceKron2Ops()
    sk = ShardedKron2(plan, ops, torch)
    T = sk.contract(svds[0][0], b_rows, svds[1][0].contiguous())
    sigma = _reduce(torch.kron, [s[1] for s in svds])
    t = T.reshape(-1) * (sigma / (sigma * sigma + lam))
    x = _kron_apply_dev([s[2] for s in svds], t.reshape(-1, 1).contiguous())[:, 0].contiguous()
    X = x.reshape(int(facs[0].shape[1]), int(facs[1].shape[1]))
    r2 = sk.residual_sumsq(facs[0], X, facs[1], b_rows)
    return x, r2 + lam * float((x * x).sum().item())


def sharded_fast_kronecker_regression(factors, b_rows, config, plan: ShardPlan, caches=None):
    """fast_kronecker_regression (solvers.py:372-462) with b row-sharded over the ranks.

    Every rank holds both factors and its rows [lo, hi) of the n0 x n1 reshape of b (``b_rows``,
    device, (hi - lo) x n1).  The sketch and the preconditioner are computed replicated (identical
    NumPy-exact streams, so every rank draws the same sketch); each rank keeps the sampled rows
    whose factor-0 index it owns, gathers their b entries locally, and the Richardson loop
    all-reduces the d^2 normal-operator partial once per iteration (sharded_richardson).  Returns
    (x, iterations, history).  With one rank it is the single-GPU algorithm through the
    per-iteration kernels."""
    import math

    import torch

    from . import _device as D
    from .kron import SparseDiagonal, sketched_kron_apply, sketched_kron_transpose_apply
    from .solvers import FactorGram, _fast_sketch_dev, _validated_problem, build_kron_preconditioner

    if len(factors) != 2:
        raise ValueError("the row-sharded fast solve covers the two-factor problem")
    n0, n1 = int(factors[0].shape[0]), int(factors[1].shape[0])
    facs = [D.to_dev(a) for a in factors]
    sdiag, grams, s = _fast_sketch_dev(facs, config, caches)
    lo, hi = plan.rows
    keys = sdiag.indices
    own = (keys >= lo * n1) & (keys < hi * n1)
    li, lv = keys[own].contiguous(), sdiag.values[own].contiguous()
    local = SparseDiagonal._trusted(li, lv)
    b_at = b_rows.reshape(-1)[li - lo * n1].contiguous()
    rhs_local = sketched_kron_transpose_apply(facs, local, (lv * b_at).contiguous())
    pre = build_kron_preconditioner([FactorGram(v=v, eigenvalues=w, matrix=None) for v, w in grams], config.lam)

    def normal_local(x):
        return sketched_kron_transpose_apply(facs, local, sketched_kron_apply(facs, local, x))

    x, iters, hist = sharded_richardson(normal_local, pre.apply, rhs_local, config.effective_damping,
                                        config.effective_max_iters, config.residual_tol, torch, config.lam)
    return x, iters, hist


# Public entry points are gated (capture vs. concurrent solves, see _state.py).
_state.gate_names(globals(), ["sharded_kronmatmul_svd_solve", "sharded_fast_kronecker_regression"])
