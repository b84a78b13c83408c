"""Row-sharded multi-GPU execution of the FastKroneckerRegression path.

The n1 x n2 reshape of b (factor 0 = slow index) and every sampled row shard by contiguous
ranges of factor-0 rows, one rank per GPU:

* exact KronMatMul  t = U1^T B U2 : each rank contracts its row block, one d1*d2 all-reduce;
* loss              ||A1 X A2^T - B||^2 : per-rank partial over its rows, one scalar all-reduce;
* fast solve        preprocessing is replicated (identical NumPy-exact streams on every rank, so
                    every rank draws the same sketch); each rank keeps the samples whose factor-0
                    row it owns, and the Richardson loop all-reduces the d1*d2 Gram partial
                    H_local x once per iteration (the only exchange in the loop); the
                    preconditioner and the update are replicated.  On the device the loop is
                    launches + NCCL collectives only (DeviceShardedLoop: apply-only launches of
                    the persistent eigenbasis kernel, an in-graph all-reduce, a one-CTA update
                    kernel with the stopping rules), captured as one CUDA graph.

Collectives go through ``torch.distributed`` (NCCL on GPUs, gloo on CPU for the tests); the local
compute is supplied by an ops object so the same plan runs the device kernels in production and
NumPy stand-ins in the CPU tests.
"""

from __future__ import annotations

import math
from ctypes import byref as ctypes_byref, c_int64 as ctypes_i64
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
    """Sum a tensor over all ranks in place (no-op without a process group; a group of one still
    runs the collective, so the single-GPU tests exercise the NCCL path)."""
    if dist is None:
        import torch.distributed as dist  # noqa: F811
    if dist.is_available() and dist.is_initialized():
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


def sharded_fast_kronecker_regression(factors, b_rows, config, plan: ShardPlan, caches=None, dist=None,
                                      use_graph: bool = True):
    """fast_kronecker_regression (solvers.py:372-462) with b row-sharded over the ranks.

    Every rank holds both factors and its rows [lo, hi) of the n0 x n1 reshape of b (``b_rows``,
    device, (hi - lo) x n1).  The sketch and the preconditioner's eigendecompositions are computed
    replicated (identical NumPy-exact streams, so every rank draws the same sketch); each rank keeps
    the sampled rows whose factor-0 index it owns and gathers their b entries locally.  The
    Richardson loop then runs on the device with no host round trip (DeviceShardedLoop): per pass
    one apply-only launch of the persistent eigenbasis kernel on the rank's samples, one NCCL
    all-reduce of the d^2 partial, and a one-CTA kernel applying the reference's step, stopping and
    divergence rules; the whole loop is captured as one CUDA graph.  Returns (x, iterations,
    history); with one rank it is the single-GPU algorithm."""
    from . import _device as D
    from .kron import SparseDiagonal, _view_for
    from .solvers import _fast_sketch_dev

    if len(factors) != 2:
        raise ValueError("the row-sharded fast solve covers the two-factor problem")
    n1 = int(factors[1].shape[0])
    facs = [D.to_dev(a) for a in factors]
    sdiag, grams, s = _fast_sketch_dev(facs, config, caches)
    lo, hi = plan.rows
    keys = sdiag.indices
    own = (keys >= lo * n1) & (keys < hi * n1)
    li, lv = keys[own].contiguous(), sdiag.values[own].contiguous()
    local = SparseDiagonal._trusted(li, lv)
    b_at = b_rows.reshape(-1)[li - lo * n1].contiguous()
    (VL, wL), (VR, wR) = grams
    view = _view_for(facs, local)
    key = None
    if use_graph:
        import torch
        key = (_state.thread_key(), torch.cuda.current_stream().cuda_stream,
               tuple((a.data_ptr(), tuple(a.shape)) for a in facs), b_rows.data_ptr(), config, plan,
               view.nnz, view.u_left)
    loop = _state.cache_get(_SHARDED_LOOPS, key) if key is not None else None
    if loop is None:
        loop = DeviceShardedLoop(facs, view, VL, wL, VR, wR, b_at, config, dist)
        if key is not None:
            _state.cache_put(_SHARDED_LOOPS, key, loop, 4)
    else:  # same shapes: repack this call's rows into the captured loop's buffers and replay it
        loop.repack(view, VL, wL, VR, wR, b_at)
    return loop.run(use_graph)


_SHARDED_LOOPS: dict = {}


class DeviceShardedLoop:
    """The row-sharded Richardson loop of one rank on the device (ks_shard_loop_* in
    ks_richardson_persistent.cu).  Collective count and order are identical on every rank (a
    rank that has stopped keeps issuing its all-reduces on stale partials), and every decision is
    taken on identical all-reduced values, so the ranks stay in lockstep."""

    def __init__(self, facs, view, VL, wL, VR, wR, b_at, config, dist=None):
        import torch
        from . import _device as D, _lib
        self.torch, self.D, self.L = torch, D, _lib
        if dist is None:
            import torch.distributed as dist  # noqa: F811
        self.dist = dist
        self.view, self.config = view, config
        self.dL, self.dR = view.dL, view.dR
        self.VL, self.VR = VL.contiguous(), VR.contiguous()
        self.wL, self.wR = wL.contiguous(), wR.contiguous()
        sizes = (ctypes_i64 * 4)()
        _lib.call("ks_shard_loop_sizes", ctypes_byref(view.struct), sizes)
        self.Lp, self.Rp, self.part = D.empty(int(sizes[0])), D.empty(int(sizes[1])), D.empty(int(sizes[2]))
        self.plan_ws = torch.empty(int(sizes[3]), dtype=torch.uint8, device=D.dev())
        self.b_at = b_at
        # the apply launches (and a captured graph of them) read the row segments through this
        # loop-owned copy, so a repack for a new sketch of the same sizes keeps the graph valid
        self.seg = view.seg.clone()
        st = view.struct
        self.struct = _lib.SketchView(st.Lmat, st.ldl, st.dL, st.Rmat, st.ldr, st.dR, st.u_left, st.nnz,
                                      self.seg.data_ptr(), st.lrow, st.rrow, st.v)
        _lib.call("ks_shard_loop_pack", ctypes_byref(view.struct), None, D.p(self.VL), D.p(self.VR), D.p(b_at),
                  D.p(view.perm_arg()), D.p(self.Lp), D.p(self.Rp), D.p(self.plan_ws), D.stream())
        self.max_iters = config.effective_max_iters
        self.x = D.zeros(self.dL, self.dR)
        self.rhs = D.zeros(self.dL, self.dR)
        self.g = D.zeros(self.dL, self.dR)
        self.hist = D.zeros(max(1, self.max_iters))
        self.state = torch.zeros(4, dtype=torch.int32, device=D.dev())
        self.aux = D.zeros(1)

    def repack(self, view, VL, wL, VR, wR, b_at):
        """New sketch / eigendecomposition of the same sizes into the existing buffers."""
        D, L = self.D, self.L
        self.view = view  # keeps the new grouped-view buffers alive; the struct is passed by value
        self.VL.copy_(VL)
        self.VR.copy_(VR)
        self.wL.copy_(wL)
        self.wR.copy_(wR)
        self.b_at = b_at
        self.seg.copy_(view.seg)
        L.call("ks_shard_loop_pack", ctypes_byref(view.struct), None, D.p(self.VL), D.p(self.VR), D.p(b_at),
               D.p(view.perm_arg()), D.p(self.Lp), D.p(self.Rp), D.p(self.plan_ws), D.stream())

    def _pass(self, it):
        D, L, c = self.D, self.L, self.config
        L.call("ks_shard_loop_apply", ctypes_byref(self.struct), D.p(self.Lp), D.p(self.Rp), D.p(self.plan_ws),
               1 if it < 0 else 2, D.p(self.x), D.p(self.g), D.p(self.state), D.p(self.part), D.stream())
        allreduce_sum(self.g, self.dist)
        L.call("ks_shard_loop_update", it, D.p(self.g), D.p(self.x), D.p(self.rhs), D.p(self.wL), D.p(self.wR),
               self.dL, self.dR, float(c.lam), float(c.effective_damping), float(c.residual_tol), D.p(self.hist),
               D.p(self.state), D.p(self.aux), D.stream())

    def body(self):
        self.state.zero_()
        self.x.zero_()
        for it in range(-1, self.max_iters):
            self._pass(it)

    graph = None

    def run(self, use_graph: bool = True):
        torch = self.torch
        if use_graph and self.graph is None:
            try:
                self.body()  # warm-up (lazy initialisations, NCCL communicator) before capture
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    self.body()
                self.graph = graph
            except Exception:
                self.graph = None
        if use_graph and self.graph is not None:
            self.graph.replay()
        else:
            self.body()
        state = self.state.cpu().tolist()
        hist = self.hist[: state[3]].cpu().tolist()
        if state[1] == 2:
            from .errors import NumericalFailureError
            raise NumericalFailureError("Richardson iteration diverged", iterations=state[2],
                                        diagnostics={"residual_history": hist})
        return self.natural_x(), state[2], hist

    def replay(self):
        """Re-run the captured loop (benchmarking); returns nothing."""
        if self.graph is not None:
            self.graph.replay()
        else:
            self.body()

    def natural_x(self):
        """x = VL x' VR^T back in the natural (grouped) order."""
        D, L = self.D, self.L
        t = D.empty(self.dL, self.dR)
        out = D.empty(self.dL, self.dR)
        L.call("ks_gemm", self.dL, self.dR, self.dL, 1.0, D.p(self.VL), self.dL, 1, 0, D.p(self.x), self.dR, 1, 0,
               0.0, D.p(t), self.dR, 1, 0, 1, D.stream())
        L.call("ks_gemm", self.dL, self.dR, self.dR, 1.0, D.p(t), self.dR, 1, 0, D.p(self.VR), 1, self.dR, 0, 0.0,
               D.p(out), self.dR, 1, 0, 1, D.stream())
        return self.view.from_groups(out)


# Public entry points are gated (capture vs. concurrent solves, see _state.py).
_state.gate_names(globals(), ["sharded_kronmatmul_svd_solve", "sharded_fast_kronecker_regression"])
