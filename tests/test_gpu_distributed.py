"""Row-sharded exact solve over NCCL on the GPU.  One B200 per test box: a
world-size-1 NCCL group runs the production collective path; the world-size-2 logic of the shard
plan is covered on CPU by tests/test_multirank_cpu.py."""

import os
import socket

import numpy as np
import pytest

from conftest import rel
from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_exact_solve_nccl_world1():
    import torch
    import torch.distributed as dist
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.distributed import ShardPlan, sharded_kronmatmul_svd_solve
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, d = 4096, 32
        facs, _ = O.synth_regression(n, d, 2, 0)
        b = np.random.default_rng(1).standard_normal(n * n)
        plan = ShardPlan(1, 0, n)
        lo, hi = plan.rows
        b_rows = torch.tensor(b.reshape(n, n)[lo:hi], device="cuda")
        x, loss = sharded_kronmatmul_svd_solve(facs, b_rows, 1e-3, plan)
        ref = K.kronmatmul_svd_solve(facs, b, 1e-3)
        assert rel(x, ref.solution) <= 1e-12
        assert loss == pytest.approx(ref.loss, rel=1e-12)
    finally:
        dist.destroy_process_group()


def test_sharded_row_blocks_sum_to_full_contraction():
    """Two row blocks contracted separately (what two ranks do) sum to the full K1 pass."""
    import torch
    from paper_2209_04876_b200.distributed import DeviceKron2Ops, ShardPlan
    n, d = 2048, 16
    facs, _ = O.synth_regression(n, d, 2, 3)
    b = np.random.default_rng(2).standard_normal((n, n))
    L, R = (torch.tensor(a, device="cuda") for a in facs)
    B = torch.tensor(b, device="cuda")
    ops = DeviceKron2Ops()
    parts = []
    for r in range(2):
        lo, hi = ShardPlan(2, r, n).rows
        parts.append(ops.contract(L[lo:hi], B[lo:hi], R))
    full = ops.contract(L, B, R)
    np.testing.assert_allclose((parts[0] + parts[1]).cpu().numpy(), full.cpu().numpy(), rtol=1e-11, atol=1e-9)
    np.testing.assert_allclose(full.cpu().numpy(), facs[0].T @ b @ facs[1], rtol=1e-10, atol=1e-8)


def test_sharded_fast_solve_nccl_world1():
    """The row-sharded fast solve (replicated sketch, rank-local samples, one d^2 NCCL all-reduce per
    Richardson pass, the loop on the device as one CUDA graph) over an NCCL world of one: same
    sketch and iterations as the single-GPU solve and the reference oracle, x and the step-norm
    history within 2x the reference's noise floor (the reductions run in another order); the
    captured graph and the eager launch sequence agree bit for bit."""
    import torch
    import torch.distributed as dist
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.distributed import ShardPlan, sharded_fast_kronecker_regression
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, d = 4096, 32
        facs, _ = O.synth_regression(n, d, 2, 0)
        b = np.random.default_rng(4).standard_normal(n * n)
        params = dict(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
        cfg = K.RegressionConfig(**params)
        plan = ShardPlan(1, 0, n)
        lo, hi = plan.rows
        b_rows = torch.tensor(b.reshape(n, n)[lo:hi], device="cuda")
        x, iters, hist = sharded_fast_kronecker_regression(facs, b_rows, cfg, plan)
        xe, iters_e, hist_e = sharded_fast_kronecker_regression(facs, b_rows, cfg, plan, use_graph=False)
        assert torch.equal(x, xe) and iters == iters_e and hist == hist_e
        ref = K.fast_kronecker_regression(facs, b, cfg)
        o = O.fast_kronecker_regression(facs, b, **params)
        assert iters == ref.iterations == o.iterations
        assert rel(x, o.solution) <= 2 * 4.6e-9  # c2 floor (tests/golden/floor.json)
        assert rel(x, ref.solution) <= 2 * 4.6e-9
        h = np.asarray(hist)
        assert np.max(np.abs(h / np.asarray(o.trace["history"]) - 1.0)) <= 2 * 2.3e-8
    finally:
        dist.destroy_process_group()
