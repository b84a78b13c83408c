"""World-size-2 gloo tests (CPU) of the row-sharded multi-GPU plan (paper_2209_04876_b200.distributed).

Local compute uses NumPy stand-ins (the oracle restatement) instead of the CUDA kernels; the plan,
sample ownership, collectives and the sharded Richardson loop are the production code."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_04876_b200.distributed import (ShardPlan, ShardedKron2, row_block_of_b, shard_sparse_diagonal,
                                               sharded_richardson, split_counts)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class NumpyOps:
    device = "cpu"

    def contract(self, L_rows, B_rows, R):
        return torch.from_numpy(L_rows.T @ B_rows @ R)

    def resid(self, L_rows, X, R, B_rows):
        e = L_rows @ X @ R.T - B_rows
        return float(np.sum(e * e))


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import kronsolve_oracle as O
        n, d = 64, 4
        facs, _ = O.synth_regression(n, d, 2, 0)
        rng = np.random.default_rng(3)
        b = rng.standard_normal(n * n)
        plan = ShardPlan(world, rank, n)
        lo, hi = plan.rows
        B_rows = row_block_of_b(b, plan, n).reshape(hi - lo, n)
        sk = ShardedKron2(plan, NumpyOps(), torch)
        T = sk.contract(facs[0], B_rows, facs[1]).numpy()
        X = rng.standard_normal((d, d))
        loss = sk.residual_sumsq(facs[0], X, facs[1], B_rows)
        # fast solve: replicated sketch, rank-local samples, sharded Richardson
        cfg = dict(eps=0.25, delta=0.1, lam=1e-2, alpha=1e-3, seed=5)  # s = 1600 < n^2: sketched path
        ref = O.fast_kronecker_regression(facs, b, **cfg)
        sd_idx, sd_val = ref.trace["sd_indices"], ref.trace["sd_values"]
        li, lv = shard_sparse_diagonal(plan, sd_idx, sd_val, n)
        pre = O.Preconditioner([O.factor_gram(a) for a in facs], cfg["lam"])

        def normal_local(x):
            xn = x.numpy()
            fwd = O.sketched_kron_apply(facs, li, lv, xn)
            return torch.from_numpy(O.sketched_kron_transpose_apply(facs, li, lv, fwd))

        rhs_local = torch.from_numpy(O.sketched_kron_transpose_apply(facs, li, lv, lv * b[li]))
        x, iters, hist = sharded_richardson(normal_local, lambda v: torch.from_numpy(pre.apply(v.numpy())),
                                            rhs_local, 1.0 - math.sqrt(cfg["eps"]),
                                            O.effective_max_iters(cfg["eps"]), 1e-9, torch, cfg["lam"])
        np.savez(os.path.join(out, f"rank{rank}.npz"), T=T, loss=loss, x=x.numpy(), iters=iters,
                 hist=np.asarray(hist), nlocal=len(li))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results(tmp_path_factory):
    # Results travel through files: a fork()ed multiprocessing.Manager leaves the parent's
    # OpenBLAS thread pool deadlocked for the tests that follow.
    world = 2
    out = str(tmp_path_factory.mktemp("multirank"))
    mp.spawn(_worker, args=(world, free_port(), out), nprocs=world, join=True)
    res = {}
    for r in range(world):
        with np.load(os.path.join(out, f"rank{r}.npz")) as z:
            res[r] = {k: (z[k].item() if z[k].ndim == 0 else z[k]) for k in z.files}
    return res


def test_shard_plan_partitions_rows():
    for n, w in [(64, 2), (65, 2), (7, 3), (16384, 8)]:
        spans = [ShardPlan(w, r, n).rows for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
        assert [hi - lo for lo, hi in spans] == split_counts(n, w)
        p = ShardPlan(w, 0, n)
        rows = np.arange(n)
        owners = p.owner_of_row(rows)
        for r, (lo, hi) in enumerate(spans):
            assert np.all(owners[lo:hi] == r)


def test_sharded_kron2_matches_unsharded(results):
    from oracle import kronsolve_oracle as O
    n, d = 64, 4
    facs, _ = O.synth_regression(n, d, 2, 0)
    rng = np.random.default_rng(3)
    b = rng.standard_normal(n * n)
    X = rng.standard_normal((d, d))
    T_ref = facs[0].T @ b.reshape(n, n) @ facs[1]
    loss_ref = float(np.sum((facs[0] @ X @ facs[1].T - b.reshape(n, n)) ** 2))
    for r in (0, 1):
        np.testing.assert_allclose(results[r]["T"], T_ref, rtol=1e-12, atol=1e-9)
        assert results[r]["loss"] == pytest.approx(loss_ref, rel=1e-12)


def test_sharded_richardson_matches_single_process(results):
    from oracle import kronsolve_oracle as O
    n, d = 64, 4
    facs, _ = O.synth_regression(n, d, 2, 0)
    b = np.random.default_rng(3).standard_normal(n * n)
    ref = O.fast_kronecker_regression(facs, b, eps=0.25, delta=0.1, lam=1e-2, alpha=1e-3, seed=5)
    assert ref.iterations > 0
    assert results[0]["nlocal"] + results[1]["nlocal"] == ref.trace["sd_indices"].size
    assert results[0]["nlocal"] > 0 and results[1]["nlocal"] > 0
    for r in (0, 1):
        assert results[r]["iters"] == ref.iterations
        np.testing.assert_allclose(results[r]["x"], ref.solution, rtol=1e-8, atol=1e-12)
    np.testing.assert_array_equal(results[0]["x"], results[1]["x"])  # identical decisions and iterates
