"""Acceptance properties on the CUDA path (the reference's pkg/tests/test_acceptance.py checks,
restated): the Kronecker leverage law, random-instance equivalence of the fast multiplies with
dense products, the (1+eps) approximation contract over 100 seeds, exact-solver agreement, the
Woodbury workspace, Tucker ALS monotonicity / interpolation and sketched-ALS quality.  Inputs are
seeded NumPy draws (the Tucker tensors come from the oracle's generator, input generation only)."""

import itertools
import math
from functools import reduce

import numpy as np
import pytest

from conftest import dense_kron
from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu


def K():
    import paper_2209_04876_b200 as k
    return k


def _dense_ridge(a, lam):
    inv = np.linalg.pinv(a.T @ a + lam * np.eye(a.shape[1]))
    return np.einsum("ij,jk,ik->i", a, inv, a)


def test_kronecker_leverage_law():
    rng = np.random.default_rng(101)
    worst_stat = worst_ridge = 0.0
    for _ in range(50):
        order = int(rng.integers(2, 4))
        shapes = [(int(rng.integers(2, 7)), int(rng.integers(1, 5))) for _ in range(order)]
        shapes = [(max(r, c), c) for r, c in shapes]
        facs = [rng.standard_normal(s) for s in shapes]
        k = dense_kron(facs)
        sampler = K().build_product_sampler([K().statistical_leverage_scores(a) for a in facs])
        joint = reduce(np.kron, [np.asarray(p.cpu() if hasattr(p, "cpu") else p)
                                 for p in sampler.per_factor_probabilities])
        full = K().statistical_leverage_scores(k).normalized()
        worst_stat = max(worst_stat, float(np.max(np.abs(joint - np.asarray(full)))))
        # ridge scores of the Kronecker product by summation over factor singular triples
        lam = float(rng.uniform(0.01, 1.0))
        svds = [K().compact_svd(a, rank_tol=0.0) for a in facs]
        got = np.zeros(k.shape[0])
        for flat, rows in enumerate(itertools.product(*[range(s[0]) for s in shapes])):
            total = 0.0
            for t in itertools.product(*[range(sv.rank) for sv in svds]):
                sig2 = math.prod(float(svds[n].sigma[t[n]]) ** 2 for n in range(order))
                u2 = math.prod(float(svds[n].u[rows[n], t[n]]) for n in range(order)) ** 2
                total += sig2 / (sig2 + lam) * u2
            got[flat] = total
        worst_ridge = max(worst_ridge, float(np.max(np.abs(got - _dense_ridge(k, lam)))))
        # and the device scores of the dense product itself
        dev = K().ridge_leverage_scores(K().compact_svd(k), lam).scores
        worst_ridge = max(worst_ridge, float(np.max(np.abs(dev - _dense_ridge(k, lam)))))
    assert worst_stat <= 1e-9 and worst_ridge <= 1e-9


def test_fast_multiply_random_instances():
    rng = np.random.default_rng(202)
    worst = 0.0
    for _ in range(100):
        order = int(rng.integers(1, 5))
        while True:
            shapes = [(int(rng.integers(1, 9)), int(rng.integers(1, 5))) for _ in range(order)]
            if math.prod(s[0] for s in shapes) <= 2000:
                break
        facs = [rng.standard_normal(s) for s in shapes]
        dense = dense_kron(facs)
        n_rows, n_cols = dense.shape
        b = rng.standard_normal((n_cols, 2))
        want = dense @ b
        worst = max(worst, np.max(np.abs(K().kron_mat_mul(facs, b) - want)) / max(1.0, np.max(np.abs(want))))
        sq = [rng.standard_normal((s[1], s[1])) for s in shapes]
        c = rng.standard_normal(n_cols)
        want = dense_kron(sq) @ c
        worst = max(worst, np.max(np.abs(K().kron_vec_square(sq, c) - want)) / max(1.0, np.max(np.abs(want))))
        nnz = int(rng.integers(1, max(2, n_rows // 3)))
        idx = np.sort(rng.choice(n_rows, size=nnz, replace=False)).astype(np.int64)
        vals = rng.standard_normal(nnz)
        sd = K().SparseDiagonal(indices=idx, values=vals)
        cv = rng.standard_normal(n_cols)
        want = vals * (dense @ cv)[idx]
        got = K().sketched_kron_apply(facs, sd, cv)
        worst = max(worst, np.max(np.abs(got - want), initial=0.0) / max(1.0, np.max(np.abs(want), initial=0.0)))
        bv = rng.standard_normal(nnz)
        want = dense[idx].T @ (vals * bv)
        got = K().sketched_kron_transpose_apply(facs, sd, bv)
        worst = max(worst, np.max(np.abs(got - want)) / max(1.0, np.max(np.abs(want))))
    assert worst <= 1e-10


def test_approximation_contract_100_seeds():
    eps, delta, lam = 0.25, 0.05, 1e-3
    hits = 0
    for seed in range(100):
        rng = np.random.default_rng(seed)
        facs = [rng.normal(1.0, math.sqrt(1e-3), (20, 3)) for _ in range(2)]
        b = rng.standard_normal(400)
        rep = K().fast_kronecker_regression(facs, b, K().RegressionConfig(eps=eps, delta=delta, lam=lam, seed=seed))
        opt = K().kronmatmul_svd_solve(facs, b, lam)
        hits += rep.loss <= (1 + eps) * opt.loss + 1e-12
    assert hits >= 95


def test_exact_solver_agreement_50_instances():
    rng = np.random.default_rng(303)
    worst = 0.0
    for i in range(50):
        order = int(rng.integers(1, 4))
        shapes = [(int(rng.integers(2, 8)), int(rng.integers(1, 4))) for _ in range(order)]
        shapes = [(max(r, c), c) for r, c in shapes]
        facs = [rng.standard_normal(s) for s in shapes]
        b = rng.standard_normal(math.prod(s[0] for s in shapes))
        lam = (0.0, 1e-3, 1.0)[i % 3]
        r1 = K().naive_normal_solve(facs, b, lam)
        r2 = K().kronmatmul_svd_solve(facs, b, lam)
        worst = max(worst, np.linalg.norm(r1.solution - r2.solution) / max(1.0, np.linalg.norm(r2.solution)))
        r3 = O.kronmatmul_svd_solve(facs, b, lam)
        worst = max(worst, np.linalg.norm(r3.solution - r2.solution) / max(1.0, np.linalg.norm(r3.solution)))
    assert worst <= 1e-8


def test_woodbury_workspace_30_cores():
    worst = 0.0
    for seed in range(30):
        rng = np.random.default_rng(seed + 500)
        rank = tuple(int(r) for r in rng.integers(2, 5, size=3))
        shape = tuple(r + int(rng.integers(1, 4)) for r in rank)
        lam = float(rng.uniform(0.0, 0.5))
        model = K().TuckerModel(core=rng.standard_normal(rank),
                                factors=[rng.standard_normal((i, r)) for i, r in zip(shape, rank)], lam=lam)
        n = int(rng.integers(0, 3))
        ws = K().build_factor_workspace(model, n, eps=0.25, lam=lam)
        kd = dense_kron([a for k, a in enumerate(model.factors) if k != n])
        g = K().unfold(model.core, n)
        gp = np.linalg.pinv(g)
        nmat = np.eye(g.shape[1]) - g.T @ np.linalg.pinv(g.T)
        mp = np.linalg.pinv(kd.T @ kd + lam * gp @ gp.T + float(ws.penalty_weight) * nmat)
        for _ in range(3):
            z = rng.standard_normal(g.shape[1])
            want = mp @ z
            got = np.asarray(ws.apply(z))
            worst = max(worst, np.linalg.norm(got - want) / max(1.0, np.linalg.norm(want)))
    assert worst <= 1e-8


def test_tucker_monotone_and_full_rank_interpolation():
    for seed in range(20):
        x = np.random.default_rng(seed + 700).standard_normal((8, 8, 8))
        _, rep = K().tucker_als(x, (3, 3, 3), lam=1e-2, sweeps=3, solver_mode="exact",
                                config=K().RegressionConfig(seed=seed))
        for a, b in zip(rep.step_losses, rep.step_losses[1:]):
            assert b <= a * (1 + 1e-10) + 1e-10
    x = np.random.default_rng(42).standard_normal((8, 8, 8))
    _, rep = K().tucker_als(x, (8, 8, 8), lam=0.0, sweeps=1, solver_mode="exact",
                            config=K().RegressionConfig(seed=0))
    assert rep.rre <= 1e-8


def test_sketched_als_quality_10_seeds():
    hits = 0
    for seed in range(10):
        x = O.synth_tucker((20, 20, 20), (4, 4, 4), 0.01, seed, relative=True)
        _, exact = K().tucker_als(x, (4, 4, 4), lam=0.0, sweeps=5, solver_mode="exact",
                                  config=K().RegressionConfig(seed=seed))
        _, fast = K().tucker_als(x, (4, 4, 4), lam=0.0, sweeps=5, solver_mode="fast",
                                 config=K().RegressionConfig(eps=0.25, delta=0.05, seed=seed))
        hits += abs(fast.rre - exact.rre) <= 0.05 * max(exact.rre, 1e-12)
    assert hits >= 9
