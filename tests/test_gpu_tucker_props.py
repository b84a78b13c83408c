"""Tucker-ALS properties on the CUDA path (the reference's pkg/tests/test_tucker.py checks,
restated): core update projection / shrinkage / fast-vs-exact quality, the naive factor update's
per-row normal equations, and the ALS driver's interpolation, rank-one recovery, stopping rule,
report structure, fast-mode quality and the shared-sketch option."""

import numpy as np
import pytest

from conftest import dense_kron
from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu


def K():
    import paper_2209_04876_b200 as k
    return k


def _model(rng, shape, rank, lam=0.0):
    return K().TuckerModel(core=rng.standard_normal(tuple(rank)),
                           factors=[rng.standard_normal((i, r)) for i, r in zip(shape, rank)], lam=lam)


def _design(model, n):
    others = [np.asarray(a) for k, a in enumerate(model.factors) if k != n]
    return dense_kron(others) @ np.asarray(K().unfold(model.core, n)).T


def _row_loss(design, y, b, lam):
    return float(np.sum((design @ y - b) ** 2) + lam * np.sum(y ** 2))


def test_core_update_projection_and_shrinkage(rng):
    qs = [np.linalg.qr(rng.standard_normal((4, 4)))[0] for _ in range(3)]
    x = rng.standard_normal((4, 4, 4))
    core = K().core_update(K().TuckerModel(core=np.zeros((4, 4, 4)), factors=qs), x, mode="exact")
    np.testing.assert_allclose(core, K().multi_mode_product(x, [q.T for q in qs]), atol=1e-10)
    m = _model(rng, (5, 4), (2, 2))
    x = rng.standard_normal((5, 4))
    plain = K().core_update(m, x, mode="exact")
    m.lam = 1e12
    assert np.linalg.norm(K().core_update(m, x, mode="exact")) <= 1e-9 * np.linalg.norm(plain)


def test_fast_core_update_quality_50_seeds():
    hits = 0
    for seed in range(50):
        x = np.random.default_rng(seed + 300).standard_normal((10, 10, 10))
        model, _ = K().tucker_als(x, (3, 3, 3), lam=1e-3, sweeps=1, solver_mode="exact",
                                  config=K().RegressionConfig(seed=seed))
        caches = [K().build_factor_cache(a) for a in model.factors]
        cfg = K().RegressionConfig(eps=0.25, delta=0.05, lam=1e-3, seed=seed, alpha=2e-4)
        fast = K().core_update(model, x, mode="fast", config=cfg, caches=caches)
        exact = K().core_update(model, x, mode="exact")
        lf = K().ridge_loss(model.factors, K().vectorize(fast), K().vectorize(x), 1e-3)
        le = K().ridge_loss(model.factors, K().vectorize(exact), K().vectorize(x), 1e-3)
        hits += lf <= (1 + cfg.eps) * le
    assert hits >= 48


def test_naive_factor_update_normal_equations(rng):
    m = _model(rng, (5, 4, 3), (2, 2, 2))
    x = K().reconstruct(m)
    before = K().regularized_loss(m, x)
    m.factors[1] = K().naive_factor_update(m, x, 1)
    assert K().regularized_loss(m, x) <= before + 1e-10
    m = _model(rng, (5, 4, 3), (2, 2, 2), lam=0.3)
    x = rng.standard_normal((5, 4, 3))
    new = K().naive_factor_update(m, x, 0)
    design, b = _design(m, 0), np.asarray(K().unfold(x, 0))
    for i in range(5):
        grad = design.T @ (design @ new[i] - b[i]) + 0.3 * new[i]
        assert np.linalg.norm(grad) <= 1e-8 * max(1.0, np.linalg.norm(b[i]))
    m = _model(rng, (6, 5), (2, 3), lam=0.05)
    x = rng.standard_normal((6, 5))
    new = K().naive_factor_update(m, x, 0)
    design, b = _design(m, 0), np.asarray(K().unfold(x, 0))
    for i in range(6):
        want = np.linalg.solve(design.T @ design + 0.05 * np.eye(2), design.T @ b[i])
        np.testing.assert_allclose(new[i], want, atol=1e-8)


def test_als_interpolation_rank_one_and_stop(rng):
    x = rng.standard_normal((4, 3, 5))
    _, rep = K().tucker_als(x, (4, 3, 5), lam=0.0, sweeps=1, solver_mode="exact",
                            config=K().RegressionConfig(seed=0))
    assert rep.rre <= 1e-8
    u, v, w = rng.standard_normal(6), rng.standard_normal(5), rng.standard_normal(4)
    _, rep = K().tucker_als(np.einsum("i,j,k->ijk", u, v, w), (1, 1, 1), lam=0.0, sweeps=5,
                            solver_mode="exact", config=K().RegressionConfig(seed=3))
    assert rep.rre <= 1e-6
    u = rng.standard_normal(5)
    _, rep = K().tucker_als(np.outer(u, u), (1, 1), lam=0.0, sweeps=50, solver_mode="exact",
                            config=K().RegressionConfig(seed=0), loss_change_tol=1e-6)
    assert len(rep.sweep_losses) < 50


def test_als_report_structure_and_validation(rng):
    x = rng.standard_normal((5, 4, 3))
    _, rep = K().tucker_als(x, (2, 2, 2), lam=0.1, sweeps=2, solver_mode="exact",
                            config=K().RegressionConfig(seed=0))
    assert isinstance(rep, K().AlsReport)
    assert len(rep.sweep_losses) == 2 and len(rep.sweep_rres) == 2
    assert len(rep.step_losses) == 1 + 2 * 4
    assert rep.rre == pytest.approx(rep.sweep_rres[-1])
    x = rng.standard_normal((4, 4))
    for kw in (dict(core_shape=(5, 2), sweeps=1), dict(core_shape=(2, 2), sweeps=0),
               dict(core_shape=(2, 2), solver_mode="bogus")):
        with pytest.raises(K().InvalidInputError):
            K().tucker_als(x, **kw)


def test_fast_mode_reaches_exact_quality():
    x = O.synth_tucker((20, 20, 20), (4, 4, 4), 0.01, seed=0, relative=True)
    _, exact = K().tucker_als(x, (4, 4, 4), lam=0.0, sweeps=5, solver_mode="exact",
                              config=K().RegressionConfig(seed=0))
    _, fast = K().tucker_als(x, (4, 4, 4), lam=0.0, sweeps=5, solver_mode="fast",
                             config=K().RegressionConfig(eps=0.25, delta=0.05, seed=0, alpha=7e-5))
    assert fast.rre <= 2.0 * exact.rre
    assert fast.rre <= 3e-4


def test_shared_sketch_update_quality(rng):
    x = rng.standard_normal((8, 8, 8))
    model, _ = K().tucker_als(x, (2, 2, 2), lam=1e-3, sweeps=1, solver_mode="exact",
                              config=K().RegressionConfig(seed=3))
    cfg = K().RegressionConfig(eps=0.25, delta=0.05, lam=1e-3, seed=3, alpha=5e-5, share_row_sketch=True)
    fast = K().fast_factor_matrix_update(model, x, 0, cfg)
    naive = K().naive_factor_update(model, x, 0)
    design, b = _design(model, 0), np.asarray(K().unfold(x, 0))
    for i in range(8):
        lf = _row_loss(design, fast[i], b[i], 1e-3)
        ln = _row_loss(design, naive[i], b[i], 1e-3)
        assert lf <= 3.0 * ln  # one sketch reused for every row: the reference's looser bound
