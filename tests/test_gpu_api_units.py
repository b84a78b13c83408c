"""Unit-level behaviour of the smaller public entry points on the device: ridge leverage scores,
sample counts, Kronecker rows, the dense tensor helpers and the Tucker model metrics.  Each test
states a property the reference's own unit tests check (pkg/tests/test_leverage.py,
test_kron.py, test_tensor.py, test_tucker.py) and checks it on the CUDA path, against the oracle
where one exists."""

import itertools

import numpy as np
import pytest
import torch

from conftest import dense_kron
from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu


def _dense_ridge(a, lam):
    inv = np.linalg.pinv(a.T @ a + lam * np.eye(a.shape[1]))
    return np.einsum("ij,jk,ik->i", a, inv, a)


# ---------------------------------------------------------------------------
# ridge leverage scores (leverage.py:51-64)
# ---------------------------------------------------------------------------

def test_ridge_scores_known_answers():
    import paper_2209_04876_b200 as K
    ls = K.ridge_leverage_scores(K.compact_svd(np.eye(3)), 0.0)
    np.testing.assert_allclose(ls.scores, np.ones(3), atol=1e-12)
    assert ls.approx_factor == 1.0 and ls.lam == 0.0
    np.testing.assert_allclose(K.ridge_leverage_scores(K.compact_svd(np.eye(2)), 1.0).scores, [0.5, 0.5],
                               atol=1e-12)
    # rank-deficient 3x2: Gram + 3 I = diag(4, 7) gives (1/4, 4/7, 0)
    a = np.array([[1.0, 0.0], [0.0, 2.0], [0.0, 0.0]])
    np.testing.assert_allclose(K.ridge_leverage_scores(K.compact_svd(a), 3.0).scores, [0.25, 4 / 7, 0.0],
                               atol=1e-12)
    with pytest.raises(K.InvalidInputError):
        K.ridge_leverage_scores(K.compact_svd(np.ones((4, 2))), -1.0)
    zero = K.ridge_leverage_scores(K.compact_svd(np.zeros((5, 3))), 0.5)
    np.testing.assert_array_equal(zero.scores, np.zeros(5))


def test_ridge_scores_match_definition_and_oracle(rng):
    import paper_2209_04876_b200 as K
    for lam in (0.0, 0.3, 5.0):
        a = rng.standard_normal((40, 6))
        got = K.ridge_leverage_scores(K.compact_svd(a), lam).scores
        assert isinstance(got, np.ndarray)
        np.testing.assert_allclose(got, _dense_ridge(a, lam), atol=1e-10)
        np.testing.assert_allclose(got, O.ridge_scores(O.compact_svd(a), lam), atol=1e-13)
        # device in, device out
        dev = K.ridge_leverage_scores(K.compact_svd(torch.tensor(a, device="cuda")), lam).scores
        assert isinstance(dev, torch.Tensor) and dev.is_cuda
        np.testing.assert_allclose(dev.cpu().numpy(), got, rtol=0, atol=1e-15)


def test_ridge_scores_bounds_and_sums(rng):
    import paper_2209_04876_b200 as K
    for _ in range(10):
        a = rng.standard_normal((10, 3))
        lam = float(rng.uniform(0, 2))
        s = K.ridge_leverage_scores(K.compact_svd(a), lam).scores
        assert np.all(s <= 1.0 + 1e-10) and np.all(s >= -1e-12)
        sig = np.linalg.svd(a, compute_uv=False)
        assert abs(s.sum() - np.sum(sig ** 2 / (sig ** 2 + lam))) < 1e-10
    # unregularised scores of a rank-r matrix sum to r
    low = rng.standard_normal((9, 2)) @ rng.standard_normal((2, 4))
    assert abs(K.statistical_leverage_scores(low).scores.sum() - 2.0) < 1e-10


def test_appending_rows_never_increases_scores(rng):
    import paper_2209_04876_b200 as K
    a = rng.standard_normal((12, 4))
    for lam in (0.0, 0.5):
        before = K.ridge_leverage_scores(K.compact_svd(a), lam).scores
        grown = np.vstack([a, rng.standard_normal((5, 4))])
        after = K.ridge_leverage_scores(K.compact_svd(grown), lam).scores[:12]
        assert np.all(after <= before + 1e-12)


def test_exact_factor_scores_and_sample_counts(rng):
    import paper_2209_04876_b200 as K
    facs = [rng.standard_normal((30, 4)), rng.standard_normal((25, 3))]
    got = K.exact_factor_scores(facs)
    for a, ls in zip(facs, got):
        np.testing.assert_allclose(ls.scores, O.ridge_scores(O.compact_svd(a), 0.0), atol=1e-13)
    caches = [K.build_factor_cache(a) for a in facs]
    for x, y in zip(K.exact_factor_scores(facs, caches), got):
        np.testing.assert_allclose(x.scores, y.scores, atol=1e-13)
    for d in (1, 4, 64, 4096):
        for eps in (0.05, 0.1, 0.5):
            assert K.regression_sample_count(d, eps) == O.regression_sample_count(d, eps)
            assert K.spectral_sample_count(d, eps, 0.01) == O.spectral_sample_count(d, eps, 0.01)
            assert K.regression_sample_count(d, eps, beta=0.5) == O.regression_sample_count(d, eps, 0.5)


# ---------------------------------------------------------------------------
# Kronecker rows and the dense helpers (kron.py:193-205, tensor.py:110-213)
# ---------------------------------------------------------------------------

def test_kron_rows_match_dense_and_errors(rng):
    import paper_2209_04876_b200 as K
    facs = [rng.standard_normal((3, 2)), rng.standard_normal((4, 3)), rng.standard_normal((2, 2))]
    dense = dense_kron(facs)
    multi = np.stack(np.unravel_index(np.arange(24), (3, 4, 2)), axis=1)
    np.testing.assert_allclose(K.kron_rows(facs, multi), dense, rtol=0, atol=1e-13)
    dev = K.kron_rows([torch.tensor(a, device="cuda") for a in facs], torch.tensor(multi, device="cuda"))
    assert dev.is_cuda
    np.testing.assert_allclose(dev.cpu().numpy(), dense, rtol=0, atol=1e-13)
    # one multi-index given as a flat vector; negative indices wrap as in NumPy
    np.testing.assert_allclose(K.kron_rows(facs, np.array([-1, 0, -2])), dense[[2 * 8 + 0 * 2 + 0]],
                               atol=1e-13)
    with pytest.raises(IndexError):
        K.kron_rows(facs, np.array([[3, 0, 0]]))
    with pytest.raises(IndexError):
        K.kron_rows(facs, torch.tensor([[0, 0, -3]], device="cuda"))
    # the device is still healthy after the rejected indices
    torch.cuda.synchronize()
    np.testing.assert_allclose(K.kron_rows([np.eye(2), np.eye(2)], np.array([[0, 0]])), [[1.0, 0, 0, 0]])


def test_explicit_kron_and_column_stacking(rng):
    import paper_2209_04876_b200 as K
    np.testing.assert_array_equal(K.explicit_kron([np.eye(2), np.eye(3)]), np.eye(6))
    facs = [rng.standard_normal((3, 2)), rng.standard_normal((2, 4)), rng.standard_normal((2, 1))]
    np.testing.assert_allclose(K.explicit_kron(facs), dense_kron(facs), rtol=0, atol=1e-14)
    a = rng.standard_normal((3, 2))
    np.testing.assert_array_equal(K.explicit_kron([a]), a)
    with pytest.raises(K.errors.SizeGuardError):
        K.explicit_kron([np.ones((2, 2))] * 4, max_entries=100)
    with pytest.raises(K.InvalidInputError):
        K.explicit_kron([])
    # colvec(B C A^T) = (A kron B) colvec(C)
    A, B, C = rng.standard_normal((3, 4)), rng.standard_normal((2, 3)), rng.standard_normal((3, 4))
    np.testing.assert_allclose(K.stack_columns(B @ C @ A.T), K.explicit_kron([A, B]) @ K.stack_columns(C),
                               atol=1e-12)
    m = rng.standard_normal((4, 2))
    assert np.array_equal(K.unstack_columns(K.stack_columns(m), (4, 2)), m)
    md = torch.tensor(m, device="cuda")
    assert torch.equal(K.unstack_columns(K.stack_columns(md), (4, 2)), md)
    with pytest.raises(K.InvalidInputError):
        K.unstack_columns(np.ones(5), (2, 3))


def test_unfold_fold_vectorize(rng):
    import paper_2209_04876_b200 as K
    x = np.array([1.0, 2.0, 3.0])
    m = K.unfold(x, 0)
    assert m.shape == (3, 1) and np.array_equal(m[:, 0], x)
    x = rng.standard_normal((2, 3, 4))
    for mode in range(3):
        m = K.unfold(x, mode)
        rest = [r for k, r in enumerate(x.shape) if k != mode]
        for j, idx in enumerate(itertools.product(*[range(r) for r in rest])):
            full = list(idx)
            full.insert(mode, slice(None))
            assert np.array_equal(m[:, j], x[tuple(full)])
        assert np.array_equal(K.fold(m, x.shape, mode), x)
        xd = torch.tensor(x, device="cuda")
        assert torch.equal(K.fold(K.unfold(xd, mode), x.shape, mode), xd)
    v = K.vectorize(x)
    assert np.array_equal(v, x.reshape(-1)) and np.array_equal(K.devectorize(v, x.shape), x)
    with pytest.raises(K.InvalidInputError):
        K.devectorize(np.ones(5), (2, 3))
    with pytest.raises(K.InvalidInputError):
        K.fold(np.ones((2, 5)), (2, 3), 0)


def test_mode_products(rng):
    import paper_2209_04876_b200 as K
    x = rng.standard_normal((2, 3, 4))
    np.testing.assert_array_equal(K.n_mode_product(x, np.eye(3), 1), x)
    v = rng.standard_normal(4)
    a = rng.standard_normal((2, 4))
    np.testing.assert_allclose(K.n_mode_product(v, a, 0), a @ v, atol=1e-13)
    y = rng.standard_normal((2, 3, 2))
    b = rng.standard_normal((4, 3))
    out = K.n_mode_product(y, b, 1)
    assert out.shape == (2, 4, 2)
    np.testing.assert_allclose(out, np.einsum("itk,jt->ijk", y, b), atol=1e-13)
    with pytest.raises(K.InvalidInputError):
        K.n_mode_product(rng.standard_normal((2, 3)), np.eye(4), 1)
    # vec(G x_1 A1 x_2 A2 x_3 A3) = (A1 kron A2 kron A3) vec(G) in row-major vectorisation
    g = rng.standard_normal((2, 3, 2))
    facs = [rng.standard_normal((3, 2)), rng.standard_normal((2, 3)), rng.standard_normal((4, 2))]
    expanded = K.multi_mode_product(g, facs)
    np.testing.assert_allclose(K.vectorize(expanded), dense_kron(facs) @ g.reshape(-1), atol=1e-12)


def test_pseudo_inverse_and_reciprocal(rng):
    import paper_2209_04876_b200 as K
    np.testing.assert_allclose(K.pseudo_inverse(np.eye(3)), np.eye(3), atol=1e-14)
    np.testing.assert_allclose(K.pseudo_inverse(np.diag([2.0, 4.0])), np.diag([0.5, 0.25]), atol=1e-14)
    a = rng.standard_normal((6, 3))
    np.testing.assert_allclose(K.pseudo_inverse(a) @ a, np.eye(3), atol=1e-12)
    a = rng.standard_normal((5, 2)) @ rng.standard_normal((2, 4))
    p = K.pseudo_inverse(a)
    np.testing.assert_allclose(a @ p @ a, a, atol=1e-8)
    np.testing.assert_allclose(p @ a @ p, p, atol=1e-8)
    np.testing.assert_allclose((a @ p).T, a @ p, atol=1e-8)
    np.testing.assert_allclose((p @ a).T, p @ a, atol=1e-8)
    np.testing.assert_allclose(p, np.linalg.pinv(a, rcond=1e-10), atol=1e-10)
    d = np.array([2.0, 0.0, -1.0, 0.5])
    np.testing.assert_array_equal(K.pseudo_reciprocal(d), [0.5, 0.0, 0.0, 2.0])
    dd = K.pseudo_reciprocal(torch.tensor(d, device="cuda"))
    assert dd.is_cuda and np.array_equal(dd.cpu().numpy(), [0.5, 0.0, 0.0, 2.0])


# ---------------------------------------------------------------------------
# Tucker model metrics (tucker.py:45-101)
# ---------------------------------------------------------------------------

def _model(K, rng, shape, rank, lam=0.0):
    return K.TuckerModel(core=rng.standard_normal(tuple(rank)),
                         factors=[rng.standard_normal((i, r)) for i, r in zip(shape, rank)], lam=lam)


def test_tucker_model_metrics(rng):
    import paper_2209_04876_b200 as K
    with pytest.raises(K.InvalidInputError):
        K.TuckerModel(core=rng.standard_normal((2, 2)), factors=[rng.standard_normal((4, 2))])
    with pytest.raises(K.InvalidInputError):
        K.TuckerModel(core=rng.standard_normal((3, 2)),
                      factors=[rng.standard_normal((2, 3)), rng.standard_normal((4, 2))])
    m = _model(K, rng, (4, 3, 5), (2, 2, 2))
    m.core = np.zeros_like(m.core)
    x = rng.standard_normal((4, 3, 5))
    assert np.all(K.reconstruct(m) == 0.0)
    assert K.relative_error(m, x) == pytest.approx(1.0)
    # rank-one hand case
    u, v, w = np.array([1.0, 2.0]), np.array([3.0, -1.0]), np.array([0.5, 4.0])
    core = np.zeros((2, 2, 2))
    core[0, 0, 0] = 1.0
    facs = [np.column_stack([t, np.zeros(2)]) for t in (u, v, w)]
    np.testing.assert_allclose(K.reconstruct(K.TuckerModel(core=core, factors=facs)),
                               np.einsum("i,j,k->ijk", u, v, w), atol=1e-14)
    m = _model(K, rng, (4, 3, 5), (2, 2, 2))
    assert K.relative_error(m, K.reconstruct(m)) == pytest.approx(0.0, abs=1e-14)
    m = _model(K, rng, (4, 3, 2), (2, 2, 2), lam=0.7)
    x = rng.standard_normal((4, 3, 2))
    err = float(np.sum((K.reconstruct(m) - x) ** 2))
    frob = float(np.sum(m.core ** 2)) + sum(float(np.sum(a ** 2)) for a in m.factors)
    assert K.regularized_loss(m, x) == pytest.approx(err + 0.7 * frob, rel=1e-12)
    m = _model(K, rng, (4, 3), (2, 2), lam=1.0)
    m.core = np.zeros_like(m.core)
    m.factors = [np.zeros_like(a) for a in m.factors]
    x = rng.standard_normal((4, 3))
    assert K.regularized_loss(m, x) == pytest.approx(float(np.sum(x ** 2)), rel=1e-12)


# ---------------------------------------------------------------------------
# exact solve properties and the generic Richardson loop on device tensors (solvers.py:201-248)
# ---------------------------------------------------------------------------

def test_exact_solve_residual_orthogonality_and_loss(rng):
    import paper_2209_04876_b200 as K
    facs = [rng.standard_normal((8, 3)), rng.standard_normal((6, 2))]
    b = rng.standard_normal(48)
    k = dense_kron(facs)
    rep = K.kronmatmul_svd_solve(facs, b, 0.0)
    assert np.linalg.norm(k.T @ (k @ rep.solution - b)) <= 1e-8 * np.linalg.norm(b)
    rep = K.kronmatmul_svd_solve(facs, b, 0.1)
    assert rep.loss == pytest.approx(K.ridge_loss(facs, rep.solution, b, 0.1), abs=1e-10)
    want = np.sum((k @ rep.solution - b) ** 2) + 0.1 * np.sum(rep.solution ** 2)
    assert rep.loss == pytest.approx(want, rel=1e-12)


def test_richardson_on_device_tensors(rng):
    import paper_2209_04876_b200 as K
    a = torch.tensor(rng.standard_normal((8, 3)), device="cuda")
    b = torch.tensor(rng.standard_normal(8), device="cuda")
    ata = a.T @ a
    m = 2.0 * ata
    minv = torch.linalg.inv(m)
    xs = torch.linalg.lstsq(a.cpu(), b.cpu()[:, None]).solution[:, 0].cuda()
    its = []
    x, it = K.richardson_solve(lambda v: ata @ v, lambda v: minv @ v, a.T @ b, 1.0,
                               K.RegressionConfig(eps=0.25, max_richardson_iters=10, residual_tol=1e-300),
                               callback=lambda xk: its.append(xk.clone()))
    assert x.is_cuda and it == 10
    e0 = float(torch.sqrt(xs @ m @ xs))
    for j, xk in enumerate(its, start=1):
        d = xk - xs
        assert float(torch.sqrt(d @ m @ d)) <= 0.5 ** j * e0 * (1 + 1e-10) + 1e-12
