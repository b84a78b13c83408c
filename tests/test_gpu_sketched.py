"""Sketched Kronecker operator vs the oracle and dense definitions (reference test_kron.py:149-235)."""

import numpy as np
import pytest

from conftest import dense_kron
from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu


def rsd(rng, n_rows, nnz):
    import paper_2209_04876_b200 as K
    idx = np.sort(rng.choice(n_rows, size=nnz, replace=False)).astype(np.int64)
    return K.SparseDiagonal(indices=idx, values=rng.standard_normal(nnz))


@pytest.mark.parametrize("shapes,nnz", [([(4, 2), (3, 2), (4, 3)], 7), ([(5, 3), (6, 2)], 5), ([(7, 2)], 3),
                                        ([(2, 3), (3, 2), (2, 2), (2, 2)], 9), ([(16, 4), (9, 16)], 20),
                                        ([(30, 16), (20, 16), (10, 4)], 300), ([(50, 4), (40, 16)], 400)])
def test_sparse_vs_dense(rng, shapes, nnz):
    import paper_2209_04876_b200 as K
    facs = [rng.standard_normal(s) for s in shapes]
    dense = dense_kron(facs)
    sd = rsd(rng, dense.shape[0], nnz)
    s = np.zeros((dense.shape[0],) * 2)
    s[sd.indices, sd.indices] = sd.values
    c = rng.standard_normal(dense.shape[1])
    np.testing.assert_allclose(K.sketched_kron_apply(facs, sd, c), (s @ dense @ c)[sd.indices], atol=1e-11)
    bv = rng.standard_normal(nnz)
    bfull = np.zeros(dense.shape[0])
    bfull[sd.indices] = bv
    np.testing.assert_allclose(K.sketched_kron_transpose_apply(facs, sd, bv), dense.T @ s @ bfull, atol=1e-11)


def test_empty_single_zero_fallback(rng):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.errors import InvalidInputError
    facs = [rng.standard_normal((3, 2)), rng.standard_normal((2, 2))]
    sd = K.SparseDiagonal(indices=np.array([], dtype=np.int64), values=np.array([]))
    assert K.sketched_kron_apply(facs, sd, rng.standard_normal(4)).size == 0
    np.testing.assert_array_equal(K.sketched_kron_transpose_apply(facs, sd, np.array([])), np.zeros(4))
    facs = [rng.standard_normal((4, 2)), rng.standard_normal((3, 3))]
    dense = dense_kron(facs)
    sd1 = K.SparseDiagonal(indices=np.array([7]), values=np.array([2.5]))
    c = rng.standard_normal(6)
    np.testing.assert_allclose(K.sketched_kron_apply(facs, sd1, c), [2.5 * dense[7] @ c], atol=1e-12)
    np.testing.assert_array_equal(K.sketched_kron_apply(facs, rsd(rng, 12, 4), np.zeros(6)), np.zeros(4))
    facs2 = [rng.standard_normal((4, 2)), rng.standard_normal((3, 2))]
    d2 = dense_kron(facs2)
    sdf = rsd(rng, 12, 10)  # nnz > rows/2: dense fallback
    s = np.zeros((12, 12)); s[sdf.indices, sdf.indices] = sdf.values
    c2 = rng.standard_normal(4)
    np.testing.assert_allclose(K.sketched_kron_apply(facs2, sdf, c2), (s @ d2 @ c2)[sdf.indices], atol=1e-12)
    with pytest.raises(InvalidInputError):
        K.sketched_kron_apply([rng.standard_normal((2, 2))] * 2, K.SparseDiagonal(np.array([5]), np.array([1.0])),
                              rng.standard_normal(4))


def test_adjoint_and_linearity(rng):
    import paper_2209_04876_b200 as K
    facs = [rng.standard_normal((40, 8)), rng.standard_normal((30, 6))]
    sd = rsd(rng, 1200, 250)
    c1, c2 = rng.standard_normal(48), rng.standard_normal(48)
    a, b = 0.7, -1.3
    np.testing.assert_allclose(K.sketched_kron_apply(facs, sd, a * c1 + b * c2),
                               a * K.sketched_kron_apply(facs, sd, c1) + b * K.sketched_kron_apply(facs, sd, c2),
                               atol=1e-10)
    bb = rng.standard_normal(250)
    lhs = K.sketched_kron_apply(facs, sd, c1) @ bb
    rhs = c1 @ K.sketched_kron_transpose_apply(facs, sd, bb)
    assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))


@pytest.mark.parametrize("n,d", [(1024, 16), (4096, 32), (16384, 64)])
def test_sketched_ops_on_baseline_sketch(golden, n, d):
    import paper_2209_04876_b200 as K
    g = golden({1024: "c1", 4096: "c2", 16384: "c3"}[n])
    facs, _ = O.synth_regression(n, d, 2, 0)
    sd = K.SparseDiagonal(g["sd_indices"], g["sd_values"])
    rng = np.random.default_rng(1)
    c = rng.standard_normal(d * d)
    want = O.sketched_kron_apply(facs, g["sd_indices"], g["sd_values"], c)
    np.testing.assert_allclose(K.sketched_kron_apply(facs, sd, c), want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
    bv = rng.standard_normal(g["sd_indices"].size)
    want_t = O.sketched_kron_transpose_apply(facs, g["sd_indices"], g["sd_values"], bv)
    np.testing.assert_allclose(K.sketched_kron_transpose_apply(facs, sd, bv), want_t, rtol=1e-12,
                               atol=1e-12 * np.abs(want_t).max())


def test_preconditioner_dense(rng):
    import paper_2209_04876_b200 as K
    facs = [rng.standard_normal((6, 2)), rng.standard_normal((5, 3))]
    pre = K.build_kron_preconditioner([K.factor_gram(a) for a in facs], 0.3)
    k = dense_kron(facs)
    x = rng.standard_normal(6)
    np.testing.assert_allclose(pre.apply(x), np.linalg.inv(k.T @ k + 0.3 * np.eye(6)) @ x, atol=1e-10)
    a = np.zeros((4, 2)); a[:, 0] = rng.standard_normal(4)
    pre = K.build_kron_preconditioner([K.factor_gram(a)], 0.0)
    x = rng.standard_normal(2)
    np.testing.assert_allclose(pre.apply(x), np.linalg.pinv(a.T @ a) @ x, atol=1e-10)
    facs3 = [rng.standard_normal((5, 2)), rng.standard_normal((4, 2)), rng.standard_normal((3, 2))]
    pre3 = K.build_kron_preconditioner([K.factor_gram(a) for a in facs3], 0.1)
    k3 = dense_kron(facs3)
    x3 = rng.standard_normal(8)
    np.testing.assert_allclose(pre3.apply(x3), np.linalg.inv(k3.T @ k3 + 0.1 * np.eye(8)) @ x3, atol=1e-10)
