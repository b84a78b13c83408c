"""Dense device primitives vs the oracle / dense definitions (reference test_kron.py,
test_tensor.py, test_solvers.py patterns)."""

import math

import numpy as np
import pytest
import torch

from conftest import dense_kron, rel

pytestmark = pytest.mark.gpu


def test_gemm_strided_batched(rng):
    from paper_2209_04876_b200 import _lib, _device as D
    a = rng.standard_normal((3, 70, 33))
    b = rng.standard_normal((3, 33, 45))
    A, B = D.to_dev(a), D.to_dev(b)
    C = D.empty(3, 70, 45)
    _lib.call("ks_gemm", 70, 45, 33, 1.0, D.p(A), 33, 1, 70 * 33, D.p(B), 45, 1, 33 * 45, 0.0, D.p(C), 45, 1, 70 * 45,
              3, D.stream())
    np.testing.assert_allclose(C.cpu().numpy(), a @ b, rtol=1e-13, atol=1e-13)


def test_gemm_tn_tall(rng):
    from paper_2209_04876_b200 import _lib, _device as D
    a = rng.standard_normal((5000, 64))
    b = rng.standard_normal((5000, 17))
    C = D.empty(64, 17)
    _lib.call("ks_gemm_tn_tall", 64, 17, 5000, 2.0, D.p(D.to_dev(a)), 64, 1, D.p(D.to_dev(b)), 17, 1, D.p(C), D.stream())
    np.testing.assert_allclose(C.cpu().numpy(), 2 * a.T @ b, rtol=1e-12, atol=1e-11)


def test_kron_mat_mul_hand_case():
    import paper_2209_04876_b200 as K
    facs = [np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[0.0, 1.0], [1.0, 0.0]])]
    np.testing.assert_allclose(K.kron_mat_mul(facs, np.array([1.0, 0.0, 0.0, 0.0])), [0.0, 1.0, 0.0, 3.0],
                               atol=1e-12)


@pytest.mark.parametrize("shapes", [[(4, 3)], [(3, 2), (2, 5)], [(2, 3), (4, 2), (3, 2)], [(5, 1), (1, 4), (2, 2)]])
def test_kron_mat_mul_dense_oracle(rng, shapes):
    import paper_2209_04876_b200 as K
    facs = [rng.standard_normal(s) for s in shapes]
    cols = math.prod(s[1] for s in shapes)
    b = rng.standard_normal((cols, 3))
    dense = dense_kron(facs)
    got = K.kron_mat_mul(facs, b)
    assert isinstance(got, np.ndarray) and got.shape == (dense.shape[0], 3)
    assert np.max(np.abs(got - dense @ b)) <= 1e-10 * max(1, np.max(np.abs(dense @ b)))


def test_kron_mat_mul_errors_and_device_io(rng):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.errors import InvalidInputError
    with pytest.raises(InvalidInputError):
        K.kron_mat_mul([rng.standard_normal((3, 2)), rng.standard_normal((2, 4))], rng.standard_normal(9))
    with pytest.raises(InvalidInputError):
        K.kron_mat_mul([np.array([[np.nan]])], np.ones(1))
    facs = [rng.standard_normal((6, 3)), rng.standard_normal((5, 2))]
    b = torch.tensor(rng.standard_normal(6), device="cuda")
    out = K.kron_mat_mul(facs, b)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    np.testing.assert_allclose(out.cpu().numpy(), dense_kron(facs) @ b.cpu().numpy(), atol=1e-12)


def test_kron_vec_square(rng):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.errors import InvalidInputError
    facs = [rng.standard_normal(s) for s in [(2, 2), (3, 3), (2, 2)]]
    c = rng.standard_normal(12)
    np.testing.assert_allclose(K.kron_vec_square(facs, c), dense_kron(facs) @ c, atol=1e-12)
    with pytest.raises(InvalidInputError):
        K.kron_vec_square([rng.standard_normal((3, 2))], rng.standard_normal(2))


class TestCompactSvd:
    def test_identity(self):
        import paper_2209_04876_b200 as K
        svd = K.compact_svd(np.eye(3), rank_tol=1e-12)
        assert svd.rank == 3
        np.testing.assert_allclose(svd.sigma, [1.0, 1.0, 1.0], atol=1e-12)
        np.testing.assert_allclose(svd.reconstruct(), np.eye(3), atol=1e-12)

    def test_rank_deficient_diagonal(self):
        import paper_2209_04876_b200 as K
        svd = K.compact_svd([[3.0, 0.0], [0.0, 0.0]], rank_tol=1e-12)
        assert svd.rank == 1
        np.testing.assert_allclose(svd.sigma, [3.0])

    @pytest.mark.parametrize("shape", [(5, 5), (17, 9), (64, 64), (40, 64), (6, 4), (3000, 64), (20000, 16),
                                       (1000, 128)])
    def test_reconstruction_sizes(self, rng, shape):
        import paper_2209_04876_b200 as K
        a = rng.standard_normal(shape)
        svd = K.compact_svd(a)
        assert np.linalg.norm(svd.reconstruct() - a) <= 1e-8 * np.linalg.norm(a)
        np.testing.assert_allclose(svd.u.T @ svd.u, np.eye(svd.rank), atol=1e-10)
        np.testing.assert_allclose(svd.v.T @ svd.v, np.eye(svd.rank), atol=1e-10)
        ref = np.linalg.svd(a, compute_uv=False)
        np.testing.assert_allclose(svd.sigma, ref[:svd.rank], rtol=1e-11)

    def test_low_rank_truncation(self, rng):
        import paper_2209_04876_b200 as K
        a = rng.standard_normal((5, 2)) @ rng.standard_normal((2, 4))
        assert K.compact_svd(a).rank == 2

    def test_zero_and_invalid(self):
        import paper_2209_04876_b200 as K
        from paper_2209_04876_b200.errors import InvalidInputError
        assert K.compact_svd(np.zeros((3, 2))).rank == 0
        with pytest.raises(InvalidInputError):
            K.compact_svd([[np.nan, 0.0], [0.0, 1.0]])
        with pytest.raises(InvalidInputError):
            K.compact_svd(np.eye(2), rank_tol=1.5)


def test_factor_gram_matches_eigh(rng):
    import paper_2209_04876_b200 as K
    from oracle import kronsolve_oracle as O
    for shape in [(50, 5), (16384, 64), (300, 3)]:
        a = rng.normal(1.0, 0.03, shape)
        fg = K.factor_gram(a)
        v, w, g = O.factor_gram(a)
        np.testing.assert_allclose(fg.eigenvalues, w, rtol=1e-9, atol=1e-12 * w[0])
        recon = fg.v @ np.diag(fg.eigenvalues) @ fg.v.T
        assert np.linalg.norm(recon - g) <= 1e-12 * np.linalg.norm(g)
        np.testing.assert_allclose(fg.matrix, g, rtol=1e-12, atol=1e-12 * np.abs(g).max())


def test_inverse_small(rng):
    from paper_2209_04876_b200.leverage import _inverse_small
    from paper_2209_04876_b200 import _device as D
    from paper_2209_04876_b200.errors import NumericalFailureError
    for d in (1, 5, 64, 128):
        m = rng.standard_normal((d, d)) + d * np.eye(d)
        x = _inverse_small(D.to_dev(m)).cpu().numpy()
        np.testing.assert_allclose(x @ m, np.eye(d), atol=1e-11)
    with pytest.raises(NumericalFailureError):
        _inverse_small(D.to_dev(np.zeros((2, 2))))


@pytest.mark.parametrize("n,d", [(4096, 16), (65536, 64), (20000, 128)])
def test_cholqr2_and_leverage_scores_tall(n, d):
    """CholeskyQR2 R (R^T R = A^T A, up to row signs the Householder R) and the fused leverage
    scores ||(A R^-1)_i||^2 against NumPy's QR / the oracle's compact-SVD scores."""
    import ctypes
    import torch
    from paper_2209_04876_b200 import _device as D, _lib
    from oracle import kronsolve_oracle as O
    rng = np.random.default_rng(n + d)
    a = rng.normal(1.0, np.sqrt(1e-3), (n, d))
    at = torch.tensor(a, device="cuda")
    r = D.empty(d, d)
    ok = ctypes.c_int32(0)
    _lib.call("ks_chol_qr2_r", D.p(at), n, d, D.p(r), ctypes.byref(ok), D.stream())
    assert ok.value == 1
    rr = r.cpu().numpy()
    _, rq = np.linalg.qr(a)
    signs = np.sign(np.diag(rq))
    np.testing.assert_allclose(rr, signs[:, None] * rq, rtol=1e-10, atol=1e-10 * np.abs(rq).max())
    sc = D.empty(n)
    _lib.call("ks_leverage_scores_tall", D.p(at), n, d, D.p(sc), ctypes.byref(ok), D.stream())
    assert ok.value == 1
    want = O.ridge_scores(O.compact_svd(a), 0.0)
    np.testing.assert_allclose(sc.cpu().numpy(), want, rtol=1e-10)
    # rank-deficient input: CholeskyQR2 declines, callers fall back to Householder / the SVD
    a[:, 1] = a[:, 0]
    _lib.call("ks_leverage_scores_tall", D.p(torch.tensor(a, device="cuda")), n, d, D.p(sc), ctypes.byref(ok),
              D.stream())
    assert ok.value == 0


@pytest.mark.parametrize("shape,rank", [((512, 512, 64), (16, 16, 4)),   # BASELINE c5 (K13)
                                        ((37, 203, 8), (2, 4, 1)),      # partial unit, n2 = 8
                                        ((9, 70, 128), (6, 8, 8)),      # n2 = 128 (32-row units)
                                        ((5, 131, 24), (4, 2, 3)),      # odd R2, n1 not a unit multiple
                                        ((300, 1, 16), (2, 2, 5)),      # n1 = 1: one row per unit
                                        ((40, 300, 40), (3, 27, 7))])   # odd ranks, R1 > 16 (two S tiles)
def test_kron3_contract_matches_oracle(rng, shape, rank):
    """K13 (ks_kron3.cu): T = (U0 kron U1 kron U2)^T b against the oracle's rightmost-first
    kron_mat_mul (kron.py:44-77) with the transposed factors."""
    from oracle import kronsolve_oracle as O
    from paper_2209_04876_b200 import _lib, _device as D
    us = [rng.standard_normal((n, r)) for n, r in zip(shape, rank)]
    b = rng.standard_normal(math.prod(shape))
    assert _lib.load().ks_kron3_supported(*shape, *rank) == 1
    T = D.empty(rank[0], rank[1] * rank[2])
    U = [D.to_dev(u) for u in us]
    _lib.call("ks_kron3_contract", D.p(U[0]), D.p(U[1]), D.p(U[2]), D.p(D.to_dev(b)), *shape, *rank, D.p(T),
              D.stream())
    want = O.kron_mat_mul([u.T for u in us], b)
    got = T.cpu().numpy().reshape(-1)
    assert rel(got, want) < 1e-13, rel(got, want)
    # with ||b||^2 from the same pass (register-streaming kernel) or a second one (TMA ring)
    T3, bsq = D.empty(rank[0], rank[1] * rank[2]), D.empty(1)
    _lib.call("ks_kron3_contract_sumsq", D.p(U[0]), D.p(U[1]), D.p(U[2]), D.p(D.to_dev(b)), *shape, *rank, D.p(T3),
              D.p(bsq), D.stream())
    assert torch.equal(T3, T)
    assert abs(float(bsq) - float(np.dot(b, b))) <= 1e-13 * float(np.dot(b, b))
    # deterministic: a second pass gives the same bits
    T2 = D.empty(rank[0], rank[1] * rank[2])
    _lib.call("ks_kron3_contract", D.p(U[0]), D.p(U[1]), D.p(U[2]), D.p(D.to_dev(b)), *shape, *rank, D.p(T2),
              D.stream())
    assert torch.equal(T, T2)

