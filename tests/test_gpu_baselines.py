"""Dense comparison baselines on the GPU: naive_normal_solve and
sketch_and_solve_ridge against the oracle (pinned bit-exact to the reference in
tests/test_oracle.py) and the reference's own unit properties (tests/test_solvers.py)."""

import numpy as np
import pytest

from conftest import dense_kron, rel
from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu


def K():
    import paper_2209_04876_b200 as k
    return k


@pytest.mark.parametrize("lam", [0.0, 1e-3, 1.0])
def test_naive_normal_solve_matches_oracle(lam):
    rng = np.random.default_rng(3)
    facs = [rng.standard_normal((8, 3)), rng.standard_normal((6, 2))]
    b = rng.standard_normal(48)
    got = K().naive_normal_solve(facs, b, lam)
    want = O.naive_normal_solve(facs, b, lam)
    assert rel(got.solution, want.solution) <= 1e-10
    assert got.loss == pytest.approx(want.loss, rel=1e-10)
    ex = K().kronmatmul_svd_solve(facs, b, lam)
    assert rel(got.solution, ex.solution) <= 1e-10


def test_naive_normal_solve_reference_properties():
    rng = np.random.default_rng(4)
    b = rng.standard_normal(6)
    np.testing.assert_allclose(K().naive_normal_solve([np.eye(2), np.eye(3)], b, 0.0).solution, b, atol=1e-10)
    facs = [rng.standard_normal((6, 2)), rng.standard_normal((5, 2))]
    b = rng.standard_normal(30)
    x = K().naive_normal_solve(facs, b, 1e12).solution
    assert np.linalg.norm(x) <= 1e-9 * np.linalg.norm(dense_kron(facs).T @ b)
    facs = [rng.standard_normal((7, 3)), rng.standard_normal((5, 2))]
    b = rng.standard_normal(35)
    x = K().naive_normal_solve(facs, b, 0.02).solution
    k = dense_kron(facs)
    assert np.linalg.norm(k.T @ (k @ x - b) + 0.02 * x) <= 1e-8 * max(1.0, np.linalg.norm(k.T @ b))
    from paper_2209_04876_b200.errors import SizeGuardError
    with pytest.raises(SizeGuardError):
        K().naive_normal_solve([rng.standard_normal((40, 30))] * 2, rng.standard_normal(1600), 0.0,
                               max_dense_entries=10_000)


@pytest.mark.parametrize("lam", [0.0, 1e-2])
def test_sketch_and_solve_matches_oracle(lam):
    rng = np.random.default_rng(77)
    facs = [rng.standard_normal((14, 3)), rng.standard_normal((12, 2))]
    b = rng.standard_normal(14 * 12)
    got = K().sketch_and_solve_ridge(facs, b, K().RegressionConfig(eps=0.5, delta=0.1, lam=lam, seed=4))
    want = O.sketch_and_solve_ridge(facs, b, eps=0.5, lam=lam, seed=4)
    assert got.sample_count == want.sample_count
    assert rel(got.solution, want.solution) <= 1e-9


def test_sketch_and_solve_reference_properties():
    rng = np.random.default_rng(5)
    facs = [rng.standard_normal((5, 2)), rng.standard_normal((4, 2))]
    b = rng.standard_normal(20)
    full = K().RowSketch(indices=np.arange(20), weights=np.ones(20))
    rep = K().sketch_and_solve_ridge(facs, b, K().RegressionConfig(lam=1e-2, seed=0), sketch=full)
    np.testing.assert_allclose(rep.solution, K().kronmatmul_svd_solve(facs, b, 1e-2).solution, atol=1e-8)
    rep = K().sketch_and_solve_ridge(facs, np.zeros(20), K().RegressionConfig(lam=1e-2, seed=0))
    np.testing.assert_allclose(rep.solution, np.zeros(4), atol=1e-12)
    sk = K().sketch_rows_of_kron(facs, full)
    np.testing.assert_allclose(sk, dense_kron(facs), rtol=1e-15)


def test_sketch_and_solve_c2_dense_path():
    """BASELINE config 2 shapes (n = 4096, d = 32: a 1024 x 1024 sampled normal matrix, above the
    Jacobi limit, so the dense symmetric eigensolver path) against the oracle."""
    facs, b = O.synth_regression(4096, 32, 2, 0)
    cfg = dict(eps=0.1, lam=1e-3, alpha=1e-5, seed=0)
    want = O.sketch_and_solve_ridge(facs, b, **cfg)
    got = K().sketch_and_solve_ridge(facs, b, K().RegressionConfig(delta=0.01, **cfg))
    assert got.sample_count == want.sample_count
    assert got.loss == pytest.approx(want.loss, rel=1e-6)
