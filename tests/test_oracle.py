"""Pin the CPU oracle (oracle/kronsolve_oracle.py) before trusting it:
  * against the committed golden fixtures produced by the reference itself, and
  * against the live reference when /root/reference is importable (build container only)."""

import math
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC, dense_kron
from oracle import kronsolve_oracle as O

CFG = dict(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)


@pytest.mark.parametrize("name,n,d", [("c1", 1024, 16), ("c2", 4096, 32)])
def test_oracle_matches_golden_fast(golden, name, n, d):
    g = golden(name)
    facs, b = O.synth_regression(n, d, 2, 0)
    rep = O.fast_kronecker_regression(facs, b, **CFG)
    assert rep.sample_count == int(g["s"]) and rep.iterations == int(g["iterations"])
    np.testing.assert_array_equal(rep.trace["indices"], g["indices"])
    np.testing.assert_array_equal(rep.trace["weights"], g["weights"])
    np.testing.assert_array_equal(rep.trace["sd_indices"], g["sd_indices"])
    np.testing.assert_array_equal(rep.trace["sd_values"], g["sd_values"])
    np.testing.assert_array_equal(rep.solution, g["x"])
    assert rep.loss == float(g["loss"])
    np.testing.assert_array_equal(np.asarray(rep.trace["history"]), g["history"])
    np.testing.assert_array_equal(rep.trace["cdfs"][0], g["cdf0"])


@pytest.mark.slow
def test_oracle_matches_golden_c3(golden):
    g = golden("c3")
    facs, b = O.synth_regression(16384, 64, 2, 0)
    rep = O.fast_kronecker_regression(facs, b, with_loss=False, **CFG)
    np.testing.assert_array_equal(rep.trace["indices"], g["indices"])
    np.testing.assert_array_equal(rep.solution, g["x"])


@pytest.mark.parametrize("name,n,d", [("c1", 1024, 16), ("c2", 4096, 32)])
def test_oracle_matches_golden_exact(golden, name, n, d):
    g = golden(name)
    facs, b = O.synth_regression(n, d, 2, 0)
    rep = O.kronmatmul_svd_solve(facs, b, 1e-3)
    np.testing.assert_array_equal(rep.solution, g["exact_x"])
    assert rep.loss == float(g["opt"])


def test_oracle_known_answers():
    # reference test_kron.py:45-49 hand case
    facs = [np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[0.0, 1.0], [1.0, 0.0]])]
    np.testing.assert_allclose(O.kron_mat_mul(facs, np.array([1.0, 0, 0, 0])), [0, 1, 0, 3], atol=1e-12)
    # test_leverage.py:44-48 ridge scores (1/4, 4/7, 0)
    a = np.array([[1.0, 0.0], [0.0, 2.0], [0.0, 0.0]])
    np.testing.assert_allclose(O.ridge_scores(O.compact_svd(a), 3.0), [0.25, 4 / 7, 0.0], atol=1e-12)
    # test_kron.py:139-145 duplicate aggregation sqrt(sum w^2) = [3, sqrt 2]
    idx, val = O.sparse_diagonal_from_sketch(np.array([2, 2, 0]), np.array([1.0, 1.0, 3.0]), (4,))
    np.testing.assert_array_equal(idx, [0, 2])
    np.testing.assert_allclose(val ** 2, [9.0, 2.0], atol=1e-12)
    # test_leverage.py:206-214 uniform weights sqrt(2) and degenerate distribution
    _, w = O.sample_rows(np.full(4, 0.25), 2, 0)
    np.testing.assert_allclose(w, [math.sqrt(2.0)] * 2, atol=1e-12)
    i3, w3 = O.sample_rows(np.array([1.0, 0.0, 0.0]), 3, 0)
    np.testing.assert_array_equal(i3, [0, 0, 0])
    np.testing.assert_allclose(w3, [1 / math.sqrt(3.0)] * 3, atol=1e-12)
    # test_solvers.py:330-333 damping 0.5 and 16 iterations at eps=0.25
    assert O.effective_max_iters(0.25) == 16
    # partitions of SURVEY Appendix A
    assert O.balanced_partition([64, 64])[:2] == ((0,), (1,))
    assert O.balanced_partition([16, 16, 4])[:2] == ((0,), (1, 2))
    assert O.balanced_partition([16, 4])[:2] == ((1,), (0,))


def test_oracle_sketched_applies_vs_dense(rng):
    facs = [rng.standard_normal((4, 2)), rng.standard_normal((3, 2)), rng.standard_normal((4, 3))]
    dense = dense_kron(facs)
    idx = np.sort(rng.choice(48, size=7, replace=False)).astype(np.int64)
    val = rng.standard_normal(7)
    c = rng.standard_normal(12)
    np.testing.assert_allclose(O.sketched_kron_apply(facs, idx, val, c), val * (dense @ c)[idx], atol=1e-12)
    bv = rng.standard_normal(7)
    full = np.zeros(48)
    full[idx] = val * bv
    np.testing.assert_allclose(O.sketched_kron_transpose_apply(facs, idx, val, bv), dense.T @ full, atol=1e-12)


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference not mounted (GPU box)")
def test_oracle_matches_live_reference_units(golden):
    sys.path.insert(0, str(REFERENCE_SRC))
    import kronsolve as ks
    rng = np.random.default_rng(3)
    for shapes in ([(3, 2), (2, 5)], [(2, 3), (4, 2), (3, 2)]):
        facs = [rng.standard_normal(s) for s in shapes]
        b = rng.standard_normal((math.prod(s[1] for s in shapes), 3))
        np.testing.assert_array_equal(O.kron_mat_mul(facs, b), ks.kron_mat_mul(facs, b))
    facs = [rng.standard_normal((15, 2)), rng.standard_normal((12, 3))]
    b = rng.standard_normal(180)
    caches_ref = [ks.build_factor_cache(a) for a in facs]
    caches_or = [O.factor_cache(a) for a in facs]
    r1 = ks.fast_kronecker_regression(facs, b, ks.RegressionConfig(eps=0.25, delta=0.1, lam=1e-2, seed=4,
                                                                   alpha=1e-3), caches=caches_ref)
    r2 = O.fast_kronecker_regression(facs, b, eps=0.25, delta=0.1, lam=1e-2, seed=4, alpha=1e-3,
                                     caches=caches_or)
    np.testing.assert_array_equal(r1.solution, r2.solution)
    u = golden("units")
    a = np.random.default_rng(12345).standard_normal((50, 5))
    sc, _ = O.jl_scores(a, a, a.T @ a, 0.25, 3)
    np.testing.assert_array_equal(sc, u["jl_scores"])


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference not mounted (GPU box)")
def test_dense_baselines_match_live_reference():
    sys.path.insert(0, str(REFERENCE_SRC))
    import kronsolve as ks
    rng = np.random.default_rng(77)
    facs = [rng.standard_normal((14, 3)), rng.standard_normal((12, 2))]
    b = rng.standard_normal(14 * 12)
    for lam in (0.0, 1e-2):
        r = ks.naive_normal_solve(facs, b, lam)
        o = O.naive_normal_solve(facs, b, lam)
        np.testing.assert_array_equal(o.solution, r.solution)
        assert o.loss == r.loss
        cfg = ks.RegressionConfig(eps=0.5, delta=0.1, lam=lam, seed=4)
        r = ks.sketch_and_solve_ridge(facs, b, cfg)
        o = O.sketch_and_solve_ridge(facs, b, eps=0.5, lam=lam, seed=4)
        np.testing.assert_array_equal(o.solution, r.solution)
        assert o.sample_count == r.sample_count


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference not mounted (GPU box)")
def test_synth_generators_match_live_reference():
    """The input generators the tests use follow experiments.py bit for bit."""
    sys.path.insert(0, str(REFERENCE_SRC))
    from kronsolve.experiments import generate_synth_regression, generate_synth_tucker
    for seed in (0, 3):
        np.testing.assert_array_equal(O.synth_tucker((9, 7, 5), (3, 2, 2), 0.01, seed, relative=True),
                                      generate_synth_tucker((9, 7, 5), (3, 2, 2), 0.01, seed))
        facs, b = O.synth_regression(64, 4, 2, seed)
        rf, rb = generate_synth_regression(64, 4, 2, seed=seed)
        np.testing.assert_array_equal(b, rb)
        for a, r in zip(facs, rf):
            np.testing.assert_array_equal(a, r)
