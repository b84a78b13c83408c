"""Sampler tables, draws, weights and sketch deduplication: bit-exact vs the oracle/NumPy
(reference test_leverage.py / test_kron.py patterns)."""

import math

import numpy as np
import pytest
import torch

from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 3, 8, 9, 100, 128, 129, 1000, 1024, 4097, 16384, 65536, 100003])
def test_sampler_tables_bit_exact(n):
    import paper_2209_04876_b200 as K
    rng = np.random.default_rng(n)
    sc = rng.random(n) ** 3 + (rng.random(n) < 0.01)
    sampler = K.build_product_sampler([K.LeverageScores(sc, 0.0)])
    ref = O.Sampler([sc])
    np.testing.assert_array_equal(sampler.per_factor_probabilities[0], ref.probs[0])
    np.testing.assert_array_equal(sampler.per_factor_cdf[0], ref.cdfs[0])


@pytest.mark.parametrize("n,kind", [(65536, "ints"), (100003, "ints"), (40000, "zeros_first"), (131072, "pow2"),
                                    (131073, "smooth"), (200000, "smooth")])
def test_sampler_tables_bit_exact_large(n, kind):
    """The n >= 32768 path (multi-CTA pairwise total, segmented exact cumsum with verification and the
    window fallback): small-integer scores (exact sums, round-half-even ties), a long zero prefix,
    power-of-two scores, and sizes past the segmented kernel's limit -- all bit-exact."""
    import paper_2209_04876_b200 as K
    rng = np.random.default_rng(n + len(kind))
    if kind == "ints":
        sc = rng.integers(0, 4, n).astype(np.float64)
        sc[0] = 1.0
    elif kind == "zeros_first":
        sc = rng.random(n)
        sc[: n // 3] = 0.0
    elif kind == "pow2":
        sc = np.ldexp(1.0, rng.integers(-40, 3, n)).astype(np.float64)
    else:
        sc = rng.random(n) + 0.25
    sampler = K.build_product_sampler([K.LeverageScores(sc, 0.0)])
    ref = O.Sampler([sc])
    np.testing.assert_array_equal(sampler.per_factor_probabilities[0], ref.probs[0])
    np.testing.assert_array_equal(sampler.per_factor_cdf[0], ref.cdfs[0])


def test_sampler_tables_with_zeros_and_validation():
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.errors import InvalidInputError
    sc = np.array([0.0, 0.0, 1e-30, 2.0, 0.0, 3.5, 0.0])
    s = K.build_product_sampler([K.LeverageScores(sc, 0.0)])
    np.testing.assert_array_equal(s.per_factor_cdf[0], np.cumsum(sc / sc.sum()))
    with pytest.raises(InvalidInputError):
        K.build_product_sampler([K.LeverageScores(np.zeros(3), 0.0)])
    with pytest.raises(InvalidInputError):
        K.build_product_sampler([K.LeverageScores(np.array([1.0, -1.0]), 0.0)])
    with pytest.raises(InvalidInputError):
        K.build_product_sampler([K.LeverageScores(np.array([1.0, np.inf]), 0.0)])


def test_product_sampler_draws_match_reference(golden):
    import paper_2209_04876_b200 as K
    u = golden("units")
    rng = np.random.default_rng(12345)
    rng.standard_normal((50, 5))
    facs = [rng.standard_normal((40, 3)), rng.standard_normal((30, 2))]
    sampler = K.build_product_sampler([K.statistical_leverage_scores(f) for f in facs])
    g = np.random.default_rng(7)
    draws = sampler.sample(1000, g)
    np.testing.assert_array_equal(draws, u["draws"])
    # the Generator advanced exactly as the reference's sample() advances it
    g2 = np.random.default_rng(7)
    g2.random(2000)
    assert g.random() == g2.random()
    sk = K.sample_rows(sampler, 500, 11)
    np.testing.assert_array_equal(sk.indices, u["sk_indices"])
    np.testing.assert_allclose(sk.weights, u["sk_weights"], rtol=1e-13)


def test_product_sampler_bit_exact_given_same_tables(rng):
    import paper_2209_04876_b200 as K
    scores = [rng.random(1024) + 0.01, rng.random(777) + 0.01]
    ref = O.Sampler(scores)
    s = 20011
    idx_ref, w_ref = O.sample_rows(ref, s, 99)
    sk = K.sample_rows(K.build_product_sampler([K.LeverageScores(x, 0.0) for x in scores]), s, 99)
    np.testing.assert_array_equal(sk.indices, idx_ref)
    np.testing.assert_array_equal(sk.weights, w_ref)


def test_explicit_distribution_sample_rows(golden):
    import paper_2209_04876_b200 as K
    u = golden("units")
    rng = np.random.default_rng(12345)
    rng.standard_normal((50, 5)); rng.standard_normal((40, 3)); rng.standard_normal((30, 2))
    p = rng.random(97)
    sk = K.sample_rows(p, 300, 5)
    np.testing.assert_array_equal(sk.indices, u["choice_indices"])
    np.testing.assert_array_equal(sk.weights, u["choice_weights"])
    sk = K.sample_rows(np.full(4, 0.25), 2, seed=0)
    np.testing.assert_allclose(sk.weights, [math.sqrt(2.0)] * 2, atol=1e-12)
    sk = K.sample_rows(np.array([1.0, 0.0, 0.0]), 3, seed=0)
    np.testing.assert_array_equal(sk.indices, [0, 0, 0])


def test_spectral_approx_rows(golden):
    import paper_2209_04876_b200 as K
    u = golden("units")
    rng = np.random.default_rng(12345)
    for shp in [(50, 5), (40, 3), (30, 2)]:
        rng.standard_normal(shp)
    rng.random(97)
    a2 = rng.standard_normal((400, 4))
    got = K.spectral_approx_rows(a2, 0.5, 0.1, seed=2, alpha=0.05)
    assert got.shape == u["spectral_rows"].shape
    np.testing.assert_allclose(got, u["spectral_rows"], rtol=1e-12, atol=1e-14)


def test_jl_scores_vs_reference(golden):
    import paper_2209_04876_b200 as K
    u = golden("units")
    a = np.random.default_rng(12345).standard_normal((50, 5))
    ls = K.approx_leverage_scores_jl(a, a, a.T @ a, 0.25, seed=3)
    np.testing.assert_allclose(ls.scores, u["jl_scores"], rtol=1e-12)
    assert ls.approx_factor == pytest.approx(1.125)


def test_jl_scores_errors(rng):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.errors import InvalidInputError, NumericalFailureError
    a = rng.standard_normal((6, 2))
    with pytest.raises(InvalidInputError):
        K.approx_leverage_scores_jl(a, a, a.T @ a, 0.5, seed=0)
    z = np.zeros((4, 2))
    with pytest.raises(NumericalFailureError):
        K.approx_leverage_scores_jl(z, z, z.T @ z, 0.25, seed=0)


@pytest.mark.parametrize("case", ["dups", "degenerate", "flat", "three"])
def test_sparse_diagonal_bit_exact(case, rng):
    import paper_2209_04876_b200 as K
    if case == "dups":
        idx = rng.integers(0, 30, size=(5000, 2)); shape = (30, 30)
    elif case == "degenerate":
        idx = np.zeros((4000, 2), dtype=np.int64); shape = (5, 7)
    elif case == "flat":
        idx = rng.integers(0, 50, size=3000); shape = (50,)
    else:
        idx = rng.integers(0, 9, size=(2000, 3)); shape = (9, 9, 9)
    w = rng.random(idx.shape[0]) + 0.1
    sd = K.sparse_diagonal_from_sketch(K.RowSketch(idx, w), shape)
    ri, rv = O.sparse_diagonal_from_sketch(idx, w, shape)
    np.testing.assert_array_equal(sd.indices, ri)
    np.testing.assert_array_equal(sd.values, rv)


def test_sparse_diagonal_known_answer():
    import paper_2209_04876_b200 as K
    sd = K.sparse_diagonal_from_sketch(K.RowSketch(np.array([2, 2, 0]), np.array([1.0, 1.0, 3.0])), (4,))
    np.testing.assert_array_equal(sd.indices, [0, 2])
    np.testing.assert_allclose(sd.values ** 2, [9.0, 2.0], atol=1e-12)


def test_large_sketch_dedup_matches_oracle():
    import paper_2209_04876_b200 as K
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 65536, size=(169767, 2))
    w = rng.random(169767)
    sd = K.sparse_diagonal_from_sketch(K.RowSketch(torch.tensor(idx, device="cuda"), torch.tensor(w, device="cuda")),
                                       (65536, 65536))
    ri, rv = O.sparse_diagonal_from_sketch(idx, w, (65536, 65536))
    np.testing.assert_array_equal(sd.indices.cpu().numpy(), ri)
    np.testing.assert_array_equal(sd.values.cpu().numpy(), rv)
