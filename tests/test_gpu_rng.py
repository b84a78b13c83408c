"""GPU PCG64 / ziggurat streams vs NumPy itself (bit-exact)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 1, 12345, np.random.SeedSequence(0).spawn(5)[4]])
@pytest.mark.parametrize("count,skip", [(1, 0), (1000, 0), (100_003, 17), (38049 * 2, 0)])
def test_uniforms_bit_exact(seed, count, skip):
    from paper_2209_04876_b200.leverage import device_uniforms
    from paper_2209_04876_b200._numpy_rng import pcg64_state
    st, inc = pcg64_state(seed)
    g = np.random.default_rng(seed)
    if skip:
        g.random(skip)
    np.testing.assert_array_equal(device_uniforms(st, inc, count, skip).cpu().numpy(), g.random(count))


@pytest.mark.parametrize("seed", [0, 3, np.random.SeedSequence(0).spawn(5)[1], np.random.SeedSequence(0).spawn(5)[3]])
@pytest.mark.parametrize("count", [1, 7, 5000, 78 * 16384])
def test_standard_normal_bit_exact(seed, count):
    from paper_2209_04876_b200.leverage import device_standard_normal
    got = device_standard_normal(seed, count).cpu().numpy()
    want = np.random.default_rng(seed).standard_normal(count)
    bad = np.flatnonzero(got != want)
    # the tail branch uses device log1p: allow ulp-level differences there only
    assert bad.size <= max(2, count // 100000), bad[:10]
    if bad.size:
        np.testing.assert_allclose(got[bad], want[bad], rtol=4e-16, atol=0)


def test_standard_normal_divisor_and_batches():
    from paper_2209_04876_b200.leverage import device_standard_normal
    n = (1 << 25) + 12345  # crosses the internal batch boundary
    got = device_standard_normal(5, n, divisor=3.0).cpu().numpy()
    want = np.random.default_rng(5).standard_normal(n) / 3.0
    assert np.count_nonzero(got != want) <= 64
    np.testing.assert_allclose(got, want, rtol=1e-15, atol=0)
