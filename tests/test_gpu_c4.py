"""BASELINE config 4 (n = 65536, d in {16, 32, 64, 128}) on one B200.

c4 is the configuration where the per-factor spectral row sampling (leverage.py:235-252) is
active (s_n < n) and, at d = 128, where the persistent loop kernel does not apply.  b has
4.29e9 entries (34.4 GB): it lives only on the device.

* sampling parity: with b = 0 (b only enters the right-hand side) the oracle finishes in seconds
  and the sketch -- spectral rows, JL scores, product sampling, sparse diagonal -- must match it
  bit for bit in the indices and to rounding in the values;
* solve quality: with b ~ N(0, 1) generated on the device from NumPy's stream
  (default_rng(0).standard_normal(n^2)), the fast solve's loss is checked against
  the exact optimum from the device KronMatMul solver."""

import math

import numpy as np
import pytest
import torch

from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu

N4 = 65536
PARAMS = dict(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)


def cfg():
    import paper_2209_04876_b200 as K
    return K.RegressionConfig(**PARAMS)


def factors(d):
    """experiments.py:106-115 at n = 65536 (A1 then A2 from one default_rng(0))."""
    gen = np.random.default_rng(0)
    return [gen.normal(1.0, math.sqrt(0.001), (N4, d)) for _ in range(2)]


@pytest.mark.parametrize("d", [16, 64])
def test_c4_sketch_matches_oracle(d):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.solvers import FastSolveTrace
    facs = factors(d)
    b_dev = torch.zeros(N4 * N4, dtype=torch.float64, device="cuda")
    tr = FastSolveTrace()
    rep = K.fast_kronecker_regression([torch.tensor(a, device="cuda") for a in facs], b_dev, cfg(), _trace=tr,
                                      with_loss=False)
    del b_dev
    torch.cuda.empty_cache()
    # the oracle with a zero-stride zero b: identical sketch, trivial Richardson (rhs = 0)
    ref = O.fast_kronecker_regression(facs, np.broadcast_to(0.0, (N4 * N4,)), with_loss=False, **PARAMS)
    t = ref.trace
    assert rep.sample_count == t["s"]
    assert tr.a_tilde_rows == t["a_tilde_rows"] and all(r < N4 for r in t["a_tilde_rows"])  # spectral branch
    np.testing.assert_array_equal(tr.sketch.indices.cpu().numpy(), t["indices"])
    np.testing.assert_allclose(tr.sketch.weights.cpu().numpy(), t["weights"], rtol=1e-9)
    np.testing.assert_array_equal(tr.sdiag.indices.cpu().numpy(), t["sd_indices"])
    np.testing.assert_allclose(tr.sdiag.values.cpu().numpy(), t["sd_values"], rtol=1e-9)
    assert np.allclose(np.asarray(rep.solution.cpu()), 0.0)


@pytest.mark.parametrize("d", [16, 64, 128])
def test_c4_fast_solve_vs_exact(d):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.leverage import device_standard_normal
    facs = [torch.tensor(a, device="cuda") for a in factors(d)]
    b = device_standard_normal(0, N4 * N4)  # default_rng(0).standard_normal(n^2), bit-exact stream
    # spot-check the device stream against NumPy on its first entries
    np.testing.assert_array_equal(b[:4096].cpu().numpy(), np.random.default_rng(0).standard_normal(4096))
    exact = K.kronmatmul_svd_solve(facs, b, PARAMS["lam"])
    fast = K.fast_kronecker_regression(facs, b, cfg())
    s = math.ceil(1e-5 * 1680 * d * d * math.log(40 * d * d) * math.log(100.0) / 0.1)
    assert fast.sample_count == s
    assert 0 < fast.iterations <= 24
    x = fast.solution.cpu().numpy()
    assert np.all(np.isfinite(x))
    # b ~ N(0, 1) is almost pure noise for a rank-d^2 model: OPT ~ ||b||^2.  At alpha = 1e-5 the
    # sample count is far below the (1 + eps) theorem's, so the reference itself lands ~20 % above
    # OPT here (a quality property of the algorithm at this alpha, as SURVEY.md notes for c5)
    assert exact.loss <= fast.loss <= 1.5 * exact.loss
    # the separate right-hand-side + loop path (other kernels, other summation orders) agrees
    from paper_2209_04876_b200 import solvers as S
    S._USE_FUSED[0] = False
    try:
        sep = K.fast_kronecker_regression(facs, b, cfg(), with_loss=False)
    finally:
        S._USE_FUSED[0] = True
    assert sep.iterations == fast.iterations
    xs = sep.solution.cpu().numpy()
    assert np.linalg.norm(xs - x) <= 1e-6 * np.linalg.norm(x)
    del b
    torch.cuda.empty_cache()
