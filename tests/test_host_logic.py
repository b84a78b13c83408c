"""Host-side logic that needs no GPU: RegressionConfig's derived settings and validation
(reference test_solvers.py TestConfig, solvers.py:41-98) and the generic Richardson iteration
driven by NumPy callables (solvers.py:201-248)."""

import math

import numpy as np
import pytest


def _lstsq(a, b):
    return np.linalg.lstsq(a, b, rcond=None)[0]


def test_config_derived_settings():
    from paper_2209_04876_b200 import RegressionConfig
    assert RegressionConfig(mode="theoretical", alpha=1e-5).effective_alpha == 1.0
    assert RegressionConfig(mode="practical", alpha=1e-5).effective_alpha == 1e-5
    cfg = RegressionConfig(eps=0.25)
    assert cfg.effective_damping == pytest.approx(0.5)
    assert cfg.effective_max_iters == 8 * math.ceil(math.log(4.0))
    cfg = RegressionConfig(eps=0.25, damping=1.0, max_richardson_iters=3)
    assert cfg.effective_damping == 1.0 and cfg.effective_max_iters == 3


@pytest.mark.parametrize("kw", [dict(eps=0.0), dict(eps=1.0), dict(delta=0.0), dict(delta=1.0), dict(lam=-1.0),
                                dict(alpha=0.0), dict(alpha=1.5), dict(mode="other")])
def test_config_range_validation(kw):
    from paper_2209_04876_b200 import InvalidInputError, RegressionConfig
    with pytest.raises(InvalidInputError):
        RegressionConfig(**kw)


def test_richardson_fixed_point_and_one_step(rng):
    from paper_2209_04876_b200 import RegressionConfig, richardson_solve
    a = rng.standard_normal((8, 3))
    b = rng.standard_normal(8)
    ata = a.T @ a
    inv = np.linalg.inv(ata)
    x, it = richardson_solve(lambda v: ata @ v, lambda v: inv @ v, a.T @ b, 1.0, RegressionConfig(eps=0.25))
    assert it == 1
    np.testing.assert_allclose(x, _lstsq(a, b), atol=1e-10)
    xs = _lstsq(a, b)
    moves = []
    x, it = richardson_solve(lambda v: ata @ v, lambda v: np.linalg.solve(ata, v), a.T @ b, 1.0,
                             RegressionConfig(eps=0.25), x0=xs, callback=moves.append)
    assert it == 0 and not moves
    np.testing.assert_allclose(x, xs, atol=1e-12)


@pytest.mark.parametrize("kappa", [2.0, 4.0])
def test_richardson_contraction_rate(rng, kappa):
    from paper_2209_04876_b200 import RegressionConfig, richardson_solve
    a = rng.standard_normal((8, 3))
    b = rng.standard_normal(8)
    ata = a.T @ a
    m = kappa * ata
    minv = np.linalg.inv(m)
    xs = _lstsq(a, b)
    its = []
    richardson_solve(lambda v: ata @ v, lambda v: minv @ v, a.T @ b, 1.0,
                     RegressionConfig(eps=0.25, max_richardson_iters=10, residual_tol=1e-300),
                     callback=lambda xk: its.append(xk.copy()))
    assert len(its) == 10
    e0 = math.sqrt(xs @ m @ xs)
    for k, xk in enumerate(its, start=1):
        d = xk - xs
        assert math.sqrt(d @ m @ d) <= (1 - 1 / kappa) ** k * e0 * (1 + 1e-10) + 1e-12


def test_richardson_x0_shape_checked(rng):
    from paper_2209_04876_b200 import InvalidInputError, RegressionConfig, richardson_solve
    with pytest.raises(InvalidInputError):
        richardson_solve(lambda v: v, lambda v: v, np.ones(3), 1.0, RegressionConfig(), x0=np.ones(4))
