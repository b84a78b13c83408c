"""Pin the Tucker factor-update oracle (oracle/tucker_oracle.py):
  * against the live reference (tucker.py) when /root/reference is importable (build container), and
  * against the committed fixture tests/golden/tucker_units.npz made by running the reference
    (tests/golden/make_golden.py tucker), so the pin travels to machines without the reference."""

import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC
from oracle import kronsolve_oracle as O
from oracle import tucker_oracle as T
from golden.tucker_inputs import ALS_CFG, UNIT_CFG, UNIT_LAM, unit_inputs as tucker_unit_inputs

live = pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference not mounted (GPU box)")


def ref():
    sys.path.insert(0, str(REFERENCE_SRC))
    import kronsolve as ks
    import kronsolve.tucker as kt
    return ks, kt


def oracle_units():
    core, facs, x = tucker_unit_inputs()
    out = {}
    for n in range(3):
        out[f"naive{n}"] = T.naive_factor_update(core, facs, UNIT_LAM, x, n)
        ws = T.build_factor_workspace(core, facs, n, 0.25, UNIT_LAM)
        out[f"w{n}"] = np.float64(ws.w)
        z = np.arange(ws.g_n.shape[1], dtype=np.float64) / 7.0 - 0.3
        out[f"apply{n}"] = ws.apply(z)
        out[f"fast{n}"] = T.fast_factor_matrix_update(core, facs, UNIT_LAM, x, n, T.Cfg(lam=UNIT_LAM, **UNIT_CFG))
    c, f, rep = T.tucker_als(x, (3, 4, 2), lam=UNIT_LAM, sweeps=2, mode="exact", cfg=T.Cfg(seed=3))
    out["als_exact_losses"] = np.asarray(rep.step_losses)
    out["als_exact_core"] = c
    c, f, rep = T.tucker_als(x, (3, 4, 2), lam=UNIT_LAM, sweeps=2, mode="fast",
                             cfg=T.Cfg(**ALS_CFG))
    out["als_fast_losses"] = np.asarray(rep.step_losses)
    out["als_fast_core"] = c
    return out


def test_oracle_matches_tucker_golden(golden):
    g = golden("tucker_units")
    o = oracle_units()
    for k, v in o.items():
        np.testing.assert_allclose(v, g[k], rtol=1e-12, atol=1e-13, err_msg=k)


@live
@pytest.mark.parametrize("n", [0, 1, 2])
def test_factor_updates_match_live_reference(n):
    ks, kt = ref()
    core, facs, x = tucker_unit_inputs()
    model = kt.TuckerModel(core=core, factors=[a.copy() for a in facs], lam=UNIT_LAM)
    np.testing.assert_array_equal(T.naive_factor_update(core, facs, UNIT_LAM, x, n),
                                  kt.naive_factor_update(model, x, n))
    ws_r = kt.build_factor_workspace(model, n, 0.25, UNIT_LAM)
    ws_o = T.build_factor_workspace(core, facs, n, 0.25, UNIT_LAM)
    assert ws_o.w == ws_r.penalty_weight
    np.testing.assert_array_equal(ws_o.mid, ws_r.correction_mid)
    z = np.linspace(-1, 1, ws_o.g_n.shape[1])
    np.testing.assert_array_equal(ws_o.apply(z), ws_r.apply(z))
    np.testing.assert_array_equal(ws_o.project_feasible(z), ws_r.project_feasible(z))
    cfg = ks.RegressionConfig(lam=UNIT_LAM, **UNIT_CFG)
    np.testing.assert_array_equal(
        T.fast_factor_matrix_update(core, facs, UNIT_LAM, x, n, T.Cfg(lam=UNIT_LAM, **UNIT_CFG)),
        kt.fast_factor_matrix_update(model, x, n, cfg))
    # shared-sketch option and explicit caches
    caches_r = [ks.build_factor_cache(a) for a in facs]
    caches_o = [O.factor_cache(a) for a in facs]
    cfg2 = ks.RegressionConfig(lam=UNIT_LAM, share_row_sketch=True, **UNIT_CFG)
    np.testing.assert_array_equal(
        T.fast_factor_matrix_update(core, facs, UNIT_LAM, x, n,
                                    T.Cfg(lam=UNIT_LAM, share_row_sketch=True, **UNIT_CFG), caches=caches_o),
        kt.fast_factor_matrix_update(model, x, n, cfg2, caches=caches_r))


@live
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_tucker_als_matches_live_reference(mode):
    ks, kt = ref()
    _, _, x = tucker_unit_inputs()
    cfg_r = ks.RegressionConfig(**ALS_CFG)
    model, rep = kt.tucker_als(x, (3, 4, 2), lam=UNIT_LAM, sweeps=2, solver_mode=mode, config=cfg_r)
    c, f, ro = T.tucker_als(x, (3, 4, 2), lam=UNIT_LAM, sweeps=2, mode=mode,
                            cfg=T.Cfg(**ALS_CFG))
    assert ro.step_labels == rep.step_labels
    np.testing.assert_array_equal(ro.step_losses, rep.step_losses)
    np.testing.assert_array_equal(c, model.core)
    for a, b in zip(f, model.factors):
        np.testing.assert_array_equal(a, b)
    assert ro.rre == rep.rre


@live
def test_power_iteration_matches_live_reference():
    _, kt = ref()
    rng = np.random.default_rng(5)
    m = rng.standard_normal((20, 20))
    m = m @ m.T
    assert T.power_iteration(lambda v: m @ v, 20) == kt._power_iteration(lambda v: m @ v, 20)
    assert T.power_iteration(lambda v: 0.0 * v, 20) == 0.0


def test_oracle_constraint_algebra():
    """tests/test_tucker.py TestFactorWorkspace.test_projector_algebra restated on the oracle."""
    core, facs, _ = tucker_unit_inputs()
    ws = T.build_factor_workspace(core, facs, 1, 0.25, 0.1)
    nm = ws.constraint_projector()
    np.testing.assert_allclose(nm @ nm, nm, atol=1e-8)
    np.testing.assert_allclose(nm @ T.unfold(core, 1).T, 0.0, atol=1e-10)
    z = np.random.default_rng(0).standard_normal(nm.shape[0])
    assert np.linalg.norm(nm @ ws.project_feasible(z)) <= 1e-6 * np.linalg.norm(ws.project_feasible(z))
