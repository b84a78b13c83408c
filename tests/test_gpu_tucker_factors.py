"""Tucker factor-matrix updates and the ALS driver on the GPU against the
reference-generated fixture tests/golden/tucker_units.npz and the oracle (oracle/tucker_oracle.py).

Tolerances: the exact update, the workspace and its applies are direct linear algebra (1e-9
relative).  The fast update runs a fixed number of Richardson steps (16 here) on problems whose
conditioning amplifies summation-order differences; its rows match to 1e-8 relative.  Sampled
indices and sketch values per row are compared exactly / to rounding."""

import math

import numpy as np
import pytest

from conftest import dense_kron, rel
from golden.tucker_inputs import ALS_CFG, UNIT_CFG, UNIT_LAM, UNIT_RANK, unit_inputs
from oracle import kronsolve_oracle as O
from oracle import tucker_oracle as T

pytestmark = pytest.mark.gpu


def K():
    import paper_2209_04876_b200 as k
    return k


def model_of(core, facs, lam=UNIT_LAM):
    return K().TuckerModel(core=core, factors=[a.copy() for a in facs], lam=lam)


@pytest.mark.parametrize("n", [0, 1, 2])
def test_factor_updates_match_reference_fixture(golden, n):
    g = golden("tucker_units")
    core, facs, x = unit_inputs()
    m = model_of(core, facs)
    assert rel(K().naive_factor_update(m, x, n), g[f"naive{n}"]) <= 1e-10
    ws = K().build_factor_workspace(m, n, 0.25, UNIT_LAM)
    assert ws.penalty_weight == pytest.approx(float(g[f"w{n}"]), rel=1e-10)
    z = np.arange(ws.g_n.shape[1], dtype=np.float64) / 7.0 - 0.3
    assert rel(ws.apply(z), g[f"apply{n}"]) <= 1e-10
    cfg = K().RegressionConfig(lam=UNIT_LAM, **UNIT_CFG)
    fast = K().fast_factor_matrix_update(m, x, n, cfg)
    assert rel(fast, g[f"fast{n}"]) <= 1e-8


@pytest.mark.parametrize("n", [0, 2])
def test_fast_update_sketch_and_iterations_match_oracle(n):
    import torch
    from paper_2209_04876_b200 import tucker as TK
    core, facs, x = unit_inputs()
    tr_o = {}
    T.fast_factor_matrix_update(core, facs, UNIT_LAM, x, n, T.Cfg(lam=UNIT_LAM, **UNIT_CFG), trace=tr_o)
    cfg = K().RegressionConfig(lam=UNIT_LAM, **UNIT_CFG)
    tr = {}
    dev = lambda a: torch.tensor(a, device="cuda")  # noqa: E731
    TK._fast_factor_update_dev(dev(core), [dev(a) for a in facs], UNIT_LAM, dev(x), n, cfg, None, trace=tr)
    assert tr["s"] == tr_o["s"]
    i_rest = x.size // x.shape[n]
    keys = tr["sd_idx"].cpu().numpy()
    vals = tr["sd_val"].cpu().numpy()
    iters = tr["iters"].cpu().numpy()
    hist = tr["hist"].cpu().numpy()
    for i, row in enumerate(tr_o["rows"]):
        sel = (keys >= i * i_rest) & (keys < (i + 1) * i_rest)
        np.testing.assert_array_equal(keys[sel] - i * i_rest, row["sd_indices"])
        np.testing.assert_allclose(vals[sel], row["sd_values"], rtol=1e-14)
        assert iters[i] == row["iters"]
        np.testing.assert_allclose(hist[i, :len(row["hist"])], row["hist"], rtol=1e-8)


def test_shared_sketch_and_caches_match_oracle():
    core, facs, x = unit_inputs()
    m = model_of(core, facs)
    caches = [K().build_factor_cache(a) for a in facs]
    cfg = K().RegressionConfig(lam=UNIT_LAM, share_row_sketch=True, **UNIT_CFG)
    got = K().fast_factor_matrix_update(m, x, 1, cfg, caches=caches)
    want = T.fast_factor_matrix_update(core, facs, UNIT_LAM, x, 1,
                                       T.Cfg(lam=UNIT_LAM, share_row_sketch=True, **UNIT_CFG),
                                       caches=[O.factor_cache(a) for a in facs])
    assert rel(got, want) <= 1e-8


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_tucker_als_matches_reference_fixture(golden, mode):
    g = golden("tucker_units")
    _, _, x = unit_inputs()
    cfg = K().RegressionConfig(seed=3) if mode == "exact" else K().RegressionConfig(**ALS_CFG)
    model, rep = K().tucker_als(x, UNIT_RANK, lam=UNIT_LAM, sweeps=2, solver_mode=mode, config=cfg)
    assert rep.step_labels[0] == "init-core" and len(rep.step_losses) == 1 + 2 * 4
    tol = 1e-9 if mode == "exact" else 1e-7
    np.testing.assert_allclose(rep.step_losses, g[f"als_{mode}_losses"], rtol=tol)
    assert rel(model.core, g[f"als_{mode}_core"]) <= (1e-8 if mode == "exact" else 1e-6)
    assert rep.rre == pytest.approx(rep.sweep_rres[-1], rel=1e-12)


def test_initial_model_is_lapack_qr():
    _, _, x = unit_inputs()
    m = K().initial_model(x, UNIT_RANK, 0.1, 3)
    want = O.initial_tucker_factors(x.shape, UNIT_RANK, 3)
    for a, b in zip(m.factors, want):
        np.testing.assert_allclose(a, b, atol=1e-13)
    assert not np.any(m.core)


def test_workspace_matches_dense_pinv():
    """tests/test_tucker.py TestFactorWorkspace.test_woodbury_matches_dense_pinv, on the device."""
    for seed in range(3):
        rng = np.random.default_rng(seed)
        rank = tuple(int(r) for r in rng.integers(2, 5, size=3))
        shape = tuple(int(r) + int(rng.integers(1, 4)) for r in rank)
        lam = float(rng.uniform(0, 0.5))
        core = rng.standard_normal(rank)
        facs = [rng.standard_normal((i, r)) for i, r in zip(shape, rank)]
        n = int(rng.integers(0, 3))
        ws = K().build_factor_workspace(model_of(core, facs, lam), n, eps=0.25, lam=lam)
        others = [a for k, a in enumerate(facs) if k != n]
        kk = dense_kron(others)
        g = T.unfold(core, n)
        gp = np.linalg.pinv(g)
        nm = np.eye(g.shape[1]) - g.T @ np.linalg.pinv(g.T)
        mm = kk.T @ kk + lam * gp @ gp.T + ws.penalty_weight * (nm.T @ nm)
        z = rng.standard_normal(g.shape[1])
        want = np.linalg.pinv(mm) @ z
        assert np.linalg.norm(ws.apply(z) - want) <= 1e-8 * max(1.0, np.linalg.norm(want))
        np.testing.assert_allclose(ws.constraint_projector() @ ws.constraint_projector(), ws.constraint_projector(),
                                   atol=1e-8)
        np.testing.assert_allclose(ws.apply_penalized_normal(z),
                                   kk.T @ kk @ z + ws.penalty_weight * z + gp @ ((lam * np.linalg.pinv(g.T) -
                                                                                 ws.penalty_weight * g) @ z),
                                   rtol=1e-9, atol=1e-9)


def test_fast_update_reference_properties():
    """test_tucker.py TestFastFactorUpdate: shortcut == naive when s >= I_rest; zero rows stay zero."""
    rng = np.random.default_rng(12345)
    x = rng.standard_normal((6, 6, 6))
    model, _ = K().tucker_als(x, (2, 2, 2), lam=0.0, sweeps=1, solver_mode="exact",
                              config=K().RegressionConfig(seed=5))
    cfg = K().RegressionConfig(eps=0.25, delta=0.05, lam=0.0, seed=6)
    np.testing.assert_allclose(K().fast_factor_matrix_update(model, x, 0, cfg), K().naive_factor_update(model, x, 0),
                               atol=1e-6)
    core, facs, x = unit_inputs()
    x = x.copy()
    x[2] = 0.0
    cfg = K().RegressionConfig(lam=UNIT_LAM, **UNIT_CFG)
    fast = K().fast_factor_matrix_update(model_of(core, facs), x, 0, cfg)
    np.testing.assert_allclose(fast[2], np.zeros(UNIT_RANK[0]), atol=1e-12)


def test_validation():
    from paper_2209_04876_b200.errors import InvalidInputError
    core, facs, x = unit_inputs()
    m = model_of(core, facs)
    with pytest.raises(InvalidInputError):
        K().fast_factor_matrix_update(m, x, 0, K().RegressionConfig(eps=0.35, seed=0))
    with pytest.raises(InvalidInputError):
        K().build_factor_workspace(m, 0, eps=0.4, lam=0.0)
    with pytest.raises(InvalidInputError):
        K().naive_factor_update(m, x, 5)
    zc = K().TuckerModel(core=np.zeros(UNIT_RANK), factors=facs, lam=0.1)
    with pytest.raises(InvalidInputError):
        K().build_factor_workspace(zc, 0, eps=0.25, lam=0.1)
    with pytest.raises(InvalidInputError):
        K().tucker_als(x, (50, 2, 2), sweeps=1)
    with pytest.raises(InvalidInputError):
        K().tucker_als(x, UNIT_RANK, solver_mode="bogus")


def test_c5_fast_factor_update_mode2_matches_oracle():
    """BASELINE config 5 shapes (512 x 512 x 64, rank (16, 16, 4)): the mode-2 update (64 rows,
    R_rest = 256, s = 3481 samples per row) against the oracle, and its rows' ridge quality."""
    x = O.synth_tucker((512, 512, 64), (16, 16, 4), 0.01, seed=0)
    facs = O.initial_tucker_factors(x.shape, (16, 16, 4), 0)
    core = O.core_update_exact(facs, x, 1e-3)
    cfg = dict(eps=0.1, delta=0.01, alpha=1e-5, seed=11)
    want = T.fast_factor_matrix_update(core, facs, 1e-3, x, 2, T.Cfg(lam=1e-3, **cfg))
    got = K().fast_factor_matrix_update(model_of(core, facs, 1e-3), x, 2, K().RegressionConfig(lam=1e-3, **cfg))
    assert rel(got, want) <= 1e-8
    naive = K().naive_factor_update(model_of(core, facs, 1e-3), x, 2)
    assert rel(naive, T.naive_factor_update(core, facs, 1e-3, x, 2)) <= 1e-10
    assert math.isfinite(float(np.sum(got)))


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_c5_als_sweep_matches_reference_fixture(golden, mode):
    """One ALS sweep at BASELINE config 5 against the reference's own run (tests/golden/c5_als.npz,
    make_golden.py c5als): step losses, final core, factor 2 and rre."""
    g = golden("c5_als")
    x = O.synth_tucker((512, 512, 64), (16, 16, 4), 0.01, seed=0)
    cfg = (K().RegressionConfig(eps=0.1, delta=0.01, alpha=1e-5, seed=0) if mode == "fast"
           else K().RegressionConfig(seed=0))
    model, rep = K().tucker_als(x, (16, 16, 4), lam=1e-3, sweeps=1, solver_mode=mode, config=cfg)
    tol = 1e-9 if mode == "exact" else 1e-7
    np.testing.assert_allclose(rep.step_losses, g[f"{mode}_losses"], rtol=tol)
    assert rep.rre == pytest.approx(float(g[f"{mode}_rre"]), rel=tol)
    assert rel(model.core, g[f"{mode}_core"]) <= 100 * tol
    assert rel(model.factors[2], g[f"{mode}_factor2"]) <= 100 * tol


@pytest.mark.parametrize("shape,rank,n", [((200, 150), (3, 2), 0), ((200, 150), (3, 2), 1),
                                          ((10, 9, 8, 7), (2, 3, 2, 2), 0), ((10, 9, 8, 7), (2, 3, 2, 2), 3)])
def test_fast_update_other_orders_match_oracle(shape, rank, n):
    """Order-2 models (one other factor: no right group) and order-4 models (three other factors:
    Khatri-Rao right rows) through the same row kernel, against the oracle."""
    rng = np.random.default_rng(len(shape) * 10 + n)
    core = rng.standard_normal(rank)
    facs = [np.linalg.qr(rng.standard_normal((i, r)))[0] for i, r in zip(shape, rank)]
    x = T.reconstruct(core, facs) + 0.05 * rng.standard_normal(shape)
    i_rest = x.size // x.shape[n]
    cfg = dict(eps=0.25, delta=0.05, alpha=1e-4, seed=5)
    s = T.factor_sample_count(int(np.prod([r for k, r in enumerate(rank) if k != n])), shape[n], T.Cfg(**cfg))
    assert s < i_rest  # the sketched path, not the exact shortcut
    want = T.fast_factor_matrix_update(core, facs, 0.02, x, n, T.Cfg(lam=0.02, **cfg))
    got = K().fast_factor_matrix_update(model_of(core, facs, 0.02), x, n, K().RegressionConfig(lam=0.02, **cfg))
    assert rel(got, want) <= 1e-8
