"""Solvers on the device vs the reference golden fixtures and the oracle.

Tolerances: loss <= 1e-9 relative; exact-path x <= 1e-9 relative; fast-path x
and the step-norm history within max(1e-9, 2x the reference's own noise floor) -- the floors are
measured by tests/golden/measure_floor.py (floor.json: c1-c3 against the reference fixtures, the
mixed-width and small sketched cases against the oracle); iterations and sample counts equal;
sampled indices bit-exact."""

import json
import math
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import dense_kron, rel
from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu

CASES = {"c1": (1024, 16), "c2": (4096, 32), "c3": (16384, 64)}
FLOOR = json.loads((Path(__file__).resolve().parent / "golden" / "floor.json").read_text())
X_TOL = {k: 2 * FLOOR[k]["x"] for k in CASES}        # 2x the reference's own noise floor (measure_floor.py)
H_TOL = {k: 2 * FLOOR[k]["history"] for k in CASES}


def cfg(**kw):
    import paper_2209_04876_b200 as K
    base = dict(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
    base.update(kw)
    return K.RegressionConfig(**base)


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_fast_regression_matches_reference(golden, name):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.solvers import FastSolveTrace
    n, d = CASES[name]
    g = golden(name)
    facs, b = O.synth_regression(n, d, 2, 0)
    tr = FastSolveTrace()
    rep = K.fast_kronecker_regression(facs, b, cfg(), _trace=tr)
    assert rep.sample_count == int(g["s"])
    assert rep.iterations == int(g["iterations"])
    np.testing.assert_array_equal(tr.sketch.indices.cpu().numpy(), g["indices"].astype(np.int64))
    # weights carry the JL score differences (gram inverse: ~kappa*u); indices are bit-exact
    np.testing.assert_allclose(tr.sketch.weights.cpu().numpy(), g["weights"], rtol=1e-10)
    np.testing.assert_array_equal(tr.sdiag.indices.cpu().numpy(), g["sd_indices"])
    np.testing.assert_allclose(tr.sdiag.values.cpu().numpy(), g["sd_values"], rtol=1e-10)
    assert rel(tr.rhs, g["rhs"]) <= 1e-10
    assert rel(rep.solution, g["x"]) <= max(1e-9, X_TOL[name])
    assert abs(rep.loss - float(g["loss"])) <= 1e-9 * float(g["loss"])
    h = np.asarray(tr.history)
    assert h.size == g["history"].size
    assert np.max(np.abs(h - g["history"]) / g["history"]) <= max(1e-9, H_TOL[name])
    assert rep.wall_time > 0


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_exact_solver_matches_reference(golden, name):
    import paper_2209_04876_b200 as K
    n, d = CASES[name]
    g = golden(name)
    facs, b = O.synth_regression(n, d, 2, 0)
    rep = K.kronmatmul_svd_solve(facs, b, 1e-3)
    assert rel(rep.solution, g["exact_x"]) <= 1e-9
    assert abs(rep.loss - float(g["opt"])) <= 1e-9 * float(g["opt"])


def test_device_resident_inputs_return_device(golden):
    import paper_2209_04876_b200 as K
    g = golden("c1")
    facs, b = O.synth_regression(1024, 16, 2, 0)
    fd = [torch.tensor(a, device="cuda") for a in facs]
    bd = torch.tensor(b, device="cuda")
    rep = K.fast_kronecker_regression(fd, bd, cfg())
    assert isinstance(rep.solution, torch.Tensor) and rep.solution.is_cuda
    assert rel(rep.solution, g["x"]) <= X_TOL["c1"]


def test_ridge_loss(rng):
    import paper_2209_04876_b200 as K
    facs = [rng.standard_normal((5, 2)), rng.standard_normal((4, 3))]
    k = dense_kron(facs)
    b = rng.standard_normal(20)
    x = rng.standard_normal(6)
    want = np.sum((k @ x - b) ** 2) + 0.05 * x @ x
    assert K.ridge_loss(facs, x, b, 0.05) == pytest.approx(want, rel=1e-10)
    assert K.ridge_loss(facs, np.zeros(6), b, 0.7) == pytest.approx(b @ b)
    facs3 = [rng.standard_normal((6, 2)), rng.standard_normal((5, 3)), rng.standard_normal((4, 2))]
    k3 = dense_kron(facs3)
    b3 = rng.standard_normal(120)
    x3 = rng.standard_normal(12)
    assert K.ridge_loss(facs3, x3, b3, 0.1) == pytest.approx(np.sum((k3 @ x3 - b3) ** 2) + 0.1 * x3 @ x3, rel=1e-10)


def test_exact_solvers_small(rng):
    import paper_2209_04876_b200 as K
    b = rng.standard_normal(6)
    rep = K.kronmatmul_svd_solve([np.eye(2), np.eye(3)], b, 0.4)
    np.testing.assert_allclose(rep.solution, b / 1.4, atol=1e-10)
    for lam in (0.0, 1e-3, 1.0):
        facs = [rng.standard_normal((8, 3)), rng.standard_normal((6, 2))]
        bb = rng.standard_normal(48)
        r1 = O.kronmatmul_svd_solve(facs, bb, lam)
        r2 = K.kronmatmul_svd_solve(facs, bb, lam)
        np.testing.assert_allclose(r2.solution, r1.solution, atol=1e-10)
        assert r2.loss == pytest.approx(r1.loss, rel=1e-10)
    facs3 = [rng.standard_normal((6, 2)), rng.standard_normal((5, 3)), rng.standard_normal((4, 2))]
    b3 = rng.standard_normal(120)
    np.testing.assert_allclose(K.kronmatmul_svd_solve(facs3, b3, 0.01).solution,
                               O.kronmatmul_svd_solve(facs3, b3, 0.01).solution, atol=1e-10)


def test_fast_regression_small_cases(rng):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.errors import InvalidInputError
    b = rng.standard_normal(6)
    rep = K.fast_kronecker_regression([np.eye(2), np.eye(3)], b, K.RegressionConfig(seed=0))
    np.testing.assert_allclose(rep.solution, b, atol=1e-10)
    with pytest.raises(InvalidInputError):
        K.fast_kronecker_regression([np.zeros((3, 2)), np.eye(2)], rng.standard_normal(6), K.RegressionConfig(seed=0))
    with pytest.raises(InvalidInputError):
        K.fast_kronecker_regression([rng.standard_normal((4, 2))], rng.standard_normal(4),
                                    K.RegressionConfig(eps=0.5, seed=0))
    # sketched path at small scale: same result as the oracle (same streams)
    for seed in range(5):
        rs = np.random.default_rng(seed + 1000)
        facs = [rs.normal(1.0, math.sqrt(1e-3), (20, 3)) for _ in range(2)]
        bb = rs.standard_normal(400)
        c = K.RegressionConfig(eps=0.25, delta=0.05, lam=1e-3, seed=seed, alpha=2e-4)
        r = K.fast_kronecker_regression(facs, bb, c)
        o = O.fast_kronecker_regression(facs, bb, eps=0.25, delta=0.05, lam=1e-3, seed=seed, alpha=2e-4)
        assert r.sample_count == o.sample_count and r.iterations == o.iterations
        assert rel(r.solution, o.solution) <= 2 * FLOOR["small_sketched"]["x"]  # measure_floor.py aux
        assert r.loss == pytest.approx(o.loss, rel=1e-9)


def test_fast_regression_scale_equivariance_and_caches(rng):
    import paper_2209_04876_b200 as K
    facs = [rng.standard_normal((12, 2)), rng.standard_normal((10, 2))]
    b = rng.standard_normal(120)
    c = K.RegressionConfig(eps=0.25, delta=0.1, lam=1e-3, seed=11, alpha=1e-3)
    r1 = K.fast_kronecker_regression(facs, b, c)
    r2 = K.fast_kronecker_regression(facs, 3.0 * b, c)
    assert r1.sample_count == r2.sample_count
    np.testing.assert_allclose(r2.solution, 3.0 * r1.solution, rtol=1e-9, atol=1e-12)
    facs = [rng.standard_normal((15, 2)), rng.standard_normal((12, 3))]
    b = rng.standard_normal(180)
    caches = [K.build_factor_cache(a) for a in facs]
    c = K.RegressionConfig(eps=0.25, delta=0.1, lam=1e-2, seed=4, alpha=1e-3)
    rep = K.fast_kronecker_regression(facs, b, c, caches=caches)
    o = O.fast_kronecker_regression(facs, b, eps=0.25, delta=0.1, lam=1e-2, seed=4, alpha=1e-3,
                                    caches=[O.factor_cache(a) for a in facs])
    assert rel(rep.solution, o.solution) <= 1e-8
    assert rep.loss <= 1.3 * O.kronmatmul_svd_solve(facs, b, 1e-2).loss


def test_richardson_generic(rng):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.errors import NumericalFailureError
    a = rng.standard_normal((8, 3))
    b = rng.standard_normal(8)
    ata = a.T @ a
    inv = np.linalg.inv(ata)
    x, it = K.richardson_solve(lambda v: ata @ v, lambda v: inv @ v, a.T @ b, 1.0, K.RegressionConfig(eps=0.25))
    assert it == 1
    bad = -inv
    with pytest.raises(NumericalFailureError) as err:
        K.richardson_solve(lambda v: ata @ v, lambda v: bad @ v, rng.standard_normal(3), 1.0,
                           K.RegressionConfig(eps=0.25, max_richardson_iters=50, residual_tol=1e-300))
    assert "residual_history" in err.value.diagnostics


def test_fused_richardson_divergence_rule(golden):
    """The device loop applies the reference's divergence rule (solvers.py:236-243)."""
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.errors import NumericalFailureError
    facs, b = O.synth_regression(1024, 16, 2, 0)
    with pytest.raises(NumericalFailureError) as err:
        K.fast_kronecker_regression(facs, b, cfg(damping=-1.0, max_richardson_iters=60))
    hist = err.value.diagnostics["residual_history"]
    assert len(hist) >= 6 and hist[-1] > 10 * hist[-6]
    with pytest.raises(O.OracleError) as oerr:
        O.fast_kronecker_regression(facs, b, eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0, damping=-1.0,
                                    max_iters=60)
    assert oerr.value.kind == "numerical" and oerr.value.iterations == err.value.iterations


def test_graph_replay_matches_eager(golden):
    """The JL/sampling stage is captured in a CUDA graph on the second solve with the same
    buffers and replayed afterwards; every solve must equal the eager one bit for bit."""
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    g = golden("c2")
    facs, b = O.synth_regression(4096, 32, 2, 0)
    fd = [torch.tensor(a, device="cuda") for a in facs]
    bd = torch.tensor(b, device="cuda")
    S._USE_GRAPHS[0] = False
    try:
        ref = K.fast_kronecker_regression(fd, bd, cfg())
    finally:
        S._USE_GRAPHS[0] = True
    S._PREFIX_GRAPHS.clear()
    S._USE_SOLVE_GRAPH[0] = False  # exercise the stage graph (used when the whole solve is not graphed)
    try:
        outs = [K.fast_kronecker_regression(fd, bd, cfg()) for _ in range(4)]  # eager, capture, replay x2
    finally:
        S._USE_SOLVE_GRAPH[0] = True
    assert any(e.graph is not None for e in S._PREFIX_GRAPHS.values())
    for rep in outs:
        assert rep.iterations == ref.iterations
        assert torch.equal(rep.solution, ref.solution)
    assert rel(outs[-1].solution, g["x"]) <= X_TOL["c2"]
    # the replayed stage reads the factors' current contents: a scaled factor changes the answer
    # exactly like an eager solve of the scaled problem
    fd[0].mul_(2.0)
    S._USE_SOLVE_GRAPH[0] = False
    try:
        rep2 = K.fast_kronecker_regression(fd, bd, cfg())
    finally:
        S._USE_SOLVE_GRAPH[0] = True
    S._USE_GRAPHS[0] = False
    try:
        ref2 = K.fast_kronecker_regression(fd, bd, cfg())
    finally:
        S._USE_GRAPHS[0] = True
    assert torch.equal(rep2.solution, ref2.solution)


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_fused_rhs_loop_matches_separate_rhs(name):
    """The fused launch (right-hand side + dinv built inside the persistent loop kernel) and the
    separate transpose-apply + loop path agree to rounding."""
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    from paper_2209_04876_b200.solvers import FastSolveTrace
    n, d = CASES[name]
    facs, b = O.synth_regression(n, d, 2, 0)
    t1, t2 = FastSolveTrace(), FastSolveTrace()
    r1 = K.fast_kronecker_regression(facs, b, cfg(), _trace=t1)
    S._USE_FUSED[0] = False
    try:
        r2 = K.fast_kronecker_regression(facs, b, cfg(), _trace=t2)
    finally:
        S._USE_FUSED[0] = True
    assert r1.iterations == r2.iterations
    assert rel(t1.rhs, t2.rhs) <= 1e-13
    # kappa(K^T K + lam I) ~ 1e8-1e9 amplifies the rhs rounding: compare at the measured floor
    assert rel(r1.solution, r2.solution) <= X_TOL[name]


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_whole_solve_graph_matches_eager(golden, name):
    """Two-factor solves with device-resident or page-locked host b run as one captured CUDA
    graph from the second call on; results equal the eager (trace) pipeline bit for bit and the
    reference golden x / step-norm history / loss (c3 is the configuration bench.py times)."""
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    from paper_2209_04876_b200.solvers import FastSolveTrace
    n, d = CASES[name]
    g = golden(name)
    facs, b = O.synth_regression(n, d, 2, 0)
    fd = [torch.tensor(a, device="cuda") for a in facs]
    bd = torch.tensor(b, device="cuda")
    ref = K.fast_kronecker_regression(fd, bd, cfg(), _trace=FastSolveTrace())  # eager
    S._SOLVE_GRAPHS.clear()
    before = dict(S._SOLVE_STATS)
    outs = [K.fast_kronecker_regression(fd, bd, cfg()) for _ in range(4)]
    assert S._SOLVE_STATS["capture"] == before["capture"] + 1
    assert S._SOLVE_STATS["replay"] >= before["replay"] + 2
    for rep in outs:
        assert rep.iterations == ref.iterations
        assert torch.equal(rep.solution, ref.solution)
    assert rel(outs[-1].solution, g["x"]) <= X_TOL[name]
    assert outs[-1].iterations == int(g["iterations"]) and outs[-1].sample_count == int(g["s"])
    h = np.asarray(S.last_solve_history())  # the replayed graph's step norms
    assert h.size == g["history"].size
    assert np.max(np.abs(h - g["history"]) / g["history"]) <= max(1e-9, H_TOL[name])
    assert abs(outs[-1].loss - float(g["loss"])) <= 1e-9 * float(g["loss"])
    # page-locked host b: the graph gathers the sampled entries through mapped host memory
    bh = torch.tensor(b).pin_memory()
    hs = [K.fast_kronecker_regression(fd, bh, cfg()) for _ in range(3)]
    for rep in hs:
        assert rep.iterations == ref.iterations
        np.testing.assert_array_equal(np.asarray(rep.solution), ref.solution.cpu().numpy())


def test_host_pinned_factor_graph_matches_device_path():
    """Page-locked host factors and b: the third and later calls replay one graph that also holds
    the factor uploads and their validation; the result equals the device-resident path bit for bit,
    and invalid factors still raise the reference's error."""
    import torch
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    from paper_2209_04876_b200.errors import InvalidInputError
    n, d = 4096, 32
    rng = np.random.default_rng(0)
    facs_h = [rng.normal(1.0, np.sqrt(1e-3), (n, d)) for _ in range(2)]
    cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
    facs_pin = [torch.from_numpy(a).pin_memory() for a in facs_h]
    b_pin = torch.ones(n * n, dtype=torch.float64).pin_memory()
    dev = K.fast_kronecker_regression([torch.tensor(a, device="cuda") for a in facs_h],
                                      torch.ones(n * n, dtype=torch.float64, device="cuda"), cfg)
    outs = [K.fast_kronecker_regression(facs_pin, b_pin, cfg) for _ in range(3)]
    assert any(k[0] == "host" for k in S._HOST_GRAPHS) and any(e.graph is not None for e in S._HOST_GRAPHS.values())
    for r in outs:
        np.testing.assert_array_equal(np.asarray(r.solution), dev.solution.cpu().numpy())
        assert r.iterations == dev.iterations and r.loss == pytest.approx(dev.loss, rel=1e-12)
    facs_pin[1][5, 3] = float("nan")
    with pytest.raises(InvalidInputError, match="factor 1 contains non-finite"):
        K.fast_kronecker_regression(facs_pin, b_pin, cfg)
    facs_pin[1][5, 3] = float("inf")
    with pytest.raises(InvalidInputError, match="factor 1 contains non-finite"):
        K.fast_kronecker_regression(facs_pin, b_pin, cfg)
    facs_pin[1][5, 3] = 1.0
    keep = facs_pin[0].clone()
    facs_pin[0].zero_()
    with pytest.raises(InvalidInputError, match="factor 0 is identically zero"):
        K.fast_kronecker_regression(facs_pin, b_pin, cfg)
    facs_pin[0].copy_(keep)
    facs_pin[1][5, 3] = 1.0
    r = K.fast_kronecker_regression(facs_pin, b_pin, cfg)  # the graph is still usable afterwards
    assert np.all(np.isfinite(np.asarray(r.solution)))


def test_device_graph_replay_validates_in_graph():
    """Device-resident inputs: once the whole-solve graph is captured, later calls replay it with the
    factor validation as a graph node (no synchronising pre-check); new invalid contents at the same
    addresses still raise the reference's errors, and valid contents give the eager result."""
    import torch
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    from paper_2209_04876_b200.errors import InvalidInputError
    n, d = 4096, 32
    rng = np.random.default_rng(1)
    facs = [torch.tensor(rng.normal(1.0, np.sqrt(1e-3), (n, d)), device="cuda") for _ in range(2)]
    b = torch.tensor(rng.standard_normal(n * n), device="cuda")
    c = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
    S._SOLVE_GRAPHS.clear()
    outs = [K.fast_kronecker_regression(facs, b, c) for _ in range(4)]
    key = S._solve_graph_key(facs, b, c)
    assert key is not None and S._SOLVE_GRAPHS[key].graph is not None
    for r in outs[1:]:
        assert torch.equal(r.solution, outs[0].solution) and r.iterations == outs[0].iterations
    replays = S._SOLVE_STATS["replay"]
    facs[1][7, 2] = float("nan")
    with pytest.raises(InvalidInputError, match="factor 1 contains non-finite"):
        K.fast_kronecker_regression(facs, b, c)
    facs[1][7, 2] = float("-inf")
    with pytest.raises(InvalidInputError, match="factor 1 contains non-finite"):
        K.fast_kronecker_regression(facs, b, c)
    assert S._SOLVE_STATS["replay"] == replays + 2  # both rejected by the in-graph check
    facs[1][7, 2] = 1.0
    keep = facs[0].clone()
    facs[0].zero_()
    with pytest.raises(InvalidInputError, match="factor 0 is identically zero"):
        K.fast_kronecker_regression(facs, b, c)
    facs[0].copy_(keep)
    facs[1][7, 2] = outs[0].solution.new_tensor(0.0) + float(np.asarray(rng.normal(1.0, 0.0316)))
    r = K.fast_kronecker_regression(facs, b, c)
    S._SOLVE_GRAPHS.clear()
    e = K.fast_kronecker_regression(facs, b, c)  # eager (first sight of the key)
    assert torch.equal(r.solution, e.solution) and r.iterations == e.iterations


def test_spectral_branch_graph_matches_eager_and_oracle():
    """n = 16384, d = 16: per-factor spectral row sampling is active (s_n < n).  The whole-solve graph
    (spectral rows, Grams, eigensolves and JL chains per factor on their own streams) equals the
    eager pipeline bit for bit, and its sketch equals the oracle's."""
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    from paper_2209_04876_b200.solvers import FastSolveTrace
    n, d = 16384, 16
    facs, _ = O.synth_regression(n, d, 2, 0)
    b = np.random.default_rng(5).standard_normal(n * n)
    fd = [torch.tensor(a, device="cuda") for a in facs]
    bd = torch.tensor(b, device="cuda")
    tr = FastSolveTrace()
    ref = K.fast_kronecker_regression(fd, bd, cfg(), _trace=tr)  # eager
    assert all(r < n for r in tr.a_tilde_rows)  # spectral branch
    oref = O.fast_kronecker_regression(facs, b, with_loss=False, eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
    np.testing.assert_array_equal(tr.sdiag.indices.cpu().numpy(), oref.trace["sd_indices"])
    assert ref.iterations == oref.iterations
    S._SOLVE_GRAPHS.clear()
    before = dict(S._SOLVE_STATS)
    outs = [K.fast_kronecker_regression(fd, bd, cfg()) for _ in range(4)]
    assert S._SOLVE_STATS["capture"] == before["capture"] + 1
    for rep in outs:
        assert rep.iterations == ref.iterations
        assert torch.equal(rep.solution, ref.solution)


@pytest.mark.parametrize("n1,n2,d1,d2", [(3000, 2500, 16, 32), (2048, 2048, 64, 16), (2500, 2100, 24, 40),
                                         (1800, 1500, 48, 8)])
def test_fast_regression_mixed_widths_vs_oracle(n1, n2, d1, d2):
    """Unequal factor shapes: graph + persistent-loop paths (widths 16/32/64, any pairing) and the
    per-iteration path (other widths), against the oracle; later calls (graph replays) repeat the
    first call's result bit for bit."""
    import paper_2209_04876_b200 as K
    rs = np.random.default_rng(n1 + d1)
    facs = [rs.normal(1.0, math.sqrt(1e-3), (n1, d1)), rs.normal(1.0, math.sqrt(1e-3), (n2, d2))]
    b = rs.standard_normal(n1 * n2)
    c = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=3)
    fd = [torch.tensor(a, device="cuda") for a in facs]
    bd = torch.tensor(b, device="cuda")
    reps = [K.fast_kronecker_regression(fd, bd, c) for _ in range(3)]
    o = O.fast_kronecker_regression(facs, b, eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=3, with_loss=False)
    for r in reps:
        assert r.sample_count == o.sample_count and r.iterations == o.iterations
        assert torch.equal(r.solution, reps[0].solution)
    assert rel(reps[0].solution, o.solution) <= 2 * FLOOR[f"mixed_{n1}_{n2}_{d1}_{d2}"]["x"]  # measure_floor.py aux


def test_concurrent_solves_on_threads_match_serial():
    """SPEC.md:394 / experiments.py:196-198: independent solves may run concurrently on threads.
    Four solves (different seeds / inputs) from a thread pool, each thread on its own stream and
    each repeated so that its whole-solve graph is captured and replayed while the other threads
    run, reproduce the serial results bit for bit; NumPy inputs on threads as well."""
    from concurrent.futures import ThreadPoolExecutor
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    n, d = 4096, 32
    probs = []
    for k in range(4):
        rs = np.random.default_rng(100 + k)
        facs = [rs.normal(1.0, math.sqrt(1e-3), (n, d)) for _ in range(2)]
        probs.append((facs, rs.standard_normal(n * n), cfg(seed=k)))
    dev = [([torch.tensor(a, device="cuda") for a in f], torch.tensor(b, device="cuda"), c) for f, b, c in probs]
    serial = [K.fast_kronecker_regression(f, b, c, with_loss=False) for f, b, c in dev]
    serial_hist = []
    for f, b, c in dev:
        K.fast_kronecker_regression(f, b, c, with_loss=False)
        serial_hist.append(S.last_solve_history())

    def work(k):
        f, b, c = dev[k]
        st = torch.cuda.Stream()
        outs = []
        with torch.cuda.stream(st):
            for _ in range(4):  # eager, capture, replays
                r = K.fast_kronecker_regression(f, b, c, with_loss=False)
                outs.append((r.solution.clone(), r.iterations, S.last_solve_history()))
        st.synchronize()
        return outs

    with ThreadPoolExecutor(4) as ex:
        got = list(ex.map(work, range(4)))
    for k in range(4):
        for x, it, h in got[k]:
            assert it == serial[k].iterations
            assert torch.equal(x, serial[k].solution)
            assert h == serial_hist[k]
    # NumPy inputs (eager path with host gathers) on threads
    with ThreadPoolExecutor(4) as ex:
        host = list(ex.map(lambda k: K.fast_kronecker_regression(probs[k][0], probs[k][1], probs[k][2],
                                                                  with_loss=False), range(4)))
    for k in range(4):
        np.testing.assert_array_equal(host[k].solution, serial[k].solution.cpu().numpy())


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_exact_solve_graph_matches_eager(golden, name):
    """kronmatmul_svd_solve with device-resident inputs: first call eager (records the factors'
    numerical ranks), then one captured graph replayed with the factors copied into its own buffers
    -- bit-identical to the eager solve, equal to the reference's exact x / loss, and a replay on NEW
    factor tensors of the same shapes (the Tucker ALS pattern) equals the eager solve on them."""
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    n, d = CASES[name]
    g = golden(name)
    facs, b = O.synth_regression(n, d, 2, 0)
    fd = [torch.tensor(a, device="cuda") for a in facs]
    bd = torch.tensor(b, device="cuda")
    S._EXACT_GRAPHS.clear()
    S._USE_GRAPHS[0] = False
    try:
        ref = K.kronmatmul_svd_solve(fd, bd, 1e-3)  # eager
    finally:
        S._USE_GRAPHS[0] = True
    outs = [K.kronmatmul_svd_solve(fd, bd, 1e-3) for _ in range(3)]  # eager (ranks), capture, replay
    assert len(S._EXACT_GRAPHS) == 1 and next(iter(S._EXACT_GRAPHS.values())).graph is not None
    for rep in outs:
        assert torch.equal(rep.solution, ref.solution)
        assert rep.loss == ref.loss
    assert rel(outs[-1].solution, g["exact_x"]) <= 1e-9
    assert abs(outs[-1].loss - float(g["opt"])) <= 1e-9 * float(g["opt"])
    # new factor tensors, same shapes: the replay copies them in
    f2 = [a * 1.5 + 0.01 for a in fd]
    got = K.kronmatmul_svd_solve(f2, bd, 1e-3)
    S._USE_GRAPHS[0] = False
    try:
        want = K.kronmatmul_svd_solve(f2, bd, 1e-3)
    finally:
        S._USE_GRAPHS[0] = True
    assert torch.equal(got.solution, want.solution) and got.loss == want.loss
    # the validation rides in the graph: a replay on non-finite / all-zero factors raises the
    # reference's errors (solvers.py:265-274)
    from paper_2209_04876_b200.errors import InvalidInputError
    bad = fd[0].clone()
    bad[3, 1] = float("nan")
    with pytest.raises(InvalidInputError, match="factor 0 contains non-finite entries"):
        K.kronmatmul_svd_solve([bad, fd[1]], bd, 1e-3)
    with pytest.raises(InvalidInputError, match="factor 1 is identically zero"):
        K.kronmatmul_svd_solve([fd[0], torch.zeros_like(fd[1])], bd, 1e-3)


def test_exact_solve_loss_identity(rng):
    """With a noisy b (loss ~ ||b||^2) the replayed exact solve takes its loss from the ||b||^2 of
    the K1 pass and the exact-solution identity ||b||^2 - sum s^2 t^2 / (s^2 + lam) (no second pass
    over b); it agrees with the direct ridge_loss pass to 1e-12."""
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    n, d = 2048, 16
    facs = [torch.tensor(rng.normal(1.0, math.sqrt(1e-3), (n, d)), device="cuda") for _ in range(2)]
    bd = torch.tensor(rng.standard_normal(n * n), device="cuda")
    S._EXACT_GRAPHS.clear()
    reps = [K.kronmatmul_svd_solve(facs, bd, 1e-3) for _ in range(3)]  # eager, capture, replay
    entry = next(iter(S._EXACT_GRAPHS.values()))
    assert entry.graph is not None and entry.identity
    direct = K.ridge_loss(facs, reps[-1].solution, bd, 1e-3)
    for rep in reps:
        assert abs(rep.loss - direct) <= 1e-12 * direct
    assert torch.equal(reps[1].solution, reps[0].solution) and torch.equal(reps[2].solution, reps[0].solution)


def test_exact_solve_graph_declined_cholqr_and_no_loss(rng):
    """An ill-conditioned factor (kappa^2 > 1e12: CholeskyQR2 declines) makes the captured exact solve
    fall back to the eager Householder path -- results equal the eager solve bit for bit; with
    with_loss=False (core_update's case) the solution is the same and the loss is nan."""
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    n, d = 2048, 16
    a0 = rng.standard_normal((n, d))
    a0[:, 3] = a0[:, 2] + 1e-9 * rng.standard_normal(n)  # nearly dependent columns
    facs = [torch.tensor(a0, device="cuda"), torch.tensor(rng.normal(1.0, 0.03, (n, d)), device="cuda")]
    bd = torch.tensor(rng.standard_normal(n * n), device="cuda")
    S._USE_GRAPHS[0] = False
    try:
        ref = K.kronmatmul_svd_solve(facs, bd, 1e-3)
    finally:
        S._USE_GRAPHS[0] = True
    S._EXACT_GRAPHS.clear()
    outs = [K.kronmatmul_svd_solve(facs, bd, 1e-3) for _ in range(3)]
    for rep in outs:
        assert torch.equal(rep.solution, ref.solution) and rep.loss == ref.loss
    nl = K.kronmatmul_svd_solve(facs, bd, 1e-3, with_loss=False)
    assert torch.equal(nl.solution, ref.solution) and math.isnan(nl.loss)


def test_exact_solve_graph_noncontiguous_factors(rng):
    """Non-contiguous device factors (transposed views) go through the graph path's row-major copies
    and give the eager solve's result."""
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import solvers as S
    n, d = 1024, 16
    facs = [torch.tensor(rng.normal(1.0, 0.03, (d, n)), device="cuda").T for _ in range(2)]
    assert not facs[0].is_contiguous()
    bd = torch.tensor(rng.standard_normal(n * n), device="cuda") * 1e-3 + 1.0  # a near fit: the direct loss pass
    S._USE_GRAPHS[0] = False
    try:
        ref = K.kronmatmul_svd_solve(facs, bd, 1e-3)
    finally:
        S._USE_GRAPHS[0] = True
    S._EXACT_GRAPHS.clear()
    outs = [K.kronmatmul_svd_solve(facs, bd, 1e-3) for _ in range(3)]
    for rep in outs:
        assert torch.equal(rep.solution, ref.solution)
        assert abs(rep.loss - ref.loss) <= 1e-12 * ref.loss
