"""Measure the reference's own numerical noise floor for the fast solver (writes floor.json).

FastKroneckerRegression runs 24 Richardson iterations on a system with condition number
~4e8..5e9, so the fast-path x and the step-norm history move far more than
1e-9 under perturbations that are all equally valid implementations of the reference
algorithm.  This script runs the oracle (bit-identical to the reference, pinned by
tests/test_oracle.py) under such variants and records the largest relative change of x, of
the history and of the loss against the reference golden fixtures:

  ulp_b      -- b perturbed by one ulp on 1% of its entries
  gram_order -- the approximate Gram A~^T A summed in a different order (einsum vs BLAS)
  eig_route  -- the Gram eigendecomposition through SVD instead of syevd
  inv_jl     -- the JL estimator through an explicit inverse (the GPU's formulation)
  combined   -- gram_order + eig_route + inv_jl

The GPU parity tests use tolerance = 2 x max(variant) (tests/test_gpu_solvers.py).
Run in the build container:  python tests/golden/measure_floor.py [c1 c2 c3 c4]

c4 (n = 65536, d in {16, 32, 64, 128}; b = default_rng(0).standard_normal(n^2), 34 GB) reads b
through the memmap of make_golden_c4.py and the oracle's ``b_at`` hook (the fast solve reads b
only at the sparse-diagonal rows); there ``ulp_b`` perturbs 1 % of the SAMPLED entries (the
others never enter the solve), and the loss is not re-evaluated (x and history floors only).
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import kronsolve_oracle as O  # noqa: E402

CASES = {"c1": (1024, 16), "c2": (4096, 32), "c3": (16384, 64)}
CFG = dict(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)


def fg_svd(a, assume_gram=False):
    a = np.asarray(a)
    gg = 0.5 * (a + a.T)
    _, s, vt = np.linalg.svd(gg)
    return np.ascontiguousarray(vt.T), s, gg


def jl_inverse(a, at, gt, eps, seed, lf=8.0, gram_order=False):
    if gram_order:
        gt = np.einsum("ij,ik->jk", at, at)
    gen = np.random.default_rng(seed)
    r = O.jl_rows(a.shape[0], lf)
    g = gen.standard_normal((r, at.shape[0])) / math.sqrt(r)
    q = (1.0 + eps / 4.0) * ((g @ at) @ np.linalg.inv(gt))
    proj = q @ a.T
    return np.einsum("ri,ri->i", proj, proj) / ((1.0 + eps / 4.0) * (1.0 - eps / 20.0)), 1.0 + eps / 2.0


def run(name, variant):
    b_at = None
    if name.startswith("c4"):
        import make_golden_c4 as MC
        d = int(name[4:])
        facs, bmm = MC.c4_factors(d), MC.c4_b()
        b = None

        def b_at(idx):
            v = np.asarray(bmm[idx], dtype=np.float64)
            if variant == "ulp_b":
                pick = np.random.default_rng(1).random(v.size) < 0.01
                v[pick] = np.nextafter(v[pick], np.inf)
            return v
    else:
        n, d = CASES[name]
        facs, b = O.synth_regression(n, d, 2, 0)
    fg0, jl0 = O.factor_gram, O.jl_scores
    try:
        if variant == "ulp_b" and b_at is None:
            rng = np.random.default_rng(1)
            pick = rng.random(b.size) < 0.01
            b = b.copy()
            b[pick] = np.nextafter(b[pick], 2.0)
        if variant == "gram_order":
            O.jl_scores = lambda a, at, gt, eps, seed, lf=8.0: jl0(a, at, np.einsum("ij,ik->jk", at, at), eps, seed, lf)
        if variant in ("eig_route", "combined"):
            O.factor_gram = fg_svd
        if variant == "inv_jl":
            O.jl_scores = jl_inverse
        if variant == "combined":
            O.jl_scores = lambda *a, **k: jl_inverse(*a, gram_order=True, **k)
        if b_at is not None:
            rep = O.fast_kronecker_regression(facs, None, with_loss=False, b_at=b_at, **CFG)
        else:
            rep = O.fast_kronecker_regression(facs, b, **CFG)
    finally:
        O.factor_gram, O.jl_scores = fg0, jl0
    return rep


def main(names):
    path = HERE / "floor.json"
    out = json.loads(path.read_text()) if path.exists() else {}
    for name in names:
        g = dict(np.load(HERE / (f"c4_d{name[4:]}.npz" if name.startswith("c4") else f"{name}.npz")))
        rows = {}
        for variant in ("ulp_b", "gram_order", "eig_route", "inv_jl", "combined"):
            rep = run(name, variant)
            h = np.asarray(rep.trace["history"])
            rows[variant] = {
                "x": float(np.linalg.norm(rep.solution - g["x"]) / np.linalg.norm(g["x"])),
                "history": float(np.max(np.abs(h / g["history"] - 1.0))),
                "loss": float(abs(rep.loss - float(g["loss"])) / float(g["loss"])) if np.isfinite(rep.loss) else None,
                "indices_equal": bool(np.array_equal(rep.trace["indices"], g["indices"])),
            }
            print(name, variant, rows[variant], flush=True)
        out[name] = {"variants": rows,
                     "x": max(r["x"] for r in rows.values()),
                     "history": max(r["history"] for r in rows.values()),
                     "loss": max((r["loss"] for r in rows.values() if r["loss"] is not None), default=None)}
        path.write_text(json.dumps(out, indent=1))


# ---------------------------------------------------------------------------------------------
# Floors of the other fast-path comparisons in the GPU tests (against the oracle, which is pinned
# to the reference): the mixed-width solves and the small sketched solves of test_gpu_solvers.py
# and the c5 fast Tucker core of test_gpu_tucker.py.  Floor = largest relative change of the
# result under the variants above (x; for the core, the core), against the unperturbed run.
# ---------------------------------------------------------------------------------------------

MIXED = [(3000, 2500, 16, 32), (2048, 2048, 64, 16), (2500, 2100, 24, 40), (1800, 1500, 48, 8)]


def _variant_solve(facs, b, params, variant):
    fg0, jl0 = O.factor_gram, O.jl_scores
    try:
        if variant == "ulp_b":
            rng = np.random.default_rng(1)
            pick = rng.random(b.size) < 0.01
            b = b.copy()
            b[pick] = np.nextafter(b[pick], np.inf)
        if variant == "gram_order":
            O.jl_scores = lambda a, at, gt, eps, seed, lf=8.0: jl0(a, at, np.einsum("ij,ik->jk", at, at), eps, seed, lf)
        if variant in ("eig_route", "combined"):
            O.factor_gram = fg_svd
        if variant == "inv_jl":
            O.jl_scores = jl_inverse
        if variant == "combined":
            O.jl_scores = lambda *a, **k: jl_inverse(*a, gram_order=True, **k)
        return O.fast_kronecker_regression(facs, b, with_loss=False, **params)
    finally:
        O.factor_gram, O.jl_scores = fg0, jl0


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def aux_floors():
    out = {}
    variants = ("ulp_b", "gram_order", "eig_route", "inv_jl", "combined")
    for n1, n2, d1, d2 in MIXED:  # test_fast_regression_mixed_widths_vs_oracle
        rs = np.random.default_rng(n1 + d1)
        facs = [rs.normal(1.0, math.sqrt(1e-3), (n1, d1)), rs.normal(1.0, math.sqrt(1e-3), (n2, d2))]
        b = rs.standard_normal(n1 * n2)
        params = dict(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=3)
        base = _variant_solve(facs, b, params, None).solution
        out[f"mixed_{n1}_{n2}_{d1}_{d2}"] = {"x": max(_rel(_variant_solve(facs, b, params, v).solution, base)
                                                       for v in variants)}
        print("mixed", n1, n2, d1, d2, out[f"mixed_{n1}_{n2}_{d1}_{d2}"], flush=True)
    small = 0.0
    for seed in range(5):  # test_fast_regression_small_cases
        rs = np.random.default_rng(seed + 1000)
        facs = [rs.normal(1.0, math.sqrt(1e-3), (20, 3)) for _ in range(2)]
        bb = rs.standard_normal(400)
        params = dict(eps=0.25, delta=0.05, lam=1e-3, seed=seed, alpha=2e-4)
        base = _variant_solve(facs, bb, params, None).solution
        small = max([small] + [_rel(_variant_solve(facs, bb, params, v).solution, base) for v in variants])
    out["small_sketched"] = {"x": small}
    print("small", small, flush=True)
    # c5 fast core (tucker.py:121-124 with caches = exact factor SVD + Gram eigendecomposition)
    x = O.synth_tucker((512, 512, 64), (16, 16, 4), 0.01, seed=0)
    facs = O.initial_tucker_factors(x.shape, (16, 16, 4), 0)
    core = O.core_update_exact(facs, x, 1e-3)
    del core
    kw = dict(eps=0.1, delta=0.01, alpha=1e-5, seed=0)
    g = dict(np.load(HERE / "c5.npz"))

    def fast_core(variant):
        xs = x
        fs = facs
        if variant == "ulp_factors":  # every stage sees a 1-ulp different input
            fs = [a.copy() for a in facs]
            for k, a in enumerate(fs):
                pick = np.random.default_rng(10 + k).random(a.shape) < 0.01
                a[pick] = np.nextafter(a[pick], np.inf)
        if variant == "ulp_b":
            pick = np.random.default_rng(1).random(x.size).reshape(x.shape) < 0.01
            xs = x.copy()
            xs[pick] = np.nextafter(xs[pick], np.inf)
        fg = fg_svd if variant in ("eig_route", "combined") else O.factor_gram
        caches = []
        for a in fs:
            m = np.einsum("ij,ik->jk", a, a) if variant in ("gram_order", "combined") else a.T @ a
            caches.append((O.compact_svd(a), fg(m, assume_gram=True)))
        return O.core_update_fast(fs, xs, 1e-3, caches, **kw)[0]

    base = fast_core(None)
    rows = {v: _rel(fast_core(v), g["core_fast"]) for v in ("ulp_b", "ulp_factors", "gram_order", "eig_route",
                                                             "combined")}
    rows["unperturbed_vs_golden"] = _rel(base, g["core_fast"])
    out["c5_fast_core"] = {"variants": rows, "core": max(rows.values())}
    print("c5 fast core", out["c5_fast_core"], flush=True)
    return out


if __name__ == "__main__":
    if sys.argv[1:] == ["aux"]:
        sys.path.insert(0, str(HERE))
        path = HERE / "floor.json"
        fl = json.loads(path.read_text())
        fl.update(aux_floors())
        path.write_text(json.dumps(fl, indent=1))
        sys.exit(0)
    sys.path.insert(0, str(HERE))
    main(sys.argv[1:] or list(CASES) + ["c4_d16", "c4_d32", "c4_d64", "c4_d128"])
