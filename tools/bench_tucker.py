"""Time the Tucker factor-matrix updates and a fast-mode ALS sweep at BASELINE config 5
(512 x 512 x 64 tensor, rank (16, 16, 4), lam 1e-3, eps 0.1, delta 0.01, alpha 1e-5).

    python tools/bench_tucker.py [--cpu] [--sweeps K]

Prints one JSON line: per-mode GPU times of fast_factor_matrix_update (device-resident inputs,
median of 5 after warm-up, host wall clock around a synchronised call) and of naive_factor_update,
the per-sweep time of tucker_als(solver_mode="fast"), and with --cpu the oracle port's times on the
host cores for the same calls (one run each)."""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2209_04876_b200 as K  # noqa: E402
from paper_2209_04876_b200 import tucker as TK  # noqa: E402


def synth(shape, rank, noise, seed):
    """experiments.py:118-131 construction (as oracle.synth_tucker), generated on the host."""
    from oracle import kronsolve_oracle as O
    return O.synth_tucker(shape, rank, noise, seed)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--sweeps", type=int, default=2)
    args = ap.parse_args()
    shape, rank, lam = (512, 512, 64), (16, 16, 4), 1e-3
    x = synth(shape, rank, 0.01, 0)
    xd = torch.tensor(x, device="cuda")
    m0 = K.initial_model(xd, rank, lam, 0)
    m0.core = TK.core_update(m0, xd, mode="exact")
    caches = [K.build_factor_cache(a) for a in m0.factors]
    cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=lam, alpha=1e-5, seed=7)
    out = {"config": "c5: 512x512x64, rank (16,16,4), lam=1e-3, eps=0.1, delta=0.01, alpha=1e-5"}
    for n in range(3):
        out[f"fast_mode{n}_s"] = timed(lambda: K.fast_factor_matrix_update(m0, xd, n, cfg, caches=caches))
        out[f"naive_mode{n}_s"] = timed(lambda: K.naive_factor_update(m0, xd, n))
    t0 = time.perf_counter()
    _, rep = K.tucker_als(xd, rank, lam=lam, sweeps=args.sweeps, solver_mode="fast",
                          config=K.RegressionConfig(eps=0.1, delta=0.01, alpha=1e-5, seed=0))
    out["als_fast_total_s"] = time.perf_counter() - t0
    out["als_fast_sweep_s"] = rep.sweep_seconds
    out["als_fast_rre"] = rep.rre
    t0 = time.perf_counter()
    _, rep = K.tucker_als(xd, rank, lam=lam, sweeps=args.sweeps, solver_mode="exact",
                          config=K.RegressionConfig(seed=0))
    out["als_exact_total_s"] = time.perf_counter() - t0
    out["als_exact_rre"] = rep.rre
    if args.cpu:
        from oracle import kronsolve_oracle as O
        from oracle import tucker_oracle as T
        core = m0.core.cpu().numpy()
        facs = [a.cpu().numpy() for a in m0.factors]
        oc = [O.factor_cache(a) for a in facs]
        for n in range(3):
            t0 = time.perf_counter()
            T.fast_factor_matrix_update(core, facs, lam, x, n, T.Cfg(lam=lam, eps=0.1, delta=0.01, alpha=1e-5, seed=7),
                                        caches=oc)
            out[f"cpu_fast_mode{n}_s"] = time.perf_counter() - t0
        out["cpu_threads"] = os.cpu_count()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
