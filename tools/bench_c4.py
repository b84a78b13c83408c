"""BASELINE config 4 timings on one B200: n = 65536, d in {16, 32, 64, 128}, b ~ N(0, 1) of length
n^2 (34 GB, generated on the device from NumPy's default_rng(0) stream), lam 1e-3, eps 0.1,
delta 0.01, alpha 1e-5.

    python tools/bench_c4.py [d ...]

Per d: fast_kronecker_regression (device-resident inputs, median of 3 after one warm-up, host
wall clock around a synchronised call, with_loss=False), kronmatmul_svd_solve's exact pass, the
loss pass, the fast loss / exact loss ratio, iterations and sample count.  One JSON line per d."""

import json
import math
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2209_04876_b200 as K  # noqa: E402
from paper_2209_04876_b200.leverage import device_standard_normal  # noqa: E402

N = 65536


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), out


def main():
    ds = [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [16, 32, 64, 128]
    fast_only = "--fast-only" in sys.argv
    b = device_standard_normal(0, N * N)
    cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
    for d in ds:
        gen = np.random.default_rng(0)
        facs = [torch.tensor(gen.normal(1.0, math.sqrt(0.001), (N, d)), device="cuda") for _ in range(2)]
        t_fast, fast = timed(lambda: K.fast_kronecker_regression(facs, b, cfg, with_loss=False))
        if fast_only:
            print(json.dumps({"d": d, "fast_solve_s": t_fast}), flush=True)
            continue
        t_exact, ex = timed(lambda: K.kronmatmul_svd_solve(facs, b, 1e-3), reps=1)
        t_loss, lf = timed(lambda: K.ridge_loss(facs, fast.solution, b, 1e-3), reps=1)
        print(json.dumps({"n": N, "d": d, "fast_solve_s": t_fast, "fast_wall_time_s": fast.wall_time,
                          "iterations": fast.iterations, "sample_count": fast.sample_count,
                          "exact_solve_incl_loss_s": t_exact, "loss_pass_s": t_loss,
                          "fast_loss_over_opt": lf / ex.loss}), flush=True)
        del facs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
