"""Time the drop-in NumPy call path at c3 (pageable factors and b) against page-locked torch inputs.

    python tools/numpy_path_probe.py"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2209_04876_b200 as K  # noqa: E402

n, d = 16384, 64
facs = bench.make_inputs(n, d)
b = np.ones(n * n)
cfg = K.RegressionConfig(**bench.PARAMS)


def timed(fn, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


out = {"numpy_no_loss_s": timed(lambda: K.fast_kronecker_regression(facs, b, cfg, with_loss=False)),
       "numpy_with_loss_s": timed(lambda: K.fast_kronecker_regression(facs, b, cfg), 3)}
fp = [torch.from_numpy(a).pin_memory() for a in facs]
bp = torch.from_numpy(b).pin_memory()
out["pinned_no_loss_s"] = timed(lambda: K.fast_kronecker_regression(fp, bp, cfg, with_loss=False))
print(out)
