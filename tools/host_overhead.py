"""Host-side cost of the public call with page-locked host inputs at c3 (the e2e path):
wall time per call, the device time of the graph replay, and a cProfile of the Python work.
python tools/host_overhead.py"""
import cProfile
import pstats
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
facs = [torch.from_numpy(a).pin_memory() for a in bench.make_inputs(n, d)]
b = torch.ones(n * n, dtype=torch.float64).pin_memory()
cfg = K.RegressionConfig(**bench.PARAMS)
for _ in range(40):
    K.fast_kronecker_regression(facs, b, cfg, with_loss=False)
walls = []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = K.fast_kronecker_regression(facs, b, cfg, with_loss=False)
    np.asarray(r.solution)
    walls.append(time.perf_counter() - t0)
print("wall median us", statistics.median(walls) * 1e6, "report wall_time us", r.wall_time * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    K.fast_kronecker_regression(facs, b, cfg, with_loss=False)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
