"""Timeline of one whole-solve graph replay at c3 (device inputs) or with host inputs (--host), or
at c4 d = 64 (--c4: n = 65536, b = default_rng(0).standard_normal(n^2) generated in HBM): device
time from the graph's start to each join.  KS_GRAPH_TIMELINE=1 python tools/graph_timeline.py [--host|--c4]"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2209_04876_b200 as K  # noqa: E402
from paper_2209_04876_b200 import solvers as S  # noqa: E402

n, d = (65536, 64) if "--c4" in sys.argv else (16384, 64)
facs_h = bench.make_inputs(n, d)
cfg = K.RegressionConfig(**bench.PARAMS)
if "--host" in sys.argv:
    facs = [torch.from_numpy(a).pin_memory() for a in facs_h]
    b = torch.ones(n * n, dtype=torch.float64).pin_memory()
    graphs = S._HOST_GRAPHS
elif "--c4" in sys.argv:
    from paper_2209_04876_b200.leverage import device_standard_normal
    facs = [torch.tensor(a, device="cuda") for a in facs_h]
    b = device_standard_normal(0, n * n)
    graphs = S._SOLVE_GRAPHS
else:
    facs = [torch.tensor(a, device="cuda") for a in facs_h]
    b = torch.ones(n * n, dtype=torch.float64, device="cuda")
    graphs = S._SOLVE_GRAPHS
rows = {}
for i in range(25):
    K.fast_kronecker_regression(facs, b, cfg, with_loss=False)
    torch.cuda.synchronize()
    if i < 10:
        continue
    tl = next(e.out["timeline"] for e in graphs.values() if e.graph is not None)
    t0 = tl[0][1]
    for name, ev in tl[1:]:
        rows.setdefault(name, []).append(t0.elapsed_time(ev) * 1e3)
for name, v in rows.items():
    print(f"{name:12s} {statistics.median(v):8.1f} us")
