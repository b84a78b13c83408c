"""Where the end-to-end (host inputs) call spends its time: host-clock offsets of the solve's phase
marks relative to the call start, and the device time between them.  python tools/e2e_phases.py"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2209_04876_b200 as K  # noqa: E402
from paper_2209_04876_b200 import solvers as S  # noqa: E402

n, d = 16384, 64
facs_h = bench.make_inputs(n, d)
cfg = K.RegressionConfig(**bench.PARAMS)
facs_pin = [torch.from_numpy(a).pin_memory() for a in facs_h]
b_host = torch.ones(n * n, dtype=torch.float64).pin_memory()
if "--device" in sys.argv:  # device-resident inputs instead (the bench's `value` path)
    facs_pin = [f.cuda() for f in facs_pin]
    b_host = b_host.cuda()
rows = []
for i in range(12):
    torch.cuda.synchronize()
    S._PHASES[0] = []
    t0 = time.perf_counter()
    r = K.fast_kronecker_regression(facs_pin, b_host, cfg, with_loss=False)
    x = r.solution if isinstance(r.solution, np.ndarray) else r.solution.shape
    t1 = time.perf_counter()
    ph = S._PHASES[0]; S._PHASES[0] = None
    if i >= 4:
        rows.append((t1 - t0, [(nm, ht - t0) for nm, ht, _ in ph],
                     [(ph[k][0], ph[k - 1][2].elapsed_time(ph[k][2]) * 1e3) for k in range(1, len(ph))]))
print("e2e median ms", statistics.median(r[0] for r in rows) * 1e3)
for nm, _ in rows[0][1]:
    hs = [dict(r[1])[nm] for r in rows]
    print(f"  host offset of {nm:20s} {statistics.median(hs) * 1e6:8.1f} us")
for nm, _ in rows[0][2]:
    ds = [dict(r[2])[nm] for r in rows]
    print(f"  device time to  {nm:20s} {statistics.median(ds):8.1f} us")
