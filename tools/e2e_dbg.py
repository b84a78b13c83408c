import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2209_04876_b200 as K
from paper_2209_04876_b200 import solvers as S
import bench
n, d = 16384, 64
facs_h = bench.make_inputs(n, d)
cfg = K.RegressionConfig(**bench.PARAMS)
b_host = torch.ones(n * n, dtype=torch.float64).pin_memory()
facs_pin = [torch.from_numpy(a).pin_memory() for a in facs_h]
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = K.fast_kronecker_regression(facs_pin, b_host, cfg, with_loss=False)
    x = np.asarray(r.solution)
    t1 = time.perf_counter()
    print(i, f"{(t1-t0)*1e3:.3f} ms wall_time {r.wall_time*1e3:.3f} ms", S._SOLVE_STATS, S._PREFIX_STATS)
