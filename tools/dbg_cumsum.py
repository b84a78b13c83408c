import ctypes, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2209_04876_b200 import _lib as L, _device as D
L.load()
for n in (40000, 65536):
    sc = torch.tensor(np.random.default_rng(n).random(n) + 0.5, device="cuda")
    p, c = D.empty(n), D.empty(n)
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    L.call("ks_sampler_tables", D.p(sc), n, 0, D.p(p), D.p(c), D.p(fl), D.stream())
    torch.cuda.synchronize()
    o = (ctypes.c_int64 * 2)()
    L.load().ks_debug_cumsum_stats(0, o)
    ref = np.cumsum(p.cpu().numpy())
    print(n, "fail", o[0], "nseg", o[1], "exact", np.array_equal(ref, c.cpu().numpy()))
