"""Time ks_leverage_scores_tall_async (CholeskyQR2 leverage scores) alone at c4 size: python tools/probe_lev.py [n] [d] [reps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2209_04876_b200 import _device as D, _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
g = torch.Generator(device="cuda").manual_seed(0)
a = 1.0 + 0.001 * torch.randn(n, d, dtype=torch.float64, device="cuda", generator=g)
sc = torch.empty(n, dtype=torch.float64, device="cuda")
info = torch.zeros(2, dtype=torch.int32, device="cuda")
ts = []
for i in range(reps + 3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("ks_leverage_scores_tall_async", D.p(a), n, d, D.p(sc), D.p(info), D.stream())
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(f"n={n} d={d} leverage scores median {ts[len(ts) // 2]:.1f} us min {ts[0]:.1f} us info {info.tolist()} sum {float(sc.sum()):.6f}")
