"""Device time of the two-factor sketch (sparse diagonal + grouped view, kron.py:147-190 /
sketch_diag_grouped2_launch) on c3-sized draws: eager launches and one graph replay.
python tools/bench_sketch.py   (KS_SKETCH_SORT=1: the flat radix-sort path)"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2209_04876_b200 import _device as D  # noqa: E402
from paper_2209_04876_b200.kron import sketch_diag_grouped2_launch  # noqa: E402

n, d, s = 16384, 64, 38049
rng = np.random.default_rng(0)
facs = [torch.zeros(n, d, dtype=torch.float64, device="cuda") for _ in range(2)]
draws = torch.tensor(rng.integers(0, n, (s, 2)), dtype=torch.int64, device="cuda")
w = torch.tensor(rng.random(s) + 0.5, dtype=torch.float64, device="cuda")
first = D.empty(s, dtype=D.I64)


def run():
    return sketch_diag_grouped2_launch(facs, draws, w, first)


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


out = run()
torch.cuda.synchronize()
print("nnz, ul:", out[5].cpu().tolist())
print("eager us", timed(run))
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run()
print("graph us", timed(g.replay))
