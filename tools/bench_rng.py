"""Device NumPy-exact standard_normal (the JL sketches of the fast solve): warm timings of one
1.28 M draw (c3: r = 78 rows x 16384), two concurrent draws on two streams, and both replayed in
a CUDA graph.  python tools/bench_rng.py"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2209_04876_b200 import leverage as _lev  # noqa: E402
from paper_2209_04876_b200.leverage import device_standard_normal  # noqa: E402

_lev._DEFERRED[0] = _lev.DeferredChecks()  # status words checked never (timing only), no host syncs

N = 78 * 16384


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


x = device_standard_normal(7, N)
ref = np.random.default_rng(7).standard_normal(N)
xd = x.cpu().numpy()
print("parity: exact", int(np.sum(xd == ref)), "of", N, "max abs diff", float(np.max(np.abs(xd - ref))))
print("one draw us", timed(lambda: device_standard_normal(7, N)))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def two():
    main = torch.cuda.current_stream()
    s1.wait_stream(main)
    s2.wait_stream(main)
    with torch.cuda.stream(s1):
        device_standard_normal(7, N)
    with torch.cuda.stream(s2):
        device_standard_normal(8, N)
    main.wait_stream(s1)
    main.wait_stream(s2)


print("two concurrent us", timed(two))
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    two()
torch.cuda.synchronize()
with torch.cuda.graph(g):
    two()
print("two concurrent, graph us", timed(g.replay))
g1 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g1):
    device_standard_normal(7, N)
print("one draw, graph us", timed(g1.replay))
