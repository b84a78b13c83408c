"""Time the two-factor n^2 passes (KronMatMul contract, loss residual) at a BASELINE size.

    python tools/bench_kron2.py [n] [d] [reps]
"""
import ctypes
import math
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2209_04876_b200 import _device as D, _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
g = torch.Generator(device="cuda").manual_seed(0)
U1 = torch.randn(n, d, dtype=torch.float64, device="cuda", generator=g)
U2 = torch.randn(n, d, dtype=torch.float64, device="cuda", generator=g)
B = torch.randn(n * n, dtype=torch.float64, device="cuda", generator=g)
X = torch.randn(d, d, dtype=torch.float64, device="cuda", generator=g)
T = torch.empty(d, d, dtype=torch.float64, device="cuda")
o = torch.empty(1, dtype=torch.float64, device="cuda")
lib = _lib.load()


def contract():
    assert lib.ks_kron2_contract(D.p(U1), D.p(B), n, D.p(U2), n, n, d, d, D.p(T), D.stream()) == 0


def resid():
    assert lib.ks_kron2_residual_sumsq(D.p(U1), D.p(X), D.p(U2), D.p(B), n, n, n, d, d, D.p(o), D.stream()) == 0


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


fl = 2.0 * n * n * d
for name, fn in (("contract", contract), ("residual", resid)):
    ms = timed(fn)
    print(f"{name}: {ms:.3f} ms  {fl / ms / 1e9:.2f} TF/s  {8.0 * n * n / ms / 1e6:.0f} GB/s")
ref = (U1.T @ B.view(n, n) @ U2)
contract()
torch.cuda.synchronize()
print("contract rel err vs cuBLAS", float((T - ref).norm() / ref.norm()))
t0 = timed(lambda: U1.T @ (B.view(n, n) @ U2))
print(f"cuBLAS U1^T (B U2): {t0:.3f} ms {fl / t0 / 1e9:.2f} TF/s")
