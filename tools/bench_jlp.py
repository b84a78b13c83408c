"""Time ks_jl_projection (Cholesky + two triangular solves) alone and print its phase stamps."""
import ctypes
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2209_04876_b200 import _device as D, _lib  # noqa: E402

lib = _lib.load()
rng = np.random.default_rng(0)
for d, r in [(16, 56), (32, 67), (64, 78)]:
    A = rng.normal(1, np.sqrt(1e-3), (4096, d))
    G = D.to_dev(A.T @ A)
    GA = D.to_dev(rng.standard_normal((r, d)))
    Q = D.empty(r, d)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    ts = []
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.ks_jl_projection(D.p(G), d, D.p(GA), r, 1.0, D.p(Q), D.p(info), D.stream())
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    st = (ctypes.c_uint64 * 4)()
    lib.ks_debug_jl_projection_stamps(st)
    ref = np.linalg.solve((A.T @ A).T, GA.cpu().numpy().T).T
    err = np.max(np.abs(Q.cpu().numpy() - ref)) / np.max(np.abs(ref))
    print(f"d={d} r={r}: {statistics.median(ts[1:]):7.1f} us  stage {(st[1]-st[0])/1e3:6.1f}  chol "
          f"{(st[2]-st[1])/1e3:6.1f}  solve {(st[3]-st[2])/1e3:6.1f} us  err {err:.1e}  info {int(info.item())}")
