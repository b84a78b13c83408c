"""Fit the persistent loop's chunk-cost model to measured per-CTA apply times.

Runs the fused loop at c3, reads the CTA stamps of iteration 5 (apply duration per CTA), rebuilds
each CTA's chunks from the view's segment offsets with the device plan's rules, and regresses
duration ~ a * chunks + b * samples + c * sum(longest row)."""
import ctypes
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2209_04876_b200 as K  # noqa: E402
from paper_2209_04876_b200 import _device as D, _lib  # noqa: E402
from paper_2209_04876_b200.solvers import FastSolveTrace  # noqa: E402

CH_ROWS, CH_S = 16, 64
n, d = 16384, 64
rng = np.random.default_rng(0)
facs = [torch.tensor(rng.normal(1.0, math.sqrt(1e-3), (n, d)), device="cuda") for _ in range(2)]
b = torch.ones(n * n, dtype=torch.float64, device="cuda")
cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
tr = FastSolveTrace()
K.fast_kronecker_regression(facs, b, cfg, _trace=tr)
view = tr.loop_inputs["view"]
seg = view.seg[: view.u_left + 1].cpu().numpy()
ul = view.u_left
chunks = []  # (rows, samples, longest)
for g0 in range(0, ul, CH_ROWS):
    ub, ue = g0, min(ul, g0 + CH_ROWS)
    sb, se = seg[ub], seg[ue]
    pieces = max(1, -(-(se - sb) // CH_S))
    for k in range(pieces):
        tb, te = sb + k * CH_S, min(se, sb + (k + 1) * CH_S)
        longest = max(min(seg[u + 1], te) - max(seg[u], tb) for u in range(ub, ue))
        chunks.append((ue - ub, te - tb, max(longest, 0)))
chunks = np.array(chunks, dtype=np.float64)
# current device model
dmma = (CH_ROWS // 16) * (d // 8) * (d // 4) + (d // 16) * (d // 8) * (CH_ROWS // 4)
cost = int(13.3 * dmma) + chunks[:, 1] * (d // 16) + chunks[:, 2] * 139
G = torch.cuda.get_device_properties(0).multi_processor_count
total = cost.sum()
mid2 = 2 * np.cumsum(cost) - cost
rng_b = [0] + [int(np.searchsorted(mid2 * G, 2 * total * bb, side="left")) for bb in range(1, G)] + [len(chunks)]
# run the loop and read the stamps
li = tr.loop_inputs
x = D.empty(view.dL, view.dR)
hist = D.zeros(max(1, li["max_iters"]))
rhs2 = D.empty(view.dL, view.dR)
it, hl = ctypes.c_int32(0), ctypes.c_int32(0)
lib = _lib.load()
for _ in range(3):
    assert lib.ks_richardson_fused(ctypes.byref(view.struct), D.p(view.perm_arg()), D.p(li["b_at"]), D.p(li["VL"]),
                                   D.p(li["wL"]), D.p(li["VR"]), D.p(li["wR"]), None, li["lam"], li["damping"],
                                   li["max_iters"], li["tol"], D.p(x), D.p(hist), D.p(rhs2), ctypes.byref(it),
                                   ctypes.byref(hl), D.stream()) == 0
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * (9 * G))()
lib.ks_debug_richardson_cta_stamps.argtypes = [ctypes.c_int32, ctypes.c_void_p]
lib.ks_debug_richardson_cta_stamps(G, buf)
st = np.array(list(buf), dtype=np.float64).reshape(G, 9)
dur = (st[:, 1] - st[:, 0]) / 1e3  # us
feats = np.array([[rng_b[bb + 1] - rng_b[bb], chunks[rng_b[bb]:rng_b[bb + 1], 1].sum(),
                   chunks[rng_b[bb]:rng_b[bb + 1], 2].sum()] for bb in range(G)])
coef, *_ = np.linalg.lstsq(np.c_[feats, np.ones(G)], dur, rcond=None)
pred = np.c_[feats, np.ones(G)] @ coef
print("chunks", len(chunks), "per CTA", feats[:, 0].min(), feats[:, 0].max())
print("apply us: median %.2f max %.2f min %.2f" % (np.median(dur), dur.max(), dur.min()))
print("fit us = %.3f*chunks + %.4f*samples + %.4f*longest + %.3f ; resid rms %.3f" % (*coef, np.sqrt(np.mean((pred - dur) ** 2))))
print("per-cycle weights (1.94 GHz): chunk %.0f, sample %.1f, longest %.1f" % tuple(c * 1940 for c in coef[:3]))
print("model cost vs duration corr:", np.corrcoef([cost[rng_b[bb]:rng_b[bb + 1]].sum() for bb in range(G)], dur)[0, 1])
