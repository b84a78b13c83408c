"""Per-phase profile of the fused (eigenbasis) Richardson launch: python tools/profile_loop_fused.py [c3]"""
import ctypes
import math
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2209_04876_b200 as K  # noqa: E402
from paper_2209_04876_b200 import _device as D, _lib  # noqa: E402
from paper_2209_04876_b200.solvers import FastSolveTrace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n, d = {"c1": (1024, 16), "c2": (4096, 32), "c3": (16384, 64)}[name]
rng = np.random.default_rng(0)
facs = [torch.tensor(rng.normal(1.0, math.sqrt(1e-3), (n, d)), device="cuda") for _ in range(2)]
b = torch.ones(n * n, dtype=torch.float64, device="cuda")
cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
tr = FastSolveTrace()
rep = K.fast_kronecker_regression(facs, b, cfg, _trace=tr)
li = tr.loop_inputs
view = li["view"]
x = D.empty(view.dL, view.dR)
hist = D.zeros(max(1, li["max_iters"]))
rhs2 = D.empty(view.dL, view.dR)
it, hl = ctypes.c_int32(0), ctypes.c_int32(0)
lib = _lib.load()


def fused():
    rc = lib.ks_richardson_fused(ctypes.byref(view.struct), D.p(view.perm_arg()), D.p(li["b_at"]), D.p(li["VL"]),
                                 D.p(li["wL"]), D.p(li["VR"]), D.p(li["wR"]), None, li["lam"], li["damping"],
                                 li["max_iters"], li["tol"], D.p(x), D.p(hist), D.p(rhs2), ctypes.byref(it),
                                 ctypes.byref(hl), D.stream())
    assert rc == 0, rc


fused()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fused()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"fused launch: median {statistics.median(ts):.1f} us, iterations {it.value}")
ph = (ctypes.c_double * 6)()
lib.ks_debug_richardson_phases(it.value, ph)
print("phases (cycles/iter):", dict(zip(["apply", "sync1", "reduce+sync2", "norm", "-", "update"], [round(v) for v in ph])))
sp = (ctypes.c_double * 4)()
lib.ks_debug_richardson_apply_split(it.value, sp)
print("apply split:", dict(zip(["wait", "Y", "samples", "G"], [round(v) for v in sp])))
nct = torch.cuda.get_device_properties(0).multi_processor_count
buf = (ctypes.c_uint64 * (9 * nct))()
lib.ks_debug_richardson_cta_stamps.argtypes = [ctypes.c_int32, ctypes.c_void_p]
lib.ks_debug_richardson_cta_stamps(nct, buf)
st = np.array(list(buf), dtype=np.float64).reshape(nct, 9)
st = (st - st[:, 0].min()) / 1e3
for k, nm in enumerate(["apply_start", "apply_end", "sync1_out", "reduce_end", "sync2_out", "norm", "-", "upd_end", "-"]):
    col = st[:, k]
    print(f"{nm:12s} min {col.min():7.2f} median {np.median(col):7.2f} max {col.max():7.2f} us")
print("x vs trace x:", float(np.linalg.norm(x.cpu().numpy().reshape(-1) - rep.solution.cpu().numpy().reshape(-1))
                             / np.linalg.norm(rep.solution.cpu().numpy())))
