"""Fast-solve profiling helper (for ncu launch lists and phase timing).

    python tools/profile_fast.py [c1|c2|c3] [reps] [--loop]

Runs `reps` fast_kronecker_regression solves on device-resident BASELINE inputs, prints the
wall time, the persistent Richardson kernel's per-phase cycle counts, and (with --loop) CUDA-event
timings of the Richardson loop alone on the solve's own inputs."""
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

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "c3"
reps = int(args[1]) if len(args) > 1 else 1
n, d = {"c1": (1024, 16), "c2": (4096, 32), "c3": (16384, 64)}[name]
rng = np.random.default_rng(0)
facs = [torch.tensor(rng.normal(1.0, math.sqrt(1e-3), (n, d)), device="cuda") for _ in range(2)]
b = torch.ones(n * n, dtype=torch.float64, device="cuda")
cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
walls = []
for _ in range(reps):
    tr = FastSolveTrace()
    rep = K.fast_kronecker_regression(facs, b, cfg, _trace=tr)
    walls.append(rep.wall_time)
torch.cuda.synchronize()
print("wall", walls, "loss", rep.loss, "iters", rep.iterations)
ph = (ctypes.c_double * 6)()
if _lib.load().ks_debug_richardson_phases(rep.iterations, ph) == 0:
    names = ["apply", "sync", "reduce+sync", "precondA+sync", "precondB+sync", "update"]
    print("richardson phases (cycles/iter):", {k: round(v) for k, v in zip(names, ph)})

if "--loop" in sys.argv:
    li = tr.loop_inputs
    view = li["view"]
    x = D.empty(view.dL, view.dR)
    hist = D.zeros(max(1, li["max_iters"]))
    it, hl = ctypes.c_int32(0), ctypes.c_int32(0)

    def run(VL, VR, dinv, rhs):
        rc = _lib.load().ks_richardson_sketched(ctypes.byref(view.struct), D.p(VL), D.p(VR), D.p(dinv), D.p(rhs),
                                                li["lam"], li["damping"], li["max_iters"], li["tol"], D.p(x), D.p(hist),
                                                ctypes.byref(it), ctypes.byref(hl), D.stream())
        assert rc == 0, rc

    def timed(*a):
        run(*a)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(*a)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(ts)

    print("loop us (solve inputs):", timed(li["VL"], li["VR"], li["dinv"], li["rhs"]), "iters", it.value)
    _lib.load().ks_debug_richardson_phases(it.value, ph)
    print("  phases:", [round(v) for v in ph])
    eyeL = torch.eye(view.dL, dtype=torch.float64, device="cuda")
    eyeR = torch.eye(view.dR, dtype=torch.float64, device="cuda")
    ones = torch.ones(view.dL * view.dR, dtype=torch.float64, device="cuda")
    print("loop us (identity precond):", timed(eyeL, eyeR, ones, li["rhs"]), "iters", it.value)
    _lib.load().ks_debug_richardson_phases(it.value, ph)
    print("  phases:", [round(v) for v in ph])

if "--cta" in sys.argv:
    nct = torch.cuda.get_device_properties(0).multi_processor_count
    buf = (ctypes.c_uint64 * (9 * nct))()
    _lib.load().ks_debug_richardson_cta_stamps.argtypes = [ctypes.c_int32, ctypes.c_void_p]
    assert _lib.load().ks_debug_richardson_cta_stamps(nct, buf) == 0
    ts = np.array(list(buf), dtype=np.float64).reshape(nct, 9)
    t0 = ts[:, 0].min()
    ts = (ts - t0) / 1e3
    names = ["apply_start", "apply_end", "sync1_out", "reduce_end", "sync2_out", "precA_end", "sync3_out",
             "precB_end", "sync4_out"]
    for k, nm in enumerate(names):
        col = ts[:, k]
        print(f"{nm:12s} min {col.min():8.2f} us  median {np.median(col):8.2f}  max {col.max():8.2f}  argmax {col.argmax()}")
    dur = ts[:, 1] - ts[:, 0]
    print("apply duration: min %.2f median %.2f max %.2f us" % (dur.min(), np.median(dur), dur.max()))
    print("slowest CTAs:", np.argsort(-dur)[:8], dur[np.argsort(-dur)[:8]].round(2))
