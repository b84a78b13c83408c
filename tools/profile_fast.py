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
n, d = {"c1": (1024, 16), "c2": (4096, 32), "c3": (16384, 64), "c4": (65536, 64), "c4d32": (65536, 32)}[name]
rng = np.random.default_rng(0)
facs = [torch.tensor(rng.normal(1.0, math.sqrt(1e-3), (n, d)), device="cuda") for _ in range(2)]
if name.startswith("c4"):
    from paper_2209_04876_b200.leverage import device_standard_normal
    b = device_standard_normal(0, n * n)
else:
    b = torch.ones(n * n, dtype=torch.float64, device="cuda")
cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
walls = []
for _ in range(reps):
    tr = FastSolveTrace()
    rep = K.fast_kronecker_regression(facs, b, cfg, _trace=tr)
    walls.append(rep.wall_time)
    if "--mem" in sys.argv:
        free, total = torch.cuda.mem_get_info()
        print(f"mem: free {free / 2**30:.1f} GiB / {total / 2**30:.1f}; torch allocated "
              f"{torch.cuda.memory_allocated() / 2**30:.2f} reserved {torch.cuda.memory_reserved() / 2**30:.2f} GiB")
torch.cuda.synchronize()
print("wall", walls, "loss", rep.loss, "iters", rep.iterations)
from paper_2209_04876_b200 import solvers as _S  # noqa: E402
print("prefix graph stats:", _S._PREFIX_STATS, "keys:", len(_S._PREFIX_GRAPHS), "solve graph stats:", _S._SOLVE_STATS)
ph = (ctypes.c_double * 6)()
if _lib.load().ks_debug_richardson_phases(rep.iterations, ph) == 0:
    names = ["apply", "barrier_1", "reduce", "barrier_2", "norm_update", "loop_overhead"]
    print("richardson phases (cycles/iter, last profiled run):", {k: round(v) for k, v in zip(names, ph)})

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
    if li.get("wL") is not None:
        rhs2 = D.empty(view.dL, view.dR)

        def fused():
            rc = _lib.load().ks_richardson_fused(ctypes.byref(view.struct), D.p(view.perm_arg()), D.p(li["b_at"]),
                                                 D.p(li["VL"]), D.p(li["wL"]), D.p(li["VR"]), D.p(li["wR"]), None,
                                                 li["lam"], li["damping"], li["max_iters"], li["tol"], D.p(x),
                                                 D.p(hist), D.p(rhs2), ctypes.byref(it), ctypes.byref(hl), D.stream())
            assert rc == 0, rc
        fused()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fused()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print("fused rhs+loop us:", statistics.median(ts), "iters", it.value)
    _lib.load().ks_debug_richardson_phases(it.value, ph)
    print("  phases:", [round(v) for v in ph])
