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
    names = ["apply", "sync", "reduce+sync", "precondA+sync", "precondB+sync", "update"]
    print("richardson phases (cycles/iter):", {k: round(v) for k, v in zip(names, ph)})
    sp = (ctypes.c_double * 4)()
    if _lib.load().ks_debug_richardson_apply_split(rep.iterations, sp) == 0:
        print("  apply split (cycles/iter):", {k: round(v) for k, v in zip(["wait", "Y", "samples", "G"], sp)})

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

if "--trace" in sys.argv:
    # kernel timeline of one solve (CUPTI via torch.profiler): start offset, duration, stream
    import json
    import tempfile
    from torch.profiler import ProfilerActivity, profile
    from paper_2209_04876_b200 import solvers as S2
    K.fast_kronecker_regression(facs, b, cfg)
    K.fast_kronecker_regression(facs, b, cfg)
    before = dict(S2._PREFIX_STATS)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        rep = K.fast_kronecker_regression(facs, b, cfg)
        torch.cuda.synchronize()
    print("prefix graph stats before/after the traced solve:", before, dict(S2._PREFIX_STATS))
    with tempfile.NamedTemporaryFile(suffix=".json", delete=False) as f:
        path = f.name
    prof.export_chrome_trace(path)
    allev = json.load(open(path))["traceEvents"]
    ev = [e for e in allev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    rt = [e for e in allev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime" and e.get("dur", 0) > 15]
    ev.sort(key=lambda e: e["ts"])
    t0 = ev[0]["ts"]
    print(f"{'start_us':>9} {'dur_us':>8} {'gap_us':>7} strm  kernel")
    prev_end = {}
    for e in ev:
        s = e["args"].get("stream", -1)
        gap = e["ts"] - prev_end.get(s, e["ts"])
        prev_end[s] = e["ts"] + e["dur"]
        print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} {gap:7.1f} {s:4}  {e['name'][:80]}")
    import collections
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in allev:
        if e.get("ph") == "X" and e.get("cat") == "cuda_runtime":
            agg[e["name"]][0] += 1
            agg[e["name"]][1] += e.get("dur", 0)
    print("runtime API totals:")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:40s} {v[0]:5d} calls {v[1]:9.1f} us")
    print("slow runtime API calls (>15 us):")
    for e in sorted(rt, key=lambda e: e["ts"]):
        print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f}   {e['name']}")
    end = max(e["ts"] + e["dur"] for e in ev)
    print(f"span {end - t0:.1f} us, wall {rep.wall_time * 1e6:.1f} us")

if "--host" in sys.argv:
    # host-side profile of one warm solve (where the wall time goes that is not GPU work)
    import cProfile
    import pstats
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    for _ in range(5):
        pr.enable()
        rep = K.fast_kronecker_regression(facs, b, cfg)
        pr.disable()
        torch.cuda.synchronize()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(45)

if "--phases" in sys.argv:
    import collections
    from paper_2209_04876_b200 import solvers as S
    gpu_t, host_t, walls2 = collections.defaultdict(list), collections.defaultdict(list), []
    order = []
    for rep_i in range(8):
        S._PHASES = []
        torch.cuda.synchronize()
        rep = K.fast_kronecker_regression(facs, b, cfg)
        torch.cuda.synchronize()
        ph, S._PHASES = S._PHASES, None
        walls2.append(rep.wall_time * 1e6)
        prev = ph[0]
        for name, th, ev in ph[1:]:
            if name not in order:
                order.append(name)
            gpu_t[name].append(prev[2].elapsed_time(ev) * 1e3)
            host_t[name].append(1e6 * (th - prev[1]))
            prev = (name, th, ev)
    print(f"phases over 8 solves: wall median {statistics.median(walls2):.0f} us min {min(walls2):.0f} us",
          "solve graph stats:", S._SOLVE_STATS)
    for name in order:
        print(f"  {name:20s} gpu median {statistics.median(gpu_t[name]):8.1f} us   host-issue median "
              f"{statistics.median(host_t[name]):8.1f} us")
