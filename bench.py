"""Benchmark: FastKroneckerRegression solve time at BASELINE config 3 (n=16384, d=64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

One step = one ``fast_kronecker_regression`` solve (SolveReport.wall_time semantics of the
reference: sampling + preprocessing + Richardson, loss excluded) on the BASELINE inputs
(A1, A2 ~ N(1, var 1e-3) seed 0, b = ones(n^2), lam=1e-3, eps=0.1, delta=0.01, alpha=1e-5).

  value  -- device-resident inputs, CUDA-event time per solve (max over ranks), seconds.
  e2e    -- the public API called with HOST inputs (numpy factors, pinned host b): wall time of
            the solve including every host<->device transfer it makes (factors up, sampled b
            entries up, indices/x down); loss excluded as in the reference.
  roofline -- dominant kernel (the fused sketched normal-operator apply of the Richardson loop)
            at algorithmic FLOPs / measured FP64 peak; KronMatMul (exact baseline n^2 pass) and
            the loss pass are reported alongside under "kernels".
  cpu_baseline -- the oracle port of the reference (NumPy/OpenBLAS) on this host's cores.

``--impl reference`` times the reference's CPU implementation (oracle port) instead.
Under torchrun (N>1) the solve is row-sharded: rank r holds rows [lo, hi) of the
n x n reshape of b, the sketch is replicated, the Richardson loop all-reduces its d^2 partial over
NCCL once per pass inside one CUDA graph (distributed.sharded_fast_kronecker_regression); rank 0
reports the max over ranks.  ``--sharded`` runs that path at N = 1 as well.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

# the solve graph's concurrent branches need more than the default 8 hardware work queues
# (paper_2209_04876_b200/__init__.py); set before any CUDA context exists
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c1": (1024, 16), "c2": (4096, 32), "c3": (16384, 64),
}
METRIC = "FastKronReg solve time (s) at n=16384,d=64"
PARAMS = dict(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_inputs(n, d):
    """experiments.py:106-115: A1, A2 ~ N(1, var 1e-3) from default_rng(0)."""
    import numpy as np
    rng = np.random.default_rng(0)
    facs = [rng.normal(1.0, math.sqrt(0.001), (n, d)) for _ in range(2)]
    return facs


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML every
    2 ms in a thread (nvidia-smi as the fallback); one sample is taken at start() and one at stop(),
    so even a short timed region has samples."""

    _REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index=0):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reason_mask)
        self.thread = None
        self.stop_flag = threading.Event()
        self.nvml = None

    def _sample(self):
        nv, h = self.nvml
        try:
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                 float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)), int(get_reasons(h))))
        except Exception:
            pass

    def _loop(self):
        while not self.stop_flag.wait(0.002):
            self._sample()

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = (nv, nv.nvmlDeviceGetHandleByIndex(self.index))
        except Exception:
            self.nvml = None
            return
        self._sample()
        self.thread = threading.Thread(target=self._loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.nvml is None:
            return self._smi_once()
        self._sample()
        self.stop_flag.set()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [x[0] for x in self.samples]
        mx = [x[1] for x in self.samples]
        reasons = sorted({nm for x in self.samples for nm, bit in self._REASONS.items() if x[2] & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(self.samples), "source": "nvml, 2 ms", "reasons": reasons}

    def _smi_once(self):
        cmd = ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
               "--format=csv,noheader,nounits"]
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=10).stdout.strip().split(",")
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            return {"sm_mhz": float(out[0]), "sm_max_mhz": float(out[1]), "samples": 1, "source": "nvidia-smi",
                    "reasons": sorted(nm for nm, v in zip(names, out[2:6]) if v.strip().lower() == "active")}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": ["clock query unavailable"]}


def fp64_peak_tflops():
    """Measured FP64 (DMMA) peak of this pool's B200s (tools/fp64_peak.cu, profiles/r01_fp64_peak.txt)."""
    p = ROOT / "profiles" / "r01_fp64_peak.txt"
    best = None
    if p.exists():
        for line in p.read_text().splitlines():
            if line.startswith("{") and '"dmma' in line:
                try:
                    v = json.loads(line)["tflops"]
                    best = v if best is None else max(best, v)
                except Exception:
                    pass
    return best or 37.1


def hbm_peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def flush_l2(buf):
    buf.add_(1.0)


def sharded_k1_timing(facs, b, n, d, ws, rank, barrier, reps=5):
    """The exact KronMatMul n^2 pass row-sharded over the ranks (BASELINE c3): rank r
    contracts rows [lo, hi) of the n x n reshape of b (ks_kron2_contract) and one d x d NCCL
    all-reduce combines the partials.  CUDA events around contract + all-reduce, median over reps,
    max over ranks."""
    import torch
    from paper_2209_04876_b200.distributed import DeviceKron2Ops, ShardPlan, allreduce_sum
    plan = ShardPlan(ws, rank, n)
    lo, hi = plan.rows
    B = b.reshape(n, n)[lo:hi]
    ops = DeviceKron2Ops()
    L, R = facs[0][lo:hi], facs[1]
    ts = []
    for i in range(reps + 1):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        allreduce_sum(ops.contract(L, B, R))
        e1.record()
        e1.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1) * 1e3)
    us = statistics.median(ts)
    if ws > 1:
        t = torch.tensor([us], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        us = float(t.item())
    flops = 2.0 * n * n * d + 2.0 * n * d * d
    return {"ranks": ws, "rows_per_rank": hi - lo, "us": us, "tflops_total": flops / (us * 1e-6) / 1e12,
            "note": "K1 pass of kronmatmul_svd_solve on each rank's row block + d^2 NCCL all-reduce, max over ranks"}


def run_ours(args):
    import numpy as np
    import torch
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import _lib, _device as D
    from paper_2209_04876_b200.solvers import FastSolveTrace

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    n, d = CONFIGS[args.config]
    facs_h = make_inputs(n, d)
    facs = [torch.tensor(a, device="cuda") for a in facs_h]
    b = torch.ones(n * n, dtype=torch.float64, device="cuda")
    cfg = K.RegressionConfig(**PARAMS)
    l2 = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 512 MB > 126 MB L2

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        K.fast_kronecker_regression(facs, b, cfg)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    times = []
    stream = torch.cuda.current_stream()
    from paper_2209_04876_b200 import solvers as S
    full_times = []  # whole public call incl. validation and the exact loss pass
    rich_live = []  # device time of the persistent Richardson launch inside the timed solves
    stage_live = []  # the same with the eigenbasis packing launches before it
    for _ in range(args.steps):
        flush_l2(l2)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        S._PHASES[0] = []
        e0.record(stream)
        rep = K.fast_kronecker_regression(facs, b, cfg)
        e1.record(stream)
        e1.synchronize()
        ph = S._PHASES[0]; S._PHASES[0] = None
        names = [p[0] for p in ph]
        # the reference's wall_time span: after validation -> end of the Richardson loop (the
        # loss pass that follows is excluded, as in solvers.py:404-462)
        times.append(ph[names.index("t0")][2].elapsed_time(ph[names.index("solve_end")][2]) / 1e3)
        full_times.append(e0.elapsed_time(e1) / 1e3)
        if S._LAST_LOOP_EVENTS[0] is not None:  # whole-solve graph: events captured around the loop
            l0, l1, lk = S._LAST_LOOP_EVENTS[0]
            rich_live.append(lk.elapsed_time(l1) * 1e3)  # the persistent kernel's launch alone
            stage_live.append(l0.elapsed_time(l1) * 1e3)  # with the eigenbasis packing launches
        elif "richardson" in names:
            i = names.index("richardson")
            rich_live.append(ph[i - 1][2].elapsed_time(ph[i][2]) * 1e3)
    barrier()
    clk = clocks.stop()
    t_step = sum(times) / len(times)
    if ws > 1:
        t = torch.tensor([t_step], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_step = float(t.item())
    x_loss = rep.loss

    # ---- e2e through the public API with host inputs: pinned host factors and b go in, the
    # solution comes back to the host; the timed region is the whole call (validation, factor
    # uploads, the sampled-b transfer, the solve, the solution download); loss excluded
    # page-locked inputs; the small factor buffers first: pinned after a 2 GB page-locked block they
    # land on scattered pages and upload at ~15-37 instead of ~53 GB/s (tools/h2d_probe.py)
    facs_pin = [torch.from_numpy(a).pin_memory() for a in facs_h]
    b_host = torch.ones(n * n, dtype=torch.float64).pin_memory()
    e2e = []
    # warm-up: graph capture, then the page-locked b pages the sampled-entry reads touch (their
    # address translations settle over the first replays)
    e2e_warm = max(args.warmup, 40)
    for i in range(e2e_warm + max(5, args.steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = K.fast_kronecker_regression(facs_pin, b_host, cfg, with_loss=False)
        x_host = np.asarray(r.solution)
        e2e_t = time.perf_counter() - t0
        if i >= e2e_warm:
            e2e.append(e2e_t)
        if os.environ.get("KS_BENCH_DEBUG"):
            print(f"e2e {i} {e2e_t * 1e3:.3f} ms", file=sys.stderr)
    if os.environ.get("KS_BENCH_DEBUG"):
        # which host<->device leg is slow in this process: factor upload, sampled-b reads
        dev_f = [torch.empty_like(f, device="cuda") for f in facs_pin]
        tu, tg = [], []
        idx = torch.randint(0, n, (38049, 2), dtype=torch.int64, device="cuda")
        out = torch.empty(38049, dtype=torch.float64, device="cuda")
        for _ in range(10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for f, df in zip(facs_pin, dev_f):
                df.copy_(f, non_blocking=True)
            torch.cuda.synchronize()
            tu.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            _lib.call("ks_gather_draws2", D.p(b_host), D.p(idx), n, 38049, D.p(out), D.stream())
            torch.cuda.synchronize()
            tg.append(time.perf_counter() - t0)
        print(f"upload {statistics.median(tu) * 1e3:.3f} ms, mapped gather {statistics.median(tg) * 1e3:.3f} ms",
              file=sys.stderr)
    t0 = time.perf_counter()
    r_full = K.fast_kronecker_regression(facs_h, b_host, cfg)
    e2e_full = time.perf_counter() - t0

    # ---- stage / kernel timing (outside the timed region)
    tr = FastSolveTrace()
    K.fast_kronecker_regression(facs, b, cfg, _trace=tr)
    nnz = tr.sdiag.nnz
    kernels = stage_timings(K, facs, b, cfg, tr, n, d)
    launches = count_launches(K, facs, b, cfg)
    try:
        kernels["kronmatmul_rowsharded"] = sharded_k1_timing(facs, b, n, d, ws, rank, barrier)
    except Exception as exc:  # reported, never fatal for the headline line
        kernels["kronmatmul_rowsharded"] = {"error": repr(exc)[:200]}

    result = None
    if rank == 0:
        peak = fp64_peak_tflops()
        rich = kernels["richardson_loop"]
        live_us = statistics.median(rich_live) if rich_live else rich["us"]
        live_tf = rich["flops_per_iter"] * rich["iterations"] / (live_us * 1e-6) / 1e12
        result = {
            "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"fast_kronecker_regression {args.config}: n={n}, d={d}, N=2, b=ones(n^2), "
                                   "lam=1e-3, eps=0.1, delta=0.01, alpha=1e-5, seed=0",
                       "n": n, "d": d, "sample_count": rep.sample_count, "iterations": rep.iterations,
                       "nnz": nnz, "parallelism": f"replicas{ws}" if ws > 1 else "single",
                       "l2": "flushed (512 MB write) before every timed solve"},
            "loss": x_loss,
            "e2e": {"value": statistics.median(e2e), "unit": "s",
                    "h2d_bytes_per_step": 2 * n * d * 8 + nnz * 8,
                    "d2h_bytes_per_step": nnz * 8 + d * d * 8,
                    "note": "whole public call fast_kronecker_regression(pinned host factors, pinned host b, "
                            "with_loss=False) timed on the host: factor uploads, sampled-b gather/upload, solve, "
                            "solution download; only the sampled entries of b cross PCIe; median of steps",
                    "full_call_with_loss_s": e2e_full},
            "full_call_device_s": statistics.median(full_times),
            "roofline": {"bound": "tensor", "kernel": "richardson_phased_kernel (eigenbasis sketched normal "
                                                        "operator, diagonal preconditioner, right-hand-side pass + "
                                                        "all iterations in one persistent launch; FP64 DMMA)",
                         "achieved": live_tf, "peak": peak, "unit": "TFLOP/s",
                         "frac": live_tf / peak, "traffic": traffic_bytes(),
                         "measured": "CUDA events captured in the solve graph on the launching stream: one "
                                     "recorded right before the persistent launch (after the packing launches), "
                                     "one after it; median over the timed solves",
                         "stage_us": statistics.median(stage_live) if stage_live else None,
                         "stage_frac": (rich["flops_per_iter"] * rich["iterations"] / (statistics.median(stage_live)
                                        * 1e-6) / 1e12 / peak) if stage_live else None,
                         "peak_source": "measured FP64 DMMA peak (tools/fp64_peak.cu, profiles/r01_fp64_peak.txt)",
                         "algorithmic_flops_per_launch": rich["flops_per_iter"] * rich["iterations"],
                         "launch_us": live_us, "standalone_launch_us": rich["us"]},
            "kernels": kernels,
            "gpu_launches": launches * args.steps,
            "gpu_launches_per_step": launches,
            "clocks": clk,
        }
        if not args.skip_cpu:
            result["cpu_baseline"] = cpu_baseline(args.config, args.cpu_reps)
        if not args.no_extra:  # the other BASELINE configurations, each with its own roofline and clocks
            del b
            torch.cuda.empty_cache()
            result["configs"] = {}
            for name, fn in (("c4_d64", extra_c4), ("c5_tucker_core", extra_c5)):
                try:
                    result["configs"][name] = fn(args, l2)
                except Exception as exc:  # reported, never fatal for the headline line
                    result["configs"][name] = {"error": repr(exc)[:300]}
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return result


def run_sharded(args):
    """N > 1 (or --sharded): the row-sharded solve of SURVEY.md 8(e).  Rank r holds both factors and
    rows [lo, hi) of the n x n reshape of b; the sketch and eigendecompositions are replicated, the
    Richardson loop runs on the rank's samples with one d^2 NCCL all-reduce per pass, all on the
    device as one CUDA graph (distributed.sharded_fast_kronecker_regression).  value = the whole
    solve's time per step (CUDA events, max over ranks); the loop alone is timed the same way for
    the roofline (algorithmic FLOPs of the full problem / loop time / (N x FP64 peak))."""
    import numpy as np
    import torch
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import distributed as DS
    from paper_2209_04876_b200.solvers import FastSolveTrace

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    import torch.distributed as dist
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, d = CONFIGS[args.config]
    facs_h = make_inputs(n, d)
    facs = [torch.tensor(a, device="cuda") for a in facs_h]
    plan = DS.ShardPlan(ws, rank, n)
    lo, hi = plan.rows
    b_rows = torch.ones((hi - lo, n), dtype=torch.float64, device="cuda")
    cfg = K.RegressionConfig(**PARAMS)
    l2 = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device="cuda")

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if ws > 1:
            t = torch.tensor([v], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            v = float(t.item())
        return v

    for _ in range(args.warmup):
        DS.sharded_fast_kronecker_regression(facs, b_rows, cfg, plan)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    times = []
    for _ in range(args.steps):
        flush_l2(l2)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, iters, hist = DS.sharded_fast_kronecker_regression(facs, b_rows, cfg, plan)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    barrier()
    clk = clocks.stop()
    t_step = max_over_ranks(sum(times) / len(times))
    # the captured loop alone (apply launches + NCCL all-reduces + update kernels)
    loop = next(iter(DS._SHARDED_LOOPS.values()))
    lts = []
    for _ in range(5):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        loop.replay()
        e1.record()
        e1.synchronize()
        lts.append(e0.elapsed_time(e1) * 1e3)
    loop_us = max_over_ranks(statistics.median(lts))
    # e2e: factors from page-locked host memory every step, the solution back to the host
    facs_pin = [torch.from_numpy(a).pin_memory() for a in facs_h]
    e2e = []
    for i in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        for f, fp in zip(facs, facs_pin):
            f.copy_(fp, non_blocking=True)
        xr, _, _ = DS.sharded_fast_kronecker_regression(facs, b_rows, cfg, plan)
        xh = xr.cpu().numpy()
        if i >= args.warmup:
            e2e.append(time.perf_counter() - t0)
    e2e_v = max_over_ranks(statistics.median(e2e))
    # full-problem sketch sizes for the algorithmic FLOPs: one traced single-GPU solve
    tr = FastSolveTrace()
    rep = K.fast_kronecker_regression(facs, torch.ones(n * n, dtype=torch.float64, device="cuda"), cfg, _trace=tr,
                                      with_loss=False)
    view = tr.loop_inputs["view"]
    u1, nnz = view.u_left, view.nnz
    flops_iter = 2.0 * u1 * d * d * 2 + 4.0 * nnz * d + 4.0 * d * d * (d + d)
    k1 = sharded_k1_timing(facs, torch.ones(n * n, dtype=torch.float64, device="cuda"), n, d, ws, rank, barrier)
    result = None
    if rank == 0:
        peak = fp64_peak_tflops()
        ach = flops_iter * iters / (loop_us * 1e-6) / 1e12
        result = {
            "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"fast_kronecker_regression {args.config}: n={n}, d={d}, N=2, b=ones(n^2), "
                                   "lam=1e-3, eps=0.1, delta=0.01, alpha=1e-5, seed=0",
                       "n": n, "d": d, "sample_count": rep.sample_count, "iterations": iters, "nnz": nnz,
                       "parallelism": f"rowsharded{ws}", "rows_per_rank": hi - lo,
                       "l2": "flushed (512 MB write) before every timed solve"},
            "e2e": {"value": e2e_v, "unit": "s", "h2d_bytes_per_step": 2 * n * d * 8, "d2h_bytes_per_step": d * d * 8,
                    "note": "factors uploaded from page-locked host memory every step, b row-sharded and resident "
                            "(only its sampled entries are read), the solution copied back; max over ranks"},
            "roofline": {"bound": "tensor", "kernel": "row-sharded Richardson loop (apply-only launches of the "
                                                        "persistent eigenbasis kernel + NCCL all-reduce + update), "
                                                        "all ranks",
                         "achieved": ach, "peak": peak * ws, "unit": "TFLOP/s", "frac": ach / (peak * ws),
                         "traffic": None, "launch_us": loop_us,
                         "algorithmic_flops_per_launch": flops_iter * iters,
                         "peak_source": f"{ws} x measured FP64 DMMA peak (profiles/r01_fp64_peak.txt)"},
            "kernels": {"richardson_loop_rowsharded": {"us": loop_us, "iterations": iters,
                                                       "us_per_iter": loop_us / max(iters, 1),
                                                       "allreduce_bytes_per_iter": 8 * d * d},
                        "kronmatmul_rowsharded": k1},
            "gpu_launches_per_step": 3 * (iters + 1),
            "gpu_launches": 3 * (iters + 1) * args.steps,
            "clocks": clk,
        }
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    del xh
    return result


def _events_median(fn, reps, flush=None):
    """Median device time (s) of fn() over reps, CUDA events on the current stream, optional L2
    flush before every rep (outside the events)."""
    import torch
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return statistics.median(ts)


def _graph_events_median(fn, reps, flush=None):
    """As _events_median, for fn captured once into a CUDA graph and replayed: the device time of
    its launches without the host-side launch latency (for kernels of tens of microseconds)."""
    import torch
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        fn()
        with torch.cuda.graph(g, stream=side):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    return _events_median(g.replay, reps, flush)


def extra_c4(args, l2):
    """BASELINE config 4 at d = 64 (and the K1 pass at d = 16): n = 65536, b = default_rng(0).
    standard_normal(n^2) regenerated in HBM (34.4 GB).  The fast solve through the public API
    (whole-solve graph), the exact solve, the KronMatMul (K1) and loss (K2) passes with their
    roofline fractions, clocks over the timed region, and the oracle port's time on the host."""
    import numpy as np
    import torch
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import _lib as L, _device as D, solvers as S
    from paper_2209_04876_b200.leverage import device_standard_normal
    n = 65536
    peak = fp64_peak_tflops()
    hbm, hbm_src = hbm_peak_gbs()
    b = device_standard_normal(0, n * n)
    cfg = K.RegressionConfig(**PARAMS)
    out = {"workload": "fast_kronecker_regression c4: n=65536, d=64, N=2, b=default_rng(0).standard_normal(n^2) "
                       "(34.4 GB, generated in HBM), lam=1e-3, eps=0.1, delta=0.01, alpha=1e-5, seed=0"}
    facs = [torch.tensor(a, device="cuda") for a in make_inputs(n, 64)]
    for _ in range(max(args.warmup, 3)):
        rep = K.fast_kronecker_regression(facs, b, cfg, with_loss=False)
    clocks = ClockSampler(0)
    clocks.start()
    loop_us = []

    def solve():
        K.fast_kronecker_regression(facs, b, cfg, with_loss=False)
    ts = []
    for _ in range(args.steps):
        ts.append(_events_median(solve, 1, lambda: flush_l2(l2)))
        if S._LAST_LOOP_EVENTS[0] is not None:
            l0, l1, lk = S._LAST_LOOP_EVENTS[0]
            loop_us.append(lk.elapsed_time(l1) * 1e3)
    for _ in range(2):  # first sight of the key (eager, records the ranks), then the graph capture
        K.kronmatmul_svd_solve(facs, b, PARAMS["lam"])
    t_exact = _events_median(lambda: K.kronmatmul_svd_solve(facs, b, PARAMS["lam"]), 3, lambda: flush_l2(l2))
    T = torch.empty(64, 64, dtype=torch.float64, device="cuda")
    k1 = lambda: L.call("ks_kron2_contract", D.p(facs[0]), D.p(b), n, D.p(facs[1]), n, n, 64, 64, D.p(T),  # noqa: E731
                        D.stream())
    t_k1 = _events_median(k1, 3, lambda: flush_l2(l2))
    X = torch.randn(64, 64, dtype=torch.float64, device="cuda")
    o = torch.empty(1, dtype=torch.float64, device="cuda")
    k2 = lambda: L.call("ks_kron2_residual_sumsq", D.p(facs[0]), D.p(X), D.p(facs[1]), D.p(b), n, n, n, 64, 64,  # noqa: E731
                        D.p(o), D.stream())
    t_k2 = _events_median(k2, 3, lambda: flush_l2(l2))
    f16 = [torch.tensor(a, device="cuda") for a in make_inputs(n, 16)]
    T16 = torch.empty(16, 16, dtype=torch.float64, device="cuda")
    k1_16 = lambda: L.call("ks_kron2_contract", D.p(f16[0]), D.p(b), n, D.p(f16[1]), n, n, 16, 16, D.p(T16),  # noqa: E731
                           D.stream())
    t_k1_16 = _events_median(k1_16, 3, lambda: flush_l2(l2))
    X16 = torch.randn(16, 16, dtype=torch.float64, device="cuda")
    k2_16 = lambda: L.call("ks_kron2_residual_sumsq", D.p(f16[0]), D.p(X16), D.p(f16[1]), D.p(b), n, n, n, 16, 16,  # noqa: E731
                           D.p(o), D.stream())
    t_k2_16 = _events_median(k2_16, 3, lambda: flush_l2(l2))
    out["clocks"] = clocks.stop()
    by = 8.0 * n * n
    fl64 = 2.0 * n * n * 64 + 2.0 * n * 64 * 64
    fl16 = 2.0 * n * n * 16 + 2.0 * n * 16 * 16
    tr = S.FastSolveTrace()
    K.fast_kronecker_regression(facs, b, cfg, _trace=tr, with_loss=False)
    view = tr.loop_inputs["view"]
    flops_iter = 2.0 * view.u_left * 64 * 64 * 2 + 4.0 * view.nnz * 64 + 4.0 * 64 * 64 * 128
    lu = statistics.median(loop_us) if loop_us else None
    out.update({
        "metric": "FastKronReg solve time (s) at n=65536,d=64", "value": statistics.median(ts), "unit": "s",
        "sample_count": rep.sample_count, "iterations": rep.iterations, "nnz": view.nnz,
        "exact_solve_s": t_exact,
        "roofline": {"bound": "tensor", "kernel": "persistent eigenbasis Richardson loop (graph-replayed launch)",
                     "achieved": flops_iter * rep.iterations / (lu * 1e-6) / 1e12 if lu else None,
                     "peak": peak, "unit": "TFLOP/s",
                     "frac": flops_iter * rep.iterations / (lu * 1e-6) / 1e12 / peak if lu else None,
                     "launch_us": lu, "traffic": None},
        "kernels": {
            "kronmatmul_d64": {"us": t_k1 * 1e6, "tflops": fl64 / t_k1 / 1e12, "frac_fp64": fl64 / t_k1 / 1e12 / peak,
                               "gbs": by / t_k1 / 1e9, "frac_hbm": by / t_k1 / 1e9 / hbm, "bound": "fp64"},
            "loss_pass_d64": {"us": t_k2 * 1e6, "frac_fp64": fl64 / t_k2 / 1e12 / peak, "frac_hbm": by / t_k2 / 1e9 / hbm},
            "kronmatmul_d16": {"us": t_k1_16 * 1e6, "gbs": by / t_k1_16 / 1e9, "frac_hbm": by / t_k1_16 / 1e9 / hbm,
                               "frac_fp64": fl16 / t_k1_16 / 1e12 / peak, "bound": "hbm",
                               "note": "K1 of the exact solve at c4 d=16: 34.4 GB of b read once"},
            "loss_pass_d16": {"us": t_k2_16 * 1e6, "gbs": by / t_k2_16 / 1e9, "frac_hbm": by / t_k2_16 / 1e9 / hbm,
                              "frac_fp64": fl16 / t_k2_16 / 1e12 / peak, "bound": "hbm",
                              "note": "K2 (ridge_loss pass) at c4 d=16: 34.4 GB of b read once"}},
        "peaks": {"fp64_tflops": peak, "hbm_gbs": hbm, "hbm_source": hbm_src},
    })
    del b
    torch.cuda.empty_cache()
    if not args.skip_cpu:
        from oracle import kronsolve_oracle as O
        fh = make_inputs(n, 64)
        t0 = time.perf_counter()
        r = O.fast_kronecker_regression(fh, None, with_loss=False, b_at=lambda idx: np.ones(len(idx)), **PARAMS)
        out["cpu_baseline"] = {"value": r.wall_time, "unit": "s", "cores": os.cpu_count(), "kind": "port",
                               "sample": "one oracle fast_kronecker_regression at c4 d=64 with b read as ones at "
                                         "the sampled rows (the solve's cost does not depend on b's values; "
                                         "streaming default_rng(0).standard_normal(n^2) on the host alone takes "
                                         "~90 s)", "run_s": time.perf_counter() - t0}
    return out


def extra_c5(args, l2):
    """BASELINE config 5: Tucker ALS core update (tucker.py:108-127) on the 512 x 512 x 64 synthetic
    tensor, rank (16, 16, 4).  The exact core (K13: U0^T B (U1 kron U2) on the TMA + DMMA K1 kernel,
    B = the 512 x 32768 reshape of X) and the fast core (cached factor SVDs / Grams), their ALS
    'sweepK-core' step times, the K13 / K14 passes against the HBM roofline, and the oracle port."""
    import numpy as np
    import torch
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200 import _lib as L, _device as D, solvers as S
    from oracle import kronsolve_oracle as O
    peak = fp64_peak_tflops()
    hbm, _ = hbm_peak_gbs()
    shape, rank, lam = (512, 512, 64), (16, 16, 4), 1e-3
    x = O.synth_tucker(shape, rank, 0.01, 0)
    xd = torch.tensor(x, device="cuda")
    cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=lam, alpha=1e-5, seed=0)
    model = K.initial_model(xd, rank, lam, 0)
    model.core = K.core_update(model, xd, mode="exact")
    caches = [K.build_factor_cache(a) for a in model.factors]
    clocks = ClockSampler(0)
    clocks.start()
    t_exact = _events_median(lambda: K.core_update(model, xd, mode="exact"), max(args.steps, 5), lambda: flush_l2(l2))
    t_fast = _events_median(lambda: K.core_update(model, xd, mode="fast", config=cfg, caches=caches),
                            max(args.steps, 5), lambda: flush_l2(l2))
    U0, Ur = model.factors[0], S._kron_dev(model.factors[1:])
    U1, U2 = model.factors[1].contiguous(), model.factors[2].contiguous()
    B = xd.reshape(512, -1)
    T = torch.empty(16, 64, dtype=torch.float64, device="cuda")
    k13 = lambda: L.call("ks_kron3_contract", D.p(U0), D.p(U1), D.p(U2), D.p(xd), 512, 512, 64, 16, 16, 4,  # noqa: E731
                         D.p(T), D.stream())
    t13 = _graph_events_median(k13, 10, lambda: flush_l2(l2))
    k13_k1 = lambda: L.call("ks_kron2_contract", D.p(U0), D.p(B), int(B.shape[1]), D.p(Ur), 512, int(B.shape[1]),  # noqa: E731
                            16, 64, D.p(T), D.stream())
    t13_k1 = _graph_events_median(k13_k1, 10, lambda: flush_l2(l2))
    Xc = torch.randn(16, 64, dtype=torch.float64, device="cuda")
    o = torch.empty(1, dtype=torch.float64, device="cuda")
    k14 = lambda: L.call("ks_kron2_residual_sumsq", D.p(U0), D.p(Xc), D.p(Ur), D.p(B), int(B.shape[1]), 512,  # noqa: E731
                         int(B.shape[1]), 16, 64, D.p(o), D.stream())
    t14 = _graph_events_median(k14, 10, lambda: flush_l2(l2))
    als = {}
    for mode in ("exact", "fast"):
        _, rep = K.tucker_als(xd, rank, lam=lam, sweeps=3, solver_mode=mode, config=cfg)
        core_steps = [s for lab, s in zip(rep.step_labels, rep.step_seconds) if lab.endswith("-core")]
        als[mode] = {"sweep_core_s": core_steps, "mean_sweep_s": rep.mean_sweep_seconds, "rre": rep.rre}
    clk = clocks.stop()
    by = 8.0 * x.size
    fl = 2.0 * x.size * 4 + 2.0 * 512 * 512 * 16 * 4 + 2.0 * 512 * 16 * 64  # rightmost-first order
    fl_k1 = 2.0 * x.size * 64 + 2.0 * 512 * 16 * 64  # U0^T B (U1 kron U2) grouping
    out = {"workload": "Tucker ALS core update c5: 512x512x64 = Tucker(core 16x16x4) + N(0, 0.01^2), rank "
                       "(16,16,4), lam=1e-3, eps=0.1, delta=0.01, alpha=1e-5, seed 0",
           "metric": "core_update time (s)", "unit": "s", "exact_core_s": t_exact, "fast_core_s": t_fast,
           "als": als, "clocks": clk,
           "roofline": {"bound": "hbm", "kernel": "K13: (U0 kron U1 kron U2)^T b, one streaming pass in the "
                                                 "reference's rightmost-first order (ks_kron3_contract)",
                        "achieved": by / t13 / 1e9, "peak": hbm,
                        "unit": "GB/s", "frac": by / t13 / 1e9 / hbm, "launch_us": t13 * 1e6,
                        "traffic": traffic_bytes("r02_k13_ncu_full.json")},
           "kernels": {"k13_exact_core_contraction": {"us": t13 * 1e6, "frac_hbm": by / t13 / 1e9 / hbm,
                                                      "frac_fp64": fl / t13 / 1e12 / peak,
                                                      "note": "both launches (streaming pass + CTA-slot sum), graph replay"},
                       "k13_via_k1_right_group": {"us": t13_k1 * 1e6, "frac_hbm": by / t13_k1 / 1e9 / hbm,
                                                  "frac_fp64": fl_k1 / t13_k1 / 1e12 / peak,
                                                  "note": "round-2 start: TMA + DMMA K1 on B (U1 kron U2)"},
                       "k14_residual": {"us": t14 * 1e6, "frac_hbm": by / t14 / 1e9 / hbm}}}
    if not args.skip_cpu:
        facs_h = [a.cpu().numpy() for a in model.factors]
        t0 = time.perf_counter()
        O.core_update_exact(facs_h, x, lam)
        te = time.perf_counter() - t0
        oc = [O.factor_cache(a) for a in facs_h]
        t0 = time.perf_counter()
        O.core_update_fast(facs_h, x, lam, oc, eps=0.1, delta=0.01, alpha=1e-5, seed=0)
        tf = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": te, "unit": "s", "cores": os.cpu_count(), "kind": "port",
                               "sample": "one oracle exact core update (and one fast, fast_s) at c5", "fast_s": tf}
    return out


def _timed(fn, reps=5):
    import torch
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def stage_timings(K, facs, b, cfg, tr, n, d):
    """Per-kernel device times (CUDA events on the launching stream) and roofline numbers."""
    import ctypes
    import torch
    from paper_2209_04876_b200 import _lib as L, _device as D
    peak = fp64_peak_tflops()
    hbm, _ = hbm_peak_gbs()
    out = {}
    li = tr.loop_inputs
    view = li["view"]
    nnz, u1 = view.nnz, view.u_left
    x = torch.empty(view.dL, view.dR, dtype=torch.float64, device="cuda")
    hist = torch.zeros(max(1, li["max_iters"]), dtype=torch.float64, device="cuda")
    it = ctypes.c_int32(0)
    hl = ctypes.c_int32(0)

    rhs2 = torch.empty(view.dL, view.dR, dtype=torch.float64, device="cuda")
    fused = li.get("wL") is not None

    def loop():
        if fused:  # the product path: right-hand side + eigenbasis loop in one persistent launch
            rc = L.load().ks_richardson_fused(ctypes.byref(view.struct), D.p(view.perm_arg()), D.p(li["b_at"]),
                                              D.p(li["VL"]), D.p(li["wL"]), D.p(li["VR"]), D.p(li["wR"]), None,
                                              li["lam"], li["damping"], li["max_iters"], li["tol"], D.p(x), D.p(hist),
                                              D.p(rhs2), ctypes.byref(it), ctypes.byref(hl), D.stream())
        else:
            rc = L.load().ks_richardson_sketched(ctypes.byref(view.struct), D.p(li["VL"]), D.p(li["VR"]),
                                                 D.p(li["dinv"]), D.p(li["rhs"]), li["lam"], li["damping"],
                                                 li["max_iters"], li["tol"], D.p(x), D.p(hist), ctypes.byref(it),
                                                 ctypes.byref(hl), D.stream())
        assert rc == 0, rc

    us_loop = _timed(loop, 5)
    iters = it.value
    ph = (ctypes.c_double * 6)()
    phases = None
    L.load().ks_debug_richardson_profile(1)  # one extra run of the instrumented instantiation
    try:
        loop()
        torch.cuda.synchronize()
    finally:
        L.load().ks_debug_richardson_profile(0)
    if L.load().ks_debug_richardson_phases(iters, ph) == 0:
        phases = dict(zip(["apply", "barrier_1", "reduce", "barrier_2", "norm_update", "loop_overhead"],
                          [round(v) for v in ph]))
        sp = (ctypes.c_double * 8)()
        if L.load().ks_debug_richardson_apply_split(iters, sp) == 0:
            phases["apply_split"] = dict(zip(["l_load_wait", "y_phase", "sample_phase", "g_phase"],
                                             [round(v) for v in (sp[0], sp[1], sp[2], sp[3] + sp[7])]))
            phases["apply_split"]["g_dmma_loop"] = round(sp[7])
            phases["apply_split"]["g_partial_stores"] = round(sp[3])
            phases["sync_split"] = dict(zip(["reduce_fetch_wait", "norm_and_rules", "step_fetch_wait"],
                                            [round(v) for v in sp[4:7]]))
        nct = torch.cuda.get_device_properties(0).multi_processor_count
        st = (ctypes.c_uint64 * (2 * nct))()
        if iters > 5 and L.load().ks_debug_richardson_cta_apply(nct, st) == 0:
            ends = [st[2 * i + 1] - st[2 * i] for i in range(nct)]
            phases["apply_ns_per_cta"] = {"min": min(ends), "median": statistics.median(ends), "max": max(ends)}
    dL, dR = view.dL, view.dR
    flops_apply = 2.0 * u1 * dL * dR * 2 + 4.0 * nnz * dR  # Y and G GEMMs over distinct left rows + dots/axpys
    flops_iter = flops_apply + 4.0 * dL * dR * (dL + dR)  # + preconditioner (four d x d x d products)
    out["richardson_loop"] = {"us": us_loop, "iterations": iters, "us_per_iter": us_loop / max(iters, 1),
                              "flops_per_iter": flops_iter, "nnz": nnz, "u_left": u1,
                              "tflops": flops_iter * iters / (us_loop * 1e-6) / 1e12,
                              "frac_fp64": flops_iter * iters / (us_loop * 1e-6) / 1e12 / peak,
                              "phase_cycles_per_iter": phases,
                              "note": "ks_richardson_fused: device work plan, eigenbasis packing of the sampled "
                                      "rows, then one persistent cooperative launch (right-hand-side pass + all "
                                      "iterations)"}
    U1, U2 = facs
    T = torch.empty(d, d, dtype=torch.float64, device="cuda")

    def kmm():
        assert L.load().ks_kron2_contract(D.p(U1), D.p(b), n, D.p(U2), n, n, d, d, D.p(T), D.stream()) == 0

    us_k_eager = _timed(kmm, 5)
    us_k = _graph_events_median(kmm, 5) * 1e6  # device time of the pass's launches (no host gaps)
    fl = 2.0 * n * n * d + 2.0 * n * d * d
    by = 8.0 * n * n
    out["kronmatmul"] = {"us": us_k, "flops": fl, "bytes": by, "tflops": fl / (us_k * 1e-6) / 1e12,
                         "gbs": by / (us_k * 1e-6) / 1e9, "frac_fp64": fl / (us_k * 1e-6) / 1e12 / peak,
                         "frac_hbm": by / (us_k * 1e-6) / 1e9 / hbm,
                         "bound": "fp64" if fl / (peak * 1e12) > by / (hbm * 1e9) else "hbm",
                         "eager_call_us": us_k_eager,
                         "note": "graph replay of ks_kron2_contract (R transpose, slot memset, the TMA + DMMA "
                                 "pass, slot reduction); eager_call_us adds the host-side launch gaps"}
    Xs = torch.randn(d, d, dtype=torch.float64, device="cuda")
    o = torch.empty(1, dtype=torch.float64, device="cuda")

    def loss():
        assert L.load().ks_kron2_residual_sumsq(D.p(U1), D.p(Xs), D.p(U2), D.p(b), n, n, n, d, d, D.p(o),
                                                D.stream()) == 0

    us_l_eager = _timed(loss, 5)
    us_l = _graph_events_median(loss, 5) * 1e6
    out["loss_pass"] = {"us": us_l, "flops": fl, "bytes": by, "tflops": fl / (us_l * 1e-6) / 1e12,
                        "frac_fp64": fl / (us_l * 1e-6) / 1e12 / peak, "eager_call_us": us_l_eager}
    return out


def count_launches(K, facs, b, cfg):
    """Kernels of libkronsolve_b200.so launched by one solve (torch profiler, outside timing)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        K.fast_kronecker_regression(facs, b, cfg)
        torch.cuda.synchronize()
    ours = 0
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name
            if "_kernel" in name and not name.startswith(("void at::", "at::", "void (anonymous namespace)::elementwise")):
                ours += 1
    return ours


def traffic_bytes(name="r02_richardson_ncu_full.json"):
    """DRAM bytes (read + write) per launch of a kernel from its committed ncu --set full capture
    (profiles/; default: the persistent Richardson kernel), or None."""
    p = ROOT / "profiles" / name
    try:
        return json.loads(p.read_text())["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None


def cpu_baseline(config, reps):
    """Oracle port of the reference (NumPy/OpenBLAS) on this host's cores."""
    from oracle import kronsolve_oracle as O
    n, d = CONFIGS[config]
    facs, b = O.synth_regression(n, d, 2, 0)
    ts = []
    for _ in range(reps):
        rep = O.fast_kronecker_regression(facs, b, with_loss=False, **PARAMS)
        ts.append(rep.wall_time)
    return {"value": statistics.median(ts), "unit": "s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"{reps} full fast_kronecker_regression solves at {config} (oracle/kronsolve_oracle.py, "
                      "NumPy 2.3.5 + OpenBLAS threads = all host cores), median wall_time"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    from oracle import kronsolve_oracle as O
    n, d = CONFIGS[args.config]
    facs, b = O.synth_regression(n, d, 2, 0)
    for _ in range(args.warmup):
        O.fast_kronecker_regression(facs, b, with_loss=False, **PARAMS)
    ts = []
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        rep = O.fast_kronecker_regression(facs, b, with_loss=False, **PARAMS)
        ts.append(rep.wall_time)
    _ = time.perf_counter() - t_wall0
    v = sum(ts) / len(ts)
    return {"metric": METRIC, "value": v, "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"fast_kronecker_regression {args.config}: n={n}, d={d}, N=2, b=ones(n^2), "
                                   "lam=1e-3, eps=0.1, delta=0.01, alpha=1e-5, seed=0", "n": n, "d": d},
            "cpu_baseline": {"value": v, "unit": "s", "cores": os.cpu_count(), "kind": "port",
                             "sample": f"{args.steps} full solves (oracle port of the reference, NumPy/OpenBLAS, "
                                       "all host threads)"},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="run the row-sharded solve also at N = 1")
    ap.add_argument("--no-extra", action="store_true", help="skip the c4 d=64 / c5 Tucker sub-results")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, _, _ = dist_env()
    if args.impl == "reference":
        res = run_reference(args)
    elif ws > 1 or args.sharded:
        res = run_sharded(args)
    else:
        res = run_ours(args)
    if res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
