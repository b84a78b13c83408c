"""Symmetric (Gram) eigensolve on the device with and without the FP32 prelude: time (CUDA events,
median of 20), FP64 sweeps, eigenvalue / eigenvector accuracy and orthogonality vs NumPy.

    KS_JACOBI_FP32=<n> python tools/jacobi_mixed.py"""
import ctypes
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2209_04876_b200 import _device as D, _lib  # noqa: E402

lib = _lib.load()
rng = np.random.default_rng(0)
for n, d in [(16384, 64), (4096, 32), (1024, 16), (65536, 128)]:
    a = rng.normal(1.0, np.sqrt(1e-3), (n, d))
    g = a.T @ a
    gt = D.to_dev(g)
    sig = D.empty(2, d)
    V = D.empty(2, d, d)
    ptrs = _lib.ptr_array(ctypes.c_void_p, [gt.data_ptr(), gt.data_ptr()])
    ts = []
    for _ in range(21):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("ks_sym_eig_batched", 2, ptrs, d, D.p(sig), D.p(V), D.stream())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    mix = (ctypes.c_longlong * 3)()
    lib.ks_debug_jacobi_mix(mix)
    sw = (ctypes.c_int32 * 8)()
    lib.ks_debug_jacobi_sweeps(sw)
    w, v = np.linalg.eigh(g)
    w, v = w[::-1], v[:, ::-1]
    s0 = sig[0].cpu().numpy()
    v0 = V[0].cpu().numpy()
    align = np.abs(np.sum(v0 * v, axis=0))
    orth = np.abs(v0.T @ v0 - np.eye(d)).max()
    resid = np.linalg.norm(g @ v0 - v0 * s0) / np.linalg.norm(g)
    print(f"d={d} fp32={os.environ.get('KS_JACOBI_FP32', 'default')} us={statistics.median(ts[1:]):.1f} "
          f"fp64_sweeps={sw[0]} eig_rel_err={np.abs(s0 - w).max() / w[0]:.2e} "
          f"min_vec_align={align.min():.15f} orth={orth:.2e} resid={resid:.2e} cycles(fp32,transition,fp64)={list(mix)}")
