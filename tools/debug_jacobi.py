"""Time the device one-sided Jacobi on representative matrices and report sweeps."""
import ctypes
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2209_04876_b200 import _device as D, _lib  # noqa: E402

lib = _lib.load()
lib.ks_debug_jacobi_sweeps.argtypes = [ctypes.c_void_p]
rng = np.random.default_rng(0)
cases = {}
for d in (16, 32, 64, 128):
    A = rng.normal(1, np.sqrt(1e-3), (16384, d))
    G = A.T @ A
    cases[f"gram{d}"] = 0.5 * (G + G.T)
cases["eye64"] = np.eye(64)
cases["randn64"] = rng.standard_normal((64, 64))
for name, M in cases.items():
    d = M.shape[0]
    Mt = D.to_dev(M)
    s = D.empty(d)
    V = D.empty(d, d)
    lib.ks_svd_small(D.p(Mt), d, D.p(s), D.p(V), D.stream())
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.ks_svd_small(D.p(Mt), d, D.p(s), D.p(V), D.stream())
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    sw = (ctypes.c_int32 * 8)()
    lib.ks_debug_jacobi_sweeps(sw)
    ref = np.linalg.svd(M, compute_uv=False)
    err = np.max(np.abs(s.cpu().numpy() - ref) / ref.max())
    print(f"{name}: {statistics.median(ts):9.1f} us  sweeps {sw[0]}  sigma err {err:.2e}")

print("two-sided symmetric (ks_sym_eig_batched):")
lib.ks_sym_eig_batched.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]
for name, M in cases.items():
    d = M.shape[0]
    if d not in (16, 32, 64) or name == "randn64":
        continue
    Mt = D.to_dev(M)
    s = D.empty(d)
    V = D.empty(d, d)
    ptrs = (ctypes.c_void_p * 1)(Mt.data_ptr())
    lib.ks_sym_eig_batched(1, ptrs, d, D.p(s), D.p(V), D.stream())
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.ks_sym_eig_batched(1, ptrs, d, D.p(s), D.p(V), D.stream())
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    sw = (ctypes.c_int32 * 8)()
    lib.ks_debug_jacobi_sweeps(sw)
    w_ref, v_ref = np.linalg.eigh(M)
    w = s.cpu().numpy()
    err = np.max(np.abs(np.sort(w) - w_ref)) / np.max(np.abs(w_ref))
    Vh = V.cpu().numpy()
    resid = np.max(np.abs(M @ Vh - Vh * w[None, :])) / np.max(np.abs(w_ref))
    orth = np.max(np.abs(Vh.T @ Vh - np.eye(d)))
    # per-pair residual relative to each eigenvalue (the small eigenpairs), numpy's own for scale
    rr = np.max(np.linalg.norm(M @ Vh - Vh * w[None, :], axis=0) / np.maximum(np.abs(w), 1e-300))
    rr_np = np.max(np.linalg.norm(M @ v_ref - v_ref * w_ref[None, :], axis=0) / np.maximum(np.abs(w_ref), 1e-300))
    print(f"{name}: {statistics.median(ts):9.1f} us  sweeps {sw[0]}  eig err {err:.2e}  resid {resid:.2e}  orth {orth:.2e}"
          f"  pair resid {rr:.2e} (numpy {rr_np:.2e})")
