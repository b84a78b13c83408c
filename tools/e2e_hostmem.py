"""e2e variance probe: the sampled-b reads cross PCIe into page-locked host memory; compare b pinned
by torch (cudaHostAlloc) with b in transparent-huge-page memory registered with cudaHostRegister.
python tools/e2e_hostmem.py"""
import ctypes
import mmap
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2209_04876_b200 as K  # noqa: E402

n, d = 16384, 64
facs_h = bench.make_inputs(n, d)
cfg = K.RegressionConfig(**bench.PARAMS)
facs_pin = [torch.from_numpy(a).pin_memory() for a in facs_h]


def thp_pinned(count):
    nbytes = count * 8
    mm = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    buf = np.frombuffer(mm, dtype=np.uint8)
    addr = buf.ctypes.data
    off = (-addr) % (2 << 20)
    libc = ctypes.CDLL("libc.so.6")
    libc.madvise(ctypes.c_void_p(addr + off), ctypes.c_size_t(nbytes), 14)  # MADV_HUGEPAGE
    arr = buf[off:off + nbytes].view(np.float64)
    arr[:] = 1.0
    t = torch.from_numpy(arr)
    rc = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
    return t, mm, rc


def run(b_host, reps=20):
    ts = []
    for i in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = K.fast_kronecker_regression(facs_pin, b_host, cfg, with_loss=False)
        np.asarray(r.solution)
        ts.append(time.perf_counter() - t0)
    return [round(x * 1e3, 3) for x in ts[8:]]


b1 = torch.ones(n * n, dtype=torch.float64).pin_memory()
print("torch pinned:", run(b1))
b2, mm, rc = thp_pinned(n * n)
print("THP registered (rc %s) pinned=%s:" % (rc, b2.is_pinned()), run(b2))
print("torch pinned again:", run(b1))
