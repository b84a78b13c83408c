"""H2D bandwidth of a 16.7 MB upload from torch-pinned vs THP-backed cudaHostRegister'ed memory
(process-to-process variance probe).  python tools/h2d_probe.py"""
import ctypes
import mmap
import statistics
import time

import numpy as np
import torch


def thp_pinned(count):
    nbytes = count * 8
    mm = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    buf = np.frombuffer(mm, dtype=np.uint8)
    off = (-buf.ctypes.data) % (2 << 20)
    ctypes.CDLL("libc.so.6").madvise(ctypes.c_void_p(buf.ctypes.data + off), ctypes.c_size_t(nbytes), 14)
    arr = buf[off:off + nbytes].view(np.float64)
    arr[:] = 1.0
    t = torch.from_numpy(arr)
    torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
    return t, mm


def bw(src, reps=20):
    dst = torch.empty(src.numel(), dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return src.numel() * 8 / statistics.median(ts[5:]) / 1e9


n = 2 * 16384 * 64
a = torch.ones(n, dtype=torch.float64).pin_memory()
t, mm = thp_pinned(n)
big = torch.ones(16384 * 16384, dtype=torch.float64).pin_memory()  # like the bench's pinned b
a2 = torch.ones(n, dtype=torch.float64).pin_memory()
print(f"torch pinned {bw(a):.1f} GB/s, THP registered {bw(t):.1f} GB/s, torch pinned after 2 GB pin {bw(a2):.1f} GB/s")
