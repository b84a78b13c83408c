"""K13 streaming probe: device time of ks_kron3_contract (graph replay, clean L2) at the c5 shape and
at 8x / 32x more slabs, with arithmetic and stream-only (TMA boxes / contiguous 1-D copies)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2209_04876_b200 import _lib as L, _device as D  # noqa: E402


def ev_median(fn, reps, flush):
    ts = []
    for _ in range(reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def graph_of(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
        with torch.cuda.graph(gr, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    return gr


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    l2 = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    clean = lambda: l2.sum()  # noqa: E731
    for n0 in (512, 4096, 16384):
        shape, rank = (n0, 512, 64), (16, 16, 4)
        x = torch.randn(*shape, dtype=torch.float64, device="cuda", generator=g)
        us = [torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g) for n, r in zip(shape, rank)]
        T = torch.empty(16, 64, dtype=torch.float64, device="cuda")
        k13 = lambda: L.call("ks_kron3_contract", D.p(us[0]), D.p(us[1]), D.p(us[2]), D.p(x), *shape, *rank,  # noqa: E731
                             D.p(T), D.stream())
        out = []
        for mode in (0, 1):
            L.call("ks_debug_kron3_stream_only", mode)
            t = ev_median(graph_of(k13).replay, 11, clean)
            out.append(f"mode{mode} {t:.1f} us {8.0 * x.numel() / t / 1e3:.0f} GB/s")
        L.call("ks_debug_kron3_stream_only", 0)
        t = ev_median(graph_of(lambda: x.sum()).replay, 11, clean)
        out.append(f"torch sum {t:.1f} us {8.0 * x.numel() / t / 1e3:.0f} GB/s")
        print(f"n0={n0} ({8.0 * x.numel() / 1e6:.0f} MB):", " | ".join(out), flush=True)
        del x


if __name__ == "__main__":
    main()
