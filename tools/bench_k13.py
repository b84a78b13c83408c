"""K13 (ks_kron3_contract) at c5 (512 x 512 x 64, rank 16/16/4): device time with L2 flushed, against
the round-2-start path (K1 on the materialised right group)."""
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


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    shape, rank = (512, 512, 64), (16, 16, 4)
    x = torch.randn(*shape, dtype=torch.float64, device="cuda", generator=g)
    us = [torch.randn(n, r, dtype=torch.float64, device="cuda", generator=g) for n, r in zip(shape, rank)]
    ur = torch.kron(us[1], us[2]).contiguous()
    T = torch.empty(16, 64, dtype=torch.float64, device="cuda")
    T1 = torch.empty_like(T)
    l2 = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    flush = lambda: l2.fill_(1.0)  # noqa: E731
    k13 = lambda: L.call("ks_kron3_contract", D.p(us[0]), D.p(us[1]), D.p(us[2]), D.p(x), *shape, *rank,  # noqa: E731
                         D.p(T), D.stream())
    k1 = lambda: L.call("ks_kron2_contract", D.p(us[0]), D.p(x), 32768, D.p(ur), 512, 32768, 16, 64, D.p(T1),  # noqa: E731
                        D.stream())
    for _ in range(3):
        k13()
        k1()
    torch.cuda.synchronize()
    rel = float((T - T1).norm() / T1.norm())
    t13, t1 = ev_median(k13, 21, flush), ev_median(k1, 21, flush)
    by = 8.0 * x.numel()
    print(f"eager call: k13 {t13:.1f} us ({by / t13 / 1e3:.0f} GB/s)  k1-group {t1:.1f} us  rel {rel:.2e}")
    # device time without the host-side preparation (tensor maps, attributes): graph replays
    gs = []
    for fn in (k13, k1):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            fn()
            with torch.cuda.graph(gr, stream=s):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        gs.append(ev_median(gr.replay, 21, flush))
        if fn is k13:
            gr13 = gr
    print(f"graph replay: k13 {gs[0]:.1f} us ({by / gs[0] / 1e3:.0f} GB/s)  k1-group {gs[1]:.1f} us")
    clean = lambda: l2.sum()  # noqa: E731  (L2 left holding clean lines)
    print(f"graph replay, clean flush: k13 {ev_median(gr13.replay, 21, clean):.1f} us")
    L.call("ks_debug_kron3_stream_only", 1)
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        k13()
        with torch.cuda.graph(gr, stream=s):
            k13()
    torch.cuda.current_stream().wait_stream(s)
    print(f"stream only (no arithmetic): dirty flush {ev_median(gr.replay, 21, flush):.1f} us, "
          f"clean flush {ev_median(gr.replay, 21, clean):.1f} us")
    L.call("ks_debug_kron3_stream_only", 2)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        k13()
        with torch.cuda.graph(gr, stream=s):
            k13()
    torch.cuda.current_stream().wait_stream(s)
    print(f"stream only, contiguous 1-D bulk copies: dirty flush {ev_median(gr.replay, 21, flush):.1f} us, "
          f"clean flush {ev_median(gr.replay, 21, clean):.1f} us")
    L.call("ks_debug_kron3_stream_only", 0)


if __name__ == "__main__":
    main()
