"""K1 / K2 (kron2 contract / residual) device times at n = 32768 (8.6 GB b) for d = 16 / 32 / 64, L2
flushed before each launch: the HBM-bound narrow widths against the FP64-bound d = 64."""
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
    n = int(next((a[2:] for a in sys.argv[1:] if a.startswith("n=")), 32768))
    g = torch.Generator(device="cuda").manual_seed(0)
    b = torch.randn(n * n, dtype=torch.float64, device="cuda", generator=g)
    l2 = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    flush = lambda: l2.fill_(1.0)  # noqa: E731
    o = torch.empty(1, dtype=torch.float64, device="cuda")
    by = 8.0 * n * n
    ds = [int(a) for a in sys.argv[1:] if not a.startswith("n=")] or [16, 32, 64]
    for d in ds:
        f = [1.0 + 0.03 * torch.randn(n, d, dtype=torch.float64, device="cuda", generator=g) for _ in range(2)]
        T = torch.empty(d, d, dtype=torch.float64, device="cuda")
        X = torch.randn(d, d, dtype=torch.float64, device="cuda", generator=g)
        k1 = lambda: L.call("ks_kron2_contract", D.p(f[0]), D.p(b), n, D.p(f[1]), n, n, d, d, D.p(T), D.stream())  # noqa: E731
        k2 = lambda: L.call("ks_kron2_residual_sumsq", D.p(f[0]), D.p(X), D.p(f[1]), D.p(b), n, n, n, d, d,  # noqa: E731
                            D.p(o), D.stream())
        k1()
        k2()
        t1, t2 = ev_median(k1, 5, flush), ev_median(k2, 5, flush)
        fl = 2.0 * n * n * d
        print(f"d={d}: K1 {t1:.0f} us {by / t1 / 1e3:.0f} GB/s {fl / t1 / 1e6:.1f} TF/s | "
              f"K2 {t2:.0f} us {by / t2 / 1e3:.0f} GB/s {fl / t2 / 1e6:.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
