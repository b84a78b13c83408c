"""ks_sampler_tables alone (one CTA per factor): device time for n = 16384 / 65536 with and without
the exact cumsum -- the split between the pairwise total + probabilities and the sequential cdf."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2209_04876_b200 import _lib as L, _device as D  # noqa: E402


def ev(fn, reps=11):
    ts = []
    for _ in range(reps):
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
    for n in (16384, 65536):
        sc = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
        p, c = D.empty(n), D.empty(n)
        fl = torch.zeros(1, dtype=torch.int32, device="cuda")
        f_nocdf = lambda: L.call("ks_sampler_tables", D.p(sc), n, 0, D.p(p), None, D.p(fl), D.stream())  # noqa: E731
        f_cdf = lambda: L.call("ks_sampler_tables", D.p(sc), n, 1, D.p(p), D.p(c), D.p(fl), D.stream())  # noqa: E731
        f_nocdf()
        f_cdf()
        torch.cuda.synchronize()
        print(f"n={n}: total+probs {ev(f_nocdf):.1f} us, with exact cdf {ev(f_cdf):.1f} us", flush=True)


if __name__ == "__main__":
    main()
