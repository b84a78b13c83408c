"""Where the Tucker exact / fast core update's time goes at c5: kernel list (torch profiler) and the
wall time of one call."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2209_04876_b200 as K  # noqa: E402
from oracle import kronsolve_oracle as O  # noqa: E402


def main():
    shape, rank, lam = (512, 512, 64), (16, 16, 4), 1e-3
    x = O.synth_tucker(shape, rank, 0.01, 0)
    xd = torch.tensor(x, device="cuda")
    model = K.initial_model(xd, rank, lam, 0)
    cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=lam, alpha=1e-5, seed=0)
    caches = [K.build_factor_cache(a) for a in model.factors]
    for mode in ("exact", "fast"):
        kw = {} if mode == "exact" else {"config": cfg, "caches": caches}
        for _ in range(3):
            K.core_update(model, xd, mode=mode, **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            K.core_update(model, xd, mode=mode, **kw)
        torch.cuda.synchronize()
        print(f"{mode}: wall {(time.perf_counter() - t0) / 10 * 1e6:.0f} us per call")
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                                torch.profiler.ProfilerActivity.CUDA]) as prof:
            K.core_update(model, xd, mode=mode, **kw)
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))


if __name__ == "__main__":
    main()
