"""Host-side profile (cProfile) of the c5 exact core update: where the wall time beyond the device
time goes."""
import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2209_04876_b200 as K  # noqa: E402
from oracle import kronsolve_oracle as O  # noqa: E402


def main():
    shape, rank, lam = (512, 512, 64), (16, 16, 4), 1e-3
    xd = torch.tensor(O.synth_tucker(shape, rank, 0.01, 0), device="cuda")
    model = K.initial_model(xd, rank, lam, 0)
    mode = sys.argv[1] if len(sys.argv) > 1 else "exact"
    kw = {}
    if mode == "fast":
        kw = {"config": K.RegressionConfig(eps=0.1, delta=0.01, lam=lam, alpha=1e-5, seed=0),
              "caches": [K.build_factor_cache(a) for a in model.factors]}
    for _ in range(3):
        K.core_update(model, xd, mode=mode, **kw)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        K.core_update(model, xd, mode=mode, **kw)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
    pstats.Stats(pr).sort_stats("tottime").print_stats(20)


if __name__ == "__main__":
    main()
