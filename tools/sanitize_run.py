"""Small end-to-end workload for compute-sanitizer (one tool per run):

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_run.py

Exercises, on tiny shapes, the kernels of the hot path: JL / spectral scores, sampler, sketch
(radix sort, sparse diagonal), the persistent eigenbasis Richardson loop (eager launch and the
whole-solve CUDA graph), the natural-basis single-role loop, the per-iteration loop, KronMatMul
(TMA + DMMA) and the loss pass."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2209_04876_b200 as K  # noqa: E402
from paper_2209_04876_b200 import solvers as S  # noqa: E402


def main():
    cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
    for (n1, n2, d1, d2) in [(256, 256, 16, 16), (320, 288, 32, 16)]:
        rng = np.random.default_rng(n1 + d1)
        facs = [torch.tensor(rng.normal(1.0, math.sqrt(1e-3), (n, d)), device="cuda") for n, d in ((n1, d1), (n2, d2))]
        b = torch.tensor(rng.standard_normal(n1 * n2), device="cuda")
        xs = [K.fast_kronecker_regression(facs, b, cfg, with_loss=(k == 2)).solution for k in range(3)]
        S._USE_FUSED[0] = False  # the separate right-hand side + per-iteration / single-role paths
        try:
            xs.append(K.fast_kronecker_regression(facs, b, cfg).solution)
        finally:
            S._USE_FUSED[0] = True
        ex = K.kronmatmul_svd_solve(facs, b, 1e-3)
        torch.cuda.synchronize()
        print(n1, n2, d1, d2, [float(torch.linalg.norm(x)) for x in xs], ex.loss, flush=True)
    print("sanitize run ok")


if __name__ == "__main__":
    main()
