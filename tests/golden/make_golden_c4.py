"""Golden fixtures for BASELINE config 4 (n = 65536, d in {16, 32, 64, 128}) by running the
REFERENCE itself.  Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_c4.py [d ...]

c4's right-hand side is b = default_rng(0).standard_normal(n^2): 4.29e9 entries,
34.4 GB.  It is streamed once, in sequential chunks of one Generator (the same stream as a single
call), into a page-cached memory map under /tmp, and the reference's own
``fast_kronecker_regression`` / ``kronmatmul_svd_solve`` read it in place (``np.asarray`` of a
memmap does not copy; the fast solve touches only ``b[sdiag.indices]``, solvers.py:448).

The one substitution: the reference's ``ridge_loss`` (solvers.py:251-262) materialises K x and
K x - b (2 x 34 GB), which does not fit this container's 62 GB.  It is replaced, for these runs
only, by the same quantity summed over row blocks of the n x n reshape of b
(||A1[blk] X A2^T - B[blk]||^2 accumulated block by block, + lam ||x||^2).  The block sum
differs from the reference's single ``r @ r`` only in summation order (relative ~1e-13; the loss
contract is 1e-9).  Everything else -- spectral row sampling, JL scores, product sampling, the
sparse diagonal, the Richardson loop, the exact SVD solve -- is the unmodified reference.

Outputs: c4_d{d}.npz next to this script (sketch indices, sparse diagonal, right-hand side,
step-norm history, fast x and loss, exact x and OPT).  The GPU box regenerates b on the device
(bit-exact stream, tests/test_gpu_c4.py) and compares against these files.
"""

from __future__ import annotations

import math
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

N4 = 65536
B_PATH = Path(os.environ.get("KS_C4_B", "/tmp/ks_c4_b.f64"))
CHUNK = 1 << 26


def c4_b():
    """default_rng(0).standard_normal(n^2) as a read-only memmap (generated once)."""
    total = N4 * N4
    if not B_PATH.exists() or B_PATH.stat().st_size != total * 8:
        t0 = time.time()
        mm = np.memmap(B_PATH, dtype=np.float64, mode="w+", shape=(total,))
        gen = np.random.default_rng(0)
        for i in range(0, total, CHUNK):
            gen.standard_normal(size=min(CHUNK, total - i), out=mm[i:i + CHUNK])
        mm.flush()
        del mm
        print(f"b generated in {time.time() - t0:.1f} s", flush=True)
    return np.memmap(B_PATH, dtype=np.float64, mode="r", shape=(N4 * N4,))


def c4_factors(d):
    """experiments.py:106-115 factors (A1 then A2 from default_rng(0)) without its all-ones b."""
    gen = np.random.default_rng(0)
    return [gen.normal(1.0, math.sqrt(0.001), (N4, d)) for _ in range(2)]


def blocked_ridge_loss(factors, x, b, lam, rows_per_block=512):
    """||K x - b||^2 + lam ||x||^2 over row blocks of the n1 x n2 reshape of b (two factors)."""
    a1, a2 = (np.asarray(f, dtype=np.float64) for f in factors)
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    xm = x.reshape(a1.shape[1], a2.shape[1])
    bm = np.asarray(b).reshape(a1.shape[0], a2.shape[0])
    right = xm @ a2.T  # d1 x n2
    acc = 0.0
    for i in range(0, a1.shape[0], rows_per_block):
        r = a1[i:i + rows_per_block] @ right
        r -= bm[i:i + rows_per_block]
        acc += float(np.einsum("ij,ij->", r, r))
    return acc + lam * float(x @ x)


def main(ds):
    import make_golden as MG
    ks, ks_solvers = MG.ks, MG.ks_solvers
    b = c4_b()
    orig_loss = ks_solvers.ridge_loss
    ks_solvers.ridge_loss = blocked_ridge_loss
    try:
        for d in ds:
            t0 = time.time()
            facs = c4_factors(d)
            cfg = ks.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
            hist, o1 = MG.capture_history()
            sk, o2 = MG.capture_sketch()
            try:
                fast = ks.fast_kronecker_regression(facs, b, cfg)
            finally:
                ks_solvers.richardson_solve = o1
                ks_solvers.sample_rows = o2
            t1 = time.time()
            exact = ks.kronmatmul_svd_solve(facs, b, 1e-3)
            sd = ks.sparse_diagonal_from_sketch(ks.RowSketch(sk["indices"], sk["weights"]), (N4, N4))
            np.savez_compressed(
                HERE / f"c4_d{d}.npz", n=N4, d=d, x=fast.solution, loss=fast.loss, iterations=fast.iterations,
                s=fast.sample_count, indices=sk["indices"].astype(np.int32), weights=sk["weights"],
                sd_indices=sd.indices, sd_values=sd.values, rhs=hist["rhs"], history=np.asarray(hist["history"]),
                exact_x=exact.solution, opt=exact.loss, fast_wall_time=fast.wall_time)
            print(f"c4 d={d}: s {fast.sample_count} iters {fast.iterations} loss {fast.loss!r} opt {exact.loss!r} "
                  f"fast wall {fast.wall_time:.2f} s (run {t1 - t0:.1f} s, exact {time.time() - t1:.1f} s)",
                  flush=True)
    finally:
        ks_solvers.ridge_loss = orig_loss


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [16, 32, 64, 128])
