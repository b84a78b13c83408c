"""Seeded small Tucker inputs shared by make_golden.py (reference run) and the tests (oracle / GPU)."""

import numpy as np

UNIT_SHAPE, UNIT_RANK = (12, 40, 30), (3, 4, 2)
UNIT_CFG = dict(eps=0.25, delta=0.05, alpha=1e-4, seed=7)
UNIT_LAM = 1e-2
ALS_CFG = dict(eps=0.25, delta=0.05, alpha=1e-4, seed=3)


def unit_inputs():
    rng = np.random.default_rng(2024)
    core = rng.standard_normal(UNIT_RANK)
    facs = [np.linalg.qr(rng.standard_normal((i, r)))[0] for i, r in zip(UNIT_SHAPE, UNIT_RANK)]
    x = core
    for mode, a in enumerate(facs):
        x = np.moveaxis(np.tensordot(a, x, axes=(1, mode)), 0, mode)
    x = x + 0.05 * rng.standard_normal(UNIT_SHAPE)
    return core, facs, x
