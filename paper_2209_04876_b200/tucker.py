"""Tucker-ALS core update on the device.

Drop-in for ``TuckerModel`` (tucker.py:45-77) and ``core_update`` (tucker.py:108-127) of
pkg/src/kronsolve/tucker.py: the core regression against the 3-factor implicit Kronecker
design is solved exactly (kronmatmul_svd_solve) or with the sketched solver (reusing cached
per-factor SVD + Gram data) -- both entirely on the GPU."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _device as D
from .errors import InvalidInputError
from .solvers import (FactorCache, RegressionConfig, fast_kronecker_regression, kronmatmul_svd_solve)
from .tensor import as_tensor, devectorize, vectorize


@dataclass
class TuckerModel:
    """Core tensor plus one loading matrix per mode (tucker.py:45-77)."""

    core: object
    factors: list
    lam: float = 0.0

    def __post_init__(self):
        host = not D.on_device(self.core)
        core = as_tensor(self.core, "core")
        self.core = D.out(core, host)
        if len(self.factors) != core.ndim:
            raise InvalidInputError(
                f"core has order {core.ndim} but got {len(self.factors)} factors")
        facs = []
        for n, a in enumerate(self.factors):
            a = a if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
            if a.ndim != 2 or a.shape[1] != core.shape[n]:
                raise InvalidInputError(
                    f"factor {n} of shape {tuple(a.shape)} does not match core dim {core.shape[n]}")
            if a.shape[0] < a.shape[1]:
                raise InvalidInputError(
                    f"factor {n} is {tuple(a.shape)}; ranks above the dimension are not supported")
            facs.append(a)
        self.factors = facs
        if self.lam < 0:
            raise InvalidInputError(f"lambda must be >= 0, got {self.lam}")

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(int(a.shape[0]) for a in self.factors)

    @property
    def core_shape(self) -> tuple[int, ...]:
        return tuple(int(s) for s in self.core.shape)


def core_update(model: TuckerModel, x, mode: str = "exact", config: RegressionConfig | None = None,
                caches: Sequence[FactorCache] | None = None):
    """Solve the core regression at fixed factors; returns the new core (tucker.py:108-127)."""
    xs = tuple(int(s) for s in x.shape) if hasattr(x, "shape") else np.asarray(x).shape
    if tuple(xs) != model.shape:
        raise InvalidInputError(f"tensor shape {tuple(xs)} != model shape {model.shape}")
    if mode == "exact":
        report = kronmatmul_svd_solve(model.factors, vectorize(x), model.lam)
    elif mode == "fast":
        cfg = (config or RegressionConfig()).with_lam(model.lam)
        report = fast_kronecker_regression(model.factors, vectorize(x), cfg, caches=caches)
    else:
        raise InvalidInputError(f"unknown core update mode {mode!r}")
    return devectorize(report.solution, model.core_shape)
