"""Tucker-ALS core update (BASELINE config 5) vs the reference golden fixture."""

import json
from pathlib import Path

import numpy as np
import pytest

from conftest import rel
from oracle import kronsolve_oracle as O

pytestmark = pytest.mark.gpu
# the reference's own noise floor of the fast core (tests/golden/measure_floor.py aux -> floor.json)
C5_FAST_FLOOR = json.loads((Path(__file__).resolve().parent / "golden" / "floor.json").read_text())["c5_fast_core"]["core"]


@pytest.fixture(scope="module")
def c5():
    x = O.synth_tucker((512, 512, 64), (16, 16, 4), 0.01, seed=0)
    facs = O.initial_tucker_factors(x.shape, (16, 16, 4), 0)
    return x, facs


def test_core_update_exact_and_fast(golden, c5):
    import paper_2209_04876_b200 as K
    g = golden("c5")
    x, facs = c5
    assert float(np.sum(x)) == pytest.approx(float(g["xsum"]), rel=1e-12)
    model = K.TuckerModel(core=np.zeros((16, 16, 4)), factors=facs, lam=1e-3)
    core = K.core_update(model, x, mode="exact")
    assert rel(core, g["core_exact"]) <= 1e-9
    model.core = core
    caches = [K.build_factor_cache(a) for a in model.factors]
    cfg = K.RegressionConfig(eps=0.1, delta=0.01, lam=1e-3, alpha=1e-5, seed=0)
    fast = K.core_update(model, x, mode="fast", config=cfg, caches=caches)
    assert rel(fast, g["core_fast"]) <= 2 * C5_FAST_FLOOR


def test_core_update_validation(c5):
    import paper_2209_04876_b200 as K
    from paper_2209_04876_b200.errors import InvalidInputError
    x, facs = c5
    model = K.TuckerModel(core=np.zeros((16, 16, 4)), factors=facs, lam=1e-3)
    with pytest.raises(InvalidInputError):
        K.core_update(model, x, mode="bogus")
    with pytest.raises(InvalidInputError):
        K.core_update(model, x[:10], mode="exact")
