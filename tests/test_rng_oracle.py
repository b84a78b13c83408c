"""The CPU restatement of NumPy's PCG64 + ziggurat (oracle/rng_oracle.py) and the ziggurat
tables the package extracts from the installed NumPy are pinned against NumPy itself."""

import numpy as np
import pytest

from oracle import rng_oracle as R
from paper_2209_04876_b200._numpy_rng import pcg64_state, ziggurat_tables


@pytest.mark.parametrize("seed", [0, 12345, np.random.SeedSequence(0).spawn(5)[4]])
def test_pcg64_raw_and_jump(seed):
    st, inc = pcg64_state(seed)
    raw = np.random.PCG64(seed).random_raw(2000)
    np.testing.assert_array_equal(R.raw_stream(st, inc, 2000), raw)
    np.testing.assert_array_equal(R.raw_stream(st, inc, 7, skip=1993), raw[1993:])
    u = np.random.default_rng(seed).random(50)
    np.testing.assert_array_equal(np.array([R.unit(r) for r in raw[:50]]), u)


def test_ziggurat_tables_shape():
    ki, wi, fi = ziggurat_tables()
    assert fi[0] == 1.0 and np.all(np.diff(fi) < 0)
    assert ki[1] == 0 and np.all(wi > 0)


@pytest.mark.parametrize("seed", [0, 7, np.random.SeedSequence(0).spawn(5)[1]])
def test_ziggurat_restatement_bit_exact(seed):
    n = 200_000  # ~50 tail draws and ~1400 wedge rejections
    raw = np.random.PCG64(seed).random_raw(int(n * 1.1) + 64)
    vals, used = R.standard_normals(raw, ziggurat_tables(), n)
    np.testing.assert_array_equal(vals, np.random.default_rng(seed).standard_normal(n))
    g = np.random.default_rng(seed)
    g.standard_normal(n)
    assert g.bit_generator.random_raw(1)[0] == raw[used]


@pytest.mark.parametrize("seed", [0, 7, 12345, 2 ** 40 + 3, 4294967295, 2 ** 70 + 11])
def test_seedseq_children_words_match_numpy(seed):
    """The vectorised SeedSequence children seeding (fast_factor_matrix_update's per-row streams)
    is bit-exact with NumPy: finishing pcg64_set_seed on the words gives PCG64(child).state."""
    from paper_2209_04876_b200._numpy_rng import seedseq_children_seed_words
    words = seedseq_children_seed_words(seed, 300)
    mult = 0x2360ED051FC65DA44385DF649FCCF645
    m128 = (1 << 128) - 1
    for i, child in enumerate(np.random.SeedSequence(seed).spawn(300)):
        initstate = (int(words[i, 0]) << 64) | int(words[i, 1])
        initseq = (int(words[i, 2]) << 64) | int(words[i, 3])
        inc = ((initseq << 1) | 1) & m128
        state = (((inc + initstate) & m128) * mult + inc) & m128
        st = np.random.PCG64(child).state["state"]
        assert (state, inc) == (int(st["state"]), int(st["inc"]))
