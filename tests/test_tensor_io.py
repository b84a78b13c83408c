"""KTN1 tensor files and CSV helpers (paper_2209_04876_b200/tensor_io.py) -- host-side parsing,
checked against the format contract of the reference (tensor_io.py) and, in the build container,
byte-for-byte against files written by the live reference."""

import csv
import struct
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC
from paper_2209_04876_b200.errors import InvalidInputError, TensorFormatError
from paper_2209_04876_b200.tensor_io import (read_matrix_csv, read_tensor, write_matrix_csv, write_results_csv,
                                             write_tensor)


@pytest.mark.parametrize("shape", [(1,), (4,), (2, 3), (3, 2, 4, 2)])
def test_roundtrip_bitwise(rng, tmp_path, shape):
    x = rng.standard_normal(shape)
    write_tensor(tmp_path / "x.ktn", x)
    back = read_tensor(tmp_path / "x.ktn")
    assert back.shape == x.shape and back.dtype == np.float64
    assert np.array_equal(back, x)


def test_exact_byte_layout(rng, tmp_path):
    x = rng.standard_normal((2, 3))
    write_tensor(tmp_path / "x.ktn", x)
    raw = (tmp_path / "x.ktn").read_bytes()
    assert len(raw) == 73 and raw[:4] == b"KTN1" and struct.unpack_from("<I", raw, 4)[0] == 1 and raw[8] == 2
    assert struct.unpack_from("<QQ", raw, 9) == (2, 3)
    np.testing.assert_array_equal(np.frombuffer(raw, dtype="<f8", offset=25).reshape(2, 3), x)


@pytest.mark.parametrize("case,code", [("magic", "bad-magic"), ("version", "bad-version"), ("trunc", "truncated"),
                                       ("overflow", "dim-overflow"), ("zero", "dim-overflow"),
                                       ("short", "truncated")])
def test_format_errors(rng, tmp_path, case, code):
    p = tmp_path / "x.ktn"
    write_tensor(p, rng.standard_normal((2, 2)))
    raw = bytearray(p.read_bytes())
    if case == "magic":
        raw = bytearray(b"NOPE" + b"\x00" * 40)
    elif case == "version":
        raw[4:8] = struct.pack("<I", 9)
    elif case == "trunc":
        raw = raw[:-5]
    elif case == "overflow":
        raw = bytearray(b"KTN1" + struct.pack("<I", 1) + struct.pack("<B", 2) + struct.pack("<QQ", 2 ** 40, 2 ** 40))
    elif case == "zero":
        raw[9:17] = struct.pack("<Q", 0)
    elif case == "short":
        raw = raw[:6]
    p.write_bytes(bytes(raw))
    with pytest.raises(TensorFormatError) as err:
        read_tensor(p)
    assert err.value.code == code


def test_non_finite_rejected(tmp_path):
    with pytest.raises(InvalidInputError):
        write_tensor(tmp_path / "x.ktn", np.array([1.0, np.nan]))


def test_csv_helpers(rng, tmp_path):
    m = rng.standard_normal((4, 3))
    write_matrix_csv(tmp_path / "m.csv", m)
    np.testing.assert_array_equal(read_matrix_csv(tmp_path / "m.csv"), m)
    (tmp_path / "bad.csv").write_text("1,2\n3\n")
    with pytest.raises(InvalidInputError):
        read_matrix_csv(tmp_path / "bad.csv")
    values = list(rng.standard_normal(50)) + [1e-300, 1e300, 1.0 / 3.0]
    write_results_csv(tmp_path / "r.csv", ["value"], [(v,) for v in values])
    with open(tmp_path / "r.csv", newline="") as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == ["value"] and [float(r[0]) for r in rows[1:]] == values
    write_results_csv(tmp_path / "h.csv", ["a", "b"], [(1.5, "x")])
    assert (tmp_path / "h.csv").read_text().splitlines()[:2] == ["a,b", "1.5,x"]


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference not mounted (GPU box)")
def test_files_identical_to_live_reference(rng, tmp_path):
    sys.path.insert(0, str(REFERENCE_SRC))
    from kronsolve import tensor_io as R
    x = rng.standard_normal((3, 5, 2))
    R.write_tensor(tmp_path / "r.ktn", x)
    write_tensor(tmp_path / "o.ktn", x)
    assert (tmp_path / "r.ktn").read_bytes() == (tmp_path / "o.ktn").read_bytes()
    assert np.array_equal(R.read_tensor(tmp_path / "o.ktn"), read_tensor(tmp_path / "r.ktn"))
    R.write_results_csv(tmp_path / "r.csv", ["a", "b"], [(1 / 3, "x"), (np.float64(2.5), 7)])
    write_results_csv(tmp_path / "o.csv", ["a", "b"], [(1 / 3, "x"), (np.float64(2.5), 7)])
    assert (tmp_path / "r.csv").read_text() == (tmp_path / "o.csv").read_text()


@pytest.mark.gpu
def test_device_read_and_write(rng, tmp_path):
    import torch
    x = rng.standard_normal((16, 8, 4))
    write_tensor(tmp_path / "x.ktn", torch.tensor(x, device="cuda"))
    t = read_tensor(tmp_path / "x.ktn", device=True)
    assert t.is_cuda and tuple(t.shape) == x.shape
    assert np.array_equal(t.cpu().numpy(), x)
