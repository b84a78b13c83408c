"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every entry point
declared in include/kronsolve_b200.h, and the ctypes binding knows them all."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "kronsolve_b200.h"
LIB = ROOT / "paper_2209_04876_b200" / "libkronsolve_b200.so"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(ks_[a-z0-9_]+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "ks_richardson_sketched" in names and "ks_kron2_contract" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    if not LIB.exists():
        pytest.skip("library not built")
    lib = ctypes.CDLL(str(LIB))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2209_04876_b200 import _lib
    assert set(declared()) == set(_lib.exported_symbols())


def test_abi_version_and_error_channel():
    if not LIB.exists():
        pytest.skip("library not built")
    from paper_2209_04876_b200 import _lib
    lib = _lib.load()
    assert lib.ks_abi_version() == _lib.ABI_VERSION
    # invalid shapes are rejected on the host side of the ABI, without touching a device
    rc = lib.ks_gemm_tn_tall(500, 4, 10, 1.0, None, 1, 1, None, 1, 1, None, None)
    assert rc == _lib.KS_EINVAL
    assert b"gemm_tn_tall" in lib.ks_last_error()


def test_error_mapping():
    from paper_2209_04876_b200 import _lib
    from paper_2209_04876_b200.errors import InvalidInputError, NumericalFailureError, SizeGuardError, \
        KronsolveError
    _lib.load()
    for rc, exc in [(_lib.KS_EINVAL, InvalidInputError), (_lib.KS_ESIZE, SizeGuardError),
                    (_lib.KS_ENUMERICAL, NumericalFailureError), (_lib.KS_EDIVERGED, NumericalFailureError),
                    (_lib.KS_ECUDA, KronsolveError)]:
        with pytest.raises(exc):
            _lib.check(rc, "x")
    assert issubclass(InvalidInputError, ValueError)


def test_kron3_supported_geometry():
    """Host-side geometry check of the K13 streaming kernel (no device work)."""
    from paper_2209_04876_b200 import _lib
    L = _lib.load()
    assert L.ks_kron3_supported(512, 512, 64, 16, 16, 4) == 1
    assert L.ks_kron3_supported(512, 512, 60, 16, 16, 4) == 0    # n2 % 8
    assert L.ks_kron3_supported(512, 512, 64, 15, 16, 4) == 1    # odd ranks are fine
    assert L.ks_kron3_supported(512, 512, 64, 2, 33, 4) == 0     # R1 > 32 (two m16 tiles of S)
    assert L.ks_kron3_supported(512, 512, 64, 64, 16, 4) == 0    # R0 R1 R2 > 2048 core entries
    assert L.ks_kron3_supported(512, 512, 256, 16, 16, 4) == 0   # n2 > 128
    assert L.ks_kron3_supported(64, 64, 64, 16, 16, 16) == 0     # R2 > 8
