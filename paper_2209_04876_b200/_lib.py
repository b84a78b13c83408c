"""ctypes binding of libkronsolve_b200.so (the C-ABI of include/kronsolve_b200.h).

Loading fails loudly: there is no CPU fallback for any hot-path operation.  Status codes map
to the reference's exception hierarchy (reference errors.py:4-37)."""

from __future__ import annotations

import ctypes
import threading
from ctypes import POINTER, c_double, c_int32, c_int64, c_uint64, c_void_p
from pathlib import Path

from .errors import InvalidInputError, KronsolveError, NumericalFailureError, SizeGuardError

LIB_PATH = Path(__file__).resolve().parent / "libkronsolve_b200.so"

KS_OK, KS_EINVAL, KS_ESIZE, KS_ENUMERICAL, KS_ECUDA, KS_EDIVERGED = range(6)
ABI_VERSION = 1

_p = c_void_p  # device pointer / stream
_i64 = c_int64
_i32 = c_int32
_d = c_double


class SketchView(ctypes.Structure):
    """Mirror of ks_sketch_view (include/kronsolve_b200.h)."""

    _fields_ = [
        ("Lmat", c_void_p), ("ldl", c_int64), ("dL", c_int32),
        ("Rmat", c_void_p), ("ldr", c_int64), ("dR", c_int32),
        ("u_left", c_int64), ("nnz", c_int64),
        ("seg", c_void_p), ("lrow", c_void_p), ("rrow", c_void_p), ("v", c_void_p),
    ]


_SIGS = {
    "ks_abi_version": ([], ctypes.c_int),
    "ks_last_error": ([], ctypes.c_char_p),
    "ks_gemm": ([_i64, _i64, _i64, _d, _p, _i64, _i64, _i64, _p, _i64, _i64, _i64, _d, _p, _i64,
                 _i64, _i64, _i64, _p], ctypes.c_int),
    "ks_gemm_tn_tall": ([_i64, _i64, _i64, _d, _p, _i64, _i64, _p, _i64, _i64, _p, _p], ctypes.c_int),
    "ks_kron_mat_mul": ([_i32, _p, _p, _p, _p, _i64, _p, _p], ctypes.c_int),
    "ks_kron2_contract": ([_p, _p, _i64, _p, _i64, _i64, _i32, _i32, _p, _p], ctypes.c_int),
    "ks_kron2_contract_sumsq": ([_p, _p, _i64, _p, _i64, _i64, _i32, _i32, _p, _p, _p], ctypes.c_int),
    "ks_kron3_contract": ([_p, _p, _p, _p, _i64, _i64, _i64, _i32, _i32, _i32, _p, _p], ctypes.c_int),
    "ks_kron3_contract_sumsq": ([_p, _p, _p, _p, _i64, _i64, _i64, _i32, _i32, _i32, _p, _p, _p], ctypes.c_int),
    "ks_kron3_supported": ([_i64, _i64, _i64, _i32, _i32, _i32], ctypes.c_int),
    "ks_debug_kron3_stream_only": ([_i32], ctypes.c_int),
    "ks_debug_loop_kernel_event": ([_p], ctypes.c_int),
    "ks_kron2_residual_sumsq": ([_p, _p, _p, _p, _i64, _i64, _i64, _i32, _i32, _p, _p], ctypes.c_int),
    "ks_sumsq_diff": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "ks_check_finite_nonzero": ([_p, _i64, _p, _p], ctypes.c_int),
    "ks_qr_r": ([_p, _i64, _i32, _p, _p], ctypes.c_int),
    "ks_svd_small": ([_p, _i32, _p, _p, _p], ctypes.c_int),
    "ks_svd_small_batched": ([_p, _i32, _i32, _p, _p, _p], ctypes.c_int),
    "ks_debug_jl_projection_stamps": ([_p], ctypes.c_int),
    "ks_richardson_fused_async": ([POINTER(SketchView), _p, _p, _p, _p, _p, _p, _p, _p, _d, _d, _i32, _d, _p, _p,
                                   _p, _p, _p, _p], ctypes.c_int),
    "ks_richardson_plan_bytes": ([_i64, _i64], ctypes.c_int64),
    "ks_shard_loop_sizes": ([POINTER(SketchView), _p], ctypes.c_int),
    "ks_shard_loop_pack": ([POINTER(SketchView), _p, _p, _p, _p, _p, _p, _p, _p, _p], ctypes.c_int),
    "ks_shard_loop_apply": ([POINTER(SketchView), _p, _p, _p, _i32, _p, _p, _p, _p, _p], ctypes.c_int),
    "ks_shard_loop_update": ([_i32, _p, _p, _p, _p, _p, _i32, _i32, _d, _d, _d, _p, _p, _p, _p], ctypes.c_int),
    "ks_richardson_plan_async": ([POINTER(SketchView), _p, _p, _p], ctypes.c_int),
    "ks_gather_count": ([_p, _p, _p, _i64, _p, _p], ctypes.c_int),
    "ks_richardson_fused": ([POINTER(SketchView), _p, _p, _p, _p, _p, _p, _p, _d, _d, _i32, _d, _p, _p, _p,
                             POINTER(c_int32), POINTER(c_int32), _p], ctypes.c_int),
    "ks_sym_eig_batched": ([_i32, _p, _i32, _p, _p, _p], ctypes.c_int),
    "ks_compact_svd": ([_p, _i64, _i32, _d, _p, _p, _p, POINTER(c_int32), _p], ctypes.c_int),
    "ks_compact_svd_async": ([_p, _i64, _i32, _d, _p, _p, _p, _p, _p], ctypes.c_int),
    "ks_inverse_small": ([_p, _i32, _p, _p, _p], ctypes.c_int),
    "ks_pcg64_random": ([c_uint64, c_uint64, c_uint64, c_uint64, c_uint64, _i64, _p, _p], ctypes.c_int),
    "ks_pcg64_standard_normal": ([c_uint64, c_uint64, c_uint64, c_uint64, _i64, _d, _p, _p, _p, _p,
                                  _p, _p], ctypes.c_int),
    "ks_jl_scores": ([_p, _i64, _i32, _p, _i32, _d, _p, _p], ctypes.c_int),
    "ks_jl_projection": ([_p, _i32, _p, _i32, _d, _p, _p, _p], ctypes.c_int),
    "ks_jl_cholesky": ([_p, _i32, _p, _p, _p], ctypes.c_int),
    "ks_jl_solve": ([_p, _i32, _p, _i32, _d, _p, _p], ctypes.c_int),
    "ks_debug_jacobi_sweeps": ([_p], ctypes.c_int),
    "ks_row_weighted_sumsq": ([_p, _i64, _i32, _p, _p, _p], ctypes.c_int),
    "ks_sampler_tables": ([_p, _i64, _i32, _p, _p, _p, _p], ctypes.c_int),
    "ks_sampler_tables_batched": ([_i32, _p, _p, _i32, _p, _p, _p, _p], ctypes.c_int),
    "ks_searchsorted_right": ([_p, _i64, _p, _i64, _p, _i64, _i64, _p], ctypes.c_int),
    "ks_sketch_weights": ([_i32, _p, _p, _i64, _p, _p], ctypes.c_int),
    "ks_sketch_diag": ([_i32, _p, _p, _p, _i64, _p, _p, POINTER(c_int64), _p], ctypes.c_int),
    "ks_gather": ([_p, _p, _i64, _p, _p], ctypes.c_int),
    "ks_sketch_diag_grouped2": ([_p, _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p, _p], ctypes.c_int),
    "ks_sketch_diag_grouped2_ex": ([_p, _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p], ctypes.c_int),
    "ks_gather_draws2": ([_p, _p, _i64, _i64, _p, _p], ctypes.c_int),
    "ks_sketch_group": ([_i32, _p, _p, _p, _i32, _p, _i32, _p, _p, _p, _i64, _p, _p, _p, _p, _p, _p,
                         _p, POINTER(c_int64), _p], ctypes.c_int),
    "ks_sketched_apply": ([POINTER(SketchView), _p, _p, _p, _p], ctypes.c_int),
    "ks_sketched_transpose_apply": ([POINTER(SketchView), _p, _p, _p, _p], ctypes.c_int),
    "ks_richardson_sketched": ([POINTER(SketchView), _p, _p, _p, _p, _d, _d, _i32, _d, _p, _p,
                                POINTER(c_int32), POINTER(c_int32), _p], ctypes.c_int),
    "ks_kron_precond_apply": ([_p, _p, _i32, _i32, _p, _p, _p, _p], ctypes.c_int),
    "ks_debug_richardson_phases": ([_i32, POINTER(c_double)], ctypes.c_int),
    "ks_debug_richardson_profile": ([_i32], ctypes.c_int),
    "ks_debug_richardson_apply_split": ([_i32, POINTER(c_double)], ctypes.c_int),
    "ks_debug_richardson_cta_apply": ([_i32, _p], ctypes.c_int),
    "ks_pcg64_random_streams": ([_p, _i32, _i64, _i32, _i64, _p, _p], ctypes.c_int),
    "ks_factor_draws_rows": ([_i32, _p, _p, _p, _p, _i64, _i64, _p, _p, _p], ctypes.c_int),
    "ks_factor_workspace": ([_i32, _p, _p, _p, _p, _i32, _p, _p, _d, _d, _p, _p, _p, _p, _p, _p, _p],
                            ctypes.c_int),
    "ks_factor_ws_apply": ([_i32, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _d, _p, _i32, _p, _p], ctypes.c_int),
    "ks_factor_rows_smem": ([_i32, _i32, _i32, _i32, _i32, _i32, _i32], ctypes.c_int64),
    "ks_factor_rows_richardson": ([_i32, _p, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _d, _p, _p, _i64, _i32,
                                   _i64, _p, _i64, _p, _p, _d, _i32, _d, _i32, _p, _p, _p, _p, _p], ctypes.c_int),
    "ks_qr_explicit": ([_p, _i64, _i32, _p, _p], ctypes.c_int),
    "ks_pinv_compose": ([_p, _i64, _p, _p, _i64, _i32, _p, _p], ctypes.c_int),
    "ks_kron_explicit2": ([_p, _i64, _i32, _p, _i64, _i32, _p, _p], ctypes.c_int),
    "ks_scaled_row_gather": ([_p, _i64, _i32, _p, _p, _i64, _d, _p, _p], ctypes.c_int),
    "ks_sketch_rows": ([_i32, _p, _p, _p, _p, _i32, _p, _i64, _p, _p], ctypes.c_int),
    "ks_chol_qr2_r": ([_p, _i64, _i32, _p, POINTER(c_int32), _p], ctypes.c_int),
    "ks_leverage_scores_tall": ([_p, _i64, _i32, _p, POINTER(c_int32), _p], ctypes.c_int),
    "ks_leverage_scores_tall_async": ([_p, _i64, _i32, _p, _p, _p], ctypes.c_int),
}

_lock = threading.Lock()
_lib = None


def exported_symbols():
    """Names of every C-ABI entry point the binding expects (include/kronsolve_b200.h)."""
    return sorted(_SIGS)


def load():
    """Load the shared library (raises if it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2209_04876_b200._build` "
                "(the B200 hot path has no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.ks_abi_version() != ABI_VERSION:
            raise ImportError("libkronsolve_b200.so ABI version mismatch; rebuild it")
        _lib = lib
    return _lib


def check(rc: int, what: str = "", **diag):
    if rc == KS_OK:
        return
    msg = (_lib.ks_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == KS_EINVAL:
        raise InvalidInputError(text)
    if rc == KS_ESIZE:
        raise SizeGuardError(text)
    if rc in (KS_ENUMERICAL, KS_EDIVERGED):
        raise NumericalFailureError(text, iterations=diag.get("iterations"),
                                    diagnostics=diag.get("diagnostics"))
    raise KronsolveError(text)


def call(name: str, *args, what: str = ""):
    lib = load()
    rc = getattr(lib, name)(*args)
    check(rc, what or name)
    return rc


def ptr_array(ctype, values):
    """Host array of plain values/pointers for the ABI's `const T*` host-side arguments."""
    return (ctype * len(values))(*values)
