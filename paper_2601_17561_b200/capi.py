"""ctypes binding of the C ABI (include/irl_capi.h) exported by libirl_b200.so.

This is plumbing for the Python host mirror (modmat.py, ccmm.py), the tests
and bench.py. It never computes anything itself: if the CUDA library is not
built, or no sm_100 device is present, loading / context creation raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libirl_b200.so"

u8p = C.POINTER(C.c_uint8)
i8p = C.POINTER(C.c_int8)
u16p = C.POINTER(C.c_uint16)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)
sz = C.c_size_t
vp = C.c_void_p

IRL_OK = 0
IRL_ERR_SHAPE_MISMATCH = 1
IRL_ERR_MODULUS_TOO_LARGE = 2
IRL_ERR_ACCUMULATION_OVERFLOW_RISK = 3
IRL_ERR_NOT_COPRIME = 4
IRL_ERR_MODULUS_BUDGET = 5
IRL_ERR_INVALID_ARGUMENT = 6
IRL_ERR_CUDA = 7
IRL_ERR_NO_DEVICE = 8
IRL_ERR_OUT_OF_MEMORY = 9
IRL_ERR_UNSUPPORTED = 10
IRL_ERR_ZERO_OVERLAP = 11
IRL_ERR_IO = 12
IRL_ERR_CONFIG = 13

IRL_EXCHANGE_AUTO, IRL_EXCHANGE_P2P, IRL_EXCHANGE_MULTICAST, IRL_EXCHANGE_COPY = 0, 1, 2, 3

# Every symbol include/irl_capi.h declares, with (restype, argtypes).
SIGNATURES = {
    "irl_abi_version": (C.c_int, []),
    "irl_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "irl_ctx_destroy": (C.c_int, [vp]),
    "irl_last_error": (C.c_char_p, [vp]),
    "irl_status_string": (C.c_char_p, [C.c_int]),
    "irl_kernel_launches": (C.c_uint64, [vp]),
    "irl_ctx_stream": (vp, [vp]),
    "irl_diag_ppmm": (C.c_int, [vp, C.c_int, C.POINTER(C.c_uint64), sz]),
    "irl_paper_basis": (sz, [u32p, u32p, sz]),
    "irl_basis_Q_bytes": (sz, [u32p, u32p, sz, u8p, sz]),
    "irl_digit_decompose": (C.c_int, [vp, i32p, sz, sz, C.c_uint32, i32p, i32p]),
    "irl_digit_recompose": (C.c_int, [vp, i32p, i32p, sz, sz, C.c_uint32, i32p]),
    "irl_small_gemm": (C.c_int, [vp, i32p, i32p, i32p, sz, sz, sz]),
    "irl_gemm_mod_psq": (C.c_int, [vp, i32p, i32p, i32p, sz, sz, sz, C.c_uint32]),
    "irl_gemm_mod_Q": (C.c_int, [vp, u8p, u8p, u8p, sz, sz, sz, sz, u32p, u32p, sz]),
    "irl_split_rows_u16": (C.c_int, [vp, vp, sz, sz, sz, sz, u32p, u32p, sz, vp, sz, vp]),
    "irl_split_cols_u16": (C.c_int, [vp, vp, sz, sz, sz, sz, u32p, u32p, sz, vp, sz, vp]),
    "irl_split_bigint": (C.c_int, [vp, vp, sz, sz, sz, C.c_int, u32p, u32p, sz, vp, sz, vp]),
    "irl_ppmm_planes": (C.c_int, [vp, vp, vp, vp, sz, sz, sz, sz, sz, u32p, u32p, sz, C.c_int, vp]),
    "irl_crt_lift": (C.c_int, [vp, vp, sz, sz, vp, sz, u32p, u32p, sz, vp]),
    "irl_synth_residue": (C.c_uint32, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "irl_synth_residues_host": (None, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint32, u16p]),
    "irl_ccmm_create": (C.c_int, [vp, sz, sz, sz, sz, u32p, u32p, sz, C.POINTER(vp)]),
    "irl_ccmm_destroy": (C.c_int, [vp]),
    "irl_ccmm_load_part": (C.c_int, [vp, sz, vp, C.c_int]),
    "irl_ccmm_load_part_bigint": (C.c_int, [vp, sz, u8p, sz]),
    "irl_ccmm_synth_db": (C.c_int, [vp, C.c_uint64, C.c_uint32]),
    "irl_ccmm_load_part_file": (C.c_int, [vp, sz, C.c_char_p]),
    "irl_ccmm_run": (C.c_int, [vp, vp, sz, vp]),
    "irl_ccmm_run_device": (C.c_int, [vp, vp, C.c_int, sz, sz, sz, vp, vp]),
    "irl_ccmm_buffers": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp)]),
    "irl_ccmm_device_bytes": (C.c_uint64, [vp]),
    "irl_ccmm_twin": (C.c_int, [vp, C.c_long, C.c_long, C.c_long, C.c_long, C.c_long, C.c_double, C.c_double,
                                C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "irl_rescale_residues": (C.c_int, [vp, vp, sz, sz, u32p, u32p, sz, sz, C.c_int, vp, sz, vp]),
    "irl_ccmm_rescale": (C.c_int, [vp, sz, sz, sz, sz, C.c_int, vp, vp]),
    "irl_ccmm_run_dq": (C.c_int, [vp, vp, sz, vp, vp]),
    "irl_iris_db_create": (C.c_int, [vp, vp, vp, sz, sz, sz, C.POINTER(vp)]),
    "irl_iris_db_destroy": (C.c_int, [vp]),
    "irl_iris_db_create_file": (C.c_int, [vp, C.c_char_p, sz, C.POINTER(vp), C.POINTER(sz), C.POINTER(sz)]),
    "irl_iris_db_match": (C.c_int, [vp, vp, vp, sz, sz, C.c_double, C.c_double, vp, vp, vp]),
    "irl_ccmm_alloc_recv": (C.c_int, [vp, sz, C.POINTER(vp), vp]),
    "irl_ccmm_set_mirrors": (C.c_int, [vp, sz, sz, vp, sz]),
    "irl_ccmm_set_mirror_ptrs": (C.c_int, [vp, sz, sz, C.POINTER(vp), sz]),
    "irl_ccmm_set_mirror_slot": (C.c_int, [vp, sz]),
    "irl_ccmm_set_mirror_parts": (C.c_int, [vp, sz]),
    "irl_ccmm_alloc_recv_parts": (C.c_int, [vp, sz, sz, C.POINTER(vp), vp]),
    "irl_ccmm_synth_part": (C.c_int, [vp, sz, C.c_uint64, C.c_uint32, C.c_uint32]),
    "irl_iris_inner_overlap": (C.c_int, [vp, vp, vp, sz, vp, vp, sz, sz, sz, vp, vp]),
    "irl_iris_match": (C.c_int, [vp, vp, vp, sz, vp, vp, sz, sz, sz, C.c_double, C.c_double, vp, vp, vp]),
    "irl_fold_stage": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "irl_fold_stage_device": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "irl_iris_db_fold": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "irl_ccmm_group_create": (C.c_int, [vp, sz, sz, sz, sz, sz, vp, vp, sz, C.POINTER(vp)]),
    "irl_ccmm_group_destroy": (C.c_int, [vp]),
    "irl_ccmm_group_engine": (C.c_int, [vp, sz, C.POINTER(vp), C.POINTER(sz), C.POINTER(sz)]),
    "irl_ccmm_group_ctx": (vp, [vp, sz]),
    "irl_ccmm_full": (C.c_int, [vp, vp, sz, vp, C.POINTER(vp), C.POINTER(C.c_int)]),
    "irl_ccmm_group_set_exchange": (C.c_int, [vp, C.c_int]),
    "irl_ccmm_group_set_query_shard": (C.c_int, [vp, C.c_int]),
    "irl_ccmm_set_mirror_multicast": (C.c_int, [vp, sz, sz, vp]),
}


class FoldParams(C.Structure):
    """irl_fold_params (include/irl_capi.h)."""
    _fields_ = [("batch", sz), ("rho", sz), ("n_db", sz), ("d", sz), ("fold_k", sz),
                ("fold_coeffs", C.POINTER(C.c_double)), ("fold_len", sz),
                ("chain_stages", sz), ("chain_centers", C.POINTER(C.c_double)),
                ("chain_lens", C.POINTER(sz)), ("chain_coeffs", C.POINTER(C.c_double)),
                ("negative_lo", C.c_double), ("negative_hi", C.c_double)]

_lib = None


class IrlLibraryMissing(RuntimeError):
    pass


def lib() -> C.CDLL:
    """Load libirl_b200.so (fails loudly when the CUDA extension is missing)."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("IRL_B200_LIB", LIB_PATH))
        if not path.exists():
            raise IrlLibraryMissing(
                f"{path} is not built; run `python -m paper_2601_17561_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def ptr(a, t=vp):
    """numpy array -> ctypes pointer; torch tensor -> raw device pointer."""
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(t)
