"""ctypes binding of the in-tree C ABI ``libpzx_gpu.so`` (include/pzx_gpu.h).

There is no fallback: if the library is missing the import fails loudly with a
pointer to ``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpzx_gpu.so")

# every symbol declared in include/pzx_gpu.h (tests check the export table)
EXPORTS = (
    "pzx_status_string", "pzx_version", "pzx_create", "pzx_destroy", "pzx_last_error",
    "pzx_launch_count", "pzx_table_upload_expr", "pzx_table_upload", "pzx_table_free",
    "pzx_table_shape", "pzx_table_term_info", "pzx_evaluate", "pzx_evaluate_range",
    "pzx_evaluate_device", "pzx_amp_to_prob_device", "pzx_synchronize",
    "pzx_debug_phase_indices", "pzx_debug_term_codes", "pzx_table_compile_host", "pzx_class_table",
    "pzx_slice_op_table", "pzx_marginal_sum", "pzx_weak_sample", "pzx_pzx1_encode", "pzx_pzx1_encode_expr",
    "pzx_pzx1_info", "pzx_pzx1_decode", "pzx_table_upload_pzx1", "pzx_backend_contract_get",
    "pzx_group_create", "pzx_group_destroy", "pzx_group_last_error", "pzx_group_upload_expr", "pzx_group_table_free",
    "pzx_group_evaluate", "pzx_microbench", "pzx_table_upload_expr_ex", "pzx_evaluate_exact",
    "pzx_evaluate_exact_range", "pzx_ringquad_sum", "pzx_ringquad_sum_device", "pzx_table_slice_stats",
    "pzx_last_kernel", "pzx_debug_slice_codes", "pzx_circuit_reduce", "pzx_expr_get_view", "pzx_expr_info",
    "pzx_expr_free", "pzx_table_page_layout", "pzx_table_page_stats",
)

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
dblp = C.POINTER(C.c_double)


class ExprView(C.Structure):
    _fields_ = [
        ("n_params", C.c_uint32), ("n_terms", C.c_uint64),
        ("term_offset", u64p), ("term_scalar", i64p),
        ("kind", u8p), ("psi_k", u8p), ("psi_mask", u64p), ("phi_k", u8p), ("phi_mask", u64p),
    ]


class TableView(C.Structure):
    _fields_ = [
        ("n_params", C.c_uint32), ("n_terms", C.c_uint64),
        ("term_row_offset", u64p), ("term_coef", i64p),
        ("psi_mask", u64p), ("phi_mask", u64p), ("k_alpha", u8p), ("k_beta", u8p),
    ]


class BackendContract(C.Structure):
    _fields_ = [("max_params", C.c_uint32), ("max_rows_per_term", C.c_uint32),
                ("max_rows_in_flight", C.c_uint64), ("preferred_batch", C.c_uint64),
                ("exact", C.c_uint32), ("deterministic", C.c_uint32), ("n_sm", C.c_uint32),
                ("tmem_accumulators", C.c_uint32)]


class TermCode(C.Structure):
    _fields_ = [("j", C.c_uint32), ("z", C.c_uint32), ("s1", C.c_uint32),
                ("a", C.c_uint32), ("b", C.c_uint32)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.pzx_status_string.restype = C.c_char_p
    L.pzx_status_string.argtypes = [C.c_int]
    L.pzx_version.restype = C.c_char_p
    L.pzx_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.pzx_destroy.argtypes = [vp]
    L.pzx_destroy.restype = None
    L.pzx_last_error.argtypes = [vp]
    L.pzx_last_error.restype = C.c_char_p
    L.pzx_launch_count.argtypes = [vp]
    L.pzx_launch_count.restype = C.c_uint64
    L.pzx_table_upload_expr.argtypes = [vp, C.POINTER(ExprView), C.POINTER(vp)]
    L.pzx_table_upload.argtypes = [vp, C.POINTER(TableView), C.POINTER(vp)]
    L.pzx_table_free.argtypes = [vp]
    L.pzx_table_free.restype = None
    L.pzx_table_shape.argtypes = [vp, C.POINTER(C.c_uint32), u64p, u64p, C.POINTER(C.c_uint32)]
    L.pzx_table_term_info.argtypes = [vp, C.c_uint64, i64p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.pzx_evaluate.argtypes = [vp, vp, u64p, C.c_uint64, dblp, dblp, C.c_uint32]
    L.pzx_evaluate_range.argtypes = [vp, vp, C.c_uint64, C.c_uint64, dblp, dblp, C.c_uint32]
    L.pzx_evaluate_exact.argtypes = [vp, vp, u64p, C.c_uint64, i64p]
    L.pzx_evaluate_exact_range.argtypes = [vp, vp, C.c_uint64, C.c_uint64, i64p]
    L.pzx_ringquad_sum.argtypes = [vp, i64p, C.c_uint32, C.c_uint64, i64p]
    L.pzx_ringquad_sum_device.argtypes = [vp, vp, C.c_uint32, C.c_uint64, vp, vp]
    L.pzx_evaluate_device.argtypes = [vp, vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                      vp, vp, C.c_uint32, vp]
    L.pzx_amp_to_prob_device.argtypes = [vp, vp, C.c_uint64, vp, C.c_uint32, vp]
    L.pzx_synchronize.argtypes = [vp]
    L.pzx_backend_contract_get.argtypes = [vp, C.POINTER(BackendContract)]
    L.pzx_table_upload_expr_ex.argtypes = [vp, C.POINTER(ExprView), C.c_uint32, C.POINTER(vp)]
    L.pzx_microbench.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double)]
    L.pzx_group_create.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]
    L.pzx_group_destroy.argtypes = [vp]
    L.pzx_group_destroy.restype = None
    L.pzx_group_last_error.argtypes = [vp]
    L.pzx_group_last_error.restype = C.c_char_p
    L.pzx_group_upload_expr.argtypes = [vp, C.POINTER(ExprView), C.c_uint32, C.POINTER(vp)]
    L.pzx_group_table_free.argtypes = [vp]
    L.pzx_group_table_free.restype = None
    L.pzx_group_evaluate.argtypes = [vp, vp, u64p, C.c_uint64, C.c_uint64, dblp, dblp, C.c_uint32]
    L.pzx_pzx1_encode.argtypes = [C.POINTER(TableView), u8p, C.c_uint64, u64p]
    L.pzx_pzx1_encode_expr.argtypes = [C.POINTER(ExprView), u8p, C.c_uint64, u64p]
    L.pzx_pzx1_info.argtypes = [u8p, C.c_uint64, C.POINTER(C.c_uint32), u64p, u64p]
    L.pzx_pzx1_decode.argtypes = [u8p, C.c_uint64, u64p, i64p, u64p, u64p, u8p, u8p]
    L.pzx_table_upload_pzx1.argtypes = [vp, u8p, C.c_uint64, C.POINTER(vp)]
    L.pzx_marginal_sum.argtypes = [vp, vp, u64p, C.c_uint64, C.c_uint32, C.c_uint32, dblp]
    L.pzx_weak_sample.argtypes = [vp, C.POINTER(vp), C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32, u64p]
    L.pzx_debug_phase_indices.argtypes = [vp, vp, u64p, C.c_uint64, u8p]
    L.pzx_debug_term_codes.argtypes = [vp, vp, u64p, C.c_uint64, C.POINTER(TermCode)]
    L.pzx_table_compile_host.argtypes = [C.POINTER(ExprView), C.POINTER(vp)]
    L.pzx_class_table.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.pzx_slice_op_table.argtypes = [C.POINTER(C.c_int32)]
    L.pzx_table_slice_stats.argtypes = [vp, u64p, u64p]
    i32p = C.POINTER(C.c_int32)
    L.pzx_last_kernel.argtypes = [vp, i32p, i32p, i32p]
    L.pzx_debug_slice_codes.argtypes = [vp, vp, u64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                        C.POINTER(TermCode)]
    L.pzx_circuit_reduce.argtypes = [C.c_uint32, vp, C.c_uint64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.c_uint32, C.c_uint64, C.POINTER(vp)]
    L.pzx_expr_get_view.argtypes = [vp, C.POINTER(ExprView)]
    L.pzx_expr_info.argtypes = [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
    L.pzx_table_page_layout.argtypes = [vp, C.POINTER(C.c_uint32), u64p, C.POINTER(C.c_uint32), u8p, u64p]
    L.pzx_table_page_stats.argtypes = [vp, u64p, u64p]
    L.pzx_expr_free.argtypes = [vp]
    L.pzx_expr_free.restype = None
    _lib = L
    return L


def ptr(arr, ctype):
    """numpy array -> ctypes pointer (None for None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(C.POINTER(ctype))
