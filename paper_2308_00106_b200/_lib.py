"""ctypes binding of libsme.so — the C-ABI declared in include/sme.h.

This module is the only place that touches the shared library.  Loading it is
lazy; a missing library or a missing CUDA device raises immediately (there is
no CPU fallback anywhere on the product path).
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libsme.so"

SME_OK, SME_EINVAL, SME_ECUDA, SME_ENOSPACE = 0, -1, -2, -3
SME_F64, SME_F32, SME_I32 = 0, 1, -1
FLAG_RANGE, FLAG_NOT_BIJECTION, FLAG_DUPLICATE, FLAG_ROWPTR, FLAG_UNSORTED = 1, 2, 4, 8, 16
SORT_SMEM_MAX = 4096

p = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
u64 = C.c_uint64
f64 = C.c_double
sz = C.c_size_t
psz = C.POINTER(C.c_size_t)
pi64 = C.POINTER(C.c_int64)

# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES: dict[str, list] = {
    "sme_last_error": [],
    "sme_version": [],
    "sme_device_sm_count": [],
    "sme_preload": [],
    "sme_device_info": [p],
    "sme_l2_set_persisting": [sz],
    "sme_l2_window": [p, sz, C.c_float, p],
    "sme_l2_reset_persisting": [],
    "sme_l2_prefetch": [p, sz, p],
    "sme_host_pcg64_permutation": [p, i64, p],
    "sme_host_pcg64_swap_partners": [p, i64, p, C.c_int],
    "sme_pcg64_swap_partners_to_device": [p, i64, p, C.c_int, p],
    "sme_pcg64_swap_partners_gpu_workspace_size": [i64, psz],
    "sme_pcg64_swap_partners_gpu": [p, i64, p, p, sz, p],
    "sme_fy_apply_workspace_size": [i64, psz],
    "sme_fy_apply": [i64, p, p, p, sz, p],
    "sme_host_mm_parse": [p, i64, C.c_int, i64, i64, i64, i64, C.c_int, C.c_int, p, p, p, p],
    "sme_host_mm_format": [p, p, p, i64, p, i64, C.c_int, p],
    "sme_perm_inverse": [i64, p, p, p, p],
    "sme_permute_vector": [C.c_int, i64, p, p, p, p],
    "sme_gather": [C.c_int, i64, p, p, p, p],
    "sme_coo_remap": [i64, p, p, p, p, p, p, p],
    "sme_row_ptr_workspace_size": [i64, psz],
    "sme_coo_row_ptr": [i64, i64, i64, p, p, p, p, p, sz, p, p],
    "sme_coo_to_csr_workspace_size": [i64, i64, i64, psz],
    "sme_coo_to_csr": [C.c_int, i64, i64, i64, p, p, p, p, p, p, p, p, p, sz, i64, p, p, p],
    "sme_permute_csr_row_ptr": [i64, p, p, p, p, sz, p],
    "sme_permute_csr_row_ptr_starts": [i64, p, p, p, p, p, sz, p],
    "sme_permute_csr_workspace_size": [i64, i64, i64, psz],
    "sme_permute_csr": [C.c_int, i64, i64, i64, p, p, p, p, p, p, p, p, p, sz, i64, p, p, p],
    "sme_long_row_nnz": [i64, p, p, p],
    "sme_map_cols_sliced": [i64, i64, p, p, p, i32, p],
    "sme_map_cols_sliced_partial": [i64, i64, p, p, p, i32, i32, p],
    "sme_csr_validate": [i64, i64, i64, p, p, p, p],
    "sme_row_stats": [i64, p, p, p],
    "sme_row_spans": [i64, p, p, i32, p, p],
    "sme_csr_expand_rows": [i64, p, p, p],
    "sme_hist2d_csr": [i64, i64, i64, p, p, i32, i32, p, p],
    "sme_hist2d_coo": [i64, i64, i64, p, p, i32, i32, p, p],
    "sme_hist2d_set_mode": [C.c_int],
    "sme_sort_rows_set_wmed": [C.c_int],
    "sme_sort_rows_set_key32": [C.c_int],
    "sme_sort_rows_set_cta": [C.c_int],
    "sme_hist2d_set_variant": [C.c_int],
    "sme_row_hist_csr": [i64, p, i32, p, p],
    "sme_entropy": [i64, p, f64, p, p, p],
    "sme_spmv_merge_tiles": [i64, i64, pi64],
    "sme_spmv_merge_plan": [i64, i64, p, p, p],
    "sme_spmv_merge_carry_bytes": [C.c_int, i64, psz],
    "sme_spmv_merge": [C.c_int, i64, i64, i64, p, p, p, p, p, p, i64, p, C.c_int, p],
    "sme_spmv_merge_set_mode": [C.c_int],
    "sme_panel_count_workspace_size": [i64, i32, psz],
    "sme_panel_row_ptrs": [i64, p, p, i32, p, p, p, sz, p],
    "sme_panel_scatter": [C.c_int, i64, p, p, p, i32, p, p, p, p, p, p],
    "sme_seg_workspace_size": [i64, i32, psz],
    "sme_seg_positions": [i64, p, p, i32, p, C.c_int, p, p, sz, p],
    "sme_seg_fill": [C.c_int, i64, p, p, p, i32, p, p, p, p, p, p, p, p, p],
    "sme_spmv_seg_warps": [C.POINTER(C.c_int32)],
    "sme_seg_set_scatter_groups": [C.c_int],
    "sme_seg_set_fill_ballot": [C.c_int],
    "sme_seg_set_fill_direct": [C.c_int],
    "sme_set_resident_grids": [C.c_int],
    "sme_spmv_seg_set_mode": [C.c_int],
    "sme_seg_plan": [i64, p, i32, p, p],
    "sme_seg_plan_split": [i64, i32, p, p],
    "sme_spmv_seg_split": [C.c_int, i32, p, p, p, p, p, p, C.c_int, p, p, p],
    "sme_spmv_seg": [C.c_int, i32, p, p, p, p, p, p, C.c_int, p],
    "sme_spmv_seg_epi": [C.c_int, i32, p, p, p, p, p, p, C.c_int, p, p, p, p, p, p, p],
    "sme_spmv_vector_epi_blocks": [i64, C.c_int, pi64],
    "sme_rows_epi_blocks": [i64, pi64],
    "sme_rows_epi": [i64, p, p, p, p, p, p, p, p, C.c_int, p],
    "sme_spmv_vector_epi": [C.c_int, i64, p, p, p, p, p, p, p, p, p, p, C.c_int, p],
    "sme_spmv_seg_epi_cg": [C.c_int, i32, p, p, p, p, p, p, p, C.c_int, p, p, p, p, p],
    "sme_spmv_seg_epi_peers": [C.c_int, i32, p, p, p, p, p, p, C.c_int, p, i64, p, i32, p, p, p, p, p],
    "sme_ipc_malloc": [sz, C.POINTER(C.c_void_p)],
    "sme_ipc_free": [p],
    "sme_ipc_get_handle": [p, p],
    "sme_ipc_open": [p, C.POINTER(C.c_void_p)],
    "sme_ipc_close": [p],
    "sme_spmv_stream_warps": [i64, i64, C.POINTER(C.c_int32)],
    "sme_spmv_stream_set_mode": [C.c_int],
    "sme_spmv_stream_set_row_cost": [C.c_int],
    "sme_spmv_stream_plan": [i64, i64, p, i32, p, p],
    "sme_spmv_stream": [C.c_int, i64, i64, i64, p, p, p, p, p, p, i32, C.c_int, i32, p],
    "sme_spmv_vector": [C.c_int, C.c_int, i64, i64, p, p, p, p, p, C.c_int, p],
    "sme_spmv_reduceat_exact": [i64, p, p, p, p, p, p],
    "sme_hash64": [p, i64, u64, p, p],
    "sme_spmv_coo": [C.c_int, i64, i64, p, p, p, p, p, p],
    "sme_spmv_coo_ordered": [C.c_int, i64, p, p, p, p, p, p, p],
    "sme_maxabs_diff": [C.c_int, i64, p, p, p, p],
    "sme_rowshard_remap_cols": [i64, i64, i32, i64, p, p, p],
    "sme_blas_partials": [pi64],
    "sme_dot": [C.c_int, i64, p, p, p, p, p, C.c_int, p],
    "sme_cg_update": [C.c_int, i64, p, p, p, p, p, p, p],
    "sme_scale": [C.c_int, i64, p, p, p, C.c_int, p],
    "sme_axpby": [C.c_int, i64, f64, p, f64, p, p],
    # sme_synth.h
    "sme_synth_laplacian5": [C.c_int, i64, p, p, p, p],
    "sme_synth_random_rows": [C.c_int, i64, i64, i32, u64, p, p, p, p],
    "sme_synth_random_rows_sel": [C.c_int, i64, p, i64, i32, u64, p, p, p, p],
    "sme_diag_gather": [p, i64, i32, i32, i32, p, p],
    "sme_synth_rmat_edges": [i64, i32, f64, f64, f64, u64, p, p, p],
    "sme_synth_row_values": [C.c_int, i64, p, u64, p, p],
    "sme_coo_to_csr_dedup": [C.c_int, i64, i64, i64, p, p, p, p, p, p, p, sz, i64, p, p],
    "sme_csr_compact_row_ptr": [i64, p, p, i32, p, p, sz, p],
    "sme_csr_compact": [C.c_int, i64, p, p, p, i32, p, p, p, p],
}
# int64 row_ptr twins (nnz >= 2^31 - 1): same argument list as the int32 namesake
WIDE_ENTRY_POINTS = (
    "sme_coo_row_ptr", "sme_coo_to_csr", "sme_permute_csr_row_ptr", "sme_permute_csr_row_ptr_starts",
    "sme_permute_csr", "sme_long_row_nnz",
    "sme_row_stats", "sme_row_spans", "sme_csr_validate", "sme_csr_expand_rows", "sme_hist2d_csr", "sme_row_hist_csr",
    "sme_seg_positions", "sme_seg_fill", "sme_spmv_vector",
)
for _n in WIDE_ENTRY_POINTS:
    SIGNATURES[_n + "_i64"] = SIGNATURES[_n]
_RESTYPES = {"sme_last_error": C.c_char_p}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load libsme.so and declare every exported signature (no CUDA needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH.name} is not built: run `python -m paper_2308_00106_b200._build` "
                    "(the max_E SpMV path has no CPU fallback)"
                )
            lib = C.CDLL(str(LIB_PATH))
            for name, argtypes in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = _RESTYPES.get(name, C.c_int)
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().sme_last_error()
    return msg.decode() if msg else ""


def call(name: str, *args) -> None:
    """Invoke an sme_* entry point; a non-zero status raises (EINVAL -> ValueError)."""
    status = getattr(load(), name)(*args)
    if status == SME_OK:
        return
    msg = f"{name}: {last_error()}"
    if status == SME_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def rp_name(name: str, row_ptr) -> str:
    """The entry point for a CSR whose row_ptr is `row_ptr` (a device tensor): the
    `_i64` twin when row_ptr is int64 (nnz >= 2^31 - 1), else `name` itself."""
    import torch

    return name + "_i64" if row_ptr.dtype == torch.int64 else name


def call_rp(name: str, row_ptr, *args) -> None:
    """call() of the int32 or int64 row_ptr variant of `name`, picked from row_ptr's dtype."""
    call(rp_name(name, row_ptr), *args)


def query_size(name: str, *args) -> int:
    out = C.c_size_t(0)
    call(name, *args, C.byref(out))
    return int(out.value)


def query_i64(name: str, *args) -> int:
    out = C.c_int64(0)
    call(name, *args, C.byref(out))
    return int(out.value)
