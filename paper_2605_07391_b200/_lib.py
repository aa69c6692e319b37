"""ctypes loader for libmerbit_b200.so (the C ABI in include/merbit_b200.h).

There is no fallback: if the in-tree shared library is missing or fails to
load, importing the package's compute API raises.  Build it with
``python -c "import __graft_entry__; __graft_entry__.build()"`` or
``make -C paper_2605_07391_b200/csrc``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MBX_LIB_PATH: load an alternative build (kernel experiments only)
LIB_PATH = os.environ.get("MBX_LIB_PATH") or os.path.join(_HERE, "libmerbit_b200.so")


class mbx_simt_config(C.Structure):
    _fields_ = [("omega", C.c_int32), ("sigma", C.c_int32), ("block_size", C.c_int32),
                ("offset_bits", C.c_int32)]


class mbx_tile_info(C.Structure):
    _fields_ = [("omega", C.c_int32), ("sigma", C.c_int32), ("n_rows", C.c_int64),
                ("nnz", C.c_int64), ("tile_num", C.c_int64), ("lane_num", C.c_int64),
                ("preprocess_seconds", C.c_double)]


class mbx_spmv_trace(C.Structure):
    _fields_ = [("fast_tiles", C.c_int64), ("normal_tiles", C.c_int64),
                ("skipped_tiles", C.c_int64)]


class mbx_pagerank_config(C.Structure):
    _fields_ = [("damping", C.c_double), ("err_tol", C.c_double), ("max_iters", C.c_int64),
                ("reference_iters", C.c_int64)]


class mbx_pagerank_result(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("final_err", C.c_double), ("status", C.c_int32),
                ("preprocess_seconds", C.c_double), ("iterate_seconds", C.c_double),
                ("l1_residual", C.c_double), ("mass", C.c_double),
                ("dangling_mass", C.c_double)]


PAGERANK_OBSERVER = C.CFUNCTYPE(C.c_int, C.c_int64, C.c_void_p, C.c_double, C.c_void_p)


class mbx_degree_stats(C.Structure):
    _fields_ = [("mean_degree", C.c_double), ("low_degree", C.c_int32), ("pad_", C.c_int32),
                ("max_degree", C.c_int64), ("empty_rows", C.c_int64)]


class mbx_bicgstab_config(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int64)]


class mbx_bicgstab_result(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("final_residual", C.c_double),
                ("status", C.c_int32), ("breakdown_reason", C.c_char * 32),
                ("preprocess_seconds", C.c_double), ("iterate_seconds", C.c_double)]


class mbx_coo(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("rows", C.POINTER(C.c_int64)), ("cols", C.POINTER(C.c_int64)),
                ("vals", C.POINTER(C.c_double))]


VP = C.c_void_p
I64P = C.POINTER(C.c_int64)
SIGNATURES = {
    "mbx_last_error": ([], C.c_char_p),
    "mbx_build_info": ([], C.c_char_p),
    "mbx_config_make": ([C.c_int, C.c_int, C.c_int, C.POINTER(mbx_simt_config)], C.c_int),
    "mbx_select_sigma": ([C.c_int, C.c_int], C.c_int),
    "mbx_tile_counts": ([C.c_int64, C.c_int64, C.POINTER(mbx_simt_config), I64P, I64P], C.c_int),
    "mbx_metadata_footprint": ([C.c_int64, C.c_int64, C.POINTER(mbx_simt_config), C.c_double],
                               C.c_double),
    "mbx_merge_search": ([VP, C.c_int64, C.c_int64, C.c_int64, I64P, I64P], C.c_int),
    "mbx_context_release_cache": ([VP], C.c_int),
    "mbx_matrix_degree_stats": ([VP, VP, C.c_int, C.POINTER(mbx_degree_stats)], C.c_int),
    "mbx_pagerank_observed": ([VP, VP, VP, VP, VP, VP, VP, VP, VP, PAGERANK_OBSERVER, VP,
                               C.POINTER(mbx_pagerank_result)], C.c_int),
    "mbx_plan_row_shards": ([VP, C.c_int64, C.c_int64, C.c_int, VP], C.c_int),
    "mbx_plan_row_shards_weighted": ([VP, C.c_int64, C.c_int64, C.c_int, C.c_double, VP], C.c_int),
    "mbx_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "mbx_context_create": ([C.c_int, C.POINTER(VP)], C.c_int),
    "mbx_context_destroy": ([VP], C.c_int),
    "mbx_context_set_stream": ([VP, VP], C.c_int),
    "mbx_context_stream": ([VP], VP),
    "mbx_context_synchronize": ([VP], C.c_int),
    "mbx_context_launch_count": ([VP], C.c_int64),
    "mbx_context_set_tuning": ([VP, C.c_int, C.c_int, C.c_int], C.c_int),
    "mbx_context_set_tuning_ex": ([VP, C.c_int, C.c_int], C.c_int),
    "mbx_context_set_layout": ([VP, C.c_int], C.c_int),
    "mbx_free": ([VP], None),
    "mbx_spmv_baseline_device": ([VP, VP, C.c_int, C.c_int, VP, VP], C.c_int),
    "mbx_bench_spmv": ([VP, VP, VP, C.POINTER(mbx_simt_config), C.c_int, C.c_int, C.c_int, VP,
                        C.POINTER(C.c_double)], C.c_int),
    "mbx_matrix_build_transition": ([VP, VP, C.POINTER(VP)], C.c_int),
    "mbx_matrix_relabel_by_degree": ([VP, VP, C.POINTER(VP), VP], C.c_int),
    "mbx_coo_free": ([C.POINTER(mbx_coo)], None),
    "mbx_mm_read": ([C.c_char_p, C.POINTER(mbx_coo)], C.c_int),
    "mbx_mm_parse": ([C.c_char_p, C.c_int64, C.c_char_p, C.POINTER(mbx_coo)], C.c_int),
    "mbx_mm_write": ([C.c_char_p, C.POINTER(mbx_coo)], C.c_int),
    "mbx_matrix_cache_write": ([C.c_char_p, C.POINTER(mbx_coo)], C.c_int),
    "mbx_matrix_cache_read": ([C.c_char_p, C.POINTER(mbx_coo)], C.c_int),
    "mbx_matrix_load_any": ([C.c_char_p, C.POINTER(mbx_coo)], C.c_int),
    "mbx_matrix_from_coo": ([VP, C.c_int, C.POINTER(mbx_coo), C.POINTER(VP)], C.c_int),
    "mbx_tile_cache_write_host": ([C.c_char_p, C.POINTER(mbx_tile_info),
                                   C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                   C.POINTER(C.c_uint32), C.c_int], C.c_int),
    "mbx_tile_cache_read_host": ([C.c_char_p, C.POINTER(mbx_tile_info),
                                  C.POINTER(C.POINTER(C.c_uint32)),
                                  C.POINTER(C.POINTER(C.c_uint32)),
                                  C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_int)], C.c_int),
    "mbx_tile_cache_write": ([VP, C.c_char_p, C.c_int], C.c_int),
    "mbx_tile_cache_load": ([VP, C.c_char_p, C.POINTER(VP), C.POINTER(C.c_int)], C.c_int),
    "mbx_bicgstab": ([VP, VP, VP, C.POINTER(mbx_simt_config), C.POINTER(mbx_bicgstab_config),
                      VP, VP, C.POINTER(C.c_double), C.POINTER(mbx_bicgstab_result)], C.c_int),
    "mbx_matrix_slot_info": ([VP, C.POINTER(C.c_int64), C.POINTER(C.c_double)], C.c_int),
    "mbx_matrix_build_xcache": ([VP, VP, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "mbx_matrix_xcache_info": ([VP, C.POINTER(C.c_int), C.POINTER(C.c_double)], C.c_int),
    "mbx_matrix_xcache_ptrs": ([VP, C.POINTER(VP), C.POINTER(VP)], C.c_int),
    "mbx_matrix_hub_columns": ([VP, VP], C.c_int),
    "mbx_matrix_gather_profile": ([VP, C.POINTER(C.c_double)], C.c_int),
    "mbx_matrix_upload": ([VP, C.c_int, C.c_int64, C.c_int64, VP, VP, VP, C.POINTER(VP)], C.c_int),
    "mbx_matrix_upload_i32": ([VP, C.c_int, C.c_int64, C.c_int64, VP, VP, VP, C.POINTER(VP)],
                              C.c_int),
    "mbx_matrix_generate_rmat": ([VP, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                  C.c_double, C.c_double, C.POINTER(VP)], C.c_int),
    "mbx_matrix_generate_stencil27": ([VP, C.c_int, C.c_int64, C.POINTER(VP)], C.c_int),
    "mbx_matrix_generate_powerlaw": ([VP, C.c_int, C.c_int, C.c_uint64, C.POINTER(VP)], C.c_int),
    "mbx_matrix_info": ([VP, C.POINTER(C.c_int), I64P, I64P, I64P], C.c_int),
    "mbx_matrix_download": ([VP, VP, VP, VP], C.c_int),
    "mbx_matrix_device_ptrs": ([VP, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP)], C.c_int),
    "mbx_matrix_destroy": ([VP], C.c_int),
    "mbx_matrix_release_caches": ([VP], C.c_int),
    "mbx_matrix_compact": ([VP, VP], C.c_int),
    "mbx_spmv_deposits": ([VP, VP, VP, C.POINTER(mbx_simt_config), VP, VP, VP, C.c_int64,
                           C.POINTER(C.c_int64)], C.c_int),
    "mbx_matrix_resident_bytes": ([VP, C.POINTER(C.c_int64)], C.c_int),
    "mbx_generate_tile": ([VP, VP, C.c_int64, C.c_int64, C.POINTER(mbx_simt_config),
                           C.POINTER(VP)], C.c_int),
    "mbx_matrix_generate_tile": ([VP, VP, C.POINTER(mbx_simt_config), C.POINTER(VP)], C.c_int),
    "mbx_tile_get_info": ([VP, C.POINTER(mbx_tile_info)], C.c_int),
    "mbx_tile_download": ([VP, VP, VP, VP], C.c_int),
    "mbx_tile_upload": ([VP, C.POINTER(mbx_tile_info), VP, VP, VP, C.POINTER(VP)], C.c_int),
    "mbx_tile_destroy": ([VP], C.c_int),
    "mbx_spmv": ([VP, VP, VP, C.POINTER(mbx_simt_config), VP, VP, C.POINTER(mbx_spmv_trace)],
                 C.c_int),
    "mbx_spmv_device": ([VP, VP, VP, C.POINTER(mbx_simt_config), VP, VP], C.c_int),
    "mbx_spmv_trace_counts": ([VP, VP, C.POINTER(mbx_spmv_trace)], C.c_int),
    "mbx_spmv_csr_device": ([VP, VP, VP, VP], C.c_int),
    "mbx_pagerank": ([VP, VP, VP, C.POINTER(mbx_simt_config), C.POINTER(mbx_pagerank_config), VP,
                      VP, VP, VP, C.POINTER(mbx_pagerank_result)], C.c_int),
    "mbx_pagerank_plan_create": ([VP, VP, VP, C.POINTER(mbx_simt_config),
                                  C.POINTER(mbx_pagerank_config), C.POINTER(VP)], C.c_int),
    "mbx_pagerank_plan_run": ([VP, VP], C.c_int),
    "mbx_pagerank_plan_result": ([VP, C.POINTER(mbx_pagerank_result), VP], C.c_int),
    "mbx_pagerank_plan_pi": ([VP], VP),
    "mbx_pagerank_plan_reference_pi": ([VP], VP),
    "mbx_pagerank_plan_destroy": ([VP], C.c_int),
    "mbx_nccl_unique_id": ([VP], C.c_int),
    "mbx_matrix_row_slice": ([VP, VP, C.c_int64, C.c_int64, C.POINTER(VP)], C.c_int),
    "mbx_shard_group_create": ([VP, C.c_int64, C.c_int, VP, C.c_int, C.c_int, VP, VP,
                                C.POINTER(mbx_simt_config), C.POINTER(mbx_pagerank_config), VP,
                                C.POINTER(VP)], C.c_int),
    "mbx_shard_group_create_peer": ([VP, C.c_int64, C.c_int, VP, C.c_int, VP, VP, VP, VP, VP],
                                    C.c_int),
    "mbx_shard_group_export": ([VP, VP], C.c_int),
    "mbx_shard_group_connect": ([VP, VP], C.c_int),
    "mbx_shard_group_quiesce": ([VP], C.c_int),
    "mbx_shard_group_run": ([VP, VP], C.c_int),
    "mbx_shard_group_result": ([VP, C.POINTER(mbx_pagerank_result), VP], C.c_int),
    "mbx_shard_group_gather_pi": ([VP, VP], C.c_int),
    "mbx_shard_group_download_local": ([VP, VP], C.c_int),
    "mbx_shard_group_destroy": ([VP], C.c_int),
}

_lib = None


def lib():
    """The loaded library.  Raises (never falls back) when it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not built: run __graft_entry__.build() "
                "(make -C paper_2605_07391_b200/csrc); there is no CPU fallback")
        try:
            # let PyTorch load its CUDA runtime pieces (and its NCCL) first;
            # the library resolves NCCL lazily and reuses an already-loaded one
            import torch  # noqa: F401
        except ImportError:
            pass
        L = C.CDLL(LIB_PATH)
        # an A/B build of an older revision (MBX_LIB_PATH) may lack newer
        # entry points: bind what it has; the in-tree library must have all
        ab_build = bool(os.environ.get("MBX_LIB_PATH"))
        for name, (args, res) in SIGNATURES.items():
            if ab_build and not hasattr(L, name):
                continue
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def exported_symbols():
    return sorted(SIGNATURES)
