"""ctypes binding of libbsp.so (the C ABI declared in include/bsp.h).

The library is built in-tree by ``paper_2507_21253_b200.build``.  Loading
fails loudly when it is missing: there is no CPU fallback in the product.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libbsp.so"

BSP_OK = 0
BSP_ERR_CONTRACT = 1
BSP_ERR_OOM = 2
BSP_ERR_CUDA = 3
BSP_ERR_NCCL = 4
BSP_ERR_IO = 5
BSP_ERR_INTERNAL = 6

i32, i64, u64, dbl, u8 = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_uint8
P = C.POINTER
vp = C.c_void_p


class bsp_csr(C.Structure):
    _fields_ = [("nrows", i64), ("ncols", i64), ("nnz", i64), ("row_ptr", vp), ("col_idx", vp),
                ("values", vp), ("owned", i32)]


class bsp_host_csr(C.Structure):
    _fields_ = [("nrows", i64), ("ncols", i64), ("nnz", i64), ("row_ptr", P(i64)),
                ("col_idx", P(i32)), ("values", P(dbl))]


class bsp_csr_cluster(C.Structure):
    _fields_ = [("nclusters", i64), ("nrows", i64), ("ncols", i64), ("ncolslots", i64),
                ("nslots", i64), ("cluster_sizes", vp), ("member_ptr", vp),
                ("cluster_col_ptr", vp), ("col_idx", vp), ("value_ptr", vp), ("values", vp),
                ("valid", vp), ("member_mask", vp), ("row_map", vp), ("csr_row_ptr", vp),
                ("csr_col_idx", vp), ("csr_values", vp), ("owned", i32), ("csr_nnz", i64)]


class bsp_host_csr_cluster(C.Structure):
    _fields_ = [("nclusters", i64), ("nrows", i64), ("ncols", i64), ("ncolslots", i64),
                ("nslots", i64), ("cluster_sizes", P(i32)), ("cluster_col_ptr", P(i64)),
                ("col_idx", P(i32)), ("value_ptr", P(i64)), ("values", P(dbl)),
                ("valid", P(u64)), ("row_map", P(i32))]


class bsp_shard_info(C.Structure):
    _fields_ = [("row_begin", i64), ("row_end", i64), ("products_local", i64),
                ("nnz_local", i64), ("nnz_global", i64), ("multiply_ms", dbl), ("gather_ms", dbl)]


BSP_NCCL_ID_BYTES = 128


class bsp_access_stats(C.Structure):
    _fields_ = [("b_row_loads", u64), ("a_inner_iters", u64), ("placeholder_skips", u64)]


class bsp_candidate(C.Structure):
    _fields_ = [("i", i32), ("j", i32), ("score", dbl)]


class bsp_exec_stats(C.Structure):
    _fields_ = [("products", i64), ("nnz_out", i64), ("units", i64 * 16),
                ("kernels_launched", i32), ("chunks", i32)]


# name -> (restype, argtypes); every symbol of include/bsp.h
SIGNATURES = {
    "bsp_last_error": (C.c_char_p, []),
    "bsp_version": (C.c_char_p, []),
    "bsp_create": (C.c_int, [C.c_int, P(vp)]),
    "bsp_destroy": (C.c_int, [vp]),
    "bsp_set_stream": (C.c_int, [vp, vp]),
    "bsp_get_stream": (vp, [vp]),
    "bsp_profile": (C.c_int, [vp, C.c_int]),
    "bsp_profile_report": (i64, [vp, C.c_char_p, i64]),
    "bsp_synchronize": (C.c_int, [vp]),
    "bsp_kernel_launches": (i64, [vp]),
    "bsp_get_exec_stats": (C.c_int, [vp, P(bsp_exec_stats)]),
    "bsp_csr_upload": (C.c_int, [vp, i64, i64, vp, vp, vp, P(bsp_csr)]),
    "bsp_csr_upload_rp32": (C.c_int, [vp, i64, i64, vp, vp, vp, P(bsp_csr)]),
    "bsp_csr_view": (C.c_int, [i64, i64, i64, vp, vp, vp, P(bsp_csr)]),
    "bsp_csr_download": (C.c_int, [vp, P(bsp_csr), vp, vp, vp]),
    "bsp_csr_download_async": (C.c_int, [vp, P(bsp_csr), vp, vp, vp]),
    "bsp_stream_wait": (C.c_int, [vp, vp]),
    "bsp_csr_free": (C.c_int, [vp, P(bsp_csr)]),
    "bsp_host_alloc": (C.c_int, [C.c_size_t, P(vp)]),
    "bsp_host_free": (C.c_int, [vp]),
    "bsp_spgemm_products": (C.c_int, [vp, P(bsp_csr), P(bsp_csr), vp, P(i64)]),
    "bsp_spgemm_symbolic": (C.c_int, [vp, P(bsp_csr), P(bsp_csr), vp]),
    "bsp_spgemm_rowwise": (C.c_int, [vp, P(bsp_csr), P(bsp_csr), P(bsp_csr)]),
    "bsp_spgemm_rowwise_range": (C.c_int, [vp, P(bsp_csr), P(bsp_csr), i64, i64, P(bsp_csr)]),
    "bsp_spgemm_rowwise_host": (C.c_int, [vp, P(bsp_host_csr), P(bsp_host_csr), P(bsp_host_csr)]),
    "bsp_partition_rows": (C.c_int, [vp, P(bsp_csr), P(bsp_csr), i32, vp]),
    "bsp_csr_cluster_build": (C.c_int, [vp, P(bsp_csr), i64, vp, vp, P(bsp_csr_cluster)]),
    "bsp_csr_cluster_free": (C.c_int, [vp, P(bsp_csr_cluster)]),
    "bsp_csr_cluster_download": (C.c_int, [vp, P(bsp_csr_cluster), P(bsp_host_csr_cluster)]),
    "bsp_host_csr_cluster_free": (None, [P(bsp_host_csr_cluster)]),
    "bsp_spgemm_clusterwise": (C.c_int, [vp, P(bsp_csr_cluster), P(bsp_csr), P(bsp_csr),
                                         P(bsp_csr_cluster)]),
    "bsp_cluster_to_csr": (C.c_int, [vp, P(bsp_csr_cluster), P(bsp_csr)]),
    "bsp_cluster_access_stats": (C.c_int, [vp, P(bsp_csr_cluster), P(bsp_csr),
                                           P(bsp_access_stats)]),
    "bsp_rowwise_access_stats": (C.c_int, [vp, P(bsp_csr), P(bsp_csr), P(bsp_access_stats)]),
    "bsp_transpose": (C.c_int, [vp, P(bsp_csr), P(bsp_csr)]),
    "bsp_generate_frontiers": (C.c_int, [vp, P(bsp_csr), C.c_int64, C.c_int64, C.c_uint64,
                                         P(bsp_csr), P(C.c_int64)]),
    "bsp_spgemm_topk": (C.c_int, [vp, P(bsp_csr), P(bsp_csr), i32, dbl, P(P(bsp_candidate)),
                                  P(i64)]),
    "bsp_minhash_candidates": (C.c_int, [vp, P(bsp_csr), i32, i32, u64, i32, dbl,
                                         P(P(bsp_candidate)), P(i64)]),
    "bsp_hierarchical_clusters": (C.c_int, [vp, P(bsp_host_csr), dbl, i32, i32, i32, i32, u64,
                                            P(i64), P(P(i64)), P(P(i32))]),
    "bsp_merge_candidates": (C.c_int, [P(bsp_host_csr), P(bsp_candidate), i64, dbl, i32, P(i64),
                                       P(P(i64)), P(P(i32)), P(i64), P(P(bsp_candidate))]),
    "bsp_variable_length_clusters": (C.c_int, [P(bsp_host_csr), dbl, i32, P(i64), P(P(i64)),
                                               P(P(i32))]),
    "bsp_fixed_length_clusters": (C.c_int, [i64, i32, P(i64), P(P(i64)), P(P(i32))]),
    "bsp_jaccard": (C.c_int, [P(bsp_host_csr), i64, i64, P(dbl)]),
    "bsp_reorder_random": (C.c_int, [i64, u64, vp]),
    "bsp_reorder_rcm": (C.c_int, [P(bsp_host_csr), vp]),
    "bsp_reorder_degree": (C.c_int, [P(bsp_host_csr), vp]),
    "bsp_bandwidth": (C.c_int, [P(bsp_host_csr), P(i64)]),
    "bsp_permute_symmetric": (C.c_int, [P(bsp_host_csr), vp, P(bsp_host_csr)]),
    "bsp_permute_rows": (C.c_int, [P(bsp_host_csr), vp, P(bsp_host_csr)]),
    "bsp_transpose_host": (C.c_int, [P(bsp_host_csr), P(bsp_host_csr)]),
    "bsp_host_csr_free": (None, [P(bsp_host_csr)]),
    "bsp_host_free_plain": (None, [vp]),
    "bsp_gen_er": (C.c_int, [i64, i32, u64, P(bsp_host_csr)]),
    "bsp_gen_hidden_clusters": (C.c_int, [i64, i32, i32, dbl, dbl, u64, u64, P(bsp_host_csr)]),
    "bsp_gen_rmat": (C.c_int, [i32, i32, dbl, dbl, dbl, u64, P(bsp_host_csr)]),
    "bsp_gen_stencil27": (C.c_int, [i32, i64, P(bsp_host_csr)]),
    "bsp_load_matrix_market": (C.c_int, [C.c_char_p, P(bsp_host_csr)]),
    "bsp_write_matrix_market": (C.c_int, [P(bsp_host_csr), C.c_char_p]),
    "bsp_load_permutation": (C.c_int, [C.c_char_p, i64, vp]),
    "bsp_write_permutation": (C.c_int, [vp, i64, C.c_char_p]),
    "bsp_nccl_unique_id": (C.c_int, [vp]),
    "bsp_comm_init": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "bsp_comm_destroy": (C.c_int, [vp]),
    "bsp_comm_rank": (C.c_int, [vp, P(C.c_int), P(C.c_int)]),
    "bsp_csr_broadcast": (C.c_int, [vp, P(bsp_csr), C.c_int, P(dbl)]),
    "bsp_csr_allgather_rows": (C.c_int, [vp, P(bsp_csr), P(bsp_csr)]),
    "bsp_spgemm_rowwise_sharded": (C.c_int, [vp, P(bsp_csr), P(bsp_csr), C.c_int, P(bsp_csr),
                                             P(bsp_shard_info)]),
    "bsp_partition_clusters": (C.c_int, [vp, P(bsp_csr_cluster), P(bsp_csr), i32, vp]),
    "bsp_csr_select_rows": (C.c_int, [vp, P(bsp_csr), vp, i64, P(bsp_csr)]),
}

_lib = None


def load() -> C.CDLL:
    """Load libbsp.so (building it first when the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() and os.environ.get("BSP_NO_AUTOBUILD") != "1":
        from . import build as _build

        _build.build(verbose=False)
    if not LIB_PATH.exists():
        raise RuntimeError(f"libbsp.so not found at {LIB_PATH}; run python -m "
                           "paper_2507_21253_b200.build (no CPU fallback exists)")
    # BSP_LIB_VARIANT=name loads libbsp_name.so (an A/B build made by tools/build_variant.py
    # with extra -D flags; experiments only)
    variant = os.environ.get("BSP_LIB_VARIANT")
    path = LIB_PATH.with_name(f"libbsp_{variant}.so") if variant else LIB_PATH
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
