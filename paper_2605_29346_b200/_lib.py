"""ctypes binding of the C ABI in include/gnn_b200.h.

This is the exact binding a maintainer of the reference would add on their
side: plain pointers, sizes and a stream handle.  The
library is loaded from the package directory (built in-tree by
``__graft_entry__.build()`` / ``make -C paper_2605_29346_b200/csrc``); if it is
missing, or there is no CUDA device, every op raises ``ExtensionMissing`` —
there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

from .errors import ExtensionMissing, RangeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgnnb200.so")
# experiment builds (tools/): GNN_LIB_PATH selects another in-tree build of the library
LIB_PATH = os.environ.get("GNN_LIB_PATH", LIB_PATH)

GNN_OK = 0
GNN_ERR_INVALID_ARGUMENT = 1
GNN_ERR_CSR_INVARIANT = 2
GNN_ERR_RANGE = 3
GNN_ERR_INDEX = 4
GNN_ERR_WORKSPACE = 5
GNN_ERR_CUDA = 6
GNN_ERR_UNSUPPORTED = 7
GNN_ERR_SOURCE_RANGE = 8

EPI_NORM = 1 << 0
EPI_SELF = 1 << 1
EPI_BIAS = 1 << 2
EPI_RELU = 1 << 3
EPI_MASK = 1 << 4
EPI_POSTNORM = 1 << 5

c_i64 = C.c_int64
c_u64 = C.c_uint64
c_ptr = C.c_void_p
c_sz = C.c_size_t
c_int = C.c_int


class CsrView(C.Structure):
    _fields_ = [
        ("num_rows", c_i64),
        ("num_cols", c_i64),
        ("nnz", c_i64),
        ("offsets", c_ptr),
        ("cols", c_ptr),
        ("vals", c_ptr),
        ("eid", c_ptr),
        ("deg_offsets", c_ptr),
        ("col_bits", C.c_int32),
        ("reserved_", C.c_int32),
        ("row_ids", c_ptr),
    ]


class Epilogue(C.Structure):
    _fields_ = [
        ("flags", C.c_uint32),
        ("self_scale", C.c_float),
        ("self_x", c_ptr),
        ("ld_self", c_i64),
        ("bias", c_ptr),
        ("mask", c_ptr),
        ("ld_mask", c_i64),
        ("post_deg_offsets", c_ptr),
    ]


class EdgeScores(C.Structure):
    _fields_ = [("s", c_ptr), ("el", c_ptr), ("er", c_ptr), ("slope", C.c_float)]


class SpmmPlan(C.Structure):
    _fields_ = [
        ("edges_per_warp", c_i64),
        ("num_warps", c_i64),
        ("chunk_row", c_ptr),
        ("chunk_split", c_ptr),
        ("num_split", c_i64),
        ("split_rows", c_ptr),
        ("split_group_base", c_ptr),
        ("num_groups", c_i64),
        ("num_empty", c_i64),
        ("empty_rows", c_ptr),
        ("short_max", c_i64),
        ("num_short", c_i64),
        ("short_rows", c_ptr),
        ("main_nnz", c_i64),
        ("dev_counts", c_ptr),
        ("row_limit", c_ptr),
    ]


# name -> (restype, argtypes).  Keep in sync with include/gnn_b200.h; the CPU
# test suite checks that every declared symbol is exported.
SIGNATURES = {
    "gnn_abi_version": (c_int, []),
    "gnn_l2_max_window": (c_i64, []),
    "gnn_l2_persist_limit": (c_int, [c_i64]),
    "gnn_l2_window": (c_int, [c_ptr, c_ptr, c_i64, C.c_float]),
    "gnn_build_id": (C.c_char_p, []),
    "gnn_strerror": (C.c_char_p, [c_int]),
    "gnn_last_cuda_error": (c_int, []),
    "gnn_device_sm_count": (c_int, []),
    "gnn_launch_counter": (c_i64, []),
    "gnn_read_probe": (c_int, [c_ptr, c_i64, c_int, c_ptr, c_ptr]),
    "gnn_memcpy2d": (c_int, [c_ptr, c_sz, c_ptr, c_sz, c_sz, c_sz, c_ptr]),
    "gnn_csr_from_edges_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_csr_from_edges": (c_int, [c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_subgraph_csr_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_subgraph_csr": (c_int, [c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_csr_validate_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_csr_validate": (c_int, [c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_degrees": (c_int, [c_i64, c_ptr, c_ptr, c_ptr]),
    "gnn_csc_from_csr_workspace": (c_sz, [c_i64, c_i64, c_i64]),
    "gnn_csc_from_csr": (
        c_int,
        [c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_csr_coalesce_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_csr_coalesce": (
        c_int,
        [c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, C.POINTER(c_i64), c_ptr, c_sz, c_ptr],
    ),
    "gnn_csr_pack_weights_workspace": (c_sz, []),
    "gnn_csr_pack_weights": (c_int, [c_i64, c_ptr, c_ptr, C.c_int32, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_generate_powerlaw_workspace": (c_sz, [c_i64]),
    "gnn_generate_powerlaw": (
        c_int,
        [c_i64, c_i64, c_ptr, c_u64, c_u64, c_u64, c_u64, c_ptr, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_powerlaw_block_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_powerlaw_block": (
        c_int,
        [c_i64, c_i64, c_ptr, c_u64, c_u64, c_u64, c_u64, c_i64, c_i64, c_i64, c_i64, c_ptr,
         c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_fill_uniform": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_u64, c_ptr]),
    "gnn_fill_labels": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_u64, c_ptr]),
    "gnn_append_dev": (c_int, [c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
    "gnn_fill_tail_dev": (c_int, [c_ptr, c_i64, c_ptr, c_i64, c_i64, c_ptr]),
    "gnn_sort_pairs_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_sort_pairs": (c_int, [c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_offsets_from_keys_workspace": (c_sz, [c_i64]),
    "gnn_offsets_from_keys": (c_int, [c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_sample_hop_workspace": (c_sz, [c_i64]),
    "gnn_sample_hop": (
        c_int,
        [c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_u64, c_u64, c_u64, c_u64, c_ptr, c_ptr,
         c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_dedup_relabel_workspace": (c_sz, [c_i64]),
    "gnn_dedup_relabel": (
        c_int,
        [c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
         c_ptr, c_sz, c_ptr],
    ),
    "gnn_sample_hop_dev_workspace": (c_sz, [c_i64]),
    "gnn_sample_hop_dev": (
        c_int,
        [c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_sz,
         c_ptr],
    ),
    "gnn_dedup_relabel_dev_workspace": (c_sz, [c_i64]),
    "gnn_dedup_relabel_dev": (
        c_int,
        [c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
         c_ptr, c_sz, c_ptr],
    ),
    "gnn_table_lookup_dev": (c_int, [c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_ptr]),
    "gnn_table_fill_dev": (c_int, [c_ptr, c_ptr, c_ptr, c_i64, C.c_int32, c_ptr]),
    "gnn_gather_rows": (c_int, [c_ptr, c_i64, c_ptr, c_i64, c_i64, c_ptr, c_i64, c_ptr]),
    "gnn_gather_rows_dev": (c_int, [c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_i64, c_ptr]),
    "gnn_table_lookup": (c_int, [c_ptr, c_ptr, c_i64, c_ptr, c_ptr]),
    "gnn_table_assign": (c_int, [c_ptr, c_ptr, c_i64, c_i64, c_ptr]),
    "gnn_spmm_plan_buffer_ints": (c_sz, [c_i64, c_i64, c_i64]),
    "gnn_spmm_plan_workspace": (c_sz, [c_i64]),
    "gnn_spmm_plan_build": (
        c_int,
        [C.POINTER(CsrView), c_i64, c_ptr, C.POINTER(SpmmPlan), c_ptr, c_sz, c_ptr],
    ),
    "gnn_spmm_plan_build_ex": (
        c_int,
        [C.POINTER(CsrView), c_i64, c_i64, c_ptr, C.POINTER(SpmmPlan), c_ptr, c_sz, c_ptr],
    ),
    "gnn_spmm_plan_build_dev": (
        c_int,
        [C.POINTER(CsrView), c_i64, c_i64, c_ptr, C.POINTER(SpmmPlan), c_ptr, c_ptr, c_ptr, c_sz,
         c_ptr],
    ),
    "gnn_spmm_workspace": (c_sz, [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64]),
    "gnn_spmm": (
        c_int,
        [
            C.POINTER(CsrView),
            C.POINTER(SpmmPlan),
            c_i64,
            c_ptr,
            c_i64,
            c_ptr,
            c_i64,
            c_i64,
            C.POINTER(Epilogue),
            c_ptr,
            c_sz,
            c_ptr,
        ],
    ),
    "gnn_spmm_shared_heads": (c_int, [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_ptr, c_i64,
                                      c_i64, c_ptr, c_i64, C.c_float, C.POINTER(Epilogue), c_ptr,
                                      c_sz, c_ptr]),
    "gnn_spmm_peer": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_i64,
         C.POINTER(Epilogue), c_ptr, c_sz, c_ptr],
    ),
    "gnn_degree_norm_inplace": (c_int, [c_i64, c_ptr, c_ptr, c_i64, c_i64, c_ptr]),
    "gnn_sddmm": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64, c_ptr, c_i64, c_ptr, c_i64, c_i64, c_ptr,
         c_ptr],
    ),
    "gnn_edge_softmax_workspace": (c_sz, [C.POINTER(SpmmPlan), c_i64]),
    "gnn_edge_softmax_fwd": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64, C.POINTER(EdgeScores), c_ptr, c_ptr,
         c_sz, c_ptr],
    ),
    "gnn_edge_softmax_bwd": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64, c_ptr, c_ptr, C.POINTER(EdgeScores),
         c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_segment_sum": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64, c_ptr, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_gat_bwd_csc_workspace": (c_sz, [C.POINTER(SpmmPlan), c_i64]),
    "gnn_gat_bwd_csc": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_i64,
         c_ptr, c_i64, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_gat_bwd_csc_mean": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64, c_ptr, c_ptr, c_i64, C.c_float, c_ptr,
         c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_gat_softmax_fwd_stats": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64, C.POINTER(EdgeScores), c_ptr, c_ptr,
         c_ptr, c_sz, c_ptr],
    ),
    "gnn_gat_rowstat": (c_int, [c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr,
                                c_ptr, c_i64, c_ptr]),
    "gnn_gat_rowstat_mean": (c_int, [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_ptr,
                                     c_i64, C.c_float, c_ptr, c_ptr, c_ptr, c_i64, c_ptr]),
    "gnn_gat_rowstat_mean_tc_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_gat_rowstat_mean_tc": (c_int, [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_ptr,
                                        c_i64, C.c_float, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_sz,
                                        c_ptr]),
    "gnn_gemm_gat_proj": (c_int, [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_i64,
                                  c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_gemm_gat_relu_stat": (c_int, [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_ptr,
                                       c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_sz,
                                       c_ptr]),
    "gnn_gat_bwd_rc_workspace": (c_sz, [C.POINTER(SpmmPlan), c_i64]),
    "gnn_gat_bwd_rc": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64, c_ptr, C.c_float, c_ptr, c_i64, c_ptr,
         c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_gat_bwd_rc_mean": (
        c_int,
        [C.POINTER(CsrView), C.POINTER(SpmmPlan), c_i64, C.c_float, c_ptr, C.c_float, c_ptr, c_i64,
         c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_invert_permutation": (c_int, [c_i64, c_ptr, c_ptr, c_ptr]),
    "gnn_gat_attn_proj": (
        c_int, [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "gnn_gat_attn_proj_bwd_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_gat_attn_proj_bwd": (
        c_int,
        [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_ptr,
         c_ptr, c_sz, c_ptr],
    ),
    "gnn_head_mean": (c_int, [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr]),
    "gnn_head_mean_bwd": (c_int, [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_ptr]),
    "gnn_gemm_workspace": (c_sz, [c_i64, c_i64, c_i64, c_int]),
    "gnn_gemm_rows_dev": (c_int, [c_i64, c_i64, c_i64, c_ptr, c_i64, c_int, c_ptr, c_i64, c_int,
                                  c_ptr, c_i64, c_ptr, c_int, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_gemm": (
        c_int,
        [c_i64, c_i64, c_i64, c_ptr, c_i64, c_int, c_ptr, c_i64, c_int, c_ptr, c_i64, c_ptr,
         c_int, c_ptr, c_sz, c_ptr],
    ),
    "gnn_colsum_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_colsum": (c_int, [c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_mask_norm_colsum_workspace": (c_sz, [c_i64, c_i64]),
    "gnn_mask_norm_colsum_dev": (c_int, [c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr,
                                         c_i64, c_ptr, c_ptr, c_ptr, c_sz, c_ptr]),
    "gnn_mask_norm_colsum": (
        c_int,
        [c_i64, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_softmax_xent_workspace": (c_sz, [c_i64]),
    "gnn_softmax_xent": (
        c_int,
        [c_i64, c_i64, c_ptr, c_i64, c_ptr, C.c_float, c_ptr, c_i64, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_gcn_head_workspace": (c_sz, [c_i64, c_i64, c_i64]),
    "gnn_gcn_head": (
        c_int,
        [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr,
         c_ptr, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_gcn_head_scaled": (
        c_int,
        [c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, C.c_float, c_ptr, c_i64,
         c_ptr, c_ptr, c_ptr, c_ptr, c_sz, c_ptr],
    ),
    "gnn_remap_ids": (c_int, [c_i64, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr]),
    "gnn_adam_step": (
        c_int,
        [c_int, c_ptr, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float, c_ptr, c_ptr],
    ),
}

_lock = threading.Lock()
_lib = None


def load_library(require_cuda: bool = True):
    """Load libgnnb200.so and bind its signatures (cached)."""
    global _lib
    if require_cuda and not torch.cuda.is_available():
        raise ExtensionMissing("no CUDA device: the sparse GNN path has no CPU fallback")
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ExtensionMissing(
                    f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _check_provenance(lib)
            _lib = lib
    return _lib


def build_id() -> str:
    """The loaded library's embedded provenance string (gnn_build_id)."""
    return load_library(False).gnn_build_id().decode()


def _check_provenance(lib) -> None:
    """Refuse a library not built from the sources next to it: the embedded
    source hash must equal buildinfo.source_hash() of the shipped csrc/ and
    include/ (GNN_ALLOW_STALE=1 skips the check, for debugging only)."""
    from . import buildinfo

    bid = lib.gnn_build_id().decode()
    want = buildinfo.source_hash()
    if f"src:{want} " not in bid + " " and os.environ.get("GNN_ALLOW_STALE") != "1":
        raise ExtensionMissing(
            f"{LIB_PATH} is stale: built from sources {bid!r}, the tree has src:{want}; "
            "rebuild with __graft_entry__.build()")


def lib():
    return load_library(True)


def strerror(status: int) -> str:
    return load_library(False).gnn_strerror(status).decode()


def check(status: int, what: str = "") -> None:
    """Map a gnn_status to the reference's exception taxonomy."""
    if status == GNN_OK:
        return
    msg = f"{what}: {strerror(status)}" if what else strerror(status)
    if status == GNN_ERR_RANGE:
        raise RangeError("target vertex id out of range")
    if status == GNN_ERR_INDEX:
        raise IndexError("edge source local id out of range")
    if status == GNN_ERR_CSR_INVARIANT:
        raise ValueError("offsets must start at 0, end at num_edges and be nondecreasing")
    if status == GNN_ERR_SOURCE_RANGE:
        raise ValueError("source vertex id outside [0, num_vertices)")
    if status in (GNN_ERR_INVALID_ARGUMENT, GNN_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if status == GNN_ERR_CUDA:
        raise RuntimeError(f"{msg} (cudaError {load_library(False).gnn_last_cuda_error()})")
    raise RuntimeError(msg)


def ptr(t) -> int | None:
    """Raw device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def workspace(nbytes: int, device) -> torch.Tensor:
    """Scratch from torch's caching allocator, so peak-memory accounting sees it."""
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def copy_rows(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst[:] = src for 2-D fp32/int tensors with unit column stride and
    possibly different row strides (host or device src), as one strided copy
    (gnn_memcpy2d) — no transient contiguous device buffer."""
    if dst.shape != src.shape or dst.dtype != src.dtype:
        raise ValueError("copy_rows: shape/dtype mismatch")
    if src.dim() != 2 or dst.stride(1) != 1 or src.stride(1) != 1:
        dst.copy_(src)
        return
    es = dst.element_size()
    check(load_library(False).gnn_memcpy2d(dst.data_ptr(), dst.stride(0) * es, src.data_ptr(),
                                           src.stride(0) * es, dst.shape[1] * es, dst.shape[0],
                                           stream_handle(dst.device)), "memcpy2d")
