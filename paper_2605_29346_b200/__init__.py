"""B200-native sparse GNN hot path (arxiv/paper_2605_29346 + GraphPy).

Drop-in for the reference's graph API (``gsbench.graph``: CsrGraph,
make_csr, csr_from_edges, generate, load_edge_list, save_csr/load_csr,
build_subgraph_csr) plus the GraphPy kernel API (SpMMv/SpMMve with degree-norm,
in-place degree-norm, SDDMM, edge-softmax) and GCN/GIN/GAT layers — all on
hand-written sm_100a kernels in libgnnb200.so, called through a C ABI
(include/gnn_b200.h).  No CPU fallback.
"""

from .errors import CapacityError, ConfigError, ExtensionMissing, ParseError, RangeError
from .graph import (
    OFFSET_DTYPE,
    TARGET_DTYPE,
    CsrGraph,
    GraphGenSpec,
    build_subgraph_csr,
    csr_from_edges,
    generate,
    load_csr,
    load_edge_list,
    make_csr,
    save_csr,
    total_degree,
)
from .ops import colsum, degree_norm_, gemm, linear, spmmv, spmmve
from .torch_ops import register_graph, release_graph  # torch.ops.gnnb200.* (torch.library)

__version__ = "0.1.0"

__all__ = [
    "CapacityError", "ConfigError", "ExtensionMissing", "ParseError", "RangeError",
    "OFFSET_DTYPE", "TARGET_DTYPE", "CsrGraph", "GraphGenSpec", "build_subgraph_csr",
    "csr_from_edges", "generate", "load_csr", "load_edge_list", "make_csr", "save_csr",
    "total_degree", "colsum", "degree_norm_", "gemm", "linear", "spmmv", "spmmve",
    "register_graph", "release_graph",
]
