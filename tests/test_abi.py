"""CPU: the C-ABI library loads and exports every symbol include/gnn_b200.h
declares; ctypes signatures cover the header; host-side argument logic."""

import ctypes
import io
import os
import re

import pytest

from paper_2605_29346_b200 import _lib
from paper_2605_29346_b200.errors import ConfigError, ParseError, RangeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gnn_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(gnn_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_functions():
    names = declared_functions()
    assert "gnn_spmm" in names and "gnn_csr_from_edges" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    assert set(declared_functions()) == set(_lib.SIGNATURES)


def test_library_loads_without_gpu_and_reports_version():
    lib = _lib.load_library(require_cuda=False)
    assert lib.gnn_abi_version() >= 1
    assert _lib.strerror(_lib.GNN_ERR_RANGE) == "target vertex id out of range"


def test_status_mapping_to_reference_exceptions():
    with pytest.raises(RangeError):
        _lib.check(_lib.GNN_ERR_RANGE)
    with pytest.raises(IndexError):
        _lib.check(_lib.GNN_ERR_INDEX)
    with pytest.raises(ValueError):
        _lib.check(_lib.GNN_ERR_CSR_INVARIANT)
    with pytest.raises(ValueError):
        _lib.check(_lib.GNN_ERR_SOURCE_RANGE)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.GNN_ERR_WORKSPACE)
    _lib.check(_lib.GNN_OK)


def test_struct_layouts_match_header():
    # 8 x 8-byte fields
    assert ctypes.sizeof(_lib.CsrView) == 80  # 8 x 8 + col_bits + reserved + row_ids
    # uint32 + float + 6 pointer/int64 fields
    assert ctypes.sizeof(_lib.Epilogue) == 8 + 6 * 8
    assert ctypes.sizeof(_lib.SpmmPlan) == 16 * 8  # + dev_counts, row_limit
    assert ctypes.sizeof(_lib.EdgeScores) == 4 * 8


def test_graphgenspec_validation_mirrors_reference():
    from paper_2605_29346_b200 import GraphGenSpec

    # test_graph.py:105-113
    with pytest.raises(ConfigError):
        GraphGenSpec("power-law", 100, 1000)
    with pytest.raises(ConfigError):
        GraphGenSpec("power-law", 100, 1000, exponent=1.0)
    with pytest.raises(ConfigError):
        GraphGenSpec("blob", 100)
    with pytest.raises(ConfigError):
        GraphGenSpec("ring", 0)
    assert GraphGenSpec("uniform-random", 100, 0.02).edge_count() == 200


def test_edge_list_parse_errors_before_any_device_work():
    from paper_2605_29346_b200 import load_edge_list

    # test_graph.py:24-33, 41-48 — raised while parsing, no GPU needed
    with pytest.raises(ParseError) as e:
        load_edge_list(io.StringIO("0 x\n"))
    assert e.value.line == 1
    with pytest.raises(ParseError) as e:
        load_edge_list(io.StringIO("# comment\n0 1\n\n1 2 3\n"))
    assert e.value.line == 4
    with pytest.raises(RangeError):
        load_edge_list(io.StringIO("n=2\n0 5\n"))
    with pytest.raises(RangeError):
        load_edge_list(io.StringIO(f"0 {2**31}\n"))
