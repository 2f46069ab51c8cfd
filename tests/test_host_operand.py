"""CPU: host-side layout transforms of SparseOperand that are pure tensor
logic — the degree-sorted form (``by_degree``: rows longest-first, row_ids
back to output rows) must hold every row's entries unchanged and in order,
including empty rows, a mega row and slab-boundary splits of the gather."""

import numpy as np
import pytest
import torch

import paper_2605_29346_b200.graph as G


@pytest.mark.parametrize("slab", [37, 1 << 24])
def test_by_degree_keeps_rows(monkeypatch, slab):
    monkeypatch.setenv("GNN_SORT_SLAB", str(slab))
    rng = np.random.default_rng(0)
    R = 1000
    deg = rng.integers(0, 50, R)
    deg[rng.integers(0, R, 100)] = 0
    deg[5] = 5000
    deg[-1] = 0
    off = torch.from_numpy(np.concatenate([[0], np.cumsum(deg)])).long()
    nnz = int(off[-1])
    cols = torch.from_numpy(rng.integers(0, R, nnz)).int()
    vals = torch.rand(nnz)
    op = G.SparseOperand(R, R, off, cols, vals=vals)
    so = op.by_degree()
    assert so.by_degree() is so and op.by_degree() is so  # cached, idempotent
    rid = so.row_ids.long()
    assert sorted(rid.tolist()) == list(range(R))
    sdeg = so.offsets[1:] - so.offsets[:-1]
    assert bool((sdeg[:-1] >= sdeg[1:]).all())  # longest first
    assert torch.equal(sdeg, torch.from_numpy(deg)[rid])
    assert torch.equal(so.deg_offsets, off)  # NORM keeps output-row degrees
    for i in range(R):
        r = int(rid[i])
        a, b = int(so.offsets[i]), int(so.offsets[i + 1])
        assert torch.equal(so.cols[a:b], cols[off[r]:off[r + 1]])
        assert torch.equal(so.vals[a:b], vals[off[r]:off[r + 1]])


def test_spmm_operand_selection(monkeypatch):
    """Which form gnn_spmm runs on: the degree-sorted copy only for topology /
    multiplicity weights, K <= 64 in float4 lanes, operands above the size
    threshold; a released operand always resolves to its sorted form."""
    monkeypatch.setattr(G, "SPMM_SORT_MIN_NNZ", 100)
    rng = np.random.default_rng(1)
    R = 300
    deg = rng.integers(0, 9, R)
    off = torch.from_numpy(np.concatenate([[0], np.cumsum(deg)])).long()
    nnz = int(off[-1])
    cols = torch.from_numpy(rng.integers(0, R, nnz)).int()
    plain = G.SparseOperand(R, R, off, cols)
    X16, Y16 = torch.zeros(R, 16), torch.zeros(R, 16)
    assert G.spmm_operand(plain, X16, Y16).row_ids is not None
    assert G.spmm_operand(plain, torch.zeros(R, 128), torch.zeros(R, 128)) is plain  # K > 64
    assert G.spmm_operand(plain, torch.zeros(R, 6), torch.zeros(R, 6)) is plain      # K % 4
    assert G.spmm_operand(plain, X16, Y16, heads=2) is plain
    assert G.spmm_operand(plain, X16, Y16, vals=torch.ones(nnz)) is plain           # edge values
    weighted = G.SparseOperand(R, R, off, cols, vals=torch.rand(nnz))
    assert G.spmm_operand(weighted, X16, Y16) is weighted  # general values: CSR edge order
    monkeypatch.setattr(G, "SPMM_SORT_MIN_NNZ", nnz + 1)
    assert G.spmm_operand(plain, X16, Y16) is plain  # small operand: row order
    plain.release_row_order()
    assert G.spmm_operand(plain, X16, Y16) is plain.by_degree()
    with pytest.raises(RuntimeError):
        plain.view()
