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
