"""GPU parity: SpMMv / SpMMve / degree-norm (+ transposes, epilogues) through
the C ABI vs the float64 oracle, tolerance of SURVEY.md Appendix A.8:
|gpu - ref| <= 1e-5 * max(|ref|, ref_abs), ref_abs = the op on |inputs|."""

import numpy as np
import pytest
import torch

from oracle import graph as og
from oracle import ops as oo

pytestmark = pytest.mark.gpu
RTOL = 1e-5


@pytest.fixture(scope="module")
def gb(cuda):
    import paper_2605_29346_b200 as gb

    return gb


def assert_close(gpu, ref, ref_abs, what=""):
    ok, worst = oo.close(gpu.detach().cpu().numpy() if torch.is_tensor(gpu) else gpu, ref,
                         ref_abs, RTOL)
    assert ok, f"{what}: worst scaled error {worst:.3e}"


@pytest.fixture(scope="module")
def graphs(gb):
    out = {}
    out["cora_pl"] = gb.generate(gb.GraphGenSpec("power-law", 2708, 10556, exponent=2.1), 42)
    out["pl_10k"] = gb.generate(gb.GraphGenSpec("power-law", 10_000, 200_000, exponent=2.1), 7)
    out["ur_5k"] = gb.generate(gb.GraphGenSpec("uniform-random", 5000, 60_000), 43)
    # heavy skew + empty rows: one mega row, many isolated vertices
    rng = np.random.default_rng(5)
    src = np.concatenate([np.zeros(300_000, np.int64), rng.integers(1, 500, 20_000)])
    dst = rng.integers(0, 4000, src.size)
    out["mega"] = gb.csr_from_edges(4000, src, dst)
    return out


def host(g):
    return g.offsets, g.targets


@pytest.mark.parametrize("gname", ["cora_pl", "pl_10k", "ur_5k", "mega"])
@pytest.mark.parametrize("K", [1, 3, 4, 16, 32, 41, 64, 128, 256, 300, 602])
def test_spmmv_forward(gb, graphs, gname, K):
    g = graphs[gname]
    off, tgt = host(g)
    rng = np.random.default_rng(K)
    X = rng.uniform(-1, 1, (g.num_vertices, K)).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    for norm in (False, True):
        Y = gb.spmmv(g, Xd, norm=norm)
        ref = oo.spmm(off, tgt, X, norm=norm)
        ra = oo.spmm(off, tgt, np.abs(X), norm=norm)
        assert_close(Y, ref, ra, f"{gname} K={K} norm={norm}")


@pytest.mark.parametrize("gname", ["cora_pl", "pl_10k", "mega"])
@pytest.mark.parametrize("K", [16, 32, 41])
def test_spmmv_transpose_and_coalesced(gb, graphs, gname, K):
    g = graphs[gname]
    off, tgt = host(g)
    t_off, t_rows, _ = og.transpose(g.num_vertices, g.num_vertices, off, tgt)
    rng = np.random.default_rng(K + 1)
    X = rng.uniform(-1, 1, (g.num_vertices, K)).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    Yt = gb.spmmv(g, Xd, transpose=True)
    assert_close(Yt, oo.spmm(t_off, t_rows, X), oo.spmm(t_off, t_rows, np.abs(X)), "transpose")
    Yc = gb.spmmv(g, Xd, norm=True, coalesced=True)
    assert_close(Yc, oo.spmm(off, tgt, X, norm=True), oo.spmm(off, tgt, np.abs(X), norm=True),
                 "coalesced")
    Ytc = gb.spmmv(g, Xd, transpose=True, coalesced=True)
    assert_close(Ytc, oo.spmm(t_off, t_rows, X), oo.spmm(t_off, t_rows, np.abs(X)), "csc coalesced")


@pytest.mark.parametrize("heads,F", [(1, 16), (4, 16), (2, 3), (3, 5), (4, 8), (4, 3)])
@pytest.mark.parametrize("gname", ["pl_10k", "mega", "pl_big"])
def test_spmmve_forward_and_transpose(gb, graphs, heads, F, gname):
    """Multi-head SpMMve and its transpose through the edge ids; four heads take
    the staged-weights path (WM_HEADS4) of the nnz-split kernel, on row-order
    (pl_10k, mega: split and empty rows) and degree-sorted (pl_big, >= 2^20
    entries) operands."""
    if gname == "pl_big" and "pl_big" not in graphs:
        graphs["pl_big"] = gb.generate(gb.GraphGenSpec("power-law", 40_000, 1_500_000,
                                                       exponent=2.1), 11)
    g = graphs[gname]
    off, tgt = host(g)
    t_off, t_rows, eid = og.transpose(g.num_vertices, g.num_vertices, off, tgt)
    rng = np.random.default_rng(heads * 10 + F)
    K = heads * F
    X = rng.uniform(-1, 1, (g.num_vertices, K)).astype(np.float32)
    ev = rng.uniform(0, 1, (g.num_edges, heads)).astype(np.float32)
    Xd, evd = torch.from_numpy(X).cuda(), torch.from_numpy(ev).cuda()
    Y = gb.spmmve(g, Xd, evd)
    assert_close(Y, oo.spmm(off, tgt, X, vals=ev, heads=heads),
                 oo.spmm(off, tgt, np.abs(X), vals=ev, heads=heads), "spmmve")
    Yt = gb.spmmve(g, Xd, evd, transpose=True)
    assert_close(Yt, oo.spmm(t_off, t_rows, X, vals=ev[eid], heads=heads),
                 oo.spmm(t_off, t_rows, np.abs(X), vals=ev[eid], heads=heads), "spmmve^T")


def test_degree_norm_inplace(gb, graphs):
    g = graphs["mega"]
    off, _ = host(g)
    X = torch.randn(g.num_vertices, 24, device="cuda")
    ref = oo.degree_norm(off, X.cpu().numpy())
    ptr = X.data_ptr()
    gb.degree_norm_(g, X)
    assert X.data_ptr() == ptr
    assert_close(X, ref, np.abs(ref), "degree_norm_")


def test_epilogues(gb, graphs):
    from paper_2605_29346_b200 import _lib
    from paper_2605_29346_b200.ops import spmm_raw

    g = graphs["mega"]
    off, tgt = host(g)
    t_off, t_rows, _ = og.transpose(g.num_vertices, g.num_vertices, off, tgt)
    V, K = g.num_vertices, 16
    rng = np.random.default_rng(9)
    X = rng.uniform(-1, 1, (V, K)).astype(np.float32)
    S = rng.uniform(-1, 1, (V, K)).astype(np.float32)
    M = rng.uniform(-1, 1, (V, K)).astype(np.float32)
    b = rng.uniform(-1, 1, K).astype(np.float32)
    Xd, Sd, Md, bd = (torch.from_numpy(a).cuda() for a in (X, S, M, b))
    f = (_lib.EPI_NORM | _lib.EPI_SELF | _lib.EPI_BIAS | _lib.EPI_RELU | _lib.EPI_MASK
         | _lib.EPI_POSTNORM)
    csc = g.csc()
    Y = spmm_raw(g.csr(), Xd, flags=f, self_x=Sd, self_scale=1.5, bias=bd, mask=Md,
                 post_deg_offsets=csc.offsets)
    pre = oo.spmm(off, tgt, X, norm=True) + 1.5 * S + b
    ref = np.maximum(pre, 0) * (M > 0)
    tdeg = np.diff(t_off).astype(np.float64)
    ref = ref * np.divide(1.0, tdeg, out=np.zeros_like(tdeg), where=tdeg > 0)[:, None]
    ra = (oo.spmm(off, tgt, np.abs(X), norm=True) + 1.5 * np.abs(S) + np.abs(b))
    ra = ra * np.divide(1.0, tdeg, out=np.zeros_like(tdeg), where=tdeg > 0)[:, None]
    assert_close(Y, ref, ra, "fused epilogue")


def test_spmmv_autograd(gb, graphs):
    g = graphs["cora_pl"]
    off, tgt = host(g)
    t_off, t_rows, _ = og.transpose(g.num_vertices, g.num_vertices, off, tgt)
    X = torch.randn(g.num_vertices, 16, device="cuda", requires_grad=True)
    dY = torch.randn(g.num_vertices, 16, device="cuda")
    Y = gb.spmmv(g, X, norm=True)
    Y.backward(dY)
    dYn = oo.degree_norm(off, dY.cpu().numpy())
    ref = oo.spmm(t_off, t_rows, dYn)
    ra = oo.spmm(t_off, t_rows, np.abs(dYn))
    assert_close(X.grad, ref, ra, "spmmv backward")


def test_deterministic(gb, graphs):
    g = graphs["mega"]
    X = torch.randn(g.num_vertices, 32, device="cuda")
    a = gb.spmmv(g, X, norm=True)
    b = gb.spmmv(g, X, norm=True)
    assert torch.equal(a, b)


@pytest.mark.slow
def test_reddit_shape_spmmv_properties(gb):
    """Full Reddit shape (V=232,965, E=114,615,892): ones -> degrees exactly,
    and sampled rows (incl. the largest mega rows) vs the float64 oracle."""
    g = gb.generate(gb.GraphGenSpec("power-law", 232_965, 114_615_892, exponent=2.1), 42)
    V = g.num_vertices
    ones = torch.ones(V, 16, device="cuda")
    deg = g.device_degrees().to(torch.float32)
    Y = gb.spmmv(g, ones)
    assert torch.equal(Y, deg[:, None].expand(V, 16))
    Yc = gb.spmmv(g, ones, coalesced=True)
    assert torch.equal(Yc, deg[:, None].expand(V, 16))
    off, tgt = g.offsets, g.targets
    d = np.diff(off)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([np.argsort(d)[-3:], rng.integers(0, V, 64)]))
    X = torch.rand(V, 16, device="cuda") * 2 - 1
    Xh = X.cpu().numpy()
    for coalesced in (False, True):
        Y = gb.spmmv(g, X, norm=True, coalesced=coalesced).cpu().numpy()
        for r in rows:
            seg = tgt[off[r]:off[r + 1]]
            ref = Xh[seg].astype(np.float64).sum(0) / len(seg)
            ra = np.abs(Xh[seg]).astype(np.float64).sum(0) / len(seg)
            assert np.all(np.abs(Y[r] - ref) <= RTOL * np.maximum(np.abs(ref), ra)), (r, coalesced)


@pytest.mark.parametrize("gname", ["cora_pl", "pl_10k", "mega"])
@pytest.mark.parametrize("K", [4, 16, 32, 64, 130])
def test_packed_multiplicity_operand_bit_identical(gb, graphs, gname, K):
    """The coalesced operands are stored packed (column | multiplicity <<
    col_bits, gnn_csr_pack_weights); the SpMM over the packed words equals the
    SpMM over the float-multiplicity form bit for bit (same order, same
    weights), with every epilogue path."""
    from paper_2605_29346_b200 import _lib
    from paper_2605_29346_b200.graph import SparseOperand
    from paper_2605_29346_b200.ops import spmm_raw

    g = graphs[gname]
    for co in (g.csr_coalesced(), g.csc_coalesced()):
        assert co.packed is not None and co.col_bits == max(1, (g.num_vertices - 1).bit_length())
        cols, vals = co.entries()
        plain = SparseOperand(co.num_rows, co.num_cols, co.offsets, cols, vals=vals,
                              deg_offsets=co.deg_offsets)
        assert plain.packed is None
        rng = np.random.default_rng(K)
        X = torch.from_numpy(rng.uniform(-1, 1, (g.num_vertices, K)).astype(np.float32)).cuda()
        b = torch.from_numpy(rng.uniform(-1, 1, K).astype(np.float32)).cuda()
        for flags in (0, _lib.EPI_NORM | _lib.EPI_BIAS | _lib.EPI_RELU):
            Ys = []
            for op in (co, plain):  # row order for both (a given plan skips the sorted form)
                Ys.append(spmm_raw(op, X, plan=op.spmm_plan(), flags=flags, bias=b))
            assert torch.equal(Ys[0], Ys[1]), (gname, K, flags)


def test_pack_weights_range_checks(gb):
    from paper_2605_29346_b200 import _lib

    lib = _lib.lib()
    ws = _lib.workspace(lib.gnn_csr_pack_weights_workspace(), torch.device("cuda"))
    out = torch.empty(3, dtype=torch.int32, device="cuda")

    def pack(cols, w, bits):
        c = torch.tensor(cols, dtype=torch.int32, device="cuda")
        v = torch.tensor(w, dtype=torch.float32, device="cuda")
        return lib.gnn_csr_pack_weights(3, c.data_ptr(), v.data_ptr(), bits, out.data_ptr(),
                                        ws.data_ptr(), ws.numel(), None)

    assert pack([0, 5, 7], [1, 2, 3], 3) == 0
    assert out.tolist() == [0 | 1 << 3, 5 | 2 << 3, 7 | 3 << 3]
    assert pack([0, 8, 7], [1, 2, 3], 3) == _lib.GNN_ERR_RANGE      # column needs 4 bits
    assert pack([0, 1, 2], [1, 2.5, 3], 3) == _lib.GNN_ERR_RANGE    # not an integer weight
    assert pack([0, 1, 2], [1, 2, 1 << 29], 3) == _lib.GNN_ERR_RANGE  # weight overflows 29 bits
    assert pack([0, 1, 2], [1, -1, 3], 3) == _lib.GNN_ERR_RANGE
    assert pack([0, 1, 2], [1, 2, 3], 0) == _lib.GNN_ERR_INVALID_ARGUMENT


def test_packed_operand_splits_large_multiplicities(gb):
    """A multiplicity above the packed word's weight field (2^(32-col_bits)-1)
    is split into several entries of the same column; the SpMM result stays
    within the A.8 tolerance of the oracle."""
    V = 1 << 20  # 20 column bits -> weights up to 4095 per word
    rng = np.random.default_rng(3)
    src = np.concatenate([np.zeros(10_000, np.int64), np.full(5000, 7), rng.integers(0, V, 50_000)])
    dst = np.concatenate([np.full(10_000, 5), np.full(5000, 5), rng.integers(0, V, 50_000)])
    g = gb.csr_from_edges(V, src, dst)
    co = g.csr_coalesced()
    assert co.packed is not None and co.col_bits == 20
    cols, vals = co.entries()
    o = co.offsets.cpu().numpy()
    c0, w0 = cols[o[0]:o[1]].cpu().numpy(), vals[o[0]:o[1]].cpu().numpy()
    assert sorted(w0[c0 == 5].tolist()) == [1810.0, 4095.0, 4095.0]  # 10000 = 2*4095 + 1810
    c7, w7 = cols[o[7]:o[8]].cpu().numpy(), vals[o[7]:o[8]].cpu().numpy()
    assert sorted(w7[c7 == 5].tolist()) == [905.0, 4095.0]
    off, tgt = g.offsets, g.targets
    X = rng.uniform(-1, 1, (V, 16)).astype(np.float32)
    Y = gb.spmmv(g, torch.from_numpy(X).cuda(), norm=True, coalesced=True)
    assert_close(Y, oo.spmm(off, tgt, X, norm=True), oo.spmm(off, tgt, np.abs(X), norm=True),
                 "split multiplicities")
    ct = g.csc_coalesced()
    t_off, t_rows, _ = og.transpose(V, V, off, tgt)
    Yt = gb.spmmv(g, torch.from_numpy(X).cuda(), transpose=True, coalesced=True)
    assert_close(Yt, oo.spmm(t_off, t_rows, X), oo.spmm(t_off, t_rows, np.abs(X)), "csc split")
    assert ct.packed is not None


@pytest.mark.parametrize("gname", ["cora_pl", "pl_10k", "ur_5k", "mega"])
@pytest.mark.parametrize("K", [4, 16, 32, 64])
def test_degree_sorted_operand_matches_row_order(gb, graphs, gname, K):
    """gnn_spmm over the degree-sorted operand (rows longest-first, row_ids
    back to output rows; the nnz-split kernel covers only the long-row prefix)
    equals the SpMM over the operand in row order — bit for bit on the short
    tail, to fp32 rounding on the long rows — for every epilogue (per-row
    inputs indexed by output row)."""
    from paper_2605_29346_b200 import _lib
    from paper_2605_29346_b200.graph import SPMM_SHORT_MAX, SPMM_SHORT_ROWORDER
    from paper_2605_29346_b200.ops import spmm_raw

    g = graphs[gname]
    V = g.num_vertices
    rng = np.random.default_rng(K + 7)
    X = torch.from_numpy(rng.uniform(-1, 1, (V, K)).astype(np.float32)).cuda()
    S = torch.from_numpy(rng.uniform(-1, 1, (V, K)).astype(np.float32)).cuda()
    M = torch.from_numpy(rng.uniform(-1, 1, (V, K)).astype(np.float32)).cuda()
    b = torch.from_numpy(rng.uniform(-1, 1, K).astype(np.float32)).cuda()
    N_, S_, B_, R_, M_, P_ = (_lib.EPI_NORM, _lib.EPI_SELF, _lib.EPI_BIAS, _lib.EPI_RELU,
                              _lib.EPI_MASK, _lib.EPI_POSTNORM)
    for op in (g.csr(), g.csc(), g.csr_coalesced(), g.csc_coalesced()):
        so = op.by_degree()
        assert so.row_ids is not None and so.nnz == op.nnz
        plan = so.spmm_plan()
        long_rows = int((so.offsets[1:] - so.offsets[:-1] > SPMM_SHORT_MAX).sum().item())
        assert plan.main_nnz == int(so.offsets[long_rows].item())
        deg = op.deg_offsets if op.deg_offsets is not None else op.offsets
        for flags in (0, N_ | B_ | R_, S_ | M_, N_ | S_ | P_):
            kw = dict(flags=flags, bias=b, self_x=S, self_scale=0.5, mask=M,
                      post_deg_offsets=g.d_offsets)
            Y0 = spmm_raw(op, X, plan=op.spmm_plan(), **kw)  # row order (plan given: no sorting)
            Y1 = spmm_raw(so, X, plan=plan, **kw)
            # the long rows' fp32 partial-sum order follows their position in
            # the edge array (warp ranges), so equal up to rounding only
            # (A.8: relative to the same contraction on absolute values)
            ra = spmm_raw(op, X.abs(), plan=op.spmm_plan(), flags=flags & N_)
            if flags & B_:
                ra = ra + b.abs()
            if flags & S_:
                ra = ra + 0.5 * S.abs()
            assert bool(((Y0 - Y1).abs() <= 1e-5 * ra + 1e-30).all()), (gname, K, flags)
            # rows both forms send to the group-per-row kernel: bit-identical
            short = (op.offsets[1:] - op.offsets[:-1]) <= min(SPMM_SHORT_MAX, SPMM_SHORT_ROWORDER)
            assert torch.equal(Y0[short], Y1[short]), (gname, K, flags)
        ref_deg = deg  # NORM of the sorted operand uses output-row degrees
        assert so.deg_offsets is ref_deg or torch.equal(so.deg_offsets, ref_deg)


def test_degree_sorted_plan_needs_short_kernel(gb, graphs):
    """A sorted operand's plan stops the nnz-split range at the short tail, so
    a call that cannot use the short-row kernel (K > 64) is refused."""
    from paper_2605_29346_b200.ops import spmm_raw

    g = graphs["pl_10k"]
    so = g.csr().by_degree()
    plan = so.spmm_plan()
    assert plan.main_nnz < so.nnz
    X = torch.ones(g.num_vertices, 128, device="cuda")
    with pytest.raises(ValueError):
        spmm_raw(so, X, plan=plan)
    Y = spmm_raw(g.csr(), X)  # the row-order operand still runs at K=128
    assert torch.equal(Y[:, 0].cpu(), torch.from_numpy(np.diff(g.offsets).astype(np.float32)))
