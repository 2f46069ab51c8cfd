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


@pytest.mark.parametrize("heads,F", [(1, 16), (4, 16), (2, 3), (3, 5)])
def test_spmmve_forward_and_transpose(gb, graphs, heads, F):
    g = graphs["pl_10k"]
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
