"""GPU parity: SDDMM, edge-softmax (given and GAT scores, forward and
backward), SpMMve's edge-value gradient, and the GAT / GIN layers (forward +
every gradient) through the C ABI vs the float64 oracle.  Tolerance of
SURVEY.md Appendix A.8: |gpu - ref| <= 1e-5 * max(|ref|, ref_abs), ref_abs =
the same contraction on |inputs|."""

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
    g = gpu.detach().cpu().numpy() if torch.is_tensor(gpu) else gpu
    ok, worst = oo.close(g.reshape(np.shape(ref)), ref, ref_abs, RTOL)
    assert ok, f"{what}: worst scaled error {worst:.3e}"


@pytest.fixture(scope="module")
def graphs(gb):
    out = {}
    out["cora_pl"] = gb.generate(gb.GraphGenSpec("power-law", 2708, 10556, exponent=2.1), 42)
    out["pl_10k"] = gb.generate(gb.GraphGenSpec("power-law", 10_000, 200_000, exponent=2.1), 7)
    rng = np.random.default_rng(5)
    src = np.concatenate([np.zeros(300_000, np.int64), rng.integers(1, 500, 20_000)])
    dst = rng.integers(0, 4000, src.size)
    out["mega"] = gb.csr_from_edges(4000, src, dst)  # one 300k-edge row + many empty rows
    return out


GNAMES = ["cora_pl", "pl_10k", "mega"]


@pytest.mark.parametrize("gname", GNAMES)
@pytest.mark.parametrize("K,heads", [(1, 1), (4, 1), (16, 1), (64, 4), (32, 2), (12, 3), (188, 4),
                                     (128, 1), (256, 2), (512, 4), (41, 1)])
def test_sddmm(gb, graphs, gname, K, heads):
    from paper_2605_29346_b200.sparse_attn import sddmm

    g = graphs[gname]
    off, tgt = g.offsets, g.targets
    rng = np.random.default_rng(K * 7 + heads)
    X = rng.uniform(-1, 1, (g.num_vertices, K)).astype(np.float32)
    Y = rng.uniform(-1, 1, (g.num_vertices, K)).astype(np.float32)
    out = sddmm(g, torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), heads=heads)
    ref = oo.sddmm(off, tgt, X, Y, heads)
    ra = oo.sddmm(off, tgt, np.abs(X), np.abs(Y), heads)
    assert_close(out, ref, ra, f"sddmm {gname} K={K} H={heads}")


@pytest.mark.parametrize("gname", GNAMES)
@pytest.mark.parametrize("heads", [1, 3, 4, 8])
def test_edge_softmax_given_scores(gb, graphs, gname, heads):
    from paper_2605_29346_b200.sparse_attn import edge_softmax

    g = graphs[gname]
    off = g.offsets
    rng = np.random.default_rng(heads)
    s = rng.normal(0, 3, (g.num_edges, heads)).astype(np.float32)
    st = torch.from_numpy(s).cuda().requires_grad_(True)
    alpha = edge_softmax(g, st)
    ref = oo.edge_softmax(off, s)
    assert_close(alpha, ref, None, f"softmax {gname} H={heads}")
    # rows sum to one
    sums = oo.spmm(off, g.targets, np.ones((g.num_vertices, heads)),
                   vals=alpha.detach().cpu().numpy().astype(np.float64), heads=heads)
    nz = np.diff(off) > 0
    assert np.allclose(sums[nz], 1.0, atol=1e-5)
    dal = rng.normal(size=s.shape).astype(np.float32)
    alpha.backward(torch.from_numpy(dal).cuda())
    dref = oo.edge_softmax_backward(off, ref, dal)
    a = np.abs(dal)
    dabs = ref * (a + np.repeat(np.add.reduceat(ref * a, off[:-1][nz], axis=0), np.diff(off)[nz],
                                axis=0))
    assert_close(st.grad, dref, dabs, f"softmax bwd {gname} H={heads}")


def test_edge_softmax_1d_and_extreme_scores(gb, graphs):
    from paper_2605_29346_b200.sparse_attn import edge_softmax

    g = graphs["mega"]
    rng = np.random.default_rng(3)
    s = (rng.normal(0, 1, g.num_edges) * 80).astype(np.float32)  # exp would overflow unshifted
    alpha = edge_softmax(g, torch.from_numpy(s).cuda())
    assert alpha.shape == (g.num_edges,)
    assert torch.isfinite(alpha).all()
    assert_close(alpha, oo.edge_softmax(g.offsets, s), None, "softmax large scores")


@pytest.mark.parametrize("gname", GNAMES)
@pytest.mark.parametrize("heads", [1, 4])
def test_gat_scores_softmax(gb, graphs, gname, heads):
    from paper_2605_29346_b200.sparse_attn import gat_attention

    g = graphs[gname]
    rng = np.random.default_rng(11 + heads)
    el = rng.normal(0, 2, (g.num_vertices, heads)).astype(np.float32)
    er = rng.normal(0, 2, (g.num_vertices, heads)).astype(np.float32)
    alpha = gat_attention(g, torch.from_numpy(el).cuda(), torch.from_numpy(er).cuda(), 0.2)
    s, _ = oo.gat_scores(g.offsets, g.targets, el, er, 0.2)
    assert_close(alpha, oo.edge_softmax(g.offsets, s), None, f"gat softmax {gname}")


@pytest.mark.parametrize("gname", ["cora_pl", "mega"])
@pytest.mark.parametrize("transpose", [False, True])
def test_spmmve_edge_value_grad(gb, graphs, gname, transpose):
    g = graphs[gname]
    off, tgt = g.offsets, g.targets
    rng = np.random.default_rng(2)
    H, F = 4, 8
    X = rng.uniform(-1, 1, (g.num_vertices, H * F)).astype(np.float32)
    ev = rng.uniform(0, 1, (g.num_edges, H)).astype(np.float32)
    evt = torch.from_numpy(ev).cuda().requires_grad_(True)
    Xt = torch.from_numpy(X).cuda().requires_grad_(True)
    Y = gb.spmmve(g, Xt, evt, transpose=transpose)
    dY = rng.uniform(-1, 1, Y.shape).astype(np.float32)
    Y.backward(torch.from_numpy(dY).cuda())
    if transpose:
        ref = oo.sddmm(off, tgt, X, dY, H)
        ra = oo.sddmm(off, tgt, np.abs(X), np.abs(dY), H)
    else:
        ref = oo.sddmm(off, tgt, dY, X, H)
        ra = oo.sddmm(off, tgt, np.abs(dY), np.abs(X), H)
    assert_close(evt.grad, ref, ra, f"spmmve d(ev) {gname} T={transpose}")


def _gat_check(gb, g, X, heads, F, mean, relu, seed):
    from paper_2605_29346_b200.models import GATConv

    off, tgt = g.offsets, g.targets
    layer = GATConv(X.shape[1], F, heads, mean=mean, seed=seed, device="cuda")
    with torch.no_grad():  # non-trivial bias and attention vectors
        rng = np.random.default_rng(seed)
        layer.bias.copy_(torch.from_numpy(rng.normal(0, 0.1, layer.bias.shape).astype(np.float32)))
    Xt = torch.from_numpy(X).cuda().requires_grad_(True)
    out = layer(g, Xt, relu=relu)
    p = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in layer.named_parameters()}
    ref, cache = oo.gat_layer_fwd(off, tgt, X, p["weight"], p["attn_l"], p["attn_r"], p["bias"],
                                  heads, mean=mean, relu=relu)
    Xa = np.abs(X.astype(np.float64))
    Wh_abs = Xa @ np.abs(p["weight"])
    ra = oo.spmm(off, tgt, Wh_abs, vals=cache["alpha"], heads=heads)
    ra = ra.reshape(len(ra), heads, F).mean(1) + np.abs(p["bias"]) if mean else ra + np.abs(p["bias"])
    assert_close(out, ref, ra, "gat forward")
    G = np.random.default_rng(seed + 1).uniform(-1, 1, ref.shape).astype(np.float32)
    out.backward(torch.from_numpy(G).cuda())
    gr = oo.gat_layer_bwd(off, tgt, cache, G)
    ga = oo.gat_layer_bwd(off, tgt, cache, G, absmode=True)
    names = {"weight": "W", "attn_l": "a_l", "attn_r": "a_r", "bias": "b"}
    for pn, on in names.items():
        assert_close(dict(layer.named_parameters())[pn].grad, gr[on], ga[on], f"gat d{pn}")
    assert_close(Xt.grad, gr["X"], ga["X"], "gat dX")


@pytest.mark.parametrize("gname", GNAMES)
def test_gat_layer_hidden_concat_relu(gb, graphs, gname):
    g = graphs[gname]
    X = np.random.default_rng(0).uniform(-1, 1, (g.num_vertices, 24)).astype(np.float32)
    _gat_check(gb, g, X, heads=4, F=16, mean=False, relu=True, seed=1)


@pytest.mark.parametrize("gname", ["cora_pl", "mega"])
@pytest.mark.parametrize("F", [7, 16])
def test_gat_layer_output_mean(gb, graphs, gname, F):
    g = graphs[gname]
    X = np.random.default_rng(1).uniform(-1, 1, (g.num_vertices, 64)).astype(np.float32)
    _gat_check(gb, g, X, heads=4, F=F, mean=True, relu=False, seed=3)


@pytest.mark.parametrize("gname", ["cora_pl", "pl_10k", "mega"])
@pytest.mark.parametrize("coalesced", [False, True])
def test_gin_layer(gb, graphs, gname, coalesced):
    from paper_2605_29346_b200.models import GINConv

    g = graphs[gname]
    off, tgt = g.offsets, g.targets
    t_off, t_rows, _ = og.transpose(g.num_vertices, g.num_vertices, off, tgt)
    rng = np.random.default_rng(4)
    X = rng.uniform(-1, 1, (g.num_vertices, 40)).astype(np.float32)
    layer = GINConv(40, 32, 9, eps=0.25, seed=2, device="cuda")
    with torch.no_grad():
        layer.b1.copy_(torch.from_numpy(rng.normal(0, 0.5, 32).astype(np.float32)))
    Xt = torch.from_numpy(X).cuda().requires_grad_(True)
    out = layer(g, Xt, coalesced=coalesced)
    p = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in layer.named_parameters()}
    ref, cache = oo.gin_layer_fwd(off, tgt, X, p["w1"], p["b1"], p["w2"], p["b2"], eps=0.25)
    absref, _ = oo.gin_layer_fwd(off, tgt, np.abs(X), np.abs(p["w1"]), np.abs(p["b1"]),
                                 np.abs(p["w2"]), np.abs(p["b2"]), eps=0.25)
    assert_close(out, ref, absref, "gin forward")
    G = rng.uniform(-1, 1, ref.shape).astype(np.float32)
    out.backward(torch.from_numpy(G).cuda())
    gr = oo.gin_layer_bwd(t_off, t_rows, cache, G)
    ga = oo.gin_layer_bwd(t_off, t_rows, cache, G, absmode=True)
    for pn in ("w1", "b1", "w2", "b2"):
        on = {"w1": "W1", "b1": "b1", "w2": "W2", "b2": "b2"}[pn]
        assert_close(dict(layer.named_parameters())[pn].grad, gr[on], ga[on], f"gin d{pn}")
    assert_close(Xt.grad, gr["X"], ga["X"], "gin dX")


def test_gat_model_trains(gb, graphs):
    """Two GAT layers through autograd + torch's optimizer: loss decreases."""
    from paper_2605_29346_b200.models import GAT

    g = graphs["cora_pl"]
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.uniform(-1, 1, (g.num_vertices, 32)).astype(np.float32)).cuda()
    y = torch.from_numpy(rng.integers(0, 7, g.num_vertices)).cuda()
    model = GAT(32, 8, 7, heads=4, device="cuda")
    opt = torch.optim.Adam(model.parameters(), lr=0.02)
    losses = []
    for _ in range(60):
        opt.zero_grad()
        loss = torch.nn.functional.cross_entropy(model(g, X), y)
        loss.backward()
        opt.step()
        losses.append(loss.item())
    assert losses[-1] < losses[0] - 0.1


@pytest.mark.parametrize("gname", GNAMES)
@pytest.mark.parametrize("heads", [1, 4, 6])
def test_segment_sum_rows_and_columns(gb, graphs, gname, heads):
    from paper_2605_29346_b200.kernels import SegmentSumCall

    g = graphs[gname]
    V, E = g.num_vertices, g.num_edges
    rng = np.random.default_rng(heads)
    vals = rng.normal(size=(E, heads)).astype(np.float32)
    vt = torch.from_numpy(vals).cuda()
    rows = torch.empty(V, heads, device="cuda")
    cols = torch.empty(V, heads, device="cuda")
    SegmentSumCall(g.csr(), vt, rows, heads)()
    SegmentSumCall(g.csc(with_eid=True), vt, cols, heads, use_eid=True)()
    ones = np.ones((V, heads))
    ref_r = oo.spmm(g.offsets, g.targets, ones, vals=vals, heads=heads)
    ref_c = np.zeros((V, heads))
    np.add.at(ref_c, g.targets, vals.astype(np.float64))
    abs_r = oo.spmm(g.offsets, g.targets, ones, vals=np.abs(vals), heads=heads)
    abs_c = np.zeros((V, heads))
    np.add.at(abs_c, g.targets, np.abs(vals).astype(np.float64))
    assert_close(rows, ref_r, abs_r, "row sums")
    assert_close(cols, ref_c, abs_c, "column sums via edge-ID")


@pytest.mark.parametrize("gname", GNAMES)
@pytest.mark.parametrize("H,F", [(4, 16), (4, 48), (4, 12), (1, 32), (2, 64), (3, 8), (8, 8),
                                 (1, 4), (4, 32)])
def test_gat_bwd_csc_fused(gb, graphs, gname, H, F):
    """dWh = SpMMve^T(alpha, dY) and dalpha = SDDMM(dY, Wh) from the fused CSC kernel."""
    from paper_2605_29346_b200.kernels import GatBwdCscCall

    g = graphs[gname]
    V, E, K = g.num_vertices, g.num_edges, H * F
    off, tgt = g.offsets, g.targets
    rng = np.random.default_rng(H * 100 + F)
    alpha = rng.uniform(0, 1, (E, H)).astype(np.float32)
    dY = rng.uniform(-1, 1, (V, K)).astype(np.float32)
    Wh = rng.uniform(-1, 1, (V, K)).astype(np.float32)
    AT = g.csc(with_eid=True)
    dWh = torch.empty(V, K, device="cuda")
    dal = torch.empty(E, H, device="cuda")
    t = [torch.from_numpy(x).cuda() for x in (alpha, dY, Wh)]
    GatBwdCscCall(AT, t[0], t[1], t[2], dWh, dal, H)()
    rows = np.repeat(np.arange(V), np.diff(off))
    ref = np.zeros((V, K))
    np.add.at(ref, tgt, (dY[rows].reshape(-1, H, F) * alpha[:, :, None]).reshape(-1, K).astype(np.float64))
    ra = np.zeros((V, K))
    np.add.at(ra, tgt, (np.abs(dY[rows]).reshape(-1, H, F) * alpha[:, :, None]).reshape(-1, K).astype(np.float64))
    assert_close(dWh, ref, ra, "fused dWh")
    assert_close(dal, oo.sddmm(off, tgt, dY, Wh, H), oo.sddmm(off, tgt, np.abs(dY), np.abs(Wh), H),
                 "fused dalpha")


@pytest.mark.parametrize("gname", GNAMES)
@pytest.mark.parametrize("H,F", [(4, 48), (4, 16), (2, 8), (1, 4), (3, 20), (4, 128), (8, 12)])
def test_gat_bwd_csc_mean_fused(gb, graphs, gname, H, F):
    """Head-mean variant: gathers dZ (F wide) once and produces every head."""
    from paper_2605_29346_b200.kernels import GatBwdCscMeanCall

    g = graphs[gname]
    V, E, K = g.num_vertices, g.num_edges, H * F
    off, tgt = g.offsets, g.targets
    rng = np.random.default_rng(H * 10 + F)
    alpha = rng.uniform(0, 1, (E, H)).astype(np.float32)
    dZ = rng.uniform(-1, 1, (V, F)).astype(np.float32)
    Wh = rng.uniform(-1, 1, (V, K)).astype(np.float32)
    AT = g.csc(with_eid=True)
    dWh = torch.empty(V, K, device="cuda")
    dal = torch.empty(E, H, device="cuda")
    t = [torch.from_numpy(x).cuda() for x in (alpha, dZ, Wh)]
    GatBwdCscMeanCall(AT, t[0], t[1], t[2], dWh, dal, H)()
    dY = np.tile(dZ.astype(np.float64) / H, (1, H))  # the concatenated-head gradient
    rows = np.repeat(np.arange(V), np.diff(off))
    ref = np.zeros((V, K))
    np.add.at(ref, tgt, (dY[rows].reshape(-1, H, F) * alpha[:, :, None]).reshape(-1, K))
    ra = np.zeros((V, K))
    np.add.at(ra, tgt, (np.abs(dY[rows]).reshape(-1, H, F) * alpha[:, :, None]).reshape(-1, K))
    assert_close(dWh, ref, ra, "mean dWh")
    assert_close(dal, oo.sddmm(off, tgt, dY, Wh, H), oo.sddmm(off, tgt, np.abs(dY), np.abs(Wh), H),
                 "mean dalpha")


@pytest.mark.parametrize("gname", ["cora_pl", "pl_10k", "mega"])
@pytest.mark.parametrize("F", [4, 16, 64])
def test_spmm_shared_heads(gb, graphs, gname, F):
    """gnn_spmm_shared_heads: Y[v, 4i+h] = s * sum_e alpha[e,h] X[col_e, i]
    (four heads over one shared row) against the float64 statement."""
    from paper_2605_29346_b200.kernels import SharedHeadsCall

    g = graphs[gname]
    off, tgt = g.offsets, g.targets
    V = g.num_vertices
    rng = np.random.default_rng(F)
    X = rng.uniform(-1, 1, (V, F)).astype(np.float32)
    al = rng.uniform(0, 1, (tgt.size, 4)).astype(np.float32)
    Y = torch.empty(V, 4 * F, device="cuda")
    SharedHeadsCall(g.csr(), torch.from_numpy(X).cuda(), torch.from_numpy(al).cuda(), Y,
                    scale=0.25)()
    rows = np.repeat(np.arange(V), np.diff(off))
    ref = np.zeros((V, F, 4))
    ra = np.zeros((V, F, 4))
    for h in range(4):
        np.add.at(ref[:, :, h], rows, al[:, h:h + 1].astype(np.float64) * X[tgt])
        np.add.at(ra[:, :, h], rows, np.abs(al[:, h:h + 1].astype(np.float64) * X[tgt]))
    ok, worst = oo.close(Y.cpu().numpy(), 0.25 * ref.reshape(V, 4 * F), 0.25 * ra.reshape(V, 4 * F))
    assert ok, worst


@pytest.mark.parametrize("V,F1,Cp", [(1000, 16, 48), (300, 64, 48), (4099, 64, 8), (129, 8, 64)])
@pytest.mark.parametrize("tc", [True, False])
def test_gat_rowstat_mean(gb, V, F1, Cp, tc, monkeypatch):
    """Head-mean layer statistics S[v,h] = scale sum_i Yc[v,4i+h] (W_h dZ[v])_i
    (tensor-core epilogue form and the SIMT kernel) packed beside er / m /
    1/sum, vs float64."""
    from paper_2605_29346_b200.kernels import GatRowStatCall

    monkeypatch.setenv("GNN_GAT_ROWSTAT_TC", "1" if tc else "0")
    g = torch.Generator(device="cuda").manual_seed(V + F1)
    dZs = torch.randn(V, Cp + 16, device="cuda", generator=g)
    dZ = dZs[:, :Cp]
    Yc = torch.randn(V, 4 * F1, device="cuda", generator=g)
    W = torch.randn(F1, 4 * Cp, device="cuda", generator=g)
    er = torch.randn(V, 4, device="cuda", generator=g)
    ms = torch.randn(V, 8, device="cuda", generator=g)
    stat = dZs[:, Cp:]
    call = GatRowStatCall(er, ms, stat, mean=(dZ, Yc, W, F1, Cp, 0.25))
    assert call.tc == tc
    call()
    got = stat.reshape(V, 4, 4).cpu().numpy()
    z = dZ.double().cpu().numpy()
    y = Yc.double().cpu().numpy().reshape(V, F1, 4)
    w = W.double().cpu().numpy().reshape(F1, 4, Cp)
    G = np.einsum("ihc,vc->vih", w, z)
    S = 0.25 * np.einsum("vih,vih->vh", y, G)
    Sa = 0.25 * np.einsum("vih,vih->vh", np.abs(y), np.einsum("ihc,vc->vih", np.abs(w), np.abs(z)))
    assert_close(got[:, :, 3], S, Sa, "S")
    assert np.array_equal(got[:, :, 0], er.cpu().numpy())
    assert np.array_equal(got[:, :, 1], ms[:, :4].cpu().numpy())
    assert np.array_equal(got[:, :, 2], ms[:, 4:].cpu().numpy())
