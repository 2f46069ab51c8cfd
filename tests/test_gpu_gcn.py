"""GPU parity: the fused GCN trainer and the autograd GCN layers vs the
float64 oracle (loss and all parameter gradients, normwise 1e-5)."""

import numpy as np
import pytest
import torch

from oracle import graph as og
from oracle import ops as oo

pytestmark = pytest.mark.gpu


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-30))


@pytest.fixture(scope="module")
def setup(cuda):
    import paper_2605_29346_b200 as gb

    V, E, F, Hd, C = 2708, 10556, 1433, 16, 7   # Cora shape (BASELINE configs[0])
    g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
    off, tgt = g.offsets, g.targets
    t_off, t_rows, _ = og.transpose(V, V, off, tgt)
    rng = np.random.default_rng(np.random.SeedSequence(0, spawn_key=(10,)))
    X = rng.uniform(-1, 1, (V, F)).astype(np.float32)
    y = np.random.default_rng(np.random.SeedSequence(0, spawn_key=(13,))).integers(0, C, V)
    return gb, g, (off, tgt, t_off, t_rows), X, y, (V, F, Hd, C)


@pytest.mark.parametrize("coalesced,sort_all", [(False, False), (True, False), (False, True),
                                               (True, True)])
def test_trainer_matches_oracle(setup, coalesced, sort_all, monkeypatch):
    """sort_all: the degree-sorted SpMM operands even at this small size (the
    default keeps operands under SPMM_SORT_MIN_NNZ entries in row order)."""
    import paper_2605_29346_b200.graph as G
    from paper_2605_29346_b200.models import GCNTrainer

    if sort_all:
        monkeypatch.setattr(G, "SPMM_SORT_MIN_NNZ", 0)
    gb, g, (off, tgt, t_off, t_rows), X, y, (V, F, Hd, C) = setup
    tr = GCNTrainer(g, F, Hd, C, seed=0, coalesced=coalesced)
    assert (tr.k_agg1.view.row_ids is not None) == sort_all
    tr.set_inputs(torch.from_numpy(X), torch.from_numpy(y))
    tr.forward_backward()
    torch.cuda.synchronize()
    p = {k: v.cpu().numpy().astype(np.float64) for k, v in tr.params().items()}
    ref = oo.gcn2_step(off, tgt, t_off, t_rows, X, p["W1"], p["b1"], p["W2"], p["b2"], y)
    assert abs(tr.loss.item() - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    for k, gv in tr.grads().items():
        ok, worst = oo.close(gv.cpu().numpy(), ref[k], ref["abs"][k])
        assert ok, (k, worst)


def test_graph_replay_equals_eager(setup):
    from paper_2605_29346_b200.models import GCNTrainer

    gb, g, _, X, y, (V, F, Hd, C) = setup
    a = GCNTrainer(g, F, Hd, C, seed=0)
    b = GCNTrainer(g, F, Hd, C, seed=0)
    for t in (a, b):
        t.set_inputs(torch.from_numpy(X), torch.from_numpy(y))
    b.capture()
    la, lb = [], []
    for _ in range(4):
        la.append(a.step().item())
        lb.append(b.run().item())
    assert la == lb
    for k in a.params():
        assert torch.equal(a.params()[k], b.params()[k])
    assert la[-1] < la[0]  # Adam makes progress


def test_autograd_layers_match_oracle(setup):
    from paper_2605_29346_b200.models import GCN

    gb, g, (off, tgt, t_off, t_rows), X, y, (V, F, Hd, C) = setup
    model = GCN(F, Hd, C, seed=0, device="cuda")
    Xd = torch.from_numpy(X).cuda()
    logits = model(g, Xd)
    W1 = model.layers[0].weight.detach().double().cpu().numpy()
    W2 = model.layers[1].weight.detach().double().cpu().numpy()
    b1 = np.zeros(Hd)
    b2 = np.zeros(C)
    ref = oo.gcn2_step(off, tgt, t_off, t_rows, X, W1, b1, W2, b2, y)
    assert rel_err(logits.detach().cpu().numpy(), ref["logits"]) <= 1e-5
    # backward of the same mean cross-entropy through our autograd ops
    Z = logits
    dZ = torch.from_numpy(oo.cross_entropy(ref["logits"], y)[1].astype(np.float32)).cuda()
    Z.backward(dZ)
    for got, k in ((model.layers[0].weight.grad, "W1"), (model.layers[1].weight.grad, "W2"),
                   (model.layers[0].bias.grad, "b1"), (model.layers[1].bias.grad, "b2")):
        ok, worst = oo.close(got.cpu().numpy(), ref[k], ref["abs"][k])
        assert ok, (k, worst)


def test_e2e_graph_matches_device_resident_epoch(setup):
    """capture_e2e (chunked H2D overlapped with X W1, loss copied back) trains
    exactly like the device-resident epoch."""
    from paper_2605_29346_b200.models import GCNTrainer

    gb, g, _, X, y, (V, F, Hd, C) = setup
    a = GCNTrainer(g, F, Hd, C, seed=0)
    b = GCNTrainer(g, F, Hd, C, seed=0)
    a.set_inputs(torch.from_numpy(X), torch.from_numpy(y))
    Xp = torch.zeros(V, b.Fpad).pin_memory()
    Xp[:, :F].copy_(torch.from_numpy(X))
    yh = torch.from_numpy(y).pin_memory()
    loss_h = torch.zeros(1).pin_memory()
    b.capture_e2e(Xp, yh, loss_h, chunks=4)
    for _ in range(3):
        la = a.step().item()
        b.run_e2e()
        torch.cuda.synchronize()
        assert la == loss_h.item()
    for k in a.params():
        assert torch.equal(a.params()[k], b.params()[k])


@pytest.mark.parametrize("padded", [True, False])
def test_e2e_pipelined_matches_device_resident_epoch(setup, padded):
    """Double-buffered e2e graphs (next step's inputs loaded under this step's
    compute) train exactly like the device-resident epoch; the host X is
    either at the device row stride or the user's [V, F] array (2-D DMA)."""
    from paper_2605_29346_b200.models import GCNTrainer

    gb, g, _, X, y, (V, F, Hd, C) = setup
    a = GCNTrainer(g, F, Hd, C, seed=0)
    b = GCNTrainer(g, F, Hd, C, seed=0)
    a.set_inputs(torch.from_numpy(X), torch.from_numpy(y))
    if padded:
        Xp = torch.zeros(V, b.Fpad).pin_memory()
        Xp[:, :F].copy_(torch.from_numpy(X))
    else:
        Xp = torch.from_numpy(np.ascontiguousarray(X)).pin_memory()
    yh = torch.from_numpy(y).pin_memory()
    loss_h = torch.zeros(1).pin_memory()
    b.capture_e2e_pipelined(Xp, yh, loss_h)
    b.prime_e2e()
    for k in range(4):
        la = a.step().item()
        b.run_e2e_pipelined(k)
        torch.cuda.synchronize()
        assert la == loss_h.item(), k
    for k2 in a.params():
        assert torch.equal(a.params()[k2], b.params()[k2])


def test_trainer_with_released_row_order_operands(setup, monkeypatch):
    """release_canonical=True keeps only the degree-sorted coalesced operands
    on the device (the row-order arrays are freed); the epoch is unchanged —
    bit-identical to the trainer that still holds both forms."""
    import paper_2605_29346_b200 as gbm
    import paper_2605_29346_b200.graph as G
    import paper_2605_29346_b200.models as Mo
    from paper_2605_29346_b200.models import GCNTrainer

    monkeypatch.setattr(G, "SPMM_SORT_MIN_NNZ", 0)
    monkeypatch.setattr(Mo, "SPMM_SORT_MIN_NNZ", 0)
    gb, g0, (off, tgt, t_off, t_rows), X, y, (V, F, Hd, C) = setup
    g = gbm.generate(gbm.GraphGenSpec("power-law", V, 10556, exponent=2.1), 42)
    a = GCNTrainer(g0, F, Hd, C, seed=0, coalesced=True)
    b = GCNTrainer(g, F, Hd, C, seed=0, coalesced=True, release_canonical=True)
    assert getattr(g.csr_coalesced(), "_released", False) and g.csr_coalesced().packed is None
    with pytest.raises(RuntimeError):
        g.csr_coalesced().view()
    for t in (a, b):
        t.set_inputs(torch.from_numpy(X), torch.from_numpy(y))
        t.forward_backward()
    torch.cuda.synchronize()
    assert torch.equal(a.loss, b.loss)
    for k, v in a.grads().items():
        assert torch.equal(v, b.grads()[k]), k


@pytest.mark.parametrize("fused", [True, False])
def test_trainer_wide_output_layer_matches_oracle(cuda, fused, monkeypatch):
    """172 classes (the papers100M shape): the fused wide output layer (class
    chunks, online softmax, no [V, C] logits) and, with the fused head turned
    off, the library-call composition (GEMM + softmax-CE + colsum + GEMMs +
    degree norm); the epoch matches the float64 oracle either way."""
    import paper_2605_29346_b200 as gb
    from paper_2605_29346_b200.kernels import HeadCall
    from paper_2605_29346_b200.models import GCNTrainer

    if not fused:
        monkeypatch.setattr(HeadCall, "FUSED_MAX", 0)

    V, E, F, Hd, C = 3000, 20000, 64, 16, 172
    g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 7)
    off, tgt = g.offsets, g.targets
    t_off, t_rows, _ = og.transpose(V, V, off, tgt)
    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (V, F)).astype(np.float32)
    y = rng.integers(0, C, V)
    for coalesced in (False, True):
        tr = GCNTrainer(g, F, Hd, C, seed=0, coalesced=coalesced)
        assert tr.k_head.fused == fused
        tr.set_inputs(torch.from_numpy(X), torch.from_numpy(y))
        tr.forward_backward()
        torch.cuda.synchronize()
        p = {k: v.cpu().numpy().astype(np.float64) for k, v in tr.params().items()}
        ref = oo.gcn2_step(off, tgt, t_off, t_rows, X, p["W1"], p["b1"], p["W2"], p["b2"], y)
        assert abs(tr.loss.item() - ref["loss"]) <= 1e-5 * abs(ref["loss"])
        for k, gv in tr.grads().items():
            ok, worst = oo.close(gv.cpu().numpy(), ref[k], ref["abs"][k])
            assert ok, (coalesced, k, worst)
