"""The torch.library registration of the hot-path operators
(paper_2605_29346_b200.torch_ops): schemas on CPU; on the GPU, forward and
backward through torch.ops.gnnb200.* equal the plain functions (same kernels),
the fake kernels give the right shapes, and torch.library.opcheck passes."""

import numpy as np
import pytest
import torch


def test_ops_registered():
    import paper_2605_29346_b200  # noqa: F401

    for name, args in (("spmmv", ["X", "graph", "norm", "transpose", "coalesced"]),
                       ("spmmve", ["X", "ev", "graph", "transpose"]),
                       ("sddmm", ["X", "Y", "graph", "heads"])):
        schema = getattr(torch.ops.gnnb200, name).default._schema
        assert [a.name for a in schema.arguments] == args


@pytest.fixture(scope="module")
def env(cuda):
    import paper_2605_29346_b200 as gb

    g = gb.generate(gb.GraphGenSpec("power-law", 3000, 40_000, exponent=2.1), 9)
    return gb, g, gb.register_graph(g)


@pytest.mark.gpu
@pytest.mark.parametrize("norm,transpose,coalesced", [(False, False, False), (True, False, False),
                                                      (False, True, False), (True, True, True)])
def test_spmmv_op_matches_function(env, norm, transpose, coalesced):
    gb, g, h = env
    X = torch.randn(g.num_vertices, 16, device="cuda", requires_grad=True)
    Y = torch.ops.gnnb200.spmmv(X, h, norm, transpose, coalesced)
    X2 = X.detach().clone().requires_grad_(True)
    Y2 = gb.spmmv(g, X2, norm=norm, transpose=transpose, coalesced=coalesced)
    assert torch.equal(Y, Y2)
    G = torch.randn_like(Y)
    Y.backward(G)
    Y2.backward(G)
    assert torch.equal(X.grad, X2.grad)


@pytest.mark.gpu
@pytest.mark.parametrize("heads", [1, 4])
@pytest.mark.parametrize("transpose", [False, True])
def test_spmmve_and_sddmm_ops(env, heads, transpose):
    gb, g, h = env
    K = 8 * heads
    X = torch.randn(g.num_vertices, K, device="cuda", requires_grad=True)
    ev = torch.rand(g.num_edges, heads, device="cuda", requires_grad=True)
    Y = torch.ops.gnnb200.spmmve(X, ev, h, transpose)
    X2, ev2 = X.detach().clone().requires_grad_(True), ev.detach().clone().requires_grad_(True)
    Y2 = gb.spmmve(g, X2, ev2, transpose=transpose)
    assert torch.equal(Y, Y2)
    G = torch.randn_like(Y)
    Y.backward(G)
    Y2.backward(G)
    assert torch.equal(X.grad, X2.grad) and torch.equal(ev.grad, ev2.grad)
    # sddmm forward + its backward (SpMMve over A and A^T) against torch on the host
    from paper_2605_29346_b200.sparse_attn import sddmm

    A = torch.randn(g.num_vertices, K, device="cuda", requires_grad=True)
    B = torch.randn(g.num_vertices, K, device="cuda", requires_grad=True)
    S = torch.ops.gnnb200.sddmm(A, B, h, heads)
    assert torch.equal(S, sddmm(g, A.detach(), B.detach(), heads=heads))
    D = torch.randn_like(S)
    S.backward(D)
    rows = np.repeat(np.arange(g.num_vertices), np.diff(g.offsets))
    cols = np.asarray(g.targets, np.int64)
    d = D.double().cpu().numpy()
    Bh, Ah = B.detach().double().cpu().numpy(), A.detach().double().cpu().numpy()
    F = K // heads
    dA = np.zeros_like(Ah)
    np.add.at(dA, rows, (d[:, :, None] * Bh[cols].reshape(-1, heads, F)).reshape(-1, K))
    dB = np.zeros_like(Bh)
    np.add.at(dB, cols, (d[:, :, None] * Ah[rows].reshape(-1, heads, F)).reshape(-1, K))
    assert np.allclose(A.grad.cpu().numpy(), dA, rtol=1e-4, atol=1e-4)
    assert np.allclose(B.grad.cpu().numpy(), dB, rtol=1e-4, atol=1e-4)


@pytest.mark.gpu
def test_opcheck_and_fake(env):
    gb, g, h = env
    X = torch.randn(g.num_vertices, 16, device="cuda")
    ev = torch.rand(g.num_edges, 4, device="cuda")
    for op, args in ((torch.ops.gnnb200.spmmv.default, (X, h, True, False, False)),
                     (torch.ops.gnnb200.spmmve.default, (X, ev, h, True)),
                     (torch.ops.gnnb200.sddmm.default, (X, X, h, 4))):
        torch.library.opcheck(op, args, test_utils=("test_schema", "test_faketensor",
                                                    "test_autograd_registration"))
    from torch._subclasses.fake_tensor import FakeTensorMode

    with FakeTensorMode() as m:
        Xf = m.from_tensor(X)
        assert torch.ops.gnnb200.spmmv(Xf, h, False, False, False).shape == X.shape
        assert torch.ops.gnnb200.sddmm(Xf, Xf, h, 4).shape == (g.num_edges, 4)
