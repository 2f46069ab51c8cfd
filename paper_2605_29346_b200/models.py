"""GNN layers (autograd) and the fused full-graph GCN trainer.

Layer math follows SURVEY.md Appendix A (GCN A.4, GIN A.5) and the GraphPy
prose: bias is part of the layer, degree-norm fused in the
forward SpMM and applied to the INPUT of the backward SpMM,
state tensors are materialised for backward.

``GCNTrainer`` is the benchmarked hot path: one epoch = forward, loss,
backward and Adam, built only from libgnnb200 kernels with every buffer
preallocated, so the whole epoch is captured in a CUDA graph and replayed.
Layer 2 aggregates before it transforms (A (Y W) = (A Y) W, width 16 < 41)
so every SpMM of the epoch runs at the hidden width.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph
from .kernels import AdamCall, GemmCall, HeadCall, MaskNormColsumCall, SpmmCall
from .ops import colsum, gemm, linear, spmm_raw


def glorot(fan_in: int, fan_out: int, seed: int, index: int = 0) -> np.ndarray:
    """Glorot-uniform weights from SeedSequence(seed, spawn_key=(12, index))
    (SURVEY.md §8d seeding idiom)."""
    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(12, index)))
    a = math.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-a, a, (fan_in, fan_out)).astype(np.float32)


# ------------------------------------------------------------ autograd layer
class _GCNAggregate(torch.autograd.Function):
    """Y = act(D^-1 A H + b) with NORM|BIAS(|RELU) fused in the SpMM epilogue."""

    @staticmethod
    def forward(ctx, H, b, g, relu, coalesced):
        op = g.csr_coalesced() if coalesced else g.csr()
        flags = _lib.EPI_NORM | _lib.EPI_BIAS | (_lib.EPI_RELU if relu else 0)
        Y = spmm_raw(op, H.contiguous(), flags=flags, bias=b.contiguous())
        ctx.save_for_backward(Y if relu else None)
        ctx.g, ctx.relu, ctx.coalesced = g, relu, coalesced
        return Y

    @staticmethod
    def backward(ctx, dY):
        (Y,) = ctx.saved_tensors
        g = ctx.g
        dY = dY.contiguous()
        lib = _lib.lib()
        dev = dY.device
        M, N = dY.shape
        dZn = torch.empty_like(dY)
        db = torch.empty(N, dtype=torch.float32, device=dev)
        ws = _lib.workspace(lib.gnn_mask_norm_colsum_workspace(M, N), dev)
        _lib.check(lib.gnn_mask_norm_colsum(
            M, N, dY.data_ptr(), dY.stride(0), Y.data_ptr() if Y is not None else None,
            Y.stride(0) if Y is not None else 0, g.d_offsets.data_ptr(), dZn.data_ptr(),
            dZn.stride(0), db.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle(dev)),
            "gcn backward")
        op = g.csc_coalesced() if ctx.coalesced else g.csc()
        dH = spmm_raw(op, dZn)
        return dH, db, None, None, None


class GCNConv(torch.nn.Module):
    """GCN layer Z = D^-1 A (X W) + b (Appendix A.4), optional fused ReLU.
    When in_feats < out_feats the aggregation runs first on the narrower side
    (same function)."""

    def __init__(self, in_feats: int, out_feats: int, seed: int = 0, index: int = 0,
                 device=None):
        super().__init__()
        self.in_feats, self.out_feats = in_feats, out_feats
        self.weight = torch.nn.Parameter(torch.from_numpy(glorot(in_feats, out_feats, seed, index)).to(device))
        self.bias = torch.nn.Parameter(torch.zeros(out_feats, device=device))

    def forward(self, g: CsrGraph, X: torch.Tensor, relu: bool = False, coalesced: bool = False):
        if self.in_feats > self.out_feats:
            H = linear(X, self.weight)
            return _GCNAggregate.apply(H, self.bias, g, relu, coalesced)
        from .ops import spmmv

        P = spmmv(g, X, norm=True, coalesced=coalesced)
        Z = linear(P, self.weight, self.bias)
        return torch.relu(Z) if relu else Z


class GCN(torch.nn.Module):
    """Stack of GCNConv layers with ReLU between them."""

    def __init__(self, in_feats: int, hidden: int, classes: int, num_layers: int = 2,
                 seed: int = 0, device=None):
        super().__init__()
        dims = [in_feats] + [hidden] * (num_layers - 1) + [classes]
        self.layers = torch.nn.ModuleList(
            GCNConv(dims[i], dims[i + 1], seed=seed, index=2 * i, device=device)
            for i in range(num_layers))

    def forward(self, g, X, coalesced: bool = False):
        h = X
        for i, layer in enumerate(self.layers):
            h = layer(g, h, relu=i < len(self.layers) - 1, coalesced=coalesced)
        return h


# ----------------------------------------------------------- fused trainer
class GCNTrainer:
    """Full-graph 2-layer GCN training step on libgnnb200 kernels only.

    Schedule of one epoch (all buffers preallocated; ``capture()`` records it
    as one CUDA graph):

      H1  = X W1                               tcgen05 3xTF32 gemm (X streamed by TMA)
      Y1  = relu(D^-1 A H1 + b1)               spmm  (NORM|BIAS|RELU epilogue)
      P2  = D^-1 A Y1                          spmm  (NORM)
      head: Z2 = P2 W2 + b2; loss, dZ2 = xent; fused output layer, one warp per row
            dP2 = D^-1 (dZ2 W2^T); dW2 = P2^T dZ2; db2 = colsum(dZ2)
      dZ1 = (A^T dP2) * [Y1 > 0]               spmm over CSC (MASK epilogue)
      db1 = colsum(dZ1); dZ1 <- D^-1 dZ1       mask_norm_colsum (in place)
      dH1 = A^T dZ1                            spmm over CSC
      dW1 = X^T dH1                            split-K gemm
      Adam(W1,b1,W2,b2)                        adam
    """

    def __init__(self, g: CsrGraph, in_feats: int, hidden: int, classes: int, *, lr=0.01,
                 seed: int = 0, coalesced: bool = False, drop_canonical_csc: bool = False,
                 release_canonical: bool = False):
        self.g = g
        dev = g.device
        self.dev = dev
        V = g.num_vertices
        self.V, self.F, self.Hd, self.C = V, in_feats, hidden, classes
        f32 = dict(dtype=torch.float32, device=dev)
        self.W1 = torch.from_numpy(glorot(in_feats, hidden, seed, 0)).to(dev)
        self.b1 = torch.zeros(hidden, **f32)
        self.W2 = torch.from_numpy(glorot(hidden, classes, seed, 2)).to(dev)
        self.b2 = torch.zeros(classes, **f32)
        self.dW1, self.db1 = torch.empty_like(self.W1), torch.empty_like(self.b1)
        self.dW2, self.db2 = torch.empty_like(self.W2), torch.empty_like(self.b2)
        # X keeps a 128-byte-multiple row stride so TMA can stream it into the
        # tcgen05 GEMM (602 floats = 2408 B is not a 16 B multiple)
        self.Fpad = -(-in_feats // 32) * 32
        self._Xstore = torch.empty(V, self.Fpad, **f32)
        self.X = self._Xstore[:, :in_feats]
        self.labels = torch.empty(V, dtype=torch.int64, device=dev)
        e = lambda k: torch.empty(V, k, **f32)  # noqa: E731
        self.H1, self.Y1, self.P2 = e(hidden), e(hidden), e(hidden)
        self.dP2, self.dZ1, self.dH1 = e(hidden), e(hidden), e(hidden)
        self.loss = torch.zeros(1, **f32)

        if coalesced:
            A, AT = g.csr_coalesced(), g.csc_coalesced()
            if drop_canonical_csc or release_canonical:
                g.drop_csc()
            if release_canonical:  # canonical CSR stays on the host only
                g.release_device_targets()
        else:
            A, AT = g.csr(), g.csc()
        self.A, self.AT = A, AT
        deg_off = g.d_offsets  # out-degree source for every norm
        N, B, R, M = _lib.EPI_NORM, _lib.EPI_BIAS, _lib.EPI_RELU, _lib.EPI_MASK
        self.k_gemm1 = GemmCall(self.X, self.W1, self.H1)
        self.k_agg1 = SpmmCall(A, self.H1, self.Y1, flags=N | B | R, bias=self.b1)
        self.k_agg2 = SpmmCall(A, self.Y1, self.P2, flags=N)
        self.k_head = HeadCall(self.P2, self.W2, self.b2, self.labels, self.dP2, self.dW2,
                               self.db2, self.loss, deg_offsets=deg_off)
        self.k_bagg2 = SpmmCall(AT, self.dP2, self.dZ1, flags=M, mask=self.Y1)
        self.k_norm1 = MaskNormColsumCall(self.dZ1, self.dZ1, deg_offsets=deg_off, colsum=self.db1)
        self.k_bagg1 = SpmmCall(AT, self.dZ1, self.dH1)
        self.k_dW1 = GemmCall(self.X, self.dH1, self.dW1, trans_a=True)
        self.k_adam = AdamCall([self.W1, self.b1, self.W2, self.b2],
                               [self.dW1, self.db1, self.dW2, self.db2], lr=lr)
        self.graph = None

    # kernels launched per epoch (our .so only)
    LAUNCHES_PER_STEP = None

    def set_inputs(self, X: torch.Tensor, labels: torch.Tensor, non_blocking: bool = False):
        self.X.copy_(X, non_blocking=non_blocking)
        self.labels.copy_(labels, non_blocking=non_blocking)

    def forward_backward(self):
        self.k_gemm1()
        self.k_agg1()
        self.k_agg2()
        self.k_head()
        self.k_bagg2()
        self.k_norm1()
        self.k_bagg1()
        self.k_dW1()

    def schedule(self):
        """(name, call) pairs of one epoch, in launch order."""
        return [("X.W1", self.k_gemm1), ("agg1", self.k_agg1), ("agg2", self.k_agg2),
                ("head", self.k_head), ("bagg2", self.k_bagg2), ("mask_norm_db1", self.k_norm1),
                ("bagg1", self.k_bagg1), ("X^T.dH1", self.k_dW1), ("adam", self.k_adam)]

    def step(self):
        self.forward_backward()
        self.k_adam()
        return self.loss

    def timed_step(self):
        """One eager epoch with CUDA events between launches on the launching
        stream (a GPU sleep first lets the host enqueue ahead, so gaps are not
        timed).  Returns {name: ms}."""
        st = torch.cuda.current_stream(self.dev)
        sched = self.schedule()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(sched) + 1)]
        torch.cuda.synchronize(self.dev)
        torch.cuda._sleep(5_000_000)
        ev[0].record(st)
        for i, (_, call) in enumerate(sched):
            call()
            ev[i + 1].record(st)
        torch.cuda.synchronize(self.dev)
        return {name: ev[i].elapsed_time(ev[i + 1]) for i, (name, _) in enumerate(sched)}

    def capture(self):
        """Record one epoch (fwd+bwd+Adam) as a CUDA graph; replay with run()."""
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            # warm the allocator-free path once outside capture
            self.forward_backward()
        torch.cuda.current_stream(self.dev).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step()
        self.graph = g
        return g

    def run(self):
        if self.graph is None:
            return self.step()
        self.graph.replay()
        return self.loss

    def params(self):
        return {"W1": self.W1, "b1": self.b1, "W2": self.W2, "b2": self.b2}

    def grads(self):
        return {"W1": self.dW1, "b1": self.db1, "W2": self.dW2, "b2": self.db2}


# ===================================================================== GAT
class _GATAggregate(torch.autograd.Function):
    """Appendix A.6 aggregation of one GAT layer, given Wh = X W:
    el/er projections, alpha = edge_softmax(LeakyReLU(el[col] + er[row]))
    (scores never materialised), Y = SpMMve(A, alpha, Wh) per head, then
    heads concatenated (+b, optional ReLU — fused in the SpMM epilogue) or
    averaged (+b).  alpha is the saved state tensor."""

    @staticmethod
    def forward(ctx, Wh, a_l, a_r, b, g, heads, mean, relu, slope):
        from .kernels import AttnProjCall, EdgeSoftmaxCall, HeadMeanCall

        Wh = Wh.contiguous()
        V, K = Wh.shape
        F = K // heads
        dev = Wh.device
        el = torch.empty(V, heads, dtype=torch.float32, device=dev)
        er = torch.empty_like(el)
        AttnProjCall(Wh, a_l.contiguous(), a_r.contiguous(), el, er, heads)()
        A = g.csr()
        alpha = torch.empty(A.nnz, heads, dtype=torch.float32, device=dev)
        EdgeSoftmaxCall(A, heads, alpha, el=el, er=er, slope=slope)()
        if mean:
            Yc = spmm_raw(A, Wh, heads=heads, vals=alpha)
            out = torch.empty(V, F, dtype=torch.float32, device=dev)
            HeadMeanCall(Yc, out, heads, F, bias=b.contiguous())()
        else:
            flags = _lib.EPI_BIAS | (_lib.EPI_RELU if relu else 0)
            out = spmm_raw(A, Wh, heads=heads, vals=alpha, flags=flags, bias=b.contiguous())
        ctx.save_for_backward(Wh, a_l, a_r, alpha, el, er, out if relu else None)
        ctx.g, ctx.heads, ctx.mean, ctx.relu, ctx.slope = g, heads, mean, relu, slope
        return out

    @staticmethod
    def backward(ctx, dout):
        from .kernels import (AttnProjBwdCall, ColsumCall, EdgeSoftmaxCall, HeadMeanCall,
                              MaskNormColsumCall, SddmmCall)

        Wh, a_l, a_r, alpha, el, er, out = ctx.saved_tensors
        g, H = ctx.g, ctx.heads
        V, K = Wh.shape
        F = K // H
        dev = Wh.device
        dout = dout.contiguous()
        db = torch.empty(dout.shape[1], dtype=torch.float32, device=dev)
        if ctx.relu:
            dY = torch.empty_like(dout)
            MaskNormColsumCall(dout, dY, mask=out, colsum=db)()
        else:
            ColsumCall(dout, db)()
            if ctx.mean:
                dY = torch.empty(V, K, dtype=torch.float32, device=dev)
                HeadMeanCall(dY, dout, H, F, backward=True)()
            else:
                dY = dout
        A, AT = g.csr(), g.csc(with_eid=True)
        dWh = spmm_raw(AT, dY, heads=H, vals=alpha, eid=AT.eid)  # SpMMve^T, alpha via edge-ID
        ds = torch.empty(A.nnz, H, dtype=torch.float32, device=dev)
        SddmmCall(A, dY, Wh, ds, heads=H)()                       # dalpha
        EdgeSoftmaxCall(A, H, ds, el=el, er=er, slope=ctx.slope, backward=True, alpha=alpha,
                        dalpha=ds)()                               # ds (in place)
        ones = torch.ones(V, H, dtype=torch.float32, device=dev)
        der = spmm_raw(A, ones, heads=H, vals=ds)
        del_ = spmm_raw(AT, ones, heads=H, vals=ds, eid=AT.eid)
        da_l = torch.empty_like(a_l)
        da_r = torch.empty_like(a_r)
        AttnProjBwdCall(Wh, a_l, a_r, del_, der, dWh, da_l, da_r, H)()
        return dWh, da_l, da_r, db, None, None, None, None, None


def glorot_heads(heads: int, F: int, seed: int, index: int) -> np.ndarray:
    """Attention vectors a_l/a_r [heads, F], Glorot-uniform over (F, 1)."""
    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(12, index)))
    a = math.sqrt(6.0 / (F + 1))
    return rng.uniform(-a, a, (heads, F)).astype(np.float32)


class GATConv(torch.nn.Module):
    """GAT layer (Appendix A.6): Wh = X W; per head h, alpha = softmax over
    row v's edges of LeakyReLU(<Wh[u,h], a_l[h]> + <Wh[v,h], a_r[h]>);
    Y_h[v] = sum_e alpha_e Wh[u,h].  ``mean=False`` concatenates heads
    (+bias, optional fused ReLU), ``mean=True`` averages them (+bias)."""

    def __init__(self, in_feats: int, out_feats: int, heads: int, *, mean: bool = False,
                 slope: float = 0.2, seed: int = 0, index: int = 0, device=None):
        super().__init__()
        self.in_feats, self.out_feats, self.heads = in_feats, out_feats, heads
        self.mean, self.slope = mean, slope
        self.weight = torch.nn.Parameter(
            torch.from_numpy(glorot(in_feats, heads * out_feats, seed, index)).to(device))
        self.attn_l = torch.nn.Parameter(
            torch.from_numpy(glorot_heads(heads, out_feats, seed, index + 100)).to(device))
        self.attn_r = torch.nn.Parameter(
            torch.from_numpy(glorot_heads(heads, out_feats, seed, index + 200)).to(device))
        nb = out_feats if mean else heads * out_feats
        self.bias = torch.nn.Parameter(torch.zeros(nb, device=device))

    def forward(self, g: CsrGraph, X: torch.Tensor, relu: bool = False):
        if relu and self.mean:
            raise ValueError("GATConv: fused ReLU is for concatenated (hidden) layers")
        Wh = linear(X, self.weight)
        return _GATAggregate.apply(Wh, self.attn_l, self.attn_r, self.bias, g, self.heads,
                                   self.mean, relu, self.slope)


class GAT(torch.nn.Module):
    """2-layer GAT: hidden layer concatenates heads (ReLU), output averages them."""

    def __init__(self, in_feats: int, hidden: int, classes: int, heads: int = 4, seed: int = 0,
                 device=None):
        super().__init__()
        self.l1 = GATConv(in_feats, hidden, heads, seed=seed, index=0, device=device)
        self.l2 = GATConv(hidden * heads, classes, heads, mean=True, seed=seed, index=2,
                          device=device)

    def forward(self, g, X):
        return self.l2(g, self.l1(g, X, relu=True))


# ===================================================================== GIN
class _GINAggregate(torch.autograd.Function):
    """U = act(A H + (1+eps) H + b): SpMMv without norm, GIN self term, bias
    and ReLU all in the SpMM epilogue.  Backward: dH = A^T dU' + (1+eps) dU'."""

    @staticmethod
    def forward(ctx, H, b, g, eps, relu, coalesced):
        H = H.contiguous()
        op = g.csr_coalesced() if coalesced else g.csr()
        flags = _lib.EPI_SELF | _lib.EPI_BIAS | (_lib.EPI_RELU if relu else 0)
        U = spmm_raw(op, H, flags=flags, bias=b.contiguous(), self_x=H, self_scale=1.0 + eps)
        ctx.save_for_backward(U if relu else None)
        ctx.g, ctx.eps, ctx.relu, ctx.coalesced = g, eps, relu, coalesced
        return U

    @staticmethod
    def backward(ctx, dU):
        from .kernels import ColsumCall, MaskNormColsumCall

        (U,) = ctx.saved_tensors
        g = ctx.g
        dU = dU.contiguous()
        db = torch.empty(dU.shape[1], dtype=torch.float32, device=dU.device)
        if ctx.relu:
            dUm = torch.empty_like(dU)
            MaskNormColsumCall(dU, dUm, mask=U, colsum=db)()
        else:
            ColsumCall(dU, db)()
            dUm = dU
        op = g.csc_coalesced() if ctx.coalesced else g.csc()
        dH = spmm_raw(op, dUm, flags=_lib.EPI_SELF, self_x=dUm, self_scale=1.0 + ctx.eps)
        return dH, db, None, None, None, None


class GINConv(torch.nn.Module):
    """GIN layer (Appendix A.5): Z = MLP((1+eps) X + A X), MLP = Linear ->
    ReLU -> Linear.  By linearity the first Linear runs before the
    aggregation, so the SpMM works at the hidden width:
    ((1+eps) X + A X) W1 = (1+eps) X W1 + A (X W1)."""

    def __init__(self, in_feats: int, hidden: int, out_feats: int, eps: float = 0.0, seed: int = 0,
                 index: int = 0, device=None):
        super().__init__()
        self.eps = float(eps)
        self.w1 = torch.nn.Parameter(torch.from_numpy(glorot(in_feats, hidden, seed, index)).to(device))
        self.b1 = torch.nn.Parameter(torch.zeros(hidden, device=device))
        self.w2 = torch.nn.Parameter(torch.from_numpy(glorot(hidden, out_feats, seed, index + 1)).to(device))
        self.b2 = torch.nn.Parameter(torch.zeros(out_feats, device=device))

    def forward(self, g: CsrGraph, X: torch.Tensor, coalesced: bool = False, relu: bool = False):
        H = linear(X, self.w1)
        U = _GINAggregate.apply(H, self.b1, g, self.eps, True, coalesced)
        return linear(U, self.w2, self.b2, relu=relu)


class GIN(torch.nn.Module):
    """2-layer GIN with ReLU between layers."""

    def __init__(self, in_feats: int, hidden: int, classes: int, eps: float = 0.0, seed: int = 0,
                 device=None):
        super().__init__()
        self.l1 = GINConv(in_feats, hidden, hidden, eps, seed=seed, index=0, device=device)
        self.l2 = GINConv(hidden, hidden, classes, eps, seed=seed, index=2, device=device)

    def forward(self, g, X, coalesced: bool = False):
        return self.l2(g, self.l1(g, X, coalesced, relu=True), coalesced)
