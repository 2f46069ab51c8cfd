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

import os

import numpy as np
import torch

from . import _lib
from .graph import SPMM_SHORT_MAX, SPMM_SORT, SPMM_SORT_MIN_NNZ, CsrGraph
from .kernels import AdamCall, GemmCall, HeadCall, MaskNormColsumCall, SpmmCall, XentCall
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
        return linear(P, self.weight, self.bias, relu=relu)


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
        self.labels = torch.zeros(V, dtype=torch.int64, device=dev)
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
                if (hidden <= 64 and hidden % 4 == 0 and SPMM_SORT and SPMM_SHORT_MAX > 0
                        and min(A.nnz, AT.nnz) >= SPMM_SORT_MIN_NNZ):
                    # every aggregation runs on the degree-sorted forms: keep only those
                    A.release_row_order()
                    AT.release_row_order()
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
        # one strided copy into the padded-stride store (no transient [V, F] buffer);
        # a pageable host source makes the copy synchronous, a pinned one async
        _lib.copy_rows(self.X, X.to(torch.float32) if X.dtype != torch.float32 else X)
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

    # ---- end-to-end step from host memory, copies overlapped with compute
    def capture_e2e(self, X_host: torch.Tensor, labels_host: torch.Tensor,
                    loss_host: torch.Tensor, chunks: int = 8):
        """Record one END-TO-END epoch as a CUDA graph: X and the labels are
        copied from pinned host memory every replay (memcpy nodes on a copy
        stream, X in ``chunks`` row blocks), the first transform X W1 runs on
        each block as soon as it lands, the rest of the epoch follows, and the
        loss is copied back to ``loss_host``.  The H2D transfer (the dominant
        e2e cost: 563 MB at the Reddit shape) overlaps the first GEMM instead
        of preceding the whole epoch.  Replay with ``run_e2e()``."""
        assert X_host.is_pinned() and labels_host.is_pinned() and loss_host.is_pinned()
        V = self.V
        # a host buffer laid out with the device row stride copies as one contiguous block
        dst = self._Xstore if X_host.shape[1] == self.Fpad else self.X
        bounds = [V * i // chunks for i in range(chunks + 1)]
        bounds = [b - b % 128 if 0 < b < V else b for b in bounds]  # tcgen05 M tiles
        gemms = [GemmCall(self.X[b0:b1], self.W1, self.H1[b0:b1])
                 for b0, b1 in zip(bounds[:-1], bounds[1:]) if b1 > b0]
        blocks = [(b0, b1) for b0, b1 in zip(bounds[:-1], bounds[1:]) if b1 > b0]
        main = torch.cuda.Stream(self.dev)
        copy = torch.cuda.Stream(self.dev)
        rest = [c for n, c in self.schedule() if n != "X.W1"]
        head_at = [n for n, _ in self.schedule() if n != "X.W1"].index("head")

        def body(adam=True):
            cur = torch.cuda.current_stream(self.dev)
            copy.wait_stream(cur)
            evs = []
            with torch.cuda.stream(copy):
                ev_lab = torch.cuda.Event()
                self.labels.copy_(labels_host, non_blocking=True)
                ev_lab.record(copy)
                for b0, b1 in blocks:
                    dst.__getitem__(slice(b0, b1)).copy_(X_host[b0:b1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
                    evs.append(ev)
            for ev, gm in zip(evs, gemms):
                cur.wait_event(ev)
                gm()
            for i, call in enumerate(rest):
                if i == head_at:
                    cur.wait_event(ev_lab)
                if call is self.k_adam and not adam:
                    continue
                call()
            loss_host.copy_(self.loss, non_blocking=True)
            cur.wait_stream(copy)

        main.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(main):
            body(adam=False)  # warm-up outside capture (no parameter update)
        torch.cuda.current_stream(self.dev).wait_stream(main)
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        self.graph_e2e = g
        self._e2e_keep = (gemms, main, copy)
        return g

    def run_e2e(self):
        self.graph_e2e.replay()

    # ---- end-to-end, double-buffered inputs: step k's H2D of the NEXT
    # step's inputs runs under step k's compute
    def capture_e2e_pipelined(self, X_host: torch.Tensor, labels_host: torch.Tensor,
                              loss_host: torch.Tensor):
        """Two CUDA graphs over two device input buffers: graph b trains on
        buffer b while a copy stream loads the next step's X / labels from the
        pinned host buffers into buffer 1-b; the loss is read back each step.
        Steady-state step time = max(H2D, epoch) instead of their sum.  Call
        ``prime_e2e()`` once (loads buffer 0), then ``run_e2e_pipelined(k)``
        for k = 0, 1, 2, ..."""
        assert X_host.is_pinned() and labels_host.is_pinned() and loss_host.is_pinned()
        # host X either already [V, Fpad] (one linear DMA: ~53 GB/s on the B200
        # box) or [V, F] (one 2-D DMA into the padded rows: correct, but pitched
        # H2D measured ~16 GB/s — keep the host copy at the device stride)
        assert X_host.shape[1] in (self.F, self.Fpad)
        f32 = dict(dtype=torch.float32, device=self.dev)
        self._Xstore_b = torch.empty(self.V, self.Fpad, **f32)
        self.labels_b = torch.zeros_like(self.labels)
        X_b = self._Xstore_b[:, :self.F]
        stores = [(self._Xstore, self.X, self.labels), (self._Xstore_b, X_b, self.labels_b)]
        self._pipe_host = (X_host, labels_host, loss_host)
        copy = torch.cuda.Stream(self.dev)
        main = torch.cuda.Stream(self.dev)
        graphs, keep = [], []
        for b in (0, 1):
            _, Xb, lab_b = stores[b]
            nxt_store, _, nxt_lab = stores[1 - b]
            k_g1 = GemmCall(Xb, self.W1, self.H1)
            k_dw = GemmCall(Xb, self.dH1, self.dW1, trans_a=True)
            k_hd = HeadCall(self.P2, self.W2, self.b2, lab_b, self.dP2, self.dW2, self.db2,
                            self.loss, deg_offsets=self.g.d_offsets)
            sched = [k_g1, self.k_agg1, self.k_agg2, k_hd, self.k_bagg2, self.k_norm1,
                     self.k_bagg1, k_dw]
            keep.append((k_g1, k_dw, k_hd))

            def body(adam=True, sched=sched, nxt_store=nxt_store, nxt_lab=nxt_lab):
                cur = torch.cuda.current_stream(self.dev)
                copy.wait_stream(cur)  # buffer 1-b is free: the previous step finished
                with torch.cuda.stream(copy):
                    self._load_x(nxt_store, X_host)
                    nxt_lab.copy_(labels_host, non_blocking=True)
                for call in sched:
                    call()
                if adam:
                    self.k_adam()
                loss_host.copy_(self.loss, non_blocking=True)
                cur.wait_stream(copy)

            main.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(main):
                body(adam=False)  # warm-up outside capture (no parameter update)
            torch.cuda.current_stream(self.dev).wait_stream(main)
            torch.cuda.synchronize(self.dev)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                body()
            graphs.append(gr)
        self._pipe = (graphs, keep, copy, main)
        return graphs

    def _load_x(self, store, X_host):
        if X_host.shape[1] == self.Fpad:
            store.copy_(X_host, non_blocking=True)
        else:
            _lib.copy_rows(store[:, :self.F], X_host)

    def prime_e2e(self):
        """Load buffer 0 from the pinned host inputs (stream-ordered)."""
        X_host, labels_host, _ = self._pipe_host
        self._load_x(self._Xstore, X_host)
        self.labels.copy_(labels_host, non_blocking=True)

    def run_e2e_pipelined(self, k: int):
        self._pipe[0][k & 1].replay()

    def params(self):
        return {"W1": self.W1, "b1": self.b1, "W2": self.W2, "b2": self.b2}

    def grads(self):
        return {"W1": self.dW1, "b1": self.db1, "W2": self.dW2, "b2": self.db2}


# ======================================================= sampled mini-batch
class SampledGCNTrainer:
    """Mini-batch 2-layer GCN on sampled subgraphs — the regime the
    reference's sampler and execution model describe (sampler.py:259-305,
    execmodel.py:430-490): per step the seed batch's F-fanout neighbourhood is
    drawn on device (``sample_minibatch``, bit-exact with the reference's
    PCG64 stream), the union of the hop edges (frontier -> drawn neighbour,
    local ids; seeds are locals 0..B-1) forms the local subgraph A_s, the
    feature rows of every sampled vertex are gathered (``gather_features``),
    and the epoch math of ``GCNTrainer`` runs on A_s with the mean
    cross-entropy over the B seeds only (loss rows = the seed batch,
    sampler.py:299-305); Adam updates the shared weights.  Everything runs on
    libgnnb200 kernels.  ``step`` rebuilds its calls per batch (the subgraph
    size changes); ``capture`` + ``run`` make one mini-batch one CUDA-graph
    replay over envelope-sized buffers (no host sync)."""

    def __init__(self, g: CsrGraph, X: torch.Tensor, labels: torch.Tensor, in_feats: int,
                 hidden: int, classes: int, config, *, lr=0.01, seed: int = 0):
        self.g, self.X, self.labels, self.cfg = g, X, labels, config
        dev = g.device
        self.dev = dev
        self.F, self.Hd, self.C = in_feats, hidden, classes
        f32 = dict(dtype=torch.float32, device=dev)
        self.W1 = torch.from_numpy(glorot(in_feats, hidden, seed, 0)).to(dev)
        self.b1 = torch.zeros(hidden, **f32)
        self.W2 = torch.from_numpy(glorot(hidden, classes, seed, 2)).to(dev)
        self.b2 = torch.zeros(classes, **f32)
        self.dW1, self.db1 = torch.empty_like(self.W1), torch.empty_like(self.b1)
        self.dW2, self.db2 = torch.empty_like(self.W2), torch.empty_like(self.b2)
        self.loss = torch.zeros(1, **f32)
        self.k_adam = AdamCall([self.W1, self.b1, self.W2, self.b2],
                               [self.dW1, self.db1, self.dW2, self.db2], lr=lr)
        self.last = None

    def subgraph(self, seeds, rng=None):
        """(local CsrGraph A_s, local->global ids, B) of one sampled batch."""
        from .graph import csr_from_edges
        from .sampling import sample_minibatch

        sg, _ = sample_minibatch(self.g, self.cfg, seeds, rng, on_device=True)
        n = sg.num_local_vertices
        es = torch.cat([h.edge_src for h in sg.hops]) if sg.hops else torch.empty(0)
        ed = torch.cat([h.edge_dst for h in sg.hops]) if sg.hops else torch.empty(0)
        A = csr_from_edges(n, es.to(torch.int64), ed.to(torch.int64), device=self.dev)
        return A, sg.local_to_global, self.cfg.batch_size

    def forward_backward(self, A: CsrGraph, l2g: torch.Tensor, B: int):
        from .sampling import gather_features

        n = A.num_vertices
        f32 = dict(dtype=torch.float32, device=self.dev)
        Xs = gather_features(self.X, l2g)
        ys = self.labels[l2g[:B]]
        e = lambda k: torch.empty(n, k, **f32)  # noqa: E731
        H1, Y1, P2, dZ1, dH1 = e(self.Hd), e(self.Hd), e(self.Hd), e(self.Hd), e(self.Hd)
        dP2 = torch.zeros(n, self.Hd, **f32)  # rows >= B: no loss, zero gradient
        op, opT = A.csr(), A.csc()
        deg = A.d_offsets
        N_, B_, R_, M_ = _lib.EPI_NORM, _lib.EPI_BIAS, _lib.EPI_RELU, _lib.EPI_MASK
        calls = [GemmCall(Xs, self.W1, H1),
                 SpmmCall(op, H1, Y1, flags=N_ | B_ | R_, bias=self.b1),
                 SpmmCall(op, Y1, P2, flags=N_),
                 HeadCall(P2[:B], self.W2, self.b2, ys, dP2[:B], self.dW2, self.db2, self.loss,
                          deg_offsets=deg[:B + 1]),
                 SpmmCall(opT, dP2, dZ1, flags=M_, mask=Y1),
                 MaskNormColsumCall(dZ1, dZ1, deg_offsets=deg, colsum=self.db1),
                 SpmmCall(opT, dZ1, dH1),
                 GemmCall(Xs, dH1, self.dW1, trans_a=True)]
        for c in calls:
            c()
        self.last = (A, l2g, B)
        return self.loss

    def step(self, seeds, rng=None):
        A, l2g, B = self.subgraph(seeds, rng)
        self.forward_backward(A, l2g, B)
        self.k_adam()
        return self.loss

    # ------------------------------------------------------------ replayed form
    def capture(self, adam: bool = True):
        """Make every later ``run`` ONE CUDA-graph replay (
        execmodel.py:430-454 ReplayGraph): device sampling
        (DeviceSampler), the local subgraph — the hop edges concatenated at
        device offsets (already in source order: hop frontiers are consecutive
        local ids, draws frontier-major), CSR offsets from the run boundaries,
        the CSC by a stable radix sort — host-sync-free SpMM schedules
        (gnn_spmm_plan_build_dev), the feature gather, the epoch kernels and
        Adam.  Every buffer is sized for the config's envelope (local vertices
        <= B + sum_h n_cap_h, edges <= sum_h n_cap_h); past the live counts the
        edge lists are padded with a dummy vertex N_cap whose row holds the
        padding edges and never reaches a seed; every kernel stops at the live
        vertex count n (device scalar: SpMM row limit, GEMM live rows, mask /
        norm rows, feature gather), so rows past it cost nothing and stay
        stale, and the math on the live rows is the eager step's (same edge
        order per row)."""
        from .graph import SPMM_SHORT_ROWORDER, SparseOperand
        from .kernels import DevicePlan
        from .sampling import DeviceSampler

        lib, dev = _lib.lib(), self.dev
        S = DeviceSampler(self.g, self.cfg)
        self.sampler = S
        B, nh = self.cfg.batch_size, len(S.hops)
        E_cap = sum(h["n_cap"] for h in S.hops)
        N_cap = B + E_cap
        R = N_cap + 1  # + the dummy vertex
        i32 = dict(dtype=torch.int32, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        self._caps = (B, E_cap, N_cap)
        self._es = torch.full((E_cap,), N_cap, **i32)
        self._ed = torch.full((E_cap,), N_cap, **i32)
        self._l2g = torch.zeros(N_cap, **i64)
        self._cur = torch.zeros(2 * nh + nh + 1, **i64)  # one device cursor per append
        self._n_dev = self._cur[3 * nh]  # live local vertices (the last l2g append's cursor)
        self._csr_off = torch.zeros(R + 1, **i64)
        self._csc_keys, self._csc_cols = torch.empty(E_cap, **i32), torch.empty(E_cap, **i32)
        self._csc_off = torch.zeros(R + 1, **i64)
        self._ws_sort = _lib.workspace(lib.gnn_sort_pairs_workspace(E_cap, R), dev)
        self._ws_off = _lib.workspace(lib.gnn_offsets_from_keys_workspace(R), dev)
        Fpad = -(-self.F // 32) * 32  # 128-byte rows (TMA)
        self._Xs_store = torch.zeros(R, Fpad, **f32)
        Xs = self._Xs_store[:, :self.F]
        self._ys = torch.zeros(B, **i64)
        e = lambda: torch.zeros(R, self.Hd, **f32)  # noqa: E731
        H1, Y1, P2, dZ1, dH1, dP2 = e(), e(), e(), e(), e(), e()  # dP2 rows >= B stay 0
        A = SparseOperand(R, R, self._csr_off, self._ed, deg_offsets=self._csr_off)
        AT = SparseOperand(R, R, self._csc_off, self._csc_cols)
        # rows past the live vertex count are never computed (their values stay
        # stale and no live row reads them): SpMMs, GEMMs and the mask/norm pass
        # all stop at n_dev
        nd = self._n_dev
        # 64-edge warp ranges: the live part (~half the envelope) still spreads
        # over thousands of warps (the CSC's hub rows are long, the rest short)
        self._pA = DevicePlan(A, SPMM_SHORT_ROWORDER, edges_per_warp=64, row_limit=nd)
        self._pAT = DevicePlan(AT, SPMM_SHORT_ROWORDER, edges_per_warp=64, row_limit=nd)
        N_, B_, R_, M_ = _lib.EPI_NORM, _lib.EPI_BIAS, _lib.EPI_RELU, _lib.EPI_MASK
        self._rcalls = [
            GemmCall(Xs, self.W1, H1, rows_dev=nd),
            SpmmCall(A, H1, Y1, flags=N_ | B_ | R_, bias=self.b1, plan=self._pA.plan),
            SpmmCall(A, Y1, P2, flags=N_, plan=self._pA.plan),
            HeadCall(P2[:B], self.W2, self.b2, self._ys, dP2[:B], self.dW2, self.db2, self.loss,
                     deg_offsets=self._csr_off[:B + 1]),
            SpmmCall(AT, dP2, dZ1, flags=M_, mask=Y1, plan=self._pAT.plan),
            MaskNormColsumCall(dZ1, dZ1, deg_offsets=self._csr_off, colsum=self.db1, rows_dev=nd),
            SpmmCall(AT, dZ1, dH1, plan=self._pAT.plan),
            GemmCall(Xs, dH1, self.dW1, trans_a=True, rows_dev=nd)]
        self._Xs, self._replay_adam = Xs, adam
        self._rkeep = (A, AT, H1, Y1, P2, dZ1, dH1, dP2)
        # warm (plans, workspaces), then capture
        S._stage(np.arange(B), 0)
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            self._replay_body()
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        self._graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._graph):
            self._replay_body()
        torch.cuda.synchronize(dev)
        return self._graph

    def _replay_body(self):
        lib, S, dev = _lib.lib(), self.sampler, self.dev
        st = _lib.stream_handle(dev)
        B, E_cap, N_cap = self._caps
        R, nh, cur = N_cap + 1, len(S.hops), self._cur
        S._launch()
        # hop edges at device offsets: hop h after hop h-1's live count; padding -> N_cap
        for k, (dst, key) in enumerate(((self._es, "src_local"), (self._ed, "dst_local"))):
            off_in = None
            for h, hop in enumerate(S.hops):
                off_out = cur[k * nh + h]
                _lib.check(lib.gnn_append_dev(dst.data_ptr(), 4, hop[key].data_ptr(),
                                              hop["count"].data_ptr(), hop["n_cap"],
                                              None if off_in is None else off_in.data_ptr(),
                                              off_out.data_ptr(), st), "append_dev")
                off_in = off_out
            _lib.check(lib.gnn_fill_tail_dev(dst.data_ptr(), 4, off_in.data_ptr(), E_cap, N_cap,
                                             st), "fill_tail_dev")
        # local -> global: seeds, then each hop's new vertices (first-occurrence order)
        segs = [(S.seeds, S.B_dev, B)] + [(h["new_globals"], h["new_count"], h["n_cap"])
                                          for h in S.hops]
        off_in = None
        for i, (src, cnt, cap) in enumerate(segs):
            off_out = cur[2 * nh + i]
            _lib.check(lib.gnn_append_dev(self._l2g.data_ptr(), 8, src.data_ptr(), cnt.data_ptr(),
                                          cap, None if off_in is None else off_in.data_ptr(),
                                          off_out.data_ptr(), st), "append_dev")
            off_in = off_out
        assert off_in.data_ptr() == self._n_dev.data_ptr()  # live local vertex count
        _lib.check(lib.gnn_offsets_from_keys(E_cap, R, self._es.data_ptr(), self._csr_off.data_ptr(),
                                             self._ws_off.data_ptr(), self._ws_off.numel(), st),
                   "offsets_from_keys")
        _lib.check(lib.gnn_sort_pairs(E_cap, R, self._ed.data_ptr(), self._es.data_ptr(),
                                      self._csc_keys.data_ptr(), self._csc_cols.data_ptr(),
                                      self._ws_sort.data_ptr(), self._ws_sort.numel(), st),
                   "sort_pairs")
        _lib.check(lib.gnn_offsets_from_keys(E_cap, R, self._csc_keys.data_ptr(),
                                             self._csc_off.data_ptr(), self._ws_off.data_ptr(),
                                             self._ws_off.numel(), st), "offsets_from_keys")
        self._pA()
        self._pAT()
        _lib.check(lib.gnn_gather_rows_dev(self.X.data_ptr(), self.X.stride(0),
                                           self._l2g.data_ptr(), self._n_dev.data_ptr(), N_cap,
                                           self.F, self._Xs.data_ptr(), self._Xs.stride(0), st),
                   "gather_rows_dev")
        torch.index_select(self.labels, 0, S.seeds, out=self._ys)
        for c in self._rcalls:
            c()
        if self._replay_adam:
            self.k_adam()

    def run(self, seeds, rng=None):
        """One mini-batch as one graph replay (``capture`` first): seeds and the
        per-hop PCG64 states staged in pinned memory, then replayed; no host
        sync.  Returns the device loss tensor."""
        S = self.sampler
        S._stage(seeds, rng)
        self._graph.replay()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev))
        S._inflight = ev
        return self.loss

    def replay_subgraph(self):
        """(offsets, targets, local->global ids, B) of the last replayed batch's
        live subgraph, read back (synchronises) — the eager ``subgraph``'s CSR."""
        torch.cuda.synchronize(self.dev)
        B, E_cap, N_cap = self._caps
        n = int(self._n_dev.item())
        off = self._csr_off[:n + 1].cpu().numpy()
        E = int(off[-1])
        return off, self._ed[:E].cpu().numpy(), self._l2g[:n].cpu().numpy(), B

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
        from .kernels import (AttnProjBwdCall, ColsumCall, EdgeSoftmaxCall, GatBwdCscCall,
                              GatBwdCscMeanCall, HeadMeanCall, MaskNormColsumCall, SddmmCall,
                              SegmentSumCall)

        Wh, a_l, a_r, alpha, el, er, out = ctx.saved_tensors
        g, H = ctx.g, ctx.heads
        V, K = Wh.shape
        F = K // H
        dev = Wh.device
        dout = dout.contiguous()
        db = torch.empty(dout.shape[1], dtype=torch.float32, device=dev)
        A, AT = g.csr(), g.csc(with_eid=True)
        ds = torch.empty(A.nnz, H, dtype=torch.float32, device=dev)
        fused_ok = F % 4 == 0 and H <= 8
        if ctx.relu:
            dY = torch.empty_like(dout)
            MaskNormColsumCall(dout, dY, mask=out, colsum=db)()
        else:
            ColsumCall(dout, db)()
            dY = dout
            if ctx.mean and not (fused_ok and F <= 128):
                dY = torch.empty(V, K, dtype=torch.float32, device=dev)
                HeadMeanCall(dY, dout, H, F, backward=True)()
        if ctx.mean and fused_ok and F <= 128:
            # gathers dZ[v] once per edge for every head (dY = dZ/H broadcast)
            dWh = torch.empty_like(Wh)
            GatBwdCscMeanCall(AT, alpha, dout, Wh, dWh, ds, H)()
        elif K % 4 == 0 and fused_ok and K <= 512:
            # SpMMve^T (alpha via edge-ID) + SDDMM (dalpha) from one gather of dY
            dWh = torch.empty_like(Wh)
            GatBwdCscCall(AT, alpha, dY, Wh, dWh, ds, H)()
        else:
            dWh = spmm_raw(AT, dY, heads=H, vals=alpha, eid=AT.eid)
            SddmmCall(A, dY, Wh, ds, heads=H)()
        EdgeSoftmaxCall(A, H, ds, el=el, er=er, slope=ctx.slope, backward=True, alpha=alpha,
                        dalpha=ds)()                               # ds (in place)
        der = torch.empty(V, H, dtype=torch.float32, device=dev)
        del_ = torch.empty_like(der)
        SegmentSumCall(A, ds, der, H)()
        SegmentSumCall(AT, ds, del_, H, use_eid=True)()
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


# ======================================================= fused trainers (2)
def _parallelize(k: dict, pairs: dict, dev) -> dict:
    """Schedule rewrite: each ``main`` name in ``pairs`` becomes one
    ParallelCall running its listed (mutually independent) side launches on a
    forked stream, at main's position; the side entries leave the list."""
    from .kernels import ParallelCall

    sides = {n for v in pairs.values() for n in v}
    out = {}
    for name, call in k.items():
        if name in sides:
            continue
        if name in pairs:
            calls = [k[n] for n in pairs[name]]

            def side(calls=calls):
                for c in calls:
                    c()
            out["|".join([name] + pairs[name])] = ParallelCall(call, side, dev)
        else:
            out[name] = call
    return out


class _FusedEpoch:
    """Shared driver of the fused full-graph trainers: ``schedule()`` lists
    the epoch's pre-bound launches; ``step()`` runs them eagerly,
    ``capture()`` records one epoch as a CUDA graph that ``run()`` replays."""

    graph = None

    def schedule(self):  # pragma: no cover - abstract
        raise NotImplementedError

    def set_inputs(self, X: torch.Tensor, labels: torch.Tensor, non_blocking: bool = False):
        # one strided copy into the padded-stride store (no transient [V, F] buffer);
        # a pageable host source makes the copy synchronous, a pinned one async
        _lib.copy_rows(self.X, X.to(torch.float32) if X.dtype != torch.float32 else X)
        self.labels.copy_(labels, non_blocking=non_blocking)

    def forward_backward(self):
        for name, call in self.schedule():
            if name != "adam":
                call()

    def step(self):
        for _, call in self.schedule():
            call()
        return self.loss

    def timed_step(self):
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
        out = {}
        for i, (name, _) in enumerate(sched):
            out[name] = out.get(name, 0.0) + ev[i].elapsed_time(ev[i + 1])
        return out

    def capture(self):
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
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


class GATTrainer(_FusedEpoch):
    """Full-graph 2-layer GAT training epoch on libgnnb200 kernels only
    (Appendix A.6; hidden layer = heads x hidden concatenated + ReLU, output
    layer = heads x classes averaged; mean cross-entropy; Adam).

    Forward per layer: Wh = X W (tcgen05 GEMM); el/er = attention
    projections; alpha = edge_softmax(LeakyReLU(el[col] + er[row])) with the
    scores recomputed inside the softmax kernels (never stored); Y =
    SpMMve(A, alpha, Wh) per head (+bias/ReLU in the epilogue, or head mean).
    Backward per layer: SpMMve^T over the CSC reading alpha through the
    edge-ID array (no eShuffle); dalpha = SDDMM(dY, Wh);
    ds = softmax+LeakyReLU backward (in place); der/del = row / column sums
    of ds; projection backward; weight gradient GEMMs.

    The output layer's per-head width is padded to a multiple of 4 (zero
    weight columns, which stay exactly zero: their gradients are zero) so
    every edge kernel takes its float4 path."""

    def __init__(self, g: CsrGraph, in_feats: int, hidden: int, classes: int, heads: int = 4, *,
                 lr=0.01, slope=0.2, seed: int = 0):
        from .kernels import (AttnProjBwdCall, AttnProjCall, ColsumCall, EdgeSoftmaxCall,
                              GatBwdCscCall, GatBwdCscMeanCall, GatBwdRcCall, GatProjGemmCall,
                              GatReluStatGemmCall, GatRowStatCall, GatSoftmaxStatsCall,
                              HeadMeanCall, SegmentSumCall, SharedHeadsCall)

        self.g = g
        dev = g.device
        self.dev = dev
        V, H = g.num_vertices, heads
        self.V, self.F, self.Hd, self.C, self.H = V, in_feats, hidden, classes, heads
        # output-layer per-head width padded to a multiple of 4 (float4 edge
        # kernels); 8 for the 4-head recompute backward (8 lanes per head)
        Cp = -(-classes // 8) * 8 if H == 4 else -(-classes // 4) * 4
        self.Cp = Cp
        f32 = dict(dtype=torch.float32, device=dev)
        K1, K2 = H * hidden, H * Cp
        # ---- parameters (oracle-facing values are the unpadded slices)
        self.W1 = torch.from_numpy(glorot(in_feats, K1, seed, 0)).to(dev)
        self.al1 = torch.from_numpy(glorot_heads(H, hidden, seed, 100)).to(dev)
        self.ar1 = torch.from_numpy(glorot_heads(H, hidden, seed, 200)).to(dev)
        self.b1 = torch.zeros(K1, **f32)
        w2 = glorot(K1, H * classes, seed, 2).reshape(K1, H, classes)
        W2p = np.zeros((K1, H, Cp), np.float32)
        W2p[:, :, :classes] = w2
        self.W2 = torch.from_numpy(W2p.reshape(K1, K2)).to(dev)
        al2 = np.zeros((H, Cp), np.float32)
        ar2 = np.zeros((H, Cp), np.float32)
        al2[:, :classes] = glorot_heads(H, classes, seed, 102)
        ar2[:, :classes] = glorot_heads(H, classes, seed, 202)
        self.al2, self.ar2 = torch.from_numpy(al2).to(dev), torch.from_numpy(ar2).to(dev)
        self.b2 = torch.zeros(Cp, **f32)
        plist = [self.W1, self.al1, self.ar1, self.b1, self.W2, self.al2, self.ar2, self.b2]
        self.grads_ = [torch.zeros_like(p) for p in plist]
        (self.dW1, self.dal1, self.dar1, self.db1, self.dW2, self.dal2, self.dar2,
         self.db2) = self.grads_
        # ---- inputs (X row stride padded to 128 B for TMA)
        self.Fpad = -(-in_feats // 32) * 32
        self._Xstore = torch.zeros(V, self.Fpad, **f32)
        self.X = self._Xstore[:, :in_feats]
        self.labels = torch.zeros(V, dtype=torch.int64, device=dev)
        # ---- activations / state tensors
        A, AT = g.csr(), g.csc(with_eid=True)
        self.A, self.AT = A, AT
        E = A.nnz
        e = lambda *s: torch.empty(*s, **f32)  # noqa: E731
        self.Wh1, self.Y1 = e(V, K1), e(V, K1)
        self.el1, self.er1, self.el2, self.er2 = e(V, H), e(V, H), e(V, H), e(V, H)
        self.alpha1, self.alpha2 = e(E, H), e(E, H)
        # layer-2 aggregation order: with 4 heads, aggregate the shared Y1 row
        # (K1 floats per edge) for every head and transform once after
        # (gnn_spmm_shared_heads + one GEMM) instead of gathering Wh2 (H*Cp)
        self.shared2 = H == 4 and os.environ.get("GNN_GAT_SHARED", "1") != "0"
        self.Wh2 = e(V, K2)
        self.Yc2 = e(V, K1 * H) if self.shared2 else e(V, K2)
        self.Z = torch.zeros(V, Cp, **f32)
        self.dWh2 = e(V, K2)
        self.ds = e(E, H)
        self.der, self.del_ = e(V, H), e(V, H)
        self.dY1, self.dWh1 = e(V, K1), e(V, K1)
        self.loss = torch.zeros(1, **f32)
        # backward form: "rc" recomputes alpha from the forward softmax's row
        # statistics inside one CSC pass per layer (gnn_gat_bwd_rc / _mean: no
        # alpha / dalpha edge-tensor round trip, softmax backward folded in
        # through S = <dY, Yagg>, del in registers, ds stored in CSR edge order
        # so der is one coalesced CSR row sum); else the fused CSC kernel +
        # softmax backward + two segment sums
        self.rc = (H == 4 and self.shared2 and K1 % 32 == 0 and K1 <= 128 and Cp <= 64
                   and os.environ.get("GNN_GAT_RC", "1") != "0")
        # the two gradients the CSC passes gather (dZ, and dY1 masked) keep 16
        # extra floats per row in the recompute form: the row's softmax / backward
        # statistics {er, m, 1/sum, S} per head, gathered with the row
        xs = 16 if self.rc else 0
        self._dZs = torch.zeros(V, Cp + xs, **f32)  # pad columns never written: stay 0
        self.dZ = self._dZs[:, :Cp]
        self._dY1ms = e(V, K1 + xs)
        self.dY1m = self._dY1ms[:, :K1]
        Bf, R = _lib.EPI_BIAS, _lib.EPI_RELU
        k = {}
        # forward
        # layer 1's attention projections ride in the X W1 GEMM's epilogue when the
        # head width is a multiple of 16 (gnn_gemm_gat_proj; 0.72 -> 0.60 ms)
        self.fp = (H == 4 and hidden % 16 == 0 and K1 <= 128 and V >= 128
                   and os.environ.get("GNN_GAT_FUSED_PROJ", "1") != "0")
        if self.fp:
            k["X.W1+proj1"] = GatProjGemmCall(self.X, self.W1, self.Wh1, self.al1, self.ar1,
                                              self.el1, self.er1)
        else:
            k["X.W1"] = GemmCall(self.X, self.W1, self.Wh1)
            k["proj1"] = AttnProjCall(self.Wh1, self.al1, self.ar1, self.el1, self.er1, H)
        if self.rc:
            self.rowstat1, self.rowstat2 = e(V, 2 * H), e(V, 2 * H)
            k["softmax1"] = GatSoftmaxStatsCall(A, H, self.alpha1, self.rowstat1, self.el1,
                                                self.er1, slope)
        else:
            k["softmax1"] = EdgeSoftmaxCall(A, H, self.alpha1, el=self.el1, er=self.er1,
                                            slope=slope)
        k["agg1"] = SpmmCall(A, self.Wh1, self.Y1, flags=Bf | R, heads=H, vals=self.alpha1,
                             bias=self.b1)
        # (layer 2's 192-column transform runs as two column blocks whose epilogue
        # then bounds it: 1.71 ms fused vs 0.99 + 0.46 separate — kept separate)
        k["Y1.W2"] = GemmCall(self.Y1, self.W2, self.Wh2)
        k["proj2"] = AttnProjCall(self.Wh2, self.al2, self.ar2, self.el2, self.er2, H)
        if self.rc:
            k["softmax2"] = GatSoftmaxStatsCall(A, H, self.alpha2, self.rowstat2, self.el2,
                                                self.er2, slope)
        else:
            k["softmax2"] = EdgeSoftmaxCall(A, H, self.alpha2, el=self.el2, er=self.er2,
                                            slope=slope)
        if self.shared2:
            k["agg2"] = SharedHeadsCall(A, self.Y1, self.alpha2, self.Yc2, scale=1.0 / H)
            # rows 4i+h of W2 viewed [K1*H, Cp] = W2[i, h*Cp:(h+1)*Cp]: the head mean
            k["mean2"] = GemmCall(self.Yc2, self.W2.view(K1 * H, Cp), self.Z, bias=self.b2)
        else:
            k["agg2"] = SpmmCall(A, self.Wh2, self.Yc2, heads=H, vals=self.alpha2)
            k["mean2"] = HeadMeanCall(self.Yc2, self.Z, H, Cp, bias=self.b2)
        k["xent"] = XentCall(self.Z[:, :classes], self.labels, self.loss, dZ=self.dZ[:, :classes])
        # backward, layer 2
        k["db2"] = ColsumCall(self.dZ, self.db2)
        if self.rc:
            # S[v,h] = <dZ/H, sum_e alpha Wh2_h[u]> = <dZ, Yc2_h W2_h> (Yc2 carries the
            # 1/H of the head mean already), packed with er / m / inv
            k["stat2"] = GatRowStatCall(self.er2, self.rowstat2, self._dZs[:, Cp:],
                                        mean=(self.dZ, self.Yc2, self.W2, K1, Cp, 1.0))
            k["bagg2+sddmm2"] = GatBwdRcCall(AT, self.el2, self.dZ, self.Wh2, self.dWh2,
                                             self.del_, self.ds, slope=slope, mean_F=Cp,
                                             scale=1.0 / H)
            k["der2"] = SegmentSumCall(A, self.ds, self.der, H)
        else:
            # head-mean layer: the concatenated-head gradient is dZ/H broadcast, so the
            # fused CSC kernel gathers dZ[v] (Cp floats) instead of H*Cp per edge
            k["bagg2+sddmm2"] = GatBwdCscMeanCall(AT, self.alpha2, self.dZ, self.Wh2, self.dWh2,
                                                  self.ds, H)
            k["softmax2_bwd"] = EdgeSoftmaxCall(A, H, self.ds, el=self.el2, er=self.er2,
                                                slope=slope, backward=True, alpha=self.alpha2,
                                                dalpha=self.ds)
            k["der2"] = SegmentSumCall(A, self.ds, self.der, H)
            k["del2"] = SegmentSumCall(AT, self.ds, self.del_, H, use_eid=True)
        k["proj2_bwd"] = AttnProjBwdCall(self.Wh2, self.al2, self.ar2, self.del_, self.der,
                                         self.dWh2, self.dal2, self.dar2, H)
        k["Y1^T.dWh2"] = GemmCall(self.Y1, self.dWh2, self.dW2, trans_a=True)
        # hidden layer's gradient: with the recompute backward and 16-column heads,
        # the GEMM's epilogue applies the ReLU backward and writes the row statistics
        # the CSC pass gathers (gnn_gemm_gat_relu_stat) — dY1 never stored
        self.fr = (self.rc and K1 in (64, 128) and V >= 128
                   and os.environ.get("GNN_GAT_FUSED_STAT", "1") != "0")
        if self.fr:
            k["dWh2.W2^T"] = GatReluStatGemmCall(self.dWh2, self.W2, self._dY1ms, self.Y1, self.b1,
                                                 self.er1, self.rowstat1)
            k["db1"] = ColsumCall(self.dY1m, self.db1)
        else:
            k["dWh2.W2^T"] = GemmCall(self.dWh2, self.W2, self.dY1, trans_b=True)
            # backward, layer 1
            k["relu1_bwd"] = MaskNormColsumCall(self.dY1, self.dY1m, mask=self.Y1, colsum=self.db1)
        if self.rc:
            if not self.fr:
                k["stat1"] = GatRowStatCall(self.er1, self.rowstat1, self._dY1ms[:, K1:],
                                            dYm=self.dY1m, Y=self.Y1, bias=self.b1)
            k["bagg1+sddmm1"] = GatBwdRcCall(AT, self.el1, self.dY1m, self.Wh1, self.dWh1,
                                             self.del_, self.ds, slope=slope)
            k["der1"] = SegmentSumCall(A, self.ds, self.der, H)
        else:
            k["bagg1+sddmm1"] = GatBwdCscCall(AT, self.alpha1, self.dY1m, self.Wh1, self.dWh1,
                                              self.ds, H)
            k["softmax1_bwd"] = EdgeSoftmaxCall(A, H, self.ds, el=self.el1, er=self.er1,
                                                slope=slope, backward=True, alpha=self.alpha1,
                                                dalpha=self.ds)
            k["der1"] = SegmentSumCall(A, self.ds, self.der, H)
            k["del1"] = SegmentSumCall(AT, self.ds, self.del_, H, use_eid=True)
        k["proj1_bwd"] = AttnProjBwdCall(self.Wh1, self.al1, self.ar1, self.del_, self.der,
                                         self.dWh1, self.dal1, self.dar1, H)
        k["X^T.dWh1"] = GemmCall(self.X, self.dWh1, self.dW1, trans_a=True)
        k["adam"] = AdamCall(plist, self.grads_, lr=lr)
        if os.environ.get("GNN_GAT_CONCURRENT", "1") != "0" and self.rc:
            k = _parallelize(k, {"Y1^T.dWh2": ["dWh2.W2^T"]}, dev)
        elif os.environ.get("GNN_GAT_CONCURRENT", "1") != "0":
            # independent pairs run as two graph branches: the CSR row sums
            # (der) beside the CSC column sums (del, random edge-id gathers),
            # and the two weight-gradient-side GEMMs of layer 2
            k = _parallelize(k, {"der2": ["del2"], "der1": ["del1"],
                                 "Y1^T.dWh2": ["dWh2.W2^T"]}, dev)
        self.k = k

    def schedule(self):
        return list(self.k.items())

    def params(self):
        """Unpadded parameters in the oracle's naming (gat2_step)."""
        H, C, Cp, K1 = self.H, self.C, self.Cp, self.H * self.Hd
        return {"W1": self.W1, "al1": self.al1, "ar1": self.ar1, "b1": self.b1,
                "W2": self.W2.reshape(K1, H, Cp)[:, :, :C].reshape(K1, H * C),
                "al2": self.al2[:, :C], "ar2": self.ar2[:, :C], "b2": self.b2[:C]}

    def grads(self):
        H, C, Cp, K1 = self.H, self.C, self.Cp, self.H * self.Hd
        return {"W1": self.dW1, "al1": self.dal1, "ar1": self.dar1, "b1": self.db1,
                "W2": self.dW2.reshape(K1, H, Cp)[:, :, :C].reshape(K1, H * C),
                "al2": self.dal2[:, :C], "ar2": self.dar2[:, :C], "b2": self.db2[:C]}

    def pad_grads(self):
        """Gradients of the padding (must stay exactly zero)."""
        H, C, Cp, K1 = self.H, self.C, self.Cp, self.H * self.Hd
        return [self.dW2.reshape(K1, H, Cp)[:, :, C:], self.dal2[:, C:], self.dar2[:, C:],
                self.db2[C:]]


class GINTrainer(_FusedEpoch):
    """Full-graph 2-layer GIN training epoch (Appendix A.5, eps fixed; hidden
    width ``hidden``; ReLU between layers; mean cross-entropy; Adam) on
    libgnnb200 kernels only.  Each layer's first Linear runs before its
    aggregation (linearity), so both SpMMs of a layer work at the hidden
    width, with the (1+eps) self term, bias and ReLU in the SpMM epilogue:

      H1 = X W1a;  U1 = relu(A H1 + (1+eps) H1 + b1a);  Y1 = relu(U1 W1b + b1b)
      H2 = Y1 W2a; U2 = relu(A H2 + (1+eps) H2 + b2a);  Z  = U2 W2b + b2b
    """

    def __init__(self, g: CsrGraph, in_feats: int, hidden: int, classes: int, *, eps=0.0,
                 lr=0.01, seed: int = 0, coalesced: bool = True):
        self.g = g
        dev = g.device
        self.dev = dev
        V = g.num_vertices
        self.V, self.F, self.Hd, self.C, self.eps = V, in_feats, hidden, classes, float(eps)
        f32 = dict(dtype=torch.float32, device=dev)
        mk = lambda fi, fo, i: torch.from_numpy(glorot(fi, fo, seed, i)).to(dev)  # noqa: E731
        self.W1a, self.W1b = mk(in_feats, hidden, 0), mk(hidden, hidden, 1)
        self.W2a, self.W2b = mk(hidden, hidden, 2), mk(hidden, classes, 3)
        self.b1a, self.b1b = torch.zeros(hidden, **f32), torch.zeros(hidden, **f32)
        self.b2a, self.b2b = torch.zeros(hidden, **f32), torch.zeros(classes, **f32)
        plist = [self.W1a, self.b1a, self.W1b, self.b1b, self.W2a, self.b2a, self.W2b, self.b2b]
        self.grads_ = [torch.zeros_like(p) for p in plist]
        (self.dW1a, self.db1a, self.dW1b, self.db1b, self.dW2a, self.db2a, self.dW2b,
         self.db2b) = self.grads_
        self.Fpad = -(-in_feats // 32) * 32
        self._Xstore = torch.zeros(V, self.Fpad, **f32)
        self.X = self._Xstore[:, :in_feats]
        self.labels = torch.zeros(V, dtype=torch.int64, device=dev)
        e = lambda k: torch.empty(V, k, **f32)  # noqa: E731
        self.H1, self.U1, self.Y1, self.H2, self.U2 = (e(hidden) for _ in range(5))
        self.dU2, self.dH2, self.dY1, self.dU1, self.dH1 = (e(hidden) for _ in range(5))
        self.loss = torch.zeros(1, **f32)
        if coalesced:
            A, AT = g.csr_coalesced(), g.csc_coalesced()
        else:
            A, AT = g.csr(), g.csc()
        self.A, self.AT = A, AT
        S, Bf, R, M = _lib.EPI_SELF, _lib.EPI_BIAS, _lib.EPI_RELU, _lib.EPI_MASK
        s1 = 1.0 + self.eps
        k = {}
        k["X.W1a"] = GemmCall(self.X, self.W1a, self.H1)
        k["agg1"] = SpmmCall(A, self.H1, self.U1, flags=S | Bf | R, self_x=self.H1, self_scale=s1,
                             bias=self.b1a)
        k["U1.W1b"] = GemmCall(self.U1, self.W1b, self.Y1, bias=self.b1b, relu=True)
        k["Y1.W2a"] = GemmCall(self.Y1, self.W2a, self.H2)
        k["agg2"] = SpmmCall(A, self.H2, self.U2, flags=S | Bf | R, self_x=self.H2, self_scale=s1,
                             bias=self.b2a)
        if hidden <= 32:  # fused output layer: weights of <= 32 x C live in registers
            k["head"] = HeadCall(self.U2, self.W2b, self.b2b, self.labels, self.dU2, self.dW2b,
                                 self.db2b, self.loss)
        else:  # wide hidden: the output layer as tensor-core GEMMs + one softmax-CE kernel
            from .kernels import ColsumCall

            Cp = -(-classes // 4) * 4
            self.Z2 = torch.zeros(V, Cp, **f32)
            self.dZ2 = torch.zeros(V, Cp, **f32)
            Z2, dZ2 = self.Z2[:, :classes], self.dZ2[:, :classes]
            k["head.Z"] = GemmCall(self.U2, self.W2b, Z2, bias=self.b2b)
            k["head.xent"] = XentCall(Z2, self.labels, self.loss, dZ=dZ2)
            k["head.dW"] = GemmCall(self.U2, dZ2, self.dW2b, trans_a=True)
            k["head.db"] = ColsumCall(dZ2, self.db2b)
            k["head.dP"] = GemmCall(dZ2, self.W2b, self.dU2, trans_b=True)
        k["relu_bwd_U2"] = MaskNormColsumCall(self.dU2, self.dU2, mask=self.U2, colsum=self.db2a)
        k["bagg2"] = SpmmCall(AT, self.dU2, self.dH2, flags=S, self_x=self.dU2, self_scale=s1)
        k["Y1^T.dH2"] = GemmCall(self.Y1, self.dH2, self.dW2a, trans_a=True)
        k["dH2.W2a^T"] = GemmCall(self.dH2, self.W2a, self.dY1, trans_b=True)
        k["relu_bwd_Y1"] = MaskNormColsumCall(self.dY1, self.dY1, mask=self.Y1, colsum=self.db1b)
        k["U1^T.dY1"] = GemmCall(self.U1, self.dY1, self.dW1b, trans_a=True)
        k["dY1.W1b^T"] = GemmCall(self.dY1, self.W1b, self.dU1, trans_b=True)
        k["relu_bwd_U1"] = MaskNormColsumCall(self.dU1, self.dU1, mask=self.U1, colsum=self.db1a)
        k["bagg1"] = SpmmCall(AT, self.dU1, self.dH1, flags=S, self_x=self.dU1, self_scale=s1)
        k["X^T.dH1"] = GemmCall(self.X, self.dH1, self.dW1a, trans_a=True)
        k["adam"] = AdamCall(plist, self.grads_, lr=lr)
        _ = M
        self.k = k

    def schedule(self):
        return list(self.k.items())

    def params(self):
        return {"W1a": self.W1a, "b1a": self.b1a, "W1b": self.W1b, "b1b": self.b1b,
                "W2a": self.W2a, "b2a": self.b2a, "W2b": self.W2b, "b2b": self.b2b}

    def grads(self):
        return {"W1a": self.dW1a, "b1a": self.db1a, "W1b": self.dW1b, "b1b": self.db1b,
                "W2a": self.dW2a, "b2a": self.db2a, "W2b": self.dW2b, "b2b": self.db2b}
