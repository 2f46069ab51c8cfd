"""Pre-bound kernel launches for the fused training engines.

Each ``*Call`` object resolves its C-ABI arguments (views, plans, epilogue,
workspace) once; ``__call__`` only reads the current CUDA stream and launches,
so a step built from these objects is cheap on the host and capturable in a
CUDA graph (no allocation, no host sync inside).
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib
from .graph import SparseOperand, spmm_operand


_L2_STATE = {}


def l2_hot_window(X) -> int:
    """Bytes of a persisting-L2 window over the gathered array's low-id prefix
    (GNN_L2_PERSIST_MB, default 48 MB; measured best on the papers100M shape),
    for arrays at least twice the size of L2 only: with a degree-ordered
    numbering (the power-law generator's hubs are its low ids) the prefix holds
    the rows most gathered, and pinning it keeps the streaming tail from
    evicting them.  0 = no window."""
    mb = int(os.environ.get("GNN_L2_PERSIST_MB", "48"))
    if mb <= 0 or X.device.type != "cuda":
        return 0
    dev = X.device.index if X.device.index is not None else torch.cuda.current_device()
    if dev not in _L2_STATE:
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        _L2_STATE[dev] = l2
        _lib.lib().gnn_l2_persist_limit(mb << 20)
    if int(X.shape[0]) * X.stride(0) * X.element_size() <= 2 * _L2_STATE[dev]:
        return 0
    return mb << 20


class _L2Window:
    """Sets / clears a stream's access-policy window around one launch (kept in
    the launches' kernel nodes when captured into a CUDA graph)."""

    def __init__(self, lib, X):
        self.lib, self.X, self.n = lib, X, l2_hot_window(X)

    def __enter__(self):
        if self.n:
            self.lib.gnn_l2_window(_lib.stream_handle(self.X.device), self.X.data_ptr(), self.n, 1.0)

    def __exit__(self, *exc):
        if self.n:
            self.lib.gnn_l2_window(_lib.stream_handle(self.X.device), None, 0, 0.0)


class SpmmCall:
    def __init__(self, op: SparseOperand, X: torch.Tensor, Y: torch.Tensor, *, flags=0, heads=1,
                 vals=None, eid=None, bias=None, self_x=None, self_scale=1.0, mask=None,
                 post_deg_offsets=None, edges_per_warp=None, plan=None):
        """``plan``: a prebuilt (e.g. device-count, DevicePlan.plan) schedule for
        ``op`` itself — the operand is then used as given (no degree-sorted form)."""
        self.lib = _lib.lib()
        self.dev = X.device
        self.K = int(X.shape[1])
        assert Y.shape[1] == self.K and X.stride(1) == 1 and Y.stride(1) == 1
        if plan is None:
            op = spmm_operand(op, X, Y, heads=heads, vals=vals, eid=eid, self_x=self_x, mask=mask,
                              bias=bias)
        self.view = op.view(vals=vals, eid=eid)
        self.plan = plan if plan is not None else op.spmm_plan(edges_per_warp)
        self.epi = _lib.Epilogue()
        self.epi.flags = flags
        self.epi.self_scale = float(self_scale)
        if self_x is not None:
            self.epi.self_x, self.epi.ld_self = self_x.data_ptr(), self_x.stride(0)
        if bias is not None:
            self.epi.bias = bias.data_ptr()
        if mask is not None:
            self.epi.mask, self.epi.ld_mask = mask.data_ptr(), mask.stride(0)
        if post_deg_offsets is not None:
            self.epi.post_deg_offsets = post_deg_offsets.data_ptr()
        self.heads = heads
        self.X, self.Y = X, Y
        self._keep = (op, vals, eid, bias, self_x, mask, post_deg_offsets)
        nbytes = self.lib.gnn_spmm_workspace(C.byref(self.view), C.byref(self.plan), self.K)
        self.ws = _lib.workspace(nbytes, self.dev)
        self.l2 = _L2Window(self.lib, X)  # hub-prefix persisting window (large X only)

    def __call__(self):
        with self.l2:
            _lib.check(self.lib.gnn_spmm(C.byref(self.view), C.byref(self.plan), self.heads,
                                         self.X.data_ptr(), self.X.stride(0), self.Y.data_ptr(),
                                         self.Y.stride(0), self.K, C.byref(self.epi),
                                         self.ws.data_ptr(), self.ws.numel(),
                                         _lib.stream_handle(self.dev)), "spmm")


class DevicePlan:
    """Host-sync-free SpMM schedule of an operand whose rows change in place
    (gnn_spmm_plan_build_dev): fixed buffers, counts on device; ``__call__``
    rebuilds it for the operand's current offsets (capturable)."""

    def __init__(self, op: SparseOperand, short_max: int, edges_per_warp: int | None = None,
                 row_limit: torch.Tensor | None = None):
        """``row_limit``: device int64 scalar, the live rows (rows past it are
        not computed by the SpMMs run on this plan)."""
        from .graph import _default_edges_per_warp

        self.lib = _lib.lib()
        self.dev = op.device
        if edges_per_warp is None:
            with torch.cuda.device(self.dev):
                edges_per_warp = _default_edges_per_warp(op.nnz, self.lib.gnn_device_sm_count())
        R = op.num_rows
        nint = self.lib.gnn_spmm_plan_buffer_ints(R, op.nnz, edges_per_warp)
        self.buf = torch.zeros(max(int(nint), 1), dtype=torch.int32, device=self.dev)
        self.counts = torch.zeros(4, dtype=torch.int64, device=self.dev)
        self.ws = _lib.workspace(self.lib.gnn_spmm_plan_workspace(R), self.dev)
        self.view = op.view()
        self.P, self.short_max, self.op = int(edges_per_warp), int(short_max), op
        self.row_limit = row_limit
        self.plan = _lib.SpmmPlan()
        self()  # fills the plan's capacities and pointers (fixed from now on)

    def __call__(self):
        _lib.check(self.lib.gnn_spmm_plan_build_dev(
            C.byref(self.view), self.P, self.short_max, self.buf.data_ptr(), C.byref(self.plan),
            self.counts.data_ptr(),
            self.row_limit.data_ptr() if self.row_limit is not None else None,
            self.ws.data_ptr(), self.ws.numel(),
            _lib.stream_handle(self.dev)), "spmm plan (device counts)")


class SharedHeadsCall:
    """Y[:, 4i+h] = scale * sum_e vals[e, h] X[col_e, i] (gnn_spmm_shared_heads):
    four heads aggregated over one shared feature row."""

    def __init__(self, op: SparseOperand, X, vals, Y, scale=1.0):
        self.lib = _lib.lib()
        self.dev = X.device
        self.F = int(X.shape[1])
        assert Y.shape[1] == 4 * self.F and vals.shape[-1] == 4
        self.view = op.view(vals=vals)
        self.plan = op.plan()
        self.X, self.Y, self.scale = X, Y, float(scale)
        self.epi = _lib.Epilogue()
        self._keep = (op, vals)
        nbytes = self.lib.gnn_spmm_workspace(C.byref(self.view), C.byref(self.plan), 4 * self.F)
        self.ws = _lib.workspace(nbytes, self.dev)

    def __call__(self):
        if not hasattr(self, "l2"):
            self.l2 = _L2Window(self.lib, self.X)
        with self.l2:
            _lib.check(self.lib.gnn_spmm_shared_heads(
                C.byref(self.view), C.byref(self.plan), self.X.data_ptr(), self.X.stride(0),
                self.F, self.Y.data_ptr(), self.Y.stride(0), self.scale, C.byref(self.epi),
                self.ws.data_ptr(), self.ws.numel(), _lib.stream_handle(self.dev)),
                "spmm_shared_heads")


class ParallelCall:
    """Two independent launches: ``side`` on a forked stream, ``main`` on the
    current one, joined before returning (fork/join events; capturable into
    the epoch's CUDA graph as two branches)."""

    def __init__(self, main, side, dev):
        self.main, self.side = main, side
        self.stream = torch.cuda.Stream(dev)

    def __call__(self):
        cur = torch.cuda.current_stream(self.stream.device)
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            self.side()
        self.main()
        cur.wait_stream(self.stream)


class GemmCall:
    """C = op(A) op(B) (+bias)(relu).  ``rows_dev``: device int64 scalar of live
    rows (C rows, or the contraction rows of A^T B) of capacity-sized operands."""

    def __init__(self, A, B, Cout, *, trans_a=False, trans_b=False, bias=None, relu=False,
                 rows_dev=None):
        self.lib = _lib.lib()
        self.dev = A.device
        self.M = A.shape[1] if trans_a else A.shape[0]
        self.Kd = A.shape[0] if trans_a else A.shape[1]
        self.N = B.shape[0] if trans_b else B.shape[1]
        assert tuple(Cout.shape) == (self.M, self.N)
        self.A, self.B, self.C, self.bias = A, B, Cout, bias
        self.ta, self.tb, self.relu = int(trans_a), int(trans_b), int(relu)
        self.ws = _lib.workspace(self.lib.gnn_gemm_workspace(self.M, self.N, self.Kd, self.ta),
                                 self.dev)
        self.rows_dev = rows_dev

    def __call__(self):
        if self.rows_dev is not None:
            _lib.check(self.lib.gnn_gemm_rows_dev(
                self.M, self.N, self.Kd, self.A.data_ptr(), self.A.stride(0), self.ta,
                self.B.data_ptr(), self.B.stride(0), self.tb, self.C.data_ptr(), self.C.stride(0),
                self.bias.data_ptr() if self.bias is not None else None, self.relu,
                self.rows_dev.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                _lib.stream_handle(self.dev)), "gemm (device rows)")
            return
        _lib.check(self.lib.gnn_gemm(self.M, self.N, self.Kd, self.A.data_ptr(),
                                     self.A.stride(0), self.ta, self.B.data_ptr(),
                                     self.B.stride(0), self.tb, self.C.data_ptr(),
                                     self.C.stride(0),
                                     self.bias.data_ptr() if self.bias is not None else None,
                                     self.relu, self.ws.data_ptr(), self.ws.numel(),
                                     _lib.stream_handle(self.dev)), "gemm")


class MaskNormColsumCall:
    def __init__(self, X, out, *, mask=None, deg_offsets=None, colsum=None, rows_dev=None):
        self.lib = _lib.lib()
        self.dev = X.device
        self.M, self.N = X.shape
        self.X, self.out, self.mask, self.deg, self.colsum = X, out, mask, deg_offsets, colsum
        self.rows_dev = rows_dev  # device int64 scalar: live rows of a capacity buffer
        self.ws = _lib.workspace(self.lib.gnn_mask_norm_colsum_workspace(self.M, self.N), self.dev)

    def __call__(self):
        args = [self.M, self.N, self.X.data_ptr(), self.X.stride(0),
                self.mask.data_ptr() if self.mask is not None else None,
                self.mask.stride(0) if self.mask is not None else 0,
                self.deg.data_ptr() if self.deg is not None else None,
                self.out.data_ptr() if self.out is not None else None,
                self.out.stride(0) if self.out is not None else 0,
                self.colsum.data_ptr() if self.colsum is not None else None]
        if self.rows_dev is not None:
            _lib.check(self.lib.gnn_mask_norm_colsum_dev(
                *args, self.rows_dev.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                _lib.stream_handle(self.dev)), "mask_norm_colsum (device rows)")
            return
        _lib.check(self.lib.gnn_mask_norm_colsum(
            *args, self.ws.data_ptr(), self.ws.numel(), _lib.stream_handle(self.dev)),
            "mask_norm_colsum")


class XentCall:
    def __init__(self, Z, labels, loss, dZ=None, grad_scale=None):
        self.lib = _lib.lib()
        self.dev = Z.device
        self.M, self.Cn = Z.shape
        self.Z, self.labels, self.loss, self.dZ = Z, labels, loss, dZ
        self.scale = float(1.0 / self.M if grad_scale is None else grad_scale)
        self.ws = _lib.workspace(self.lib.gnn_softmax_xent_workspace(self.M), self.dev)

    def __call__(self):
        _lib.check(self.lib.gnn_softmax_xent(
            self.M, self.Cn, self.Z.data_ptr(), self.Z.stride(0), self.labels.data_ptr(),
            self.scale, self.dZ.data_ptr() if self.dZ is not None else None,
            self.dZ.stride(0) if self.dZ is not None else 0, self.loss.data_ptr(),
            self.ws.data_ptr(), self.ws.numel(), _lib.stream_handle(self.dev)), "softmax_xent")


class AdamCall:
    def __init__(self, params, grads, lr=0.01, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0):
        self.lib = _lib.lib()
        self.dev = params[0].device
        self.params, self.grads = list(params), list(grads)
        self.m = [torch.zeros_like(p) for p in self.params]
        self.v = [torch.zeros_like(p) for p in self.params]
        rows = [[p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), p.numel()]
                for p, g, m, v in zip(self.params, self.grads, self.m, self.v)]
        self.table = torch.tensor(rows, dtype=torch.int64, device=self.dev)
        self.step = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.lr, self.b1, self.b2, self.eps, self.wd = lr, betas[0], betas[1], eps, weight_decay

    def __call__(self):
        _lib.check(self.lib.gnn_adam_step(len(self.params), self.table.data_ptr(), self.lr,
                                          self.b1, self.b2, self.eps, self.wd,
                                          self.step.data_ptr(), _lib.stream_handle(self.dev)),
                   "adam")


class HeadCall:
    """Fused output layer: logits, mean cross-entropy, dP (degree-normed), dW, db.

    The fused kernel (gnn_gcn_head_scaled) covers Din, C <= 64 and, with the
    wide form (class chunks, online softmax, logits never stored), Din <= 32
    with C <= 256 — the 172 classes of the papers100M shape; other shapes run
    the same math as library calls: Z = P W + b, softmax-CE (dZ scaled),
    dW = P^T dZ, db = colsum(dZ), dP = (dZ W^T) / deg.  ``scale`` multiplies the summed
    loss and dZ: 1/M (the default) is the mean over these rows; a row-
    partitioned rank passes 1/V_global so the all-reduced loss and gradients
    equal the single-GPU mean."""

    FUSED_MAX = int(os.environ.get("GNN_HEAD_FUSED_MAX", "64"))

    def __init__(self, P, W, b, labels, dP, dW, db, loss, deg_offsets=None, scale=None):
        self.lib = _lib.lib()
        self.dev = P.device
        self.M, self.Din = P.shape
        self.C = W.shape[1]
        self.scale = float(1.0 / self.M if scale is None else scale)
        self.P, self.W, self.b, self.labels, self.dP = P, W, b, labels, dP
        self.dW, self.db, self.loss, self.deg = dW, db, loss, deg_offsets
        self.fused = ((self.Din <= self.FUSED_MAX and self.C <= self.FUSED_MAX)
                      or (self.FUSED_MAX > 0 and self.Din <= 32 and 64 < self.C <= 256))
        if not self.fused:
            f32 = dict(dtype=torch.float32, device=self.dev)
            self.Z = torch.empty(self.M, self.C, **f32)
            self.dZ = torch.empty(self.M, self.C, **f32)
            self._parts = [GemmCall(P, W, self.Z, bias=b),
                           XentCall(self.Z, labels, loss, dZ=self.dZ, grad_scale=self.scale),
                           GemmCall(P, self.dZ, dW, trans_a=True),
                           ColsumCall(self.dZ, db),
                           GemmCall(self.dZ, W, dP, trans_b=True)]
            if deg_offsets is not None:
                self._parts.append(MaskNormColsumCall(dP, dP, deg_offsets=deg_offsets))
            return
        self.ws = _lib.workspace(self.lib.gnn_gcn_head_workspace(self.M, self.Din, self.C),
                                 self.dev)

    def __call__(self):
        if not self.fused:
            for c in self._parts:
                c()
            if self.scale * self.M != 1.0:  # softmax_xent's loss is the mean over M rows
                self.loss.mul_(self.scale * self.M)
            return
        _lib.check(self.lib.gnn_gcn_head_scaled(
            self.M, self.Din, self.C, self.P.data_ptr(), self.P.stride(0), self.W.data_ptr(),
            self.b.data_ptr(), self.labels.data_ptr(),
            self.deg.data_ptr() if self.deg is not None else None, self.scale,
            self.dP.data_ptr(), self.dP.stride(0), self.dW.data_ptr(), self.db.data_ptr(),
            self.loss.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
            _lib.stream_handle(self.dev)), "gcn_head")


class ColsumCall:
    def __init__(self, X, out):
        self.lib = _lib.lib()
        self.dev = X.device
        self.M, self.N = X.shape
        self.X, self.out = X, out
        self.ws = _lib.workspace(self.lib.gnn_colsum_workspace(self.M, self.N), self.dev)

    def __call__(self):
        _lib.check(self.lib.gnn_colsum(self.M, self.N, self.X.data_ptr(), self.X.stride(0),
                                       self.out.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                                       _lib.stream_handle(self.dev)), "colsum")


class SddmmCall:
    """out[e,h] = <X[row_e,h,:], Y[col_e,h,:]> over op's edges."""

    def __init__(self, op: SparseOperand, X, Y, out, heads=1):
        self.lib = _lib.lib()
        self.dev = X.device
        self.K = int(X.shape[1])
        self.view, self.plan = op.view(), op.plan()
        self.X, self.Y, self.out, self.heads, self._op = X, Y, out, heads, op

    def __call__(self):
        _lib.check(self.lib.gnn_sddmm(C.byref(self.view), C.byref(self.plan), self.heads,
                                      self.X.data_ptr(), self.X.stride(0), self.Y.data_ptr(),
                                      self.Y.stride(0), self.K, self.out.data_ptr(),
                                      _lib.stream_handle(self.dev)), "sddmm")


class EdgeSoftmaxCall:
    """Forward (alpha from s, or from GAT el/er) or backward (ds from alpha,
    dalpha[, GAT el/er]) edge softmax over op's rows."""

    def __init__(self, op: SparseOperand, heads, out, *, s=None, el=None, er=None, slope=0.2,
                 backward=False, alpha=None, dalpha=None):
        self.lib = _lib.lib()
        self.dev = out.device
        self.view, self.plan = op.view(), op.plan()
        self.heads, self.out, self.backward = heads, out, backward
        self.sc = _lib.EdgeScores()
        self.sc.s = s.data_ptr() if s is not None else None
        self.sc.el = el.data_ptr() if el is not None else None
        self.sc.er = er.data_ptr() if er is not None else None
        self.sc.slope = float(slope)
        self.alpha, self.dalpha = alpha, dalpha
        self._keep = (op, s, el, er)
        self.ws = _lib.workspace(self.lib.gnn_edge_softmax_workspace(C.byref(self.plan), heads),
                                 self.dev)

    def __call__(self):
        st = _lib.stream_handle(self.dev)
        if self.backward:
            _lib.check(self.lib.gnn_edge_softmax_bwd(
                C.byref(self.view), C.byref(self.plan), self.heads, self.alpha.data_ptr(),
                self.dalpha.data_ptr(), C.byref(self.sc), self.out.data_ptr(),
                self.ws.data_ptr(), self.ws.numel(), st), "edge_softmax backward")
        else:
            _lib.check(self.lib.gnn_edge_softmax_fwd(
                C.byref(self.view), C.byref(self.plan), self.heads, C.byref(self.sc),
                self.out.data_ptr(), self.ws.data_ptr(), self.ws.numel(), st), "edge_softmax")


class AttnProjCall:
    def __init__(self, Wh, a_l, a_r, el, er, heads):
        self.lib = _lib.lib()
        self.dev = Wh.device
        self.V = int(Wh.shape[0])
        self.H = heads
        self.F = int(a_l.numel()) // heads
        self.Wh, self.a_l, self.a_r, self.el, self.er = Wh, a_l, a_r, el, er

    def __call__(self):
        _lib.check(self.lib.gnn_gat_attn_proj(self.V, self.H, self.F, self.Wh.data_ptr(),
                                              self.Wh.stride(0), self.a_l.data_ptr(),
                                              self.a_r.data_ptr(), self.el.data_ptr(),
                                              self.er.data_ptr(), _lib.stream_handle(self.dev)),
                   "gat attn_proj")


class AttnProjBwdCall:
    def __init__(self, Wh, a_l, a_r, del_, der, dWh, da_l, da_r, heads):
        self.lib = _lib.lib()
        self.dev = Wh.device
        self.V = int(Wh.shape[0])
        self.H = heads
        self.F = int(a_l.numel()) // heads
        self.t = (Wh, a_l, a_r, del_, der, dWh, da_l, da_r)
        self.ws = _lib.workspace(self.lib.gnn_gat_attn_proj_bwd_workspace(self.H, self.F),
                                 self.dev)

    def __call__(self):
        Wh, a_l, a_r, del_, der, dWh, da_l, da_r = self.t
        _lib.check(self.lib.gnn_gat_attn_proj_bwd(
            self.V, self.H, self.F, Wh.data_ptr(), Wh.stride(0), a_l.data_ptr(), a_r.data_ptr(),
            del_.data_ptr(), der.data_ptr(), dWh.data_ptr(), dWh.stride(0), da_l.data_ptr(),
            da_r.data_ptr(), self.ws.data_ptr(), self.ws.numel(), _lib.stream_handle(self.dev)),
            "gat attn_proj backward")


class HeadMeanCall:
    """out[v,f] = mean_h Y[v,h*F+f] (+bias); backward=True: Y <- dout/heads broadcast."""

    def __init__(self, Y, out, heads, F, bias=None, backward=False):
        self.lib = _lib.lib()
        self.dev = Y.device
        self.V = int(Y.shape[0])
        self.H, self.F = heads, F
        self.Y, self.out, self.bias, self.backward = Y, out, bias, backward

    def __call__(self):
        st = _lib.stream_handle(self.dev)
        if self.backward:
            _lib.check(self.lib.gnn_head_mean_bwd(self.V, self.H, self.F, self.out.data_ptr(),
                                                  self.out.stride(0), self.Y.data_ptr(),
                                                  self.Y.stride(0), st), "head_mean backward")
        else:
            _lib.check(self.lib.gnn_head_mean(
                self.V, self.H, self.F, self.Y.data_ptr(), self.Y.stride(0),
                self.bias.data_ptr() if self.bias is not None else None, self.out.data_ptr(),
                self.out.stride(0), st), "head_mean")


class SegmentSumCall:
    """out[r,h] = sum over op's row r of vals[(eid ? eid[j] : j), h] (row sums of
    an edge tensor; column sums through the CSC + edge-ID)."""

    def __init__(self, op: SparseOperand, vals, out, heads, use_eid=False, eid=None):
        self.lib = _lib.lib()
        self.dev = out.device
        self.view = op.view(vals=vals, eid=op.eid if use_eid else None)
        if eid is not None:  # an explicit position map (e.g. CSR -> CSC positions)
            self.view.eid = eid.data_ptr()
            self._eid = eid
        elif not use_eid:
            self.view.eid = None
        self.plan = op.plan()
        self.heads, self.vals, self.out, self._op = heads, vals, out, op
        self.ws = _lib.workspace(self.lib.gnn_edge_softmax_workspace(C.byref(self.plan), heads),
                                 self.dev)

    def __call__(self):
        _lib.check(self.lib.gnn_segment_sum(C.byref(self.view), C.byref(self.plan), self.heads,
                                            self.vals.data_ptr(), self.out.data_ptr(),
                                            self.ws.data_ptr(), self.ws.numel(),
                                            _lib.stream_handle(self.dev)), "segment_sum")


class GatBwdCscCall:
    """Fused GAT backward over the CSC (edge-ID view): dWh = SpMMve^T(alpha, dY)
    and dalpha = SDDMM(dY, Wh) from one gather of dY per edge."""

    def __init__(self, AT: SparseOperand, alpha, dY, Wh, dWh, dalpha, heads):
        self.lib = _lib.lib()
        self.dev = dY.device
        self.view = AT.view(vals=alpha, eid=AT.eid)
        self.plan = AT.plan()
        self.K = int(dY.shape[1])
        self.t = (alpha, dY, Wh, dWh, dalpha)
        self.heads, self._op = heads, AT
        self.ws = _lib.workspace(self.lib.gnn_gat_bwd_csc_workspace(C.byref(self.plan), self.K),
                                 self.dev)

    def __call__(self):
        alpha, dY, Wh, dWh, dalpha = self.t
        _lib.check(self.lib.gnn_gat_bwd_csc(
            C.byref(self.view), C.byref(self.plan), self.heads, alpha.data_ptr(), dY.data_ptr(),
            dY.stride(0), Wh.data_ptr(), Wh.stride(0), self.K, dWh.data_ptr(), dWh.stride(0),
            dalpha.data_ptr(), self.ws.data_ptr(), self.ws.numel(), _lib.stream_handle(self.dev)),
            "gat_bwd_csc")


class GatBwdCscMeanCall:
    """Fused GAT backward of a head-mean layer over the CSC: gathers dZ[v]
    (F floats) once per edge and produces dWh (all heads) and dalpha."""

    def __init__(self, AT: SparseOperand, alpha, dZ, Wh, dWh, dalpha, heads, scale=None):
        self.lib = _lib.lib()
        self.dev = dZ.device
        self.view = AT.view(vals=alpha, eid=AT.eid)
        self.plan = AT.plan()
        self.F = int(dZ.shape[1])
        self.heads = heads
        self.scale = float(1.0 / heads if scale is None else scale)
        self.t = (alpha, dZ, Wh, dWh, dalpha)
        self._op = AT
        self.ws = _lib.workspace(
            self.lib.gnn_gat_bwd_csc_workspace(C.byref(self.plan), heads * self.F), self.dev)

    def __call__(self):
        alpha, dZ, Wh, dWh, dalpha = self.t
        _lib.check(self.lib.gnn_gat_bwd_csc_mean(
            C.byref(self.view), C.byref(self.plan), self.heads, alpha.data_ptr(), dZ.data_ptr(),
            dZ.stride(0), self.scale, Wh.data_ptr(), Wh.stride(0), self.F, dWh.data_ptr(),
            dWh.stride(0), dalpha.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
            _lib.stream_handle(self.dev)), "gat_bwd_csc_mean")


class GatSoftmaxStatsCall:
    """GAT edge softmax (scores from el / er) that also keeps the per-row
    (max, 1/sum) statistics the recompute backward needs."""

    def __init__(self, op: SparseOperand, heads, alpha, rowstat, el, er, slope=0.2):
        self.lib = _lib.lib()
        self.dev = alpha.device
        self.view, self.plan = op.view(), op.plan()
        self.heads, self.alpha, self.rowstat = heads, alpha, rowstat
        self.sc = _lib.EdgeScores()
        self.sc.s = None
        self.sc.el, self.sc.er, self.sc.slope = el.data_ptr(), er.data_ptr(), float(slope)
        self._keep = (op, el, er)
        self.ws = _lib.workspace(self.lib.gnn_edge_softmax_workspace(C.byref(self.plan), heads),
                                 self.dev)

    def __call__(self):
        _lib.check(self.lib.gnn_gat_softmax_fwd_stats(
            C.byref(self.view), C.byref(self.plan), self.heads, C.byref(self.sc),
            self.alpha.data_ptr(), self.rowstat.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
            _lib.stream_handle(self.dev)), "gat_softmax_fwd_stats")


class GatRowStatCall:
    """Per-row backward statistics {er, m, 1/sum, S} of a GAT layer, written as
    four float4 into ``stat`` (a [V, 16] view, usually the 16 columns after
    the gradient row the recompute backward gathers).  Concatenated heads:
    S = <dYm_h, Y_h - b_h>.  ``mean`` (head-mean output layer,
    aggregate-then-transform): S = scale <dZ, Yc_h W_h>, on the tensor cores
    (gnn_gat_rowstat_mean_tc: dZ W_h^T reduced against Yc in the GEMM
    epilogue) where the shapes allow, else the SIMT kernel."""

    def __init__(self, er, rowstat, stat, *, dYm=None, Y=None, bias=None, mean=None):
        self.lib = _lib.lib()
        self.dev = er.device
        self.V = int(er.shape[0])
        self.er, self.rowstat, self.stat = er, rowstat, stat
        self.dYm, self.Y, self.bias, self.mean = dYm, Y, bias, mean
        self.tc = False
        if mean is not None and os.environ.get("GNN_GAT_ROWSTAT_TC", "1") != "0":
            dZ, Yc, W, F1, Cp, _ = mean
            self.tc = (self.V >= 128 and W.stride(0) == 4 * Cp and dZ.stride(0) % 4 == 0
                       and dZ.data_ptr() % 16 == 0 and Yc.stride(0) % 4 == 0
                       and Yc.data_ptr() % 16 == 0)
            if self.tc:
                self.ws = _lib.workspace(self.lib.gnn_gat_rowstat_mean_tc_workspace(F1, Cp),
                                         self.dev)

    def __call__(self):
        st = _lib.stream_handle(self.dev)
        if self.mean is None:
            K = int(self.dYm.shape[1])
            _lib.check(self.lib.gnn_gat_rowstat(
                self.V, K, self.dYm.data_ptr(), self.dYm.stride(0), self.Y.data_ptr(),
                self.Y.stride(0), self.bias.data_ptr() if self.bias is not None else None,
                self.er.data_ptr(), self.rowstat.data_ptr(), self.stat.data_ptr(),
                self.stat.stride(0), st), "gat_rowstat")
        else:
            dZ, Yc, W, F1, Cp, scale = self.mean
            if self.tc:
                _lib.check(self.lib.gnn_gat_rowstat_mean_tc(
                    self.V, F1, Cp, dZ.data_ptr(), dZ.stride(0), Yc.data_ptr(), Yc.stride(0),
                    W.data_ptr(), W.stride(0), scale, self.er.data_ptr(), self.rowstat.data_ptr(),
                    self.stat.data_ptr(), self.stat.stride(0), self.ws.data_ptr(), self.ws.numel(),
                    st), "gat_rowstat_mean_tc")
                return
            _lib.check(self.lib.gnn_gat_rowstat_mean(
                self.V, F1, Cp, dZ.data_ptr(), dZ.stride(0), Yc.data_ptr(), Yc.stride(0),
                W.data_ptr(), W.stride(0), scale, self.er.data_ptr(), self.rowstat.data_ptr(),
                self.stat.data_ptr(), self.stat.stride(0), st), "gat_rowstat_mean")


class GatProjGemmCall:
    """Wh = X W with the GAT attention projections el / er (4 heads of F =
    N/4 columns) in the same tcgen05 pass (gnn_gemm_gat_proj): Wh is not read
    back for them."""

    def __init__(self, X, W, Wh, a_l, a_r, el, er):
        self.lib = _lib.lib()
        self.dev = X.device
        self.M, self.Kd = int(X.shape[0]), int(X.shape[1])
        self.N = int(W.shape[1])
        self.F = self.N // 4
        self.t = (X, W, Wh, a_l, a_r, el, er)
        self.ws = _lib.workspace(self.lib.gnn_gemm_workspace(self.M, self.N, self.Kd, 0), self.dev)

    def __call__(self):
        X, W, Wh, a_l, a_r, el, er = self.t
        _lib.check(self.lib.gnn_gemm_gat_proj(
            self.M, self.N, self.Kd, X.data_ptr(), X.stride(0), W.data_ptr(), W.stride(0),
            Wh.data_ptr(), Wh.stride(0), self.F, a_l.data_ptr(), a_r.data_ptr(), el.data_ptr(),
            er.data_ptr(), self.ws.data_ptr(), self.ws.numel(), _lib.stream_handle(self.dev)),
            "gemm_gat_proj")


class GatReluStatGemmCall:
    """dYm = ReLU'(Y) * (A W^T) with the recompute backward's per-head row
    statistics {er, m, 1/sum, S} written after each row's N columns, in the
    tcgen05 GEMM's epilogue (gnn_gemm_gat_relu_stat): the GAT hidden layer's
    dY = dWh2 W2^T, its ReLU backward and its statistics in one pass."""

    def __init__(self, A, Wt, dYms, Y, bias, er, rowstat):
        self.lib = _lib.lib()
        self.dev = A.device
        self.M, self.Kd = int(A.shape[0]), int(A.shape[1])
        self.N = int(Wt.shape[0])
        self.t = (A, Wt, dYms, Y, bias, er, rowstat)
        self.ws = _lib.workspace(self.lib.gnn_gemm_workspace(self.M, self.N, self.Kd, 0), self.dev)

    def __call__(self):
        A, Wt, C_, Y, bias, er, rs = self.t
        _lib.check(self.lib.gnn_gemm_gat_relu_stat(
            self.M, self.N, self.Kd, A.data_ptr(), A.stride(0), Wt.data_ptr(), Wt.stride(0),
            C_.data_ptr(), C_.stride(0), Y.data_ptr(), Y.stride(0), bias.data_ptr(), er.data_ptr(),
            rs.data_ptr(), self.ws.data_ptr(), self.ws.numel(), _lib.stream_handle(self.dev)),
            "gemm_gat_relu_stat")


class GatBwdRcCall:
    """GAT backward over the CSC with alpha recomputed from the row statistics
    (gnn_gat_bwd_rc / _mean): dWh, del and ds (CSR edge order) in one pass.
    ``dY`` is a [V, R] view whose rows continue with the 16 statistics floats
    (row stride >= R + 16)."""

    def __init__(self, AT: SparseOperand, el, dY, Wh, dWh, del_, ds, *, slope=0.2,
                 mean_F=None, scale=None):
        self.lib = _lib.lib()
        self.dev = dY.device
        self.view, self.plan = AT.view(), AT.plan()
        self.view.eid = AT.eid.data_ptr()  # ds lands in CSR edge order
        self.mean_F = mean_F
        self.K = int(dWh.shape[1])
        self.scale = float(0.25 if scale is None else scale)
        self.slope = float(slope)
        self.t = (el, dY, Wh, dWh, del_, ds)
        self._op = AT
        self.ws = _lib.workspace(self.lib.gnn_gat_bwd_rc_workspace(C.byref(self.plan), self.K),
                                 self.dev)

    def __call__(self):
        el, dY, Wh, dWh, del_, ds = self.t
        if not hasattr(self, "l2"):
            self.l2 = _L2Window(self.lib, dY)  # the gathered gradient rows' hub prefix
        with self.l2:
            self._launch(el, dY, Wh, dWh, del_, ds)

    def _launch(self, el, dY, Wh, dWh, del_, ds):
        st = _lib.stream_handle(self.dev)
        if self.mean_F is None:
            _lib.check(self.lib.gnn_gat_bwd_rc(
                C.byref(self.view), C.byref(self.plan), self.K, el.data_ptr(), self.slope,
                dY.data_ptr(), dY.stride(0), Wh.data_ptr(), Wh.stride(0), dWh.data_ptr(),
                dWh.stride(0), del_.data_ptr(), ds.data_ptr(), self.ws.data_ptr(),
                self.ws.numel(), st), "gat_bwd_rc")
        else:
            _lib.check(self.lib.gnn_gat_bwd_rc_mean(
                C.byref(self.view), C.byref(self.plan), self.mean_F, self.scale, el.data_ptr(),
                self.slope, dY.data_ptr(), dY.stride(0), Wh.data_ptr(), Wh.stride(0),
                dWh.data_ptr(), dWh.stride(0), del_.data_ptr(), ds.data_ptr(),
                self.ws.data_ptr(), self.ws.numel(), st), "gat_bwd_rc_mean")


def invert_permutation(perm: torch.Tensor) -> torch.Tensor:
    """inv[perm[i]] = i on device (libgnnb200)."""
    inv = torch.empty_like(perm)
    lib = _lib.lib()
    _lib.check(lib.gnn_invert_permutation(perm.numel(), perm.data_ptr(), inv.data_ptr(),
                                          _lib.stream_handle(perm.device)), "invert_permutation")
    return inv


class PeerSpmmCall:
    """gnn_spmm_peer: Y = epilogue(op . X) where X is row-partitioned across
    ``parts`` (device pointers, one per rank; rows of part q are the global
    columns [q << log2, (q+1) << log2)) and every gathered row is read in place
    from its owner — peer-mapped NVLink memory on a multi-GPU box."""

    def __init__(self, op: SparseOperand, part_ptrs, part_rows_log2: int, ldx: int, K: int,
                 Y: torch.Tensor, *, flags=0, bias=None, mask=None, keep=()):
        self.lib = _lib.lib()
        self.dev = Y.device
        self.view = op.view()
        self.plan = op.spmm_plan()
        self.parts = (C.c_void_p * len(part_ptrs))(*[int(p) for p in part_ptrs])
        self.nparts, self.log2, self.ldx, self.K, self.Y = len(part_ptrs), part_rows_log2, ldx, K, Y
        self.epi = _lib.Epilogue()
        self.epi.flags = flags
        if bias is not None:
            self.epi.bias = bias.data_ptr()
        if mask is not None:
            self.epi.mask, self.epi.ld_mask = mask.data_ptr(), mask.stride(0)
        self._keep = (op, bias, mask, keep)
        self.ws = _lib.workspace(self.lib.gnn_spmm_workspace(C.byref(self.view), C.byref(self.plan),
                                                             K), self.dev)

    def __call__(self):
        _lib.check(self.lib.gnn_spmm_peer(
            C.byref(self.view), C.byref(self.plan), self.parts, self.nparts, self.log2, self.ldx,
            self.Y.data_ptr(), self.Y.stride(0), self.K, C.byref(self.epi), self.ws.data_ptr(),
            self.ws.numel(), _lib.stream_handle(self.dev)), "spmm_peer")
