"""SDDMM and edge-softmax (GraphPy class-A kernels, PAPER.md:281-287 and
606-617) on libgnnb200, as plain functions and autograd Functions.

    sddmm(g, X, Y, heads=1)            out[e,h] = <X[row_e,h,:], Y[col_e,h,:]>  (CSR edge order)
    edge_softmax(g, s)                 alpha = softmax of s over each CSR row (per head)
    gat_scores_softmax(g, el, er)      alpha from the GAT score LeakyReLU(el[col]+er[row])

All tensors are fp32 CUDA tensors; edge tensors are [E] or [E, H] in CSR
edge order.  There is no CPU path.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .graph import CsrGraph, SparseOperand


def _check(t: torch.Tensor, what: str):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor")
    if t.dtype != torch.float32:
        raise ValueError(f"{what}: expected float32, got {t.dtype}")


def _heads_of(t: torch.Tensor) -> int:
    return 1 if t.dim() == 1 else int(t.shape[1])


def sddmm_raw(op: SparseOperand, X: torch.Tensor, Y: torch.Tensor, heads: int = 1,
              out: torch.Tensor | None = None) -> torch.Tensor:
    """out[e,h] = <X[row_e, h*F:(h+1)*F], Y[col_e, h*F:(h+1)*F]> over op's edges."""
    lib = _lib.lib()
    _check(X, "sddmm X")
    _check(Y, "sddmm Y")
    K = int(X.shape[1])
    if X.dim() != 2 or Y.dim() != 2 or Y.shape[1] != K:
        raise ValueError("sddmm: X and Y must be 2-D with the same width")
    if X.shape[0] != op.num_rows or Y.shape[0] != op.num_cols:
        raise ValueError(f"sddmm: expected X [{op.num_rows}, K] and Y [{op.num_cols}, K]")
    if heads <= 0 or K % heads:
        raise ValueError("sddmm: width must be a multiple of heads")
    if X.stride(1) != 1 or Y.stride(1) != 1:
        raise ValueError("sddmm: rows must be contiguous")
    if out is None:
        out = torch.empty(op.nnz, heads, dtype=torch.float32, device=X.device)
    view = op.view()
    plan = op.plan()
    with torch.cuda.device(X.device):
        _lib.check(lib.gnn_sddmm(C.byref(view), C.byref(plan), heads, X.data_ptr(), X.stride(0),
                                 Y.data_ptr(), Y.stride(0), K, out.data_ptr(),
                                 _lib.stream_handle(X.device)), "sddmm")
    return out


def _scores(s=None, el=None, er=None, slope=0.2):
    sc = _lib.EdgeScores()
    sc.s = s.data_ptr() if s is not None else None
    sc.el = el.data_ptr() if el is not None else None
    sc.er = er.data_ptr() if er is not None else None
    sc.slope = float(slope)
    return sc


def edge_softmax_fwd_raw(op: SparseOperand, heads: int, *, s=None, el=None, er=None, slope=0.2,
                         out=None) -> torch.Tensor:
    lib = _lib.lib()
    dev = op.device
    if out is None:
        out = torch.empty(op.nnz, heads, dtype=torch.float32, device=dev)
    view, plan = op.view(), op.plan()
    sc = _scores(s, el, er, slope)
    with torch.cuda.device(dev):
        ws = _lib.workspace(lib.gnn_edge_softmax_workspace(C.byref(plan), heads), dev)
        _lib.check(lib.gnn_edge_softmax_fwd(C.byref(view), C.byref(plan), heads, C.byref(sc),
                                            out.data_ptr(), ws.data_ptr(), ws.numel(),
                                            _lib.stream_handle(dev)), "edge_softmax")
    return out


def edge_softmax_bwd_raw(op: SparseOperand, heads: int, alpha, dalpha, *, el=None, er=None,
                         slope=0.2, out=None) -> torch.Tensor:
    lib = _lib.lib()
    dev = op.device
    if out is None:
        out = torch.empty(op.nnz, heads, dtype=torch.float32, device=dev)
    view, plan = op.view(), op.plan()
    sc = _scores(None, el, er, slope)
    with torch.cuda.device(dev):
        ws = _lib.workspace(lib.gnn_edge_softmax_workspace(C.byref(plan), heads), dev)
        _lib.check(lib.gnn_edge_softmax_bwd(C.byref(view), C.byref(plan), heads,
                                            alpha.data_ptr(), dalpha.data_ptr(), C.byref(sc),
                                            out.data_ptr(), ws.data_ptr(), ws.numel(),
                                            _lib.stream_handle(dev)), "edge_softmax backward")
    return out


class _Sddmm(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X, Y, g, heads):
        ctx.save_for_backward(X, Y)
        ctx.g, ctx.heads = g, heads
        return sddmm_raw(g.csr(), X.contiguous(), Y.contiguous(), heads)

    @staticmethod
    def backward(ctx, dout):
        from .ops import spmm_raw

        X, Y = ctx.saved_tensors
        g, heads = ctx.g, ctx.heads
        d = dout.contiguous()
        dX = dY = None
        if ctx.needs_input_grad[0]:  # dX[r] = sum_e dout_e Y[col_e]
            dX = spmm_raw(g.csr(), Y.contiguous(), heads=heads, vals=d)
        if ctx.needs_input_grad[1]:  # dY[c] = sum_e dout_e X[row_e]   (A^T via edge-ID)
            csc = g.csc(with_eid=True)
            dY = spmm_raw(csc, X.contiguous(), heads=heads, vals=d, eid=csc.eid)
        return dX, dY, None, None


def sddmm(g: CsrGraph, X: torch.Tensor, Y: torch.Tensor, heads: int = 1) -> torch.Tensor:
    """SDDMM: out[e,h] = <X[row_e,h,:], Y[col_e,h,:]>,
    [E, heads] in CSR edge order.  Differentiable w.r.t. X and Y."""
    return _Sddmm.apply(X, Y, g, int(heads))


class _EdgeSoftmax(torch.autograd.Function):
    @staticmethod
    def forward(ctx, s, g):
        heads = _heads_of(s)
        s2 = s.contiguous().reshape(s.shape[0], heads)
        alpha = edge_softmax_fwd_raw(g.csr(), heads, s=s2)
        ctx.save_for_backward(alpha)
        ctx.g, ctx.shape = g, s.shape
        return alpha.reshape(s.shape)

    @staticmethod
    def backward(ctx, dalpha):
        (alpha,) = ctx.saved_tensors
        heads = alpha.shape[1]
        da = dalpha.contiguous().reshape(alpha.shape)
        ds = edge_softmax_bwd_raw(ctx.g.csr(), heads, alpha, da)
        return ds.reshape(ctx.shape), None


def edge_softmax(g: CsrGraph, s: torch.Tensor) -> torch.Tensor:
    """alpha_e = exp(s_e - max_row) / sum_row exp(s - max_row) per head, over
    each CSR row (the attention state tensor of PAPER.md:606-617)."""
    _check(s, "edge_softmax scores")
    if s.shape[0] != g.num_edges:
        raise ValueError(f"edge_softmax: expected {g.num_edges} edge scores, got {s.shape[0]}")
    return _EdgeSoftmax.apply(s, g)


def gat_attention(g: CsrGraph, el: torch.Tensor, er: torch.Tensor, slope: float = 0.2):
    """alpha = edge_softmax(LeakyReLU(el[col] + er[row])) with the scores
    computed inside the softmax kernels (never materialised).  Not
    differentiable by itself; the GAT layer owns its backward."""
    heads = _heads_of(el)
    return edge_softmax_fwd_raw(g.csr(), heads, el=el.contiguous(), er=er.contiguous(),
                                slope=slope)
