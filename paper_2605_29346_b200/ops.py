"""Sparse and dense operators of the GNN hot path (GraphPy kernel API,
PAPER.md:264-287) on libgnnb200, as plain functions and autograd Functions.

    spmmv(g, X, norm=False, transpose=False)      Y = [D^-1] A X   (or A^T X)
    spmmve(g, X, ev, transpose=False)             Y = A_ev X       (edge values ev[E(,H)])
    degree_norm_(g, X, transpose=False)           X[v] /= deg(v)   in place
    linear(X, W, b=None, relu=False)              X W (+b) fp32-accurate
    colsum(X)                                     sum over rows

All tensors are fp32 CUDA tensors; there is no CPU path.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .graph import CsrGraph, SparseOperand, spmm_operand


def _check_features(X: torch.Tensor, rows: int, what: str):
    if not isinstance(X, torch.Tensor) or not X.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor")
    if X.dtype != torch.float32:
        raise ValueError(f"{what}: expected float32, got {X.dtype}")
    if X.dim() != 2 or X.shape[0] != rows:
        raise ValueError(f"{what}: expected shape [{rows}, K], got {tuple(X.shape)}")
    if X.stride(1) != 1:
        raise ValueError(f"{what}: rows must be contiguous")


def spmm_raw(op: SparseOperand, X: torch.Tensor, *, heads: int = 1, vals=None, eid=None,
             flags: int = 0, bias=None, self_x=None, self_scale: float = 1.0, mask=None,
             post_deg_offsets=None, out=None, plan=None) -> torch.Tensor:
    """Y = epilogue(op . X) through gnn_spmm; X is [num_cols, K] with unit column stride."""
    lib = _lib.lib()
    K = int(X.shape[1])
    _check_features(X, op.num_cols, "spmm input")
    dev = X.device
    if out is None:
        out = torch.empty(op.num_rows, K, dtype=torch.float32, device=dev)
    else:
        _check_features(out, op.num_rows, "spmm output")
    if plan is None:
        op = spmm_operand(op, X, out, heads=heads, vals=vals, eid=eid, self_x=self_x, mask=mask,
                          bias=bias)
        plan = op.spmm_plan()
    view = op.view(vals=vals, eid=eid)
    epi = _lib.Epilogue()
    epi.flags = flags
    epi.self_scale = float(self_scale)
    if self_x is not None:
        epi.self_x = self_x.data_ptr()
        epi.ld_self = self_x.stride(0)
    if bias is not None:
        epi.bias = bias.data_ptr()
    if mask is not None:
        epi.mask = mask.data_ptr()
        epi.ld_mask = mask.stride(0)
    if post_deg_offsets is not None:
        epi.post_deg_offsets = post_deg_offsets.data_ptr()
    with torch.cuda.device(dev):
        ws = _lib.workspace(lib.gnn_spmm_workspace(C.byref(view), C.byref(plan), K), dev)
        _lib.check(lib.gnn_spmm(C.byref(view), C.byref(plan), heads, X.data_ptr(), X.stride(0),
                                out.data_ptr(), out.stride(0), K, C.byref(epi), ws.data_ptr(),
                                ws.numel(), _lib.stream_handle(dev)), "spmm")
    return out


def degree_norm_(g: CsrGraph, X: torch.Tensor, transpose: bool = False) -> torch.Tensor:
    """In-place X[v,:] /= deg(v) (rows of degree 0 become 0; no clamp buffer).
    transpose=True uses in-degrees (the CSC's row lengths).  PAPER.md:275,278."""
    lib = _lib.lib()
    op = g.csc() if transpose else g.csr()
    _check_features(X, op.num_rows, "degree_norm_")
    with torch.cuda.device(X.device):
        _lib.check(lib.gnn_degree_norm_inplace(op.num_rows, op.offsets.data_ptr(), X.data_ptr(),
                                               X.stride(0), X.shape[1],
                                               _lib.stream_handle(X.device)), "degree_norm_")
    return X


def _operand(g: CsrGraph, transpose: bool, coalesced: bool) -> SparseOperand:
    if coalesced:
        return g.csc_coalesced() if transpose else g.csr_coalesced()
    return g.csc() if transpose else g.csr()


class _SpMMv(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X, g, norm, transpose, coalesced):
        op = _operand(g, transpose, coalesced)
        Y = spmm_raw(op, X.contiguous(), flags=_lib.EPI_NORM if norm else 0)
        ctx.g, ctx.norm, ctx.transpose, ctx.coalesced = g, norm, transpose, coalesced
        return Y

    @staticmethod
    def backward(ctx, dY):
        g = ctx.g
        dY = dY.contiguous()
        if ctx.norm:
            # norm sits on the OUTPUT of forward, so backward applies it to the
            # INPUT of the transposed SpMM; dY is not ours
            # to overwrite, so normalise a copy in place.
            dY = degree_norm_(g, dY.clone(), transpose=ctx.transpose)
        op = _operand(g, not ctx.transpose, ctx.coalesced)
        return spmm_raw(op, dY), None, None, None, None


def spmmv(g: CsrGraph, X: torch.Tensor, norm: bool = False, transpose: bool = False,
          coalesced: bool = False) -> torch.Tensor:
    """SpMMv: Y[v] = sum_{e in row v} X[col_e], divided by
    deg(v) when ``norm`` (fused in the same kernel).  No edge tensor.
    ``transpose`` aggregates over A^T through the CSC.  ``coalesced`` uses the
    multiplicity-weighted unique-pair structure (same result, fewer gathers on
    multigraphs).  Differentiable w.r.t. X."""
    return _SpMMv.apply(X, g, bool(norm), bool(transpose), bool(coalesced))


class _SpMMve(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X, ev, g, transpose):
        heads = 1 if ev.dim() == 1 else int(ev.shape[1])
        ev_c = ev.contiguous()
        if transpose:
            csc = g.csc(with_eid=True)
            Y = spmm_raw(csc, X.contiguous(), heads=heads, vals=ev_c, eid=csc.eid)
        else:
            Y = spmm_raw(g.csr(), X.contiguous(), heads=heads, vals=ev_c)
        ctx.save_for_backward(X, ev_c)
        ctx.g, ctx.transpose, ctx.heads = g, transpose, heads
        return Y

    @staticmethod
    def backward(ctx, dY):
        X, ev = ctx.saved_tensors
        g, heads = ctx.g, ctx.heads
        dY = dY.contiguous()
        dX = dev = None
        if ctx.needs_input_grad[0]:
            if ctx.transpose:
                dX = spmm_raw(g.csr(), dY, heads=heads, vals=ev)
            else:
                csc = g.csc(with_eid=True)
                dX = spmm_raw(csc, dY, heads=heads, vals=ev, eid=csc.eid)
        if ctx.needs_input_grad[1]:
            from .sparse_attn import sddmm

            if ctx.transpose:
                # Y = A^T_ev X: dev_e(row r, col c of A) = <dY[c], X[r]>
                d = sddmm(g, X, dY, heads=heads)
            else:
                d = sddmm(g, dY, X, heads=heads)
            dev = d if ev.dim() == 2 else d.reshape(-1)
        return dX, dev, None, None


def spmmve(g: CsrGraph, X: torch.Tensor, ev: torch.Tensor, transpose: bool = False):
    """SpMMve: Y[v] = sum_e ev_e * X[col_e]; ev is [E] or
    [E, H] in CSR edge order (H heads split the feature dim).  ``transpose``
    runs over the CSC and fetches ev through the edge-ID array — no eShuffle."""
    return _SpMMve.apply(X, ev, g, bool(transpose))


# ------------------------------------------------------------------ dense
def gemm(A: torch.Tensor, B: torch.Tensor, *, trans_a: bool = False, trans_b: bool = False,
         bias=None, relu: bool = False, out=None) -> torch.Tensor:
    """C = op(A) op(B) (+bias)(relu), fp32 in/out on libgnnb200."""
    lib = _lib.lib()
    if A.stride(1) != 1 or B.stride(1) != 1:
        raise ValueError("gemm: operands must have unit column stride")
    M = A.shape[1] if trans_a else A.shape[0]
    Kd = A.shape[0] if trans_a else A.shape[1]
    N = B.shape[0] if trans_b else B.shape[1]
    Kb = B.shape[1] if trans_b else B.shape[0]
    if Kb != Kd:
        raise ValueError(f"gemm: inner dimensions differ ({Kd} vs {Kb})")
    dev = A.device
    if out is None:
        out = torch.empty(M, N, dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        ws = _lib.workspace(lib.gnn_gemm_workspace(M, N, Kd, int(trans_a)), dev)
        _lib.check(lib.gnn_gemm(M, N, Kd, A.data_ptr(), A.stride(0), int(trans_a), B.data_ptr(),
                                B.stride(0), int(trans_b), out.data_ptr(), out.stride(0),
                                bias.data_ptr() if bias is not None else None, int(relu),
                                ws.data_ptr(), ws.numel(), _lib.stream_handle(dev)), "gemm")
    return out


def colsum(X: torch.Tensor, out=None) -> torch.Tensor:
    lib = _lib.lib()
    M, N = X.shape
    if out is None:
        out = torch.empty(N, dtype=torch.float32, device=X.device)
    with torch.cuda.device(X.device):
        ws = _lib.workspace(lib.gnn_colsum_workspace(M, N), X.device)
        _lib.check(lib.gnn_colsum(M, N, X.data_ptr(), X.stride(0), out.data_ptr(), ws.data_ptr(),
                                  ws.numel(), _lib.stream_handle(X.device)), "colsum")
    return out


class _Linear(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X, W, b, relu):
        Y = gemm(X.contiguous(), W.contiguous(), bias=b, relu=relu)
        ctx.save_for_backward(X, W, Y if relu else None)
        ctx.has_b, ctx.relu = b is not None, relu
        return Y

    @staticmethod
    def backward(ctx, dY):
        X, W, Y = ctx.saved_tensors
        dY = dY.contiguous()
        db = None
        if ctx.relu:  # ReLU backward against the saved output, bias grad in the same pass
            from .kernels import MaskNormColsumCall

            dYm = torch.empty_like(dY)
            db = torch.empty(dY.shape[1], dtype=torch.float32, device=dY.device)
            MaskNormColsumCall(dY, dYm, mask=Y, colsum=db if ctx.has_b else None)()
            dY = dYm
        dX = gemm(dY, W, trans_b=True) if ctx.needs_input_grad[0] else None
        dW = gemm(X, dY, trans_a=True) if ctx.needs_input_grad[1] else None
        if ctx.has_b and ctx.needs_input_grad[2] and db is None:
            db = colsum(dY)
        return dX, dW, db if ctx.has_b else None, None


def linear(X: torch.Tensor, W: torch.Tensor, b=None, relu: bool = False) -> torch.Tensor:
    """X[M,Kin] . W[Kin,N] (+ b)(ReLU fused), differentiable, on libgnnb200."""
    return _Linear.apply(X, W, b, bool(relu))
