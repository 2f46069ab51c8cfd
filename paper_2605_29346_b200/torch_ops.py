"""The hot-path operators registered as PyTorch custom ops (torch.library):

    torch.ops.gnnb200.spmmv(X, graph, norm, transpose, coalesced)
    torch.ops.gnnb200.spmmve(X, ev, graph, transpose)
    torch.ops.gnnb200.sddmm(X, Y, graph, heads)

each with a fake (meta) kernel and an autograd formula, so torch.fx /
torch.compile / torch.export see them as opaque, differentiable ops over the
same libgnnb200 kernels the plain functions of ``ops`` / ``sparse_attn`` call
(no second implementation).  A CSR graph is not a tensor, so the ops take an
integer handle: ``h = register_graph(g)`` (``release_graph(h)`` drops it).
"""

from __future__ import annotations

import torch

from . import _lib
from .graph import CsrGraph
from .ops import _operand, degree_norm_, spmm_raw

_GRAPHS: dict[int, CsrGraph] = {}


def register_graph(g: CsrGraph) -> int:
    """Handle of ``g`` for the torch.ops.gnnb200 operators (kept alive until
    release_graph)."""
    h = id(g)
    _GRAPHS[h] = g
    return h


def release_graph(handle: int) -> None:
    _GRAPHS.pop(int(handle), None)


def _graph(handle: int) -> CsrGraph:
    try:
        return _GRAPHS[int(handle)]
    except KeyError:
        raise ValueError(f"unknown graph handle {handle} (register_graph first)") from None


# ---------------------------------------------------------------- SpMMv
@torch.library.custom_op("gnnb200::spmmv", mutates_args=())
def spmmv(X: torch.Tensor, graph: int, norm: bool, transpose: bool,
          coalesced: bool) -> torch.Tensor:
    op = _operand(_graph(graph), transpose, coalesced)
    return spmm_raw(op, X.contiguous(), flags=_lib.EPI_NORM if norm else 0)


@spmmv.register_fake
def _spmmv_fake(X, graph, norm, transpose, coalesced):
    return X.new_empty(_graph(graph).num_vertices, X.shape[1])


def _spmmv_setup(ctx, inputs, output):
    _, ctx.graph, ctx.norm, ctx.transpose, ctx.coalesced = inputs


def _spmmv_backward(ctx, dY):
    dY = dY.contiguous()
    if ctx.norm:  # the norm sits on forward's output: applied to the transposed SpMM's input
        dY = degree_norm_(_graph(ctx.graph), dY.clone(), transpose=ctx.transpose)
    return spmmv(dY, ctx.graph, False, not ctx.transpose, ctx.coalesced), None, None, None, None


spmmv.register_autograd(_spmmv_backward, setup_context=_spmmv_setup)


# ---------------------------------------------------------------- SpMMve
@torch.library.custom_op("gnnb200::spmmve", mutates_args=())
def spmmve(X: torch.Tensor, ev: torch.Tensor, graph: int, transpose: bool) -> torch.Tensor:
    g = _graph(graph)
    heads = 1 if ev.dim() == 1 else int(ev.shape[1])
    ev_c = ev.contiguous()
    if transpose:
        csc = g.csc(with_eid=True)
        return spmm_raw(csc, X.contiguous(), heads=heads, vals=ev_c, eid=csc.eid)
    return spmm_raw(g.csr(), X.contiguous(), heads=heads, vals=ev_c)


@spmmve.register_fake
def _spmmve_fake(X, ev, graph, transpose):
    return X.new_empty(_graph(graph).num_vertices, X.shape[1])


def _spmmve_setup(ctx, inputs, output):
    X, ev, ctx.graph, ctx.transpose = inputs
    ctx.save_for_backward(X, ev)


def _spmmve_backward(ctx, dY):
    X, ev = ctx.saved_tensors
    heads = 1 if ev.dim() == 1 else int(ev.shape[1])
    dY = dY.contiguous()
    dX = dev = None
    if ctx.needs_input_grad[0]:
        dX = spmmve(dY, ev, ctx.graph, not ctx.transpose)
    if ctx.needs_input_grad[1]:
        # dev_e (row r, col c of A) = <dY[r], X[c]> (forward), <dY[c], X[r]> (transpose)
        d = sddmm(X, dY, ctx.graph, heads) if ctx.transpose else sddmm(dY, X, ctx.graph, heads)
        dev = d if ev.dim() == 2 else d.reshape(-1)
    return dX, dev, None, None


spmmve.register_autograd(_spmmve_backward, setup_context=_spmmve_setup)


# ---------------------------------------------------------------- SDDMM
@torch.library.custom_op("gnnb200::sddmm", mutates_args=())
def sddmm(X: torch.Tensor, Y: torch.Tensor, graph: int, heads: int) -> torch.Tensor:
    """out[e, h] = <X[row_e, head h], Y[col_e, head h]> in CSR edge order."""
    from .sparse_attn import sddmm_raw

    return sddmm_raw(_graph(graph).csr(), X.contiguous(), Y.contiguous(), heads=heads)


@sddmm.register_fake
def _sddmm_fake(X, Y, graph, heads):
    return X.new_empty(_graph(graph).num_edges, heads)


def _sddmm_setup(ctx, inputs, output):
    X, Y, ctx.graph, ctx.heads = inputs
    ctx.save_for_backward(X, Y)


def _sddmm_backward(ctx, dout):
    X, Y = ctx.saved_tensors
    dout = dout.contiguous()
    dX = dY = None
    if ctx.needs_input_grad[0]:  # dX[r] = sum_e dout_e Y[c_e]  (SpMMve over A)
        dX = spmmve(Y, dout, ctx.graph, False)
    if ctx.needs_input_grad[1]:  # dY[c] = sum_e dout_e X[r_e]  (SpMMve over A^T)
        dY = spmmve(X, dout, ctx.graph, True)
    return dX, dY, None, None


sddmm.register_autograd(_sddmm_backward, setup_context=_sddmm_setup)
