"""Device-resident CSR graph with the reference's graph API.

Mirrors ``gsbench.graph`` (graph.py:19-262) and ``gsbench.build_subgraph_csr``
(sampler.py:242-256) name for name, argument for argument, and exception for
exception, but every array-sized step runs on the GPU through libgnnb200:

* ``csr_from_edges`` / ``build_subgraph_csr`` -> stable device radix sort
  (bit-exact with numpy's ``argsort(kind="stable")`` build);
* ``make_csr`` -> device invariant check;
* ``generate`` power-law -> on-device PCG64 jump-ahead draws, bit-exact with
  ``numpy.random.default_rng(SeedSequence(seed)).random`` + ``searchsorted``;
* the transposed CSR (CSC + edge-ID), multigraph coalescing and the SpMM
  schedules are built lazily, once, on device.

Host views (``offsets``, ``targets``, ``degrees``) are materialised on first
access, read-only, with the reference's dtypes (int64 / int32 / int64).
"""

from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass
from pathlib import Path
from typing import IO, Iterable, Union

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, ExtensionMissing, ParseError, RangeError

OFFSET_DTYPE = np.int64
TARGET_DTYPE = np.int32
MAX_VERTEX_ID = int(np.iinfo(TARGET_DTYPE).max)
_CSR_MAGIC = b"CSR1"

GraphSource = Union[str, Path, IO[str], Iterable[str]]


def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise ExtensionMissing("no CUDA device: the graph builders run on the GPU only")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"graphs live on a CUDA device, got {d}")
    if d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return d


def _to_device_i64(a, dev) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=torch.int64).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    return torch.from_numpy(arr).to(dev)


def _readonly(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


def _default_edges_per_warp(nnz: int, sms: int) -> int:
    """Edge range per warp of the SpMM (a multiple of 4: 16-byte aligned index
    vectors).  2048-edge ranges (measured best on Reddit-size graphs: long
    enough to amortise row-bound loads and split-row arrivals, short enough for
    ~56k warps of parallelism); smaller graphs shrink it so every SM still
    gets several waves."""
    p = int(os.environ.get("GNN_SPMM_P", "2048"))
    while p > 256 and nnz // p < sms * 64:
        p //= 2
    return p // 4 * 4


# rows of degree <= this go to the SpMM's group-per-row kernel (power-law tail):
# a degree-sorted operand hands it a contiguous, length-ordered tail (512); a
# row-order operand keeps it to the shortest rows (its nnz-split kernel walks
# every row anyway, and staged edge values beat the tail's global loads)
SPMM_SHORT_MAX = int(os.environ.get("GNN_SPMM_SHORT", "512"))
SPMM_SHORT_ROWORDER = int(os.environ.get("GNN_SPMM_SHORT_ROWORDER", "32"))


# GNN_SPMM_SORT=0 keeps gnn_spmm on the operand's own row order; operands
# below SPMM_SORT_MIN_NNZ entries stay in row order (building the sorted copy
# costs more than it saves on a small, e.g. per-mini-batch, subgraph)
SPMM_SORT = os.environ.get("GNN_SPMM_SORT", "1") != "0"
SPMM_SORT_MIN_NNZ = int(os.environ.get("GNN_SPMM_SORT_MIN_NNZ", str(1 << 20)))


def _al16(t) -> bool:
    return t is None or (t.data_ptr() % 16 == 0 and (t.dim() < 2 or t.stride(0) % 4 == 0))


def spmm_operand(op: "SparseOperand", X, Y, *, heads=1, vals=None, eid=None, self_x=None,
                 mask=None, bias=None) -> "SparseOperand":
    """The operand form gnn_spmm should run on: the degree-sorted one
    (``by_degree``) where its group-per-row tail applies — topology or
    multiplicity weights only, K <= 64 in float4 lanes — else ``op``."""
    K = int(X.shape[1])
    if getattr(op, "_released", False):  # only the sorted form is left
        return op.by_degree()
    if (not SPMM_SORT or SPMM_SHORT_MAX <= 0 or heads != 1 or vals is not None
            or eid is not None or (op._vals is not None and not op.mult) or op.nnz == 0
            or op.nnz < SPMM_SORT_MIN_NNZ or K > 64 or K % 4
            or not all(_al16(t) for t in (X, Y, self_x, mask, bias))):
        return op
    return op.by_degree()


# GNN_SPMM_PACK=0 keeps multiplicity-weighted operands in the float form
SPMM_PACK = os.environ.get("GNN_SPMM_PACK", "1") != "0"


class SparseOperand:
    """One device sparse matrix in CSR layout (a graph's CSR, or its CSC which
    is the CSR of the transpose), plus cached SpMM schedules.

    ``mult=True`` marks ``vals`` as integer multiplicities (the coalesced
    multigraph forms); such an operand is stored packed when it fits — column
    id in the low ``col_bits`` bits, multiplicity above (gnn_csr_pack_weights)
    — one 4-byte word per edge instead of 8.  ``cols`` / ``vals`` then
    unpack on demand (setup-time consumers); the SpMM reads the packed words."""

    def __init__(self, num_rows, num_cols, offsets, cols, vals=None, eid=None, deg_offsets=None,
                 mult: bool = False, row_ids=None, pack: bool = True):
        self.num_rows = int(num_rows)
        self.num_cols = int(num_cols)
        self.nnz = int(cols.numel())
        self.offsets = offsets
        self._cols = cols
        self._vals = vals
        self.eid = eid
        self.deg_offsets = deg_offsets
        self.mult = bool(mult)
        self.row_ids = row_ids  # permuted operand: row i -> output row row_ids[i]
        self._sorted = None
        self.col_bits = 0
        self.packed = None
        self._plain = None
        self._plans = {}
        if pack and mult and vals is not None and eid is None and SPMM_PACK and self.nnz > 0:
            self._try_pack()

    def _try_pack(self):
        bits = max(1, (self.num_cols - 1).bit_length())
        if bits > 28:  # < 16 per word
            return
        maxw = (1 << (32 - bits)) - 1
        cols, vals, offsets = self._cols, self._vals, self.offsets
        reps = torch.div(vals.to(torch.int64) + (maxw - 1), maxw, rounding_mode="floor")
        reps.clamp_(min=1)
        if bits > 24 and int(reps.sum().item()) > 1.05 * self.nnz:
            # a narrow weight field (>= 2^25 columns, e.g. papers100M) splits
            # hub pairs into too many words: keep the float form
            return
        if int(reps.max().item()) > 1:
            # a multiplicity above the word's weight field (hub pairs of a
            # power-law multigraph: Reddit's top pair repeats ~2e5 times) is
            # split into several entries of the same column; the SpMM sums
            # them (same value, fp32 rounding of the split product)
            n2 = int(reps.sum().item())
            idx = torch.repeat_interleave(torch.arange(self.nnz, device=cols.device), reps,
                                          output_size=n2)
            first = torch.cumsum(reps, 0) - reps
            pos = torch.arange(n2, device=cols.device) - first[idx]
            r = reps[idx]
            w = torch.where(pos < r - 1, torch.full_like(pos, maxw),
                            vals[idx].to(torch.int64) - maxw * (r - 1))
            extra = torch.zeros(self.nnz + 1, dtype=torch.int64, device=cols.device)
            torch.cumsum(reps - 1, 0, out=extra[1:])
            offsets = offsets + extra[offsets]
            cols, vals = cols[idx].contiguous(), w.to(torch.float32)
            del idx, first, pos, r, w, extra
        lib = _lib.lib()
        dev = self.device
        out = torch.empty(cols.numel(), dtype=torch.int32, device=dev)
        with torch.cuda.device(dev):
            ws = _lib.workspace(lib.gnn_csr_pack_weights_workspace(), dev)
            rc = lib.gnn_csr_pack_weights(cols.numel(), cols.data_ptr(), vals.data_ptr(),
                                          bits, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                          _lib.stream_handle(dev))
        if rc != 0:  # not representable: keep the float form
            return
        self.packed, self.col_bits, self.offsets = out, bits, offsets
        self.nnz = int(out.numel())
        self._cols = self._vals = None

    def by_degree(self) -> "SparseOperand":
        """Degree-sorted form for gnn_spmm (cached): rows longest-first with
        ``row_ids`` mapping each back to its output row; the nnz-split kernel
        then covers only the long-row prefix and the group-per-row kernel the
        contiguous, length-ordered tail (SPMM_SHORT_MAX).  Same entries per
        row, same order within a row: results are bit-identical."""
        if self.row_ids is not None:
            return self
        if self._sorted is None:
            if getattr(self, "_released", False):
                raise RuntimeError("row-order storage of this operand was released")
            dev = self.device
            deg = self.offsets[1:] - self.offsets[:-1]
            order = torch.sort(deg, descending=True, stable=True).indices
            sdeg = deg[order]
            off = torch.zeros(self.num_rows + 1, dtype=torch.int64, device=dev)
            torch.cumsum(sdeg, 0, out=off[1:])
            # shift[i] = old start - new start of sorted row i: entry j of the
            # new array comes from j + shift[row(j)] (gathered in slabs of rows
            # to bound the int64 temporaries)
            shift = self.offsets[order] - off[:-1]
            words = self.packed if self.packed is not None else self._cols
            cols = torch.empty_like(words)
            vals = (torch.empty_like(self._vals) if (self.packed is None and self._vals is not None)
                    else None)
            slab = int(os.environ.get("GNN_SORT_SLAB", 1 << 24))
            r0 = 0
            while r0 < self.num_rows:
                e0 = int(off[r0].item())
                if e0 >= self.nnz:  # only empty rows left
                    break
                e1 = min(self.nnz, e0 + slab)
                r1 = int(torch.searchsorted(off, e1, right=True).item()) - 1
                r1 = min(max(r1, r0 + 1), self.num_rows)
                e1 = int(off[r1].item())
                row = torch.repeat_interleave(torch.arange(r0, r1, device=dev), sdeg[r0:r1],
                                              output_size=e1 - e0)
                src = torch.arange(e0, e1, device=dev) + shift[row]
                cols[e0:e1] = words[src]
                if vals is not None:
                    vals[e0:e1] = self._vals[src]
                del row, src
                r0 = r1
            del shift
            deg_off = self.deg_offsets if self.deg_offsets is not None else self.offsets
            if self.packed is not None:
                op = SparseOperand(self.num_rows, self.num_cols, off, cols,
                                   deg_offsets=deg_off, row_ids=order.to(torch.int32))
                op.packed, op.col_bits, op._cols, op.mult = op._cols, self.col_bits, None, True
            else:
                op = SparseOperand(self.num_rows, self.num_cols, off, cols, vals=vals,
                                   deg_offsets=deg_off, row_ids=order.to(torch.int32))
            self._sorted = op
        return self._sorted

    def release_row_order(self) -> None:
        """Keep only the degree-sorted form (built now if needed) and free the
        row-order index arrays: for trainers whose every use of this operand is
        a gnn_spmm (which runs on the sorted form) — halves its footprint.
        Afterwards ``cols`` / ``vals`` / ``entries`` / ``view`` are unavailable."""
        so = self.by_degree()
        if so is self:
            return
        self.packed = self._cols = self._vals = self._plain = None
        self._released = True

    def entries(self, e0: int = 0, e1: int | None = None):
        """(cols, vals) of entries [e0, e1) in plain form (vals None if none)."""
        e1 = self.nnz if e1 is None else e1
        if self.packed is None:
            v = self._vals[e0:e1] if self._vals is not None else None
            return self._cols[e0:e1], v
        pk = self.packed[e0:e1]
        w = torch.bitwise_right_shift(pk, self.col_bits) & ((1 << (32 - self.col_bits)) - 1)
        return pk & ((1 << self.col_bits) - 1), w.to(torch.float32)

    @property
    def cols(self) -> torch.Tensor:
        if self.packed is None:
            return self._cols
        return self.packed & ((1 << self.col_bits) - 1)

    @property
    def vals(self):
        if self.packed is None:
            return self._vals
        w = torch.bitwise_right_shift(self.packed, self.col_bits) & ((1 << (32 - self.col_bits)) - 1)
        return w.to(torch.float32)

    @property
    def device(self):
        return self.offsets.device

    def view(self, vals=None, eid=None) -> _lib.CsrView:
        if getattr(self, "_released", False):
            raise RuntimeError("row-order storage of this operand was released "
                               "(release_row_order): use by_degree()")
        v = _lib.CsrView()
        v.num_rows = self.num_rows
        v.num_cols = self.num_cols
        v.nnz = self.nnz
        v.offsets = self.offsets.data_ptr()
        v.row_ids = self.row_ids.data_ptr() if self.row_ids is not None else None
        if self.packed is not None and vals is None:
            # packed multiplicities: the SpMM decodes column + weight per word
            v.cols = self.packed.data_ptr()
            v.col_bits = self.col_bits
            v.vals = None
            v.eid = None
            v.deg_offsets = self.deg_offsets.data_ptr() if self.deg_offsets is not None else None
            return v
        if self.packed is not None:  # explicit edge values over a packed operand
            if self._plain is None:
                self._plain = self.cols
            v.cols = self._plain.data_ptr()
        else:
            v.cols = self.cols.data_ptr() if self.nnz else None
        vv = vals if vals is not None else self.vals
        v.vals = vv.data_ptr() if vv is not None else None
        ee = eid if eid is not None else self.eid
        # the edge-ID indirection only applies to edge values (SpMMve^T); a
        # topology-only SpMMv over a CSC that happens to carry eid ignores it
        v.eid = ee.data_ptr() if (ee is not None and vv is not None) else None
        v.deg_offsets = self.deg_offsets.data_ptr() if self.deg_offsets is not None else None
        return v

    def plan(self, edges_per_warp: int | None = None, short_max: int = 0) -> _lib.SpmmPlan:
        """Chunk schedule shared by every edge kernel.  ``short_max`` > 0 gives
        the degree-binned SpMM plan (rows of degree <= short_max handled by the
        group-per-row kernel); the edge-softmax / SDDMM / GAT kernels use 0."""
        lib = _lib.lib()
        if edges_per_warp is None:
            with torch.cuda.device(self.device):
                sms = lib.gnn_device_sm_count()
            edges_per_warp = _default_edges_per_warp(self.nnz, sms)
        key = (int(edges_per_warp), int(short_max))
        if key in self._plans:
            return self._plans[key][0]
        dev = self.device
        with torch.cuda.device(dev):
            nint = lib.gnn_spmm_plan_buffer_ints(self.num_rows, self.nnz, key[0])
            buf = torch.empty(max(int(nint), 1), dtype=torch.int32, device=dev)
            ws = _lib.workspace(lib.gnn_spmm_plan_workspace(self.num_rows), dev)
            plan = _lib.SpmmPlan()
            view = self.view()
            _lib.check(
                lib.gnn_spmm_plan_build_ex(C.byref(view), key[0], key[1], buf.data_ptr(),
                                           C.byref(plan), ws.data_ptr(), ws.numel(),
                                           _lib.stream_handle(dev)),
                "spmm plan",
            )
        self._plans[key] = (plan, buf)
        return plan

    def spmm_plan(self, edges_per_warp: int | None = None) -> _lib.SpmmPlan:
        """Plan for gnn_spmm: degree-binned, short_max = SPMM_SHORT_MAX for the
        degree-sorted form, SPMM_SHORT_ROWORDER otherwise."""
        return self.plan(edges_per_warp, short_max=SPMM_SHORT_MAX if self.row_ids is not None
                         else SPMM_SHORT_ROWORDER)

    def nbytes(self) -> int:
        n = self.offsets.numel() * 8 + self.nnz * 4
        if self._vals is not None:
            n += self._vals.numel() * self._vals.element_size()
        if self.eid is not None:
            n += self.eid.numel() * 4
        for _, buf in self._plans.values():
            n += buf.numel() * 4
        return n


class CsrGraph:
    """Compressed sparse row adjacency, immutable after construction.

    Same public surface as ``gsbench.graph.CsrGraph`` (graph.py:30-47):
    ``num_vertices``, ``num_edges``, ``offsets`` (int64, V+1), ``targets``
    (int32, E), ``degrees``, ``degree(v)``, ``neighbors(v)``; the arrays live
    on a CUDA device (``d_offsets`` / ``d_targets``) and the host views are
    lazily copied, read-only.
    """

    __slots__ = ("num_vertices", "num_edges", "d_offsets", "d_targets", "_h_offsets",
                 "_h_targets", "_csr", "_csc", "_csr_co", "_csc_co", "__weakref__")

    def __init__(self, num_vertices: int, num_edges: int, d_offsets: torch.Tensor,
                 d_targets: torch.Tensor, h_offsets=None, h_targets=None):
        object.__setattr__(self, "num_vertices", int(num_vertices))
        object.__setattr__(self, "num_edges", int(num_edges))
        object.__setattr__(self, "d_offsets", d_offsets)
        object.__setattr__(self, "d_targets", d_targets)
        object.__setattr__(self, "_h_offsets", h_offsets)
        object.__setattr__(self, "_h_targets", h_targets)
        object.__setattr__(self, "_csr", None)
        object.__setattr__(self, "_csc", None)
        object.__setattr__(self, "_csr_co", None)
        object.__setattr__(self, "_csc_co", None)

    def __setattr__(self, name, value):
        raise AttributeError("CsrGraph is immutable")

    # ---- host views (reference surface)
    @property
    def offsets(self) -> np.ndarray:
        if self._h_offsets is None:
            object.__setattr__(self, "_h_offsets", _readonly(self.d_offsets.cpu().numpy()))
        return self._h_offsets

    @property
    def targets(self) -> np.ndarray:
        if self._h_targets is None:
            if self.d_targets is None:
                raise RuntimeError("targets released without a host view")
            object.__setattr__(self, "_h_targets", _readonly(self.d_targets.cpu().numpy()))
        return self._h_targets

    @property
    def degrees(self) -> np.ndarray:
        return self.device_degrees().cpu().numpy()

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])

    def neighbors(self, v: int) -> np.ndarray:
        return self.targets[self.offsets[v]: self.offsets[v + 1]]

    # ---- device side
    @property
    def device(self) -> torch.device:
        return self.d_offsets.device

    def device_degrees(self) -> torch.Tensor:
        """int64 [V] out-degrees computed on device (graph.py:39-41)."""
        lib = _lib.lib()
        with torch.cuda.device(self.device):
            deg = torch.empty(self.num_vertices, dtype=torch.int64, device=self.device)
            _lib.check(lib.gnn_degrees(self.num_vertices, self.d_offsets.data_ptr(),
                                       deg.data_ptr() if self.num_vertices else None,
                                       _lib.stream_handle(self.device)), "degrees")
        return deg

    def csr(self) -> SparseOperand:
        if self._csr is None:
            object.__setattr__(self, "_csr", SparseOperand(self.num_vertices, self.num_vertices,
                                                           self.d_offsets, self._device_targets()))
        return self._csr

    def csc(self, with_eid: bool = False) -> SparseOperand:
        """Transposed CSR; with the edge-ID array only when
        asked — GCN's backward needs the topology alone,
        so the |E| edge-ID array is not allocated for it."""
        if self._csc is None or (with_eid and self._csc.eid is None):
            t_off, t_rows, t_eid = _transpose(self.num_vertices, self.num_vertices,
                                              self.d_offsets, self._device_targets(),
                                              with_eid=with_eid)
            object.__setattr__(self, "_csc", SparseOperand(self.num_vertices, self.num_vertices,
                                                           t_off, t_rows, eid=t_eid))
        return self._csc

    def drop_csc(self) -> None:
        """Release the canonical CSC (e.g. after building the coalesced forms)."""
        object.__setattr__(self, "_csc", None)

    def release_device_targets(self) -> None:
        """Keep the canonical targets only as the (materialised) host view and
        free the device copy — for trainers that run on the coalesced forms.
        Degree-norms keep using the device offsets; any later op that needs
        the canonical device CSR re-uploads it."""
        _ = self.targets  # materialise the read-only host view first
        object.__setattr__(self, "d_targets", None)
        object.__setattr__(self, "_csr", None)

    def _device_targets(self) -> torch.Tensor:
        if self.d_targets is None:
            object.__setattr__(self, "d_targets", torch.from_numpy(
                np.ascontiguousarray(self._h_targets)).to(self.d_offsets.device))
        return self.d_targets

    def csr_coalesced(self) -> SparseOperand:
        """Unique (row,col) pairs with multiplicities, columns ascending per row.
        An internal SpMM accelerator for multigraphs; NORM still uses the
        canonical degree (duplicates counted), so results equal the canonical
        SpMMv up to fp32 summation order."""
        if self._csr_co is None:
            csc = self.csc()
            s_off, s_cols, _ = _transpose(self.num_vertices, self.num_vertices, csc.offsets,
                                          csc.cols, with_eid=False)
            off, cols, mult = _coalesce(self.num_vertices, s_off, s_cols)
            del s_off, s_cols
            object.__setattr__(self, "_csr_co", SparseOperand(
                self.num_vertices, self.num_vertices, off, cols, vals=mult,
                deg_offsets=self.d_offsets, mult=True))
        return self._csr_co

    def csc_coalesced(self) -> SparseOperand:
        if self._csc_co is None:
            csc = self.csc()
            off, cols, mult = _coalesce(self.num_vertices, csc.offsets, csc.cols)
            object.__setattr__(self, "_csc_co", SparseOperand(
                self.num_vertices, self.num_vertices, off, cols, vals=mult,
                deg_offsets=csc.offsets, mult=True))
        return self._csc_co

    def operand(self, kind: str) -> SparseOperand:
        return {"csr": self.csr, "csc": self.csc, "csr_coalesced": self.csr_coalesced,
                "csc_coalesced": self.csc_coalesced}[kind]()

    def device_nbytes(self) -> int:
        n = 0
        for op in (self._csr, self._csc, self._csr_co, self._csc_co):
            if op is not None:
                n += op.nbytes()
        if self._csr is None:
            n += self.d_offsets.numel() * 8
            if self.d_targets is not None:
                n += self.d_targets.numel() * 4
        return n

    def __repr__(self):
        return f"CsrGraph(num_vertices={self.num_vertices}, num_edges={self.num_edges}, device={self.device})"


# --------------------------------------------------------------- builders
def _transpose(R, Ccols, offsets, cols, with_eid):
    lib = _lib.lib()
    dev = offsets.device
    nnz = cols.numel()
    with torch.cuda.device(dev):
        t_off = torch.empty(Ccols + 1, dtype=torch.int64, device=dev)
        t_rows = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)[:nnz]
        t_eid = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)[:nnz] if with_eid else None
        ws = _lib.workspace(lib.gnn_csc_from_csr_workspace(R, Ccols, nnz), dev)
        _lib.check(lib.gnn_csc_from_csr(R, Ccols, nnz, offsets.data_ptr(),
                                        cols.data_ptr() if nnz else None, t_off.data_ptr(),
                                        t_rows.data_ptr() if nnz else None,
                                        t_eid.data_ptr() if (with_eid and nnz) else None,
                                        ws.data_ptr(), ws.numel(), _lib.stream_handle(dev)),
                   "csc_from_csr")
    return t_off, t_rows, t_eid


def _coalesce(R, offsets, cols):
    lib = _lib.lib()
    dev = offsets.device
    nnz = cols.numel()
    with torch.cuda.device(dev):
        out_off = torch.empty(R + 1, dtype=torch.int64, device=dev)
        out_cols = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        out_mult = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
        n_out = C.c_int64(0)
        ws = _lib.workspace(lib.gnn_csr_coalesce_workspace(R, nnz), dev)
        _lib.check(lib.gnn_csr_coalesce(R, nnz, offsets.data_ptr(), cols.data_ptr() if nnz else None,
                                        out_off.data_ptr(), out_cols.data_ptr(),
                                        out_mult.data_ptr(), C.byref(n_out), ws.data_ptr(),
                                        ws.numel(), _lib.stream_handle(dev)), "coalesce")
        u = int(n_out.value)
        out_cols = out_cols[:u].clone()
        out_mult = out_mult[:u].clone()
    return out_off, out_cols, out_mult


def _build_from_edges(fn_ws, fn, n, src, dst, device, what):
    lib = _lib.lib()
    dev = _device(device)
    s = _to_device_i64(src, dev)
    d = _to_device_i64(dst, dev)
    if s.numel() != d.numel():
        raise ValueError("src and dst must have the same length")
    E = int(s.numel())
    with torch.cuda.device(dev):
        offsets = torch.empty(max(n, 0) + 1, dtype=torch.int64, device=dev)
        targets = torch.empty(max(E, 1), dtype=torch.int32, device=dev)[:E]
        ws = _lib.workspace(getattr(lib, fn_ws)(n, E), dev)
        _lib.check(getattr(lib, fn)(n, E, s.data_ptr() if E else None, d.data_ptr() if E else None,
                                    offsets.data_ptr(), targets.data_ptr() if E else None,
                                    ws.data_ptr(), ws.numel(), _lib.stream_handle(dev)), what)
    return offsets, targets


def make_csr(num_vertices: int, offsets, targets, device=None) -> CsrGraph:
    """Validate the CSR invariants and build an immutable graph (graph.py:91-103).

    Same checks and exception types: ValueError for a bad offsets shape, a
    wrong first/last offset, or decreasing offsets; RangeError for a target
    outside [0, num_vertices)."""
    dev = _device(device)
    if isinstance(offsets, torch.Tensor):
        d_off = offsets.to(device=dev, dtype=torch.int64).contiguous()
    else:
        d_off = torch.from_numpy(np.ascontiguousarray(offsets, dtype=OFFSET_DTYPE)).to(dev)
    if isinstance(targets, torch.Tensor):
        d_tgt = targets.to(device=dev, dtype=torch.int32).contiguous()
    else:
        d_tgt = torch.from_numpy(np.ascontiguousarray(targets, dtype=TARGET_DTYPE)).to(dev)
    if tuple(d_off.shape) != (num_vertices + 1,):
        raise ValueError("offsets must have length num_vertices + 1")
    lib = _lib.lib()
    E = int(d_tgt.numel())
    with torch.cuda.device(dev):
        ws = _lib.workspace(lib.gnn_csr_validate_workspace(num_vertices, E), dev)
        _lib.check(lib.gnn_csr_validate(num_vertices, E, d_off.data_ptr(),
                                        d_tgt.data_ptr() if E else None, ws.data_ptr(),
                                        ws.numel(), _lib.stream_handle(dev)), "make_csr")
    return CsrGraph(num_vertices, E, d_off, d_tgt)


def csr_from_edges(num_vertices: int, src, dst, device=None) -> CsrGraph:
    """Counting-sort edge pairs into CSR; stable within each source segment
    (graph.py:106-114), on device."""
    off, tgt = _build_from_edges("gnn_csr_from_edges_workspace", "gnn_csr_from_edges",
                                 int(num_vertices), src, dst, device, "csr_from_edges")
    return CsrGraph(num_vertices, int(tgt.numel()), off, tgt)


def build_subgraph_csr(edge_src, edge_dst, num_local_src: int, device=None):
    """Exclusive prefix sum of per-source degrees plus stable grouping
    (sampler.py:242-256).  Returns host ``(offsets int64, targets int32)`` like
    the reference when given host arrays, device tensors when given CUDA
    tensors.  IndexError if a source id is outside [0, num_local_src)."""
    on_device = isinstance(edge_src, torch.Tensor) and edge_src.is_cuda
    off, tgt = _build_from_edges("gnn_subgraph_csr_workspace", "gnn_subgraph_csr",
                                 int(num_local_src), edge_src, edge_dst,
                                 edge_src.device if on_device else device, "build_subgraph_csr")
    if on_device:
        return off, tgt
    return off.cpu().numpy(), tgt.cpu().numpy()


def total_degree(graph: CsrGraph) -> int:
    """Sum of out-degrees; equals num_edges by the CSR invariant (graph.py:117-119)."""
    return int(graph.d_offsets[-1].item())


# ------------------------------------------------------------ edge-list IO
def _lines(source: GraphSource):
    if isinstance(source, (str, Path)):
        with open(source, "r", encoding="utf-8") as fh:
            yield from fh
    else:
        yield from source


def load_edge_list(source: GraphSource, *, symmetrize: bool = False, compact_ids: bool = False,
                   device=None) -> CsrGraph:
    """Parse "src dst" lines into a CsrGraph (graph.py:134-196 semantics):
    '#' comments, optional "n=<count>" header, ParseError with the 1-based
    line number, RangeError for ids beyond 32 bits or the declared count,
    optional symmetrize / compact_ids.  Parsing is host text IO; the CSR build
    runs on device."""
    pairs_s: list[int] = []
    pairs_d: list[int] = []
    declared = None
    for lineno, raw in enumerate(_lines(source), start=1):
        text = raw.strip()
        if not text or text[0] == "#":
            continue
        if text.startswith("n="):
            try:
                declared = int(text[2:])
            except ValueError:
                raise ParseError(lineno, f"bad vertex-count header {text!r}") from None
            if declared < 0:
                raise ParseError(lineno, "declared vertex count must be nonnegative")
            continue
        fields = text.split()
        if len(fields) != 2:
            raise ParseError(lineno, f"expected 'src dst', got {text!r}")
        try:
            a, b = int(fields[0]), int(fields[1])
        except ValueError:
            raise ParseError(lineno, f"expected 'src dst', got {text!r}") from None
        if a < 0 or b < 0:
            raise ParseError(lineno, "vertex ids must be nonnegative")
        if a > MAX_VERTEX_ID or b > MAX_VERTEX_ID:
            raise RangeError(f"line {lineno}: vertex id exceeds 32-bit id space")
        pairs_s.append(a)
        pairs_d.append(b)
    src = np.asarray(pairs_s, dtype=np.int64)
    dst = np.asarray(pairs_d, dtype=np.int64)
    if symmetrize and src.size:
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    if compact_ids:
        ids = np.unique(np.concatenate([src, dst]))
        src = np.searchsorted(ids, src)
        dst = np.searchsorted(ids, dst)
        n = int(ids.size)
    else:
        top = max(int(src.max()) if src.size else -1, int(dst.max()) if dst.size else -1)
        n = top + 1
        if declared is not None:
            if declared < n:
                raise RangeError(f"vertex id {top} outside declared range n={declared}")
            n = declared
    return csr_from_edges(n, src, dst, device=device)


# ------------------------------------------------------------- binary IO
def save_csr(graph: CsrGraph, path) -> None:
    """Binary "CSR1" file: magic, <QQ (V, E), <i8 offsets, <i4 targets (graph.py:199-209)."""
    with open(path, "wb") as fh:
        fh.write(_CSR_MAGIC)
        fh.write(struct.pack("<QQ", graph.num_vertices, graph.num_edges))
        fh.write(np.asarray(graph.offsets, dtype="<i8").tobytes())
        fh.write(np.asarray(graph.targets, dtype="<i4").tobytes())


def _stream_to_device(fh, dst: torch.Tensor, nbytes: int, chunk: int = 64 << 20) -> None:
    """Read ``nbytes`` from ``fh`` straight into device tensor ``dst`` through
    two pinned staging buffers: the read of chunk i+1 overlaps the H2D copy of
    chunk i; no full host copy of the array ever exists."""
    if nbytes == 0:
        return
    dev = dst.device
    st = torch.cuda.current_stream(dev)
    bufs = [torch.empty(min(chunk, nbytes), dtype=torch.uint8).pin_memory() for _ in range(2)]
    done = [None, None]
    flat = dst.view(torch.uint8).reshape(-1)
    pos = 0
    k = 0
    while pos < nbytes:
        n = min(chunk, nbytes - pos)
        b = bufs[k & 1]
        if done[k & 1] is not None:
            done[k & 1].synchronize()  # the copy that last used this buffer has landed
        view = memoryview(b.numpy())[:n]
        got = 0
        while got < n:  # raw readinto may return short counts (pipes, FUSE, network FS)
            r = fh.readinto(view[got:])
            if not r:
                break
            got += r
        if got != n:
            # the reference's load_csr hits make_csr's shape check on a short
            # array (graph.py:218-220, 95-96): ValueError, not ParseError
            raise ValueError("truncated CSR1 file: offsets/targets shorter than the header says")
        flat[pos:pos + n].copy_(b[:n], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(st)
        done[k & 1] = ev
        pos += n
        k += 1
    st.synchronize()


def load_csr(path, device=None) -> CsrGraph:
    """Read a "CSR1" file (graph.py:212-220) straight into device memory —
    the <i8 offsets and <i4 targets are streamed through pinned staging
    buffers (read overlapped with H2D, no full host copy)
    — and validate it on device; ParseError on a bad magic, the reference's
    ValueError / RangeError on invariant violations."""
    dev = _device(device)
    with open(path, "rb", buffering=0) as fh:
        magic = fh.read(4)
        if magic != _CSR_MAGIC:
            raise ParseError(1, f"bad magic {magic!r}, expected {_CSR_MAGIC!r}")
        n, m = struct.unpack("<QQ", fh.read(16))  # struct.error on a short header, as the reference
        n, m = int(n), int(m)
        d_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        d_tgt = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
        with torch.cuda.device(dev):
            _stream_to_device(fh, d_off, 8 * (n + 1))
            _stream_to_device(fh, d_tgt, 4 * m)
    return make_csr(n, d_off, d_tgt, device=dev)


# -------------------------------------------------------------- generators
@dataclass(frozen=True)
class GraphGenSpec:
    """Parameters for one synthetic graph family (graph.py:50-83)."""

    kind: str  # uniform-random | power-law | star | ring | complete
    num_vertices: int
    target_edges: int | float | None = None
    exponent: float | None = None

    _KINDS = ("uniform-random", "power-law", "star", "ring", "complete")

    def __post_init__(self):
        if self.kind not in self._KINDS:
            raise ConfigError(f"unknown graph kind {self.kind!r}")
        if self.num_vertices < 1:
            raise ConfigError("num_vertices must be positive")
        if self.kind in ("uniform-random", "power-law"):
            if self.target_edges is None:
                raise ConfigError(f"{self.kind} requires target_edges")
            if isinstance(self.target_edges, float) and not 0 < self.target_edges < 1:
                raise ConfigError("edge probability must lie in (0, 1)")
        if self.kind == "power-law" and (self.exponent is None or self.exponent <= 1):
            raise ConfigError("power-law requires exponent > 1")

    def edge_count(self) -> int:
        n = self.num_vertices
        if isinstance(self.target_edges, float):
            return int(round(self.target_edges * n * n))
        return int(self.target_edges or 0)


def powerlaw_cdf(n: int, exponent: float) -> np.ndarray:
    """The float64 CDF of graph.py:256-259 (host, numpy pairwise sum — the
    device draws must search exactly this array to stay bit-exact)."""
    w = (np.arange(n, dtype=np.float64) + 1.0) ** (-1.0 / (exponent - 1.0))
    cdf = np.cumsum(w / w.sum())
    cdf[-1] = 1.0
    return cdf


def pcg64_seed_state(seed: int) -> tuple[int, int]:
    """(state, inc) of numpy's PCG64 seeded by SeedSequence(seed) — the
    generator graph.py:230 builds."""
    st = np.random.PCG64(np.random.SeedSequence(seed)).state["state"]
    return int(st["state"]), int(st["inc"])


def powerlaw_edges_device(n: int, m: int, exponent: float, seed: int, device=None):
    """Device (src, dst) int64 draws of graph.py:260-261, bit-exact."""
    lib = _lib.lib()
    dev = _device(device)
    cdf = torch.from_numpy(powerlaw_cdf(n, exponent)).to(dev)
    state, inc = pcg64_seed_state(seed)
    mask = (1 << 64) - 1
    with torch.cuda.device(dev):
        src = torch.empty(max(m, 1), dtype=torch.int64, device=dev)[:m]
        dst = torch.empty(max(m, 1), dtype=torch.int64, device=dev)[:m]
        ws = _lib.workspace(lib.gnn_generate_powerlaw_workspace(n), dev)
        _lib.check(lib.gnn_generate_powerlaw(n, m, cdf.data_ptr(), state >> 64, state & mask,
                                             inc >> 64, inc & mask,
                                             src.data_ptr() if m else None,
                                             dst.data_ptr() if m else None, ws.data_ptr(),
                                             ws.numel(), _lib.stream_handle(dev)),
                   "generate_powerlaw")
    return src, dst


def generate(spec: GraphGenSpec, seed: int, device=None) -> CsrGraph:
    """Deterministically generate a graph from (spec, seed) (graph.py:227-262).

    power-law: draws and CSR build on device, bit-exact with the reference.
    uniform-random: numpy's bounded-integer stream is not position-addressable,
    so the draws stay on the host (same calls as the reference) and only the
    CSR build runs on device.  star / ring / complete: closed-form CSR."""
    n = spec.num_vertices
    dev = _device(device)
    if spec.kind == "star":
        off = np.full(n + 1, n - 1, dtype=OFFSET_DTYPE)
        off[0] = 0
        return make_csr(n, off, np.arange(1, n, dtype=TARGET_DTYPE), device=dev)
    if spec.kind == "ring":
        off = np.arange(n + 1, dtype=OFFSET_DTYPE)
        tgt = ((np.arange(n, dtype=np.int64) + 1) % n).astype(TARGET_DTYPE)
        return make_csr(n, off, tgt, device=dev)
    if spec.kind == "complete":
        off = np.arange(n + 1, dtype=OFFSET_DTYPE) * (n - 1)
        ids = np.arange(n, dtype=np.int64)
        tgt = np.broadcast_to(ids, (n, n))[~np.eye(n, dtype=bool)].astype(TARGET_DTYPE)
        return make_csr(n, off, tgt, device=dev)
    m = spec.edge_count()
    if m > n * n:
        raise ConfigError(f"target_edges {m} exceeds n^2 = {n * n}")
    if spec.kind == "uniform-random":
        rng = np.random.default_rng(np.random.SeedSequence(seed))
        src = rng.integers(0, n, size=m, dtype=np.int64)
        dst = rng.integers(0, n, size=m, dtype=np.int64)
        return csr_from_edges(n, src, dst, device=dev)
    src, dst = powerlaw_edges_device(n, m, spec.exponent, seed, device=dev)
    g = csr_from_edges(n, src, dst, device=dev)
    del src, dst
    return g


# ------------------------------------------------ row-block (per-rank) build
def _sort_pairs(keys: torch.Tensor, vals: torch.Tensor, key_limit: int):
    """Stable device radix sort of int32 (key, val) pairs by key (gnn_sort_pairs)."""
    lib = _lib.lib()
    dev = keys.device
    n = int(keys.numel())
    ko = torch.empty(max(n, 1), dtype=torch.int32, device=dev)[:n]
    vo = torch.empty(max(n, 1), dtype=torch.int32, device=dev)[:n]
    with torch.cuda.device(dev):
        ws = _lib.workspace(lib.gnn_sort_pairs_workspace(n, max(int(key_limit), 1)), dev)
        _lib.check(lib.gnn_sort_pairs(n, max(int(key_limit), 1), keys.data_ptr() if n else None,
                                      vals.data_ptr() if n else None, ko.data_ptr() if n else None,
                                      vo.data_ptr() if n else None, ws.data_ptr(), ws.numel(),
                                      _lib.stream_handle(dev)), "sort_pairs")
        del ws
    return ko, vo


def _offsets_from_keys(sorted_keys: torch.Tensor, R: int) -> torch.Tensor:
    lib = _lib.lib()
    dev = sorted_keys.device
    n = int(sorted_keys.numel())
    off = torch.empty(R + 1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        ws = _lib.workspace(lib.gnn_offsets_from_keys_workspace(R), dev)
        _lib.check(lib.gnn_offsets_from_keys(n, R, sorted_keys.data_ptr() if n else None,
                                             off.data_ptr(), ws.data_ptr(), ws.numel(),
                                             _lib.stream_handle(dev)), "offsets_from_keys")
    return off


class RowBlock:
    """Rows [lo, hi) of a graph's CSR and of its transposed CSR (CSC), built
    on device without the rest of the graph (SURVEY §8e per-rank build).

    ``csr_offsets`` / ``csr_targets``: rows lo..hi-1 of csr_from_edges
    (graph.py:106-114), local row ids, global column ids; ``csc_offsets`` /
    ``csc_rows``: rows lo..hi-1 of the transposed CSR (in-edges of the owned
    vertices, source ids ascending, stream order within equal sources) —
    both bit-exact with the reference's arrays sliced to the block.
    ``csr_coalesced()`` / ``csc_coalesced()`` are the multiplicity-weighted
    unique-pair forms the trainers aggregate over; ``deg_offsets`` the
    canonical out-degree prefix of the block rows (every degree-norm)."""

    def __init__(self, num_vertices, num_edges, lo, hi, deg_offsets, csr=None, csc=None,
                 csr_co=None, csc_co=None, in_deg_offsets=None):
        self.num_vertices, self.num_edges = int(num_vertices), int(num_edges)
        self.lo, self.hi, self.rows = int(lo), int(hi), int(hi) - int(lo)
        self.deg_offsets = deg_offsets
        self.in_deg_offsets = in_deg_offsets
        self.csr_offsets, self.csr_targets = csr if csr is not None else (None, None)
        self.csc_offsets, self.csc_rows = csc if csc is not None else (None, None)
        self._csr_co, self._csc_co = csr_co, csc_co

    @property
    def device(self):
        return self.deg_offsets.device

    def csr_coalesced(self) -> SparseOperand:
        return self._csr_co

    def csc_coalesced(self) -> SparseOperand:
        return self._csc_co

    def nbytes(self) -> int:
        n = 0
        for t in (self.deg_offsets, self.in_deg_offsets, self.csr_offsets, self.csr_targets,
                  self.csc_offsets, self.csc_rows):
            if t is not None:
                n += t.numel() * t.element_size()
        for op in (self._csr_co, self._csc_co):
            if op is not None:
                n += op.nbytes()
        return n


def _block_capacity(spec: GraphGenSpec, lo: int, hi: int, cdf: np.ndarray) -> int:
    """Expected edges with an endpoint draw in [lo, hi) plus a 6-sigma margin
    (the block builder re-runs with the exact count if a block exceeds it)."""
    m = spec.edge_count()
    p = float(cdf[hi - 1] - (cdf[lo - 1] if lo > 0 else 0.0)) if hi > lo else 0.0
    mu = m * p
    return int(min(m, mu + 6.0 * np.sqrt(max(mu, 1.0)) + 8192))


def powerlaw_row_block(spec: GraphGenSpec, seed: int, lo: int, hi: int, device=None, *,
                       canonical: bool = False, coalesced: bool = True,
                       chunk: int = 1 << 26, pack: bool = True) -> RowBlock:
    """Build rows [lo, hi) of ``generate(spec, seed)`` (power-law) and of its
    transpose on device.  The bit-exact edge stream of graph.py:256-261 is
    regenerated in ``chunk``-edge pieces (gnn_powerlaw_block), keeping in
    stream order the edges with src (CSR) or dst (CSC) in the block; stable
    radix sorts then give the block's rows exactly as the reference's CSR and
    transposed CSR hold them.  Memory is O(block), not O(E): a rank of the
    row partition never holds the whole papers100M graph.  ``pack=False``
    keeps the coalesced forms unpacked (a partition re-packs after its id
    remap)."""
    if spec.kind != "power-law":
        raise ConfigError("row-block build covers the power-law generator")
    lib = _lib.lib()
    dev = _device(device)
    n, m = spec.num_vertices, spec.edge_count()
    if not 0 <= lo <= hi <= n:
        raise ValueError("block bounds outside [0, V]")
    R = hi - lo
    cdf_h = powerlaw_cdf(n, spec.exponent)
    cdf = torch.from_numpy(cdf_h).to(dev)
    state, inc = pcg64_seed_state(seed)
    mask = (1 << 64) - 1
    chunk = max(int(chunk), 4096)
    cap = _block_capacity(spec, lo, hi, cdf_h)
    i32 = dict(dtype=torch.int32, device=dev)
    count = torch.zeros(2, dtype=torch.int64, device=dev)
    for _attempt in range(2):
        rk, rv = torch.empty(max(cap, 1), **i32), torch.empty(max(cap, 1), **i32)
        ck, cv = torch.empty(max(cap, 1), **i32), torch.empty(max(cap, 1), **i32)
        with torch.cuda.device(dev):
            ws = _lib.workspace(lib.gnn_powerlaw_block_workspace(n, chunk), dev)
            _lib.check(lib.gnn_powerlaw_block(n, m, cdf.data_ptr(), state >> 64, state & mask,
                                              inc >> 64, inc & mask, lo, hi, chunk, cap,
                                              rk.data_ptr(), rv.data_ptr(), ck.data_ptr(),
                                              cv.data_ptr(), count.data_ptr(), ws.data_ptr(),
                                              ws.numel(), _lib.stream_handle(dev)),
                       "powerlaw_block")
            del ws
        nr, nc = (int(x) for x in count.tolist())
        if max(nr, nc) <= cap:
            break
        del rk, rv, ck, cv
        cap = max(nr, nc)  # rare: the block exceeded the 6-sigma margin; exact re-run
    del cdf
    rk, rv, ck, cv = rk[:nr], rv[:nr], ck[:nc], cv[:nc]
    # ---- CSR rows: stable by row (stream order within a row) = the canonical block
    csr = None
    if canonical:
        k1, t1 = _sort_pairs(rk, rv, R)
        csr = (_offsets_from_keys(k1, R), t1)
        del k1
    csr_co = None
    if coalesced:
        # (row, col) order: stable by col, then stable by row; then run-length coalesce
        c1, r1 = _sort_pairs(rv, rk, n)
        del rk, rv
        r2, c2 = _sort_pairs(r1, c1, R)
        del c1, r1
        deg_off = _offsets_from_keys(r2, R)
        del r2
        off, cols, mult = _coalesce(R, deg_off, c2)
        del c2
        csr_co = SparseOperand(R, n, off, cols, vals=mult, deg_offsets=deg_off, mult=True,
                               pack=pack)
    else:
        deg_off = csr[0] if csr is not None else _offsets_from_keys(_sort_pairs(rk, rv, R)[0], R)
        del rk, rv
    if csr is not None:
        deg_off = csr[0]
        if csr_co is not None:
            csr_co.deg_offsets = deg_off
    # ---- CSC rows: stable by source then by destination = the transposed CSR
    s1, d1 = _sort_pairs(cv, ck, n)
    del ck, cv
    d2, s2 = _sort_pairs(d1, s1, R)
    del s1, d1
    in_off = _offsets_from_keys(d2, R)
    del d2
    csc = (in_off, s2) if canonical else None
    csc_co = None
    if coalesced:
        off, rows, mult = _coalesce(R, in_off, s2)
        csc_co = SparseOperand(R, n, off, rows, vals=mult, deg_offsets=in_off, mult=True,
                               pack=pack)
    del s2
    return RowBlock(n, m, lo, hi, deg_off, csr=csr, csc=csc, csr_co=csr_co, csc_co=csc_co,
                    in_deg_offsets=in_off)


def fill_uniform(X: torch.Tensor, row0: int, seed: int) -> torch.Tensor:
    """X[i, k] = U[-1, 1) hash of (seed, (row0 + i) * K + k) in place
    (gnn_fill_uniform): rows of a global synthetic feature matrix, identical
    however the rows are partitioned."""
    lib = _lib.lib()
    with torch.cuda.device(X.device):
        _lib.check(lib.gnn_fill_uniform(X.data_ptr(), X.stride(0), X.shape[0], X.shape[1], row0,
                                        seed & ((1 << 64) - 1), _lib.stream_handle(X.device)),
                   "fill_uniform")
    return X


def fill_labels(y: torch.Tensor, row0: int, classes: int, seed: int) -> torch.Tensor:
    lib = _lib.lib()
    with torch.cuda.device(y.device):
        _lib.check(lib.gnn_fill_labels(y.data_ptr(), y.numel(), row0, classes,
                                       seed & ((1 << 64) - 1), _lib.stream_handle(y.device)),
                   "fill_labels")
    return y
