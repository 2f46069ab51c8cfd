"""1D row-partitioned multi-GPU GCN training.

One process per GPU.  Rank p owns the vertex range [bounds[p], bounds[p+1])
— contiguous row blocks balanced by EDGE count, not vertex count (the
power-law skew puts 28% of Reddit's edges in 115 rows) — and holds

  * its rows of the CSR (forward aggregation) and its rows of the CSC
    (= in-edges of its vertices, for the backward aggregation; SURVEY §8e
    option 1, symmetric with the forward so the kernels are identical);
  * column ids remapped once, on device, from global vertex ids to positions
    in a padded exchange buffer [P * Bmax, width]: vertex v of block q lives
    at q * Bmax + (v - bounds[q]).

Every layer writes its rows straight into its own slot of that buffer, and
one in-place all-gather (NCCL over NVLink / NVSwitch) fills the other slots
before the aggregation that needs them: four [V, hidden] all-gathers per GCN
epoch (H1, Y1 forward; dP2, dZ1 backward) plus one all-reduce of the ~42 KB of
weight gradients and the loss.  The exchanges are pluggable so the same
schedule runs on NCCL (``TorchDistExchange``) or as P virtual ranks inside one
process (``LocalExchange``, used by the single-GPU parity tests).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph, SparseOperand
from .kernels import AdamCall, GemmCall, MaskNormColsumCall, SpmmCall
from .models import glorot


# ----------------------------------------------------------- host logic
# Per-row cost of the GCN epoch in edge-equivalents: the SpMMs cost ~15 ps per
# (canonical) edge, the row-proportional work (X.W1 and X^T.dH1 at 602
# features, the fused head, mask/norm) ~2.6 ns per row on B200 (bench.py
# kernels_ms, Reddit shape) -> ~170 edges.  Balancing deg(r) + ROW_COST keeps
# both the sparse and the dense work even across ranks.
ROW_COST = 170


def partition_bounds(offsets: np.ndarray, parts: int, row_cost: float = 0.0) -> np.ndarray:
    """Row boundaries [P+1] of contiguous blocks of ~equal cost
    sum_r (deg(r) + row_cost); row_cost = 0 balances edges only
    (searchsorted on the cumulative cost; every block non-empty when V >= P)."""
    offsets = np.asarray(offsets)
    V = offsets.size - 1
    if parts <= 0:
        raise ValueError("parts must be positive")
    cum = offsets.astype(np.float64) + row_cost * np.arange(V + 1, dtype=np.float64)
    total = cum[-1]
    targets = total * np.arange(parts + 1, dtype=np.float64) / parts
    b = np.searchsorted(cum, targets, side="left").astype(np.int64)
    b[0], b[-1] = 0, V
    b = np.maximum.accumulate(np.minimum(b, V))
    # keep every block non-empty in rows when possible (P <= V)
    if V >= parts:
        for p in range(1, parts):
            b[p] = min(max(b[p], b[p - 1] + 1), V - (parts - p))
    return b


def expected_bounds(spec, parts: int, row_cost: float = 0.0) -> np.ndarray:
    """Row bounds for the power-law generator WITHOUT building the graph: the
    expected out-degree prefix of graph.py:256-261 is m * cdf (every edge's
    source is a draw from that CDF), so blocks of equal expected cost are
    found from the CDF alone.  Realised block sums differ from expectation by
    O(sqrt) — a fraction of a percent at the papers100M shape."""
    from .graph import powerlaw_cdf

    cdf = powerlaw_cdf(spec.num_vertices, spec.exponent)
    cum = np.concatenate([[0.0], spec.edge_count() * cdf])
    return partition_bounds(cum, parts, row_cost)


def remap_ids_host(ids: np.ndarray, bounds: np.ndarray, stride: int) -> np.ndarray:
    """Host statement of gnn_remap_ids (used by the CPU tests)."""
    ids = np.asarray(ids, dtype=np.int64)
    owner = np.searchsorted(bounds[1:-1], ids, side="right")
    return (owner * stride + ids - bounds[owner]).astype(np.int32)


def block_stride(bounds: np.ndarray) -> int:
    return int(max(1, np.max(np.diff(bounds))))


# ---------------------------------------------------------- exchanges
class TorchDistExchange:
    """All-gather / all-reduce through torch.distributed (NCCL on GPUs, gloo
    on CPU for the host-logic tests).  The all-gather is in place: the local
    block already sits in its slot of the padded buffer."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather(self, full: torch.Tensor, stride_rows: int, async_op: bool = False):
        d = self.dist
        mine = full[self.rank * stride_rows:(self.rank + 1) * stride_rows]
        if d.get_backend(self.group) == "nccl":
            return d.all_gather_into_tensor(full, mine, group=self.group, async_op=async_op)
        parts = list(full.split(stride_rows))
        return d.all_gather(parts, mine.clone(), group=self.group, async_op=async_op)

    def all_reduce(self, t: torch.Tensor):
        self.dist.all_reduce(t, group=self.group)

    def all_gather_start(self, full: torch.Tensor, stride_rows: int):
        """Launch the in-place all-gather (NCCL's own stream, ordered after the
        producer kernels) and return its work handle."""
        return self.all_gather(full, stride_rows, async_op=True)

    def all_gather_wait(self, handle):
        handle.wait()  # NCCL: the current stream waits on the collective, no host sync


class PeerExchange:
    """Peer-memory form of the exchange (one process per GPU): every rank's
    exchanged blocks live in torch symmetric memory, mapped into every peer
    over NVLink / NVSwitch; the aggregation kernels (gnn_spmm_peer) read the
    rows they need straight from the owner, so a phase boundary is only a
    device-side barrier — no all-gather copy.  Gradients still use one NCCL
    all-reduce.

    Opt-in (bench: GNN_DIST_EXCHANGE=peer), not the default: an aggregation
    re-reads every source row ~deg times, so in-place remote gathers move
    nnz*K*4 bytes over NVLink (Reddit, K=16: 4.4 GB, ~5 ms at 900 GB/s) where
    the all-gather moves each remote row once (V*K*4 = 15 MB) and the gathers
    then hit local L2/HBM.  Peer loads pay off for single-use operands (GEMM
    tiles), not for SpMM's high-reuse gathers."""

    def __init__(self, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        self.dist, self.symm, self.group = dist, symm, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.group_name = (group or dist.group.WORLD).group_name
        if hasattr(symm, "enable_symm_mem_for_group"):
            symm.enable_symm_mem_for_group(self.group_name)
        self.handles = []
        self.ptrs = {}

    def alloc(self, rows: int, width: int, device) -> torch.Tensor:
        """A [rows, width] fp32 block in symmetric memory (collective: every
        rank allocates its blocks in the same order); its peers' pointers are
        recorded under ptrs[id(tensor)]."""
        t = self.symm.empty(rows, width, dtype=torch.float32, device=device)
        t.zero_()
        h = self.symm.rendezvous(t, self.group_name)
        self.handles.append(h)
        self.ptrs[t.data_ptr()] = [int(p) for p in h.buffer_ptrs]
        return t

    def peer_ptrs(self, trainer) -> dict:
        return {n: self.ptrs[b.data_ptr()] for n, b in trainer.blocks().items()}

    def barrier(self):
        # device-side barrier over the group, stream-ordered (no host sync)
        self.handles[0].barrier(channel=0, timeout_ms=60_000)

    def all_reduce(self, t: torch.Tensor):
        self.dist.all_reduce(t, group=self.group)


class NullExchange:
    """The exchange of a single rank (N=1): every slot is already local."""

    world, rank = 1, 0

    def all_gather(self, full, stride_rows, async_op=False):
        return None

    def all_gather_start(self, full, stride_rows):
        return None

    def all_gather_wait(self, handle):
        pass

    def all_reduce(self, t):
        pass


class LocalExchange:
    """P virtual ranks in one process (one GPU): the exchanges copy slots
    between the ranks' buffers.  Used to test the partitioned schedule."""

    def __init__(self, world: int):
        self.world = world
        self.pending = {}

    def all_gather_many(self, fulls, stride_rows):
        for q, src in enumerate(fulls):
            blk = src[q * stride_rows:(q + 1) * stride_rows]
            for p, dst in enumerate(fulls):
                if p != q:
                    dst[q * stride_rows:(q + 1) * stride_rows].copy_(blk)

    def all_reduce_many(self, ts):
        tot = torch.stack(ts).sum(0)
        for t in ts:
            t.copy_(tot)


# ------------------------------------------------------------ partition
class RowPartition:
    """Rank ``rank``'s share of graph ``g`` (global CSR/CSC on this device)."""

    def __init__(self, g: CsrGraph, parts: int, rank: int, *, coalesced: bool = True,
                 bounds: np.ndarray | None = None, pow2_stride: bool = False):
        self.g = g
        self._setup(g.num_vertices, g.device, parts, rank,
                    partition_bounds(g.offsets, parts, ROW_COST) if bounds is None else bounds,
                    pow2_stride)
        cols_total = parts * self.stride
        # canonical row degrees of the owned rows (every degree-norm uses them)
        self.deg_offsets = (g.d_offsets[self.lo:self.hi + 1] - g.d_offsets[self.lo]).contiguous()
        if coalesced:
            A, AT = g.csr_coalesced(), g.csc_coalesced()
        else:
            A, AT = g.csr(), g.csc()
        self.A = self._slice(A, cols_total, deg=self.deg_offsets)
        self.AT = self._slice(AT, cols_total, deg=None)

    def _setup(self, num_vertices, device, parts, rank, bounds, pow2_stride):
        self.num_vertices, self.device = int(num_vertices), device
        self.parts, self.rank = parts, rank
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.stride = block_stride(self.bounds)
        if pow2_stride:  # peer mode: owner = id >> log2(stride), row = id & (stride - 1)
            self.stride = 1 << max(0, (self.stride - 1).bit_length())
        self.stride_log2 = self.stride.bit_length() - 1 if pow2_stride else None
        self.lo, self.hi = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.rows = self.hi - self.lo
        self.d_bounds = torch.from_numpy(self.bounds).to(device)

    @classmethod
    def from_block(cls, block, parts: int, rank: int, bounds, *,
                   pow2_stride: bool = False) -> "RowPartition":
        """Partition from this rank's own RowBlock (graph.powerlaw_row_block):
        the per-rank build, no global graph anywhere.  ``block`` must hold
        rows [bounds[rank], bounds[rank+1]) with coalesced forms."""
        self = cls.__new__(cls)
        self.g = None
        self._setup(block.num_vertices, block.device, parts, rank, bounds, pow2_stride)
        if (block.lo, block.hi) != (self.lo, self.hi):
            raise ValueError("row block does not match the partition bounds")
        cols_total = parts * self.stride
        self.deg_offsets = block.deg_offsets
        self.A = self._remap(block.csr_coalesced(), cols_total, deg=self.deg_offsets)
        self.AT = self._remap(block.csc_coalesced(), cols_total, deg=None)
        return self

    def _remap(self, op: SparseOperand, cols_total: int, deg) -> SparseOperand:
        """Block operand with global column ids -> exchange-buffer positions."""
        lib = _lib.lib()
        cols, vals = op.entries()
        nnz = int(cols.numel())
        out = torch.empty(max(nnz, 1), dtype=torch.int32, device=cols.device)[:nnz]
        with torch.cuda.device(cols.device):
            _lib.check(lib.gnn_remap_ids(nnz, cols.data_ptr() if nnz else None,
                                         self.d_bounds.data_ptr(), self.parts, self.stride,
                                         out.data_ptr() if nnz else None,
                                         _lib.stream_handle(cols.device)), "remap_ids")
        vals = vals.contiguous() if vals is not None else None
        del cols
        return SparseOperand(self.rows, cols_total, op.offsets, out, vals=vals,
                             deg_offsets=deg, mult=op.mult)

    def _slice(self, op: SparseOperand, cols_total: int, deg) -> SparseOperand:
        lib = _lib.lib()
        off = op.offsets[self.lo:self.hi + 1]
        e0, e1 = int(off[0].item()), int(off[-1].item())
        loc_off = (off - e0).contiguous()
        cols, vals = op.entries(e0, e1)
        out = torch.empty(e1 - e0, dtype=torch.int32, device=cols.device)
        with torch.cuda.device(cols.device):
            _lib.check(lib.gnn_remap_ids(e1 - e0, cols.data_ptr() if e1 > e0 else None,
                                         self.d_bounds.data_ptr(), self.parts, self.stride,
                                         out.data_ptr() if e1 > e0 else None,
                                         _lib.stream_handle(cols.device)), "remap_ids")
        vals = vals.contiguous() if vals is not None else None
        return SparseOperand(self.rows, cols_total, loc_off, out, vals=vals,
                             deg_offsets=deg if deg is not None else None, mult=op.mult)

    def split_local_remote(self, op: SparseOperand):
        """(local, remote) parts of a sliced operand: entries whose column is
        in this rank's own slot vs the others (order within a row kept).  The
        local part can aggregate while the all-gather of the other slots is
        still in flight (SURVEY §8e pipelining)."""
        dev = op.offsets.device
        R = op.num_rows
        lo, hi = self.rank * self.stride, (self.rank + 1) * self.stride
        deg = (op.offsets[1:] - op.offsets[:-1])
        rows = torch.repeat_interleave(torch.arange(R, device=dev), deg)
        cols, vals_all = op.entries()
        is_loc = (cols >= lo) & (cols < hi)
        out = []
        for sel in (is_loc, ~is_loc):
            idx = torch.nonzero(sel).squeeze(1)  # keeps row-major, in-row order
            cnt = torch.bincount(rows[idx], minlength=R)
            off = torch.zeros(R + 1, dtype=torch.int64, device=dev)
            torch.cumsum(cnt, 0, out=off[1:])
            vals = vals_all[idx].contiguous() if vals_all is not None else None
            out.append(SparseOperand(R, op.num_cols, off, cols[idx].contiguous(), vals=vals,
                                     deg_offsets=op.deg_offsets, mult=op.mult))
        return out[0], out[1]

    def local_rows(self, t: torch.Tensor) -> torch.Tensor:
        return t[self.lo:self.hi]


# ------------------------------------------------------------- trainer
class DistGCNTrainer:
    """One rank of the row-partitioned 2-layer GCN epoch (same math and
    kernels as ``models.GCNTrainer``; see the module docstring).

    Phases (exchanges between them):
      A  H1[slot] = X_loc W1                         -> all-gather H1
      B  Y1[slot] = relu(D^-1 A_loc H1 + b1)          -> all-gather Y1
      C  P2 = D^-1 A_loc Y1; head (loss scaled 1/V): dP2[slot], dW2, db2
                                                     -> all-gather dP2
      D  dZ1 = (A^T_loc dP2) * [Y1 > 0]; dZ1n[slot] = D^-1 dZ1, db1
                                                     -> all-gather dZ1n
      E  dH1 = A^T_loc dZ1n; dW1 = X_loc^T dH1       -> all-reduce grads+loss
      F  Adam (identical on every rank)
    """

    def __init__(self, part: RowPartition, in_feats: int, hidden: int, classes: int, *,
                 lr=0.01, seed: int = 0, peer: bool = False, alloc=None,
                 overlap: bool = False):
        """``peer``: exchanged blocks are read in place by gnn_spmm_peer (see
        PeerExchange / bind_peers) instead of being all-gathered; ``alloc``
        (rows, width, device) -> tensor provides the block storage (torch
        symmetric memory for real ranks, plain tensors for virtual ones).

        ``overlap`` (all-gather mode): every aggregation is split by source
        owner — the entries whose column is this rank's own slot aggregate
        while the all-gather of the other slots is in flight (on a comm
        stream), then the remote entries finish the row with the local partial
        as the SELF term (NORM distributes: acc_loc/d + acc_rem/d).  Same
        math, different fp32 summation order (tolerance, not bit-exact, vs
        the unsplit schedule)."""
        from .kernels import HeadCall

        self.part = part
        self.peer = peer
        if overlap and peer:
            raise ValueError("overlap applies to the all-gather exchange, not peer mode")
        self.overlap = overlap
        dev = part.device
        self.dev = dev
        V, n, S, P = part.num_vertices, part.rows, part.stride, part.parts
        self.V, self.F, self.Hd, self.C = V, in_feats, hidden, classes
        f32 = dict(dtype=torch.float32, device=dev)
        self.W1 = torch.from_numpy(glorot(in_feats, hidden, seed, 0)).to(dev)
        self.b1 = torch.zeros(hidden, **f32)
        self.W2 = torch.from_numpy(glorot(hidden, classes, seed, 2)).to(dev)
        self.b2 = torch.zeros(classes, **f32)
        # one flat gradient buffer (+ loss) -> a single all-reduce
        sizes = [in_feats * hidden, hidden, hidden * classes, classes, 1]
        self.flat = torch.zeros(sum(sizes), **f32)
        views = list(self.flat.split(sizes))
        self.dW1 = views[0].view(in_feats, hidden)
        self.db1, self.db2 = views[1], views[3]
        self.dW2 = views[2].view(hidden, classes)
        self.loss = views[4]
        self.Fpad = -(-in_feats // 32) * 32
        self._Xstore = torch.zeros(max(n, 1), self.Fpad, **f32)
        self.X = self._Xstore[:n, :in_feats]
        self.labels = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)[:n]
        if peer:
            if part.stride_log2 is None:
                raise ValueError("peer mode needs RowPartition(..., pow2_stride=True)")
            mk = alloc or (lambda r, w, d: torch.zeros(r, w, dtype=torch.float32, device=d))
            # local blocks only; peers' blocks are read in place
            self.H1f, self.Y1f, self.dP2f, self.dZ1f = (mk(S, hidden, dev) for _ in range(4))
            sl = slice(0, n)
        else:
            full = lambda: torch.zeros(P * S, hidden, **f32)  # noqa: E731
            self.H1f, self.Y1f, self.dP2f, self.dZ1f = full(), full(), full(), full()
            sl = slice(part.rank * S, part.rank * S + n)
        self.H1, self.Y1 = self.H1f[sl], self.Y1f[sl]
        self.dP2, self.dZ1n = self.dP2f[sl], self.dZ1f[sl]
        e = lambda: torch.empty(max(n, 1), hidden, **f32)[:n]  # noqa: E731
        self.P2, self.dZ1, self.dH1 = e(), e(), e()
        A, AT = part.A, part.AT
        N_, B_, R_, M_ = _lib.EPI_NORM, _lib.EPI_BIAS, _lib.EPI_RELU, _lib.EPI_MASK
        deg = part.deg_offsets
        self.phases = []
        self._lazy = {}  # peer mode: aggregation calls built by bind_peers()
        # overlap: pre[name] runs before the pending all-gather is waited on
        pre = {k: [] for k in ("agg1", "agg2", "bagg2", "bagg1")}
        if n > 0 and overlap:
            S_ = _lib.EPI_SELF
            self.tmp = e()
            A_l, A_r = part.split_local_remote(A)
            AT_l, AT_r = part.split_local_remote(AT)
            self.split_nnz = {"A": (A_l.nnz, A_r.nnz), "AT": (AT_l.nnz, AT_r.nnz)}
            t = self.tmp
            pre["agg1"] = [("agg1.local", SpmmCall(A_l, self.H1f, t, flags=N_))]
            k_agg1 = SpmmCall(A_r, self.H1f, self.Y1, flags=N_ | S_ | B_ | R_, bias=self.b1,
                              self_x=t)
            pre["agg2"] = [("agg2.local", SpmmCall(A_l, self.Y1f, t, flags=N_))]
            k_agg2 = SpmmCall(A_r, self.Y1f, self.P2, flags=N_ | S_, self_x=t)
            pre["bagg2"] = [("bagg2.local", SpmmCall(AT_l, self.dP2f, t))]
            k_bagg2_ov = SpmmCall(AT_r, self.dP2f, self.dZ1, flags=S_ | M_, self_x=t,
                                  mask=self.Y1)
            pre["bagg1"] = [("bagg1.local", SpmmCall(AT_l, self.dZ1f, t))]
            k_bagg1_ov = SpmmCall(AT_r, self.dZ1f, self.dH1, flags=S_, self_x=t)
        if n > 0:
            k_gemm1 = GemmCall(self.X, self.W1, self.H1)
            if peer:
                k_agg1 = self._deferred("agg1")
                k_agg2 = self._deferred("agg2")
            elif not overlap:
                k_agg1 = SpmmCall(A, self.H1f, self.Y1, flags=N_ | B_ | R_, bias=self.b1)
                k_agg2 = SpmmCall(A, self.Y1f, self.P2, flags=N_)
            # loss and dZ scaled 1/V_global: the all-reduce sums to the single-GPU mean
            k_head = HeadCall(self.P2, self.W2, self.b2, self.labels, self.dP2, self.dW2,
                              self.db2, self.loss, deg_offsets=deg, scale=1.0 / V)
            if peer:
                k_bagg2 = self._deferred("bagg2")
                k_bagg1 = self._deferred("bagg1")
            elif overlap:
                k_bagg2, k_bagg1 = k_bagg2_ov, k_bagg1_ov
            else:
                k_bagg2 = SpmmCall(AT, self.dP2f, self.dZ1, flags=M_, mask=self.Y1)
                k_bagg1 = SpmmCall(AT, self.dZ1f, self.dH1)
            k_norm1 = MaskNormColsumCall(self.dZ1, self.dZ1n, deg_offsets=deg, colsum=self.db1)
            k_dW1 = GemmCall(self.X, self.dH1, self.dW1, trans_a=True)
            zero = lambda: None  # noqa: E731
        else:  # a rank without rows still takes part in every exchange
            k_gemm1 = k_agg1 = k_agg2 = k_bagg2 = k_norm1 = k_bagg1 = k_dW1 = lambda: None  # noqa: E731
            k_head = None
            zero = self.flat.zero_
        self._head = k_head
        # (name, calls before the previous exchange is waited on, calls after, exchange)
        self.phases = [
            ("A", [], [("X.W1", k_gemm1)], ("gather", self.H1f)),
            ("B", pre["agg1"], [("agg1", k_agg1)], ("gather", self.Y1f)),
            ("C", pre["agg2"], [("agg2", k_agg2), ("head", k_head if n > 0 else zero)],
             ("gather", self.dP2f)),
            ("D", pre["bagg2"], [("bagg2", k_bagg2), ("mask_norm_db1", k_norm1)],
             ("gather", self.dZ1f)),
            ("E", pre["bagg1"], [("bagg1", k_bagg1), ("X^T.dH1", k_dW1)], ("reduce", self.flat)),
        ]
        self.k_adam = AdamCall([self.W1, self.b1, self.W2, self.b2],
                               [self.dW1, self.db1, self.dW2, self.db2], lr=lr)

    def _deferred(self, name):
        def call():
            self._lazy[name]()
        return call

    def blocks(self) -> dict:
        """The exchanged blocks of this rank (peer mode: what peers read)."""
        return {"H1": self.H1f, "Y1": self.Y1f, "dP2": self.dP2f, "dZ1": self.dZ1f}

    def bind_peers(self, ptrs: dict) -> None:
        """Peer mode: ``ptrs[name][q]`` = device pointer of rank q's block
        ``name`` (peer-mapped for real ranks); builds the gnn_spmm_peer calls."""
        from .kernels import PeerSpmmCall

        if self.part.rows == 0:
            return
        part, hd = self.part, self.Hd
        lg, ld = part.stride_log2, hd
        N_, B_, R_, M_ = _lib.EPI_NORM, _lib.EPI_BIAS, _lib.EPI_RELU, _lib.EPI_MASK
        self._lazy = {
            "agg1": PeerSpmmCall(part.A, ptrs["H1"], lg, ld, hd, self.Y1, flags=N_ | B_ | R_,
                                 bias=self.b1),
            "agg2": PeerSpmmCall(part.A, ptrs["Y1"], lg, ld, hd, self.P2, flags=N_),
            "bagg2": PeerSpmmCall(part.AT, ptrs["dP2"], lg, ld, hd, self.dZ1, flags=M_,
                                  mask=self.Y1),
            "bagg1": PeerSpmmCall(part.AT, ptrs["dZ1"], lg, ld, hd, self.dH1),
        }

    def set_inputs(self, X_local, labels_local, non_blocking=False):
        """X_local: [rows, F], or [rows, Fpad] already at the device row stride
        (one linear copy — a pitched H2D copy is ~3x slower over PCIe)."""
        n = self.part.rows
        if X_local.shape[1] == self.Fpad and X_local.shape[1] != self.F:
            self._Xstore[:n].copy_(X_local, non_blocking=non_blocking)
        else:
            _lib.copy_rows(self.X, X_local)
        self.labels.copy_(labels_local, non_blocking=non_blocking)

    def step(self, ex):
        S = self.part.stride
        pending = None
        for _, pre, calls, (kind, buf) in self.phases:
            for _, c in pre:  # own-slot aggregation, overlapping the all-gather
                c()
            if pending is not None:
                ex.all_gather_wait(pending)
                pending = None
            for _, c in calls:
                c()
            if kind == "gather":
                if self.peer:
                    ex.barrier()  # the block is complete on every rank; peers read it in place
                elif self.overlap:
                    pending = ex.all_gather_start(buf, S)
                else:
                    ex.all_gather(buf, S)
            else:
                ex.all_reduce(buf)
        self.k_adam()
        return self.loss

    def timed_step(self, ex) -> dict:
        """One epoch with CUDA events around every launch and exchange on the
        current stream (exchanges unoverlapped, so each is timed alone);
        returns {name: ms}."""
        st = torch.cuda.current_stream(self.dev)
        S = self.part.stride
        marks = []

        def mark(name, fn):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            marks.append((name, a, b))

        torch.cuda.synchronize(self.dev)
        for _, pre, calls, (kind, buf) in self.phases:
            for name, c in list(pre) + list(calls):
                mark(name, c)
            if kind == "gather":
                if self.peer:
                    mark("barrier", ex.barrier)
                else:
                    mark("all_gather", lambda: ex.all_gather(buf, S))
            else:
                mark("all_reduce", lambda: ex.all_reduce(buf))
        mark("adam", self.k_adam)
        torch.cuda.synchronize(self.dev)
        out = {}
        for name, a, b in marks:
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out

    def params(self):
        return {"W1": self.W1, "b1": self.b1, "W2": self.W2, "b2": self.b2}

    def grads(self):
        return {"W1": self.dW1, "b1": self.db1, "W2": self.dW2, "b2": self.db2}


def bind_virtual_peers(trainers) -> None:
    """Peer mode with P virtual ranks on one GPU: every rank reads the other
    ranks' blocks directly (same device), exactly as real ranks read peer-
    mapped NVLink memory."""
    names = ("H1", "Y1", "dP2", "dZ1")
    ptrs = {n: [t.blocks()[n].data_ptr() for t in trainers] for n in names}
    for t in trainers:
        t.bind_peers(ptrs)


def step_virtual(trainers, ex: LocalExchange, adam: bool = True):
    """One epoch of P virtual ranks (``trainers[p]`` = rank p) in lockstep.
    Peer-mode trainers need no exchange: phase order on the one stream is the
    barrier."""
    S = trainers[0].part.stride
    pending = None
    for i in range(len(trainers[0].phases)):
        for t in trainers:  # overlap: own-slot parts run before the slots land
            for _, c in t.phases[i][1]:
                c()
        if pending is not None:
            ex.all_gather_many(pending, S)
            pending = None
        for t in trainers:
            for _, c in t.phases[i][2]:
                c()
        kind = trainers[0].phases[i][3][0]
        bufs = [t.phases[i][3][1] for t in trainers]
        if kind == "gather" and trainers[0].overlap:
            pending = bufs
        elif kind == "gather":
            if not trainers[0].peer:
                ex.all_gather_many(bufs, S)
        else:
            ex.all_reduce_many(bufs)
    if adam:
        for t in trainers:
            t.k_adam()
    return trainers[0].loss
