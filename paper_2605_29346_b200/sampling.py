"""Device sampled-block pipeline: the reference's
per-iteration sampler (``gsbench/sampler.py``) with the same names, argument
meaning, RNG contract and exceptions, running on libgnnb200 kernels:

  * ``sample_hop``      sampler.py:118-144 — draws bit-exact with numpy's PCG64
                        stream (device jump-ahead), ``pick = floor(u * deg)``;
  * ``SubgraphBuilder`` sampler.py:146-188 — device global->local table;
  * ``dedup_relabel``   sampler.py:191-239 — first-occurrence local ids
                        (deterministic: atomicMin of positions + stable scan);
  * ``build_subgraph_csr`` sampler.py:242-256 — device stable CSR build;
  * ``sample_minibatch`` sampler.py:259-296 — one count read per hop (to size
                        the next frontier); everything else stays on device.

Results (``HopBlock`` / ``SampledSubgraph`` / ``IterationMetadata``) hold
numpy arrays like the reference's, copied from device once per mini-batch;
``sample_minibatch(..., on_device=True)`` keeps them as device tensors.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Union

import numpy as np
import torch

from . import _lib
from .errors import ConfigError
from .graph import CsrGraph
from .graph import build_subgraph_csr as _device_subgraph_csr

LOCAL_DTYPE = np.int32
SeedLike = Union[int, np.random.SeedSequence, None]
_INT32_MAX = 2**31 - 1


@dataclass(frozen=True)
class SampleConfig:
    """Mini-batch size B and per-hop fanouts F_1..F_N (sampler.py:29-47)."""

    batch_size: int
    fanouts: tuple
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "fanouts", tuple(int(f) for f in self.fanouts))
        if self.batch_size < 1:
            raise ConfigError("batch_size must be >= 1")
        if len(self.fanouts) < 1:
            raise ConfigError("at least one hop is required")
        if any(f < 0 for f in self.fanouts):
            raise ConfigError("fanouts must be nonnegative")

    @property
    def num_hops(self) -> int:
        return len(self.fanouts)


@dataclass
class HopBlock:
    hop_index: int
    src_local: object
    dst_unique_local: object
    edge_src: object
    edge_dst: object
    raw_draw_count: int


@dataclass
class SampledSubgraph:
    hops: list
    local_to_global: object

    @property
    def num_local_vertices(self) -> int:
        return int(self.local_to_global.shape[0])


@dataclass(frozen=True)
class IterationMetadata:
    batch_size: int
    per_hop_vertex_counts: tuple
    per_hop_edge_counts: tuple
    total_unique_vertices: int
    total_edges: int

    @property
    def num_hops(self) -> int:
        return len(self.per_hop_vertex_counts)


def _as_seed_sequence(rng: SeedLike, default_seed: int) -> np.random.SeedSequence:
    if rng is None:
        return np.random.SeedSequence(default_seed)
    if isinstance(rng, np.random.SeedSequence):
        return rng
    return np.random.SeedSequence(int(rng))


def hop_state(base: np.random.SeedSequence, hop: int) -> tuple[int, int]:
    """(state, inc) of the hop's PCG64 stream: sampler.py:99-107 appends the
    1-based hop index to the base spawn key."""
    if base.entropy is None:
        raise ConfigError("entropy-less seed sequences cannot be re-derived on device")
    child = np.random.SeedSequence(base.entropy, spawn_key=tuple(base.spawn_key) + (hop,))
    st = np.random.PCG64(child).state["state"]
    return int(st["state"]), int(st["inc"])


def _i64(x, dev) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.int64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64)).to(dev)


def _pcg64_words(rng) -> tuple[int, int]:
    """(state, inc) of a numpy PCG64 stream: a ``np.random.Generator`` over
    PCG64 (the reference's argument, sampler.py:118-123) or a raw
    ``(state, inc)`` tuple."""
    if isinstance(rng, np.random.Generator):
        bg = rng.bit_generator
        if not isinstance(bg, np.random.PCG64):
            raise ConfigError("device sample_hop reproduces numpy's PCG64 stream only")
        st = bg.state["state"]
        return int(st["state"]), int(st["inc"])
    s, inc = rng
    return int(s), int(inc)


def sample_hop(graph: CsrGraph, frontier, fanout: int, rng):
    """Device sample_hop (sampler.py:118-144): (src, dst) int64 device tensors
    of the hop's draws, bit-exact with the reference for the same generator.

    ``rng`` is the reference's ``np.random.Generator`` (PCG64): the draws use
    its current stream position and, like ``rng.random(n)`` in the reference,
    the generator is advanced past the n doubles consumed.  A raw PCG64
    ``(state, inc)`` tuple is accepted too (used by the device pipeline)."""
    lib = _lib.lib()
    dev = graph.device
    fr = _i64(frontier, dev)
    F = int(fr.numel())
    cap = F * int(fanout)
    src = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    dst = torch.empty_like(src)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    s, inc = _pcg64_words(rng)
    mask = (1 << 64) - 1
    with torch.cuda.device(dev):
        ws = _lib.workspace(lib.gnn_sample_hop_workspace(F), dev)
        _lib.check(lib.gnn_sample_hop(graph.num_vertices, graph.d_offsets.data_ptr(),
                                      graph._device_targets().data_ptr(),
                                      fr.data_ptr() if F else None, F, int(fanout), s >> 64,
                                      s & mask, inc >> 64, inc & mask, src.data_ptr(),
                                      dst.data_ptr(), count.data_ptr(), ws.data_ptr(), ws.numel(),
                                      _lib.stream_handle(dev)), "sample_hop")
    n = int(count.item())  # one read per hop: sizes the next hop
    if isinstance(rng, np.random.Generator) and n:
        rng.bit_generator.advance(n)  # the reference consumed n doubles (sampler.py:142)
    return src[:n], dst[:n]


def _check_seeds(seeds, num_vertices: int) -> np.ndarray:
    """The reference's seed-batch checks (sampler.py:153-160): non-empty,
    distinct, inside [0, V) — ConfigError otherwise."""
    s = np.asarray(seeds.cpu() if isinstance(seeds, torch.Tensor) else seeds, dtype=np.int64)
    s = s.reshape(-1)
    if s.size == 0:
        raise ConfigError("seed batch must be non-empty")
    if np.unique(s).size != s.size:
        raise ConfigError("seed vertices must be distinct")
    if s.min() < 0 or s.max() >= num_vertices:
        raise ConfigError("seed vertex id out of range")
    return s


class SubgraphBuilder:
    """Device twin of sampler.py:146-188: seeds take locals 0..B-1; the
    global->local table is an int32 device array over the base graph."""

    def __init__(self, num_vertices: int, seeds, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        s = _check_seeds(seeds, num_vertices)
        self.dev = dev
        self.num_vertices = num_vertices
        self.table = torch.full((num_vertices,), -1, dtype=torch.int32, device=dev)
        self.firstpos = torch.full((num_vertices,), _INT32_MAX, dtype=torch.int32, device=dev)
        seeds_d = torch.from_numpy(s).to(dev)
        lib = _lib.lib()
        with torch.cuda.device(dev):
            _lib.check(lib.gnn_table_assign(self.table.data_ptr(), seeds_d.data_ptr(), s.size, 0,
                                            _lib.stream_handle(dev)), "table_assign")
        self._chunks = [seeds_d]
        self._size = int(s.size)
        self.hops: list[HopBlock] = []

    @property
    def num_local_vertices(self) -> int:
        return self._size

    def add_hop(self, hop_index: int, frontier, src_global, dst_global) -> HopBlock:
        block = dedup_relabel(src_global, dst_global, self, hop_index, frontier=frontier)
        self.hops.append(block)
        return block

    def finish(self) -> SampledSubgraph:
        l2g = torch.cat(self._chunks) if len(self._chunks) > 1 else self._chunks[0]
        return SampledSubgraph(hops=self.hops, local_to_global=l2g)


def dedup_relabel(src_global, dst_global, builder: SubgraphBuilder, hop_index: int,
                  frontier=None) -> HopBlock:
    """sampler.py:191-239 on device: ValueError when a draw's source is not
    yet in the subgraph; first-seen destinations get fresh locals in
    first-occurrence order."""
    lib = _lib.lib()
    dev = builder.dev
    sg = _i64(src_global, dev)
    dg = _i64(dst_global, dev)
    n = int(sg.numel())
    src_l = torch.empty(max(n, 1), dtype=torch.int32, device=dev)[:n]
    dst_l = torch.empty(max(n, 1), dtype=torch.int32, device=dev)[:n]
    new_g = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    start = builder._size
    with torch.cuda.device(dev):
        ws = _lib.workspace(lib.gnn_dedup_relabel_workspace(n), dev)
        _lib.check(lib.gnn_dedup_relabel(
            builder.num_vertices, builder.table.data_ptr(), builder.firstpos.data_ptr(),
            sg.data_ptr() if n else None, dg.data_ptr() if n else None, n, start,
            src_l.data_ptr() if n else None, dst_l.data_ptr() if n else None, new_g.data_ptr(),
            cnt.data_ptr(), err.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle(dev)),
            "dedup_relabel")
    k = int(cnt.item())
    if int(err.item()):
        raise ValueError("hop source vertex not present in subgraph")
    new_g = new_g[:k]
    if k:
        builder._chunks.append(new_g)
        builder._size = start + k
    new_locals = torch.arange(start, start + k, dtype=torch.int32, device=dev)
    if frontier is not None:
        fr = _i64(frontier, dev)
        fl = torch.empty(max(fr.numel(), 1), dtype=torch.int32, device=dev)[:fr.numel()]
        if fr.numel():
            with torch.cuda.device(dev):
                _lib.check(lib.gnn_table_lookup(builder.table.data_ptr(), fr.data_ptr(),
                                                fr.numel(), fl.data_ptr(),
                                                _lib.stream_handle(dev)), "table_lookup")
    else:  # the draw sources, unique in first-occurrence order (host fallback path)
        u, pos = np.unique(src_l.cpu().numpy(), return_index=True)
        fl = torch.from_numpy(u[np.argsort(pos, kind="stable")].astype(LOCAL_DTYPE)).to(dev)
    return HopBlock(hop_index=hop_index, src_local=fl, dst_unique_local=new_locals,
                    edge_src=src_l, edge_dst=dst_l, raw_draw_count=n)


def build_subgraph_csr(edge_src, edge_dst, num_local_src: int):
    """sampler.py:242-256 on device (stable CSR of a sampled block)."""
    return _device_subgraph_csr(edge_src, edge_dst, num_local_src)


def _to_host(sg: SampledSubgraph) -> SampledSubgraph:
    hops = [HopBlock(b.hop_index, b.src_local.cpu().numpy(), b.dst_unique_local.cpu().numpy(),
                     b.edge_src.cpu().numpy(), b.edge_dst.cpu().numpy(), b.raw_draw_count)
            for b in sg.hops]
    l2g = sg.local_to_global.cpu().numpy()
    l2g.setflags(write=False)
    return SampledSubgraph(hops=hops, local_to_global=l2g)


def sample_minibatch(graph: CsrGraph, config: SampleConfig, seed_vertices, rng: SeedLike = None,
                     on_device: bool = False):
    """sampler.py:259-296 on device: hop h's frontier is hop h-1's new
    destinations (hop 1: the seeds); deterministic for fixed (seeds, rng)."""
    seeds = np.asarray(seed_vertices.cpu() if isinstance(seed_vertices, torch.Tensor)
                       else seed_vertices, dtype=np.int64)
    if seeds.size != config.batch_size:
        raise ConfigError(f"expected {config.batch_size} seed vertices, got {seeds.size}")
    base = _as_seed_sequence(rng, config.seed)
    builder = SubgraphBuilder(graph.num_vertices, seeds, device=graph.device)
    vc, ec = [], []
    frontier = builder._chunks[0]
    for hop, fanout in enumerate(config.fanouts, 1):
        src, dst = sample_hop(graph, frontier, fanout, hop_state(base, hop))
        block = builder.add_hop(hop, frontier, src, dst)
        vc.append(builder.num_local_vertices)
        ec.append(block.raw_draw_count)
        frontier = (builder._chunks[-1] if block.dst_unique_local.numel()
                    else torch.empty(0, dtype=torch.int64, device=graph.device))
    sg = builder.finish()
    meta = IterationMetadata(batch_size=int(seeds.size), per_hop_vertex_counts=tuple(vc),
                             per_hop_edge_counts=tuple(ec),
                             total_unique_vertices=builder.num_local_vertices,
                             total_edges=int(sum(ec)))
    return (sg if on_device else _to_host(sg)), meta


def gather_indices(subgraph: SampledSubgraph):
    """sampler.py:299-305: feature rows = every sampled vertex, label rows =
    the seed batch."""
    batch = subgraph.hops[0].src_local.shape[0] if subgraph.hops else 0
    l2g = subgraph.local_to_global
    feat = l2g.clone() if isinstance(l2g, torch.Tensor) else np.array(l2g, copy=True)
    return feat, feat[:batch].clone() if isinstance(feat, torch.Tensor) else feat[:batch].copy()


class DeviceSampler:
    """Host-sync-free, replayable ``sample_minibatch`` (ZeroGNN's device-
    resident metadata + capture/replay; the
    reference models it in execmodel.py:430-490).  Every buffer is
    provisioned for the worst-case envelope of ``config`` (hop h: frontier ≤
    B·Π_{i<h} F_i, draws ≤ frontier·F_h); counts live in device scalars;
    kernels cover the capacity and exit early past the live count.  One
    mini-batch = one CUDA graph replay that also copies the seeds and the
    per-hop PCG64 states in from pinned host memory.  ``result()`` reads the
    sampled blocks back (bit-exact with ``sample_minibatch``)."""

    def __init__(self, graph: CsrGraph, config: SampleConfig):
        lib = _lib.lib()
        self.lib, self.g, self.cfg = lib, graph, config
        dev = graph.device
        self.dev = dev
        B, H = config.batch_size, config.num_hops
        i64 = dict(dtype=torch.int64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self.table = torch.full((graph.num_vertices,), -1, **i32)
        self.firstpos = torch.full((graph.num_vertices,), _INT32_MAX, **i32)
        self.size = torch.zeros(1, **i64)
        self.err = torch.zeros(1, **i32)
        self.seeds = torch.zeros(B, **i64)
        self.B_dev = torch.full((1,), B, **i64)
        self.rng = torch.zeros(H, 4, dtype=torch.int64, device=dev)  # uint64 words
        self.seeds_h = torch.zeros(B, dtype=torch.int64).pin_memory()
        self.rng_h = torch.zeros(H, 4, dtype=torch.int64).pin_memory()
        self._inflight = None  # event after the last replay's staging copies
        self.hops = []
        f_cap = B
        for h, fan in enumerate(config.fanouts):
            n_cap = f_cap * fan
            hop = dict(
                f_cap=f_cap, n_cap=n_cap, fanout=fan,
                src=torch.empty(max(n_cap, 1), **i64), dst=torch.empty(max(n_cap, 1), **i64),
                count=torch.zeros(1, **i64), new_count=torch.zeros(1, **i64),
                src_local=torch.empty(max(n_cap, 1), **i32),
                dst_local=torch.empty(max(n_cap, 1), **i32),
                new_globals=torch.empty(max(n_cap, 1), **i64),
                frontier_local=torch.empty(max(f_cap, 1), **i32),
                ws_s=_lib.workspace(lib.gnn_sample_hop_dev_workspace(f_cap), dev),
                ws_d=_lib.workspace(lib.gnn_dedup_relabel_dev_workspace(n_cap), dev))
            self.hops.append(hop)
            f_cap = n_cap
        self.graph = None

    def _launch(self):
        lib, g, st = self.lib, self.g, _lib.stream_handle(self.dev)
        B = self.cfg.batch_size
        self.err.zero_()  # an error flag never sticks to later batches
        self.seeds.copy_(self.seeds_h, non_blocking=True)
        self.rng.copy_(self.rng_h, non_blocking=True)
        _lib.check(lib.gnn_table_assign(self.table.data_ptr(), self.seeds.data_ptr(), B, 0, st),
                   "table_assign")
        self.size.fill_(B)
        frontier, f_dev = self.seeds, self.B_dev
        tgt = g._device_targets()
        for h, hop in enumerate(self.hops):
            _lib.check(lib.gnn_sample_hop_dev(
                g.num_vertices, g.d_offsets.data_ptr(), tgt.data_ptr(), frontier.data_ptr(),
                f_dev.data_ptr(), hop["f_cap"], hop["fanout"], self.rng[h].data_ptr(),
                hop["src"].data_ptr(), hop["dst"].data_ptr(), hop["count"].data_ptr(),
                hop["ws_s"].data_ptr(), hop["ws_s"].numel(), st), "sample_hop_dev")
            _lib.check(lib.gnn_dedup_relabel_dev(
                g.num_vertices, self.table.data_ptr(), self.firstpos.data_ptr(),
                hop["src"].data_ptr(), hop["dst"].data_ptr(), hop["count"].data_ptr(),
                hop["n_cap"], self.size.data_ptr(), hop["src_local"].data_ptr(),
                hop["dst_local"].data_ptr(), hop["new_globals"].data_ptr(),
                hop["new_count"].data_ptr(), self.err.data_ptr(), hop["ws_d"].data_ptr(),
                hop["ws_d"].numel(), st), "dedup_relabel_dev")
            _lib.check(lib.gnn_table_lookup_dev(self.table.data_ptr(), frontier.data_ptr(),
                                                f_dev.data_ptr(), hop["f_cap"],
                                                hop["frontier_local"].data_ptr(), st),
                       "table_lookup_dev")
            frontier, f_dev = hop["new_globals"], hop["new_count"]
        # reset the table for the next mini-batch (seeds + every hop's new vertices)
        _lib.check(lib.gnn_table_fill_dev(self.table.data_ptr(), self.seeds.data_ptr(), None, B,
                                          -1, st), "table_fill_dev")
        for hop in self.hops:
            _lib.check(lib.gnn_table_fill_dev(self.table.data_ptr(), hop["new_globals"].data_ptr(),
                                              hop["new_count"].data_ptr(), hop["n_cap"], -1, st),
                       "table_fill_dev")

    def _stage(self, seeds, rng: SeedLike):
        s = np.asarray(seeds.cpu() if isinstance(seeds, torch.Tensor) else seeds, dtype=np.int64)
        if s.size != self.cfg.batch_size:
            raise ConfigError(f"expected {self.cfg.batch_size} seed vertices, got {s.size}")
        s = _check_seeds(s, self.g.num_vertices)  # out-of-range ids would index offsets[] OOB
        base = _as_seed_sequence(rng, self.cfg.seed)
        if self._inflight is not None:
            # the previous replay's H2D copies read these pinned buffers: wait for them
            self._inflight.synchronize()
            self._inflight = None
        self.seeds_h.copy_(torch.from_numpy(s))
        words = []
        for h in range(1, self.cfg.num_hops + 1):
            st, inc = hop_state(base, h)
            words.append([st >> 64, st & ((1 << 64) - 1), inc >> 64, inc & ((1 << 64) - 1)])
        self.rng_h.copy_(torch.from_numpy(np.array(words, dtype=np.uint64).view(np.int64)))

    def capture(self):
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            self._launch()
        torch.cuda.current_stream(self.dev).wait_stream(s)
        torch.cuda.synchronize(self.dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self._launch()
        self.graph = graph
        return graph

    def run(self, seeds, rng: SeedLike = None):
        """One mini-batch: stage seeds + RNG states in pinned memory, replay."""
        self._stage(seeds, rng)
        if self.graph is None:
            self._launch()
        else:
            self.graph.replay()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev))
        self._inflight = ev

    def result(self):
        """(SampledSubgraph, IterationMetadata) with host arrays (synchronises)."""
        torch.cuda.synchronize(self.dev)
        if int(self.err.item()):
            raise ValueError("hop source vertex not present in subgraph")
        B = self.cfg.batch_size
        chunks = [self.seeds.cpu().numpy()]
        hops, vc, ec = [], [], []
        size = B
        for h, hop in enumerate(self.hops):
            n, k = int(hop["count"].item()), int(hop["new_count"].item())
            f = B if h == 0 else int(self.hops[h - 1]["new_count"].item())
            new_l = np.arange(size, size + k, dtype=LOCAL_DTYPE)
            size += k
            chunks.append(hop["new_globals"][:k].cpu().numpy())
            hops.append(HopBlock(h + 1, hop["frontier_local"][:f].cpu().numpy(), new_l,
                                 hop["src_local"][:n].cpu().numpy(),
                                 hop["dst_local"][:n].cpu().numpy(), n))
            vc.append(size)
            ec.append(n)
        l2g = np.concatenate(chunks)
        meta = IterationMetadata(B, tuple(vc), tuple(ec), size, int(sum(ec)))
        return SampledSubgraph(hops=hops, local_to_global=l2g), meta


def gather_features(X: torch.Tensor, ids: torch.Tensor, out: torch.Tensor | None = None):
    """out[i] = X[ids[i]] on libgnnb200 (the mini-batch feature gather)."""
    lib = _lib.lib()
    ids = ids.to(device=X.device, dtype=torch.int64).contiguous()
    n, K = int(ids.numel()), int(X.shape[1])
    if out is None:
        out = torch.empty(n, K, dtype=torch.float32, device=X.device)
    with torch.cuda.device(X.device):
        _lib.check(lib.gnn_gather_rows(X.data_ptr(), X.stride(0), ids.data_ptr() if n else None,
                                       n, K, out.data_ptr(), out.stride(0),
                                       _lib.stream_handle(X.device)), "gather_rows")
    return out
