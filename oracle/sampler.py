"""numpy restatement of the reference sampling pipeline (test oracle only):
gsbench/sampler.py — hop_generator 99-107, sample_hop 118-144,
SubgraphBuilder 146-188, dedup_relabel 191-239, sample_minibatch 259-296.
Pinned against tests/golden/sampling.json (produced by the unmodified
reference, tests/golden/make_golden_sampling.py)."""

from __future__ import annotations

import numpy as np


def hop_seed_sequence(base: np.random.SeedSequence, hop: int) -> np.random.SeedSequence:
    """sampler.py:99-107: the hop's stream appends the 1-based hop index."""
    return np.random.SeedSequence(base.entropy, spawn_key=tuple(base.spawn_key) + (hop,))


def sample_hop(offsets, targets, frontier, fanout, rng):
    """sampler.py:118-144: fanout draws with replacement per frontier vertex
    of nonzero degree; pick = floor(u * deg) with u = rng.random()."""
    frontier = np.asarray(frontier, dtype=np.int64)
    empty = (np.empty(0, np.int64), np.empty(0, np.int64))
    if fanout == 0 or frontier.size == 0:
        return empty
    deg = np.diff(offsets)[frontier]
    active = frontier[deg > 0]
    if active.size == 0:
        return empty
    src = np.repeat(active, fanout)
    base = np.repeat(offsets[active], fanout)
    span = np.repeat(deg[deg > 0], fanout)
    pick = (rng.random(src.size) * span).astype(np.int64)
    return src, targets[base + pick].astype(np.int64)


class SubgraphBuilder:
    """sampler.py:146-188 + dedup_relabel 191-239 (first-occurrence local ids)."""

    def __init__(self, num_vertices, seeds):
        seeds = np.asarray(seeds, dtype=np.int64)
        self.table = np.full(num_vertices, -1, dtype=np.int32)
        self.table[seeds] = np.arange(seeds.size, dtype=np.int32)
        self.chunks = [seeds.copy()]
        self.size = int(seeds.size)
        self.hops = []

    def add_hop(self, hop, frontier, src_g, dst_g):
        t = self.table
        src_l = t[src_g]
        if src_l.size and src_l.min() < 0:
            raise ValueError("hop source vertex not present in subgraph")
        dst_l = t[dst_g]
        fresh = dst_l < 0
        if fresh.any():
            uniq, first = np.unique(dst_g[fresh], return_index=True)
            new = uniq[np.argsort(first, kind="stable")]
            start = self.size
            t[new] = np.arange(start, start + new.size, dtype=np.int32)
            self.chunks.append(new)
            self.size = start + int(new.size)
            dst_l = t[dst_g]
            new_l = np.arange(start, self.size, dtype=np.int32)
        else:
            new_l = np.empty(0, np.int32)
        block = {"hop": hop, "frontier_local": t[np.asarray(frontier, np.int64)].astype(np.int32),
                 "new_unique_local": new_l, "edge_src": src_l.astype(np.int32),
                 "edge_dst": dst_l.astype(np.int32)}
        self.hops.append(block)
        return block


def sample_minibatch(offsets, targets, seeds, fanouts, sample_seed):
    """sampler.py:259-296; returns (local_to_global, hop blocks, vertex counts, edge counts)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    base = np.random.SeedSequence(sample_seed)
    b = SubgraphBuilder(offsets.size - 1, seeds)
    frontier = np.asarray(seeds, dtype=np.int64)
    vc, ec = [], []
    for hop, f in enumerate(fanouts, 1):
        gen = np.random.default_rng(hop_seed_sequence(base, hop))
        src, dst = sample_hop(offsets, targets, frontier, f, gen)
        block = b.add_hop(hop, frontier, src, dst)
        vc.append(b.size)
        ec.append(int(src.size))
        frontier = b.chunks[-1] if block["new_unique_local"].size else np.empty(0, np.int64)
    return np.concatenate(b.chunks), b.hops, vc, ec
