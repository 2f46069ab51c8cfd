"""numpy restatement of the reference graph substrate (test oracle only).

Each function names the reference lines it restates.  The integer results
are the parity target for the device builders: bit-exact.
"""

from __future__ import annotations

import numpy as np

OFFSET_DTYPE = np.int64
TARGET_DTYPE = np.int32


def make_csr(num_vertices, offsets, targets):
    """graph.py:91-103 — returns (offsets int64, targets int32) after the checks."""
    offsets = np.ascontiguousarray(offsets, dtype=OFFSET_DTYPE)
    targets = np.ascontiguousarray(targets, dtype=TARGET_DTYPE)
    if offsets.shape != (num_vertices + 1,):
        raise ValueError("offsets shape")
    if offsets[0] != 0 or offsets[-1] != targets.size:
        raise ValueError("offsets ends")
    if np.any(offsets[1:] < offsets[:-1]):
        raise ValueError("offsets decreasing")
    if targets.size and (targets.min() < 0 or targets.max() >= num_vertices):
        raise IndexError("target out of range")  # RangeError in the reference
    return offsets, targets


def csr_from_edges(num_vertices, src, dst):
    """graph.py:106-114: bincount -> cumsum -> stable argsort -> gather."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    counts = np.bincount(src, minlength=num_vertices)
    if counts.size != num_vertices:
        raise ValueError("source id out of range")
    offsets = np.empty(num_vertices + 1, dtype=OFFSET_DTYPE)
    offsets[0] = 0
    np.cumsum(counts, out=offsets[1:])
    perm = np.argsort(src, kind="stable")
    return make_csr(num_vertices, offsets, dst[perm].astype(TARGET_DTYPE))


def build_subgraph_csr(edge_src, edge_dst, num_local_src):
    """sampler.py:242-256 (IndexError on a source outside [0, n))."""
    edge_src = np.asarray(edge_src, dtype=np.int64)
    edge_dst = np.asarray(edge_dst, dtype=np.int64)
    if edge_src.size and (edge_src.min() < 0 or edge_src.max() >= num_local_src):
        raise IndexError("edge source local id out of range")
    counts = np.bincount(edge_src, minlength=num_local_src)
    offsets = np.zeros(num_local_src + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    perm = np.argsort(edge_src, kind="stable")
    return offsets, edge_dst[perm].astype(np.int32)


def row_ids(offsets):
    """Row of every CSR entry (expanded offsets)."""
    return np.repeat(np.arange(offsets.size - 1, dtype=np.int64), np.diff(offsets))


def transpose(num_rows, num_cols, offsets, targets):
    """Transposed CSR + edge ids: csr_from_edges(num_cols, targets, rows)
    (SURVEY.md §8a a5), eid = argsort(targets, stable)."""
    rows = row_ids(offsets)
    eid = np.argsort(targets, kind="stable")
    t_off = np.zeros(num_cols + 1, dtype=np.int64)
    np.cumsum(np.bincount(targets, minlength=num_cols), out=t_off[1:])
    return t_off, rows[eid].astype(np.int32), eid.astype(np.int32)


def coalesce(num_rows, offsets, targets):
    """Unique (row, col) pairs sorted by (row, col) with multiplicities."""
    rows = row_ids(offsets)
    key = rows * (int(targets.max()) + 1 if targets.size else 1) + targets
    uniq, counts = np.unique(key, return_counts=True)
    ncol = int(targets.max()) + 1 if targets.size else 1
    u_rows = uniq // ncol
    u_cols = (uniq % ncol).astype(np.int32)
    off = np.zeros(num_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(u_rows, minlength=num_rows), out=off[1:])
    return off, u_cols, counts.astype(np.float64)


def powerlaw_cdf(n, exponent):
    """graph.py:256-259."""
    weights = (np.arange(n, dtype=np.float64) + 1.0) ** (-1.0 / (exponent - 1.0))
    cdf = np.cumsum(weights / weights.sum())
    cdf[-1] = 1.0
    return cdf


def generate_powerlaw(n, m, exponent, seed):
    """graph.py:230, 254-262: PCG64 via default_rng(SeedSequence(seed))."""
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    cdf = powerlaw_cdf(n, exponent)
    src = np.searchsorted(cdf, rng.random(m), side="right").astype(np.int64)
    dst = np.searchsorted(cdf, rng.random(m), side="right").astype(np.int64)
    return csr_from_edges(n, src, dst)


def powerlaw_edges(n, m, exponent, seed):
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    cdf = powerlaw_cdf(n, exponent)
    src = np.searchsorted(cdf, rng.random(m), side="right").astype(np.int64)
    dst = np.searchsorted(cdf, rng.random(m), side="right").astype(np.int64)
    return src, dst


def generate_uniform(n, m, seed):
    """graph.py:249-252."""
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    src = rng.integers(0, n, size=m, dtype=np.int64)
    dst = rng.integers(0, n, size=m, dtype=np.int64)
    return csr_from_edges(n, src, dst)
