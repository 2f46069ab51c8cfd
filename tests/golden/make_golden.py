"""Generate the golden fixtures for the graph-substrate parity tests by
importing the UNMODIFIED reference (gsbench) from /root/reference.

Run in the build container (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --large    # + Reddit/products-shape digests (~3 min)

Outputs (committed): tests/golden/graph_small.npz, tests/golden/csr1_small.bin,
tests/golden/digests.json.
"""

from __future__ import annotations

import argparse
import hashlib
import io
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import gsbench as g  # noqa: E402
from gsbench.graph import csr_from_edges  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def small(out):
    fx = {}
    # generator families (graph.py:227-262)
    specs = {
        "pl_1000_20000_s42": (g.GraphGenSpec("power-law", 1000, 20000, exponent=2.1), 42),
        "pl_10000_200000_s7": (g.GraphGenSpec("power-law", 10_000, 200_000, exponent=2.1), 7),
        "pl_2708_10556_s42": (g.GraphGenSpec("power-law", 2708, 10556, exponent=2.1), 42),
        "pl_3000_30000_e25_s5": (g.GraphGenSpec("power-law", 3000, 30000, exponent=2.5), 5),
        "ur_500_5000_s43": (g.GraphGenSpec("uniform-random", 500, 5000), 43),
        "ur_100_p002_s5": (g.GraphGenSpec("uniform-random", 100, 0.02), 5),
        "star_5": (g.GraphGenSpec("star", 5), 0),
        "ring_4": (g.GraphGenSpec("ring", 4), 0),
        "complete_3": (g.GraphGenSpec("complete", 3), 0),
        "complete_17": (g.GraphGenSpec("complete", 17), 0),
    }
    for name, (spec, seed) in specs.items():
        gr = g.generate(spec, seed)
        fx[f"{name}/offsets"] = gr.offsets
        fx[f"{name}/targets"] = gr.targets
    # transposed CSR of a power-law graph via the reference builder
    gr = g.generate(specs["pl_1000_20000_s42"][0], 42)
    rows = np.repeat(np.arange(gr.num_vertices), np.diff(gr.offsets))
    t = csr_from_edges(gr.num_vertices, gr.targets, rows)
    fx["pl_1000_20000_s42/csc_offsets"] = t.offsets
    fx["pl_1000_20000_s42/csc_rows"] = t.targets
    # raw shuffled edge lists through csr_from_edges (stability within rows)
    rng = np.random.default_rng(1234)
    for name, (n, m) in {"edges_64_4000": (64, 4000), "edges_70000_300000": (70_000, 300_000)}.items():
        src = rng.integers(0, n, size=m)
        dst = rng.integers(0, n, size=m)
        gr = csr_from_edges(n, src, dst)
        fx[f"{name}/src"] = src.astype(np.int64)
        fx[f"{name}/dst"] = dst.astype(np.int64)
        fx[f"{name}/offsets"] = gr.offsets
        fx[f"{name}/targets"] = gr.targets
    # build_subgraph_csr on a real sampled block (sampler.py:242-296)
    base = g.generate(specs["pl_10000_200000_s7"][0], 7)
    cfg = g.SampleConfig(batch_size=8, fanouts=(5, 5))
    sg, _ = g.sample_minibatch(base, cfg, np.arange(8), 3)
    for h, block in enumerate(sg.hops):
        off, tgt = g.build_subgraph_csr(block.edge_src, block.edge_dst, sg.num_local_vertices)
        fx[f"subgraph_hop{h}/edge_src"] = np.asarray(block.edge_src, dtype=np.int64)
        fx[f"subgraph_hop{h}/edge_dst"] = np.asarray(block.edge_dst, dtype=np.int64)
        fx[f"subgraph_hop{h}/num_local"] = np.array([sg.num_local_vertices], dtype=np.int64)
        fx[f"subgraph_hop{h}/offsets"] = off
        fx[f"subgraph_hop{h}/targets"] = tgt
    # edge-list parsing (graph.py:134-196)
    text = "# c\n0 5\n1 2\n0 3\n0 5\n7 1\nn=9\n"
    gr = g.load_edge_list(io.StringIO(text))
    fx["edgelist_a/offsets"] = gr.offsets
    fx["edgelist_a/targets"] = gr.targets
    gr = g.load_edge_list(io.StringIO("5 1000\n1000 7\n7 5\n"), symmetrize=True, compact_ids=True)
    fx["edgelist_b/offsets"] = gr.offsets
    fx["edgelist_b/targets"] = gr.targets
    np.savez_compressed(os.path.join(out, "graph_small.npz"), **fx)
    # CSR1 bytes written by the reference (graph.py:204-209)
    g.save_csr(g.generate(specs["pl_1000_20000_s42"][0], 42), os.path.join(out, "csr1_small.bin"))


def large(out):
    res = {}
    shapes = {
        "reddit_s42": (232_965, 114_615_892, 2.1, 42),
        "products_s42": (2_449_029, 123_718_280, 2.1, 42),
    }
    for name, (n, m, ex, seed) in shapes.items():
        t0 = time.time()
        gr = g.generate(g.GraphGenSpec("power-law", n, m, exponent=ex), seed)
        t1 = time.time()
        rows = np.repeat(np.arange(gr.num_vertices, dtype=np.int64), np.diff(gr.offsets))
        tt = csr_from_edges(gr.num_vertices, gr.targets, rows)
        t2 = time.time()
        deg = gr.degrees
        res[name] = {
            "num_vertices": n, "num_edges": m, "exponent": ex, "seed": seed,
            "offsets_sha256": digest(gr.offsets), "targets_sha256": digest(gr.targets),
            "csc_offsets_sha256": digest(tt.offsets), "csc_rows_sha256": digest(tt.targets),
            "degree_max": int(deg.max()), "degree_sum": int(deg.sum()),
            "generate_s": round(t1 - t0, 2), "transpose_s": round(t2 - t1, 2),
        }
        print(name, res[name], flush=True)
        del gr, tt, rows
    with open(os.path.join(out, "digests.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    a = ap.parse_args()
    small(HERE)
    if a.large:
        large(HERE)
