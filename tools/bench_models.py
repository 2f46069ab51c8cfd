"""Model-level measurements beside bench.py's headline (GCN epoch):

  gin      2-layer GIN epoch, Reddit shape (K=602 -> 64 -> 41)        [BASELINE configs[2]]
  gat      2-layer GAT epoch, products shape (K=100 -> 4x16 -> 4x47)   [BASELINE configs[3]]
  sweep    SpMMv / SpMMve K sweep 16..256, Reddit shape               [BASELINE configs[1]]
  sampling device sample_minibatch / DeviceSampler vs the reference sampler (host)
  minibatch sampled mini-batch GCN training step, Reddit shape (SampledGCNTrainer)
  build    device CSR / CSC(+eid) builders at the Reddit shape vs the reference port
  variants GCN epoch + SpMMv K=32 on the canonical layout, the uniform-random control,
           seeds 43 / 44
  papers100m 2-layer GCN epoch, ogbn-papers100M shape (V=111M, E=1.6B, K=128 -> 16 -> 172),
           row-partitioned over the N ranks of the run, per-rank block build [configs[4]]

Prints one JSON object per item: device-timed ms (CUDA-graph replay), per-
kernel ms inside eager epochs, peak memory.  Usage:
    python tools/bench_models.py gin gat sweep
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_29346_b200 as gb
from paper_2605_29346_b200 import _lib
from paper_2605_29346_b200.kernels import SpmmCall

REDDIT = dict(V=232_965, E=114_615_892)
PAPERS100M = dict(V=111_059_956, E=1_615_685_872, F=128, H=16, C=172, seed=42)
# row-proportional cost of the papers100M epoch in edge-equivalents (X.W1 and
# X^T.dH1 stream 512 B per row, the 172-class head ~0.3 ns per row, vs ~15 ps
# per edge for each of the four SpMMs)
PAPERS100M_ROW_COST = 40.0
PRODUCTS = dict(V=2_449_029, E=123_718_280)


def peak_hbm():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(__file__), "..",
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def time_graph(tr, steps=10, warmup=3):
    tr.capture()
    for _ in range(warmup):
        tr.run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        tr.run()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def kernel_ms(tr, reps=3):
    per = [tr.timed_step() for _ in range(reps)]
    return {k: round(statistics.median(p[k] for p in per), 4) for k in per[0]}


def run_gin():
    from paper_2605_29346_b200.models import GINTrainer

    g = gb.generate(gb.GraphGenSpec("power-law", REDDIT["V"], REDDIT["E"], exponent=2.1), 42)
    V = g.num_vertices
    torch.cuda.reset_peak_memory_stats()
    tr = GINTrainer(g, 602, 64, 41, seed=42, coalesced=True)
    g.drop_csc()
    X = torch.rand(V, 602) * 2e-3 - 1e-3
    y = torch.randint(0, 41, (V,))
    tr.set_inputs(X, y)
    c0 = _lib.lib().gnn_launch_counter()
    tr.step()
    torch.cuda.synchronize()
    launches = _lib.lib().gnn_launch_counter() - c0
    ms = time_graph(tr)
    return {"item": "gin_epoch_ms", "workload": "2-layer GIN (hidden 64) full-graph epoch, Reddit shape",
            "ms": round(ms, 4), "launches_per_step": int(launches), "kernels_ms": kernel_ms(tr),
            "peak_mb": round(torch.cuda.max_memory_allocated() / 2**20, 1),
            "loss": float(tr.loss.item())}


def run_gat():
    from paper_2605_29346_b200.models import GATTrainer

    t0 = time.perf_counter()
    g = gb.generate(gb.GraphGenSpec("power-law", PRODUCTS["V"], PRODUCTS["E"], exponent=2.1), 42)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    V = g.num_vertices
    torch.cuda.reset_peak_memory_stats()
    tr = GATTrainer(g, 100, 16, 47, heads=4, seed=42)
    X = torch.rand(V, 100) * 2 - 1
    y = torch.randint(0, 47, (V,))
    tr.set_inputs(X, y)
    c0 = _lib.lib().gnn_launch_counter()
    tr.step()
    torch.cuda.synchronize()
    launches = _lib.lib().gnn_launch_counter() - c0
    ms = time_graph(tr)
    km = kernel_ms(tr)
    E, H = g.num_edges, 4
    # SURVEY §8d official bytes: fused score+softmax 8(V+1)+4E+8VH+4EH; SDDMM F=16 per head
    b_soft = 8 * (V + 1) + 4 * E + 8 * V * H + 4 * E * H
    if tr.rc:
        # alpha-recompute CSC pass (gnn_gat_bwd_rc): offsets, rows, ds (CSC order) + dY,
        # row stats {er, m, inv, S}, Wh, dWh, del — every operand once
        b_bwd1 = 8 * (V + 1) + 4 * E + 4 * E * H + 12 * V * H * 16 + 16 * V * H + 4 * V * H
    else:
        # fused SpMMve^T + SDDMM over the CSC: offsets, rows, eid, alpha, dalpha + dY, Wh, dWh
        b_bwd1 = 8 * (V + 1) + 8 * E + 8 * E * H + 12 * V * H * 16
    hbm = peak_hbm()
    return {"item": "gat_epoch_ms",
            "workload": "2-layer GAT (4 heads x 16 hidden, 4 x 47 out averaged) full-graph epoch, products shape",
            "ms": round(ms, 4), "launches_per_step": int(launches), "kernels_ms": km,
            "softmax1_gbs": round(b_soft / (km["softmax1"] * 1e-3) / 1e9, 1),
            "bwd1_fused_gbs": round(b_bwd1 / (km["bagg1+sddmm1"] * 1e-3) / 1e9, 1),
            "bwd1_bytes": b_bwd1, "backward_form": "alpha recomputed (rc)" if tr.rc else "alpha read",
            "hbm_peak": hbm,
            "peak_mb": round(torch.cuda.max_memory_allocated() / 2**20, 1), "generate_s": round(t_gen, 2),
            "loss": float(tr.loss.item())}


def run_sweep():
    V, E = REDDIT["V"], REDDIT["E"]
    g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
    g.csc()
    flush = torch.empty(64 * 2**20, device="cuda")
    hbm = peak_hbm()
    out = []
    ev = torch.rand(E, device="cuda")
    for K in (16, 32, 64, 128, 256):
        X = torch.rand(V, K, device="cuda")
        Y = torch.empty_like(X)
        row = {"item": "spmm_sweep", "K": K}
        for name, call in (
                ("spmmv_norm", SpmmCall(g.csr(), X, Y, flags=_lib.EPI_NORM)),
                ("spmmv_norm_coalesced", SpmmCall(g.csr_coalesced(), X, Y, flags=_lib.EPI_NORM)),
                ("spmmve", SpmmCall(g.csr(), X, Y, vals=ev)),
                ("spmmvT", SpmmCall(g.csc(), X, Y))):
            ts = []
            for _ in range(12):
                flush.add_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                call()
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts[2:])
            byt = 8 * (V + 1) + 4 * E + 8 * V * K + (4 * E if name == "spmmve" else 0)
            row[name] = {"ms": round(ms, 4), "gbs": round(byt / (ms * 1e-3) / 1e9, 1),
                         "frac": round(byt / (ms * 1e-3) / 1e9 / hbm, 4),
                         "gather_tbs": round(4 * E * K / (ms * 1e-3) / 1e12, 2)}
        out.append(row)
    return out


def run_sampling():
    """Reference default sampling config (configs/default.json: power-law
    n=1e5, m=2e7, exponent 2.1; B=256, fanouts [10,10]) — device
    sample_minibatch vs the reference algorithm on the host (oracle port)."""
    from oracle import sampler as osm
    from paper_2605_29346_b200.sampling import SampleConfig, sample_minibatch

    g = gb.generate(gb.GraphGenSpec("power-law", 100_000, 20_000_000, exponent=2.1), 42)
    off, tgt = g.offsets, g.targets
    out = {}
    for B, fan, reps in ((256, (10, 10), 20), (8192, (25, 10), 5)):
        cfg = SampleConfig(B, fan)
        rng = np.random.default_rng(0)
        batches = [rng.choice(100_000, B, replace=False) for _ in range(reps)]
        for s in batches[:2]:
            sample_minibatch(g, cfg, s, 1, on_device=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(batches):
            sample_minibatch(g, cfg, s, i, on_device=True)
        torch.cuda.synchronize()
        dev_ms = (time.perf_counter() - t0) * 1e3 / reps
        # replayed: device-resident counts, one CUDA graph per mini-batch
        from paper_2605_29346_b200.sampling import DeviceSampler

        ds = DeviceSampler(g, cfg)
        ds.capture()
        for i, s in enumerate(batches[:2]):
            ds.run(s, i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(batches):
            ds.run(s, i)
        torch.cuda.synchronize()
        replay_ms = (time.perf_counter() - t0) * 1e3 / reps
        t0 = time.perf_counter()
        for i, s in enumerate(batches):
            osm.sample_minibatch(off, tgt, s, cfg.fanouts, i)
        cpu_ms = (time.perf_counter() - t0) * 1e3 / reps
        out[f"B{B}_F{'x'.join(map(str, fan))}"] = {"device_ms": round(dev_ms, 3),
                                                  "device_replay_ms": round(replay_ms, 3),
                                                  "cpu_reference_port_ms": round(cpu_ms, 3)}
    return {"item": "sample_minibatch_ms",
            "workload": "reference default graph (configs/default.json: power-law 1e5/2e7, "
                        "exponent 2.1)", **out,
            "note": "wall clock per mini-batch: device_ms = host-synchronous API (one count read "
                    "per hop); device_replay_ms = DeviceSampler, one CUDA-graph replay incl. the "
                    "seed / RNG-state H2D copies, no host sync"}


def run_minibatch():
    """Sampled mini-batch GCN training (SampledGCNTrainer) on the Reddit shape:
    B=1024 seeds, fanouts (25, 10), K=602 -> 16 -> 41 — sampling, subgraph
    CSR/CSC build, feature gather, the epoch kernels on the subgraph and Adam,
    wall clock per step."""
    from paper_2605_29346_b200.models import SampledGCNTrainer
    from paper_2605_29346_b200.sampling import SampleConfig

    V, E = REDDIT["V"], REDDIT["E"]
    g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
    X = torch.rand(V, 602, device="cuda") * 2 - 1
    y = torch.randint(0, 41, (V,), device="cuda")
    B, fan = 1024, (25, 10)
    tr = SampledGCNTrainer(g, X, y, 602, 16, 41, SampleConfig(B, fan), seed=42)
    rng = np.random.default_rng(0)
    batches = [rng.choice(V, B, replace=False) for _ in range(12)]
    for i, s in enumerate(batches[:2]):
        tr.step(s, rng=i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sizes = []
    for i, s in enumerate(batches[2:]):
        tr.step(s, rng=100 + i)
        sizes.append((tr.last[0].num_vertices, tr.last[0].num_edges))
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / (len(batches) - 2)
    # replayed form: one CUDA graph per mini-batch (capture + run), no host sync
    tr2 = SampledGCNTrainer(g, X, y, 602, 16, 41, SampleConfig(B, fan), seed=42)
    tr2.capture()
    many = [rng.choice(V, B, replace=False) for _ in range(50)]
    for i, s in enumerate(many[:5]):
        tr2.run(s, rng=i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for i, s in enumerate(many[5:]):
        tr2.run(s, rng=200 + i)
    ev1.record()
    torch.cuda.synchronize()
    ms_replay = (time.perf_counter() - t0) * 1e3 / (len(many) - 5)
    ms_replay_dev = ev0.elapsed_time(ev1) / (len(many) - 5)
    return {"item": "minibatch_gcn_step_ms", "ms": round(ms_replay, 3),
            "ms_device": round(ms_replay_dev, 3), "ms_eager": round(ms, 3),
            "workload": f"Reddit shape, B={B}, fanouts {fan}, GCN 602->16->41, Adam",
            "mean_subgraph_vertices": int(np.mean([v for v, _ in sizes])),
            "mean_subgraph_edges": int(np.mean([e for _, e in sizes])),
            "envelope": {"edges": tr2._caps[1], "vertices": tr2._caps[2]},
            "loss": float(tr2.loss.item()),
            "note": "ms: wall clock per step of the replayed form (capture + run: one CUDA graph "
                    "per mini-batch incl. the seed / RNG-state staging, device sampling, subgraph "
                    "CSR/CSC build, device-count SpMM plans, feature gather, epoch kernels, Adam; "
                    "no host sync); ms_device: CUDA events over the same loop; ms_eager: the "
                    "per-batch rebuilt calls (SampledGCNTrainer.step)"}


def run_build(reps=5):
    """Device CSR / CSC builders in isolation on the Reddit shape (BASELINE
    configs[1] graph): csr_from_edges from the device int64 (src, dst) stream
    (reference graph.py:106-114) and the transposed build with the edge-ID
    array, CUDA-event medians; roofline on SURVEY §8d's
    algorithmic bytes (CSR 16E + 4E + 8(V+1); CSC+eid 8(V+1) + 4E + 8(V+1) +
    4E + 4E).  Beside them the reference algorithm (oracle numpy port, one
    host thread like the reference) on a bounded sample: the first 1/8 of the
    same edge stream, whole V."""
    from oracle import graph as og

    V, E = REDDIT["V"], REDDIT["E"]
    hbm = peak_hbm()
    src, dst = gb.graph.powerlaw_edges_device(V, E, 2.1, 42)
    torch.cuda.synchronize()

    def timed(fn):
        ts = []
        for _ in range(reps + 1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
            del r
        return statistics.median(ts[1:])

    t_csr = timed(lambda: gb.csr_from_edges(V, src, dst, device="cuda"))
    g = gb.csr_from_edges(V, src, dst, device="cuda")

    def csc():
        g.drop_csc()
        return g.csc(with_eid=True)

    t_csc = timed(csc)
    b_csr = 16 * E + 4 * E + 8 * (V + 1)
    b_csc = 8 * (V + 1) + 4 * E + 8 * (V + 1) + 4 * E + 4 * E
    ns = E // 8
    hs, hd = src[:ns].cpu().numpy(), dst[:ns].cpu().numpy()
    del src, dst
    t0 = time.perf_counter()
    off, tgt = og.csr_from_edges(V, hs, hd)
    c_csr = time.perf_counter() - t0
    t0 = time.perf_counter()
    og.transpose(V, V, off, tgt)
    c_csc = time.perf_counter() - t0
    return {"item": "csr_csc_build", "V": V, "E": E,
            "csr_from_edges": {"ms": round(t_csr, 3), "bytes": b_csr,
                               "gbs": round(b_csr / (t_csr * 1e-3) / 1e9, 1),
                               "frac": round(b_csr / (t_csr * 1e-3) / 1e9 / hbm, 4)},
            "csc_with_eid": {"ms": round(t_csc, 3), "bytes": b_csc,
                             "gbs": round(b_csc / (t_csc * 1e-3) / 1e9, 1),
                             "frac": round(b_csc / (t_csc * 1e-3) / 1e9 / hbm, 4)},
            "cpu_reference_port": {"sample": f"first {ns} edges of the stream (1/8), V={V}",
                                   "csr_from_edges_ms": round(c_csr * 1e3, 1),
                                   "transpose_ms": round(c_csc * 1e3, 1), "threads": 1}}


def run_variants():
    """Simple-graph and seed controls of the headline: the GCN
    epoch (device-timed CUDA-graph replay, 602 -> 16 -> 41, Adam) and SpMMv
    K=32 (degree-norm fused, L2 flushed between reps, median of 15) on
      * the canonical layout of the seed-42 power-law graph (every stored edge
        gathered: what a simple graph without duplicate pairs gets);
      * the uniform-random control (reference pkg/tests/conftest.py:40-42),
        generated with the reference's own stream (host draws, device CSR);
      * seeds 43 and 44 (reference configs/default.json:3-6).
    The headline itself runs on the coalesced layout of seed 42."""
    from paper_2605_29346_b200.models import GCNTrainer

    V, E = REDDIT["V"], REDDIT["E"]
    hbm = peak_hbm()
    flush = torch.empty(64 * 2**20, device="cuda")
    out = []
    for name, kind, seed, coalesced in (("powerlaw_s42_canonical", "power-law", 42, False),
                                        ("uniform_s42", "uniform-random", 42, True),
                                        ("powerlaw_s43", "power-law", 43, True),
                                        ("powerlaw_s44", "power-law", 44, True)):
        t0 = time.perf_counter()
        g = gb.generate(gb.GraphGenSpec(kind, V, E, exponent=2.1), seed, device="cuda")
        torch.cuda.synchronize()
        t_gen = time.perf_counter() - t0
        nnz = g.csr_coalesced().nnz if coalesced else E
        X = torch.rand(V, 602, device="cuda") * 2 - 1
        y = torch.randint(0, 41, (V,), device="cuda")
        tr = GCNTrainer(g, 602, 16, 41, seed=seed, coalesced=coalesced)
        tr.set_inputs(X, y)
        tr.step()
        ms = time_graph(tr)
        km = kernel_ms(tr)
        del tr
        X32 = torch.rand(V, 32, device="cuda") * 2 - 1
        Y32 = torch.empty_like(X32)
        call = SpmmCall(g.operand("csr_coalesced" if coalesced else "csr"), X32, Y32,
                        flags=_lib.EPI_NORM)
        ts = []
        for _ in range(15):
            flush.add_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        t32 = statistics.median(ts[3:])
        b32 = 8 * (V + 1) + 4 * E + 8 * V * 32
        out.append({"item": "gcn_epoch_variant", "graph": name, "layout":
                    "coalesced" if coalesced else "canonical", "unique_pairs": int(nnz),
                    "duplicate_frac": round(1 - g.csr_coalesced().nnz / E, 4),
                    "epoch_ms": round(ms, 4), "kernels_ms": km,
                    "spmmv_k32": {"ms": round(t32, 4), "gbs": round(b32 / (t32 * 1e-3) / 1e9, 1),
                                  "frac": round(b32 / (t32 * 1e-3) / 1e9 / hbm, 4),
                                  "gather_tbs": round(4 * nnz * 32 / (t32 * 1e-3) / 1e12, 2)},
                    "generate_s": round(t_gen, 2)})
        del call, g, X, y, X32, Y32
        torch.cuda.empty_cache()
    return out


def run_papers100m(rank=0, world=1, steps=10, warmup=3, scale=None):
    """2-layer GCN epoch on the ogbn-papers100M-shaped power-law graph
    (BASELINE configs[4]), row-partitioned over the run's ranks.  Every rank
    builds only its own block (graph.powerlaw_row_block: the bit-exact edge
    stream regenerated and filtered, no whole graph anywhere), fills its rows
    of the synthetic [V, 128] features / labels on device (hash-based,
    partition independent), and trains with DistGCNTrainer (N=1: one block,
    no exchange; N>1: NCCL all-gathers of the [V, 16] blocks overlapped with
    the own-slot aggregation + one gradient all-reduce).  Output layer: the
    fused 172-class head (logits never stored).  ``scale`` (or
    GNN_C5_SCALE) shrinks V and E for smoke runs."""
    from paper_2605_29346_b200.dist import (DistGCNTrainer, NullExchange, RowPartition,
                                            TorchDistExchange, expected_bounds)

    scale = float(os.environ.get("GNN_C5_SCALE", "1")) if scale is None else scale
    P = PAPERS100M
    V, E = int(P["V"] * scale), int(P["E"] * scale)
    F, Hd, C = P["F"], P["H"], P["C"]
    dev = torch.device("cuda", torch.cuda.current_device())
    spec = gb.GraphGenSpec("power-law", V, E, exponent=2.1)
    bounds = expected_bounds(spec, world, PAPERS100M_ROW_COST)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    t0 = time.perf_counter()
    blk = gb.graph.powerlaw_row_block(spec, P["seed"], lo, hi, pack=False)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    build_peak = torch.cuda.max_memory_allocated(dev)
    nnz_csr, nnz_csc = blk.csr_coalesced().nnz, blk.csc_coalesced().nnz
    deg_edges = int(blk.deg_offsets[-1].item())
    part = RowPartition.from_block(blk, world, rank, bounds)
    del blk
    torch.cuda.synchronize()
    t_part = time.perf_counter() - t0 - t_build
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats(dev)
    overlap = world > 1
    tr = DistGCNTrainer(part, F, Hd, C, seed=P["seed"], overlap=overlap)
    if overlap:
        part.A = part.AT = None
    else:  # every aggregation runs on the degree-sorted forms: keep only those
        part.A.release_row_order()
        part.AT.release_row_order()
    torch.cuda.empty_cache()
    gb.graph.fill_uniform(tr.X, lo, P["seed"])
    gb.graph.fill_labels(tr.labels, lo, C, P["seed"])
    ex = NullExchange() if world == 1 else TorchDistExchange()
    lib = _lib.lib()
    c0 = lib.gnn_launch_counter()
    tr.step(ex)
    torch.cuda.synchronize()
    launches = lib.gnn_launch_counter() - c0
    for _ in range(warmup):
        tr.step(ex)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(steps):
        tr.step(ex)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    peak = torch.cuda.max_memory_allocated(dev)
    per = [tr.timed_step(ex) for _ in range(3)]
    kern = {k: round(statistics.median(p[k] for p in per), 3) for k in per[0]}
    t = torch.tensor([ms, peak / 2**20, build_peak / 2**20, t_build], device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    # analytic per-rank footprint: block CSR+CSC (coalesced, packed words + int64
    # offsets), X rows, 4 exchanged [V,16] buffers (+ 3 local [rows,16])
    rows = hi - lo
    analytic = (8 * 2 * (rows + 1) + 4 * (nnz_csr + nnz_csc) + 4 * rows * F
                + 4 * Hd * (4 * world * part.stride + 3 * rows))
    return {"item": "gcn_papers100m_epoch_ms",
            "workload": "2-layer GCN full-graph epoch, ogbn-papers100M-shaped power-law graph "
                        f"(V={V}, E={E}, K={F} -> {Hd} -> {C}), row-partitioned over {world} "
                        "rank(s), per-rank block build",
            "scale": scale, "n_gpus": world, "ms": round(float(t[0]), 3),
            "steps": steps, "warmup": warmup, "timing": "CUDA events, max over ranks",
            "loss": float(tr.loss.item()), "launches_per_step": int(launches),
            "rank0_kernels_ms": kern,
            "rank0_rows": rows, "rank0_edges": deg_edges, "rank0_unique_pairs_csr": nnz_csr,
            "rank0_unique_pairs_csc": nnz_csc,
            "peak_mb_train": round(float(t[1]), 1), "peak_mb_build": round(float(t[2]), 1),
            "rank0_analytic_mb": round(analytic / 2**20, 1),
            "build_s": round(float(t[3]), 2), "partition_s": round(t_part, 2),
            "inputs": "X / labels hashed on device (gnn_fill_uniform / gnn_fill_labels)",
            "exchange": "none (one rank)" if world == 1 else "NCCL all-gather, own-slot overlap"}


if __name__ == "__main__":
    for item in sys.argv[1:] or ["gin", "gat", "sweep"]:
        r = {"gin": run_gin, "gat": run_gat, "sweep": run_sweep, "sampling": run_sampling,
             "minibatch": run_minibatch, "papers100m": run_papers100m,
             "variants": run_variants, "build": run_build}[item]()
        for x in (r if isinstance(r, list) else [r]):
            print(json.dumps(x), flush=True)
        torch.cuda.empty_cache()
