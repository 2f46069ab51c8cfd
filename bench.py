"""Benchmark of the sparse GNN hot path on B200 (BASELINE.json metric:
"GCN epoch ms & SpMMv HBM GB/s (Reddit-shape, K=32) vs roofline; peak MB").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  A "step" is one full-graph GCN training epoch
(forward, mean cross-entropy, backward, Adam) on the Reddit-shaped synthetic
power-law graph (|V|=232,965, |E|=114,615,892, K=602 -> 16 -> 41), generated
on device bit-exactly as gsbench.generate(power-law, exponent 2.1, seed 42)
would.  value = device-timed ms per epoch (CUDA events, max over ranks);
e2e = the same epoch through the public trainer API with the step's inputs
(X, labels) copied from pinned host memory and the loss read back.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REDDIT = dict(V=232_965, E=114_615_892, F=602, H=16, C=41, exponent=2.1, seed=42)
L2_BYTES = 126 * 1024 * 1024


def local_device() -> int:
    """GPU of this rank: LOCAL_RANK (wrapped onto the visible devices, so a
    gloo test run can put several ranks on one GPU)."""
    import torch

    return int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count())


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "model": model}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def spmm_bytes(V, E, K):
    """SURVEY.md §8d official algorithmic bytes of one SpMMv: 8(V+1)+4E+4VK+4VK."""
    return 8 * (V + 1) + 4 * E + 8 * V * K


def l2_read_gbs(lib, dev, mb=64, reps=100):
    """Measured L2 -> SM read bandwidth (GB/s): an L2-resident buffer streamed
    with 128-bit loads by every SM (gnn_read_probe)."""
    import torch

    n = mb * 2**20 // 4
    buf = torch.rand(n, device=dev)
    out = torch.zeros(1, device=dev)
    st = torch.cuda.current_stream()
    for _ in range(3):
        lib.gnn_read_probe(buf.data_ptr(), n, reps, out.data_ptr(), st.cuda_stream)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        lib.gnn_read_probe(buf.data_ptr(), n, reps, out.data_ptr(), st.cuda_stream)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return n * 4 * reps / (min(ts) * 1e-3) / 1e9


def flush_l2(buf):
    buf.add_(1.0)


def time_call(fn, reps, flush=None, stream=None):
    import torch

    st = stream or torch.cuda.current_stream()
    times = []
    for _ in range(reps):
        if flush is not None:
            flush()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        times.append(a.elapsed_time(b))
    return times


# ------------------------------------------------------------ CPU baseline
def workload_config(world):
    """config block shared by both arms (the driver compares them key by key)."""
    P = REDDIT
    return {"workload": "2-layer GCN full-graph epoch, Reddit-shape power-law graph",
            "V": P["V"], "E": P["E"], "K": P["F"], "hidden": P["H"], "classes": P["C"],
            "graph": f"power-law exponent {P['exponent']}, seed {P['seed']}",
            "optimizer": "adam", "parallelism": f"rowpart{world}" if world > 1 else "single"}


class CpuGcnEpoch:
    """The oracle's GCN epoch on the host (float64 numpy; SURVEY §8d CPU
    baseline): forward, mean cross-entropy, backward and Adam at FULL size —
    no sampling, no extrapolation.  Dense ops on the BLAS threads; the four
    SpMMs (two over the CSR with the degree-norm, two over the CSC) on every
    host core through oracle.parallel.ForkSpmmPool.  Same schedule as
    GCNTrainer (layer 2 aggregates the 16-wide Y1, then applies W2)."""

    def __init__(self, off, tgt, t_off, t_rows, X, y, W1, b1, W2, b2, lr=0.01):
        from oracle.parallel import ForkSpmmPool

        self.off = np.asarray(off, dtype=np.int64)
        V = self.off.size - 1
        d = np.diff(self.off).astype(np.float64)
        self.inv = np.divide(1.0, d, out=np.zeros_like(d), where=d > 0)[:, None]
        self.X = np.asarray(X, dtype=np.float64)  # resident float64 input
        self.y = np.asarray(y)
        self.p = [np.array(t, dtype=np.float64) for t in (W1, b1, W2, b2)]
        self.m = [np.zeros_like(t) for t in self.p]
        self.v = [np.zeros_like(t) for t in self.p]
        self.t, self.lr = 0, lr
        self.pool = ForkSpmmPool({"csr": (self.off, tgt), "csc": (t_off, t_rows)}, V,
                                 W1.shape[1])
        self.workers = self.pool.workers

    def step(self):
        from oracle import ops as oo

        W1, b1, W2, b2 = self.p
        H1 = self.X @ W1
        Y1 = np.maximum(self.pool.spmm("csr", H1, norm=True) + b1, 0.0)
        P2 = self.pool.spmm("csr", Y1, norm=True)
        Z2 = P2 @ W2 + b2
        loss, dZ2 = oo.cross_entropy(Z2, self.y)
        dW2, db2 = P2.T @ dZ2, dZ2.sum(axis=0)
        dP2 = (dZ2 @ W2.T) * self.inv
        dZ1 = self.pool.spmm("csc", dP2) * (Y1 > 0)
        db1 = dZ1.sum(axis=0)
        dH1 = self.pool.spmm("csc", dZ1 * self.inv)
        dW1 = self.X.T @ dH1
        self.t += 1
        b1c, b2c = 1 - 0.9 ** self.t, 1 - 0.999 ** self.t
        for p, g, m, v in zip(self.p, (dW1, db1, dW2, db2), self.m, self.v):
            m *= 0.9
            m += 0.1 * g
            v *= 0.999
            v += 0.001 * g * g
            p -= self.lr * (m / b1c) / (np.sqrt(v / b2c) + 1e-8)
        return float(loss)

    def close(self):
        self.pool.close()

    def describe(self):
        return (f"oracle float64 GCN epoch at full size (all {self.off[-1]} edges, no sampling): "
                f"dense ops on the BLAS threads, 4 SpMMs on {self.workers} fork()ed host "
                f"workers (oracle.parallel), mean cross-entropy, Adam")


# -------------------------------------------------------------- our arm
def run_ours(args, rank, world):
    import torch

    import paper_2605_29346_b200 as gb
    from paper_2605_29346_b200 import _lib
    from paper_2605_29346_b200.kernels import SpmmCall
    from paper_2605_29346_b200.models import GCNTrainer

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    lib = _lib.lib()
    P = REDDIT
    V, E, F, Hd, C = P["V"], P["E"], P["F"], P["H"], P["C"]

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=P["exponent"]), P["seed"],
                    device=dev)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    g.csc()
    torch.cuda.synchronize()
    t_csc = time.perf_counter() - t0
    h_off = g.offsets  # host views for the CPU baseline (before any release)
    h_tgt = g.targets
    h_toff = g.csc().offsets.cpu().numpy()
    h_trows = g.csc().cols.cpu().numpy()
    if args.layout == "coalesced":
        t0 = time.perf_counter()
        g.csr_coalesced()
        g.csc_coalesced()
        torch.cuda.synchronize()
        t_co = time.perf_counter() - t0
        g.drop_csc()
        g.release_device_targets()  # training runs on the coalesced forms only
        # every aggregation of the epoch runs on the degree-sorted forms: keep only those
        g.csr_coalesced().release_row_order()
        g.csc_coalesced().release_row_order()
    else:
        t_co = 0.0

    # synthetic inputs (SURVEY §8d seeding): X ~ U[-1,1), labels uniform
    rng = np.random.default_rng(np.random.SeedSequence(P["seed"], spawn_key=(10,)))
    X_h = torch.from_numpy(rng.random((V, F), dtype=np.float32) * 2 - 1).pin_memory()
    y_h = torch.from_numpy(np.random.default_rng(np.random.SeedSequence(P["seed"], spawn_key=(13,)))
                           .integers(0, C, V)).pin_memory()

    setup_peak = torch.cuda.max_memory_allocated(dev)
    torch.cuda.empty_cache()  # return the setup temporaries (radix-sort scratch) to the driver
    torch.cuda.reset_peak_memory_stats(dev)
    base_alloc = torch.cuda.memory_allocated(dev)
    tr = GCNTrainer(g, F, Hd, C, seed=P["seed"], coalesced=args.layout == "coalesced")
    tr.set_inputs(X_h, y_h)
    p0 = [t.double().cpu().numpy() for t in (tr.W1, tr.b1, tr.W2, tr.b2)]
    c0 = lib.gnn_launch_counter()
    tr.step()
    torch.cuda.synchronize()
    launches_per_step = lib.gnn_launch_counter() - c0
    tr.capture()
    torch.cuda.synchronize()

    # ---- device-timed epochs (inputs resident; X 561 MB and the graph exceed L2)
    for _ in range(args.warmup):
        tr.run()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    with ClockSampler(dev.index) as clk:
        st = torch.cuda.current_stream()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(args.steps):
            tr.run()
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.steps
    if world > 1:
        torch.distributed.barrier()
    peak_train = torch.cuda.max_memory_allocated(dev)
    # SURVEY §8d cross-check: the driver's view (cudaMemGetInfo) of device memory in use
    free_b, total_b = torch.cuda.mem_get_info(dev)
    dev_used = total_b - free_b
    torch_reserved = torch.cuda.memory_reserved(dev)
    loss_val = float(tr.loss.item())

    # ---- e2e: host buffers in, loss out, copies inside the timed region.  The
    # host X is laid out with the trainer's 128-byte row stride (608 floats) so
    # it copies as one contiguous block.  Inputs are double-buffered: each step
    # (one CUDA graph) trains on one device buffer while the copy stream loads
    # the next step's X / labels into the other; the first step's copy (prime)
    # is inside the timed region too.
    loss_h = torch.empty(1, dtype=torch.float32).pin_memory()
    # pinned host X at the device row stride (608): one linear DMA per step.
    # (A [V, 602] host array works too — one 2-D DMA into the padded rows — but
    # pitched H2D runs at ~16 GB/s here vs ~53 GB/s linear.)
    Xp_h = torch.zeros(V, tr.Fpad, dtype=torch.float32).pin_memory()
    Xp_h[:, :F].copy_(X_h)
    tr.capture_e2e_pipelined(Xp_h, y_h, loss_h)
    tr.prime_e2e()
    for k in range(2):
        tr.run_e2e_pipelined(k)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    tr.prime_e2e()
    for k in range(args.steps):
        tr.run_e2e_pipelined(k)
    b.record(st)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / args.steps
    e2e_loss = float(loss_h.item())

    # ---- per-kernel times inside real (eager) epochs: dominant kernel = the SpMMs
    per = [tr.timed_step() for _ in range(5)]
    kern_ms = {k: statistics.median(p[k] for p in per) for k in per[0]}
    spmm_keys = ["agg1", "agg2", "bagg2", "bagg1"]
    hbm_peak, peak_src = peaks()
    b16 = spmm_bytes(V, E, Hd)
    avg_spmm = statistics.mean(kern_ms[k] for k in spmm_keys)
    ach16 = b16 / (avg_spmm * 1e-3) / 1e9
    flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)

    # ---- SpMMv K=32 (BASELINE headline kernel), canonical CSR, NORM fused
    X32 = torch.rand(V, 32, device=dev) * 2 - 1
    Y32 = torch.empty_like(X32)
    k32 = {}
    for layout in ("csr", "csr_coalesced"):
        if layout == "csr" and args.layout == "coalesced":
            continue  # canonical device CSR released for training; measured in the canonical run
        call = SpmmCall(g.operand(layout), X32, Y32, flags=_lib.EPI_NORM)
        t32 = time_call(call, 20, flush=lambda: flush_l2(flush_buf))
        med = statistics.median(t32)
        k32[layout] = {"ms": round(med, 4),
                       "gbs": round(spmm_bytes(V, E, 32) / (med * 1e-3) / 1e9, 1)}
    t32 = k32["csr"]["ms"] if "csr" in k32 else k32["csr_coalesced"]["ms"]
    ach32 = spmm_bytes(V, E, 32) / (t32 * 1e-3) / 1e9
    # hierarchical bound: max(B_comp/BW_hbm, 4EK/BW_L2) with BW_L2 = 2x HBM (nominal)
    # hierarchical bound: max(B_comp/BW_hbm, 4*nnz*K/BW_L2), BW_L2 measured
    # here by an L2-resident 128-bit read probe (libgnnb200 gnn_read_probe)
    l2_gbs = l2_read_gbs(lib, dev)
    nnz32 = g.operand("csr_coalesced" if "csr" not in k32 else "csr").nnz
    hier32 = max(spmm_bytes(V, E, 32) / (hbm_peak * 1e9), 4 * nnz32 * 32 / (l2_gbs * 1e9)) * 1e3

    # width-16 gathers: one 64-byte feature row per stored (coalesced) entry
    gather16 = 4 * Hd * g.csr_coalesced().nnz if args.layout == "coalesced" else 4 * Hd * E
    traffic16 = None
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                         "r2_spmm16_traffic.json")
    if os.path.exists(tpath) and args.layout == "coalesced":
        with open(tpath) as f:
            traffic16 = json.load(f)["traffic_bytes_per_launch"]
    # BASELINE.md analytic footprint: canonical CSR+CSC (int64 offsets, int32 ids),
    # X, and the epoch's [V,hidden] activations/gradients
    analytic = (g.d_offsets.numel() * 8 + E * 4) * 2 + V * F * 4 + V * 6 * Hd * 4
    res = {
        "metric": "gcn_epoch_ms",
        "value": round(ms, 4),
        "unit": "ms",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": False,
        "scaling": "strong",  # the whole Reddit-shape epoch is fixed at every N
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (device power-law generator, bit-exact gsbench.generate seed 42; "
                "X~U[-1,1) f32, labels uniform)",
        "config": workload_config(world),
        "layout": args.layout,
        "l2": "inputs larger than L2 (X 561 MB, graph 0.9-1.1 GB): no flush needed; "
              "spmmv_k32 flushes L2 (252 MB write) between reps",
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms",
                "h2d_bytes_per_step": int(Xp_h.numel() * 4 + y_h.numel() * 8),
                "d2h_bytes_per_step": 4, "loss_read_back": e2e_loss,
                "how": "one CUDA graph per step trains on one device input buffer while a copy "
                       "stream loads the next step's X (row stride 608) and labels from pinned "
                       "host memory into the other; loss copied back every step; the first "
                       "step's copy is inside the timed region"},
        "gpu_launches": int(launches_per_step * args.steps),
        "roofline": {"kernel": "spmm width-16 (4 per epoch, avg, timed in-epoch)", "bound": "hbm",
                     "achieved": round(ach16, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(ach16 / hbm_peak, 4), "traffic": traffic16,
                     "traffic_source": "profiles/r2_spmm16_traffic.json (ncu --set full)",
                     "bytes_per_launch": b16, "peak_source": peak_src,
                     # the binding unit is the L2->SM gather return, not HBM
                     "gather_bytes_per_launch": gather16,
                     "gather_tbs": round(gather16 / (avg_spmm * 1e-3) / 1e12, 2),
                     "l2_read_tbs": round(l2_gbs / 1e3, 2),
                     "gather_frac_of_l2_roof": round(gather16 / (avg_spmm * 1e-3) / (l2_gbs * 1e9), 4)},
        "spmmv_k32": {"ms": t32, "gbs": round(ach32, 1), "frac": round(ach32 / hbm_peak, 4),
                      "hierarchical_bound_ms": round(hier32, 4),
                      "hierarchical_frac": round(hier32 / t32, 4), "l2_read_gbs": round(l2_gbs, 1),
                      "gather_bytes": 4 * nnz32 * 32, "layouts": k32},
        "kernels_ms": {k: round(v, 4) for k, v in kern_ms.items()},
        "peak_mb": {"train_phase": round(peak_train / 2**20, 1),
                    "allocated_before_train": round(base_alloc / 2**20, 1),
                    "analytic_graph_plus_tensors": round(analytic / 2**20, 1),
                    "train_over_analytic": round(peak_train / analytic, 3),
                    "setup_peak_incl_device_build": round(setup_peak / 2**20, 1),
                    "cudaMemGetInfo_used_mb": round(dev_used / 2**20, 1),
                    "torch_reserved_mb": round(torch_reserved / 2**20, 1),
                    "note": "train phase: resident degree-sorted coalesced CSR+CSC (packed column + "
                            "multiplicity words, row_ids), X at "
                            "row stride 608, activations, workspaces; analytic = canonical "
                            "CSR+CSC (int64 offsets, int32 ids) + X + 6 [V,16] tensors"},
        "setup_s": {"generate+csr": round(t_gen, 3), "csc": round(t_csc, 3),
                    "coalesce": round(t_co, 3)},
        "loss": loss_val,
        "launches_per_step": int(launches_per_step),
    }
    res["clocks"] = clk.summary()

    if rank == 0 and not args.no_cpu_baseline:
        # one full-size oracle epoch on the host cores (after one untimed epoch
        # that faults the arrays in): SURVEY §8d CPU baseline, measured, not scaled
        cpu = CpuGcnEpoch(h_off, h_tgt, h_toff, h_trows, X_h.numpy(), y_h.numpy(), *p0)
        try:
            cpu.step()
            t0 = time.perf_counter()
            cpu_loss = cpu.step()
            cms = (time.perf_counter() - t0) * 1e3
        finally:
            cpu.close()
        res["cpu_baseline"] = {"value": round(cms, 1), "unit": "ms", "cores": cpu.workers,
                               "kind": "port", "sample": cpu.describe() + "; 1 timed epoch "
                               "after 1 warm-up", "loss_epoch2": cpu_loss, **cpu_info()}
    if not args.no_extras:
        # the other BASELINE configs, measured in the same run (not the headline)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_models as bm

        del tr
        torch.cuda.empty_cache()
        extras = {}
        for name, fn in (("gin_reddit", bm.run_gin), ("gat_products", bm.run_gat),
                         ("spmm_sweep_reddit", bm.run_sweep), ("sampling", bm.run_sampling),
                         ("minibatch_gcn_reddit", bm.run_minibatch),
                         ("gcn_reddit_variants", bm.run_variants),
                         ("csr_csc_build_reddit", bm.run_build),
                         ("gcn_papers100m", lambda: bm.run_papers100m(0, 1, steps=10, warmup=3))):
            try:
                extras[name] = fn()
            except Exception as exc:  # report, never hide
                extras[name] = {"error": repr(exc)[:300]}
            torch.cuda.empty_cache()
        res["extras"] = extras
    return res


# ------------------------------------------------- our arm, N > 1 ranks
def run_dist(args, rank, world):
    """Row-partitioned GCN epoch: every rank builds only its own
    cost-balanced row block of the CSR/CSC (bit-exact edge stream regenerated
    and filtered on its GPU) and exchanges [V, hidden] blocks with in-place
    NCCL all-gathers; one all-reduce of the weight gradients.  Strong
    scaling: the whole Reddit-shape epoch is fixed, split over N GPUs."""
    import torch

    import paper_2605_29346_b200 as gb
    from paper_2605_29346_b200 import _lib
    from paper_2605_29346_b200.dist import DistGCNTrainer, RowPartition, TorchDistExchange

    dev = torch.device("cuda", local_device())
    torch.cuda.set_device(dev)
    lib = _lib.lib()
    P = REDDIT
    V, E, F, Hd, C = P["V"], P["E"], P["F"], P["H"], P["C"]
    # per-rank build: this rank regenerates the bit-exact edge stream and keeps
    # only its rows of the CSR and CSC (graph.powerlaw_row_block) — no rank
    # ever holds the whole graph; bounds from the expected degree prefix
    from paper_2605_29346_b200.dist import ROW_COST, expected_bounds

    spec = gb.GraphGenSpec("power-law", V, E, exponent=P["exponent"])
    bounds = expected_bounds(spec, world, ROW_COST)
    blk = gb.graph.powerlaw_row_block(spec, P["seed"], int(bounds[rank]), int(bounds[rank + 1]),
                                      pack=False)
    # exchange: NCCL all-gathers (default) or, with GNN_DIST_EXCHANGE=peer, the
    # peer-memory form (gnn_spmm_peer reads every rank's block in place through
    # torch symmetric memory; phase boundaries are device-side barriers)
    mode = os.environ.get("GNN_DIST_EXCHANGE", "nccl")
    part = RowPartition.from_block(blk, world, rank, bounds, pow2_stride=(mode == "peer"))
    del blk
    g = None
    torch.cuda.empty_cache()
    rng = np.random.default_rng(np.random.SeedSequence(P["seed"], spawn_key=(10,)))
    X_all = rng.random((V, F), dtype=np.float32) * 2 - 1
    y_all = np.random.default_rng(np.random.SeedSequence(P["seed"], spawn_key=(13,))).integers(0, C, V)
    # this rank's rows, pinned at the device row stride (one linear H2D per step)
    Fpad = -(-F // 32) * 32
    X_h = torch.zeros(part.rows, Fpad, dtype=torch.float32).pin_memory()
    X_h[:, :F].copy_(torch.from_numpy(X_all[part.lo:part.hi]))
    y_h = torch.from_numpy(np.ascontiguousarray(y_all[part.lo:part.hi])).pin_memory()
    del X_all
    torch.cuda.reset_peak_memory_stats(dev)
    if mode == "peer":
        from paper_2605_29346_b200.dist import PeerExchange

        ex = PeerExchange()
        tr = DistGCNTrainer(part, F, Hd, C, seed=P["seed"], peer=True, alloc=lambda r, w, d: ex.alloc(r, w, d))
        tr.bind_peers(ex.peer_ptrs(tr))
    else:
        ex = TorchDistExchange()
        # overlap the all-gathers with the own-slot part of each aggregation
        # (GNN_DIST_OVERLAP=0 turns it off; no use with a single rank)
        overlap = world > 1 and os.environ.get("GNN_DIST_OVERLAP", "1") != "0"
        tr = DistGCNTrainer(part, F, Hd, C, seed=P["seed"], overlap=overlap)
        if overlap:  # the trainer holds the own-slot / other-slot parts; drop the unsplit slices
            part.A = part.AT = None
            torch.cuda.empty_cache()
    tr.set_inputs(X_h, y_h)
    c0 = lib.gnn_launch_counter()
    tr.step(ex)
    torch.cuda.synchronize()
    launches = lib.gnn_launch_counter() - c0
    for _ in range(args.warmup):
        tr.step(ex)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    with ClockSampler(dev.index) as clk:
        st = torch.cuda.current_stream()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(args.steps):
            tr.step(ex)
        b.record(st)
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    torch.distributed.barrier()
    loss_h = torch.empty(1, dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    torch.distributed.barrier()
    a.record(st)
    for _ in range(args.steps):
        tr.set_inputs(X_h, y_h, non_blocking=True)
        tr.step(ex)
        loss_h.copy_(tr.loss, non_blocking=True)
    b.record(st)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / args.steps
    t = torch.tensor([ms, e2e_ms], device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms, e2e_ms = float(t[0]), float(t[1])
    loss_val = float(tr.loss.item())
    peak_mb = round(torch.cuda.max_memory_allocated(dev) / 2**20, 1)
    clocks = clk.summary()
    overlapped = mode != "peer" and tr.overlap
    rows_rank0, bounds_l = part.rows, [int(x) for x in part.bounds]
    extras = {}
    if not args.no_extras:
        # BASELINE configs[4]: the papers100M-shaped epoch, row-partitioned over
        # these N ranks (per-rank block build; every rank runs it)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_models as bm

        del tr, part, g
        torch.cuda.empty_cache()
        try:
            extras["gcn_papers100m"] = bm.run_papers100m(rank, world, steps=10, warmup=3)
        except Exception as exc:  # report, never hide
            extras["gcn_papers100m"] = {"error": repr(exc)[:300]}
    return {
        "metric": "gcn_epoch_ms", "value": round(ms, 4), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (device power-law generator, bit-exact gsbench.generate seed 42; "
                "X~U[-1,1) f32, labels uniform)",
        "config": workload_config(world),
        "partition": {"how": "1D row partition (cost-balanced: deg + 170 per row) + "
                             + ("peer-memory SpMM (symmetric memory, NVLink loads)"
                                if mode == "peer" else "NCCL all-gathers"
                                + (" overlapped with own-slot aggregation"
                                   if overlapped else "")),
                      "rows_rank0": rows_rank0, "bounds": bounds_l},
        "layout": "coalesced", "l2": "inputs larger than L2: no flush needed",
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms",
                "h2d_bytes_per_step": int(X_h.numel() * 4 + y_h.numel() * 8),
                "d2h_bytes_per_step": 4},
        "gpu_launches": int(launches * args.steps),
        "peak_mb": {"train_phase": peak_mb},
        "loss": loss_val, "clocks": clocks,
        "dist": {"backend": torch.distributed.get_backend(), "world_size": world,
                 "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                 "nccl_log": "NCCL_DEBUG=INFO (INIT) on stderr: nranks per communicator"},
        "extras": extras,
    }


# -------------------------------------------------------- reference arm
def run_reference(args):
    """The reference CPU path of this workload: the oracle port (float64 numpy
    restatement of the reference's graph build + the GCN epoch, oracle/),
    timed on the host cores.  Honours --steps / --warmup: each step is one
    full-size epoch (no sampling).  Graph generation and the CSC build (the
    reference's own numpy algorithms, ~2 min) are setup, not timed."""
    from oracle import graph as og

    P = REDDIT
    V, E, F, Hd, C = P["V"], P["E"], P["F"], P["H"], P["C"]
    t0 = time.perf_counter()
    src, dst = og.powerlaw_edges(V, E, P["exponent"], P["seed"])
    off, tgt = og.csr_from_edges(V, src, dst)
    del src, dst
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    t_off, t_rows, _ = og.transpose(V, V, off, tgt)
    t_csc = time.perf_counter() - t0
    rng = np.random.default_rng(np.random.SeedSequence(P["seed"], spawn_key=(10,)))
    X = rng.random((V, F), dtype=np.float32) * 2 - 1
    y = np.random.default_rng(np.random.SeedSequence(P["seed"], spawn_key=(13,))).integers(0, C, V)

    def glorot(fi, fo, idx):  # same seeded init as the trainer (SURVEY §8d spawn_key 12)
        r = np.random.default_rng(np.random.SeedSequence(P["seed"], spawn_key=(12, idx)))
        a = (6.0 / (fi + fo)) ** 0.5
        return r.uniform(-a, a, (fi, fo)).astype(np.float32).astype(np.float64)

    cpu = CpuGcnEpoch(off, tgt, t_off, t_rows, X, y, glorot(F, Hd, 0), np.zeros(Hd),
                      glorot(Hd, C, 2), np.zeros(C))
    times = []
    try:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            loss = cpu.step()
            if i >= args.warmup:
                times.append((time.perf_counter() - t0) * 1e3)
    finally:
        cpu.close()
    v = statistics.mean(times)
    return {"metric": "gcn_epoch_ms", "value": round(v, 1), "unit": "ms", "n_gpus": args.gpus,
            "device": "cpu (the reference path is host code; n_gpus = the run's N)",
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v, 1),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gsbench power-law restatement, seed 42; X~U[-1,1), labels uniform)",
            "config": workload_config(args.gpus),
            "impl": "reference",
            "cpu_baseline": {"value": round(v, 1), "unit": "ms", "cores": cpu.workers,
                             "kind": "port", "sample": cpu.describe() + "; every step one epoch",
                             **cpu_info()},
            "e2e": {"value": round(v, 1), "unit": "ms", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "loss_last": loss,
            "setup_s": {"generate+csr": round(t_gen, 1), "csc": round(t_csc, 1)}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--layout", choices=["canonical", "coalesced"], default="coalesced")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the GIN / GAT / SpMM-sweep lines of the other BASELINE configs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch

        torch.cuda.set_device(local_device())
        # NCCL's init log (nranks, rings / NVLS) on stderr, so the scaling run can
        # verify the communicator size; stdout keeps the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        # NCCL over NVLink/NVSwitch; GNN_DIST_BACKEND=gloo lets the partitioned path be
        # exercised with several ranks sharing one GPU (test only, not a bench number)
        torch.distributed.init_process_group(os.environ.get("GNN_DIST_BACKEND", "nccl"))
        res = run_dist(args, rank, world)
        torch.distributed.destroy_process_group()
    else:
        res = run_ours(args, rank, world)
    if rank == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
