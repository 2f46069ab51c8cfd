"""SpMM micro-sweep on the Reddit-shape graph: layouts x K x edges-per-warp."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_29346_b200 as gb
from paper_2605_29346_b200 import _lib
from paper_2605_29346_b200.kernels import SpmmCall

V, E = 232_965, 114_615_892
g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
g.csc()
g.csr_coalesced()
g.csc_coalesced()
flush = torch.empty(64 * 2**20, device="cuda")
res = {}
for K in [int(k) for k in (sys.argv[1:] or ["16", "32"])]:
    X = torch.rand(V, K, device="cuda")
    Y = torch.empty_like(X)
    for layout in ("csr", "csr_coalesced", "csc", "csc_coalesced"):
        for P in [int(x) for x in os.environ.get('SWEEP_P', '512,1024,2048').split(',')]:
            call = SpmmCall(g.operand(layout), X, Y, flags=_lib.EPI_NORM if "csr" in layout else 0,
                            edges_per_warp=P)
            ts = []
            for _ in range(12):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                torch.cuda._sleep(3_000_000)  # host runs ahead: no launch gap in the window
                a.record()
                call()
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            res[f"K{K} {layout} P{P}"] = round(statistics.median(ts[2:]), 4)
            print(f"K={K:3d} {layout:14s} P={P:5d}  {res[f'K{K} {layout} P{P}']:.4f} ms", flush=True)
