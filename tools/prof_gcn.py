"""Profiling driver (run under ncu on the GPU box): builds the Reddit-shape
graph on device, then runs eager GCN epochs and standalone SpMMv calls."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_29346_b200 as gb
from paper_2605_29346_b200 import _lib
from paper_2605_29346_b200.kernels import SpmmCall
from paper_2605_29346_b200.models import GCNTrainer

ap = argparse.ArgumentParser()
ap.add_argument("--epochs", type=int, default=2)
ap.add_argument("--spmm-k", type=int, nargs="*", default=[32])
ap.add_argument("--layout", default="canonical")
a = ap.parse_args()
V, E = 232_965, 114_615_892
g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
tr = GCNTrainer(g, 602, 16, 41, seed=42, coalesced=a.layout == "coalesced")
X = torch.rand(V, 602) * 2 - 1
y = torch.randint(0, 41, (V,))
tr.set_inputs(X, y)
tr.step()  # warm (plans, workspaces)
torch.cuda.synchronize()
# ncu --profile-from-start off: only the epochs below are captured
torch.cuda.profiler.start()
for _ in range(a.epochs):
    tr.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
for K in a.spmm_k:
    Xk = torch.rand(V, K, device="cuda")
    Yk = torch.empty_like(Xk)
    for layout in ("csr", "csr_coalesced"):
        SpmmCall(g.operand(layout), Xk, Yk, flags=_lib.EPI_NORM)()
torch.cuda.synchronize()
print("done")
