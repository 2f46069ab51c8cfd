"""Profiling driver: one SpMMv (NORM) on the Reddit-shape graph, layout and K
from argv (default csr_coalesced 16)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_29346_b200 as gb
from paper_2605_29346_b200 import _lib
from paper_2605_29346_b200.kernels import SpmmCall

layout = sys.argv[1] if len(sys.argv) > 1 else "csr_coalesced"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = gb.generate(gb.GraphGenSpec("power-law", 232_965, 114_615_892, exponent=2.1), 42)
op = g.operand(layout)
X = torch.rand(232_965, K, device="cuda")
Y = torch.empty_like(X)
call = SpmmCall(op, X, Y, flags=_lib.EPI_NORM if "csr" in layout else 0)
for _ in range(3):
    call()
torch.cuda.synchronize()
print("done")
