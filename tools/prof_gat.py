"""Profiling driver (run under ncu on the GPU box): products-shape GAT
trainer, eager epochs, so every GAT kernel launches with its real inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_29346_b200 as gb
from paper_2605_29346_b200.models import GATTrainer

V, E = 2_449_029, 123_718_280
g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
tr = GATTrainer(g, 100, 16, 47, heads=4, seed=42)
tr.set_inputs(torch.rand(V, 100) * 2 - 1, torch.randint(0, 47, (V,)))
tr.step()  # warm (plans, workspaces); ncu --profile-from-start off sees only the epochs below
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(int(os.environ.get("EPOCHS", "1"))):
    tr.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
