"""Launch list of the replayed sampled mini-batch step (run under ncu):
capture, then two replays (Reddit shape, B=1024, fanouts (25, 10))."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_29346_b200 as gb
from paper_2605_29346_b200.models import SampledGCNTrainer
from paper_2605_29346_b200.sampling import SampleConfig

V, E = 232_965, 114_615_892
g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
X = torch.rand(V, 602, device="cuda") * 2 - 1
y = torch.randint(0, 41, (V,), device="cuda")
tr = SampledGCNTrainer(g, X, y, 602, 16, 41, SampleConfig(1024, (25, 10)), seed=42)
tr.capture()
rng = np.random.default_rng(0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for i in range(2):
    tr.run(rng.choice(V, 1024, replace=False), rng=i)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
