"""Times the GAT trainer's kernels (eager epoch) on the products shape; env
vars select kernel variants.  Prints {name: ms} for the listed kernels."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_29346_b200 as gb
from paper_2605_29346_b200.models import GATTrainer
V, E = 2_449_029, 123_718_280
g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
tr = GATTrainer(g, 100, 16, 47, heads=4, seed=42)
tr.set_inputs(torch.rand(V, 100) * 2 - 1, torch.randint(0, 47, (V,)))
tr.step()
per = [tr.timed_step() for _ in range(3)]
km = {k: round(statistics.median(p[k] for p in per), 3) for k in per[0]}
keys = sys.argv[1:] or list(km)
print(json.dumps({k: km[k] for k in keys}))
