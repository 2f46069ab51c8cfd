import sys, os, shutil; sys.path.insert(0,'.')
lib = sys.argv[1]
if lib != "default":
    shutil.copy(lib, "paper_2605_29346_b200/libgnnb200.so")
import torch, statistics
import paper_2605_29346_b200 as gb
from paper_2605_29346_b200.models import GCNTrainer
g = gb.generate(gb.GraphGenSpec("power-law", 232965, 114615892, exponent=2.1), 42)
tr = GCNTrainer(g, 602, 16, 41, seed=42, coalesced=True)
tr.set_inputs(torch.rand(232965, 602), torch.randint(0, 41, (232965,)))
tr.step()
per = [tr.timed_step() for _ in range(5)]
print(lib, {k: round(statistics.median(p[k] for p in per), 4) for k in ("head", "X.W1", "X^T.dH1", "mask_norm_db1")})
