"""Smoke of the overlapped all-gather path with a 1-rank NCCL group (the only
multi-process form one GPU allows): async all_gather_into_tensor + work.wait
around the own-slot / other-slot split aggregations, several epochs vs the
non-overlapped schedule and the single-GPU trainer."""
import os
import sys

sys.path.insert(0, '.')
import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29613")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
import paper_2605_29346_b200 as gb
from paper_2605_29346_b200.dist import DistGCNTrainer, RowPartition, TorchDistExchange
from paper_2605_29346_b200.models import GCNTrainer

g = gb.generate(gb.GraphGenSpec("power-law", 20000, 400000, exponent=2.1), 1)
X = torch.rand(20000, 64)
y = torch.randint(0, 7, (20000,))
ex = TorchDistExchange()
a = DistGCNTrainer(RowPartition(g, 1, 0), 64, 16, 7, seed=0, overlap=True)
b = DistGCNTrainer(RowPartition(g, 1, 0), 64, 16, 7, seed=0)
s = GCNTrainer(g, 64, 16, 7, seed=0, coalesced=True)
for t in (a, b, s):
    t.set_inputs(X, y)
for k in range(5):
    la, lb, ls = a.step(ex).item(), b.step(ex).item(), s.step().item()
    print(k, la, lb, ls, flush=True)
torch.cuda.synchronize()
ok = all(torch.allclose(p, q, rtol=1e-4, atol=1e-6) for p, q in zip(a.params().values(), s.params().values()))
print("overlap params match single-GPU:", ok)
dist.destroy_process_group()
