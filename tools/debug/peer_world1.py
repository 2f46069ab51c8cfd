"""Smoke of the PeerExchange plumbing with a 1-rank NCCL group (the only
multi-process form one GPU allows): symmetric-memory alloc + rendezvous +
device barrier + bind_peers, then one peer-mode epoch vs the all-gather mode."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29611")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
import paper_2605_29346_b200 as gb
from paper_2605_29346_b200.dist import DistGCNTrainer, PeerExchange, RowPartition, TorchDistExchange
g = gb.generate(gb.GraphGenSpec("power-law", 20000, 400000, exponent=2.1), 1)
X = torch.rand(20000, 64); y = torch.randint(0, 7, (20000,))
ex = PeerExchange()
p = RowPartition(g, 1, 0, pow2_stride=True)
t = DistGCNTrainer(p, 64, 16, 7, seed=0, peer=True, alloc=lambda r, w, d: ex.alloc(r, w, d))
t.bind_peers(ex.peer_ptrs(t))
t.set_inputs(X, y)
l1 = t.step(ex).item()
t2 = DistGCNTrainer(RowPartition(g, 1, 0), 64, 16, 7, seed=0)
t2.set_inputs(X, y)
l2 = t2.step(TorchDistExchange()).item()
torch.cuda.synchronize()
print("peer", l1, "nccl", l2, "equal", l1 == l2,
      all(torch.equal(a, b) for a, b in zip(t.params().values(), t2.params().values())))
dist.destroy_process_group()
