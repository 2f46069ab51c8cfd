"""Small end-to-end exercise of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): SpMM (row order, degree-sorted, packed,
shared heads, split rows), SDDMM, edge softmax, GAT backward, GEMMs, fused
heads, GCN/GAT trainer steps, sampling.  Sizes are tiny so the sanitizers
finish in minutes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_29346_b200 as gb
from paper_2605_29346_b200 import _lib
from paper_2605_29346_b200.kernels import SharedHeadsCall, SpmmCall
from paper_2605_29346_b200.models import GATTrainer, GCNTrainer, GINTrainer

torch.manual_seed(0)
rng = np.random.default_rng(0)
# a mega row + empty rows + a power-law body, so split rows and every plan path run
src = np.concatenate([np.zeros(20_000, np.int64), rng.integers(1, 300, 4000), rng.integers(0, 3000, 30_000)])
dst = rng.integers(0, 3000, src.size)
g = gb.csr_from_edges(3000, src, dst)
for K in (4, 16, 32, 64, 130):
    X = torch.rand(3000, K, device="cuda")
    for op in (g.csr(), g.csc(), g.csr_coalesced(), g.csc_coalesced()):
        Y = torch.empty(3000, K, device="cuda")
        SpmmCall(op, X, Y, flags=_lib.EPI_NORM if op.deg_offsets is not None else 0)()
al = torch.rand(g.num_edges, 4, device="cuda")
SharedHeadsCall(g.csr(), torch.rand(3000, 16, device="cuda"), al, torch.empty(3000, 64, device="cuda"), 0.25)()
pl = gb.generate(gb.GraphGenSpec("power-law", 2000, 20_000, exponent=2.1), 3)
Xh = torch.rand(2000, 40)
yh = torch.randint(0, 7, (2000,))
for co in (False, True):
    t = GCNTrainer(pl, 40, 16, 7, seed=0, coalesced=co)
    t.set_inputs(Xh, yh)
    t.step()
t = GCNTrainer(pl, 40, 16, 90, seed=0)  # wide output layer (tcgen05 head, head_tc.cu)
t.set_inputs(Xh, torch.randint(0, 90, (2000,)))
t.step()
t = GCNTrainer(pl, 40, 16, 172, seed=0)  # 172 classes: both epilogue halves, both dW blocks
t.set_inputs(Xh, torch.randint(0, 172, (2000,)))
t.step()
# device builders: stable radix sorts (1-3 passes), offsets with long empty gaps
from paper_2605_29346_b200.graph import _offsets_from_keys, _sort_pairs  # noqa: E402

for R in (300, 100_000, 1 << 27):
    k = torch.randint(0, R, (50_001,), device="cuda", dtype=torch.int32)
    ko, vo = _sort_pairs(k, torch.arange(50_001, device="cuda", dtype=torch.int32), R)
    _offsets_from_keys(ko, R if R < (1 << 20) else 1 << 20) if R < (1 << 20) else None
gb.csr_from_edges(3000, src, dst).csc(with_eid=True)
# replayed sampled mini-batch step (device-count plans, live-row limits)
from paper_2605_29346_b200.models import SampledGCNTrainer  # noqa: E402
from paper_2605_29346_b200.sampling import SampleConfig  # noqa: E402

st = SampledGCNTrainer(pl, Xh.cuda(), yh.cuda(), 40, 16, 7, SampleConfig(batch_size=64, fanouts=(5, 4)),
                       seed=0)
st.capture()
for i in range(2):
    st.run(rng.choice(2000, 64, replace=False), rng=i)
t = GINTrainer(pl, 40, 64, 7, seed=0)
t.set_inputs(Xh, yh)
t.step()
t = GATTrainer(pl, 40, 16, 7, heads=4, seed=0)
t.set_inputs(Xh, yh)
t.step()
torch.cuda.synchronize()
print("sanitize smoke done")
