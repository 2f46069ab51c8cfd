"""Launch list of the device CSR / CSC(+eid) builders on the Reddit shape
(run under ncu --metrics gpu__time_duration.sum): one warm call each, then
the profiled pair between NVTX-free markers (cudaDeviceSynchronize)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2605_29346_b200 as gb
V, E = 232_965, 114_615_892
src, dst = gb.graph.powerlaw_edges_device(V, E, 2.1, 42)
for rep in range(2):
    torch.cuda.synchronize()
    g = gb.csr_from_edges(V, src, dst, device="cuda")
    torch.cuda.synchronize()
    g.csc(with_eid=True)
    torch.cuda.synchronize()
    del g
print("ok")
