"""Does tcgen05 kind::tf32 truncate fp32 operands (ignore the low 13 mantissa bits)?
Compare the TC GEMM with GNN_TC_RAWHI=1 (A_hi not written back) to float64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_29346_b200 as gb
rng = np.random.default_rng(0)
M, K, N = 4096, 608, 16
a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
b = rng.uniform(-1, 1, (K, N)).astype(np.float32)
C = gb.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
ref = a.astype(np.float64) @ b.astype(np.float64)
sc = np.abs(a).astype(np.float64) @ np.abs(b)
print(os.environ.get("GNN_TC_RAWHI", "0"), "max scaled err", np.max(np.abs(C - ref) / sc))
