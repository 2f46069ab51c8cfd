import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_29346_b200 as gb
K, M, N = 1024, 128, 16
A = torch.arange(K * M, device="cuda", dtype=torch.float32).reshape(K, M) % 7 + 1
B = torch.ones(K, N, device="cuda")
C = gb.gemm(A, B, trans_a=True)
torch.cuda.synchronize()
print("C[:2,:4]", C[:2, :4].tolist(), "ref", (A.T @ B)[:2, :4].tolist())
