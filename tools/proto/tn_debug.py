import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_29346_b200 as gb
K, M, N = 1024, 128, 16
torch.manual_seed(0)
# test A layout: B = e_n at row k=n -> C[m,n] = A[n,m]
A = torch.randn(K, M, device="cuda"); B = torch.zeros(K, N, device="cuda")
for n in range(N): B[n, n] = 1.0
C = gb.gemm(A, B, trans_a=True).cpu(); ref = (A.T @ B).cpu()
print("A-test max err", (C - ref).abs().max().item())
bad = ((C - ref).abs() > 1e-3).nonzero()
print("bad (m,n) sample", bad[:10].tolist())
# test B layout: A = ones -> C[m,n] = sum_k B[k,n]
A = torch.ones(K, M, device="cuda"); B = torch.randn(K, N, device="cuda")
C = gb.gemm(A, B, trans_a=True).cpu(); ref = (A.T @ B).cpu()
print("B-test max err", (C - ref).abs().max().item(), "rel", ((C-ref).abs().max()/ref.abs().max()).item())
# only first k-block nonzero
B2 = torch.zeros(K, N, device="cuda"); B2[:32] = torch.randn(32, N, device="cuda")
A2 = torch.randn(K, M, device="cuda")
C = gb.gemm(A2, B2, trans_a=True).cpu(); ref = (A2.T @ B2).cpu()
print("kblock0 max err", (C - ref).abs().max().item())
for r in range(0, 32, 8):
    B3 = torch.zeros(K, N, device="cuda"); B3[r:r+8] = torch.randn(8, N, device="cuda")
    C = gb.gemm(A2, B3, trans_a=True).cpu(); ref = (A2.T @ B3).cpu()
    print(f"rows {r}-{r+7} max err", (C - ref).abs().max().item())
# precision: random both
A = torch.randn(K, M, device="cuda"); B = torch.randn(K, N, device="cuda")
C = gb.gemm(A, B, trans_a=True).double().cpu(); ref = A.double().T.cpu() @ B.double().cpu()
print("random rel", ((C - ref).abs().max() / ref.abs().max()).item())
