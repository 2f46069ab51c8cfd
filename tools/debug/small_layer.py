import sys; sys.path.insert(0,'.')
import torch
import paper_2605_29346_b200 as gb
from paper_2605_29346_b200 import _lib
from paper_2605_29346_b200.kernels import GemmCall, SpmmCall
for (V,E) in [(2000,20000),(2000,400000),(20000,200000)]:
    g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 0)
    A, AT = g.csr(), g.csc()
    K=128
    X = torch.rand(V, K, device="cuda"); W = torch.rand(K, 16, device="cuda")
    H, Y, dY, dH = (torch.empty(V, 16, device="cuda") for _ in range(4)); dW = torch.empty(K, 16, device="cuda")
    calls = {"gemm": GemmCall(X, W, H), "spmm": SpmmCall(A, H, Y, flags=_lib.EPI_NORM), "spmmT": SpmmCall(AT, dY, dH), "gemmT": GemmCall(X, dH, dW, trans_a=True)}
    for n,c in calls.items():
        for _ in range(3): c()
        torch.cuda.synchronize()
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2000000)
        a.record()
        for _ in range(20): c()
        b.record(); torch.cuda.synchronize()
        print(V,E,n, round(a.elapsed_time(b)*1e3/20,2), "us", "P=",A.plan().edges_per_warp, "nsplit",A.plan().num_split, "T nsplit", AT.plan().num_split)
