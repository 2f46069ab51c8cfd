"""Time the fused output layer alone (gnn_gcn_head_scaled) at a given shape.
    python tools/prof_head.py [M] [Din] [C]      (default: papers100M 111059956 16 172)
GNN_HEAD_LANES=1 selects the lane-per-class wide form instead of thread-per-row."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_29346_b200.kernels import HeadCall

M, Din, C = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (111_059_956, 16, 172)))
dev = torch.device("cuda")
P = torch.rand(M, Din, device=dev) * 2 - 1
W = torch.rand(Din, C, device=dev) - 0.5
b = torch.zeros(C, device=dev)
y = torch.randint(0, C, (M,), device=dev)
deg = torch.arange(M + 1, device=dev, dtype=torch.int64) * 3
dP = torch.empty_like(P)
dW, db, loss = torch.empty(Din, C, device=dev), torch.empty(C, device=dev), torch.empty(1, device=dev)
h = HeadCall(P, W, b, y, dP, dW, db, loss, deg_offsets=deg)
for _ in range(2):
    h()
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    h()
e.record()
torch.cuda.synchronize()
ms = a.elapsed_time(e) / 5
print(f"head M={M} Din={Din} C={C} lanes={os.environ.get('GNN_HEAD_LANES', '1')}: {ms:.3f} ms, "
      f"{2 * 3 * M * Din * C / ms / 1e9:.1f} TFLOP/s (3 x 2*Din*C flop/row), loss {loss.item():.4f}")
