import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2605_29346_b200 as gb
from paper_2605_29346_b200.models import GINTrainer
from oracle import ops as oo, graph as og
g = gb.generate(gb.GraphGenSpec("power-law", 2708, 10556, exponent=2.1), 42)
V, F, Hd, C = g.num_vertices, 70, 32, 9
X = np.random.default_rng(1).uniform(-1, 1, (V, F)).astype(np.float32) * 1e-3
y = np.random.default_rng(2).integers(0, C, V)
tr = GINTrainer(g, F, Hd, C, eps=0.1, seed=4, coalesced=False)
tr.set_inputs(torch.from_numpy(X), torch.from_numpy(y))
tr.forward_backward(); torch.cuda.synchronize()
p = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in tr.params().items()}
off, tgt = g.offsets, g.targets
t_off, t_rows, _ = og.transpose(V, V, off, tgt)
Xd = X.astype(np.float64)
H1 = Xd @ p["W1a"]; U1 = np.maximum(oo.spmm(off, tgt, H1) + 1.1 * H1 + p["b1a"], 0)
Y1 = np.maximum(U1 @ p["W1b"] + p["b1b"], 0)
H2 = Y1 @ p["W2a"]; U2 = np.maximum(oo.spmm(off, tgt, H2) + 1.1 * H2 + p["b2a"], 0)
Z = U2 @ p["W2b"] + p["b2b"]
loss, dZ = oo.cross_entropy(Z, y)
dU2 = (dZ @ p["W2b"].T) * (U2 > 0)
dH2 = oo.spmm(t_off, t_rows, dU2) + 1.1 * dU2
def cmp(name, got, ref):
    got = got.detach().cpu().numpy().astype(np.float64)
    print(name, np.abs(got - ref).max() / np.abs(ref).max())
cmp("H1", tr.H1, H1); cmp("U1", tr.U1, U1); cmp("Y1", tr.Y1, Y1); cmp("H2", tr.H2, H2); cmp("U2", tr.U2, U2)
cmp("dU2", tr.dU2, dU2); cmp("dH2", tr.dH2, dH2)
cmp("dW2a", tr.dW2a, Y1.T @ dH2)
cmp("dW2a_from_gpu_inputs", tr.dW2a, tr.Y1.double().cpu().numpy().T @ tr.dH2.double().cpu().numpy())
print("ref dW2a max", np.abs(Y1.T @ dH2).max(), "abs", (np.abs(Y1).T @ np.abs(dH2)).max())
