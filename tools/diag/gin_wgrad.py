"""Diagnostic: isolate the GIN full-size weight-gradient GEMMs (device inputs,
float64 host product) to see which stage carries the W1b error."""
import numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2605_29346_b200 as gb
from paper_2605_29346_b200.models import GINTrainer
V, E, F, C = 232_965, 114_615_892, 602, 41
g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
rng = np.random.default_rng(np.random.SeedSequence(42, spawn_key=(10,)))
X = (rng.random((V, F), dtype=np.float32) * 2 - 1)
y = np.random.default_rng(np.random.SeedSequence(42, spawn_key=(13,))).integers(0, C, V)
tr = GINTrainer(g, F, 64, C, eps=0.1, seed=42)
tr.set_inputs(torch.from_numpy(X), torch.from_numpy(y))
tr.forward_backward(); torch.cuda.synchronize()
def chk(name, A, B, D):
    A = A.cpu().double().numpy(); B = B.cpu().double().numpy(); D = D.cpu().double().numpy()
    ref = A.T @ B; ab = np.abs(A).T @ np.abs(B)
    s = np.maximum(np.abs(ref), ab)
    e = np.abs(D - ref) / s
    i = np.unravel_index(np.argmax(e), e.shape)
    print(name, "max scaled err %.3e at %s ref %.4e abs %.4e dev %.4e; median %.2e" % (e.max(), i, ref[i], ab[i], D[i], np.median(e)))
    # same with fp32-cast inputs sums in float32 sequential blocks for comparison
chk("W1b=U1^T dY1", tr.U1, tr.dY1, tr.dW1b)
chk("W2a=Y1^T dH2", tr.Y1, tr.dH2, tr.dW2a)
chk("W1a=X^T dH1", tr.X, tr.dH1, tr.dW1a)
U1 = tr.U1.cpu().double().numpy(); dY1 = tr.dY1.cpu().double().numpy()
print("U1 max %.3e dY1 max %.3e; rows with |U1|>1e3: %d" % (np.abs(U1).max(), np.abs(dY1).max(), (np.abs(U1).max(1) > 1e3).sum()))
# emulate: fp32 sequential accumulation chains of length L
for L in (1024, 8192, 65536):
    acc = np.zeros((64, 64), np.float32)
    for r0 in range(0, V, L):
        acc += (U1[r0:r0+L].T @ dY1[r0:r0+L]).astype(np.float32)
    ref = U1.T @ dY1; ab = np.abs(U1).T @ np.abs(dY1)
    print("block-f32 L=%d scaled err %.3e" % (L, (np.abs(acc - ref) / np.maximum(np.abs(ref), ab)).max()))
# 1xTF32 emulation error bound for reference
def tf32(a):
    a = a.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000); return a.view(np.float32).astype(np.float64)
U32 = tr.U1.cpu().numpy(); d32 = tr.dY1.cpu().numpy()
Uh, dh = tf32(U32), tf32(d32); Ul, dl = tf32(U32 - Uh), tf32(d32 - dh)
e3 = Uh.T @ dh + Uh.T @ dl + Ul.T @ dh
ref = U1.T @ dY1; ab = np.abs(U1).T @ np.abs(dY1)
print("3xTF32 exact-acc emulation scaled err %.3e" % (np.abs(e3 - ref) / np.maximum(np.abs(ref), ab)).max())
