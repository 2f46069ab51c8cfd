"""Full-size GAT parity (BASELINE configs[3]): one products-shaped epoch
(V=2,449,029, E=123,718,280, power-law 2.1, seed 42; K=100 -> 4 x 16 hidden
-> 4 x 47 averaged; the bench's GATTrainer in its default backward form),
checked stage by stage against float64 restatements of oracle/ops.py
gat_layer_fwd / gat_layer_bwd / cross_entropy, elementwise (SURVEY.md
Appendix A.8: |gpu - ref| <= 1e-5 * max(|ref|, ref_abs), ref_abs = the same
contraction on |inputs|).

Staged: every stage takes the device's own outputs of the stages before it
as inputs (each already checked), so an error is attributed to the launch
that made it.  The oracle's whole-graph gat2_step is out of reach at this
size (float64 edge tensors of E x H), so the per-row and per-column stages
run on samples that include the graph's hubs:

* rows R: every row whose out-degree is in the top until >= 900k edges,
  plus 4096 random rows — alpha, both aggregations, ds and der are checked
  on all of their edges (>= 1M edges);
* columns U: the top in-degree columns until >= 900k in-edges, plus 4096
  random columns — del and dWh (the SpMMve^T over the CSC) on all of their
  in-edges;
* whole-graph reductions (db, da_l, da_r, dW) are checked over all V rows,
  the float64 sums streamed from the device in row chunks.

The layer-2 ds / der / del are snapshotted right after the layer-2
backward (the trainer reuses those buffers for layer 1)."""

import numpy as np
import pytest
import torch

from oracle import ops as oo

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RTOL = 1e-5
V, E, F, HID, C, H = 2_449_029, 123_718_280, 100, 16, 47, 4
SLOPE = 0.2
CHUNK = 1 << 18


def _close(name, got, ref, ref_abs=None):
    ok, worst = oo.close(got, ref, ref_abs, RTOL)
    assert ok, (name, worst)
    print(f"{name}: {np.size(got)} values, worst |err| / (1e-5 scale) = {worst / RTOL:.3f}")
    return worst


def _edges_of(off, rows):
    """CSR positions of the rows' edges; local offsets."""
    starts = off[rows]
    deg = off[rows + 1] - starts
    lofs = np.zeros(rows.size + 1, np.int64)
    np.cumsum(deg, out=lofs[1:])
    idx = np.repeat(starts - lofs[:-1], deg) + np.arange(lofs[-1], dtype=np.int64)
    return idx, lofs


def _seg(x, lofs, op=np.add):
    deg = np.diff(lofs)
    out = np.zeros((deg.size,) + x.shape[1:], np.float64)
    nz = deg > 0
    if np.any(nz):
        out[nz] = op.reduceat(x, lofs[:-1][nz], axis=0)
    return out


def _sample(deg, rng, need=900_000, extra=4096):
    order = np.argsort(-deg, kind="stable")
    k = int(np.searchsorted(np.cumsum(deg[order]), need)) + 1
    pick = np.union1d(order[:k], rng.choice(deg.size, extra, replace=False))
    return pick.astype(np.int64)


def _rows(t, idx):
    """Device rows -> float64 host (idx: host int64)."""
    return t[torch.from_numpy(idx).to(t.device)].double().cpu().numpy()


def _stream(*ts):
    """Float64 host chunks of equal-row device tensors."""
    n = ts[0].shape[0]
    for r0 in range(0, n, CHUNK):
        yield [t[r0:r0 + CHUNK].double().cpu().numpy() for t in ts]


def _proj(Wh, a):
    Whr = Wh.reshape(Wh.shape[0], H, -1)
    return (Whr * a[None]).sum(-1), (np.abs(Whr) * np.abs(a)[None]).sum(-1)


def _softmax_rows(el_u, er_v, lofs):
    """alpha per edge (rows = local CSR segments) and the pre-activation."""
    pre = el_u + er_v
    s = np.where(pre > 0, pre, SLOPE * pre)
    deg = np.diff(lofs)
    m = _seg(s, lofs, np.maximum)
    ex = np.exp(s - np.repeat(m, deg, axis=0))
    sm = _seg(ex, lofs)
    return ex / np.repeat(sm, deg, axis=0), pre


def _agg(alpha, Xu, lofs, Fh):
    """Y[v, h*Fh+f] = sum_e alpha[e,h] X[u_e, h*Fh+f] and its |.| scale."""
    n = alpha.shape[0]
    prod = alpha[:, :, None] * Xu.reshape(n, H, Fh)
    y = _seg(prod.reshape(n, H * Fh), lofs)
    ya = _seg(np.abs(prod).reshape(n, H * Fh), lofs)
    return y, ya


def _ds(alpha, dalpha, dalpha_abs, pre, lofs):
    """Edge-softmax + LeakyReLU backward (oracle edge_softmax_backward), with
    its scale: the subtraction dalpha - S turned into an addition."""
    deg = np.diff(lofs)
    S = np.repeat(_seg(alpha * dalpha, lofs), deg, axis=0)
    Sa = np.repeat(_seg(alpha * dalpha_abs, lofs), deg, axis=0)
    lr = np.where(pre > 0, 1.0, SLOPE)
    return alpha * (dalpha - S) * lr, alpha * (dalpha_abs + Sa) * lr


@pytest.fixture(scope="module")
def epoch(cuda):
    import paper_2605_29346_b200 as gb
    from paper_2605_29346_b200.models import GATTrainer

    g = gb.generate(gb.GraphGenSpec("power-law", V, E, exponent=2.1), 42)
    rng = np.random.default_rng(np.random.SeedSequence(42, spawn_key=(20,)))
    X = rng.random((V, F), dtype=np.float32) * 2 - 1
    y = rng.integers(0, C, V)
    tr = GATTrainer(g, F, HID, C, heads=H, seed=42)
    tr.set_inputs(torch.from_numpy(X), torch.from_numpy(y))
    p = {k: v.detach().double().cpu().numpy() for k, v in tr.params().items()}
    off = np.asarray(g.offsets, np.int64)
    tgt = np.asarray(g.targets)
    R = _sample(np.diff(off), rng)
    idxR, lofsR = _edges_of(off, R)
    AT = tr.AT
    t_off = AT.offsets.cpu().numpy().astype(np.int64)
    U = _sample(np.diff(t_off), rng)
    idxU, lofsU = _edges_of(t_off, U)
    dev_idxU = torch.from_numpy(idxU).to(cuda)
    teid = AT.eid[dev_idxU].long()
    trows = AT.cols[dev_idxU].long().cpu().numpy()
    dev_idxR = torch.from_numpy(idxR).to(cuda)
    snap = {}
    names = [n for n, _ in tr.schedule()]
    assert "proj2_bwd" in names and tr.rc and tr.fr, names
    for name, call in tr.schedule():
        if name == "adam":
            continue
        call()
        if name == "proj2_bwd":  # layer-2 edge / vertex gradients, before layer 1 reuses them
            snap = {"ds_R": tr.ds[dev_idxR].double().cpu().numpy(),
                    "ds_U": tr.ds[teid].double().cpu().numpy(),
                    "der": tr.der.double().cpu().numpy(),
                    "del": tr.del_.double().cpu().numpy()}
    torch.cuda.synchronize()
    assert idxR.size >= 1_000_000 and idxU.size >= 1_000_000
    print(f"sample: {R.size} rows / {idxR.size} edges (max out-degree {np.diff(off).max()}), "
          f"{U.size} columns / {idxU.size} in-edges (max in-degree {np.diff(t_off).max()})")
    return dict(tr=tr, p=p, X=X, y=y, R=R, idxR=idxR, lofsR=lofsR, uR=tgt[idxR].astype(np.int64),
                U=U, lofsU=lofsU, vU=trows, teid=teid, dev_idxR=dev_idxR, snap=snap)


def _layer_forward(d, Wh, el, er, alpha, label, Xin, W, a_l, a_r, Fh):
    """Stages: Wh rows, el/er, alpha on R's edges.  Returns the f64 alpha and
    the pre-activations (the backward stages use them)."""
    R, idxR, lofsR, uR = d["R"], d["idxR"], d["lofsR"], d["uR"]
    Xr = Xin(R)
    _close(f"Wh{label}", _rows(Wh, R), Xr @ W, np.abs(Xr) @ np.abs(W))
    chk = np.union1d(R, d["U"])
    Whc = _rows(Wh, chk)
    for nm, dev, a in (("el", el, a_l), ("er", er, a_r)):
        ref, ra = _proj(Whc, a)
        _close(f"{nm}{label}", _rows(dev, chk), ref, ra)
    alpha_ref, pre = _softmax_rows(_rows(el, uR), np.repeat(_rows(er, R), np.diff(lofsR), axis=0),
                                   lofsR)
    _close(f"alpha{label}", alpha[d["dev_idxR"]].double().cpu().numpy(), alpha_ref)
    return alpha_ref, pre


def test_products_gat_forward(epoch):
    d, tr, p = epoch, epoch["tr"], epoch["p"]
    R, lofsR, uR = d["R"], d["lofsR"], d["uR"]
    Cp, K1 = tr.Cp, H * HID
    # layer 1
    _layer_forward(d, tr.Wh1, tr.el1, tr.er1, tr.alpha1, "1", lambda r: d["X"][r].astype(np.float64),
                   p["W1"], p["al1"], p["ar1"], HID)
    a1 = tr.alpha1[d["dev_idxR"]].double().cpu().numpy()
    pre, pa = _agg(a1, _rows(tr.Wh1, uR), lofsR, HID)
    _close("Y1", _rows(tr.Y1, R), np.maximum(pre + p["b1"], 0), pa + np.abs(p["b1"]))
    # layer 2 (padded head width Cp: the padding columns of W2 are zero)
    W2 = tr.W2.double().cpu().numpy()
    al2, ar2 = tr.al2.double().cpu().numpy(), tr.ar2.double().cpu().numpy()
    _layer_forward(d, tr.Wh2, tr.el2, tr.er2, tr.alpha2, "2", lambda r: _rows(tr.Y1, r), W2,
                   al2, ar2, Cp)
    a2 = tr.alpha2[d["dev_idxR"]].double().cpu().numpy()
    assert tr.shared2
    # Yc2[v, 4i+h] = (1/H) sum_e alpha2[e,h] Y1[u,i]  (shared-heads aggregation)
    Y1u = _rows(tr.Y1, uR)
    prod = a2[:, None, :] * Y1u[:, :, None] / H  # [e, i, h]
    n = prod.shape[0]
    yc = _seg(prod.reshape(n, K1 * H), lofsR)
    yca = _seg(np.abs(prod).reshape(n, K1 * H), lofsR)
    _close("Yc2", _rows(tr.Yc2, R), yc, yca)
    # Z = Yc2 W2v + b2  (the head mean folded into the transform)
    Ycd = _rows(tr.Yc2, R)
    W2v = W2.reshape(K1 * H, Cp)
    b2 = tr.b2.double().cpu().numpy()
    _close("Z", _rows(tr.Z, R), Ycd @ W2v + b2, np.abs(Ycd) @ np.abs(W2v) + np.abs(b2))
    assert not torch.any(tr.Z[:, C:] != 0)
    # loss over all V, dZ on R: float64 softmax of the device logits
    Zd = tr.Z[:, :C].double().cpu().numpy()
    loss, dz = oo.cross_entropy(Zd, d["y"])
    assert abs(tr.loss.item() - loss) <= RTOL * abs(loss), (tr.loss.item(), loss)
    del Zd
    dZd = _rows(tr.dZ, R)[:, :C]
    dzr = dz[R]
    assert np.all(np.abs(dZd - dzr) <= RTOL * np.maximum(np.abs(dzr), 1.0 / V)), "dZ"


def _layer_backward(d, label, alpha_R, pre_R, Wh, dY_rows, alpha_dev, Fh, snap_ds, snap_ds_U,
                    der, del_, dWh, a_l, a_r):
    """ds on R's edges, der on R, del on U, dWh on U.  dY_rows(idx) returns the
    per-head output gradient rows [n, H*Fh] the layer's aggregation receives
    (dZ/H broadcast to the heads for the mean layer)."""
    R, lofsR, uR, U, lofsU, vU = d["R"], d["lofsR"], d["uR"], d["U"], d["lofsU"], d["vU"]
    n = uR.size
    dal = np.zeros((n, H))
    dala = np.zeros((n, H))
    dYr = dY_rows(R)
    for e0 in range(0, n, CHUNK):
        e1 = min(n, e0 + CHUNK)
        Whu = _rows(Wh, uR[e0:e1]).reshape(e1 - e0, H, -1)[:, :, :Fh]
        rv = np.searchsorted(lofsR, np.arange(e0, e1), side="right") - 1
        dY = dYr[rv].reshape(e1 - e0, H, Fh)
        dal[e0:e1] = (dY * Whu).sum(-1)
        dala[e0:e1] = (np.abs(dY) * np.abs(Whu)).sum(-1)
    ds_ref, ds_abs = _ds(alpha_R, dal, dala, pre_R, lofsR)
    _close(f"ds{label}", snap_ds, ds_ref, ds_abs)
    # der[v] = row sum of ds (CSR order), del[u] = column sum (CSC, via edge ids)
    _close(f"der{label}", der[R], _seg(snap_ds, lofsR), _seg(np.abs(snap_ds), lofsR))
    _close(f"del{label}", del_[U], _seg(snap_ds_U, lofsU), _seg(np.abs(snap_ds_U), lofsU))
    # dWh[u] = sum_{e=(v,u)} alpha[e,h] dY[v,h,:] + del[u,h] a_l[h] + der[u,h] a_r[h]
    aU = alpha_dev[d["teid"]].double().cpu().numpy()
    dYv = dY_rows(vU).reshape(vU.size, H, Fh)
    prod = aU[:, :, None] * dYv
    g = _seg(prod.reshape(vU.size, H * Fh), lofsU).reshape(U.size, H, Fh)
    ga = _seg(np.abs(prod).reshape(vU.size, H * Fh), lofsU).reshape(U.size, H, Fh)
    g += del_[U][:, :, None] * a_l[None] + der[U][:, :, None] * a_r[None]
    ga += np.abs(del_[U])[:, :, None] * np.abs(a_l)[None] + np.abs(der[U])[:, :, None] * np.abs(a_r)[None]
    got = _rows(dWh, U).reshape(U.size, H, -1)
    _close(f"dWh{label}", got[:, :, :Fh], g, ga)
    assert not np.any(got[:, :, Fh:] != 0)


def test_products_gat_backward(epoch):
    d, tr, p, snap = epoch, epoch["tr"], epoch["p"], epoch["snap"]
    R, lofsR, uR = d["R"], d["lofsR"], d["uR"]
    Cp, K1 = tr.Cp, H * HID
    W2 = tr.W2.double().cpu().numpy()
    al2, ar2 = tr.al2.double().cpu().numpy(), tr.ar2.double().cpu().numpy()
    degR = np.diff(lofsR)
    # the f64 alpha of R's edges from the device scores (the forward test checks
    # the device's stored alpha against it)
    alpha2, pre2 = _softmax_rows(_rows(tr.el2, uR), np.repeat(_rows(tr.er2, R), degR, axis=0), lofsR)
    alpha1, pre1 = _softmax_rows(_rows(tr.el1, uR), np.repeat(_rows(tr.er1, R), degR, axis=0), lofsR)
    # db2 = column sum of dZ (all V)
    s = np.zeros(Cp)
    sa = np.zeros(Cp)
    for (dz,) in _stream(tr.dZ):
        s += dz.sum(0)
        sa += np.abs(dz).sum(0)
    _close("db2", tr.db2.double().cpu().numpy(), s, sa)
    # layer 2: the mean layer's aggregation receives dZ / H on every head
    mean_dY = lambda idx: np.tile(_rows(tr.dZ, idx) / H, (1, H))  # noqa: E731
    _layer_backward(d, "2", alpha2, pre2, tr.Wh2, mean_dY, tr.alpha2, Cp,
                    snap["ds_R"], snap["ds_U"], snap["der"], snap["del"], tr.dWh2,
                    al2, ar2)
    # da_l / da_r (all V), dW2 = Y1^T dWh2 (all V)
    dal = np.zeros((H, Cp))
    dar = np.zeros((H, Cp))
    dala = np.zeros((H, Cp))
    dara = np.zeros((H, Cp))
    dW = np.zeros((K1, H * Cp))
    dWa = np.zeros((K1, H * Cp))
    for r0, (wh, y1, dwh) in zip(range(0, V, CHUNK), _stream(tr.Wh2, tr.Y1, tr.dWh2)):
        dl, dr = snap["del"][r0:r0 + CHUNK], snap["der"][r0:r0 + CHUNK]
        whr = wh.reshape(-1, H, Cp)
        dal += (whr * dl[:, :, None]).sum(0)
        dar += (whr * dr[:, :, None]).sum(0)
        dala += (np.abs(whr) * np.abs(dl)[:, :, None]).sum(0)
        dara += (np.abs(whr) * np.abs(dr)[:, :, None]).sum(0)
        dW += y1.T @ dwh
        dWa += np.abs(y1).T @ np.abs(dwh)
    _close("dal2", tr.dal2.double().cpu().numpy(), dal, dala)
    _close("dar2", tr.dar2.double().cpu().numpy(), dar, dara)
    _close("dW2", tr.dW2.double().cpu().numpy(), dW, dWa)
    # dY1 = dWh2 W2^T on R; relu backward exact; db1 over all V
    dwhR = _rows(tr.dWh2, R)
    if tr.fr:  # the GEMM's epilogue applies the ReLU backward: dY1 itself is never stored
        mk = _rows(tr.Y1, R) > 0
        _close("dY1m", _rows(tr.dY1m, R), (dwhR @ W2.T) * mk, (np.abs(dwhR) @ np.abs(W2.T)) * mk)
    else:
        _close("dY1", _rows(tr.dY1, R), dwhR @ W2.T, np.abs(dwhR) @ np.abs(W2.T))
        m = _rows(tr.dY1m, R)
        assert np.array_equal(m, _rows(tr.dY1, R) * (_rows(tr.Y1, R) > 0)), "dY1m"
    s = np.zeros(K1)
    sa = np.zeros(K1)
    for (dy,) in _stream(tr.dY1m):
        s += dy.sum(0)
        sa += np.abs(dy).sum(0)
    _close("db1", tr.db1.double().cpu().numpy(), s, sa)
    # layer 1 (ds / der / del hold layer 1's values now)
    ds1_R = tr.ds[d["dev_idxR"]].double().cpu().numpy()
    ds1_U = tr.ds[d["teid"]].double().cpu().numpy()
    der1, del1 = tr.der.double().cpu().numpy(), tr.del_.double().cpu().numpy()
    _layer_backward(d, "1", alpha1, pre1, tr.Wh1, lambda idx: _rows(tr.dY1m, idx),
                    tr.alpha1, HID, ds1_R, ds1_U, der1, del1, tr.dWh1,
                    p["al1"], p["ar1"])
    dal = np.zeros((H, HID))
    dar = np.zeros((H, HID))
    dala = np.zeros((H, HID))
    dara = np.zeros((H, HID))
    dW = np.zeros((F, K1))
    dWa = np.zeros((F, K1))
    for r0, (wh, dwh) in zip(range(0, V, CHUNK), _stream(tr.Wh1, tr.dWh1)):
        dl, dr = del1[r0:r0 + CHUNK], der1[r0:r0 + CHUNK]
        whr = wh.reshape(-1, H, HID)
        dal += (whr * dl[:, :, None]).sum(0)
        dar += (whr * dr[:, :, None]).sum(0)
        dala += (np.abs(whr) * np.abs(dl)[:, :, None]).sum(0)
        dara += (np.abs(whr) * np.abs(dr)[:, :, None]).sum(0)
        x = d["X"][r0:r0 + CHUNK].astype(np.float64)
        dW += x.T @ dwh
        dWa += np.abs(x).T @ np.abs(dwh)
    _close("dal1", tr.dal1.double().cpu().numpy(), dal, dala)
    _close("dar1", tr.dar1.double().cpu().numpy(), dar, dara)
    _close("dW1", tr.dW1.double().cpu().numpy(), dW, dWa)
