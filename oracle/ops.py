"""float64 restatement of the GraphPy kernel semantics and GCN math (test
oracle only; PARITY UNPINNED — the reference has no implementation of these,
SURVEY.md §8c).  Semantics follow SURVEY.md Appendix A:

* A[v,u] = multiplicity of (v,u) in CSR row v (duplicates summed, A.1);
* deg(v) = offsets[v+1]-offsets[v]; degree-norm divides by deg(v), rows with
  deg 0 give 0 (A.2, A.3);
* SpMMv: Y = A X (no edge tensor); SpMMve: Y[v] =
  sum_e ev_e X[col_e] per head;
* SDDMM: out[e,h] = <X[row_e,h,:], Y[col_e,h,:]> (A.7);
* GCN: Z = norm_A(X W) + b, ReLU between layers, mean cross-entropy (A.4).
"""

from __future__ import annotations

import contextlib

import numpy as np

_CHUNK = 1 << 24  # gathered elements per block (bounds oracle memory)


def _row_blocks(offsets, K):
    R = offsets.size - 1
    per = max(1, _CHUNK // max(K, 1))
    r0 = 0
    while r0 < R:
        # grow the block until it holds ~per edges (at least one row)
        target = offsets[r0] + per
        r1 = int(np.searchsorted(offsets, target, side="right")) - 1
        r1 = min(max(r1, r0 + 1), R)
        yield r0, r1
        r0 = r1


_POOL = None  # oracle.parallel.ForkSpmmPool while inside parallel(pool)


@contextlib.contextmanager
def parallel(pool):
    """Run every eligible spmm() on ``pool`` (oracle.parallel.ForkSpmmPool):
    same per-row float64 sums, all host cores."""
    global _POOL
    prev, _POOL = _POOL, pool
    try:
        yield pool
    finally:
        _POOL = prev


def spmm(offsets, cols, X, vals=None, heads=1, norm=False, deg_offsets=None):
    """Y[v] = sum_{e in row v} w_e * X[cols_e] (w_e = vals[e, head] or 1)."""
    if _POOL is not None and vals is None and deg_offsets is None:
        name = _POOL.lookup(offsets, cols, X)
        if name is not None:
            return _POOL.spmm(name, X, norm=norm)
    return _spmm_serial(offsets, cols, X, vals, heads, norm, deg_offsets)


def _spmm_serial(offsets, cols, X, vals=None, heads=1, norm=False, deg_offsets=None):
    offsets = np.asarray(offsets, dtype=np.int64)
    X = np.asarray(X, dtype=np.float64)
    R = offsets.size - 1
    K = X.shape[1]
    F = K // heads
    Y = np.zeros((R, K), dtype=np.float64)
    for r0, r1 in _row_blocks(offsets, K):
        e0, e1 = int(offsets[r0]), int(offsets[r1])
        if e1 == e0:
            continue
        G = X[cols[e0:e1]]
        if vals is not None:
            w = np.asarray(vals[e0:e1], dtype=np.float64).reshape(e1 - e0, heads)
            G = (G.reshape(e1 - e0, heads, F) * w[:, :, None]).reshape(e1 - e0, K)
        starts = offsets[r0:r1] - e0
        nz = np.nonzero(offsets[r0 + 1:r1 + 1] > offsets[r0:r1])[0]
        Y[r0 + nz] = np.add.reduceat(G, starts[nz], axis=0)
    if norm:
        d = np.diff(offsets if deg_offsets is None else np.asarray(deg_offsets)).astype(np.float64)
        inv = np.divide(1.0, d, out=np.zeros_like(d), where=d > 0)
        Y *= inv[:, None]
    return Y


def degree_norm(offsets, X):
    d = np.diff(np.asarray(offsets)).astype(np.float64)
    inv = np.divide(1.0, d, out=np.zeros_like(d), where=d > 0)
    return np.asarray(X, dtype=np.float64) * inv[:, None]


def sddmm(offsets, cols, X, Y, heads=1):
    """out[e,h] = <X[row_e,h,:], Y[col_e,h,:]> in CSR edge order."""
    offsets = np.asarray(offsets, dtype=np.int64)
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    K = X.shape[1]
    F = K // heads
    E = int(offsets[-1])
    out = np.zeros((E, heads), dtype=np.float64)
    rows = np.repeat(np.arange(offsets.size - 1), np.diff(offsets))
    step = max(1, _CHUNK // max(K, 1))
    for e0 in range(0, E, step):
        e1 = min(E, e0 + step)
        p = X[rows[e0:e1]].reshape(-1, heads, F) * Y[cols[e0:e1]].reshape(-1, heads, F)
        out[e0:e1] = p.sum(axis=2)
    return out


def edge_softmax(offsets, s):
    """alpha_e = exp(s_e - max_row) / sum_row exp(...) per head, CSR rows."""
    offsets = np.asarray(offsets, dtype=np.int64)
    s = np.asarray(s, dtype=np.float64)
    s2 = s.reshape(s.shape[0], -1)
    out = np.zeros_like(s2)
    nz = np.nonzero(np.diff(offsets) > 0)[0]
    if nz.size == 0:
        return out.reshape(s.shape)
    starts = offsets[nz]
    deg = np.diff(offsets)[nz]
    mx = np.maximum.reduceat(s2, starts, axis=0)
    ex = np.exp(s2 - np.repeat(mx, deg, axis=0))
    sm = np.add.reduceat(ex, starts, axis=0)
    out[:] = ex / np.repeat(sm, deg, axis=0)
    return out.reshape(s.shape)


def edge_softmax_backward(offsets, alpha, dalpha):
    """dS = alpha * (dalpha - sum_row alpha * dalpha)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    a = np.asarray(alpha, dtype=np.float64).reshape(alpha.shape[0], -1)
    da = np.asarray(dalpha, dtype=np.float64).reshape(a.shape)
    nz = np.nonzero(np.diff(offsets) > 0)[0]
    out = np.zeros_like(a)
    if nz.size:
        starts = offsets[nz]
        deg = np.diff(offsets)[nz]
        dot = np.add.reduceat(a * da, starts, axis=0)
        out[:] = a * (da - np.repeat(dot, deg, axis=0))
    return out.reshape(np.shape(alpha))


def cross_entropy(logits, labels):
    """Mean softmax cross-entropy and its gradient w.r.t. the logits."""
    z = np.asarray(logits, dtype=np.float64)
    z = z - z.max(axis=1, keepdims=True)
    lse = np.log(np.exp(z).sum(axis=1))
    n = z.shape[0]
    loss = float(np.mean(lse - z[np.arange(n), labels]))
    p = np.exp(z - lse[:, None])
    p[np.arange(n), labels] -= 1.0
    return loss, p / n


def gcn2_step(offsets, cols, t_offsets, t_cols, X, W1, b1, W2, b2, labels, loss_rows=None):
    """2-layer GCN forward + backward (Appendix A.4): returns loss, logits and
    the parameter gradients, all float64.  ``loss_rows`` = B restricts the
    mean cross-entropy to the first B rows (the seed vertices of a sampled
    mini-batch subgraph, sampler.py:299-305: labels = the seed batch); the
    other rows get zero logit gradient."""
    X = np.asarray(X, dtype=np.float64)
    H1 = X @ W1
    P1 = spmm(offsets, cols, H1, norm=True)
    Z1 = P1 + b1
    Y1 = np.maximum(Z1, 0.0)
    H2 = Y1 @ W2
    Z2 = spmm(offsets, cols, H2, norm=True) + b2
    if loss_rows is None:
        loss, dZ2 = cross_entropy(Z2, labels)
    else:
        loss, dz = cross_entropy(Z2[:loss_rows], np.asarray(labels)[:loss_rows])
        dZ2 = np.zeros_like(Z2)
        dZ2[:loss_rows] = dz
    db2 = dZ2.sum(axis=0)
    dH2 = spmm(t_offsets, t_cols, degree_norm(offsets, dZ2))
    dW2 = Y1.T @ dH2
    dY1 = dH2 @ W2.T
    dZ1 = dY1 * (Z1 > 0)
    db1 = dZ1.sum(axis=0)
    dH1 = spmm(t_offsets, t_cols, degree_norm(offsets, dZ1))
    dW1 = X.T @ dH1
    # Appendix A.8 scale: the same contractions on absolute values (guards the
    # cancellation in bias sums and weight gradients)
    absd = {
        "W1": np.abs(X).T @ spmm(t_offsets, t_cols, degree_norm(offsets, np.abs(dZ1))),
        "b1": np.abs(dZ1).sum(axis=0),
        "W2": np.abs(Y1).T @ spmm(t_offsets, t_cols, degree_norm(offsets, np.abs(dZ2))),
        "b2": np.abs(dZ2).sum(axis=0),
    }
    return {"loss": loss, "logits": Z2, "W1": dW1, "b1": db1, "W2": dW2, "b2": db2, "abs": absd}


def close(gpu, ref, ref_abs=None, rtol=1e-5):
    """Appendix A.8 criterion: |gpu-ref| <= rtol * max(|ref|, ref_abs)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = np.abs(ref) if ref_abs is None else np.maximum(np.abs(ref), np.asarray(ref_abs))
    err = np.abs(gpu - ref)
    ok = err <= rtol * scale + 1e-30
    return bool(np.all(ok)), float(np.max(err / np.maximum(scale, 1e-30))) if err.size else 0.0


# ------------------------------------------------------------------- GAT
def leaky_relu(x, slope):
    return np.where(x > 0, x, slope * x)


def _rows_of(offsets):
    offsets = np.asarray(offsets, dtype=np.int64)
    return np.repeat(np.arange(offsets.size - 1), np.diff(offsets))


def gat_scores(offsets, cols, el, er, slope=0.2):
    """Appendix A.6: s_e,h = LeakyReLU(el[col_e,h] + er[row_e,h]) for NZE
    e = (row v, col u) — the degenerate (K=1) SDDMM of PAPER.md:281-283.
    Returns (s, pre)."""
    el = np.asarray(el, dtype=np.float64)
    er = np.asarray(er, dtype=np.float64)
    pre = el[np.asarray(cols)] + er[_rows_of(offsets)]
    return leaky_relu(pre, slope), pre


def attn_proj(Wh, a, heads):
    """el[v,h] = <Wh[v,h,:], a[h,:]> (a is [heads, F])."""
    V = Wh.shape[0]
    return (np.asarray(Wh, np.float64).reshape(V, heads, -1) * np.asarray(a, np.float64)[None]).sum(-1)


def gat_layer_fwd(offsets, cols, X, W, a_l, a_r, b, heads, mean=False, relu=False, slope=0.2):
    """One GAT layer (Appendix A.6; state tensor alpha saved):
    Wh = X W; el/er = attention projections; alpha = edge_softmax(scores);
    Y = SpMMve(A, alpha, Wh) per head; heads concatenated (+b, optional ReLU)
    or averaged (+b) in the last layer."""
    X = np.asarray(X, dtype=np.float64)
    Wh = X @ np.asarray(W, np.float64)
    V = Wh.shape[0]
    F = Wh.shape[1] // heads
    el, er = attn_proj(Wh, a_l, heads), attn_proj(Wh, a_r, heads)
    s, pre = gat_scores(offsets, cols, el, er, slope)
    alpha = edge_softmax(offsets, s)
    Yc = spmm(offsets, cols, Wh, vals=alpha, heads=heads)
    if mean:
        Z = Yc.reshape(V, heads, F).mean(axis=1) + b
    else:
        Z = Yc + b
    out = np.maximum(Z, 0.0) if relu else Z
    cache = dict(X=X, W=np.asarray(W, np.float64), Wh=Wh, el=el, er=er, pre=pre, alpha=alpha,
                 Z=Z, a_l=np.asarray(a_l, np.float64), a_r=np.asarray(a_r, np.float64),
                 heads=heads, mean=mean, relu=relu, slope=slope)
    return out, cache


def gat_layer_bwd(offsets, cols, c, dout, absmode=False):
    """Hand-derived backward of gat_layer_fwd.  SpMMve^T for dWh (PAPER.md:
    264-265), dalpha by the dot SDDMM, softmax backward, LeakyReLU backward,
    attention-projection backward, then the dense transform.  absmode=True
    runs the same contractions on absolute values with every subtraction
    turned into an addition: the Appendix A.8 ``ref_abs`` scale."""
    A = np.abs if absmode else (lambda t: t)
    offsets = np.asarray(offsets, dtype=np.int64)
    cols = np.asarray(cols)
    H, mean, slope = c["heads"], c["mean"], c["slope"]
    V = c["Wh"].shape[0]
    F = c["Wh"].shape[1] // H
    dZ = A(np.asarray(dout, np.float64))
    if c["relu"]:
        dZ = dZ * (c["Z"] > 0)
    db = dZ.sum(axis=0)
    dY = np.repeat(dZ[:, None, :] / H, H, axis=1).reshape(V, H * F) if mean else dZ
    Wh, alpha = A(c["Wh"]), c["alpha"]
    rows = _rows_of(offsets)
    # dWh (aggregation part) = A^T_alpha dY: scatter-add over the edge list
    dWh = np.zeros_like(Wh)
    contrib = dY[rows].reshape(-1, H, F) * alpha[:, :, None]
    np.add.at(dWh, cols, contrib.reshape(-1, H * F))
    dalpha = sddmm(offsets, cols, dY, Wh, heads=H)
    if absmode:
        srow = spmm(offsets, cols, np.ones((V, H)), vals=alpha * dalpha, heads=H)
        ds = alpha * (dalpha + srow[rows])
        ds = ds * np.where(c["pre"] > 0, 1.0, abs(slope))
    else:
        ds = edge_softmax_backward(offsets, alpha, dalpha) * np.where(c["pre"] > 0, 1.0, slope)
    der = spmm(offsets, cols, np.ones((V, H)), vals=ds, heads=H)
    dl = np.zeros((V, H))
    np.add.at(dl, cols, ds)
    a_l, a_r = A(c["a_l"]), A(c["a_r"])
    dWh = dWh + (dl[:, :, None] * a_l[None] + der[:, :, None] * a_r[None]).reshape(V, H * F)
    da_l = (Wh.reshape(V, H, F) * dl[:, :, None]).sum(axis=0)
    da_r = (Wh.reshape(V, H, F) * der[:, :, None]).sum(axis=0)
    dW = A(c["X"]).T @ dWh
    dX = dWh @ A(c["W"]).T
    return {"W": dW, "a_l": da_l, "a_r": da_r, "b": db, "X": dX, "Wh": dWh, "alpha": dalpha,
            "ds": ds, "el": dl, "er": der}


# ------------------------------------------------------------------- GIN
def gin_layer_fwd(offsets, cols, X, W1, b1, W2, b2, eps=0.0, relu_out=False,
                  transform_first=False):
    """Appendix A.5: Z = MLP((1+eps) X + A X), MLP = Linear -> ReLU -> Linear
    (SpMMv without norm, PAPER.md:2320-2321 class B).

    ``transform_first``: evaluate Hs W1 as (1+eps) (X W1) + A (X W1) — the same
    value in exact arithmetic (A is linear), float64 rounding apart — so a
    wide input (Reddit K=602) is aggregated at the hidden width; Hs itself is
    then never formed (the backward takes dW1 = X^T ((1+eps) dU + A^T dU))."""
    X = np.asarray(X, dtype=np.float64)
    if transform_first:
        XW = X @ W1
        Hs = None
        U = (1.0 + eps) * XW + spmm(offsets, cols, XW) + b1
    else:
        Hs = (1.0 + eps) * X + spmm(offsets, cols, X)
        U = Hs @ W1 + b1
    Ur = np.maximum(U, 0.0)
    Z = Ur @ W2 + b2
    out = np.maximum(Z, 0.0) if relu_out else Z
    return out, dict(X=X, Hs=Hs, U=U, Ur=Ur, Z=Z, W1=W1, W2=W2, eps=eps, relu_out=relu_out)


def gin2_forward(offsets, cols, X, p, eps=0.0, transform_first=False):
    """Forward caches (c1, c2) of gin2_step (each with its layer output "out")."""
    tf = transform_first
    h1, c1 = gin_layer_fwd(offsets, cols, X, p["W1a"], p["b1a"], p["W1b"], p["b1b"], eps,
                           relu_out=True, transform_first=tf)
    Z, c2 = gin_layer_fwd(offsets, cols, h1, p["W2a"], p["b2a"], p["W2b"], p["b2b"], eps,
                          transform_first=tf)
    c1["out"], c2["out"] = h1, Z
    return c1, c2


def gin2_forward_abs(offsets, cols, X, p, eps=0.0):
    """Appendix A.8 ref_abs scales of the three ReLU pre-activations of
    gin2_forward(transform_first=True): the same contractions on absolute
    values (|X| |W1a| aggregated, and so on through the layers)."""
    e = 1.0 + abs(eps)
    A = lambda k: np.abs(np.asarray(p[k], np.float64))  # noqa: E731
    XW = np.abs(np.asarray(X, np.float64)) @ A("W1a")
    U1 = e * XW + spmm(offsets, cols, XW) + A("b1a")
    Z1 = U1 @ A("W1b") + A("b1b")
    HW = Z1 @ A("W2a")
    U2 = e * HW + spmm(offsets, cols, HW) + A("b2a")
    return {"U1": U1, "Z1": Z1, "U2": U2}


def gin_layer_bwd(t_offsets, t_cols, c, dout, absmode=False, need_dx=True):
    A = np.abs if absmode else (lambda t: t)
    dZ = A(np.asarray(dout, np.float64))
    if c["relu_out"]:
        dZ = dZ * c.get("mask_Z", c["Z"] > 0)
    db2 = dZ.sum(axis=0)
    dW2 = A(c["Ur"]).T @ dZ
    dU = (dZ @ A(np.asarray(c["W2"], np.float64)).T) * c.get("mask_U", c["U"] > 0)
    db1 = dU.sum(axis=0)
    W1 = A(np.asarray(c["W1"], np.float64))
    eps = abs(c["eps"]) if absmode else c["eps"]
    if c["Hs"] is None:  # transform_first: Hs^T dU = X^T ((1+eps) dU + A^T dU)
        dXW = (1.0 + eps) * dU + spmm(t_offsets, t_cols, dU)
        dW1 = A(c["X"]).T @ dXW
        dX = dXW @ W1.T if need_dx else None
    else:
        dW1 = A(c["Hs"]).T @ dU
        dHs = dU @ W1.T
        dX = (1.0 + eps) * dHs + spmm(t_offsets, t_cols, dHs) if need_dx else None
    return {"W1": dW1, "b1": db1, "W2": dW2, "b2": db2, "X": dX}


def gat2_step(offsets, cols, X, p, labels, heads, slope=0.2):
    """2-layer GAT (hidden: heads concatenated + ReLU; output: heads
    averaged), mean cross-entropy, all gradients (+ Appendix A.8 scales)."""
    h1, c1 = gat_layer_fwd(offsets, cols, X, p["W1"], p["al1"], p["ar1"], p["b1"], heads,
                           relu=True, slope=slope)
    Z, c2 = gat_layer_fwd(offsets, cols, h1, p["W2"], p["al2"], p["ar2"], p["b2"], heads,
                          mean=True, slope=slope)
    loss, dZ = cross_entropy(Z, labels)
    g2 = gat_layer_bwd(offsets, cols, c2, dZ)
    g1 = gat_layer_bwd(offsets, cols, c1, g2["X"])
    a2 = gat_layer_bwd(offsets, cols, c2, dZ, absmode=True)
    a1 = gat_layer_bwd(offsets, cols, c1, a2["X"], absmode=True)
    names = {"W": "W", "a_l": "al", "a_r": "ar", "b": "b"}
    grads, absd = {}, {}
    for k, n in names.items():
        grads[n + "1"], grads[n + "2"] = g1[k], g2[k]
        absd[n + "1"], absd[n + "2"] = a1[k], a2[k]
    return {"loss": loss, "logits": Z, "alpha1": c1["alpha"], "alpha2": c2["alpha"], **grads,
            "abs": absd}


def gin2_step(offsets, cols, t_offsets, t_cols, X, p, labels, eps=0.0, transform_first=False,
              masks=None, forward=None, dlogits=None, fwd_abs=None):
    """2-layer GIN (ReLU between layers), mean cross-entropy, all gradients.
    ``transform_first`` applies each layer's first Linear before its
    aggregation (see gin_layer_fwd).  ``forward`` = (c1, c2) reuses caches of
    gin2_forward.  ``masks`` = {"U1", "Z1", "U2": bool [V, w]} sets the ReLU
    branch the backward takes for those pre-activations (the caller passes
    the device's branches for units whose pre-activation lies within the
    forward tolerance of zero, where either branch is a correct result).
    ``dlogits`` starts the backward from a given logit gradient (the
    device's, checked separately) instead of the oracle's own.
    ``fwd_abs`` = gin2_forward_abs(...) makes the A.8 scales of the weight
    gradients follow "the same op on |inputs|" through the forward too: the
    activations a weight gradient contracts (relu(U1), Y1, relu(U2)) enter
    the abs pass at their forward abs scale (masked by the taken ReLU branch)
    instead of at |activation|, so a forward value that is small only through
    cancellation carries its forward tolerance into the gradient's bound."""
    c1, c2 = forward if forward is not None else gin2_forward(
        offsets, cols, X, p, eps, transform_first)
    h1, Z = c1["out"], c2["out"]
    for name, (c, key) in {"U1": (c1, "mask_U"), "Z1": (c1, "mask_Z"),
                           "U2": (c2, "mask_U")}.items():
        c.pop(key, None)
        if masks and name in masks:
            c[key] = masks[name]
    loss, dZ = cross_entropy(Z, labels)
    if dlogits is not None:
        dZ = np.asarray(dlogits, dtype=np.float64)
    g2 = gin_layer_bwd(t_offsets, t_cols, c2, dZ)
    g1 = gin_layer_bwd(t_offsets, t_cols, c1, g2["X"], need_dx=False)
    ca1, ca2 = c1, c2
    if fwd_abs is not None:
        m = lambda c, key, v: c.get(key, v > 0)  # noqa: E731
        ca1 = dict(c1, Ur=fwd_abs["U1"] * m(c1, "mask_U", c1["U"]))
        ca2 = dict(c2, Ur=fwd_abs["U2"] * m(c2, "mask_U", c2["U"]),
                   X=fwd_abs["Z1"] * m(c1, "mask_Z", c1["Z"]))
        if ca2["Hs"] is not None:  # aggregate-first: Hs = (1+eps) X + A X on the abs scale
            e = 1.0 + abs(eps)
            ca2["Hs"] = e * ca2["X"] + spmm(offsets, cols, ca2["X"])
    a2 = gin_layer_bwd(t_offsets, t_cols, ca2, dZ, absmode=True)
    a1 = gin_layer_bwd(t_offsets, t_cols, ca1, a2["X"], absmode=True, need_dx=False)
    grads, absd = {}, {}
    for k, n in {"W1": "W{}a", "b1": "b{}a", "W2": "W{}b", "b2": "b{}b"}.items():
        grads[n.format(1)], grads[n.format(2)] = g1[k], g2[k]
        absd[n.format(1)], absd[n.format(2)] = a1[k], a2[k]
    return {"loss": loss, "logits": Z, **grads, "abs": absd}
