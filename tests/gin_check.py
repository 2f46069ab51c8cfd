"""Staged GIN parity check shared by the small-graph and full-size tests
(elementwise):

1. forward: every ReLU pre-activation (U1, Z1, U2) vs the float64 oracle at
   its forward abs scale; a unit may take the other ReLU branch only where the
   oracle's pre-activation lies within the forward tolerance of zero, and the
   oracle's backward then follows the device's branch for exactly those units;
2. logits (wide head, stored) vs the oracle; dZ vs the float64 softmax of the
   device's own logits; the backward starts from the device's dZ (a row whose
   top logits tie within their fp32 forward tolerance has an ill-determined
   dZ).  With the fused head (hidden <= 32, logits never stored) the oracle's
   own dZ is used;
3. all eight gradients vs the oracle, scales per gin2_step(fwd_abs=...)."""

import numpy as np

from oracle import ops as oo


def gin_staged_check(tr, off, tgt, t_off, t_rows, X, y, p, eps, rtol=1e-5):
    V, C = tr.V, tr.C
    fwd = oo.gin2_forward(off, tgt, X, p, eps=eps, transform_first=True)
    scale = oo.gin2_forward_abs(off, tgt, X, p, eps=eps)
    masks = {}
    for name, ref, dev in (("U1", fwd[0]["U"], tr.U1), ("Z1", fwd[0]["Z"], tr.Y1),
                           ("U2", fwd[1]["U"], tr.U2)):
        got = dev.cpu().numpy()
        ok, worst = oo.close(got, np.maximum(ref, 0.0), scale[name], rtol)
        assert ok, (name, worst)  # forward values
        m = got > 0
        flip = m != (ref > 0)
        assert np.all(np.abs(ref[flip]) <= rtol * scale[name][flip]), name
        assert flip.sum() <= max(1, 1e-5 * flip.size), (name, int(flip.sum()))
        masks[name] = m
    dZd = None
    if hasattr(tr, "Z2"):
        Zd = tr.Z2[:, :C].cpu().numpy().astype(np.float64)
        zabs = np.maximum(scale["U2"], 0) @ np.abs(p["W2b"]) + np.abs(p["b2b"])
        ok, worst = oo.close(Zd, fwd[1]["out"], zabs, rtol)
        assert ok, ("logits", worst)
        _, dz_ref = oo.cross_entropy(Zd, y)  # float64 softmax of the device logits
        dZd = tr.dZ2[:, :C].cpu().numpy()
        assert np.all(np.abs(dZd - dz_ref) <= rtol * np.maximum(np.abs(dz_ref), 1.0 / V)), "dZ"
    ref = oo.gin2_step(off, tgt, t_off, t_rows, X, p, y, eps=eps, transform_first=True,
                       forward=fwd, masks=masks, dlogits=dZd, fwd_abs=scale)
    assert abs(tr.loss.item() - ref["loss"]) <= rtol * abs(ref["loss"]), (tr.loss.item(),
                                                                          ref["loss"])
    grads = tr.grads()
    for k in p:
        ok, worst = oo.close(grads[k].detach().cpu().numpy(), ref[k], ref["abs"][k], rtol)
        assert ok, (k, worst)
