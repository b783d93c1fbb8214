"""CPU restatement of the MoE-layer BACKWARD — TEST INFRASTRUCTURE ONLY.

The reference has no backward for the expert FFN, permute or combine (SURVEY
§8(c)): the only gradient it ships is ``aux_loss_grad_wr`` (reference
``pkg/src/moelab/routing.py:123-137``). This module restates the analytic
gradient of the reference FORWARD (``route`` :71-108 -> ``apply_capacity``
:226-247 -> ``combine_standard`` :189-201 / ``combine_mem_efficient`` :204-223
-> residual :254-262, plus ``aux_loss`` :111-120) with the scalar loss

    L = <dY, y> + aux_loss(decision, coeff)

following SURVEY Appendix C. Selection (top-k set, drops, token fractions f) is
piecewise constant and therefore a constant of the backward.

Pinning: ``tests/test_oracle.py`` checks this against central finite
differences of the oracle forward (``oracle/routing_ref.py``, itself pinned to
the reference's golden vectors), and its W_r aux part against the reference's
``aux_loss_grad_wr``. The module is dtype-generic: fp64 for parity, fp32 for
the CPU baseline timed by ``bench.py``.
"""
from __future__ import annotations

import numpy as np

from . import routing_ref as R


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def moe_forward_backward(x, w_r, params: R.ExpertParams, dy, *, score="softmax", top_k=1,
                         coeff=0.0, variant="standard", capacity=None, selection_bias=None,
                         decision=None, want_grads=True):
    """Forward y and all gradients of L = <dy, y> + aux.

    capacity: None (dropless) or (capacity_factor, pad). variant: "standard" |
    "mem_efficient". Returns a dict with y, aux, decision and (if want_grads)
    dx, dw_r, dw1, dw2, dgate (lists per expert, same layout as params).
    """
    if decision is None:
        decision = R.route(x, w_r, score=score, top_k=top_k, selection_bias=selection_bias)
        if capacity is not None:
            decision = R.apply_capacity(decision, capacity[0], pad=capacity[1])
    d = decision
    t, h = x.shape
    n_exp = d.num_experts
    gated = params.gate is not None
    permuted, rmap = R.permute(x, d)
    prow = R._row_probs(d, rmap)
    dt = x.dtype

    y = np.zeros((t, params.w2[0].shape[0]), dtype=dt)
    dx = np.zeros_like(x)
    dw1 = [np.zeros_like(w) for w in params.w1]
    dw2 = [np.zeros_like(w) for w in params.w2]
    dg_w = [np.zeros_like(w) for w in params.gate] if gated else None
    ds = np.zeros((t, n_exp), dtype=dt)

    for e, sl in R.expert_slices(d):
        if sl.stop <= sl.start:
            continue
        xs = permuted[sl]
        src = rmap[sl]
        real = src >= 0
        p = np.where(real, prow[sl], 0.0).astype(dt)
        w1, w2 = params.w1[e], params.w2[e]
        z = xs @ w1.T
        if gated:
            g = xs @ params.gate[e].T
            sg = _sigmoid(g)
            a = g * sg * z
        else:
            sz = _sigmoid(z)
            a = z * sz
        dys = np.zeros((xs.shape[0], y.shape[1]), dtype=dt)
        dys[real] = dy[src[real]]
        if variant == "standard":
            o = a @ w2.T
            np.add.at(y, src[real], (o * p[:, None])[real])
            if not want_grads:
                continue
            dp = (dys * o).sum(axis=1)
            do = p[:, None] * dys
            da = do @ w2
            dw2[e] += do.T @ a
        elif variant == "mem_efficient":
            pa = np.where(real[:, None], a * p[:, None], a)
            o = pa @ w2.T
            np.add.at(y, src[real], o[real])
            if not want_grads:
                continue
            gpa = dys @ w2
            dp = (gpa * a).sum(axis=1)
            da = np.where(real[:, None], gpa * p[:, None], gpa)
            dw2[e] += dys.T @ pa
        else:
            raise ValueError(f"unknown variant {variant!r}")
        if gated:
            dz = da * g * sg
            dgg = da * z * sg * (1.0 + g * (1.0 - sg))
            dg_w[e] += dgg.T @ xs
            dxs = dz @ w1 + dgg @ params.gate[e]
        else:
            dz = da * sz * (1.0 + z * (1.0 - sz))
            dxs = dz @ w1
        dw1[e] += dz.T @ xs
        np.add.at(dx, src[real], dxs[real])
        ds[src[real], e] += dp[real]

    aux = R.aux_loss(d, coeff)
    alive = None
    if d.dropped is not None:
        alive = (d.routing_map & ~d.dropped).any(axis=1)
        y[~alive] += x[~alive]
    out = {"y": y, "aux": aux, "decision": d}
    if not want_grads:
        return out

    # score gradient: combine term (kept selections) + aux term (all rows)
    f = d.counts / max(int(d.routing_map.sum()), 1)
    ds += (coeff * n_exp * f / t)[None, :].astype(dt)
    logits = x @ w_r
    s = d.scores
    inner = (ds * s).sum(axis=1, keepdims=True)
    if score == "softmax":
        dl = s * (ds - inner)
    elif score == "sigmoid":
        sig = _sigmoid(logits)
        dl = sig * (1.0 - sig) / sig.sum(axis=1, keepdims=True) * (ds - inner)
    else:
        raise ValueError(f"unknown score function {score!r}")
    dw_r = x.T @ dl
    dx += dl @ w_r.T
    if alive is not None:
        dx[~alive] += dy[~alive]
    out.update(dx=dx, dw_r=dw_r, dw1=dw1, dw2=dw2, dgate=dg_w, dlogits=dl, ds=ds)
    return out


def loss(x, w_r, params, dy, **kw):
    """Scalar L = <dy, y> + aux used by the finite-difference pin."""
    r = moe_forward_backward(x, w_r, params, dy, want_grads=False, **kw)
    return float((dy * r["y"]).sum() + r["aux"])
