"""torch restatement of oracle/backward_ref.py — TEST INFRASTRUCTURE ONLY.

Same algorithm as ``backward_ref.moe_forward_backward`` (the analytic gradient of the
reference forward ``route`` -> ``apply_capacity`` -> ``combine_standard`` /
``combine_mem_efficient`` -> residual, plus ``aux_loss``; reference
``pkg/src/moelab/routing.py:71-262``), written with torch tensor ops so
it runs on any device in any dtype. Its purpose is the GPU parity tests at the BASELINE.json
shapes (Mixtral h=4096/m=14336/T=16384, Qwen3 E=128/K=8, DeepSeek E=256/h=7168), where
the numpy fp64 oracle would take CPU-hours: the tests run this module in fp32 on the GPU
(TF32 off) against the bf16 kernels.

Pinning: ``tests/test_torch_ref.py`` checks it in fp64 on the CPU against
``backward_ref`` (itself pinned by finite differences and the reference's own goldens) on
every variant: softmax / sigmoid, standard / mem-efficient, dropless / capacity+pad,
shared expert. Only ``tests/`` may import it; the product never does.

The decision is an input (``topk_idx`` [T, K], ascending expert ids, from the device
router whose selections the tests check bit-exactly against ``routing_ref.route`` first),
so the selection itself is not recomputed here; scores, drops, counts and every value are.
"""
from __future__ import annotations

import torch


def _scores(logits, score):
    """routing.py:85-91"""
    if score == "softmax":
        return torch.softmax(logits, dim=1)
    if score == "sigmoid":
        s = torch.sigmoid(logits)
        return s / s.sum(dim=1, keepdim=True)
    raise ValueError(f"unknown score function {score!r}")


def kept_mask(topk_idx, num_experts, capacity=None):
    """[T, K] bool: selection survives apply_capacity (routing.py:240-243: the first C
    selections of each expert by token index)."""
    if capacity is None or capacity < 0:
        return torch.ones_like(topk_idx, dtype=torch.bool)
    t, k = topk_idx.shape
    onehot = torch.zeros((t, num_experts), dtype=torch.int64, device=topk_idx.device)
    onehot.scatter_(1, topk_idx.long(), 1)
    rank = torch.cumsum(onehot, dim=0) - 1                      # rank within the expert column
    return torch.gather(rank, 1, topk_idx.long()) < capacity


def moe_forward_backward(x, w_r, gate, up, w2, dy, topk_idx, *, score="softmax", coeff=0.0,
                         variant="standard", capacity=None, shared=None, dtype=None,
                         want_grads=True):
    """Forward y and the gradients of L = <dy, y> + aux.

    x [T,h], w_r [h,E], gate/up [E,m,h] (or gate None: ungated), w2 [E,h,m], dy [T,h];
    topk_idx [T,K]; capacity: per-expert C or None; shared: (gate_s, up_s, w2_s) [m_s,h] /
    [h,m_s] computed on every token with weight 1 (latent_moe_forward's shared term,
    routing.py:276-278). Weights may be any dtype/device; they are cast per expert to
    `dtype` (default x.dtype). Returns dict y, aux, dx, dw_r, dgate, dup, dw2 (lists per
    expert, None for experts without rows), and the shared gradients.
    """
    dt = dtype or x.dtype
    dev = x.device
    xf = x.to(dt)
    dyf = dy.to(dt)
    wr = w_r.to(device=dev, dtype=dt)
    t, h = xf.shape
    n_exp = wr.shape[1]
    k = topk_idx.shape[1]
    idx = topk_idx.to(dev).long()
    logits = xf @ wr
    s = _scores(logits, score)
    keep = kept_mask(idx, n_exp, capacity)
    p_sel = torch.gather(s, 1, idx)                                # probs, not renormalised
    counts = torch.bincount(idx.reshape(-1), minlength=n_exp).to(dt)  # pre-drop counts
    f = counts / max(t * k, 1)
    aux = coeff * n_exp * float((f * s.mean(dim=0)).sum())

    # expert-major order, ascending token within an expert (permute, routing.py:155-163)
    flat_e = idx.reshape(-1)
    flat_keep = keep.reshape(-1)
    order = torch.argsort(flat_e * (t * k) + torch.arange(t * k, device=dev), stable=True)
    order = order[flat_keep[order]]
    tok_of = order // k
    sel_e = flat_e[order]
    bounds = torch.bincount(sel_e, minlength=n_exp).cumsum(0).tolist()

    y = torch.zeros((t, w2.shape[1]), dtype=dt, device=dev)
    dx = torch.zeros_like(xf)
    ds = torch.zeros((t, n_exp), dtype=dt, device=dev)
    dgate, dup, dw2 = [None] * n_exp, [None] * n_exp, [None] * n_exp
    gated = gate is not None
    start = 0
    for e in range(n_exp):
        stop = bounds[e]
        if stop <= start:
            start = stop
            continue
        sel = order[start:stop]
        tok = tok_of[start:stop]
        start = stop
        xs = xf[tok]
        w_up = up[e].to(device=dev, dtype=dt)
        w_dn = w2[e].to(device=dev, dtype=dt)
        z = xs @ w_up.T
        if gated:
            w_g = gate[e].to(device=dev, dtype=dt)
            g = xs @ w_g.T
            sg = torch.sigmoid(g)
            a = g * sg * z
        else:
            sz = torch.sigmoid(z)
            a = z * sz
        p = p_sel.reshape(-1)[sel][:, None]
        dys = dyf[tok]
        if variant == "standard":
            o = a @ w_dn.T
            y.index_add_(0, tok, o * p)
            if not want_grads:
                continue
            dp = (dys * o).sum(dim=1)
            do = p * dys
            da = do @ w_dn
            dw2[e] = do.T @ a
        elif variant == "mem_efficient":
            pa = a * p
            y.index_add_(0, tok, pa @ w_dn.T)
            if not want_grads:
                continue
            gpa = dys @ w_dn
            dp = (gpa * a).sum(dim=1)
            da = gpa * p
            dw2[e] = dys.T @ pa
        else:
            raise ValueError(f"unknown variant {variant!r}")
        if gated:
            dz = da * g * sg
            dgg = da * z * sg * (1.0 + g * (1.0 - sg))
            dgate[e] = dgg.T @ xs
            dxs = dz @ w_up + dgg @ w_g
        else:
            dz = da * sz * (1.0 + z * (1.0 - sz))
            dxs = dz @ w_up
        dup[e] = dz.T @ xs
        dx.index_add_(0, tok, dxs)
        ds[tok, e] += dp

    alive = keep.any(dim=1)
    if capacity is not None and capacity >= 0:
        y[~alive] += xf[~alive]
    out = {"y": y, "aux": aux, "kept": keep}
    sh = None
    if shared is not None:
        gs, us, w2s = (w.to(device=dev, dtype=dt) for w in shared)
        gsh = xf @ gs.T
        zsh = xf @ us.T
        ssh = torch.sigmoid(gsh)
        ash = gsh * ssh * zsh
        y += ash @ w2s.T
        if want_grads:
            dash = dyf @ w2s
            dzs = dash * gsh * ssh
            dgs = dash * zsh * ssh * (1.0 + gsh * (1.0 - ssh))
            dx += dzs @ us + dgs @ gs
            sh = {"dgate": dgs.T @ xf, "dup": dzs.T @ xf, "dw2": dyf.T @ ash}
    if not want_grads:
        return out

    # score gradient: combine term (kept selections) + aux term (pre-drop counts)
    ds += (coeff * n_exp * f / t)[None, :]
    inner = (ds * s).sum(dim=1, keepdim=True)
    if score == "softmax":
        dl = s * (ds - inner)
    else:
        sig = torch.sigmoid(logits)
        dl = sig * (1.0 - sig) / sig.sum(dim=1, keepdim=True) * (ds - inner)
    dw_r = xf.T @ dl
    dx += dl @ wr.T
    if capacity is not None and capacity >= 0:
        dx[~alive] += dyf[~alive]
    out.update(dx=dx, dw_r=dw_r, dgate=dgate, dup=dup, dw2=dw2, shared=sh, dlogits=dl)
    return out
