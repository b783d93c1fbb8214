"""Shared EP parity body: one rank's check of the EP layer against the
single-process GLOBAL oracle. Used by tests/test_ep_gpu.py (one process per GPU, NCCL) and
tests/test_ep_loopback_gpu.py (n ranks as threads on one GPU, paper_2603_07685_b200.loopback).

Rank r owns tokens [r*T, (r+1)*T) of one global batch and experts [r*E/n, (r+1)*E/n). The
oracle runs the whole layer on the global batch (decision taken from the GPUs' own fp32
logits, i.e. parity at the logits boundary); every rank checks its slice of y and dX, its
experts' dW1/dW2, the all-reduced dW_r and the global aux.
"""
import numpy as np
import torch

CASES = {
    "dropless_softmax": dict(E=8, K=2, h=256, m=256, T=256, score="softmax", cf=None, pad=False),
    "capacity_pad": dict(E=8, K=2, h=256, m=256, T=256, score="softmax", cf=1.0, pad=True,
                         skew=True),
    "sigmoid_many": dict(E=16, K=4, h=256, m=256, T=192, score="sigmoid", cf=None, pad=False),
    "mem_efficient": dict(E=8, K=2, h=256, m=256, T=128, score="softmax", cf=None, pad=False,
                          mem=True),
    "top8": dict(E=16, K=8, h=256, m=256, T=160, score="softmax", cf=None, pad=False),
}
# the 256-row CTA-pair plan (ops.pick_align(n*T, K, E) == 256 at n = 4) under EP
PAIR_CASES = {
    "pair_engine": dict(E=8, K=2, h=256, m=256, T=2048, score="softmax", cf=None, pad=False),
    "pair_capacity": dict(E=8, K=2, h=256, m=512, T=2048, score="softmax", cf=1.0, pad=True,
                          skew=True),
}
# MXFP8 expert GEMMs under EP (tolerance of the recipe: tests/test_layer_gpu.py)
MX_CASES = {
    "mxfp8": dict(E=8, K=2, h=256, m=256, T=256, score="softmax", cf=None, pad=False,
                  precision="mxfp8", y_tol=0.1, g_tol=0.12),
}
# ECHO hot-expert cloning (dropless, a strongly preferred expert): the cloned computation
# must equal the un-cloned global oracle exactly as any other EP run.
ECHO_CASES = {
    "echo_hot_expert": dict(E=8, K=2, h=256, m=256, T=256, score="softmax", cf=None, pad=False,
                            hot=0.4, echo=2),
    "echo_hot_top4": dict(E=16, K=4, h=256, m=256, T=192, score="sigmoid", cf=None, pad=False,
                          hot=0.4, echo=1),
}


def rank_check(ep, case, transport, dev, direct=False):
    """Run the EP layer fwd+bwd on this rank and compare with the global oracle; returns
    "ok" or a description of the errors. direct=True calls the transport's Function
    directly (loopback ranks share autograd's device thread)."""
    from oracle import backward_ref as B
    from oracle import routing_ref as R
    from paper_2603_07685_b200 import gemm, ops
    from paper_2603_07685_b200.dispatcher import check_ep_status, last_echo, moe_forward_ep
    from paper_2603_07685_b200.layer import MoEConfig

    rank, world = ep.rank, ep.n
    E, K, h, m, T = case["E"], case["K"], case["h"], case["m"], case["T"]
    cfg = MoEConfig(E, K, h, m, score=case["score"], aux_loss_coeff=1e-2,
                    capacity_factor=case["cf"], pad_to_capacity=case["pad"],
                    mem_efficient=case.get("mem", False),
                    precision=case.get("precision", "bf16"))
    g = torch.Generator().manual_seed(11)
    bf = torch.bfloat16
    x_g = torch.randn((world * T, h), generator=g).to(bf)
    w_r = (torch.randn((h, E), generator=g) * h ** -0.5)
    if case.get("skew"):
        # push routing towards low expert ids (capacity drops on the global batch)
        x_g = (x_g.float() + torch.linspace(1.0, 0.0, h)[None, :] * 0.5).to(bf)
        w_r[:, 0] += 0.05
    if case.get("hot"):
        # one hot expert: a constant feature whose router weight favours expert 0
        x_g[:, 0] = 1.0
        w_r[0, 0] += case["hot"] * h ** 0.5
    w_r = w_r.to(bf)
    up = (torch.randn((E, m, h), generator=g) * h ** -0.5).to(bf)
    gate = (torch.randn((E, m, h), generator=g) * h ** -0.5).to(bf)
    w2 = (torch.randn((E, h, m), generator=g) * m ** -0.5).to(bf)
    dy_g = torch.randn((world * T, h), generator=g).to(bf)
    el = E // world
    mine = slice(rank * el, (rank + 1) * el)
    sl = slice(rank * T, (rank + 1) * T)

    x = x_g[sl].to(dev).requires_grad_(True)
    w_rd = w_r.to(dev).requires_grad_(True)
    w1d = gemm.interleave_gate_up(gate[mine].to(dev), up[mine].to(dev)).requires_grad_(True)
    w2d = w2[mine].to(dev).contiguous().requires_grad_(True)
    echo = case.get("echo", 0)
    sf = transport in ("p2p_sync_free", "p2p_graph")
    tr = "p2p" if sf else transport
    leaves = (x, w_rd, w1d, w2d)
    dyd = dy_g[sl].to(dev)
    if direct:
        from paper_2603_07685_b200.loopback import forward_backward

        y, aux, grads = forward_backward(x.detach(), w_rd.detach(), w1d.detach(), w2d.detach(),
                                         cfg, ep, dyd, steps=2, transport=tr, echo_slots=echo,
                                         sync_free=sf)
        gx, gwr, gw1, gw2 = grads[:4]
    elif transport == "p2p_graph":
        # the whole sync-free fwd+bwd step captured in one CUDA graph, replayed twice
        def stepf():
            y_, aux_ = moe_forward_ep(x, w_rd, w1d, w2d, cfg, ep, transport="p2p",
                                      sync_free=True)
            torch.autograd.backward([y_, aux_], [dyd, torch.ones_like(aux_)])
            return y_, aux_

        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                for p_ in leaves:
                    p_.grad = None
                stepf()
        torch.cuda.current_stream().wait_stream(side)
        for p_ in leaves:
            p_.grad = None
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            y, aux = stepf()
        graph.replay()
        graph.replay()
        gx, gwr, gw1, gw2 = x.grad, w_rd.grad, w1d.grad, w2d.grad
    else:
        y, aux = moe_forward_ep(x, w_rd, w1d, w2d, cfg, ep, transport=tr, echo_slots=echo,
                                sync_free=sf)
        # a second step exercises buffer reuse across steps (symmetric pools, barriers)
        for p_ in leaves:
            p_.grad = None
        y, aux = moe_forward_ep(x, w_rd, w1d, w2d, cfg, ep, transport=tr, echo_slots=echo,
                                sync_free=sf)
        torch.autograd.backward([y, aux], [dyd, torch.ones_like(aux)])
        gx, gwr, gw1, gw2 = x.grad, w_rd.grad, w1d.grad, w2d.grad
    if echo and not last_echo.get("clones"):
        raise AssertionError(f"ECHO made no clones: {last_echo}")
    check_ep_status()  # no overlapped GEMM timed out waiting for a source rank
    dwr = gwr.float().clone()
    ep.all_reduce(dwr)
    # global decision from the GPUs' own logits
    r = ops.router_forward(x.detach(), w_rd.detach(), K, cfg.score)
    lg = r.logits[:T, :E].contiguous()
    lg_all = torch.empty((world * T, E), dtype=torch.float32, device=dev)
    ep.all_gather_into_tensor(lg_all, lg)
    torch.cuda.current_stream().synchronize()

    f64 = lambda t: t.detach().double().cpu().numpy()  # noqa: E731
    dec = R.route(f64(lg_all), np.eye(E), score=cfg.score, top_k=K)
    if cfg.capacity_factor is not None:
        dec = R.apply_capacity(dec, cfg.capacity_factor, pad=cfg.pad_to_capacity)
    params = R.ExpertParams(w1=list(f64(up)), w2=list(f64(w2)), gate=list(f64(gate)))
    ref = B.moe_forward_backward(f64(x_g), f64(w_r), params, f64(dy_g), score=cfg.score,
                                 top_k=K, coeff=1e-2, decision=dec,
                                 variant="mem_efficient" if cfg.mem_efficient else "standard")

    def rel(a, b):
        return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))

    errs = {
        "y": rel(f64(y), ref["y"][sl]),
        "dx": rel(f64(gx), ref["dx"][sl]),
        "dwr": rel(f64(dwr), ref["dw_r"]),
    }
    dg, du = gemm.split_gate_up(gw1)
    for j in range(el):
        e = rank * el + j
        if dec.effective_counts()[e] == 0:
            continue
        errs[f"dgate{e}"] = rel(f64(dg[j]), ref["dgate"][e])
        errs[f"dup{e}"] = rel(f64(du[j]), ref["dw1"][e])
        errs[f"dw2_{e}"] = rel(f64(gw2[j]), ref["dw2"][e])
    aux_err = abs(float(aux.detach()) - ref["aux"]) / max(abs(ref["aux"]), 1e-9)
    y_tol, g_tol = case.get("y_tol", 1e-2), case.get("g_tol", 2e-2)
    bad = {k: v for k, v in errs.items() if v > (y_tol if k == "y" else g_tol)}
    if aux_err > 1e-4:
        bad["aux"] = aux_err
    return "ok" if not bad else f"errors {bad}"
