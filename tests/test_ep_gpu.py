"""EP layer on N GPUs (NCCL) vs the single-process GLOBAL oracle.

Each rank owns tokens [r*T, (r+1)*T) of one global batch and experts
[r*E/N, (r+1)*E/N). The oracle runs the whole layer on the global batch (decision taken
from the GPUs' own fp32 logits, i.e. parity at the logits boundary); every rank checks
its slice of y and dX, its experts' dW1/dW2, the all-reduced dW_r and the global aux.
Skipped unless >= 2 GPUs are visible (gpurun --gpus 2|4).
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = {
    "dropless_softmax": dict(E=8, K=2, h=256, m=256, T=256, score="softmax", cf=None, pad=False),
    "capacity_pad": dict(E=8, K=2, h=256, m=256, T=256, score="softmax", cf=1.0, pad=True,
                         skew=True),
    "sigmoid_many": dict(E=16, K=4, h=256, m=256, T=192, score="sigmoid", cf=None, pad=False),
    "mem_efficient": dict(E=8, K=2, h=256, m=256, T=128, score="softmax", cf=None, pad=False,
                          mem=True),
    "top8": dict(E=16, K=8, h=256, m=256, T=160, score="softmax", cf=None, pad=False),
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


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exit_worker(q):
    """Flush the result queue and leave without NCCL / symmetric-memory teardown: a
    teardown that blocks would keep the GPUs busy for the next test."""
    try:
        torch.cuda.synchronize()
    except Exception:  # pragma: no cover
        pass
    q.close()
    q.join_thread()
    os._exit(0)


def _join_all(procs):
    for p in procs:
        p.join(timeout=30)
    for p in procs:
        if p.is_alive():
            p.kill()
            p.join(timeout=10)


def _worker(rank, world, port, case, q, transport):
    try:
        import torch.distributed as dist

        from oracle import backward_ref as B
        from oracle import routing_ref as R
        from paper_2603_07685_b200 import gemm, ops
        from paper_2603_07685_b200.dispatcher import EPGroup, moe_forward_ep
        from paper_2603_07685_b200.layer import MoEConfig

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
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
        ep = EPGroup()
        echo = case.get("echo", 0)
        sf = transport in ("p2p_sync_free", "p2p_graph")
        tr = "p2p" if sf else transport
        leaves = (x, w_rd, w1d, w2d)
        dyd = dy_g[sl].to(dev)
        if transport == "p2p_graph":
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
        else:
            y, aux = moe_forward_ep(x, w_rd, w1d, w2d, cfg, ep, transport=tr, echo_slots=echo,
                                    sync_free=sf)
            # a second step exercises buffer reuse across steps (symmetric pools, barriers)
            for p_ in leaves:
                p_.grad = None
            y, aux = moe_forward_ep(x, w_rd, w1d, w2d, cfg, ep, transport=tr, echo_slots=echo,
                                    sync_free=sf)
            if echo:
                from paper_2603_07685_b200.dispatcher import last_echo
                if not last_echo.get("clones"):
                    raise AssertionError(f"ECHO made no clones: {last_echo}")
            torch.autograd.backward([y, aux], [dyd, torch.ones_like(aux)])
        from paper_2603_07685_b200.dispatcher import check_ep_status
        check_ep_status()  # no overlapped GEMM timed out waiting for a source rank
        dwr = w_rd.grad.float().clone()
        dist.all_reduce(dwr)
        # global decision from the GPUs' own logits
        r = ops.router_forward(x.detach(), w_rd.detach(), K, cfg.score)
        lg = r.logits[:T, :E].contiguous()
        lg_all = torch.empty((world * T, E), dtype=torch.float32, device=dev)
        dist.all_gather_into_tensor(lg_all, lg)
        torch.cuda.synchronize()

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
            "dx": rel(f64(x.grad), ref["dx"][sl]),
            "dwr": rel(f64(dwr), ref["dw_r"]),
        }
        dg, du = gemm.split_gate_up(w1d.grad)
        for j in range(el):
            e = rank * el + j
            if dec.effective_counts()[e] == 0:
                continue
            errs[f"dgate{e}"] = rel(f64(dg[j]), ref["dgate"][e])
            errs[f"dup{e}"] = rel(f64(du[j]), ref["dw1"][e])
            errs[f"dw2_{e}"] = rel(f64(w2d.grad[j]), ref["dw2"][e])
        aux_err = abs(float(aux.detach()) - ref["aux"]) / max(abs(ref["aux"]), 1e-9)
        y_tol, g_tol = case.get("y_tol", 1e-2), case.get("g_tol", 2e-2)
        bad = {k: v for k, v in errs.items() if v > (y_tol if k == "y" else g_tol)}
        if aux_err > 1e-4:
            bad["aux"] = aux_err
        q.put((rank, "ok" if not bad else f"errors {bad}"))
    except Exception as exc:  # pragma: no cover
        import traceback

        q.put((rank, traceback.format_exc() + repr(exc)))
    _exit_worker(q)


@pytest.mark.parametrize("transport", ["p2p", "p2p_sync_free", "p2p_graph", "p2p_overlap",
                                       "p2p_pull", "p2p_dedup", "nccl"])
@pytest.mark.parametrize("name", list(CASES))
def test_ep_layer_matches_global_oracle(name, transport):
    _run(CASES[name], transport)


@pytest.mark.parametrize("transport", ["p2p", "p2p_sync_free", "p2p_pull"])
@pytest.mark.parametrize("name", list(MX_CASES))
def test_ep_mxfp8_matches_global_oracle(name, transport):
    _run(MX_CASES[name], transport)


@pytest.mark.parametrize("name", list(ECHO_CASES))
def test_ep_echo_matches_global_oracle(name):
    _run(ECHO_CASES[name], "p2p")


def _run(case, transport):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    # validated at 2 and 4 ranks; MOE_TEST_MAX_WORLD=8 runs the whole EP group of a box
    world = min(torch.cuda.device_count(), int(os.environ.get("MOE_TEST_MAX_WORLD", "4")))
    while case["E"] % world:
        world -= 1
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, transport))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=int(os.environ.get("MOE_TEST_TIMEOUT", "300")))
               for _ in range(world)]
    finally:
        _join_all(procs)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"


def _stash_worker(rank, world, port, q):
    """Two stacked EP layers (sync-free p2p): Paged Stashing with one shared tmp buffer set
    must give bit-identical outputs and gradients to per-layer buffers."""
    try:
        import torch.distributed as dist

        from paper_2603_07685_b200.dispatcher import EPGroup, check_ep_status, moe_forward_ep
        from paper_2603_07685_b200.layer import MoEConfig
        from paper_2603_07685_b200.stash import PagedStashBuffer

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        E, K, h, m, T = 8, 2, 256, 256, 256
        cfg = MoEConfig(E, K, h, m, score="softmax", aux_loss_coeff=1e-2)
        g = torch.Generator().manual_seed(5 + rank)
        bf = torch.bfloat16
        el = E // world
        layers = []
        for li in range(2):
            gw = torch.Generator().manual_seed(100 + li)
            w_r = (torch.randn((h, E), generator=gw) * h ** -0.5).to(bf).to(dev)
            w1 = (torch.randn((el, 2 * m, h), generator=g) * h ** -0.5).to(bf).to(dev)
            w2 = (torch.randn((el, h, m), generator=g) * m ** -0.5).to(bf).to(dev)
            layers.append([w_r.requires_grad_(), w1.requires_grad_(), w2.requires_grad_()])
        x0 = torch.randn((T, h), generator=g).to(bf).to(dev)
        dy = torch.randn((T, h), generator=g).to(bf).to(dev)
        ep = EPGroup()
        rows_w = {"xp": h * 2, "preact": 4 * m, "act": 2 * m, "o": h * 2}

        def run(stash, overlap=False):
            for ws in layers:
                for w in ws:
                    w.grad = None
            x = x0.clone().requires_grad_(True)
            y = x
            auxes = []
            for li, (w_r, w1, w2) in enumerate(layers):
                if stash is None:
                    tag = f"layer{li}"
                else:  # overlapped stashing double-buffers the tmp set (two tags)
                    tag = f"ov{li % 2}" if overlap else "shared"
                y, aux = moe_forward_ep(y, w_r, w1, w2, cfg, ep, transport="p2p", sync_free=True,
                                        tag=tag, stash=stash, layer_id=li,
                                        stash_overlap=overlap)
                auxes.append(aux)
            torch.autograd.backward([y] + auxes, [dy] + [torch.ones_like(a) for a in auxes])
            torch.cuda.synchronize()
            return [y.detach().clone(), x.grad.clone()] + [w.grad.clone() for ws in layers
                                                          for w in ws]

        ref = run(None)
        buf = PagedStashBuffer(256, rows_w, page_rows=64, device=dev)
        got = run(buf)
        got_ov = run(buf, overlap=True)
        buf.check()
        check_ep_status()
        st = buf.stats()
        bad = [i for i, (a, b) in enumerate(zip(ref, got)) if not torch.equal(a, b)]
        bad += [f"overlap {i}" for i, (a, b) in enumerate(zip(ref, got_ov))
                if not torch.equal(a, b)]
        if st["free_pages"] != 256 or st["peak_pages_used"] == 0:
            bad.append(f"pages {st}")
        q.put((rank, "ok" if not bad else f"mismatch {bad}"))
    except Exception as exc:  # pragma: no cover
        import traceback

        q.put((rank, traceback.format_exc() + repr(exc)))
    _exit_worker(q)


def test_ep_paged_stash_two_layers():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_stash_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=int(os.environ.get("MOE_TEST_TIMEOUT", "300")))
               for _ in range(world)]
    finally:
        _join_all(procs)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"
