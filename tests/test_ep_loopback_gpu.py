"""The EP data plane on ONE GPU: 4 simulated EP ranks (paper_2603_07685_b200.loopback,
threads with their own streams) run the unchanged dispatcher and exchange kernels, and
every rank is checked against the single-process GLOBAL oracle (tests/ep_cases.py, the
same body as the multi-GPU tests/test_ep_gpu.py).

What runs here, per transport:
  * p2p / p2p_sync_free: moe_ep_dispatch_push into the peers' padded plans (or the device
    planner moe_ep_plan_device), the fc2-forward / fc1-dgrad row-scatter epilogues
    (moe_gg_fc2_fwd_scatter, moe_gg_fc1_dgrad_scatter: TMA bulk stores to peer addresses),
    moe_ep_row_dst, moe_ep_combine_bwd_push, the local combines;
  * p2p_pull: moe_ep_combine_pull (forward and dX), the dprob pull;
  * p2p_dedup: moe_ep_token_ranks, moe_ep_dispatch_dedup, moe_ep_fill_pad_map,
    moe_ep_expand_grad, the per-token pre-reduction and its pull;
  * nccl: permute -> all_to_all_single -> moe_ep_regroup_map / gather and back;
  * ECHO (p2p): moe_ep_echo_rewrite + clone weights pulled from the home rank + the clone
    weight-gradient reduction;
  * MXFP8 under EP: moe_ep_scatter_rows;
  * Paged Stashing on two stacked layers (bit-identical to per-layer buffers).
The peer buffers are the other ranks' allocations on the same device, so the kernels store
through the same generic addresses as over NVLink; p2p_overlap (a GEMM spin-waiting on
another rank's push kernel) and graph capture need real peers (tests/test_ep_gpu.py).
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

from ep_cases import CASES, ECHO_CASES, MX_CASES, PAIR_CASES, rank_check  # noqa: E402

N = 4


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch.device("cuda:0")


def _run(case, transport, dev, n=N):
    from paper_2603_07685_b200.loopback import run_ranks

    res = run_ranks(n, lambda ep: rank_check(ep, case, transport, dev, direct=True), dev)
    assert all(r == "ok" for r in res), res


ALL = {**CASES, **PAIR_CASES}


@pytest.mark.parametrize("transport", ["p2p", "p2p_sync_free", "p2p_pull", "p2p_dedup", "nccl"])
@pytest.mark.parametrize("name", list(ALL))
def test_loopback_ep_matches_global_oracle(name, transport, dev):
    _run(ALL[name], transport, dev)


def test_loopback_ep_two_ranks(dev):
    _run(CASES["capacity_pad"], "p2p", dev, n=2)


@pytest.mark.parametrize("transport", ["p2p", "p2p_sync_free", "p2p_pull"])
def test_loopback_ep_mxfp8(transport, dev):
    _run(MX_CASES["mxfp8"], transport, dev)


@pytest.mark.parametrize("name", list(ECHO_CASES))
def test_loopback_ep_echo(name, dev):
    _run(ECHO_CASES[name], "p2p", dev)


def test_loopback_paged_stash_two_layers(dev):
    """Two stacked EP layers (sync-free p2p): Paged Stashing with one shared tmp buffer set
    gives bit-identical outputs and gradients to per-layer buffers."""
    from paper_2603_07685_b200 import dispatcher as D
    from paper_2603_07685_b200.layer import MoEConfig
    from paper_2603_07685_b200.loopback import _Ctx, run_ranks
    from paper_2603_07685_b200.stash import PagedStashBuffer

    E, K, h, m, T = 8, 2, 256, 256, 256
    cfg = MoEConfig(E, K, h, m, score="softmax", aux_loss_coeff=1e-2)

    def body(ep):
        rank, world = ep.rank, ep.n
        g = torch.Generator().manual_seed(5 + rank)
        bf = torch.bfloat16
        el = E // world
        layers = []
        for li in range(2):
            gw = torch.Generator().manual_seed(100 + li)
            w_r = (torch.randn((h, E), generator=gw) * h ** -0.5).to(bf).to(dev)
            w1 = (torch.randn((el, 2 * m, h), generator=g) * h ** -0.5).to(bf).to(dev)
            w2 = (torch.randn((el, h, m), generator=g) * m ** -0.5).to(bf).to(dev)
            layers.append((w_r, w1, w2))
        x0 = torch.randn((T, h), generator=g).to(bf).to(dev)
        dy = torch.randn((T, h), generator=g).to(bf).to(dev)

        def run(stash):
            ctxs, y = [], x0
            with torch.no_grad():
                for li, (w_r, w1, w2) in enumerate(layers):
                    fn, args = D.ep_function(y, w_r, w1, w2, cfg, ep, transport="p2p",
                                             sync_free=True,
                                             tag=f"layer{li}" if stash is None else "shared",
                                             stash=stash, layer_id=li)
                    ctx = _Ctx()
                    y, aux = fn.forward(ctx, *args)
                    ctxs.append((fn, ctx, aux))
                out = [y.clone()]
                d = dy
                for fn, ctx, aux in reversed(ctxs):
                    gr = fn.backward(ctx, d, torch.ones_like(aux))
                    d = gr[0]
                    out += [gr[1].clone(), gr[2].clone(), gr[3].clone()]
                out.append(d.clone())
            torch.cuda.current_stream().synchronize()
            return out

        ref = run(None)
        buf = PagedStashBuffer(256, {"xp": h * 2, "preact": 4 * m, "act": 2 * m, "o": h * 2},
                               page_rows=64, device=dev)
        got = run(buf)
        buf.check()
        D.check_ep_status()
        st = buf.stats()
        bad = [i for i, (a, b) in enumerate(zip(ref, got)) if not torch.equal(a, b)]
        if st["free_pages"] != 256 or st["peak_pages_used"] == 0:
            bad.append(f"pages {st}")
        return "ok" if not bad else f"mismatch {bad}"

    res = run_ranks(N, body, dev)
    assert all(r == "ok" for r in res), res


@pytest.mark.parametrize("sync_free", [False, True])
def test_loopback_ep_unequal_tokens_rejected(sync_free, dev):
    """Ranks with different token counts: the host-planned transports raise on
    every rank before any exchange; the sync-free device planner poisons the plan (no
    push, pull or scatter touches a peer's buffers) and check_ep_status() raises."""
    from paper_2603_07685_b200 import _lib
    from paper_2603_07685_b200.dispatcher import check_ep_status
    from paper_2603_07685_b200.layer import MoEConfig
    from paper_2603_07685_b200.loopback import forward_backward, run_ranks

    E, K, h, m = 8, 2, 256, 256
    cfg = MoEConfig(E, K, h, m, aux_loss_coeff=1e-2)

    def body(ep):
        T = 256 if ep.rank == 0 else 192
        g = torch.Generator(device=dev).manual_seed(ep.rank)
        bf = torch.bfloat16
        el = E // ep.n
        x = torch.randn((T, h), device=dev, generator=g).to(bf)
        w_r = (torch.randn((h, E), device=dev, generator=g) / 16).to(bf)
        w1 = (torch.randn((el, 2 * m, h), device=dev, generator=g) / 16).to(bf)
        w2 = (torch.randn((el, h, m), device=dev, generator=g) / 16).to(bf)
        forward_backward(x, w_r, w1, w2, cfg, ep, torch.ones_like(x), transport="p2p",
                         sync_free=sync_free, tag=f"unequal{int(sync_free)}")
        torch.cuda.current_stream().synchronize()
        try:
            check_ep_status()
        except _lib.MoEKernelError as exc:
            return str(exc)
        return "no error"

    from paper_2603_07685_b200 import dispatcher as D

    try:
        if sync_free:
            res = run_ranks(2, body, dev)
            assert all("inconsistent" in r for r in res), res
        else:
            with pytest.raises(RuntimeError, match="same number of tokens"):
                run_ranks(2, body, dev)
    finally:  # drop the poisoned pools: later check_ep_status() calls look at every pool
        for key in [k for k in D._POOLS if str(k[2]).startswith("unequal")]:
            del D._POOLS[key]


@pytest.mark.parametrize("transport", ["p2p", "p2p_sync_free", "nccl"])
@pytest.mark.parametrize("name", ["dropless_softmax", "capacity_pad", "top8"])
def test_loopback_ep8(name, transport, dev):
    """EP = 8, the whole EP group of a B200 box (one expert per rank at E = 8): the layout the
    8-GPU scaling run uses, here as 8 loopback ranks on one GPU."""
    _run(CASES[name], transport, dev, n=8)
