"""EP layer on N GPUs (NCCL) vs the single-process GLOBAL oracle.

Each rank owns tokens [r*T, (r+1)*T) of one global batch and experts
[r*E/N, (r+1)*E/N). The oracle runs the whole layer on the global batch (decision taken
from the GPUs' own fp32 logits, i.e. parity at the logits boundary); every rank checks
its slice of y and dX, its experts' dW1/dW2, the all-reduced dW_r and the global aux.
Skipped unless >= 2 GPUs are visible (gpurun --gpus 2|4).
"""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

from ep_cases import CASES, ECHO_CASES, MX_CASES, PAIR_CASES, rank_check  # noqa: E402


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


def _worker_diag(rank, port, transport):
    """MOE_TEST_WORKER_LOG=dir: this worker's stderr goes to dir/ep_<port>_<transport>_r<rank>.log
    and a hung worker dumps every thread's Python stack there shortly before the test's queue
    timeout (diagnosing a rank that never reports)."""
    d = os.environ.get("MOE_TEST_WORKER_LOG")
    if not d:
        return
    import faulthandler

    os.makedirs(d, exist_ok=True)
    f = open(os.path.join(d, f"ep_{port}_{transport}_r{rank}.log"), "w")
    os.dup2(f.fileno(), 2)
    faulthandler.enable(file=f)
    faulthandler.dump_traceback_later(
        max(int(os.environ.get("MOE_TEST_TIMEOUT", "300")) - 20, 10), exit=False, file=f)


def _worker(rank, world, port, case, q, transport):
    _worker_diag(rank, port, transport)
    try:
        import torch.distributed as dist

        from paper_2603_07685_b200.dispatcher import EPGroup

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        q.put((rank, rank_check(EPGroup(), case, transport, dev)))
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


@pytest.mark.parametrize("transport", ["p2p", "p2p_sync_free", "nccl"])
@pytest.mark.parametrize("name", list(PAIR_CASES))
def test_ep_pair_engine_matches_global_oracle(name, transport):
    _run(PAIR_CASES[name], transport)


def _run(case, transport, attempt=0):
    """One EP group of spawned ranks on the box's GPUs. A group in which no rank reported
    anything (no error, no result: a process-group start-up that never completed; seen twice
    in ~200 four-GPU runs, not reproducible on a re-run) is retried once on a fresh port; a
    rank that reports an error fails the test at once."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    # the whole EP group of the box (all visible GPUs: EP=8 on an 8-GPU box);
    # MOE_TEST_MAX_WORLD caps it
    world = min(torch.cuda.device_count(), int(os.environ.get("MOE_TEST_MAX_WORLD", "8")))
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
    import queue as _queue

    res = []
    try:
        for _ in range(world):
            res.append(q.get(timeout=int(os.environ.get("MOE_TEST_TIMEOUT", "300"))))
    except _queue.Empty:
        pass
    finally:
        _join_all(procs)
    # a rank that failed reports first; the others then wait on it in a collective
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"
    if not res and attempt == 0:
        import warnings

        warnings.warn(f"EP group {case} / {transport}: no rank reported; retrying once")
        return _run(case, transport, attempt=1)
    assert len(res) == world, f"only ranks {[r for r, _ in res]} of {world} reported"


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
    import queue as _queue

    res = []
    try:
        for _ in range(world):
            res.append(q.get(timeout=int(os.environ.get("MOE_TEST_TIMEOUT", "300"))))
    except _queue.Empty:
        pass
    finally:
        _join_all(procs)
    # a rank that failed reports first; the others then wait on it in a collective
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"
    assert len(res) == world, f"only ranks {[r for r, _ in res]} of {world} reported"
