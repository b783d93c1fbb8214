"""EP host logic (paper_2603_07685_b200/dispatcher.py) on CPU with torch.distributed gloo.

Each rank routes its slice [r*T, (r+1)*T) of one global batch with the oracle, the ranks
all-gather their per-expert counts (as the GPU path does over NCCL), build the exchange
plan, emulate the all-to-all + regroup in numpy, and compare every local expert block
with the GLOBAL oracle permute: row ids (global token index) and rows
must be bit-identical, including global-position capacity drops and phantom rows; the
global aux loss must equal the oracle's aux on the global batch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import routing_ref as R
from paper_2603_07685_b200.dispatcher import (ep_host_plan, global_aux,
                                              regroup_maps_numpy)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [
    dict(E=8, K=2, T=37, cf=None, pad=False, skew=0.0),
    dict(E=8, K=2, T=64, cf=1.0, pad=True, skew=1.0),
    dict(E=6, K=3, T=50, cf=0.5, pad=False, skew=2.0),
    dict(E=4, K=1, T=33, cf=1.25, pad=True, skew=0.5),
]


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E, K, T = case["E"], case["K"], case["T"]
        rng = np.random.default_rng(7)
        h = 5
        logits_g = rng.normal(size=(world * T, E)) - case["skew"] * np.log1p(np.arange(E))
        x_g = rng.normal(size=(world * T, h))
        sl = slice(rank * T, (rank + 1) * T)
        d_loc = R.route(logits_g[sl], np.eye(E), top_k=K)
        stats = torch.tensor(np.concatenate([d_loc.counts, d_loc.scores.mean(0)]),
                             dtype=torch.float64)
        gathered = [torch.zeros_like(stats) for _ in range(world)]
        dist.all_gather(gathered, stats)
        g = torch.stack(gathered).numpy()
        counts_all = np.rint(g[:, :E]).astype(np.int64)
        cap = -1 if case["cf"] is None else R.expert_capacity(case["cf"], world * T, K, E)
        hp = ep_host_plan(counts_all, rank, cap, case["pad"])

        # ---- send side: local compact permute with this rank's per-expert capacity
        send_rows, send_ids = [], []
        for e in range(E):
            src = np.flatnonzero(d_loc.routing_map[:, e])
            if hp.cap_local is not None:
                src = src[: hp.cap_local[e]]
            send_ids.append(src + rank * T)
            send_rows.append(x_g[sl][src])
        send_ids = np.concatenate(send_ids)
        send_rows = np.concatenate(send_rows)
        assert len(send_ids) == sum(hp.send_splits)
        # ---- emulated all-to-all (all_gather of everyone's send buffers + splits)
        pack = torch.tensor(np.concatenate([send_ids[:, None], send_rows], axis=1))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([len(send_ids)]))
        mx = int(max(s.item() for s in sizes))
        padded = torch.zeros((mx, h + 1), dtype=torch.float64)
        padded[: len(send_ids)] = pack
        allp = [torch.zeros_like(padded) for _ in range(world)]
        dist.all_gather(allp, padded)
        recv = []
        for s in range(world):
            splits_s = ep_host_plan(counts_all, s, cap, case["pad"]).send_splits
            off = sum(splits_s[:rank])
            recv.append(allp[s].numpy()[off: off + splits_s[rank]])
        recv = np.concatenate(recv)
        assert len(recv) == sum(hp.recv_splits)
        # ---- regroup into the local padded plan
        map_pad, map_recv = regroup_maps_numpy(hp)
        ids_pad = np.where(map_pad >= 0, recv[np.maximum(map_pad, 0), 0], -1)
        rows_pad = np.where((map_pad >= 0)[:, None], recv[np.maximum(map_pad, 0), 1:], 0.0)
        assert np.array_equal(map_recv[map_pad[map_pad >= 0]], np.flatnonzero(map_pad >= 0))

        # ---- global oracle
        d_g = R.route(logits_g, np.eye(E), top_k=K)
        if cap >= 0:
            d_g = R.apply_capacity(d_g, case["cf"], pad=case["pad"])
        perm_g, rmap_g = R.permute(x_g, d_g)
        sl_g = R.expert_slices(d_g)
        for j in range(hp.el):
            e = rank * hp.el + j
            _, gs = sl_g[e]
            blk = slice(int(hp.off_pad[j]), int(hp.off_pad[j]) + int(hp.eff[j]))
            assert np.array_equal(ids_pad[blk].astype(np.int64), rmap_g[gs]), (rank, e)
            assert np.array_equal(rows_pad[blk], perm_g[gs]), (rank, e)
            # padding rows beyond eff are zero and unmapped
            tail = slice(blk.stop, int(hp.off_pad[j + 1]))
            assert np.all(map_pad[tail] == -1)
        aux, aux_grad = global_aux(counts_all, g[:, E:], T, K, 0.01)
        assert aux == pytest.approx(R.aux_loss(R.route(logits_g, np.eye(E), top_k=K), 0.01),
                                    rel=1e-12)
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, traceback.format_exc() + repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES, ids=[str(i) for i in range(len(CASES))])
@pytest.mark.parametrize("world", [2])
def test_ep_plan_matches_global_oracle(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"


def test_ep_plan_single_process_world4():
    """All four ranks' plans, computed in one process, tile the global expert blocks."""
    rng = np.random.default_rng(3)
    n, E, K, T = 4, 8, 2, 40
    logits_g = rng.normal(size=(n * T, E))
    counts_all = np.stack([R.route(logits_g[r * T:(r + 1) * T], np.eye(E), top_k=K).counts
                           for r in range(n)])
    cap = R.expert_capacity(0.8, n * T, K, E)
    d_g = R.apply_capacity(R.route(logits_g, np.eye(E), top_k=K), 0.8, pad=True)
    eff_g = d_g.effective_counts()
    for r in range(n):
        hp = ep_host_plan(counts_all, r, cap, True)
        assert np.array_equal(hp.eff, eff_g[r * 2:(r + 1) * 2])
        assert sum(hp.recv_splits) == int(hp.real.sum())
    # total bytes sent off-rank vs the reference byte model (uniform routing is its mean)
    sent = sum(sum(ep_host_plan(counts_all, r, -1).send_splits) -
               ep_host_plan(counts_all, r, -1).send_splits[r] for r in range(n))
    assert sent <= n * T * K


def test_static_rows_bound_every_plan():
    """Sync-free EP buffers (dispatcher.ep_static_rows) bound every rank's padded plan,
    including all-to-one routing and capacity with pad."""
    from paper_2603_07685_b200 import ops
    from paper_2603_07685_b200.dispatcher import ep_static_rows, p2p_tables

    rng = np.random.default_rng(41)
    for _ in range(200):
        n = int(rng.choice([2, 4, 8]))
        el = int(rng.integers(1, 5))
        E, T, K = n * el, int(rng.integers(1, 300)), int(rng.integers(1, min(4, n * el) + 1))
        cf = [None, 0.5, 1.0, 2.0][int(rng.integers(0, 4))]
        pad = bool(rng.integers(0, 2))
        cap = -1 if cf is None else -(-int(round(cf * n * T * K)) // E)
        align = ops.pick_align(n * T, K, E)
        if rng.random() < 0.3:  # everything onto rank 0's first expert
            counts = np.zeros((n, E), dtype=np.int64)
            counts[:, 0] = T * K
        else:
            counts = np.stack([rng.multinomial(T * K, rng.dirichlet(np.ones(E) * 0.3))
                               for _ in range(n)])
        bound = ep_static_rows(n, T, K, E, cap, align)
        for me in range(n):
            _, rows_all, hp = p2p_tables(counts, me, cap, pad, align)
            assert max(rows_all) <= bound, (n, E, T, K, cf, pad)
            assert hp.rows_pad % align == 0


def test_mx_interleave_layouts():
    """The MXFP8 fc1 weight layouts (64-row gate/up blocks, or the bf16 engine's 128) keep
    every (gate, up) pair inside one GEMM tile of the matching width."""
    from paper_2603_07685_b200 import gemm

    E, m, h = 2, 256, 8
    gate = torch.arange(E * m * h, dtype=torch.float32).reshape(E, m, h)
    up = -gate
    w64 = gemm.interleave_gate_up_mx(gate, up)
    w128 = gemm.interleave_gate_up(gate, up)
    for w, blk in ((w64, 64), (w128, 128)):
        v = w.reshape(E, m // blk, 2, blk, h)
        assert torch.equal(v[:, :, 0].reshape(E, m, h), gate)
        assert torch.equal(v[:, :, 1].reshape(E, m, h), up)


def test_sync_free_worst_case_buffers_fit_hbm_at_ep8():
    """The sync-free transport sizes its buffers for the worst case (every selection of the
    group on one rank: n*T*K rows). At EP=2/4/8 for every BASELINE.json config the per-rank
    total must fit the 180 GB of one B200 with margin (<= 75%)."""
    from paper_2603_07685_b200.dispatcher import sync_free_bytes

    configs = {  # BASELINE.json configs[1..4] (T per GPU; DeepSeek T per SURVEY §8 table)
        "mixtral": dict(E=8, K=2, h=4096, m=14336, T=16384, cap=-1),
        "qwen3": dict(E=128, K=8, h=4096, m=1536, T=32768, cap=-1),
        "deepseek": dict(E=256, K=8, h=7168, m=2048, T=4096, cap=-1),
        "capacity": dict(E=8, K=2, h=4096, m=14336, T=16384, cap=1),
    }
    hbm = 180e9
    for name, c in configs.items():
        for n in (2, 4, 8):
            if c["E"] % n:
                continue
            cap = -(-(n * c["T"] * c["K"]) // c["E"]) if c["cap"] > 0 else -1
            b = sync_free_bytes(n, c["T"], c["K"], c["E"], c["h"], c["m"], cap)
            assert b["total"] <= 0.75 * hbm, (name, n, {k: v / 1e9 for k, v in b.items()})
