"""Expert-parallel (EP) token dispatcher: experts shard over the ranks of one box and
tokens move by NCCL all-to-all over NVLink (Megatron's all-to-all dispatcher,
PAPER.md:204-211; the reference models only its bytes, pkg/src/moelab/perf.py:62-70).

Placement follows the reference convention: expert e lives on rank e // (E / EP)
(planners.py:299, tests/test_perf.py:27-33); the EP group is all ranks of the box
(tests/test_folding.py:41-45).

Per forward:
  1. local router on this rank's T tokens;
  2. ONE all-gather of [counts | mean scores] (2E floats per rank): sizes every
     exchange, gives the global aux loss (the global aux != mean of per-rank aux), and
     the per-rank prefix that reproduces the oracle's GLOBAL-position capacity drops
     (keep slot j of expert e on rank r iff sum_{r'<r} counts[r',e] + j < C_global);
  3. local permute into the compact expert-major send buffer (expert-major order is
     already destination-rank order);
  4. NCCL all_to_all_single -> receive layout [src rank][local expert];
  5. regroup into the local 128-row padded plan (phantom rows created here, on the
     expert's home rank) -> the same tcgen05 grouped GEMMs as EP = 1;
  6. reverse regroup + all_to_all_single back, combine on the source rank.
The backward mirrors it (dY dispatch, dX combine). The only host synchronisation is
the D2H copy of the gathered [EP, 2E] statistics in step 2 (sync-free dispatch is the
SURVEY §8(f) "next" item 2).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, gemm, ops
from . import echo as echo_mod
from .layer import OVERLAP_WGRAD, MoEConfig, shared_expert_backward, shared_expert_forward


class EPGroup:
    """The EP process group (one rank per GPU, NCCL). Every collective the dispatcher
    issues goes through these methods, so another group implementation (the single-GPU
    loopback group of :mod:`paper_2603_07685_b200.loopback`) can stand in for it."""

    def __init__(self, group=None):
        self.group = group if group is not None else dist.group.WORLD
        self.n = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)

    @property
    def key(self):
        return id(self.group)

    def all_gather_into_tensor(self, out, inp):
        dist.all_gather_into_tensor(out, inp, group=self.group)

    def all_reduce(self, t):
        dist.all_reduce(t, group=self.group)

    def all_to_all_single(self, out, inp, out_splits, in_splits):
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def symm_empty(self, numel: int, dtype, dev):
        """A symmetric (peer-mapped over NVLink) buffer: (tensor, [n] peer base pointers,
        handle with get_remote_tensor(peer, shape, dtype)). Collective."""
        import torch.distributed._symmetric_memory as symm

        t = symm.empty(numel, dtype=dtype, device=dev)
        h = symm.rendezvous(t, self.group)
        ptrs = [int(p) for p in h.buffer_ptrs]
        off = int(getattr(h, "offset", 0))
        if ptrs[self.rank] != t.data_ptr():
            ptrs = [p + off for p in ptrs]
        assert ptrs[self.rank] == t.data_ptr(), "symmetric-memory peer pointers"
        return t, ptrs, h


@dataclass
class EPHostPlan:
    """Host-side exchange plan computed identically on every rank from counts_all."""

    n: int
    rank: int
    el: int                    # local experts
    kept: np.ndarray           # [n, E] rows rank s sends for expert e (after capacity)
    cap_local: np.ndarray | None  # [E] this rank's per-expert capacity (None = dropless)
    send_splits: list          # rows to each destination rank
    recv_splits: list          # rows from each source rank
    table: np.ndarray          # int32 regroup table (moe_ep_regroup_map)
    off_pad: np.ndarray        # [el+1] local padded offsets
    block_expert: np.ndarray   # [rows_pad/128]
    rows_pad: int
    real: np.ndarray           # [el] real (non-phantom) rows per local expert
    eff: np.ndarray            # [el] real + phantom


def check_uniform_tokens(counts_all: np.ndarray, t: int, K: int) -> None:
    """Every rank must route the same T tokens (capacity, buffer sizes and the symmetric
    pools are derived from the local T): each rank's pre-drop counts sum to T*K."""
    tot = np.asarray(counts_all, dtype=np.int64).sum(axis=1)
    if not np.all(tot == t * K):
        raise ValueError(f"EP ranks must hold the same number of tokens: per-rank "
                         f"selections {tot.tolist()}, expected {t * K} each")


def _excl_cumsum(a, axis=-1):
    c = np.cumsum(a, axis=axis)
    return c - a


def ep_host_plan(counts_all: np.ndarray, rank: int, capacity: int = -1,
                 pad: bool = False, align: int = ops.ALIGN) -> EPHostPlan:
    """Exchange plan from the all-gathered per-rank expert counts [n, E].

    capacity: global per-expert capacity C (apply_capacity() on the global batch,
    routing.py:226-247), -1 = dropless. pad: phantom rows fill each expert to C.
    """
    counts_all = np.asarray(counts_all, dtype=np.int64)
    n, E = counts_all.shape
    el = E // n
    if capacity < 0:
        kept = counts_all.copy()
        cap_local = None
    else:
        prefix = _excl_cumsum(counts_all, axis=0)  # tokens of lower ranks (lower global index)
        kept = np.clip(capacity - prefix, 0, counts_all)
        cap_local = np.maximum(capacity - prefix[rank], 0)
    send_splits = [int(kept[rank, d * el:(d + 1) * el].sum()) for d in range(n)]
    mine = slice(rank * el, (rank + 1) * el)
    kept_mine = kept[:, mine]                                   # [n, el]
    recv_splits = [int(v) for v in kept_mine.sum(axis=1)]
    recv_base = _excl_cumsum(np.asarray(recv_splits, dtype=np.int64))
    recv_off = recv_base[:, None] + _excl_cumsum(kept_mine, axis=1)   # [n, el]
    real = kept_mine.sum(axis=0)
    phantom = np.zeros(el, dtype=np.int64)
    if capacity >= 0 and pad:
        phantom = capacity - np.minimum(counts_all[:, mine].sum(axis=0), capacity)
    eff = real + phantom
    padded = -(-eff // align) * align
    off_pad = np.concatenate([[0], np.cumsum(padded)]).astype(np.int64)
    rows_pad = int(off_pad[-1])
    # one entry per 128-row GEMM block (also for 256-row aligned plans)
    block_expert = np.repeat(np.arange(el), padded // ops.ALIGN) if align >= ops.ALIGN else (
        np.zeros(0, dtype=np.int64))
    table = np.concatenate([kept_mine.ravel(), recv_off.ravel(), off_pad, real]).astype(np.int32)
    return EPHostPlan(n, rank, el, kept, cap_local, send_splits, recv_splits, table, off_pad,
                      block_expert, rows_pad, real, eff)


def regroup_maps_numpy(hp: EPHostPlan):
    """numpy restatement of csrc/permute.cu regroup_map_kernel (CPU tests)."""
    n, el = hp.n, hp.el
    kept = hp.table[: n * el].reshape(n, el)
    recv_off = hp.table[n * el: 2 * n * el].reshape(n, el)
    map_pad = np.full(hp.rows_pad, -1, dtype=np.int64)
    total_recv = int(sum(hp.recv_splits))
    map_recv = np.full(total_recv, -1, dtype=np.int64)
    for e in range(el):
        j = 0
        for s in range(n):
            for q in range(int(kept[s, e])):
                r = int(hp.off_pad[e]) + j
                map_pad[r] = int(recv_off[s, e]) + q
                map_recv[map_pad[r]] = r
                j += 1
    return map_pad, map_recv


def global_aux(counts_all, mean_scores_all, T, K, coeff):
    """aux_loss (routing.py:111-120) of the GLOBAL batch and d aux / d s_te (all ranks)."""
    counts = counts_all.sum(axis=0).astype(np.float64)
    n, E = counts_all.shape
    f = counts / max(n * T * K, 1)
    P = mean_scores_all.astype(np.float64).mean(axis=0)  # equal T per rank
    aux = coeff * E * float(np.dot(f, P))
    aux_grad = coeff * E * f / max(n * T, 1)
    return aux, aux_grad


class _Exchange:
    """Device-side state of one forward's exchange (kept for the backward)."""

    def __init__(self, hp: EPHostPlan, dev):
        self.hp = hp
        tab = torch.from_numpy(np.concatenate([
            hp.table, hp.block_expert.astype(np.int32), np.array([hp.rows_pad // ops.ALIGN],
                                                                 dtype=np.int32)]))
        tab = tab.pin_memory().to(dev, non_blocking=True)
        nt = hp.table.size
        self.table = tab[:nt]
        n, el = hp.n, hp.el
        self.off_pad = self.table[2 * n * el: 2 * n * el + el + 1]
        self.block_expert = tab[nt: nt + hp.block_expert.size]
        self.num_m_blocks = tab[nt + hp.block_expert.size:]
        self.rows_alloc = max(hp.rows_pad, 2 * ops.ALIGN)
        self.total_recv = int(sum(hp.recv_splits))
        self.total_send = int(sum(hp.send_splits))
        i32 = dict(dtype=torch.int32, device=dev)
        self.map_pad = torch.empty((self.rows_alloc,), **i32)
        self.map_recv = torch.empty((max(self.total_recv, 1),), **i32)
        if hp.rows_pad:
            _lib.call("moe_ep_regroup_map", self.table.data_ptr(), n, el, hp.rows_pad,
                      self.map_pad.data_ptr(), self.map_recv.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)

    def a2a(self, send, forward: bool, group):
        """forward: send layout -> receive layout; else the reverse."""
        hp = self.hp
        out_rows = self.total_recv if forward else self.total_send
        out = torch.empty((out_rows,) + tuple(send.shape[1:]), dtype=send.dtype,
                          device=send.device)
        group.all_to_all_single(out, send, hp.recv_splits if forward else hp.send_splits,
                                hp.send_splits if forward else hp.recv_splits)
        return out

    def to_padded(self, recv):
        out = torch.empty((self.rows_alloc, recv.shape[1]), dtype=recv.dtype, device=recv.device)
        src = recv if recv.shape[0] else torch.zeros((1, recv.shape[1]), dtype=recv.dtype,
                                                     device=recv.device)
        ops.gather_rows(src, self.map_pad, n=self.rows_alloc, out=out)
        return out

    def from_padded(self, rows):
        out = torch.empty((self.total_recv, rows.shape[1]), dtype=rows.dtype, device=rows.device)
        if self.total_recv:
            ops.gather_rows(rows, self.map_recv, n=self.total_recv, out=out)
        return out


class _MoEEPFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w_r, w1, w2, sel_bias, w1s, w2s, cfg: MoEConfig, ep: EPGroup):
        t, h = x.shape
        E, K = cfg.num_experts, cfg.top_k
        n = ep.n
        dev = x.device
        w_r_t, w_r_pad = ops.stage_router(w_r)
        r = ops.router_forward(x, w_r, K, cfg.score, sel_bias, 0.0, w_r_t=w_r_t)
        stats = torch.cat([r.counts.float(), r.mean_scores])
        gathered = torch.empty((n, 2 * E), dtype=torch.float32, device=dev)
        ep.all_gather_into_tensor(gathered, stats)
        g = gathered.cpu().numpy()  # the one host sync of the EP forward
        counts_all = np.rint(g[:, :E]).astype(np.int64)
        check_uniform_tokens(counts_all, t, K)
        cap = cfg.capacity(n * t)  # global capacity on the global batch
        align = ops.pick_align(n * t, K, E)
        hp = ep_host_plan(counts_all, ep.rank, cap, cfg.pad_to_capacity, align)
        _record_exchange(hp, h)
        pair = align == 2 * ops.ALIGN
        aux_v, aux_g = global_aux(counts_all, g[:, E:], t, K, cfg.aux_loss_coeff)
        small = torch.from_numpy(np.concatenate([[aux_v], aux_g]).astype(np.float32))
        small = small.pin_memory().to(dev, non_blocking=True)
        aux = small[0].clone()
        r.aux_grad = small[1:]
        cap_e = None
        if hp.cap_local is not None:
            cap_e = torch.from_numpy(hp.cap_local.astype(np.int32)).pin_memory().to(
                dev, non_blocking=True)
        xc = _Exchange(hp, dev)
        splan = ops.build_plan(r.topk_idx, r.topk_prob, E, -1, False, cap_e=cap_e, compact=True)
        send = ops.permute_gather(x, splan, out=torch.empty((max(xc.total_send, 1), h),
                                                            dtype=x.dtype, device=dev))
        recv = xc.a2a(send[: xc.total_send], True, ep)
        xp = xc.to_padded(recv)
        row_prob = None
        if cfg.mem_efficient:
            prob_recv = xc.a2a(splan.row_prob[: xc.total_send].contiguous(), True, ep)
            mp = xc.map_pad.long()
            row_prob = torch.where(mp >= 0, prob_recv[mp.clamp(min=0)] if xc.total_recv else
                                   torch.zeros_like(mp, dtype=torch.float32),
                                   torch.zeros((), device=dev)).float().contiguous()
        preact, act = gemm.fc1_fwd(xp, w1, xc.block_expert, xc.num_m_blocks, row_prob,
                                   pair=pair)
        o = gemm.fc2_fwd(act, w2, xc.block_expert, xc.num_m_blocks, pair=pair)
        o_local = xc.a2a(xc.from_padded(o), False, ep)
        shared = shared_expert_forward(x, w1s, w2s) if w1s is not None else None
        y = ops.combine(o_local, splan, None if cfg.mem_efficient else r.topk_prob,
                        resid=x if cap >= 0 else None,
                        extra=shared[-1] if shared is not None else None)
        ctx.cfg, ctx.ep, ctx.r, ctx.splan, ctx.xc, ctx.cap = cfg, ep, r, splan, xc, cap
        ctx.row_prob = row_prob
        ctx.pair = pair
        ctx.shared = shared[:-1] if shared is not None else None
        ctx.save_for_backward(x, w_r_pad, w1, w2, xp, preact, act, o_local, w1s, w2s)
        return y, aux

    @staticmethod
    def backward(ctx, dy, daux):
        cfg, ep, r, splan, xc = ctx.cfg, ctx.ep, ctx.r, ctx.splan, ctx.xc
        x, w_r_pad, w1, w2, xp, preact, act, o_local, w1s, w2s = ctx.saved_tensors
        dev = x.device
        h = x.shape[1]
        el = xc.hp.el
        dy = dy.contiguous()
        d_send = torch.empty((max(xc.total_send, 1), h), dtype=dy.dtype, device=dev)
        if cfg.mem_efficient:
            d_send, _ = ops.combine_backward(dy, splan, None, None, d_rows=d_send)
        else:
            d_send, dprob = ops.combine_backward(dy, splan, o_local, r.topk_prob, d_rows=d_send)
        d_o = xc.to_padded(xc.a2a(d_send[: xc.total_send], True, ep))
        if cfg.mem_efficient:
            d_pre, part = gemm.fc2_dgrad(d_o, w2, preact, xc.block_expert, xc.num_m_blocks,
                                         row_prob=ctx.row_prob, want_dprob=True, pair=ctx.pair)
            dp_pad = part.sum(dim=1)
            dp_recv = dp_pad[xc.map_recv.long()] if xc.total_recv else dp_pad[:0]
            dp_send = xc.a2a(dp_recv.contiguous(), False, ep)
            inv = splan.inv_map.long()
            dprob = torch.where(inv >= 0, dp_send[inv.clamp(min=0)] if xc.total_send else
                                torch.zeros_like(inv, dtype=torch.float32),
                                torch.zeros((), device=dev)).float().contiguous()
        else:
            d_pre, _ = gemm.fc2_dgrad(d_o, w2, preact, xc.block_expert, xc.num_m_blocks,
                                      pair=ctx.pair)
        dw2 = gemm.wgrad(d_o, act, xc.off_pad, el, overlap_prev=OVERLAP_WGRAD)
        dxp = gemm.fc1_dgrad(d_pre, w1, xc.block_expert, xc.num_m_blocks, pair=ctx.pair)
        dw1 = gemm.wgrad(d_pre, xp, xc.off_pad, el, overlap_prev=OVERLAP_WGRAD)
        dxp_local = xc.a2a(xc.from_padded(dxp), False, ep)
        aux_scale = None if daux is None else daux.float()
        dw_r, dx_router = ops.router_backward(x, w_r_pad, r, dprob, cfg.score,
                                              aux_scale=aux_scale)
        dx_shared = dw1s = dw2s = None
        if ctx.shared is not None:
            dx_shared, dw1s, dw2s = shared_expert_backward(x, dy, w1s, w2s, ctx.shared)
        dx = ops.combine(dxp_local, splan, None, resid=dy if ctx.cap >= 0 else None,
                         extra=dx_router, extra2=dx_shared)
        return (dx, dw_r.to(torch.bfloat16), dw1, dw2, None, dw1s, dw2s, None, None)


# ----------------------------------------------------------------------------------------
# NVLink peer-memory transport: the exchange is fused into the permute / combine kernels
# (csrc/ep.cu). Token rows are pushed straight into the expert rank's padded plan and the
# expert outputs / dX rows are pulled back inside the combine; no send buffer, no NCCL
# all-to-all, no regroup copies. Stream-ordered NCCL barriers order pushes vs. consumers.


class SymmPool:
    """Symmetric (peer-mapped) buffers of one EP group. Every rank requests the same sizes
    in the same order (sizes come from the all-gathered counts), so growth is collective."""

    def __init__(self, ep: EPGroup, dev):
        self.ep = ep
        self.dev = dev
        self.bufs = {}
        self.bar = torch.zeros((1,), dtype=torch.float32, device=dev)
        # dispatch/GEMM overlap: per-dispatch epoch (same sequence on every rank), the side
        # stream the pushes run on, and the GEMMs' wait-timeout flag
        self.epoch = 0
        self.epoch_dev = torch.zeros((1,), dtype=torch.int32, device=dev)
        self.comm = torch.cuda.Stream(device=dev)
        _lib.call("moe_ep_prepare")  # load the side-stream kernels now (lazy loading)
        self.status = torch.zeros((8,), dtype=torch.int32, device=dev)

    def next_epoch(self) -> int:
        self.epoch += 1
        return self.epoch

    def get(self, name: str, numel: int, dtype):
        cur = self.bufs.get(name)
        if cur is None or cur[0].numel() < numel or cur[0].dtype != dtype:
            cap = int(numel * 1.25) + 4096
            t, ptrs, h = self.ep.symm_empty(cap, dtype, self.dev)
            peers = torch.tensor(ptrs, dtype=torch.int64, device=self.dev)
            # start from zeros (no NaN garbage in rows that are never pushed) before any
            # peer can write into it
            t.zero_()
            self.barrier()
            cur = (t, peers, h)
            self.bufs[name] = cur
        return cur[0], cur[1]

    def local(self, name: str, numel: int, dtype):
        """A (non-symmetric) tmp buffer owned by the pool, grown on demand: the worst-case
        tmp set that every layer of this tag computes in (Paged Stashing)."""
        key = "local:" + name
        cur = self.bufs.get(key)
        if cur is None or cur.numel() < numel or cur.dtype != dtype:
            cur = torch.empty((numel,), dtype=dtype, device=self.dev)
            self.bufs[key] = cur
        return cur[:numel]

    def remote(self, name: str, peer: int, numel: int, dtype):
        """Tensor view of `peer`'s copy of buffer `name` (NVLink peer memory)."""
        t, _, h = self.bufs[name]
        return h.get_remote_tensor(peer, (t.numel(),), dtype)[:numel]

    def barrier(self):
        """Stream-ordered cross-rank barrier (an NCCL all-reduce of one float)."""
        self.ep.all_reduce(self.bar)


_POOLS: dict = {}

# Last ECHO plan (measurement only): clones, pre/post max rank load.
last_echo: dict = {}

# Exact rows / bytes of the last forward's exchange on this rank (measurement only):
# rows this rank sends to other ranks and receives from them; each of the four exchanges
# of a fwd+bwd step (x dispatch, output combine, dO dispatch, dX combine) moves one
# direction's bytes of this amount over NVLink.
last_exchange: dict = {}


def _record_exchange(hp: EPHostPlan, h: int, width: int = 2):
    me = hp.rank
    el = hp.el
    sent_remote = sum(s for d, s in enumerate(hp.send_splits) if d != me)
    recv_remote = sum(s for d, s in enumerate(hp.recv_splits) if d != me)
    last_exchange.update(rows_sent_remote=int(sent_remote), rows_recv_remote=int(recv_remote),
                         bytes_sent_remote=int(sent_remote) * h * width,
                         bytes_recv_remote=int(recv_remote) * h * width,
                         local_experts=el)


# inputs of the last sync-free forward's device plan (exchange statistics on demand)
last_plan_inputs: dict = {}


def ep_static_rows(n: int, t: int, K: int, E: int, capacity: int, align: int) -> int:
    """Worst-case rows of one rank's padded plan (sync-free buffers): every selection of
    the group on this rank's experts (dropless), or el experts at capacity."""
    el = E // n
    if capacity >= 0:
        rows = el * (-(-capacity // align) * align)
    else:
        rows = n * t * K + el * (align - 1)
    return max(-(-rows // align) * align, 2 * ops.ALIGN)


def sync_free_bytes(n: int, t: int, K: int, E: int, h: int, m: int, capacity: int = -1,
                    mem_efficient: bool = False) -> dict:
    """Per-rank HBM of one sync-free p2p layer (worst-case static buffers, the default
    transport of bench.py at EP > 1), by buffer: the symmetric pools (allocated at 1.25x
    their request, SymmPool.get), the fc1 / dSwiGLU outputs and the rank's expert weights and
    their gradients. Activations of the caller (x, dY, dX) are included once each."""
    align = ops.pick_align(n * t, K, E)
    rows = ep_static_rows(n, t, K, E, capacity, align)
    el = E // n
    sym = lambda numel, w: int(numel * 1.25 + 4096) * w  # noqa: E731
    b = {
        "xp (symmetric)": sym(rows * h, 2),
        "d_o (symmetric)": sym(rows * h, 2),
        "orecv + dxrecv (symmetric)": 2 * sym(t * K * h, 2),
        "preact": rows * 2 * m * 2,
        "act": rows * m * 2,
        "d_preact": rows * 2 * m * 2,
        "row tables": rows * (2 * 8 + 4) + 4 * E * n,
        "expert weights + grads": 2 * el * 3 * h * m * 2,
        "x, dY, dX, y": 4 * t * h * 2,
    }
    if mem_efficient:
        b["prob + dprob partials (symmetric)"] = sym(rows, 4) + sym(rows * (m // 256), 4)
    b["total"] = sum(b.values())
    b["rows_static"] = rows
    return b


def exchange_stats_from_device():
    """Fill last_exchange from the last sync-free forward's gathered counts (syncs)."""
    d = last_plan_inputs
    if not d:
        return
    g = d["gathered"].cpu().numpy()
    counts_all = np.rint(g[:, :d["E"]]).astype(np.int64)
    _, _, hp = p2p_tables(counts_all, d["rank"], d["cap"], d["pad"], d["align"])
    _record_exchange(hp, d["h"])


def check_ep_status():
    """Raise if an overlapped EP GEMM timed out waiting for a source rank (synchronises)."""
    for key, pool in _POOLS.items():
        st = pool.status.tolist()
        if st[7]:
            raise _lib.MoEKernelError(
                f"EP plan inconsistent (pool {key}): token counts differ across ranks or a "
                "plan exceeds the static buffers; no rows were exchanged")
        if st[0]:
            raise _lib.MoEKernelError(
                f"EP dispatch wait timed out (pool {key}): block {st[1]}, missing sources "
                f"mask {st[2]:#x}, epoch {st[3]}, flags[0:4] {st[4:]}")


def _overlapped_push(pool, ep, push_one, stream_main):
    """Run push_one(dest, stream) for dest = me, me+1, ... on the pool's side stream, each
    followed by a release-store of this dispatch's epoch into dest's flag slot `me`; the
    consumer GEMM on the main stream waits per block on those flags."""
    n, me = ep.n, ep.rank
    pool.next_epoch()
    flags, flag_peers = pool.get("flags", 32, torch.int32)
    # the epoch lives on the device (bumped in stream order), so a captured CUDA graph
    # replays with a fresh epoch every time
    _lib.call("moe_ep_epoch_bump", pool.epoch_dev.data_ptr(), stream_main.cuda_stream)
    ev = torch.cuda.Event()
    ev.record(stream_main)
    comm = pool.comm
    comm.wait_event(ev)
    cs = comm.cuda_stream
    with torch.cuda.stream(comm):  # (also where _lib's optional timing events go)
        for i in range(n):
            d = (me + i) % n
            push_one(d, cs)
            _lib.call("moe_ep_signal", flag_peers.data_ptr(), d, me, pool.epoch_dev.data_ptr(),
                      cs)
    return flags, pool.epoch_dev


def _pool(ep: EPGroup, dev, tag: str = "") -> SymmPool:
    """Symmetric buffers per (EP group, device, tag). Layers that are alive at the same time
    (several MoE layers before their backward) must use distinct tags: a layer's received
    rows stay in its pool until its backward has run."""
    key = (ep.key, dev.index, tag)
    if key not in _POOLS:
        _POOLS[key] = SymmPool(ep, dev)
    return _POOLS[key]


def p2p_tables(counts_all: np.ndarray, rank: int, capacity: int, pad: bool, align: int):
    """Host tables of the fused transport, identical math on every rank.

    Returns (base[E] for this source rank, rows_pad of every rank, this rank's EPHostPlan).
    base[e] = padded offset of expert e on its rank + rows of lower source ranks for e
              - this rank's compact offset of e, so dest row = base[e] + inv_c[t, k].
    """
    counts_all = np.asarray(counts_all, dtype=np.int64)
    n, E = counts_all.shape
    el = E // n
    plans = [ep_host_plan(counts_all, r, capacity, pad, align) for r in range(n)]
    kept = plans[0].kept                                     # [n, E], same on every rank
    prefix = _excl_cumsum(kept, axis=0)[rank]                # rows of lower ranks, per e
    off_c = _excl_cumsum(kept[rank])                         # compact offsets on this rank
    off_pad_e = np.concatenate([plans[e // el].off_pad[e % el: e % el + 1] for e in range(E)])
    base = (off_pad_e + prefix - off_c).astype(np.int64)
    return base, [p.rows_pad for p in plans], plans[rank]


def _echo_route(r, counts_all, E, K, n, me, slots, dev, stream):
    """ECHO plan + virtual-expert rewrite of this rank's selections (see echo.py)."""
    el = E // n
    plan = echo_mod.echo_plan(counts_all.sum(axis=0), el, slots)
    layout = echo_mod.echo_layout(counts_all, plan, el, slots)
    t = r.topk_idx.shape[0]
    splan0 = ops.build_plan(r.topk_idx, r.topk_prob, E, -1, False, compact=True)
    prefix_me = (np.cumsum(counts_all, axis=0) - counts_all)[me]
    gbase = prefix_me - (np.cumsum(counts_all[me]) - counts_all[me])
    ns = layout.seg_start.shape[1]
    tab = np.concatenate([gbase, layout.seg_start.ravel(), layout.seg_v.ravel()])
    tab = torch.from_numpy(tab.astype(np.int32)).pin_memory().to(dev, non_blocking=True)
    gbase_d, start_d, v_d = torch.split(tab, [E, E * ns, E * ns])
    topk_v = torch.empty_like(r.topk_idx)
    _lib.call("moe_ep_echo_rewrite", r.topk_idx.data_ptr(), splan0.inv_map.data_ptr(), t, K, ns,
              gbase_d.data_ptr(), start_d.data_ptr(), v_d.data_ptr(), topk_v.data_ptr(), stream)
    last_echo.clear()
    last_echo.update(clones=[(c.expert, c.rank, c.tokens) for c in plan.clones],
                     pre_max_load=plan.pre_max_load, post_max_load=plan.post_max_load,
                     target_load=plan.target_load)
    return topk_v, n * layout.el_v, layout.counts_v, layout


def _echo_weights(pool, ep, w1, w2, layout):
    """Stacked weights of this rank's virtual experts: own experts, then its clone slots
    filled with the home experts' weights pulled over NVLink."""
    el = w1.shape[0]
    me = ep.rank
    out = []
    for w, name in ((w1, "echo_w1"), (w2, "echo_w2")):
        exp, _ = pool.get(name, w.numel(), w.dtype)
        exp[: w.numel()].copy_(w.reshape(-1))
        pool.barrier()
        ext = torch.empty((el + layout.slots,) + tuple(w.shape[1:]), dtype=w.dtype,
                          device=w.device)
        ext[:el].copy_(w)
        per = w[0].numel()
        for g in range(layout.slots):
            e = int(layout.slot_expert[me, g])
            if e < 0:
                ext[el + g].zero_()
                continue
            home, j = e // el, e % el
            src = pool.remote(name, home, w.numel(), w.dtype)[j * per:(j + 1) * per]
            ext[el + g].copy_(src.view(w.shape[1:]))
        out.append(ext)
    return out[0], out[1]


def _echo_reduce(pool, ep, dw_ext, layout, el, name):
    """echo_grad_reduce (planners.py:379-387): home gradient + clone gradients, plan order."""
    me = ep.rank
    slots = layout.slots
    per = dw_ext[0].numel()
    exp, _ = pool.get(name, max(slots, 1) * per, dw_ext.dtype)
    if slots:
        exp[: slots * per].copy_(dw_ext[el:].reshape(-1))
    pool.barrier()
    own = dw_ext[:el].float()
    slot_of = {}
    for r in range(layout.slot_expert.shape[0]):
        for g in range(slots):
            if layout.slot_expert[r, g] >= 0:
                slot_of[(int(layout.slot_expert[r, g]), r)] = g
    for c in layout.plan.clones:
        if c.expert // el != me:
            continue
        g = slot_of[(c.expert, c.rank)]
        src = pool.remote(name, c.rank, slots * per, dw_ext.dtype)[g * per:(g + 1) * per]
        own[c.expert % el] += src.view(dw_ext.shape[1:]).float()
    pool.barrier()
    return own.to(dw_ext.dtype)


class _MoEEPP2PFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w_r, w1, w2, sel_bias, w1s, w2s, cfg: MoEConfig, ep: EPGroup,
                echo_slots: int = 0, scatter: bool = True, tag: str = "",
                overlap: bool = True, sync_free: bool = False, stash=None,
                layer_id: int = 0, stash_overlap: bool = False):
        t, h = x.shape
        E, K = cfg.num_experts, cfg.top_k
        mx = cfg.precision == "mxfp8"
        if mx and (cfg.mem_efficient or overlap or echo_slots or stash is not None):
            raise ValueError("MXFP8 experts under EP: standard combine, p2p / p2p_pull "
                             "transport, no ECHO / stash")
        n = ep.n
        dev = x.device
        pool = _pool(ep, dev, tag)
        stream = torch.cuda.current_stream().cuda_stream
        w_r_t, w_r_pad = ops.stage_router(w_r)
        r = ops.router_forward(x, w_r, K, cfg.score, sel_bias, 0.0, w_r_t=w_r_t)
        stats = torch.cat([r.counts.float(), r.mean_scores])
        gathered = torch.empty((n, 2 * E), dtype=torch.float32, device=dev)
        if stash is not None and stash_overlap:
            # this tag's tmp buffers are free once the stash of its previous layer (on the
            # pack stream) has read them; ordering the all-gather after that also keeps
            # peers from pushing into xp early
            for ev in getattr(pool, "stash_done", ()):
                torch.cuda.current_stream().wait_event(ev)
        ep.all_gather_into_tensor(gathered, stats)  # also the reuse barrier
        cap = cfg.capacity(n * t)
        layout = None
        topk_use, E_use = r.topk_idx, E
        if sync_free and not echo_slots:
            # ---- device-side planning: no host read of the counts (CUDA-graph capturable);
            # buffers are sized for the worst case (every selection on one rank)
            align = ops.pick_align(n * t, K, E)
            el = E // n
            rows_alloc = ep_static_rows(n, t, K, E, cap, align)
            rows_bound = rows_alloc
            i32 = dict(dtype=torch.int32, device=dev)
            tab = torch.empty((E + E + 2 * n * el + 2 * el + 1 + rows_alloc // ops.ALIGN + 3
                               + n * el,), **i32)
            lens = [E, E, 2 * n * el + 2 * el + 1, rows_alloc // ops.ALIGN, 3, n * el]
            base_d, cap_d, table_d, be_d, meta_d, dst_off_d = torch.split(tab, lens)
            smallf = torch.empty((1 + E,), dtype=torch.float32, device=dev)
            _lib.call("moe_ep_plan_device", gathered.data_ptr(), 2 * E, n, E, ep.rank, t, K, cap,
                      int(cfg.pad_to_capacity), align, float(cfg.aux_loss_coeff), rows_alloc,
                      base_d.data_ptr(), cap_d.data_ptr(), table_d.data_ptr(), be_d.data_ptr(),
                      rows_alloc // ops.ALIGN, meta_d.data_ptr(), dst_off_d.data_ptr(),
                      smallf.data_ptr(), smallf[1:].data_ptr(), pool.status[7:].data_ptr(),
                      stream)
            aux = smallf[0]
            r.aux_grad = smallf[1:]
            last_plan_inputs.update(gathered=gathered, rank=ep.rank, cap=cap,
                                    pad=cfg.pad_to_capacity, align=align, h=h, E=E)
            has_cap = cap >= 0
        else:
            g = gathered.cpu().numpy()  # the one host sync of the EP forward
            counts_all = np.rint(g[:, :E]).astype(np.int64)
            check_uniform_tokens(counts_all, t, K)
            # ECHO: route to virtual experts (expert segments on their serving ranks)
            counts_use = counts_all
            if echo_slots:
                if cap >= 0:
                    raise ValueError("ECHO cloning applies to dropless routing (no capacity)")
                topk_use, E_use, counts_use, layout = _echo_route(r, counts_all, E, K, n,
                                                                  ep.rank, echo_slots, dev,
                                                                  stream)
            align = ops.pick_align(n * t, K, E_use)
            base, rows_all, hp = p2p_tables(counts_use, ep.rank, cap, cfg.pad_to_capacity, align)
            _record_exchange(hp, h)
            aux_v, aux_g = global_aux(counts_all, g[:, E:], t, K, cfg.aux_loss_coeff)
            rows_alloc = max(max(rows_all), 2 * ops.ALIGN)
            rows_bound = hp.rows_pad
            el = hp.el
            # one pinned H2D copy of every small table
            cap_local = hp.cap_local if hp.cap_local is not None else np.full(E_use, -1)
            meta = np.array([hp.rows_pad // ops.ALIGN, hp.rows_pad, 0], dtype=np.int64)
            # dst_off[s, j]: source s's compact offset of this rank's j-th (virtual) expert,
            # where the scatter epilogues return that expert's rows
            dst_off = _excl_cumsum(hp.kept, axis=1)[:, ep.rank * el:(ep.rank + 1) * el].ravel()
            parts = [base, cap_local, hp.table.astype(np.int64), hp.block_expert, meta, dst_off]
            lens = [len(p) for p in parts]
            tab = torch.from_numpy(np.concatenate(parts).astype(np.int32)).pin_memory().to(
                dev, non_blocking=True)
            base_d, cap_d, table_d, be_d, meta_d, dst_off_d = torch.split(tab, lens)
            smallf = torch.from_numpy(np.concatenate([[aux_v], aux_g]).astype(np.float32))
            smallf = smallf.pin_memory().to(dev, non_blocking=True)
            aux = smallf[0].clone()
            r.aux_grad = smallf[1:]
            has_cap = hp.cap_local is not None
        pair = align == 2 * ops.ALIGN
        ctx_topk = topk_use
        nmb = meta_d[0:1]
        off_pad_d = table_d[2 * n * el: 2 * n * el + el + 1]

        splan = ops.build_plan(topk_use, r.topk_prob, E_use, -1, False,
                               cap_e=cap_d if has_cap else None, compact=True)
        if layout is not None:
            w1, w2 = _echo_weights(pool, ep, w1, w2, layout)
        xp, xp_peers = pool.get("xp", rows_alloc * h, torch.bfloat16)
        xp = xp[: rows_alloc * h].view(rows_alloc, h)
        prob_peers = None
        row_prob = None
        if cfg.mem_efficient:
            pr, prob_peers = pool.get("prob", rows_alloc, torch.float32)
            row_prob = pr[:rows_alloc]
        map_pad = torch.empty((rows_alloc,), dtype=torch.int32, device=dev)
        if rows_bound:
            _lib.call("moe_ep_regroup_map", table_d.data_ptr(), n, el, rows_bound,
                      map_pad.data_ptr(), None, stream)
        # zero this rank's padding / phantom rows (disjoint from the rows peers push)
        _lib.call("moe_zero_pad_rows", meta_d.data_ptr(), map_pad.data_ptr(), h, xp.data_ptr(),
                  stream)
        # (row_prob of padding rows: zero at allocation, else a stale finite prob of a row
        # whose activation is exactly zero; never cleared here, peers may already be pushing)
        push_args = (x.data_ptr(), t, K, h, ctx_topk.data_ptr(), splan.inv_map.data_ptr(),
                     base_d.data_ptr(), el, xp_peers.data_ptr(),
                     r.topk_prob.data_ptr() if cfg.mem_efficient else None,
                     prob_peers.data_ptr() if prob_peers is not None else None)
        overlap = overlap and scatter
        wait = None
        if overlap:
            # pushes run destination by destination on a side stream while fc1 consumes the
            # rows block by block as their sources signal (no barrier)
            cg = 2 if pair else 1
            nblocks = rows_bound // ops.ALIGN
            need = torch.zeros((max(rows_alloc // ops.ALIGN, 1),), dtype=torch.int32, device=dev)
            order = torch.empty((max(nblocks // cg, 1),), dtype=torch.int32, device=dev)
            if nblocks:
                _lib.call("moe_ep_block_need", table_d.data_ptr(), n, el, ep.rank,
                          nblocks - nblocks % cg, cg,
                          need.data_ptr(), order.data_ptr(), stream)
            main = torch.cuda.current_stream()
            flags, epoch = _overlapped_push(
                pool, ep, lambda d, cs: _lib.call("moe_ep_dispatch_push_dest", *push_args, d, cs),
                main)
            wait = (flags, epoch, need, order, pool.status)
            preact, act = gemm.fc1_fwd(xp, w1, be_d, nmb, row_prob, pair=pair, wait=wait,
                                       **_tmp_preact_act(pool, stash, rows_alloc, w1))
            main.wait_stream(pool.comm)
            ctx.need_order = (need, order)
        else:
            _lib.call("moe_ep_dispatch_push", *push_args, stream)
            pool.barrier()
            if not mx:
                preact, act = gemm.fc1_fwd(xp, w1, be_d, nmb, row_prob, pair=pair,
                                           **_tmp_preact_act(pool, stash, rows_alloc, w1))
        ctx.overlap = overlap
        o_mx = None
        ctx.act_t = None
        if mx:  # MXFP8 experts: fc1 + SwiGLU and fc2 into a local buffer
            preact, ctx.act_t, o_mx = gemm.mxfp8_experts_fwd(xp, w1, w2, be_d, nmb, pair)
            act = None
        y = torch.empty_like(x)
        row_dst_dx = None
        if scatter:
            # expert outputs go straight from fc2's epilogue into each source rank's compact
            # buffer over NVLink; the combine is then purely local
            rows_c = max(t * K, 1)
            orecv, orecv_peers = pool.get("orecv", rows_c * h, torch.bfloat16)
            o_local = orecv[: rows_c * h].view(rows_c, h)
            _, dxrecv_peers = pool.get("dxrecv", rows_c * h, torch.bfloat16)
            row_dst = torch.empty((2, rows_alloc), dtype=torch.int64, device=dev)
            for i, pp in enumerate((orecv_peers, dxrecv_peers)):
                _lib.call("moe_ep_row_dst", table_d.data_ptr(), n, el, rows_bound,
                          dst_off_d.data_ptr(), pp.data_ptr(), h * 2, row_dst[i].data_ptr(),
                          stream)
            row_dst_dx = row_dst[1]
            if mx:  # the MXFP8 engine has no scatter epilogue: push the rows afterwards
                _lib.call("moe_ep_scatter_rows", o_mx.data_ptr(), rows_bound, h,
                          row_dst[0].data_ptr(), stream)
            else:
                gemm.fc2_fwd_scatter(act, w2, be_d, nmb, row_dst[0], pair=pair)
            shared = shared_expert_forward(x, w1s, w2s) if w1s is not None else None
            pool.barrier()
            _lib.call("moe_combine", o_local.data_ptr(), t, K, h, splan.inv_map.data_ptr(),
                      None if cfg.mem_efficient else r.topk_prob.data_ptr(),
                      x.data_ptr() if cap >= 0 else None,
                      shared[-1].data_ptr() if shared is not None else None, None,
                      y.data_ptr(), stream)
        else:
            o, o_peers = pool.get("o", rows_alloc * h, torch.bfloat16)
            o = o[: rows_alloc * h].view(rows_alloc, h)
            if mx:
                o.copy_(o_mx)
            else:
                gemm.fc2_fwd(act, w2, be_d, nmb, out=o, pair=pair)
            shared = shared_expert_forward(x, w1s, w2s) if w1s is not None else None
            pool.barrier()
            # local compact copy of the pulled expert outputs: the backward's dprob = <dY, O>
            # then reads local memory instead of pulling O over NVLink a second time
            o_local = None
            if not cfg.mem_efficient:
                o_local = torch.empty((max(t * K, 1), h), dtype=x.dtype,
                                      device=dev)
            _lib.call("moe_ep_combine_pull", o_peers.data_ptr(), t, K, h, ctx_topk.data_ptr(),
                      splan.inv_map.data_ptr(), base_d.data_ptr(), el,
                      None if cfg.mem_efficient else r.topk_prob.data_ptr(),
                      x.data_ptr() if cap >= 0 else None,
                      shared[-1].data_ptr() if shared is not None else None, None, y.data_ptr(),
                      o_local.data_ptr() if o_local is not None else None, stream)
        if stash is not None:
            # Paged Stashing: keep only this layer's actual rows (device counts) in pages; the
            # worst-case tmp buffers (xp, preact, act, received outputs) serve the next layer
            if not sync_free or cfg.mem_efficient or layout is not None or not scatter:
                raise ValueError("paged stashing needs the sync-free p2p transport with the "
                                 "standard combine")
            st_plan, st_out = _stash_pair(stash)
            if stash_overlap:  # copies on the pack stream, overlapping the next layer
                pool.stash_done = (
                    st_plan.stash_async(2 * layer_id, {"xp": xp, "preact": preact, "act": act},
                                        rows_dev=meta_d[1:2]),
                    st_out.stash_async(2 * layer_id + 1, {"o": o_local},
                                       rows_dev=splan.meta[2:3]))
            else:
                st_plan.stash(2 * layer_id, {"xp": xp, "preact": preact, "act": act},
                              rows_dev=meta_d[1:2])
                st_out.stash(2 * layer_id + 1, {"o": o_local}, rows_dev=splan.meta[2:3])
            preact = act = None
        ctx.stash, ctx.layer_id, ctx.stash_overlap = stash, layer_id, stash_overlap
        ctx.rows_bound = rows_bound
        ctx.scatter, ctx.tag, ctx.row_dst_dx = scatter, tag, row_dst_dx
        ctx.cfg, ctx.ep, ctx.r, ctx.splan, ctx.cap, ctx.pair = cfg, ep, r, splan, cap, pair
        ctx.topk_use, ctx.layout, ctx.el_own = topk_use, layout, E // n
        ctx.o_local = o_local
        ctx.tabs = (base_d, be_d, nmb, meta_d, off_pad_d, map_pad, rows_alloc, el)
        ctx.row_prob = row_prob
        ctx.shared = shared[:-1] if shared is not None else None
        ctx.save_for_backward(x, w_r_pad, w1, w2, preact, act, w1s, w2s)
        return y, aux

    @staticmethod
    def backward(ctx, dy, daux):
        cfg, ep, r, splan = ctx.cfg, ctx.ep, ctx.r, ctx.splan
        base_d, be_d, nmb, meta_d, off_pad_d, map_pad, rows_alloc, el = ctx.tabs
        ctx_topk = ctx.topk_use
        x, w_r_pad, w1, w2, preact, act, w1s, w2s = ctx.saved_tensors
        t, h = x.shape
        K = cfg.top_k
        dev = x.device
        pool = _pool(ep, dev, ctx.tag)
        stream = torch.cuda.current_stream().cuda_stream
        dy = dy.contiguous()
        xp, _ = pool.get("xp", rows_alloc * h, torch.bfloat16)
        xp = xp[: rows_alloc * h].view(rows_alloc, h)
        if ctx.stash is not None:  # reload this layer's rows into the shared tmp buffers
            tmp = _tmp_preact_act(pool, ctx.stash, rows_alloc, w1)
            preact, act = tmp["preact"], tmp["act"]
            st_plan, st_out = _stash_pair(ctx.stash)
            st_plan.reload(2 * ctx.layer_id, {"xp": xp, "preact": preact, "act": act},
                           rows_dev=meta_d[1:2])
            st_out.reload(2 * ctx.layer_id + 1, {"o": ctx.o_local}, rows_dev=splan.meta[2:3])
            if ctx.stash_overlap and ctx.layer_id > 0:
                # prefetch the previous layer's rows (other tag: its buffers were last used
                # by the backward that just finished) while this layer's backward computes
                st_plan.prefetch(2 * (ctx.layer_id - 1))
                st_out.prefetch(2 * (ctx.layer_id - 1) + 1)
        d_o, d_peers = pool.get("do", rows_alloc * h, torch.bfloat16)
        d_o = d_o[: rows_alloc * h].view(rows_alloc, h)
        _lib.call("moe_zero_pad_rows", meta_d.data_ptr(), map_pad.data_ptr(), h, d_o.data_ptr(),
                  stream)
        push_args = (dy.data_ptr(), None if cfg.mem_efficient else ctx.o_local.data_ptr(),
                     d_peers.data_ptr(), t, K, h, ctx_topk.data_ptr(), splan.inv_map.data_ptr(),
                     base_d.data_ptr(), el,
                     None if cfg.mem_efficient else r.topk_prob.data_ptr())
        part_peers = part = None
        if cfg.mem_efficient:
            ldp = gemm.dprob_partials(w2.shape[2])
            part, part_peers = pool.get("part", rows_alloc * ldp, torch.float32)
            part = part[: rows_alloc * ldp].view(rows_alloc, ldp)
        wait = None
        main = torch.cuda.current_stream()
        if ctx.overlap:
            # per-destination passes write dprob only for their own selections
            dprob = torch.zeros((t, K), dtype=torch.float32, device=dev)
            dp_ptr = None if cfg.mem_efficient else dprob.data_ptr()
            flags, epoch = _overlapped_push(
                pool, ep, lambda d, cs: _lib.call("moe_ep_combine_bwd_push_dest", *push_args,
                                                  dp_ptr, d, cs), main)
            wait = (flags, epoch, *ctx.need_order, pool.status)
        else:
            dprob = torch.empty((t, K), dtype=torch.float32, device=dev)
            _lib.call("moe_ep_combine_bwd_push", *push_args,
                      None if cfg.mem_efficient else dprob.data_ptr(), stream)
            pool.barrier()
        mx = cfg.precision == "mxfp8"
        dxp_mx = None
        if mx:
            dxp_mx, dw1, dw2 = gemm.mxfp8_experts_bwd(d_o, xp, w1, w2, preact, ctx.act_t, be_d,
                                                      nmb, off_pad_d, ctx.pair)
        elif cfg.mem_efficient:
            d_pre, _ = gemm.fc2_dgrad(d_o, w2, preact, be_d, nmb, row_prob=ctx.row_prob,
                                      pair=ctx.pair, part=part, wait=wait)
        else:
            d_pre, _ = gemm.fc2_dgrad(d_o, w2, preact, be_d, nmb, pair=ctx.pair, wait=wait)
        if ctx.overlap:
            main.wait_stream(pool.comm)
        if not mx:
            dw2 = gemm.wgrad(d_o, act, off_pad_d, el, overlap_prev=OVERLAP_WGRAD)
        if ctx.scatter:  # dX rows return from fc1_dgrad's epilogue into the source ranks
            if mx:
                _lib.call("moe_ep_scatter_rows", dxp_mx.data_ptr(), ctx.rows_bound, h,
                          ctx.row_dst_dx.data_ptr(), stream)
            else:
                gemm.fc1_dgrad_scatter(d_pre, w1, be_d, nmb, ctx.row_dst_dx, pair=ctx.pair)
        else:
            dxp, dxp_peers = pool.get("dxp", rows_alloc * h, torch.bfloat16)
            dxp = dxp[: rows_alloc * h].view(rows_alloc, h)
            if mx:
                dxp.copy_(dxp_mx)
            else:
                gemm.fc1_dgrad(d_pre, w1, be_d, nmb, out=dxp, pair=ctx.pair)
        if not mx:
            dw1 = gemm.wgrad(d_pre, xp, off_pad_d, el, overlap_prev=OVERLAP_WGRAD)
        # also orders every rank's reads of its symmetric buffers (xp, d_o) before any
        # peer's next write into them
        pool.barrier()
        if cfg.mem_efficient:
            _lib.call("moe_ep_dprob_pull", part_peers.data_ptr(), t, K, ctx_topk.data_ptr(),
                      splan.inv_map.data_ptr(), base_d.data_ptr(), el,
                      gemm.dprob_partials(w2.shape[2]),
                      dprob.data_ptr(), stream)
        aux_scale = None if daux is None else daux.float()
        dw_r, dx_router = ops.router_backward(x, w_r_pad, r, dprob, cfg.score,
                                              aux_scale=aux_scale)
        dx_shared = dw1s = dw2s = None
        if ctx.shared is not None:
            dx_shared, dw1s, dw2s = shared_expert_backward(x, dy, w1s, w2s, ctx.shared)
        dx = torch.empty_like(x)
        if ctx.scatter:
            rows_c = max(t * K, 1)
            dxrecv, _ = pool.get("dxrecv", rows_c * h, torch.bfloat16)
            _lib.call("moe_combine", dxrecv.data_ptr(), t, K, h, splan.inv_map.data_ptr(), None,
                      dy.data_ptr() if ctx.cap >= 0 else None, dx_router.data_ptr(),
                      dx_shared.data_ptr() if dx_shared is not None else None, dx.data_ptr(),
                      stream)
        else:
            _lib.call("moe_ep_combine_pull", dxp_peers.data_ptr(), t, K, h, ctx_topk.data_ptr(),
                      splan.inv_map.data_ptr(), base_d.data_ptr(), el, None,
                      dy.data_ptr() if ctx.cap >= 0 else None, dx_router.data_ptr(),
                      dx_shared.data_ptr() if dx_shared is not None else None, dx.data_ptr(),
                      None, stream)
            # no rank may overwrite the symmetric buffers before every rank has pulled
            pool.barrier()
        if ctx.layout is not None:  # clone weight gradients back into the home experts
            dw1 = _echo_reduce(pool, ep, dw1, ctx.layout, ctx.el_own, "echo_dw1")
            dw2 = _echo_reduce(pool, ep, dw2, ctx.layout, ctx.el_own, "echo_dw2")
        return (dx, dw_r.to(torch.bfloat16), dw1, dw2, None, dw1s, dw2s, None, None, None, None,
                None, None, None, None, None, None)


def _stash_pair(stash):
    """(buffer for the plan rows {xp, preact, act}, buffer for the returned outputs {o}):
    one PagedStashBuffer for both, or a pair (pages sized per row group)."""
    if isinstance(stash, (tuple, list)):
        return stash[0], stash[1]
    return stash, stash


def _tmp_preact_act(pool, stash, rows_alloc, w1):
    """With Paged Stashing, fc1's outputs go to the pool's shared tmp buffers."""
    if stash is None:
        return {}
    m2 = w1.shape[1]
    pre = pool.local("preact", rows_alloc * m2, torch.bfloat16).view(rows_alloc, m2)
    act = pool.local("act", rows_alloc * (m2 // 2), torch.bfloat16).view(rows_alloc, m2 // 2)
    return {"preact": pre, "act": act}


def _excl(a):
    a = np.asarray(a, dtype=np.int64)
    return np.cumsum(a) - a


class _MoEEPDedupFunction(torch.autograd.Function):
    """p2p transport with token de-duplication: one row per (token, destination rank) over
    NVLink each way; destinations expand rows locally and pre-reduce per-token outputs."""

    @staticmethod
    def forward(ctx, x, w_r, w1, w2, sel_bias, w1s, w2s, cfg: MoEConfig, ep: EPGroup,
                tag: str = ""):
        t, h = x.shape
        E, K = cfg.num_experts, cfg.top_k
        n = ep.n
        me = ep.rank
        dev = x.device
        pool = _pool(ep, dev, tag)
        stream = torch.cuda.current_stream().cuda_stream
        i32 = dict(dtype=torch.int32, device=dev)
        w_r_t, w_r_pad = ops.stage_router(w_r)
        r = ops.router_forward(x, w_r, K, cfg.score, sel_bias, 0.0, w_r_t=w_r_t)
        cap = cfg.capacity(n * t)
        el = E // n

        def token_ranks(splan_):
            rank_idx = torch.empty((t, K), **i32)
            sel_j = torch.empty((t, K), **i32)
            sel_pos = torch.empty((t, K), **i32)
            _lib.call("moe_ep_token_ranks", r.topk_idx.data_ptr(), splan_.inv_map.data_ptr(), t, K,
                      el, rank_idx.data_ptr(), sel_j.data_ptr(), sel_pos.data_ptr(), stream)
            rplan_ = ops.build_plan(rank_idx, None, n, -1, False, compact=True)
            return rank_idx, sel_j, sel_pos, rplan_

        if cap < 0:
            splan = ops.build_plan(r.topk_idx, r.topk_prob, E, -1, False, compact=True)
            rank_idx, sel_j, sel_pos, rplan = token_ranks(splan)
            stats = torch.cat([r.counts.float(), r.mean_scores, rplan.counts.float()])
            gathered = torch.empty((n, 2 * E + n), dtype=torch.float32, device=dev)
            ep.all_gather_into_tensor(gathered, stats)
            g = gathered.cpu().numpy()  # the one host sync of the forward
            counts_all = np.rint(g[:, :E]).astype(np.int64)
            check_uniform_tokens(counts_all, t, K)
            ntok = np.rint(g[:, 2 * E:]).astype(np.int64)
        else:
            stats = torch.cat([r.counts.float(), r.mean_scores])
            gathered = torch.empty((n, 2 * E), dtype=torch.float32, device=dev)
            ep.all_gather_into_tensor(gathered, stats)
            g = gathered.cpu().numpy()
            counts_all = np.rint(g[:, :E]).astype(np.int64)
            check_uniform_tokens(counts_all, t, K)
        align = ops.pick_align(n * t, K, E)
        pair = align == 2 * ops.ALIGN
        base, rows_all, hp = p2p_tables(counts_all, me, cap, cfg.pad_to_capacity, align)
        _record_exchange(hp, h)
        if cap >= 0:  # capacity: the local plan needs the global prefix first
            cap_e = torch.from_numpy(hp.cap_local.astype(np.int32)).pin_memory().to(
                dev, non_blocking=True)
            splan = ops.build_plan(r.topk_idx, r.topk_prob, E, -1, False, cap_e=cap_e,
                                   compact=True)
            rank_idx, sel_j, sel_pos, rplan = token_ranks(splan)
            tc = rplan.counts.float()
            gat2 = torch.empty((n, n), dtype=torch.float32, device=dev)
            ep.all_gather_into_tensor(gat2, tc)
            ntok = np.rint(gat2.cpu().numpy()).astype(np.int64)
        aux_v, aux_g = global_aux(counts_all, g[:, E:2 * E], t, K, cfg.aux_loss_coeff)
        # token-slot tables: this rank as source (tbase) and as destination (tok rows)
        # ntok[s, d] = tokens source s sends to destination d (one row each)
        recv_tok_off = np.stack([_excl(ntok[:, d]) for d in range(n)], axis=1)  # [s, d]
        tbase = recv_tok_off[me] - _excl(ntok[me])
        tok_recv = int(ntok[:, me].sum())
        tok_cap = max(int(ntok.sum(axis=0).max()), 1)
        rows_alloc = max(max(rows_all), 2 * ops.ALIGN)
        meta = np.array([hp.rows_pad // ops.ALIGN, hp.rows_pad, 0], dtype=np.int64)
        parts = [base, hp.table.astype(np.int64), hp.block_expert, meta, tbase]
        lens = [len(p_) for p_ in parts]
        tab = torch.from_numpy(np.concatenate(parts).astype(np.int32)).pin_memory().to(
            dev, non_blocking=True)
        base_d, table_d, be_d, meta_d, tbase_d = torch.split(tab, lens)
        smallf = torch.from_numpy(np.concatenate([[aux_v], aux_g]).astype(np.float32))
        smallf = smallf.pin_memory().to(dev, non_blocking=True)
        aux = smallf[0].clone()
        r.aux_grad = smallf[1:]
        nmb = meta_d[0:1]
        off_pad_d = table_d[2 * n * el: 2 * n * el + el + 1]

        tok, tok_peers = pool.get("dd_tok", tok_cap * h, torch.bfloat16)
        mp, map_peers = pool.get("dd_map", rows_alloc, torch.int32)
        srows, srows_peers = pool.get("dd_srows", tok_cap * K, torch.int32)
        sprob, sprob_peers = pool.get("dd_sprob", tok_cap * K, torch.float32)
        rprob, rprob_peers = pool.get("dd_rprob", rows_alloc, torch.float32)
        partial, partial_peers = pool.get("dd_partial", tok_cap * h, torch.bfloat16)
        tok = tok[: tok_cap * h].view(tok_cap, h)
        partial = partial[: tok_cap * h].view(tok_cap, h)
        map_pad = torch.empty((rows_alloc,), **i32)
        if hp.rows_pad:
            _lib.call("moe_ep_regroup_map", table_d.data_ptr(), n, el, hp.rows_pad,
                      map_pad.data_ptr(), None, stream)
        _lib.call("moe_ep_fill_pad_map", map_pad.data_ptr(), hp.rows_pad, mp.data_ptr(), stream)
        _lib.call("moe_ep_dispatch_dedup", x.data_ptr(), t, K, h, r.topk_idx.data_ptr(),
                  splan.inv_map.data_ptr(), base_d.data_ptr(), el, rank_idx.data_ptr(),
                  rplan.inv_map.data_ptr(), tbase_d.data_ptr(), sel_j.data_ptr(),
                  sel_pos.data_ptr(), r.topk_prob.data_ptr(), tok_peers.data_ptr(),
                  map_peers.data_ptr(), srows_peers.data_ptr(), sprob_peers.data_ptr(),
                  rprob_peers.data_ptr(), stream)
        pool.barrier()
        xp = torch.empty((rows_alloc, h), dtype=x.dtype, device=dev)
        if hp.rows_pad:
            ops.gather_rows(tok, mp[:rows_alloc], n=hp.rows_pad, out=xp)
        row_prob = rprob[:rows_alloc] if cfg.mem_efficient else None
        preact, act = gemm.fc1_fwd(xp, w1, be_d, nmb, row_prob, pair=pair)
        o = gemm.fc2_fwd(act, w2, be_d, nmb, pair=pair)
        if tok_recv:
            _lib.call("moe_combine", o.data_ptr(), tok_recv, K, h, srows.data_ptr(),
                      None if cfg.mem_efficient else sprob.data_ptr(), None, None, None,
                      partial.data_ptr(), stream)
        shared = shared_expert_forward(x, w1s, w2s) if w1s is not None else None
        pool.barrier()
        y = torch.empty_like(x)
        _lib.call("moe_ep_combine_pull", partial_peers.data_ptr(), t, K, h,
                  rank_idx.data_ptr(), rplan.inv_map.data_ptr(), tbase_d.data_ptr(), 1, None,
                  x.data_ptr() if cap >= 0 else None,
                  shared[-1].data_ptr() if shared is not None else None, None, y.data_ptr(),
                  None, stream)
        ctx.cfg, ctx.ep, ctx.r, ctx.cap, ctx.pair, ctx.tag = cfg, ep, r, cap, pair, tag
        ctx.st = (splan, rplan, rank_idx, base_d, tbase_d, be_d, nmb, off_pad_d, rows_alloc,
                  hp.rows_pad, tok_cap, tok_recv, el)
        ctx.shared = shared[:-1] if shared is not None else None
        ctx.save_for_backward(x, w_r_pad, w1, w2, xp, preact, act, o, w1s, w2s)
        return y, aux

    @staticmethod
    def backward(ctx, dy, daux):
        cfg, ep, r = ctx.cfg, ctx.ep, ctx.r
        (splan, rplan, rank_idx, base_d, tbase_d, be_d, nmb, off_pad_d, rows_alloc, rows_pad,
         tok_cap, tok_recv, el) = ctx.st
        x, w_r_pad, w1, w2, xp, preact, act, o, w1s, w2s = ctx.saved_tensors
        t, h = x.shape
        K = cfg.top_k
        dev = x.device
        pool = _pool(ep, dev, ctx.tag)
        stream = torch.cuda.current_stream().cuda_stream
        dy = dy.contiguous()
        tok, tok_peers = pool.get("dd_tok", tok_cap * h, torch.bfloat16)
        tok = tok[: tok_cap * h].view(tok_cap, h)
        mp, _ = pool.get("dd_map", rows_alloc, torch.int32)
        srows, _ = pool.get("dd_srows", tok_cap * K, torch.int32)
        rprob, _ = pool.get("dd_rprob", rows_alloc, torch.float32)
        partial, partial_peers = pool.get("dd_partial", tok_cap * h, torch.bfloat16)
        partial = partial[: tok_cap * h].view(tok_cap, h)
        dprows, dprows_peers = pool.get("dd_dprob_rows", rows_alloc, torch.float32)
        # dY once per (token, rank)
        _lib.call("moe_ep_dispatch_push", dy.data_ptr(), t, K, h, rank_idx.data_ptr(),
                  rplan.inv_map.data_ptr(), tbase_d.data_ptr(), 1, tok_peers.data_ptr(), None,
                  None, stream)
        pool.barrier()
        d_o = torch.empty((rows_alloc, h), dtype=dy.dtype, device=dev)
        _lib.call("moe_ep_expand_grad", tok.data_ptr(), mp.data_ptr(), rows_pad, h,
                  None if cfg.mem_efficient else rprob.data_ptr(),
                  None if cfg.mem_efficient else o.data_ptr(), d_o.data_ptr(),
                  None if cfg.mem_efficient else dprows.data_ptr(), stream)
        part_peers = None
        if cfg.mem_efficient:
            ldp = gemm.dprob_partials(w2.shape[2])
            part, part_peers = pool.get("part", rows_alloc * ldp, torch.float32)
            part = part[: rows_alloc * ldp].view(rows_alloc, ldp)
            d_pre, _ = gemm.fc2_dgrad(d_o, w2, preact, be_d, nmb, row_prob=rprob[:rows_alloc],
                                      pair=ctx.pair, part=part)
        else:
            d_pre, _ = gemm.fc2_dgrad(d_o, w2, preact, be_d, nmb, pair=ctx.pair)
        dw2 = gemm.wgrad(d_o, act, off_pad_d, el, overlap_prev=OVERLAP_WGRAD)
        dxp = gemm.fc1_dgrad(d_pre, w1, be_d, nmb, pair=ctx.pair)
        dw1 = gemm.wgrad(d_pre, xp, off_pad_d, el, overlap_prev=OVERLAP_WGRAD)
        if tok_recv:
            _lib.call("moe_combine", dxp.data_ptr(), tok_recv, K, h, srows.data_ptr(), None,
                      None, None, None, partial.data_ptr(), stream)
        pool.barrier()
        dprob = torch.empty((t, K), dtype=torch.float32, device=dev)
        if cfg.mem_efficient:
            _lib.call("moe_ep_dprob_pull", part_peers.data_ptr(), t, K, r.topk_idx.data_ptr(),
                      splan.inv_map.data_ptr(), base_d.data_ptr(), el,
                      gemm.dprob_partials(w2.shape[2]), dprob.data_ptr(), stream)
        else:
            _lib.call("moe_ep_dprob_pull", dprows_peers.data_ptr(), t, K, r.topk_idx.data_ptr(),
                      splan.inv_map.data_ptr(), base_d.data_ptr(), el, 1, dprob.data_ptr(),
                      stream)
        aux_scale = None if daux is None else daux.float()
        dw_r, dx_router = ops.router_backward(x, w_r_pad, r, dprob, cfg.score,
                                              aux_scale=aux_scale)
        dx_shared = dw1s = dw2s = None
        if ctx.shared is not None:
            dx_shared, dw1s, dw2s = shared_expert_backward(x, dy, w1s, w2s, ctx.shared)
        dx = torch.empty_like(x)
        _lib.call("moe_ep_combine_pull", partial_peers.data_ptr(), t, K, h, rank_idx.data_ptr(),
                  rplan.inv_map.data_ptr(), tbase_d.data_ptr(), 1, None,
                  dy.data_ptr() if ctx.cap >= 0 else None, dx_router.data_ptr(),
                  dx_shared.data_ptr() if dx_shared is not None else None, dx.data_ptr(), None,
                  stream)
        pool.barrier()
        return (dx, dw_r.to(torch.bfloat16), dw1, dw2, None, dw1s, dw2s, None, None, None)


def moe_forward_ep(x, w_r, w1_local, w2_local, cfg: MoEConfig, ep: EPGroup,
                   selection_bias=None, w1_shared=None, w2_shared=None, transport: str = "auto",
                   echo_slots: int = 0, tag: str = "", sync_free: bool = False,
                   stash=None, layer_id: int = 0, stash_overlap: bool = False):
    """EP MoE layer: w1_local [E/EP, 2m, h], w2_local [E/EP, h, m] are this rank's experts
    (global experts [rank*E/EP, (rank+1)*E/EP)). Returns (y [T,h], global aux).

    transport:
      "auto" (default): "p2p".
      "p2p": tokens are pushed over NVLink peer memory straight into the expert rank's
        padded plan (csrc/ep.cu); expert outputs and dX rows return from the fc2 / fc1-dgrad
        GEMM epilogues, which store each row (TMA bulk stores) into its source rank's
        buffer over NVLink, so both combines are local.
      "p2p_overlap": "p2p" with the dispatches overlapped with their consuming GEMMs: the
        pushes run destination by destination on a side stream and fc1 fwd / fc2 dgrad
        start each 128-row block as soon as its source ranks have signalled (per-block
        flags, no barrier). Correct, but not faster under the 1 kW power cap (measured).
      "p2p_pull": the previous p2p variant, where the combines pull the rows back over
        NVLink (kept for A/B measurement).
      "p2p_dedup": token de-duplication (one row per (token, destination rank) each way;
        HybridEP-style).
      "nccl": permute -> NCCL all_to_all_single -> regroup (the baseline dispatcher).
    tag: buffer namespace; give every MoE layer that is alive at the same time its own.
    sync_free (p2p transports, no ECHO): plan the exchange on the device
      (moe_ep_plan_device) with worst-case static buffers, so the step never reads the
      counts on the host and can be captured in a CUDA graph.
    stash (a stash.PagedStashBuffer with pools "xp", "preact", "act", "o", or a pair of
      buffers for {xp, preact, act} and {o}; sync_free p2p, standard combine): Paged
      Stashing.
      Layers sharing a `tag` compute in one set of worst-case tmp buffers; each layer's
      actual rows are copied into pages after its forward and back before its backward, so
      memory is O(worst case + sum of actual rows) instead of O(layers x worst case).
      layer_id: this layer's stash record key (unique among live layers).
      Out of pages (the reference's MemoryError, planners.py:441-446): a stash that finds
      too few free pages records nothing and its reload fills the layer's rows with NaN, so
      the gradients come out NaN rather than silently wrong; PagedStashBuffer.check()
      (a host sync) raises the MemoryError.
    stash_overlap: run the stash copies on a pack stream while the next layer computes and
      prefetch reloads on an unpack stream during the later layer's backward.
      Needs two alternating tags (layer i uses tag of parity i % 2: double-buffered tmp
      sets) and layer ids 0, 1, 2, ... in forward order.

    The router weight gradient returned is this rank's partial sum over its own tokens;
    W_r is replicated, so its all-reduce belongs to the data-parallel gradient sync.
    """
    fn, args = ep_function(x, w_r, w1_local, w2_local, cfg, ep, selection_bias, w1_shared,
                           w2_shared, transport, echo_slots, tag, sync_free, stash, layer_id,
                           stash_overlap)
    return fn.apply(*args)


def ep_function(x, w_r, w1_local, w2_local, cfg: MoEConfig, ep: EPGroup,
                selection_bias=None, w1_shared=None, w2_shared=None, transport: str = "auto",
                echo_slots: int = 0, tag: str = "", sync_free: bool = False,
                stash=None, layer_id: int = 0, stash_overlap: bool = False):
    """(autograd.Function, apply-args) of moe_forward_ep's transport (same arguments)."""
    if cfg.num_experts % ep.n:
        raise ValueError(f"num_experts {cfg.num_experts} not divisible by EP {ep.n}")
    if transport == "auto":
        # measured on B200 at EP=4 (profiles/r01_summary.md): p2p with the scatter epilogues
        # beats dedup (Qwen3 4.12M vs 3.94M tok/s, DeepSeek 1.25M vs 1.18M, Mixtral 2.06M vs
        # 2.02M) and the overlapped variant under the 1 kW power cap
        transport = "p2p"
    args = (x, w_r, w1_local, w2_local, selection_bias, w1_shared, w2_shared, cfg, ep)
    if echo_slots or transport in ("p2p", "p2p_overlap", "p2p_pull"):
        # ECHO hot-expert cloning runs on the p2p transport (virtual experts)
        return _MoEEPP2PFunction, (*args, int(echo_slots), transport != "p2p_pull", tag,
                                   transport == "p2p_overlap", sync_free and not echo_slots,
                                   stash, int(layer_id), bool(stash_overlap))
    if cfg.precision != "bf16":
        raise ValueError(f"precision {cfg.precision!r} runs on the p2p / p2p_pull transports")
    if transport == "p2p_dedup":
        return _MoEEPDedupFunction, (*args, tag)
    if transport == "nccl":
        return _MoEEPFunction, args
    raise ValueError(f"unknown transport {transport!r}")
