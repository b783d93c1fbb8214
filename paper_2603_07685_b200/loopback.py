"""Loopback EP group: n expert-parallel ranks simulated by n threads on ONE GPU.

Every rank runs the unchanged dispatcher (paper_2603_07685_b200.dispatcher) and the same
exchange kernels (csrc/ep.cu pushes / pulls, the fc2 / fc1-dgrad scatter epilogues, the
dedup and ECHO kernels, moe_ep_plan_device) on its own CUDA stream. The "peer" buffers of
the symmetric pool are ordinary allocations of the other ranks on the same device, so
the kernels store through exactly the same generic peer addresses they use over NVLink;
only the transport under them is local HBM instead of NVLink.

Collectives are host-side: each rank drains its stream, then meets the others at a
thread barrier (two barriers per collective so no rank reuses a slot early). That is
slower than NCCL but ordering-equivalent to the stream-ordered NCCL all-reduce barrier the
p2p transports rely on, so it tests the data plane, not the synchronisation of the
overlapped variant (``p2p_overlap`` spin-waits inside a persistent GEMM for flags written
by another rank's push kernel; on one GPU those kernels compete for the same SMs, so that
transport and CUDA-graph capture are not supported here).

Use ``run_ranks(n, fn)``; inside ``fn(ep)`` call the layer through
``forward_backward(...)`` (autograd's CUDA worker thread is shared by all threads of a
device, so the ranks call the Function's forward / backward directly).
"""
from __future__ import annotations

import threading
import traceback

import torch

from . import dispatcher as D


class LoopbackWorld:
    def __init__(self, n: int, dev, timeout: float = 300.0):
        self.n = n
        self.dev = dev
        self.barrier = threading.Barrier(n, timeout=timeout)
        self.slots: list = [None] * n


class _RemoteHandle:
    """The get_remote_tensor() part of torch symmetric memory's handle."""

    def __init__(self, tensors):
        self.tensors = tensors

    def get_remote_tensor(self, peer: int, shape, dtype):
        t = self.tensors[peer]
        numel = 1
        for d in shape:
            numel *= int(d)
        return t.view(dtype)[:numel].view(tuple(shape))


class LoopbackEPGroup:
    """Drop-in for dispatcher.EPGroup (same methods), rank `rank` of a LoopbackWorld."""

    def __init__(self, world: LoopbackWorld, rank: int):
        self.world = world
        self.n = world.n
        self.rank = rank
        self.group = self

    @property
    def key(self):
        return ("loopback", id(self.world), self.rank)

    # every collective: drain this rank's stream, publish, meet, read, drain, meet
    def _sync(self):
        if self.world.dev.type == "cuda":
            torch.cuda.current_stream().synchronize()

    def _meet(self):
        self.world.barrier.wait()

    def _publish(self, obj):
        self._sync()
        self.world.slots[self.rank] = obj
        self._meet()
        return list(self.world.slots)

    def _done(self):
        self._sync()
        self._meet()

    def all_gather_into_tensor(self, out, inp):
        slots = self._publish(inp)
        o = out.view(self.n, -1)
        for s in range(self.n):
            o[s].copy_(slots[s].reshape(-1))
        self._done()

    def all_reduce(self, t):
        slots = self._publish(t)
        acc = slots[0].clone()
        for s in range(1, self.n):
            acc += slots[s]
        self._done()
        t.copy_(acc)
        self._sync()

    def all_to_all_single(self, out, inp, out_splits, in_splits):
        slots = self._publish((inp, list(in_splits)))
        dst = 0
        for s in range(self.n):
            src, splits = slots[s]
            off = sum(splits[: self.rank])
            cnt = splits[self.rank]
            assert cnt == out_splits[s], "all_to_all_single split mismatch"
            if cnt:
                out[dst: dst + cnt].copy_(src[off: off + cnt])
            dst += cnt
        self._done()

    def symm_empty(self, numel: int, dtype, dev):
        t = torch.zeros((numel,), dtype=dtype, device=dev)
        slots = self._publish(t)
        ptrs = [x.data_ptr() for x in slots]
        self._done()
        return t, ptrs, _RemoteHandle(slots)


class _Ctx:
    """Stand-in for the autograd context of a torch.autograd.Function."""

    def save_for_backward(self, *tensors):
        self.saved_tensors = tensors


def forward_backward(x, w_r, w1_local, w2_local, cfg, ep, dy, steps: int = 1, **kw):
    """moe_forward_ep fwd (+ bwd with upstream dy and d aux = 1) called directly on the
    transport's Function. Returns (y, aux, grads of (x, w_r, w1, w2, w1s, w2s))."""
    fn, args = D.ep_function(x, w_r, w1_local, w2_local, cfg, ep, **kw)
    with torch.no_grad():
        for _ in range(steps):  # later steps reuse the pools' buffers
            ctx = _Ctx()
            y, aux = fn.forward(ctx, *args)
        g = fn.backward(ctx, dy.contiguous(), torch.ones_like(aux))
    return y, aux, (g[0], g[1], g[2], g[3], g[5], g[6])


def run_ranks(n: int, fn, dev=None):
    """Run fn(ep) for ranks 0..n-1 concurrently (one thread and CUDA stream each) on one
    device; returns the per-rank results. Any rank's exception aborts all and re-raises."""
    dev = torch.device("cuda", torch.cuda.current_device()) if dev is None else torch.device(dev)
    world = LoopbackWorld(n, dev)
    results: list = [None] * n
    errors: list = [None] * n

    def body(r):
        try:
            if dev.type != "cuda":  # host tensors (tests of the collectives themselves)
                results[r] = fn(LoopbackEPGroup(world, r))
                return
            torch.cuda.set_device(dev)
            s = torch.cuda.Stream(device=dev)
            with torch.cuda.stream(s):
                results[r] = fn(LoopbackEPGroup(world, r))
            s.synchronize()
        except BaseException:  # noqa: BLE001
            errors[r] = traceback.format_exc()
            world.barrier.abort()

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(n)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    first = next((e for e in errors if e and "BrokenBarrierError" not in e), None)
    first = first or next((e for e in errors if e), None)
    if first:
        raise RuntimeError(f"loopback EP rank failed:\n{first}")
    return results
