"""Can a push kernel run beside a persistent grouped GEMM that waits for it?

The GEMM (fc1_fwd_ep / fc2_dgrad_ep) is launched first and spins on a flag; after a host
delay, a push kernel variant + the signal kernel are launched on a second stream. If the
push cannot be co-scheduled, the GEMM's wait times out (2 s) and status[0] = 1.
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_07685_b200 import _lib, gemm  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    bf = torch.bfloat16
    E, h, m, rows = 4, 4096, 1536, 8192
    nblk = rows // 128
    be = torch.arange(nblk, device=dev, dtype=torch.int32) // (nblk // E)
    nmb = torch.tensor([nblk], device=dev, dtype=torch.int32)
    need = torch.ones((nblk,), dtype=torch.int32, device=dev)
    order = torch.arange(nblk // 2, dtype=torch.int32, device=dev)
    w1 = torch.randn((E, 2 * m, h), device=dev).to(bf)
    w2 = torch.randn((E, h, m), device=dev).to(bf)
    xp = torch.randn((rows, h), device=dev).to(bf)
    preact = torch.randn((rows, 2 * m), device=dev).to(bf)
    T, K = 32768, 8
    x = torch.randn((T, h), device=dev).to(bf)
    topk = torch.randint(0, E, (T, K), device=dev, dtype=torch.int32)
    inv = torch.randint(0, rows, (T, K), device=dev, dtype=torch.int32)
    base = torch.zeros((E,), dtype=torch.int32, device=dev)
    dst = torch.empty((rows * 2, h), dtype=bf, device=dev)
    peers = torch.tensor([dst.data_ptr()], dtype=torch.int64, device=dev)
    prob = torch.rand((T, K), device=dev)
    dprob = torch.zeros((T, K), device=dev)
    flags = torch.zeros((32,), dtype=torch.int32, device=dev)
    epoch_dev = torch.zeros((1,), dtype=torch.int32, device=dev)
    fpeers = torch.tensor([flags.data_ptr()], dtype=torch.int64, device=dev)
    side = torch.cuda.Stream()
    _lib.call("moe_ep_prepare")
    main_s = torch.cuda.current_stream()
    epoch = 0
    for gname in ("fc1_fwd_ep", "fc2_dgrad_ep"):
        for pname in ("none", "dispatch_push", "bwd_push"):
            epoch += 1
            status = torch.zeros((8,), dtype=torch.int32, device=dev)
            _lib.call("moe_ep_epoch_bump", epoch_dev.data_ptr(), main_s.cuda_stream)
            wait = (flags, epoch_dev, need, order, status)
            torch.cuda.synchronize()
            t0 = time.time()
            if gname == "fc1_fwd_ep":
                gemm.fc1_fwd(xp, w1, be, nmb, pair=True, wait=wait)
            else:
                gemm.fc2_dgrad(xp, w2, preact, be, nmb, pair=True, wait=wait)
            time.sleep(0.05)
            cs = side.cuda_stream
            with torch.cuda.stream(side):
                if pname == "dispatch_push":
                    _lib.call("moe_ep_dispatch_push_dest", x.data_ptr(), T, K, h, topk.data_ptr(),
                              inv.data_ptr(), base.data_ptr(), E, peers.data_ptr(), None, None,
                              0, cs)
                elif pname == "bwd_push":
                    _lib.call("moe_ep_combine_bwd_push_dest", x.data_ptr(), None,
                              peers.data_ptr(), T, K, h, topk.data_ptr(), inv.data_ptr(),
                              base.data_ptr(), E, prob.data_ptr(), None, 0, cs)
                _lib.call("moe_ep_signal", fpeers.data_ptr(), 0, 0, epoch_dev.data_ptr(), cs)
            torch.cuda.synchronize()
            st = status.tolist()
            print(f"{gname:14s} + {pname:14s}: {1e3 * (time.time() - t0):8.1f} ms  status {st}",
                  flush=True)


if __name__ == "__main__":
    main()
