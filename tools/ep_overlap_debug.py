"""Debug/measure the overlapped EP dispatch: runs fwd+bwd steps of one EP layer with a
synchronise + status check after each step, printing per-rank step times.

  torchrun --nproc-per-node 4 tools/ep_overlap_debug.py --config qwen3 --transport p2p
"""
import argparse
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import CONFIGS  # noqa: E402
from paper_2603_07685_b200 import gemm  # noqa: E402
from paper_2603_07685_b200.dispatcher import EPGroup, check_ep_status, moe_forward_ep  # noqa
from paper_2603_07685_b200.layer import MoEConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen3")
    ap.add_argument("--transport", default="p2p")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--tokens", type=int, default=0)
    a = ap.parse_args()
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    n = dist.get_world_size()
    c = CONFIGS[a.config]
    E, K, h, m = c["E"], c["K"], c["h"], c["m"]
    T = a.tokens or c["T"]
    cfg = MoEConfig(E, K, h, m, score=c["score"], aux_loss_coeff=1e-2)
    g = torch.Generator(device=dev).manual_seed(rank)
    bf = torch.bfloat16
    x = torch.randn((T, h), generator=g, device=dev).to(bf).requires_grad_(True)
    w_r = (torch.randn((h, E), generator=g, device=dev) * h ** -0.5).to(bf).requires_grad_(True)
    el = E // n
    w1 = (torch.randn((el, 2 * m, h), generator=g, device=dev) * h ** -0.5).to(bf)
    w1.requires_grad_(True)
    w2 = (torch.randn((el, h, m), generator=g, device=dev) * m ** -0.5).to(bf)
    w2.requires_grad_(True)
    dy = torch.randn((T, h), generator=g, device=dev).to(bf)
    ep = EPGroup()
    log = open(f"gpurun_out/dbg_rank{rank}.log", "w")
    for i in range(a.steps):
        torch.cuda.synchronize()
        t0 = time.time()
        y, aux = moe_forward_ep(x, w_r, w1, w2, cfg, ep, transport=a.transport)
        torch.cuda.synchronize()
        t1 = time.time()
        torch.autograd.backward([y, aux], [dy, torch.ones_like(aux)])
        torch.cuda.synchronize()
        t2 = time.time()
        try:
            check_ep_status()
            st = "ok"
        except Exception as e:  # noqa: BLE001
            st = str(e)
        print(f"rank {rank} step {i}: fwd {1e3*(t1-t0):.1f} ms bwd {1e3*(t2-t1):.1f} ms {st}",
              file=log, flush=True)
        if st != "ok":
            break
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
