"""Bisect CUDA-graph capture of the EP=1 layer step."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_07685_b200 import gemm, ops  # noqa: E402
from paper_2603_07685_b200.layer import MoEConfig, moe_forward  # noqa: E402

dev = torch.device("cuda", 0)
if "--set-device" in sys.argv:
    torch.cuda.set_device(0)
E, K, h, m, T = [int(v) for v in (sys.argv[1:6] or (8, 2, 256, 256, 512))]
cfg = MoEConfig(E, K, h, m, aux_loss_coeff=1e-2)
bf = torch.bfloat16
gen = torch.Generator(device=dev).manual_seed(5) if "--cuda-gen" in sys.argv else None
x0 = torch.randn((T, h), device=dev, generator=gen).to(bf)
dy = torch.randn((T, h), device=dev, generator=gen).to(bf)
w_r = (torch.randn((h, E), device=dev, generator=gen) * h ** -0.5).to(bf).requires_grad_()
w1 = (torch.randn((E, 2 * m, h), device=dev, generator=gen) * h ** -0.5).to(bf).requires_grad_()
w2 = (torch.randn((E, h, m), device=dev, generator=gen) * m ** -0.5).to(bf).requires_grad_()


def fwd_only():
    with torch.no_grad():
        return moe_forward(x0, w_r, w1, w2, cfg)


def fwd_bwd():
    for p in (w_r, w1, w2):
        p.grad = None
    x = x0.detach().requires_grad_(True)
    y, aux = moe_forward(x, w_r, w1, w2, cfg)
    torch.autograd.backward([y, aux], [dy, torch.ones_like(aux)])
    return y


def router_only():
    return ops.router_forward(x0, w_r.detach(), K, "softmax")


for name, fn in (() if "--bench-like" in sys.argv else
                 (("router", router_only), ("fwd", fwd_only), ("fwd_bwd", fwd_bwd))):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        print(name, "captured OK", flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, "FAILED:", str(e).splitlines()[0], flush=True)
        break

# bench-like sequence: eager warm-up on the default stream first, NVML thread running
if "--bench-like" in sys.argv:
    import threading
    import time

    import pynvml

    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    stop = threading.Event()

    def poll():
        while not stop.is_set():
            pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM)
            time.sleep(0.02)

    th = threading.Thread(target=poll, daemon=True)
    th.start()
    if "--no-default-warmup" not in sys.argv:
        for _ in range(3):
            fwd_bwd()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            fwd_bwd()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            fwd_bwd()
        g.replay()
        torch.cuda.synchronize()
        print("bench-like captured OK", flush=True)
    except Exception as e:  # noqa: BLE001
        print("bench-like FAILED:", str(e).splitlines()[0], flush=True)
    stop.set()
