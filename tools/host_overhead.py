"""Host enqueue time vs device time per layer step (EP=1): is the step launch-bound?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_07685_b200.layer import MoEConfig, moe_forward  # noqa: E402

for cname in sys.argv[1:] or ["mixtral", "qwen3", "tiny"]:
    c = bench.CONFIGS[cname]
    dev = torch.device("cuda:0")
    T, E, K, h, m = c["T"], c["E"], c["K"], c["h"], c["m"]
    cfg = MoEConfig(E, K, h, m, score=c["score"], aux_loss_coeff=1e-2)
    bf = torch.bfloat16
    x = torch.randn((T, h), device=dev).to(bf)
    dy = torch.randn((T, h), device=dev).to(bf)
    w_r = (torch.randn((h, E), device=dev) * h ** -0.5).to(bf).requires_grad_()
    w1 = (torch.randn((E, 2 * m, h), device=dev) * h ** -0.5).to(bf).requires_grad_()
    w2 = (torch.randn((E, h, m), device=dev) * m ** -0.5).to(bf).requires_grad_()

    def step():
        for p in (w_r, w1, w2):
            p.grad = None
        xx = x.detach().requires_grad_(True)
        y, aux = moe_forward(xx, w_r, w1, w2, cfg)
        torch.autograd.backward([y, aux], [dy, torch.ones_like(aux)])

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    n = 10
    # host-only cost: block the GPU behind a long sleep kernel so enqueue never waits
    torch.cuda._sleep(int(2e9))
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n):
        step()
    e.record()
    torch.cuda.synchronize()
    print(f"{cname:8s} host enqueue {1e3 * (t1 - t0) / n:7.3f} ms/step   device {s.elapsed_time(e) / n:7.3f} ms/step")
    del x, dy, w_r, w1, w2
    torch.cuda.empty_cache()
