"""Run N fwd+bwd steps of one MoE layer (EP=1) — a short target for ncu captures.

    python tools/layer_step.py [config] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_07685_b200.layer import MoEConfig, moe_forward  # noqa: E402

cname = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
c = bench.CONFIGS[cname]
dev = torch.device("cuda:0")
T, E, K, h, m = c["T"], c["E"], c["K"], c["h"], c["m"]
cfg = MoEConfig(E, K, h, m, score=c["score"], aux_loss_coeff=1e-2,
                shared_ffn_hidden=c.get("shared", 0))
g = torch.Generator(device=dev).manual_seed(0)
bf = torch.bfloat16
x = torch.randn((T, h), device=dev, generator=g).to(bf)
dy = torch.randn((T, h), device=dev, generator=g).to(bf)
w_r = (torch.randn((h, E), device=dev, generator=g) * h ** -0.5).to(bf).requires_grad_()
w1 = (torch.randn((E, 2 * m, h), device=dev, generator=g) * h ** -0.5).to(bf).requires_grad_()
w2 = (torch.randn((E, h, m), device=dev, generator=g) * m ** -0.5).to(bf).requires_grad_()
for _ in range(steps):
    for p in (w_r, w1, w2):
        p.grad = None
    xx = x.detach().requires_grad_(True)
    y, aux = moe_forward(xx, w_r, w1, w2, cfg)
    torch.autograd.backward([y, aux], [dy, torch.ones_like(aux)])
torch.cuda.synchronize()
print("ok", cname, steps)
