"""One router forward + backward at a BASELINE shape (a short ncu target).

    python tools/router_one.py [mixtral|qwen3|deepseek] [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_07685_b200 import ops  # noqa: E402

SHAPES = {"mixtral": (16384, 4096, 8, 2, "softmax", False),
          "qwen3": (32768, 4096, 128, 8, "softmax", False),
          "deepseek": (4096, 7168, 256, 8, "sigmoid", True)}
T, h, E, K, score, bias = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "mixtral"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((T, h), device=dev, generator=g).to(torch.bfloat16)
w_r = (torch.randn((h, E), device=dev, generator=g) * h ** -0.5).to(torch.bfloat16)
sb = torch.rand((E,), device=dev, generator=g) * 0.05 if bias else None
dprob = torch.randn((T, K), device=dev, generator=g)
for _ in range(iters):
    r = ops.router_forward(x, w_r, K, score, sb, 1e-2)
    ops.router_backward(x, None, r, dprob, score, aux_scale=1.0)
torch.cuda.synchronize()
print("ok", r.path)
