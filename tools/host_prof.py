"""cProfile of the host side of one layer step while the GPU is held busy (enqueue cost)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_07685_b200.layer import MoEConfig, moe_forward  # noqa: E402

cname = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
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
torch.cuda._sleep(int(3e9))
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
