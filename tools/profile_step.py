"""torch.profiler view of one MoE layer fwd+bwd step (CPU vs GPU time, gaps)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_07685_b200.layer import MoEConfig, moe_forward  # noqa: E402

cname = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
c = bench.CONFIGS[cname]
dev = torch.device("cuda:0")
T, E, K, h, m = c["T"], c["E"], c["K"], c["h"], c["m"]
cfg = MoEConfig(E, K, h, m, score=c["score"], aux_loss_coeff=1e-2,
                shared_ffn_hidden=c.get("shared", 0))
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
t0 = time.perf_counter()
for _ in range(3):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3 * (t1 - t0) / 3:.2f} ms/step, wall {1e3 * (t2 - t0) / 3:.2f} ms/step")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(f"gpurun_out/trace_{cname}.json")
