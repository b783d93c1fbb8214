"""GPU time of the router forward and backward (CUDA-graph replays, so no host launch gaps)
at the BASELINE shapes, per path.

    python tools/router_bench.py [tc|gemm] [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_07685_b200 import ops  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "tc"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ops.ROUTER_TC = mode == "tc"
dev = torch.device("cuda:0")
SHAPES = {"mixtral": (16384, 4096, 8, 2, "softmax", False),
          "qwen3": (32768, 4096, 128, 8, "softmax", False),
          "deepseek": (4096, 7168, 256, 8, "sigmoid", True)}
for name, (T, h, E, K, score, bias) in SHAPES.items():
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((T, h), device=dev, generator=g).to(torch.bfloat16)
    w_r = (torch.randn((h, E), device=dev, generator=g) * h ** -0.5).to(torch.bfloat16)
    sb = torch.rand((E,), device=dev, generator=g) * 0.05 if bias else None
    dprob = torch.randn((T, K), device=dev, generator=g)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            r = ops.router_forward(x, w_r, K, score, sb, 1e-2)
            ops.router_backward(x, None, r, dprob, score, aux_scale=1.0)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf):
        r = ops.router_forward(x, w_r, K, score, sb, 1e-2)
    with torch.cuda.graph(gb):
        ops.router_backward(x, None, r, dprob, score, aux_scale=1.0)
    res = {}
    for k, gr in (("fwd", gf), ("bwd", gb)):
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(iters):
            gr.replay()
        b.record()
        torch.cuda.synchronize()
        res[k] = a.elapsed_time(b) / iters * 1e3
    xb = T * h * 2
    print(f"{name:9s} {mode}: fwd {res['fwd']:7.1f} us ({xb / res['fwd'] / 1e6:5.2f} TB/s on x, "
          f"{xb / res['fwd'] / 1e6 / 6.5478:.2f} of HBM)  bwd {res['bwd']:7.1f} us", flush=True)
