"""Router chain timing (forward: logits + score/top-k + finalize; backward: score Jacobian +
dW_r + router dX) per C-ABI call on three paths: "tc" (the default small-N tensor-core router,
csrc/router_tc.cu), "gemm" (round-1: logits GEMM padded to 256 columns + warp-per-token top-k)
and "small" (CUDA-core, E <= 16).

    python tools/router_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_07685_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda:0")
SHAPES = {"mixtral": (16384, 4096, 8, 2), "mixtral_T32k": (32768, 4096, 8, 2),
          "e16": (16384, 4096, 16, 4), "qwen3": (32768, 4096, 128, 8),
          "deepseek": (4096, 7168, 256, 8)}


def run(T, h, E, K, mode, iters=20):
    ops.ROUTER_TC = mode == "tc"
    ops.ROUTER_SMALL = mode == "small"
    small = mode != "gemm"
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((T, h), device=dev, generator=g).to(torch.bfloat16)
    w_r = (torch.randn((h, E), device=dev, generator=g) * h ** -0.5).to(torch.bfloat16)
    dprob = torch.randn((T, K), device=dev, generator=g)

    def step():
        w_t, w_pad = (None, None) if small else ops.stage_router_weight(w_r)
        r = ops.router_forward(x, w_r, K, "softmax", None, 1e-2, w_r_t=w_t)
        ops.router_backward(x, w_pad, r, dprob, "softmax", aux_scale=1.0)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    _lib.stats.timing = True
    _lib.stats.events = []
    for _ in range(iters):
        step()
    torch.cuda.synchronize()
    _lib.stats.timing = False
    per = {}
    for nm, s, e in _lib.stats.events:
        per[nm] = per.get(nm, 0.0) + s.elapsed_time(e) / iters
    tot = sum(per.values())
    xbytes = T * h * 2
    # compulsory HBM bytes of the chain: x read in the forward and in dW_r, dX written (bf16)
    alg = 2 * xbytes + xbytes
    print(f"T={T} h={h} E={E} K={K} {mode}: {tot * 1e3:8.1f} us "
          f"(alg {alg / 1e6:.0f} MB -> {alg / (tot / 1e3) / 1e12:.2f} TB/s) "
          + " ".join(f"{k}={v * 1e3:.1f}" for k, v in sorted(per.items(), key=lambda kv: -kv[1])),
          flush=True)


for name, (T, h, E, K) in SHAPES.items():
    run(T, h, E, K, "tc")
    run(T, h, E, K, "gemm")
    if E <= 16:
        run(T, h, E, K, "small")
