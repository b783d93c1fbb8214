"""Event-timed bandwidth of the HBM-bound data-movement kernels at the BASELINE shapes:
permute gather (x -> expert-major rows), combine (rows -> y), combine backward.

    python tools/hbm_probe.py [iters]      (MOE_B200_GATHER_TMA=0|1 selects the gather)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_07685_b200 import ops  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda:0")
HBM = 6540.8
for name, (E, K, h, T) in {"mixtral": (8, 2, 4096, 16384), "qwen3": (128, 8, 4096, 32768),
                           "deepseek": (256, 8, 7168, 4096)}.items():
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((T, h), device=dev, generator=g).to(torch.bfloat16)
    w_r = (torch.randn((h, E), device=dev, generator=g) * h ** -0.5).to(torch.bfloat16)
    r = ops.router_forward(x, w_r, K, "softmax")
    plan = ops.build_plan(r.topk_idx, r.topk_prob, E, -1, False, align=ops.pick_align(T, K, E))
    xp = ops.permute_gather(x, plan)
    o = torch.randn_like(xp)
    y = torch.empty_like(x)
    dy = torch.randn_like(x)
    d_rows = torch.empty_like(xp)
    R, w = T * K, 2
    cases = {
        "permute_gather": (lambda: ops.permute_gather(x, plan, out=xp), T * h * w + R * h * w),
        "combine": (lambda: ops.combine(o, plan, r.topk_prob, out=y), R * h * w + T * h * w),
        "combine_bwd": (lambda: ops.combine_backward(dy, plan, o, r.topk_prob, d_rows=d_rows),
                        T * h * w + 2 * R * h * w),
        # the dX combine: unweighted row sum + the router dX (`extra`), as in the backward
        "combine_dx": (lambda: ops.combine(o, plan, None, extra=dy, out=y),
                       R * h * w + 2 * T * h * w),
    }
    for k, (fn, nbytes) in cases.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        gbs = nbytes / (ms / 1e3) / 1e9
        print(f"{name:9s} {k:15s} {ms * 1e3:8.1f} us {nbytes / 1e6:8.1f} MB {gbs:7.0f} GB/s "
              f"({gbs / HBM:.2f} of measured HBM)", flush=True)

# reference points for the write-heavy / read-heavy kernels above: torch's own write-only
# (zero_), read-only (sum) and copy kernels over 2 GiB
buf = torch.empty((1 << 30,), dtype=torch.bfloat16, device=dev)
buf2 = torch.empty_like(buf)
for k, (fn, nbytes) in {"write_only": (lambda: buf.zero_(), buf.numel() * 2),
                        "read_only": (lambda: buf.sum(), buf.numel() * 2),
                        "copy": (lambda: buf2.copy_(buf), buf.numel() * 4)}.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    gbs = nbytes / (ms / 1e3) / 1e9
    print(f"torch     {k:15s} {ms * 1e3:8.1f} us {nbytes / 1e6:8.1f} MB {gbs:7.0f} GB/s "
          f"({gbs / HBM:.2f} of measured HBM)", flush=True)
