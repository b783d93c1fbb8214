"""Time each bf16 expert GEMM of the Mixtral-shape layer on the engine bench.py uses
(256-row CTA-pair plan), and optionally run only one kind (a short ncu target).

    python tools/gemm_kinds.py [mixtral|qwen3|deepseek] [kind|all] [iters]
kinds: fc1_fwd fc2_fwd fc2_dgrad fc1_dgrad fc2_wgrad fc1_wgrad
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_07685_b200 import gemm, ops  # noqa: E402

SHAPES = {"mixtral": (8, 2, 4096, 14336, 16384), "qwen3": (128, 8, 4096, 1536, 32768),
          "deepseek": (256, 8, 7168, 2048, 4096)}
name = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
only = sys.argv[2] if len(sys.argv) > 2 else "all"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
E, K, h, m, T = SHAPES[name]
dev = torch.device("cuda:0")
R = T * K
align = ops.pick_align(T, K, E)
pair = align == 256
counts = [R // E] * E
if os.environ.get("GEMM_KINDS_COUNTS") == "random":
    # per-expert counts of seeded uniform top-K routing (K distinct experts per token), as
    # the bench step sees them (DeepSeek: 128 +- 11 rows; 128-row padding doubles about half)
    gen = torch.Generator().manual_seed(0)
    sel = torch.rand((T, E), generator=gen).topk(K, dim=1).indices
    counts = torch.bincount(sel.flatten(), minlength=E).tolist()
offs, be = [0], []
for e, c in enumerate(counts):
    nb = (c + align - 1) // align * (align // 128)
    be += [e] * nb
    offs.append(offs[-1] + nb * 128)
rows = offs[-1]
be_t = torch.tensor(be, dtype=torch.int32, device=dev)
nmb = torch.tensor([len(be)], dtype=torch.int32, device=dev)
offs_t = torch.tensor(offs, dtype=torch.int32, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
xp = torch.randn((rows, h), device=dev, generator=g).to(torch.bfloat16)
w1 = (torch.randn((E, 2 * m, h), device=dev, generator=g) / h ** 0.5).to(torch.bfloat16)
w2 = (torch.randn((E, h, m), device=dev, generator=g) / m ** 0.5).to(torch.bfloat16)
dout = torch.randn((rows, h), device=dev, generator=g).to(torch.bfloat16)
preact, act = gemm.fc1_fwd(xp, w1, be_t, nmb, pair=pair)
out = torch.empty((rows, h), device=dev, dtype=torch.bfloat16)
dpre = torch.empty((rows, 2 * m), device=dev, dtype=torch.bfloat16)
dx = torch.empty((rows, h), device=dev, dtype=torch.bfloat16)
dw2 = torch.empty((E, h, m), device=dev, dtype=torch.bfloat16)
dw1 = torch.empty((E, 2 * m, h), device=dev, dtype=torch.bfloat16)
gemm.fc2_dgrad(dout, w2, preact, be_t, nmb, d_preact=dpre, pair=pair)

fns = {
    "fc1_fwd": lambda: gemm.fc1_fwd(xp, w1, be_t, nmb, preact=preact, act=act, pair=pair),
    "fc2_fwd": lambda: gemm.fc2_fwd(act, w2, be_t, nmb, out=out, pair=pair),
    "fc2_dgrad": lambda: gemm.fc2_dgrad(dout, w2, preact, be_t, nmb, d_preact=dpre, pair=pair),
    "fc1_dgrad": lambda: gemm.fc1_dgrad(dpre, w1, be_t, nmb, out=dx, pair=pair),
    "fc2_wgrad": lambda: gemm.wgrad(dout, act, offs_t, E, out=dw2),
    "fc1_wgrad": lambda: gemm.wgrad(dpre, xp, offs_t, E, out=dw1),
}
flop = {"fc1_fwd": 4.0 * R * h * m, "fc2_fwd": 2.0 * R * h * m, "fc2_dgrad": 2.0 * R * h * m,
        "fc1_dgrad": 4.0 * R * h * m, "fc2_wgrad": 2.0 * R * h * m, "fc1_wgrad": 4.0 * R * h * m}


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


res = {}
for k, fn in fns.items():
    if only not in ("all", k):
        continue
    ms = timeit(fn)
    res[k] = {"ms": round(ms, 4), "tflops": round(flop[k] / ms / 1e9, 1)}
    print(f"{name} {k:10s} {ms:8.3f} ms {flop[k] / ms / 1e9:8.1f} TFLOP/s", flush=True)
print(json.dumps({"shape": name, "pair": pair, "res": res}))
