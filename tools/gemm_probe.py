"""Time the grouped GEMMs at the Mixtral-shape layer (one GPU, all 8 experts)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_07685_b200 import gemm

dev = torch.device("cuda:0")
E, K, h, m, T = 8, 2, 4096, 14336, 16384
if len(sys.argv) > 1 and sys.argv[1] == "qwen":
    E, K, h, m, T = 128, 8, 4096, 1536, 32768
if len(sys.argv) > 1 and sys.argv[1] == "deepseek":
    E, K, h, m, T = 256, 8, 7168, 2048, 4096
R = T * K
counts = [R // E] * E
offs = [0]
be = []
for e, c in enumerate(counts):
    nb = (c + 127) // 128
    be += [e] * nb
    offs.append(offs[-1] + nb * 128)
rows = offs[-1]
be_t = torch.tensor(be, dtype=torch.int32, device=dev)
nmb = torch.tensor([len(be)], dtype=torch.int32, device=dev)
offs_t = torch.tensor(offs, dtype=torch.int32, device=dev)
xp = torch.randn((rows, h), device=dev, dtype=torch.bfloat16)
w1 = (torch.randn((E, 2 * m, h), device=dev) / h ** 0.5).to(torch.bfloat16)
w2 = (torch.randn((E, h, m), device=dev) / m ** 0.5).to(torch.bfloat16)
dout = torch.randn((rows, h), device=dev, dtype=torch.bfloat16)

def timeit(fn, iters=10):
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

preact, act = gemm.fc1_fwd(xp, w1, be_t, nmb)
res = {}
flop_fc1 = 2.0 * rows * h * 2 * m
flop_fc2 = 2.0 * rows * m * h
res["fc1_fwd"] = timeit(lambda: gemm.fc1_fwd(xp, w1, be_t, nmb, preact=preact, act=act))
out = gemm.fc2_fwd(act, w2, be_t, nmb)
res["fc2_fwd"] = timeit(lambda: gemm.fc2_fwd(act, w2, be_t, nmb, out=out))
dpre, _ = gemm.fc2_dgrad(dout, w2, preact, be_t, nmb)
res["fc2_dgrad"] = timeit(lambda: gemm.fc2_dgrad(dout, w2, preact, be_t, nmb, d_preact=dpre))
dx = gemm.fc1_dgrad(dpre, w1, be_t, nmb)
res["fc1_dgrad"] = timeit(lambda: gemm.fc1_dgrad(dpre, w1, be_t, nmb, out=dx))
dw2 = gemm.wgrad(dout, act, offs_t, E)
res["fc2_wgrad"] = timeit(lambda: gemm.wgrad(dout, act, offs_t, E, out=dw2))
dw1 = gemm.wgrad(dpre, xp, offs_t, E)
res["fc1_wgrad"] = timeit(lambda: gemm.wgrad(dpre, xp, offs_t, E, out=dw1))
fl = {"fc1_fwd": flop_fc1, "fc2_fwd": flop_fc2, "fc2_dgrad": flop_fc2, "fc1_dgrad": flop_fc1,
      "fc2_wgrad": flop_fc2, "fc1_wgrad": flop_fc1}
for k, v in res.items():
    print(f"{k:10s} {v:8.3f} ms  {fl[k] / v / 1e9:8.1f} TFLOP/s")
# cuBLAS comparator on one expert's dense GEMM (context only)
a = xp[: counts[0]]
wt = w1[0]
t = timeit(lambda: a @ wt.T)
print(f"cublas e0 fc1 {t:.3f} ms {2.0 * a.shape[0] * h * 2 * m / t / 1e9:.1f} TFLOP/s")
