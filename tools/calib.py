"""Same-box calibration under the power cap: cuBLAS bf16 8192^3 vs our grouped GEMM
(1-CTA and CTA-pair engines) at the Mixtral fc1 shape, each looped for ~4 s with the SM
clock sampled by nvidia-smi. Prints TFLOP/s, median clock and TFLOP/s per GHz."""
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_07685_b200 import gemm  # noqa: E402


def sample(fn, flops, seconds=4.0):
    lines = []
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "100", "-i", "0"],
                         stdout=subprocess.PIPE, text=True)
    th = threading.Thread(target=lambda: [lines.append(x) for x in p.stdout], daemon=True)
    th.start()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    time.sleep(0.5)
    lines.clear()
    n = 0
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    t0 = time.time()
    while time.time() - t0 < seconds:
        for _ in range(5):
            fn()
        n += 5
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    p.terminate()
    ms = s.elapsed_time(e) / n
    clk = [float(x.split(",")[0]) for x in lines if x.strip()]
    pw = [float(x.split(",")[1]) for x in lines if x.strip()]
    mhz = statistics.median(clk) if clk else float("nan")
    tf = flops / ms / 1e9
    return tf, mhz, (statistics.median(pw) if pw else float("nan"))


dev = torch.device("cuda:0")
a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
res = {}
res["cublas_8192"] = sample(lambda: a @ b, 2 * 8192 ** 3)
del a, b

E, h, m = 8, 4096, 14336
rows_per = 4096
for pair in (False, True):
    align = 256 if pair else 128
    rows = E * rows_per
    be = torch.repeat_interleave(torch.arange(E, dtype=torch.int32), rows_per // 128).to(dev)
    nmb = torch.tensor([rows // 128], dtype=torch.int32, device=dev)
    xp = torch.randn((rows, h), device=dev, dtype=torch.bfloat16)
    w1 = (torch.randn((E, 2 * m, h), device=dev) * h ** -0.5).to(torch.bfloat16)
    pre = torch.empty((rows, 2 * m), device=dev, dtype=torch.bfloat16)
    act = torch.empty((rows, m), device=dev, dtype=torch.bfloat16)
    fl = 2.0 * rows * h * 2 * m
    res[f"fc1_fwd_{'pair' if pair else 'cta1'}"] = sample(
        lambda: gemm.fc1_fwd(xp, w1, be, nmb, preact=pre, act=act, pair=pair), fl)
    offs = torch.arange(E + 1, dtype=torch.int32, device=dev) * rows_per
    res[f"fc1_wgrad_{'pair' if pair else 'cta1'}"] = (None,) if not pair else sample(
        lambda: gemm.wgrad(pre, xp, offs, E), fl)
    del xp, w1, pre, act
for k, v in res.items():
    if v[0] is None:
        continue
    tf, mhz, pw = v
    print(f"{k:18s} {tf:8.1f} TFLOP/s  {mhz:6.0f} MHz  {pw:6.0f} W  {tf / mhz * 1000:7.1f} TFLOP/s/GHz")
