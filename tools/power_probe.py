"""Energy per FLOP of each expert GEMM kind (Mixtral shape, CTA-pair engine) next to cuBLAS:
each kind runs back to back for ~2 s while NVML samples power and SM clock.

    python tools/power_probe.py
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

sys.argv = [sys.argv[0], os.environ.get("POWER_CONFIG", "mixtral"), "none"]
import gemm_kinds as G  # noqa: E402  (tools/ on sys.path via the script dir)

pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)


def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetPowerUsage(hdl) / 1e3,
                    pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM)))
        time.sleep(0.02)


def measure(fn, flops, seconds=2.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n = 0
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    stop, samples = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, samples))
    t0 = time.time()
    s.record()
    th.start()
    while time.time() - t0 < seconds:
        fn()
        n += 1
        if n % 4 == 0:
            torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / n
    tail = samples[len(samples) // 3:]  # steady state
    p = sum(x[0] for x in tail) / max(len(tail), 1)
    clk = sorted(x[1] for x in tail)[len(tail) // 2] if tail else 0
    tf = flops / (ms / 1e3) / 1e12
    return ms, tf, p, clk


res = {}
only = os.environ.get("POWER_KINDS")
for k, fn in G.fns.items():
    if only and k not in only.split(","):
        continue
    ms, tf, p, clk = measure(fn, G.flop[k])
    print(f"{k:10s} {ms:7.3f} ms {tf:7.1f} TF/s  {p:6.0f} W  {clk:5d} MHz  "
          f"{p / tf:5.3f} W per TF/s  {tf / clk * 1e3:6.1f} GF/s per MHz", flush=True)
if os.environ.get("POWER_NO_CUBLAS"):
    sys.exit(0)
a = torch.randn((8192, 8192), device="cuda", dtype=torch.bfloat16)
b = torch.randn((8192, 8192), device="cuda", dtype=torch.bfloat16)
ms, tf, p, clk = measure(lambda: a @ b, 2.0 * 8192 ** 3)
print(f"{'cublas':10s} {ms:7.3f} ms {tf:7.1f} TF/s  {p:6.0f} W  {clk:5d} MHz  "
      f"{p / tf:5.3f} W per TF/s  {tf / clk * 1e3:6.1f} GF/s per MHz", flush=True)
