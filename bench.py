#!/usr/bin/env python
"""Benchmark: MoE layer fwd+bwd tokens/s & grouped-GEMM TFLOPS on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config mixtral]
    python bench.py --impl reference ...      # the reference CPU path (oracle port)

N>1 is launched by torchrun (one rank per GPU, NCCL): expert parallelism over the
N ranks with T tokens per GPU (weak scaling). One step = router -> permute ->
grouped-GEMM SwiGLU experts -> combine forward + the full backward, on one batch of
synthetic tokens already resident in HBM. Prints ONE JSON line on rank 0.

The ``e2e`` number repeats the step through the public layer API with the step's
inputs (x, dY) copied from pinned host memory and the loss read back every step.
The ``cpu_baseline`` (rank 0, N=1) times the oracle port (oracle/backward_ref.py,
numpy fp32, all host threads) on a bounded token sample of the same layer.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # BASELINE.json configs[1]: the metric's workload (fits one GPU at EP=1)
    "mixtral": dict(E=8, K=2, h=4096, m=14336, T=16384, score="softmax",
                    name="Mixtral-8x7B-shape MoE layer"),
    "qwen3": dict(E=128, K=8, h=4096, m=1536, T=32768, score="softmax",
                  name="Qwen3-235B-shape MoE layer"),
    "deepseek": dict(E=256, K=8, h=7168, m=2048, T=4096, score="sigmoid", shared=2048,
                     name="DeepSeek-V3-shape MoE layer (+1 shared expert)"),
    "capacity": dict(E=8, K=2, h=4096, m=14336, T=16384, score="softmax", cf=1.0, pad=True,
                     name="Mixtral-shape, capacity factor 1.0 drop-and-pad"),
    "tiny": dict(E=8, K=2, h=256, m=512, T=4096, score="softmax", name="tiny MoE layer"),
    "skewed": dict(E=8, K=2, h=4096, m=14336, T=16384, score="softmax", skew=1.0,
                   name="Mixtral-shape, dropless, skewed router (ECHO target)"),
}
AUX_COEFF = 1e-2
METRIC = "MoE layer fwd+bwd tokens/s & grouped-GEMM TFLOPS at 1/2/4/8 B200 (EP)"


def flops_per_token(c) -> float:
    """Algorithmic fwd+bwd FLOPs per token: 18*K*h*m routed, 18*h*m_s shared,
    6*h*E router."""
    return 18.0 * c["K"] * c["h"] * c["m"] + 18.0 * c["h"] * c.get("shared", 0) + 6.0 * c["h"] * c["E"]


def gemm_flops_per_token(c) -> float:
    return 18.0 * c["K"] * c["h"] * c["m"] + 18.0 * c["h"] * c.get("shared", 0)


# ----------------------------------------------------------------------------- clocks
class NvmlClockSampler:
    """In-process NVML sampling of the same fields nvidia-smi's clocks line reports (SM clock,
    max SM clock, clock-event reasons), every 20 ms inside the timed window. NVML is the
    library nvidia-smi itself calls; reading it directly timestamps every sample inside the
    window (a polling nvidia-smi process delivered lines late through its pipe)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int = 0):
        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        self.samples: list[tuple[float, int, int, int]] = []
        self.t0 = self.t1 = None
        self.lines = [True]  # started immediately (ClockSampler interface)
        self._stop = threading.Event()
        self._reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        self.t = threading.Thread(target=self._run, daemon=True)

    def start(self):
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            if self.t0 is not None and self.t1 is None:
                try:
                    sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                    rs = self._reasons(self.h)
                    self.samples.append((time.time(), sm, smax, rs))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(0.02)
            else:
                time.sleep(0.005)

    def window(self, start: bool):
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self) -> dict:
        self._stop.set()
        self.t.join(timeout=2)
        sm = [x[1] for x in self.samples]
        smax = [x[2] for x in self.samples]
        reasons = sorted({nm for x in self.samples for nm, bit in self.REASONS.items()
                          if x[3] & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(sm), "source": "NVML (nvidia-smi's library), every 20 ms"}


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md).

    Each sample carries nvidia-smi's own timestamp; only samples inside the timed window
    [window(start), window(end)] count (the pipe may deliver lines late, and samples from
    idle set-up phases must not enter the median)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int = 0):
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.gpu = gpu_index
        self.t0 = self.t1 = None

    def start(self):
        import shutil

        ms = os.environ.get("MOE_BENCH_SMI_MS", "100")
        if ms == "0" or os.environ.get("MOE_BENCH_CLOCKS") == "0":
            return
        cmd = ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
               "-i", str(self.gpu), "-lms", ms]
        if shutil.which("stdbuf"):
            cmd = ["stdbuf", "-oL"] + cmd
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def window(self, start: bool):
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    @staticmethod
    def _stamp(s: str):
        import datetime

        for fmt in ("%Y/%m/%d %H:%M:%S.%f", "%Y/%m/%d %H:%M:%S"):
            try:
                return datetime.datetime.strptime(s, fmt).timestamp()
            except ValueError:
                pass
        return None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)  # let the samples of the window's tail arrive
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for arrived, ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 10:
                continue
            ts = self._stamp(parts[0])
            if ts is None:
                ts = arrived
            if self.t0 is not None and not (self.t0 <= ts <= (self.t1 or ts)):
                continue
            try:
                sm.append(float(parts[2]))
                smax.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[6:10]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_baseline(c, sample_tokens: int, threads: int, reps: int = 1) -> dict:
    """Oracle port (numpy fp32) fwd+bwd of the same layer on `sample_tokens` tokens."""
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    import numpy as np

    from oracle import backward_ref as B
    from oracle import routing_ref as R

    rng = np.random.default_rng(0)
    h, m, e, k = c["h"], c["m"], c["E"], c["K"]
    f32 = np.float32
    x = rng.standard_normal((sample_tokens, h), dtype=f32)
    w_r = (rng.standard_normal((h, e), dtype=f32) * h ** -0.5).astype(f32)
    # every expert has its own weights (the layer's full parameter set, E x 3 x m x h fp32)
    # up to 8 GB of host memory; beyond that (DeepSeek shape: 45 GB) the experts share one
    # set -- same FLOPs per expert, stated in the sample description
    def expert_w(shape, fan_in):
        return (rng.standard_normal(shape, dtype=f32) * fan_in ** -0.5).astype(f32)

    distinct = e * 3 * m * h * 4 <= 8e9
    nw = e if distinct else 1
    up = [expert_w((m, h), h) for _ in range(nw)]
    w2 = [expert_w((h, m), m) for _ in range(nw)]
    gate = [expert_w((m, h), h) for _ in range(nw)]
    params = R.ExpertParams(w1=(up if distinct else up * e), w2=(w2 if distinct else w2 * e),
                            gate=(gate if distinct else gate * e))
    dy = rng.standard_normal((sample_tokens, h), dtype=f32)
    def one_step() -> float:
        t0 = time.perf_counter()
        B.moe_forward_backward(x, w_r, params, dy, score=c["score"], top_k=k, coeff=AUX_COEFF)
        return time.perf_counter() - t0

    times = [one_step() for _ in range(reps)]
    best = min(times)
    return {"value": sample_tokens / best, "unit": "tokens/s", "cores": threads,
            "kind": "port", "seconds": best, "times": times, "step": one_step,
            "sample": (f"{sample_tokens} tokens of the {c['name']} (E={e},K={k},h={h},m={m}, "
                       + (f"all {e} experts' own weights" if distinct else
                          "experts sharing one weight set (host memory)")
                       + "), fwd+bwd, oracle/backward_ref.py "
                       f"(the pinned numpy restatement of moelab.routing + its analytic "
                       f"backward) fp32, best of {reps}")}


def gemm_traffic(config: str, n: int):
    """DRAM bytes of the routed grouped-GEMM launches of one step (ncu --metrics pass over
    tools/layer_step.py, reduced by tools/step_traffic.py into profiles/), next to their
    algorithmic bytes. EP=1 captures only (the per-rank GEMMs at EP>1 see the same shapes
    per expert but fewer experts)."""
    if n != 1:
        return None
    f = ROOT / "profiles" / f"r02_step_traffic_{config}.json"
    if not f.exists():
        return None
    d = json.loads(f.read_text())
    g = d["routed_gemm_traffic"]
    tot = sum(v["traffic_GB"] for v in g.values())
    alg = sum(v["algorithmic_GB"] for v in g.values())
    return {"bytes": int(tot * 1e9), "bytes_per_launch": int(tot * 1e9 / max(len(g), 1)),
            "algorithmic_bytes": int(alg * 1e9), "ratio": round(tot / alg, 2),
            "per_gemm_GB": {k: v["traffic_GB"] for k, v in g.items()},
            "source": f"profiles/{f.name} (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                      "one step of tools/layer_step.py)"}


def gemm_floor_model(c, n: int, per_kernel: dict, steps: int, peak_tf: float, hbm_gbs: float):
    """Per-GEMM roofline floor of one step: each expert GEMM kind's time floor is
    max(FLOPs / sustained tensor peak, compulsory bytes / copy bandwidth), with the compulsory
    bytes of SURVEY §8(d) (operands read once, outputs written once, bf16; routed experts E/n
    per rank with T*K rows, plus the shared expert as one T-row group). Decides the GEMM set's
    bound: Mixtral/Qwen3 are tensor-bound, DeepSeek's 128-row-per-expert GEMMs stream
    15 GB of fc1 weights per pass and are HBM-bound at EP=1."""
    w = 2
    groups = [(c["E"] // n, c["T"] * c["K"], c["m"])]
    if c.get("shared"):
        groups.append((1, c["T"], c["shared"]))
    h = c["h"]
    kinds = {}
    for el, r, m in groups:
        per = {  # (flops, bytes)
            "fc1_fwd": (4.0 * r * h * m, r * h * w + el * 2 * m * h * w + r * 3 * m * w),
            "fc2_fwd": (2.0 * r * h * m, r * m * w + el * h * m * w + r * h * w),
            "fc2_dgrad": (2.0 * r * h * m, r * h * w + el * h * m * w + r * 4 * m * w),
            "fc1_dgrad": (4.0 * r * h * m, r * 2 * m * w + el * 2 * m * h * w + r * h * w),
            "wgrad": (6.0 * r * h * m, el * 3 * h * m * w + 2 * r * h * w + 3 * r * m * w),
        }
        for k, (f, b) in per.items():
            a = kinds.setdefault(k, [0.0, 0.0, 0.0])
            a[0] += f
            a[1] += b
            a[2] += max(f / (peak_tf * 1e12), b / (hbm_gbs * 1e9)) * 1e3
    out, floor_ms, meas_ms, t_ms, m_ms = {}, 0.0, 0.0, 0.0, 0.0
    for k, (f, b, fl) in kinds.items():
        ms = sum(sum(v) for nm, v in per_kernel.items()
                 if k in nm and nm.startswith("moe_gg_") and not nm.endswith("_f32")) / steps
        tt, tm = f / (peak_tf * 1e12) * 1e3, b / (hbm_gbs * 1e9) * 1e3
        out[k] = {"TFLOP": round(f / 1e12, 3), "GB": round(b / 1e9, 3),
                  "tensor_ms": round(tt, 3), "hbm_ms": round(tm, 3),
                  "bound": "tensor" if tt >= tm else "hbm", "floor_ms": round(fl, 3),
                  "measured_ms": round(ms, 4) if ms else None,
                  "frac_of_floor": round(fl / ms, 3) if ms else None}
        floor_ms += fl
        meas_ms += ms
        t_ms += tt
        m_ms += tm
    return {"per_gemm": out, "floor_ms": round(floor_ms, 3),
            "measured_ms": round(meas_ms, 4) if meas_ms else None,
            "frac_of_floor": round(floor_ms / meas_ms, 3) if meas_ms else None,
            "bound": "tensor" if t_ms >= m_ms else "hbm",
            "tflop": sum(v[0] for v in kinds.values()) / 1e12,
            "bytes": sum(v[1] for v in kinds.values()),
            "assumes": f"tensor peak {peak_tf} TF/s sustained, copy {hbm_gbs} GB/s; "
                       f"{c['E'] // n} routed experts x {c['T'] * c['K']} rows per rank"}


def measure_write_gbs(nbytes: int = 1 << 31, iters: int = 10) -> float:
    """HBM write-only bandwidth of this GPU (torch zero_ over 2 GiB, CUDA events, best of
    `iters`): the bound of write-dominated kernels, which B200 serves well below the copy
    rate (measured ~3.95 TB/s write-only vs ~6.5 TB/s copy, tools/hbm_probe.py)."""
    import torch

    buf = torch.empty((nbytes // 2,), dtype=torch.bfloat16, device="cuda")
    src = torch.ones((1,), dtype=torch.bfloat16, device="cuda").expand(nbytes // 2)
    buf.zero_()
    best = None
    # the best of six write-only kernels: torch's fill with 0 / fill with 1 / broadcast copy
    # (fill alone measured 2.88-3.95 TB/s on different boxes) and the library's probes
    # (16-byte stores, streaming stores, TMA bulk stores of a zeroed smem chunk)
    from paper_2603_07685_b200 import _lib

    lib = _lib.load()

    def probe(mode):
        st = lib.moe_hbm_write_probe(buf.data_ptr(), nbytes, mode,
                                     torch.cuda.current_stream().cuda_stream)
        _lib.check(st, "moe_hbm_write_probe")

    methods = {"torch_zero": lambda: buf.zero_(), "torch_fill": lambda: buf.fill_(1.0),
               "torch_broadcast_copy": lambda: buf.copy_(src), "probe_st16": lambda: probe(0),
               "probe_st16_cs": lambda: probe(1), "probe_tma_bulk": lambda: probe(2)}
    per = {}
    for nm, fn in methods.items():
        for _ in range(iters):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            ms = s.elapsed_time(e)
            best = ms if best is None else min(best, ms)
            per[nm] = min(per.get(nm, ms), ms)
    del buf
    measure_write_gbs.per_method = {k: round(nbytes / (v / 1e3) / 1e9, 1) for k, v in per.items()}
    return nbytes / (best / 1e3) / 1e9


def hbm_kernels(c, per_kernel: dict, steps: int, hbm_gbs: float, write_gbs: float | None = None):
    """Event-timed bandwidth of the HBM-bound data-movement kernels (SURVEY §8(d) bytes):
    permute gather (x read, R rows written), combine (forward y and backward dX), combine
    backward (dY + O rows read, dO rows written), and the small-N router (x read in the
    forward and in dW_r). `frac_of_bound`: the kernel's time floor max(bytes / copy
    bandwidth, written bytes / write-only bandwidth) over its measured time."""
    T, K, h = c["T"], c["K"], c["h"]
    R, w = T * K, 2
    sh = T * h * w if c.get("shared") else 0
    # (algorithmic bytes, of which written)
    alg = {
        "moe_permute_gather": (T * h * w + R * h * w + R * 4, R * h * w),
        # forward: R rows + probs + map read, y written (+ the shared-expert output read);
        # backward dX: R rows + map + the router dX (+ shared-expert dX) read, dX written
        "moe_combine": ((R * h * w + R * 8 + T * h * w + sh)
                        + (R * h * w + R * 4 + T * h * w + sh + T * h * w), 2 * T * h * w),
        "moe_combine_bwd": (T * h * w + 2 * R * h * w + R * 12, R * h * w),
        "moe_router_tc_fwd": (T * h * w + T * c["E"] * 4, T * c["E"] * 4),
        "moe_router_tc_wgrad": (T * h * w, 0),
    }
    out = {}
    for k, (b, wb) in alg.items():
        if k in per_kernel:
            ms = sum(per_kernel[k]) / steps
            gbs = b / (ms / 1e3) / 1e9
            floor_ms = max(b / hbm_gbs, wb / write_gbs if write_gbs else 0.0) / 1e6
            out[k] = {"ms_per_step": round(ms, 4), "algorithmic_MB": round(b / 1e6, 1),
                      "written_MB": round(wb / 1e6, 1),
                      "achieved_GBps": round(gbs, 1), "frac_of_measured_hbm": round(gbs / hbm_gbs, 3),
                      "frac_of_bound": round(floor_ms / ms, 3)}
    return out


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args, c) -> None:
    import torch
    import torch.distributed as dist

    from paper_2603_07685_b200 import _lib, gemm
    from paper_2603_07685_b200.layer import MoEConfig, moe_forward

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = world
    T, E, K, h, m = c["T"], c["E"], c["K"], c["h"], c["m"]
    if E % n:
        raise SystemExit(f"E={E} not divisible by {n} ranks")
    cfg = MoEConfig(E, K, h, m, score=c["score"], aux_loss_coeff=AUX_COEFF,
                    precision=args.precision,
                    capacity_factor=c.get("cf"), pad_to_capacity=c.get("pad", False),
                    shared_ffn_hidden=c.get("shared", 0))
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    bf = torch.bfloat16
    x = torch.randn((T, h), device=dev, generator=g).to(bf)
    dy = torch.randn((T, h), device=dev, generator=g).to(bf)
    gw = torch.Generator(device=dev).manual_seed(99)  # weights identical on every rank
    w_r = (torch.randn((h, E), device=dev, generator=gw) * h ** -0.5).to(bf).requires_grad_()
    skew = args.skew if args.skew is not None else c.get("skew", 0.0)
    if skew:
        # config 5 skewed routing: logits += alpha * b_e, b_e = -log(1+e),
        # exactly, through one constant-1 input feature whose router weights are alpha*b
        x[:, 0] = 1.0
        with torch.no_grad():
            b = -torch.log1p(torch.arange(E, device=dev, dtype=torch.float32)) * skew
            w_r[0, :] = b.to(bf)
    e_loc = E // n
    w1 = (torch.randn((e_loc, 2 * m, h), device=dev, generator=g) * h ** -0.5).to(bf)
    w2 = (torch.randn((e_loc, h, m), device=dev, generator=g) * m ** -0.5).to(bf)
    w1.requires_grad_()
    w2.requires_grad_()
    w1s = w2s = None
    if c.get("shared"):
        ms = c["shared"]
        w1s = (torch.randn((1, 2 * ms, h), device=dev, generator=g) * h ** -0.5).to(bf)
        w2s = (torch.randn((1, h, ms), device=dev, generator=g) * ms ** -0.5).to(bf)
        w1s.requires_grad_()
        w2s.requires_grad_()
    params = [w_r, w1, w2] + ([w1s, w2s] if w1s is not None else [])

    if n > 1:
        from paper_2603_07685_b200.dispatcher import EPGroup, moe_forward_ep

        ep = EPGroup(dist.group.WORLD)

        def layer(xx):
            return moe_forward_ep(xx, w_r, w1, w2, cfg, ep, None, w1s, w2s,
                                  transport=args.ep_transport, echo_slots=args.echo_slots,
                                  sync_free=args.sync_free or args.graph)
    else:
        def layer(xx):
            return moe_forward(xx, w_r, w1, w2, cfg, None, w1s, w2s)

    def step(xx, dyy):
        for p in params:
            p.grad = None
        xx = xx.detach().requires_grad_(True)
        y, aux = layer(xx)
        torch.autograd.backward([y, aux], [dyy, torch.ones_like(aux)])
        return y, aux

    def barrier():
        if n > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # nvidia-smi start-up contends with the driver: start sampling before the warm-up and
    # wait for its first sample so the timed region only sees the steady 100 ms polling.
    try:
        if os.environ.get("MOE_BENCH_SMI") == "1" or os.environ.get("MOE_BENCH_CLOCKS") == "0":
            raise ImportError
        clocks = NvmlClockSampler(dev.index if dev.index is not None else 0)
    except Exception:  # noqa: BLE001  (no pynvml / NVML: the nvidia-smi process)
        clocks = ClockSampler(dev.index if dev.index is not None else 0)
    if rank == 0:
        clocks.start()
        t_wait = time.time()
        while not clocks.lines and time.time() - t_wait < 10:
            time.sleep(0.05)
    # Python's cyclic GC can pause the host long enough to drain the GPU queue in the
    # middle of a timed step (seen as isolated 34-43 ms steps in A/B runs whose GEMM time
    # was unchanged): collect once now, keep it off through warm-up and every timed region
    import gc

    gc.collect()
    gc.disable()
    if not args.graph:
        for _ in range(args.warmup):
            step(x, dy)
    barrier()

    run = step
    graph_launches = None
    graph_error = None
    graph_events = None
    if args.graph:
        # whole fwd+bwd step (router, EP planning on the device, exchanges, GEMMs, NCCL
        # all-gather / barriers) captured once and replayed: no host work per step
        # warm-up on a side stream only: eager steps on the legacy default stream before
        # the capture make it fail (cudaErrorStreamCaptureImplicit, measured at EP=1)
        try:
            sx, sdy = x.clone(), dy.clone()
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for _ in range(max(args.warmup, 2)):
                    step(sx, sdy)
            torch.cuda.current_stream().wait_stream(side)
            barrier()
            graph = torch.cuda.CUDAGraph()
            l0 = _lib.stats.launches
            # per-call CUDA events (roofline) captured into the graph as event-record nodes:
            # every replay re-records them, so after the timed region they hold the last
            # timed step's per-kernel durations, measured live
            graph_events = None
            if os.environ.get("MOE_BENCH_KERNEL_EVENTS", "1") != "0":
                _lib.stats.prepare(128, external=True)
                _lib.stats.events = []
                _lib.stats.timing = True
            try:
                with torch.cuda.graph(graph):
                    g_out = step(sx, sdy)
                graph_events = list(_lib.stats.events) if _lib.stats.timing else None
            except Exception:  # noqa: BLE001  (capture again without the event nodes)
                if not _lib.stats.timing:
                    raise
                _lib.stats.timing = False
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    g_out = step(sx, sdy)
            _lib.stats.timing = False
            _lib.stats.events = []
            graph_launches = _lib.stats.launches - l0
            barrier()

            def run(xx, dyy):
                if xx is not sx:
                    sx.copy_(xx, non_blocking=True)
                    sdy.copy_(dyy, non_blocking=True)
                graph.replay()
                return g_out

            x, dy = sx, sdy
            for _ in range(2):
                run(x, dy)
            barrier()
        except Exception as exc:  # noqa: BLE001  (a capture failure falls back to eager)
            if n > 1:
                raise
            graph_error = f"{type(exc).__name__}: {exc}"[:200]
            print(f"bench: CUDA-graph capture failed ({graph_error}); timing eager steps",
                  file=sys.stderr)
            args.graph = False
            run = step
            graph_launches = None
            torch.cuda.synchronize()
            for _ in range(args.warmup):
                step(x, dy)
            barrier()

    # ---- timed region: device-resident inputs ------------------------------------
    if rank == 0:
        clocks.lines.clear()
    _lib.stats.launches = 0
    # per-launch CUDA events ride inside the timed region (the roofline's "achieved" is
    # measured live); MOE_BENCH_KERNEL_EVENTS=0 moves them to an instrumented pass after it
    live_events = os.environ.get("MOE_BENCH_KERNEL_EVENTS", "1") != "0"
    _lib.stats.timing = live_events and not args.graph
    _lib.stats.events = []
    _lib.stats.prepare(64 * args.steps)  # event pairs created before the clock starts
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    clocks.window(True)
    t_start.record()
    for _ in range(args.steps):
        run(x, dy)
    t_end.record()
    barrier()
    clocks.window(False)
    launches = _lib.stats.launches if graph_launches is None else graph_launches * args.steps
    ms_total = t_start.elapsed_time(t_end)
    ev_steps = args.steps  # timed steps the per-kernel events cover
    kernel_events = "live, every timed step"
    if args.graph and graph_events:
        ev = graph_events
        ev_steps = 1
        kernel_events = "live, the last timed step (event-record nodes in the replayed graph)"
    else:
        if args.graph or not live_events:
            # per-kernel timings (roofline) from eager instrumented steps after the timed region
            _lib.stats.prepare(64 * args.steps)
            _lib.stats.timing = True
            for _ in range(args.steps):
                step(x, dy)
            barrier()
            kernel_events = "eager instrumented steps after the timed region"
        ev = _lib.stats.events
    _lib.stats.timing = False
    per_kernel: dict[str, list] = {}
    for nm, s, e in ev:
        per_kernel.setdefault(nm, []).append(s.elapsed_time(e))
    # GEMM busy time: programmatic dependent launches (the split-unit tail, the weight
    # gradients) start while the GEMM before them drains, so their event spans overlap it.
    # Each GEMM interval is clipped at the end of the ones before it (the union of the GEMM
    # intervals, the overlap attributed to the earlier launch): per-kind exclusive times
    gemm_excl: dict[str, list] = {}
    gemm_ms = 0.0
    if ev:
        ref = ev[0][1]
        iv = sorted((ref.elapsed_time(s), ref.elapsed_time(e), nm) for nm, s, e in ev
                    if nm.startswith("moe_gg_"))
        cur = float("-inf")
        for t0_, t1_, nm in iv:
            span = max(0.0, t1_ - max(t0_, cur))
            gemm_excl.setdefault(nm, []).append(span)
            gemm_ms += span
            cur = max(cur, t1_)
    clk = clocks.stop() if rank == 0 else None

    t_tensor = torch.tensor([ms_total, gemm_ms], dtype=torch.float64, device=dev)
    if n > 1:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
    ms_total, gemm_ms_max = t_tensor.tolist()
    ms_step = ms_total / args.steps
    tokens = T * n
    value = tokens / (ms_step / 1e3)

    if args.graph and graph_launches is not None:
        # the e2e region runs the eager public API: release the graph and its private memory
        # pool first (kept alive, it leaves the eager steps short of cached blocks; DeepSeek
        # shape measured 25 ms eager steps instead of 19)
        run = step
        for p_ in params:  # (the captured backward's gradients live in the graph's pool)
            p_.grad = None
        del graph, g_out
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    # ---- e2e: host buffers through the public API ----------------------------------
    # Each step's x and dY come from pinned host memory (H2D on a copy stream, double
    # buffered so step i+1's copy overlaps step i's compute, like a data-loader prefetch);
    # the step's results go back to pinned host memory: the output y (the activation the
    # layer hands on) and the aux loss, D2H on a second copy stream that overlaps the next
    # step. All copies are inside the timed region; the region ends when the last y is on
    # the host.
    x_host = x.cpu().pin_memory()
    dy_host = dy.cpu().pin_memory()
    loss_host = torch.empty((max(args.steps, 2),), dtype=torch.float32).pin_memory()
    y_host = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for _ in range(2)]
    bufs = [(torch.empty_like(x), torch.empty_like(dy)) for _ in range(2)]
    copy_stream = torch.cuda.Stream(device=dev)
    d2h_stream = torch.cuda.Stream(device=dev)
    landed = [torch.cuda.Event() for _ in range(2)]
    released = [torch.cuda.Event() for _ in range(2)]
    main = torch.cuda.current_stream()

    def h2d(slot):
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(released[slot])
            bufs[slot][0].copy_(x_host, non_blocking=True)
            bufs[slot][1].copy_(dy_host, non_blocking=True)
            landed[slot].record(copy_stream)

    def e2e_run(steps):
        for s in range(2):
            released[s].record(main)
        h2d(0)
        for i in range(steps):
            slot = i % 2
            if i + 1 < steps:
                h2d(1 - slot)
            main.wait_event(landed[slot])
            # the public API, eagerly (as a user calls it), whatever the timed region used
            y, aux = step(*bufs[slot])
            released[slot].record(main)
            ev = torch.cuda.Event()
            ev.record(main)
            with torch.cuda.stream(d2h_stream):
                d2h_stream.wait_event(ev)
                yd = y.detach()
                yd.record_stream(d2h_stream)
                y_host[slot].copy_(yd, non_blocking=True)
                loss_host[i].copy_(aux.detach(), non_blocking=True)
        main.wait_stream(d2h_stream)

    e2e_run(2)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    e2e_run(args.steps)
    e1.record()
    barrier()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if n > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())

    # ---- drop-in function API (the reference's moelab.routing surface): numpy in, numpy
    # out, forward only (the reference API has no backward). route() + combine_standard() on
    # this step's x with the same expert weights, host<->device copies included.
    dropin = None
    if n == 1 and not args.no_dropin and c.get("shared", 0) == 0:
        import numpy as np

        from paper_2603_07685_b200 import routing as G

        gate_w, up_w = gemm.split_gate_up(w1.detach())
        params_np = G.ExpertParams(w1=list(up_w.float().cpu().numpy()),
                                   w2=list(w2.detach().float().cpu().numpy()),
                                   gate=list(gate_w.float().cpu().numpy()))
        x_np = x.float().cpu().numpy()
        w_r_np = w_r.detach().float().cpu().numpy()

        def dropin_call():
            dec = G.route(x_np, w_r_np, score=c["score"], top_k=K)
            if cfg.capacity_factor is not None:
                dec = G.apply_capacity(dec, cfg.capacity_factor, pad=cfg.pad_to_capacity)
                return G.moe_output_with_residual(x_np, dec, params_np)
            return G.combine_standard(x_np, dec, params_np)

        dropin_call()  # warm-up: uploads and stacks the expert weights once (then cached)
        times = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            y_np = dropin_call()
            times.append(time.perf_counter() - t0)
        assert isinstance(y_np, np.ndarray) and y_np.shape == (T, h)
        dsec = statistics.median(times)
        dropin = {"value": round(T / dsec, 1), "unit": "tokens/s", "ms_per_call": round(dsec * 1e3, 2),
                  "api": "paper_2603_07685_b200.routing.route + combine_standard (numpy fp32 "
                         "in, float64 out; forward only, as the reference API); host wall clock "
                         "with the host<->device copies, median of 3 after a warm-up call",
                  "h2d_bytes_per_call": int(x_np.nbytes), "d2h_bytes_per_call": int(T * h * 8)}
        del params_np, x_np

    # ---- routing statistics of this workload (global counts; config 5 drop fraction) ----
    from paper_2603_07685_b200 import ops

    with torch.no_grad():
        rr = ops.router_forward(x, w_r.detach(), K, c["score"])
        cnt = rr.counts.to(torch.int64)
        if n > 1:
            allc = torch.empty((n, E), dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(allc, cnt)
            cnt = allc.sum(0)
    cnt = cnt.cpu().double()
    cap_g = cfg.capacity(n * T)
    # ---- NVLink traffic of the EP exchange (exact, from this step's device counts) -------
    nvlink_stats = None
    if n > 1:
        from oracle.routing_ref import a2a_send_volume  # the reference byte model (perf.py:62)

        from paper_2603_07685_b200.dispatcher import exchange_stats_from_device, last_exchange

        if args.sync_free or args.graph:
            exchange_stats_from_device()  # the sync-free forward never read the counts

        ex_names = ("moe_ep_dispatch_push", "moe_ep_combine_pull", "moe_ep_combine_bwd_push",
                    "moe_gather_rows", "moe_ep_dispatch_dedup", "moe_ep_expand_grad",
                    "moe_ep_dispatch_push_dest", "moe_ep_combine_bwd_push_dest")
        ex_ms = sum(sum(v) for k_, v in per_kernel.items() if k_ in ex_names) / ev_steps
        # per step: 4 one-way transfers of this rank's remote rows (x, O, dO, dX); with
        # balanced routing each direction of the NVLink port carries ~4 x sent bytes
        out_bytes = 2 * last_exchange["bytes_sent_remote"] + 2 * last_exchange["bytes_recv_remote"]
        tr = args.ep_transport
        if tr == "auto":
            tr = "p2p"
        # p2p: the two return transfers (O, dX) run inside the fc2 / fc1-dgrad epilogues,
        # so only the two pushes (x, dO) are standalone exchange kernels
        standalone_bytes = (2 * last_exchange["bytes_sent_remote"] if tr in ("p2p", "p2p_overlap")
                            else out_bytes)
        nvlink_stats = {
            "transport": tr,
            "bytes_out_per_step_per_gpu": out_bytes,
            "model_bytes_per_step_per_gpu": 4 * a2a_send_volume(T, K, h, n, 2),
            "exchange_kernel_ms_per_step": round(ex_ms, 4),
            "returns_fused_in_gemm_epilogue": tr in ("p2p", "p2p_overlap"),
            "dispatch_overlapped_with_gemm": tr == "p2p_overlap",
            "achieved_GBps_per_direction": (round(standalone_bytes / (ex_ms / 1e3) / 1e9, 1)
                                            if ex_ms and tr in ("p2p", "p2p_overlap", "p2p_pull")
                                            else None),
            "note": ("p2p_dedup sends one row per (token, rank): fewer bytes than counted here"
                     if tr == "p2p_dedup" else None),
            "peak_GBps_per_direction": 770.0,
            "peak_source": "B200_PROFILING.md measured peer copy (nominal 900)",
        }
    routing_stats = {
        "skew_alpha": skew,
        "max_over_mean_expert_load": round(float(cnt.max() / cnt.mean()), 4),
        "capacity_per_expert": cap_g if cap_g >= 0 else None,
        "drop_fraction": (round(float(1 - cnt.clamp(max=cap_g).sum() / cnt.sum()), 5)
                          if cap_g >= 0 else 0.0),
    }

    if rank == 0:
        peaks = {}
        pk = ROOT / "MEASURED_PEAKS.json"
        if pk.exists():
            peaks = json.loads(pk.read_text())
        # the GEMMs run back to back inside a long step under the 1 kW cap: sustained peak
        peak_tf = peaks.get("bf16_tflops_sustained", 1400.0)
        peak_src = ("measured sustained cuBLAS bf16 (MEASURED_PEAKS.json bf16_tflops_sustained)"
                    if peaks else "fallback ~1.4 PF sustained (B200_PROFILING.md)")
        gemm_flops_step = gemm_flops_per_token(c) * T  # per rank
        burst_tf = peaks.get("bf16_tflops", 1590.0)
        hbm_gbs = peaks.get("hbm_gbs", 6650.0)
        traffic = gemm_traffic(args.config, n)
        write_gbs = measure_write_gbs()
        hbm = hbm_kernels(c, per_kernel, ev_steps, hbm_gbs, write_gbs)
        hbm["_peaks"] = {"copy_GBps": hbm_gbs, "write_only_GBps": round(write_gbs, 1),
                         "copy_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
                         "write_source": "measured in this run (best of torch zero_ / fill_ / "
                                         "broadcast copy and moe_hbm_write_probe's 16-byte, "
                                         "streaming and TMA bulk stores, over 2 GiB)",
                         "write_GBps_by_method": getattr(measure_write_gbs, "per_method", None)}
        gemm_tflops = gemm_flops_step * ev_steps / (gemm_ms / 1e3) / 1e12 if gemm_ms else None
        floor = gemm_floor_model(c, n, gemm_excl, ev_steps, peak_tf, hbm_gbs)
        # an HBM-bound GEMM set (DeepSeek at EP=1) reports compulsory bytes over its time
        hbm_ach = (floor.pop("bytes") / (floor["measured_ms"] / 1e3) / 1e9
                   if floor["measured_ms"] else None)
        floor.pop("tflop")
        gemm_launches = sum(len(v) for k_, v in per_kernel.items() if k_.startswith("moe_gg_"))
        out = {
            "metric": METRIC,
            "value": round(value, 1),
            "unit": "tokens/s",
            "n_gpus": n,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": ("bf16" if args.precision == "bf16" else
                      "mxfp8 (all six expert GEMMs: E4M3 with 1x32 E8M0 block scales)"),
            "data": "synthetic (seeded N(0,1) tokens, N(0,1/fan_in) random-init weights)",
            "config": {
                "workload": f"{c['name']}: E={E}, top-{K}, h={h}, ffn={m}, {T} tokens/GPU, "
                            f"{c['score']} router, aux coeff {AUX_COEFF}"
                            + (f", shared expert {c['shared']}" if c.get("shared") else "")
                            + (f", capacity factor {c['cf']} pad" if c.get("cf") else ", dropless")
                            + (f", router skew alpha {skew} (b_e = -log(1+e))" if skew else ""),
                "global_batch": tokens,
                "tokens_per_gpu": T,
                "parallelism": f"ep{n}",
                "ep_transport": args.ep_transport if n > 1 else None,
                "cuda_graph": bool(args.graph),
                "cuda_graph_error": graph_error,
                "sync_free": bool(args.sync_free or args.graph) if n > 1 else None,
                "l2": "inputs larger than L2 (x alone is "
                      f"{T * h * 2 / 1e6:.0f} MB; expert weights {E * 3 * h * m * 2 / 1e9:.2f} GB)",
            },
            "grouped_gemm_tflops": round(gemm_tflops, 1) if gemm_tflops else None,
            "layer_tflops": round(flops_per_token(c) * tokens / (ms_step / 1e3) / 1e12 / n, 1),
            "roofline": {
                "bound": floor["bound"],
                "kernel": "grouped GEMM (all tcgen05 launches: fc1/fc2 fwd, dgrad, wgrad)",
                **({"achieved": round(gemm_tflops, 1) if gemm_tflops else None,
                    "peak": peak_tf, "peak_source": peak_src, "unit": "TFLOP/s",
                    "frac": round(gemm_tflops / peak_tf, 4) if gemm_tflops else None}
                   if floor["bound"] == "tensor" or not hbm_ach else
                   {"achieved": round(hbm_ach, 1), "peak": hbm_gbs,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if peaks else "fallback",
                    "unit": "GB/s", "frac": round(hbm_ach / hbm_gbs, 4),
                    "tensor": {"achieved": round(gemm_tflops, 1) if gemm_tflops else None,
                               "peak": peak_tf, "unit": "TFLOP/s",
                               "frac": round(gemm_tflops / peak_tf, 4) if gemm_tflops else None}}),
                "floor_model": floor,
                "frac_vs": ({"sustained_measured": round(gemm_tflops / peak_tf, 4),
                             "burst_measured": round(gemm_tflops / burst_tf, 4),
                             "datasheet_dense_2250": round(gemm_tflops / 2250.0, 4),
                             # the dense bf16 tensor pipe at the SM clock the run actually
                             # held under the 1 kW cap: 8192 FLOP/clk/SM x 148 SMs x the
                             # median sampled clock (2.25 PF corresponds to ~1.86 GHz)
                             "clock_adjusted_dense": (
                                 round(gemm_tflops / (8192 * 148 * clk["sm_mhz"] * 1e6 / 1e12), 4)
                                 if clk and clk.get("sm_mhz") else None),
                             "clock_adjusted_peak_tflops": (
                                 round(8192 * 148 * clk["sm_mhz"] * 1e6 / 1e12, 1)
                                 if clk and clk.get("sm_mhz") else None)}
                            if gemm_tflops else None),
                "traffic": traffic["bytes"] if traffic else None,
                "traffic_detail": traffic,
                "algorithmic": f"18*K*h*m FLOP/token = {gemm_flops_per_token(c) / 1e9:.3f} "
                               "GFLOP/token (fwd 6, dgrad 6, wgrad 6)",
                "gemm_share_of_step": round(gemm_ms / ev_steps / ms_step, 4) if gemm_ms else None,
                "gemm_ms_per_step": round(gemm_ms / ev_steps, 4) if gemm_ms else None,
                "gemm_time": "union of the GEMM launches' event spans (a programmatic dependent "
                             "launch's overlap with the GEMM before it counted once)",
                "kernel_events": kernel_events,
            },
            "hbm_kernels": hbm,
            "e2e": {
                "value": round(tokens / (e2e_ms / 1e3), 1),
                "unit": "tokens/s",
                "ms_per_step": round(e2e_ms, 4),
                "h2d_bytes_per_step": int(x.numel() * 2 + dy.numel() * 2),
                "d2h_bytes_per_step": int(x.numel() * 2 + 4),
                "copies": "x, dY pinned H2D (copy stream, prefetched one step ahead); y and "
                          "the aux loss D2H to pinned host (second copy stream)",
                "api": "eager moe_forward + autograd backward (the public layer API) every "
                       "step, also when the device-resident timed region replays a graph",
            },
            "gpu_launches": launches,
            "gpu_launches_per_step": launches / args.steps,
            "gemm_launches": gemm_launches,
            "gemm_exclusive_ms_per_step": {k_: round(sum(v) / ev_steps, 4) for k_, v in
                                           gemm_excl.items()},
            "kernel_ms_per_step": {k_: round(sum(v) / ev_steps, 4) for k_, v in
                                   sorted(per_kernel.items(), key=lambda kv: -sum(kv[1]))},
            "clocks": clk,
            "routing": routing_stats,
            "echo": (dict(slots=args.echo_slots, **__import__(
                "paper_2603_07685_b200.dispatcher", fromlist=["x"]).last_echo)
                if args.echo_slots and n > 1 else None),
            "nvlink": nvlink_stats,
            "dropin": dropin,
        }
        if n == 1 and not args.no_cpu_baseline:
            thr = cpu_threads()
            cb = cpu_baseline(c, args.cpu_sample_tokens, thr)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        emit(out)
    gc.enable()
    if n > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, c) -> None:
    """Reference arm: the reference CPU path (oracle port of pkg/src/moelab/routing.py plus
    the restated backward) on the host cores, all threads, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    n = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    thr = cpu_threads()
    # inputs and weights are built once; warm-up steps run untimed, then K timed steps
    base = cpu_baseline(c, args.cpu_sample_tokens, thr, reps=1)
    for _ in range(max(args.warmup - 1, 0)):
        base["step"]()
    times = [base["step"]() for _ in range(args.steps)]
    sec = statistics.mean(times)
    value = args.cpu_sample_tokens / sec
    out = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "tokens/s",
        "n_gpus": n,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32",
        "data": "synthetic",
        "config": {"workload": f"{c['name']}: E={c['E']}, top-{c['K']}, h={c['h']}, "
                               f"ffn={c['m']}, CPU sample of {args.cpu_sample_tokens} tokens",
                   "parallelism": "host CPU (all threads)"},
        "cpu_baseline": {**{k: base[k] for k in ("cores", "kind", "sample")},
                         "value": round(value, 2), "unit": "tokens/s"},
        "e2e": {"value": round(value, 2), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # 60 steps (~1.7 s at Mixtral): the 1 kW power limiter needs ~1 s to settle, and 20-step
    # windows read ~3.5% fast (profiles/r02_power_window.txt)
    # (the reference arm's CPU steps take ~3 s each: it defaults to 10)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="mixtral", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-tokens", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dropin", action="store_true",
                    help="skip timing the numpy-in/numpy-out drop-in function API")
    ap.add_argument("--ep-transport", default="auto",
                    choices=["auto", "p2p", "p2p_overlap", "p2p_pull", "p2p_dedup", "nccl"],
                    help="EP exchange: fused NVLink peer-memory kernels (p2p) or NCCL a2a")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "mxfp8"],
                    help="expert GEMMs: bf16 (headline) or MXFP8 (block-scaled tcgen05 for "
                         "all six: fc1/fc2 forward, both data gradients, both weight "
                         "gradients)")
    ap.add_argument("--sync-free", action=argparse.BooleanOptionalAction, default=True,
                    help="EP: plan the exchange on the device (no host read of the counts; "
                         "worst-case static buffers). Default on: +2%% at EP=4 (measured)")
    ap.add_argument("--graph", action=argparse.BooleanOptionalAction, default=None,
                    help="capture the whole fwd+bwd step in a CUDA graph and replay it in the "
                         "timed region (EP: implies --sync-free). Default: on at N=1 (no host "
                         "work per step: immune to host pauses that drain the GPU queue), "
                         "off under EP (measured 1%% slower at EP=4)")
    ap.add_argument("--echo-slots", type=int, default=0,
                    help="ECHO hot-expert clone slots per rank (EP, dropless)")
    ap.add_argument("--skew", type=float, default=None,
                    help="router logit skew alpha (config 5 sweep: 0, 0.5, 1, 2)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 10 if args.impl == "reference" else 60
    if args.warmup < 3:
        args.warmup = 3
    if args.graph is None:
        args.graph = int(os.environ.get("WORLD_SIZE", str(args.gpus))) == 1 and args.gpus == 1
    c = CONFIGS[args.config]
    # stdout carries exactly one JSON line: everything else (NCCL's version banner, library
    # chatter) is routed to stderr at the fd level; the JSON goes to the saved stdout fd.
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.impl == "reference":
        run_reference(args, c)
    else:
        run_gpu(args, c)


_JSON_OUT = None


def emit(out: dict) -> None:
    stream = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    stream.write(json.dumps(out) + "\n")
    stream.flush()


if __name__ == "__main__":
    main()
