"""bench.py contract checks that run without a GPU: the reference arm (the CPU oracle port
timed on the host) emits exactly one JSON line on stdout carrying the contract's keys."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--config", "tiny", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"]


def test_gpu_bench_json_line():
    """The GPU arm on the tiny config: one JSON line with the contract's keys, the whole-step
    CUDA graph in the timed region (N=1 default), per-kernel events captured in the graph,
    the eager e2e with its host<->device bytes, our kernels counted."""
    import pytest
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "tiny", "--steps",
                        "3", "--warmup", "3", "--no-cpu-baseline", "--no-dropin"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3
    assert d["config"]["cuda_graph"] is True and d["config"]["cuda_graph_error"] is None
    for k in ("bound", "achieved", "peak", "unit", "frac"):
        assert k in d["roofline"], k
    assert d["roofline"]["kernel_events"].startswith("live")
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and any(k.startswith("moe_gg") for k in d["kernel_ms_per_step"])


test_gpu_bench_json_line = __import__("pytest").mark.gpu(test_gpu_bench_json_line)


def test_gemm_floor_model_bounds():
    """The per-GEMM roofline floor (bench.gemm_floor_model): Mixtral is tensor-bound in every
    kind, DeepSeek at EP=1 HBM-bound in every kind (fc1 streams E*2*m*h bf16 weights for
    ~128 rows per expert) and tensor-bound at EP=2 (twice the rows per expert); the floor
    is the sum of per-kind max(compute, bytes) and frac_of_floor = floor / measured."""
    sys.path.insert(0, str(ROOT))
    import bench

    peak_tf, hbm = 1379.5, 6547.8
    kinds = ("fc1_fwd", "fc2_fwd", "fc2_dgrad", "fc1_dgrad", "wgrad")
    mx = bench.gemm_floor_model(bench.CONFIGS["mixtral"], 1, {}, 1, peak_tf, hbm)
    assert mx["bound"] == "tensor" and all(mx["per_gemm"][k]["bound"] == "tensor" for k in kinds)
    # 18*K*h*m*T FLOP at the sustained peak
    c = bench.CONFIGS["mixtral"]
    t_ms = 18.0 * c["K"] * c["h"] * c["m"] * c["T"] / (peak_tf * 1e12) * 1e3
    assert abs(mx["floor_ms"] - t_ms) < 1e-2 and mx["measured_ms"] is None
    ds = bench.gemm_floor_model(bench.CONFIGS["deepseek"], 1, {}, 1, peak_tf, hbm)
    assert ds["bound"] == "hbm" and all(ds["per_gemm"][k]["bound"] == "hbm" for k in kinds)
    w1 = 256 * 2 * 2048 * 7168 * 2  # the routed fc1 weights, bytes
    assert ds["per_gemm"]["fc1_fwd"]["GB"] * 1e9 > w1
    assert bench.gemm_floor_model(bench.CONFIGS["deepseek"], 2, {}, 1, peak_tf, hbm)["bound"] \
        == "tensor"
    # measured per-kind exclusive times (ms lists per launch name) -> frac_of_floor
    per = {"moe_gg_fc1_fwd": [2 * mx["per_gemm"]["fc1_fwd"]["floor_ms"]],
           "moe_gg_wgrad_ex": [mx["per_gemm"]["wgrad"]["floor_ms"]],
           "moe_gg_wgrad_f32": [100.0]}  # the router's fp32 split-K GEMM is not an expert kind
    f = bench.gemm_floor_model(c, 1, per, 1, peak_tf, hbm)
    assert f["per_gemm"]["fc1_fwd"]["frac_of_floor"] == 0.5
    assert f["per_gemm"]["wgrad"]["frac_of_floor"] == 1.0
