"""Per-kernel DRAM traffic of one MoE-layer fwd+bwd step from an ncu metrics CSV
(tools/layer_step.py under `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,...`),
next to each kernel's algorithmic (compulsory) bytes and FLOPs. Writes the JSON bench.py
reads for roofline.traffic.

    python tools/step_traffic.py gpurun_out/r2o_step_mixtral.csv mixtral profiles/r02_step_traffic_mixtral.json
"""
import csv
import json
import sys
from collections import OrderedDict

SHAPES = {"mixtral": dict(E=8, K=2, h=4096, m=14336, T=16384, ms=0),
          "qwen3": dict(E=128, K=8, h=4096, m=1536, T=32768, ms=0),
          "deepseek": dict(E=256, K=8, h=7168, m=2048, T=4096, ms=2048)}

GEMM_KIND = {  # grouped_gemm_kernel<A_MN, B_MN, GROUPED_K, EPI, ...>
    ("0", "0", "0", "1"): "fc1_fwd", ("0", "0", "0", "0"): "fc2_fwd",
    ("0", "1", "0", "2"): "fc2_dgrad", ("0", "1", "0", "0"): "fc1_dgrad",
    ("1", "1", "1", "0"): "wgrad", ("0", "0", "0", "3"): "router_logits_gemm",
    ("1", "1", "1", "3"): "router_wgrad_gemm",
}


def kind_of(name):
    if "grouped_gemm_kernel<" in name:
        args = tuple(a.strip() for a in name.split("<", 1)[1].split(">")[0].split(","))
        return GEMM_KIND.get(args[:4], "gemm" + str(args))
    return name.split("(")[0].replace("void ", "").split("::")[-1]


def main():
    path, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ii, ik, im, iv = (hdr.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    launches = OrderedDict()
    for r in data:
        d = launches.setdefault(int(r[ii]), {"name": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    ours = [d for d in launches.values() if "moe::" in d["name"] or "grouped_gemm" in d["name"]
            or any(k in d["name"] for k in ("router", "perm", "combine", "gather", "topk",
                                            "finalize", "bwd_kernel", "zero_pad", "reduce"))]
    # the last of the 4 steps: its launches start at the last router forward (the small-N
    # router kernel, or the round-1 chain's weight staging)
    starts = [i for i, d in enumerate(ours) if "stage_router_weight" in d["name"]
              or ("router_tc_kernel<" in d["name"] and ", 0, " in d["name"])]
    step = ours[starts[-1]:] if starts else ours[-len(ours) // 4:]
    s = SHAPES[cfg]
    E, K, h, m, T, ms = s["E"], s["K"], s["h"], s["m"], s["T"], s["ms"]
    R = T * K
    w = 2
    alg_bytes = {  # compulsory HBM bytes per launch of the routed-expert GEMMs (bf16)
        "fc1_fwd": R * h * w + E * 2 * m * h * w + R * 2 * m * w + R * m * w,
        "fc2_fwd": R * m * w + E * h * m * w + R * h * w,
        "fc2_dgrad": R * h * w + E * h * m * w + R * 2 * m * w * 2,
        "fc1_dgrad": R * 2 * m * w + E * 2 * m * h * w + R * h * w,
    }
    flops = {"fc1_fwd": 4.0 * R * h * m, "fc2_fwd": 2.0 * R * h * m, "fc2_dgrad": 2.0 * R * h * m,
             "fc1_dgrad": 4.0 * R * h * m}
    table = []
    for d in step:
        k = kind_of(d["name"])
        dur = d.get("gpu__time_duration.sum", 0.0) / 1e6  # ms
        rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        e = {"kernel": k, "ms": round(dur, 4), "dram_read_GB": round(rd / 1e9, 4),
             "dram_write_GB": round(wr / 1e9, 4),
             "dram_TBps": round((rd + wr) / (dur / 1e3) / 1e12, 3) if dur else None,
             "tensor_active_pct": d.get(
                 "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
             "sm_ghz": round(d.get("sm__cycles_elapsed.avg.per_second", 0.0) / 1e9, 3)}
        table.append(e)
    # the routed GEMMs in step order: fc1_fwd, fc2_fwd (first), fc2_dgrad, wgrad x2, fc1_dgrad
    gemm_traffic = {}
    seen = {}
    prev = None
    for e in table:
        k = e["kernel"]
        seen[k] = seen.get(k, 0) + 1
        if k in alg_bytes and seen[k] == 1:
            gemm_traffic[k] = {"traffic_GB": round(e["dram_read_GB"] + e["dram_write_GB"], 3),
                               "algorithmic_GB": round(alg_bytes[k] / 1e9, 3),
                               "ratio": round((e["dram_read_GB"] + e["dram_write_GB"])
                                              / (alg_bytes[k] / 1e9), 2),
                               "ms_ncu": e["ms"], "tensor_active_pct": e["tensor_active_pct"],
                               "tflops_ncu": round(flops[k] / (e["ms"] / 1e3) / 1e12, 1),
                               "launches": 1}
        elif k in alg_bytes and seen[k] == 2 and prev == k:
            # split units: the 1-CTA tail launch right behind the pair launch of the same GEMM
            g = gemm_traffic[k]
            g["traffic_GB"] = round(g["traffic_GB"] + e["dram_read_GB"] + e["dram_write_GB"], 3)
            g["ratio"] = round(g["traffic_GB"] / g["algorithmic_GB"], 2)
            g["ms_ncu"] = round(g["ms_ncu"] + e["ms"], 4)
            g["tflops_ncu"] = round(flops[k] / (g["ms_ncu"] / 1e3) / 1e12, 1)
            g["launches"] = 2
        prev = k
    wg = [e for e in table if e["kernel"] == "wgrad"]
    if len(wg) >= 2:
        a2 = E * h * m * w + R * h * w + R * m * w       # dW2: read dO, act; write dW2
        a1 = E * 2 * m * h * w + R * 2 * m * w + R * h * w  # dW1: read d_preact, xp; write dW1
        for name, e, a in (("wgrad_dW2", wg[0], a2), ("wgrad_dW1", wg[1], a1)):
            gemm_traffic[name] = {"traffic_GB": round(e["dram_read_GB"] + e["dram_write_GB"], 3),
                                  "algorithmic_GB": round(a / 1e9, 3),
                                  "ratio": round((e["dram_read_GB"] + e["dram_write_GB"])
                                                 / (a / 1e9), 2),
                                  "ms_ncu": e["ms"], "tensor_active_pct": e["tensor_active_pct"]}
    res = {"config": cfg, "source": path, "step_launches": table,
           "routed_gemm_traffic": gemm_traffic,
           "note": "ncu --metrics pass (cold caches, serialised launches, unlocked clocks): "
                   "per-launch DRAM bytes are the evidence; absolute times are not bench times"}
    json.dump(res, open(out, "w"), indent=1)
    for k, v in gemm_traffic.items():
        print(cfg, k, v)


if __name__ == "__main__":
    main()
