"""Per-kind share of one step from an ncu launch list (gpu__time_duration.sum pass of
bench.py) next to the bench line's live CUDA-event shares: ncu serialises launches with
cold caches, so absolute times differ; the shares must agree.

    python tools/launch_share.py profiles/r02_final6/launches.csv profiles/r02_final6/bench1.json
"""
import csv
import json
import sys

KINDS = [("fc1_fwd", ("grouped_gemm_kernel<0, 0, 0, 1",)),
         ("fc2_fwd", ("grouped_gemm_kernel<0, 0, 0, 0",)),
         ("fc2_dgrad", ("grouped_gemm_kernel<0, 1, 0, 2",)),
         ("fc1_dgrad", ("grouped_gemm_kernel<0, 1, 0, 0",)),
         ("wgrad", ("grouped_gemm_kernel<1, 1, 1, 0",)),
         ("router", ("router_tc_kernel", "finalize_kernel", "bwd_kernel", "reduce_cm",
                     "stage_router", "router_bwd")),
         ("permute+gather", ("plan", "scan", "gather_tokens", "zero_pad", "split_units",
                             "count", "offsets", "scatter")),
         ("combine", ("combine",))]
BENCH = {"fc1_fwd": ["moe_gg_fc1_fwd"], "fc2_fwd": ["moe_gg_fc2_fwd"],
         "fc2_dgrad": ["moe_gg_fc2_dgrad"], "fc1_dgrad": ["moe_gg_fc1_dgrad"],
         "wgrad": ["moe_gg_wgrad_ex", "moe_gg_wgrad"],
         "router": ["moe_router_tc_fwd", "moe_router_tc_wgrad", "moe_router_bwd2",
                    "moe_stage_router_weight", "moe_router_finalize_tiles"],
         "permute+gather": ["moe_permute_plan", "moe_permute_gather", "moe_zero_pad_rows",
                            "moe_split_units"],
         "combine": ["moe_combine", "moe_combine_bwd"]}


def kind(name):
    for k, pats in KINDS:
        if any(p in name for p in pats):
            return k
    return None


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14]
    hdr, data = rows[0], rows[1:]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    ours = [(r[ik], float(r[iv].replace(",", ""))) for r in data
            if r[im] == "gpu__time_duration.sum" and kind(r[ik])]
    starts = [i for i, (n, _) in enumerate(ours) if "router_tc_kernel" in n and ", 0, " in n]
    # the last complete step: between the last two router forward launches
    step = ours[starts[-2]:starts[-1]] if len(starts) >= 2 else ours
    ncu = {}
    for n, ns in step:
        ncu[kind(n)] = ncu.get(kind(n), 0.0) + ns / 1e6
    tot = sum(ncu.values())
    b = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    kms = b["kernel_ms_per_step"]
    ev = {k: sum(kms.get(n, 0.0) for n in names) for k, names in BENCH.items()}
    etot = sum(ev.values())
    print(f"{'kind':16s} {'ncu ms':>8s} {'ncu share':>9s} {'bench ms':>9s} {'bench share':>11s}")
    for k, _ in KINDS:
        print(f"{k:16s} {ncu.get(k, 0):8.3f} {ncu.get(k, 0) / tot:9.3f} {ev[k]:9.3f} "
              f"{ev[k] / etot:11.3f}")
    print(f"{'total':16s} {tot:8.3f} {'':9s} {etot:9.3f}   (bench ms_per_step {b['ms_per_step']})")


if __name__ == "__main__":
    main()
