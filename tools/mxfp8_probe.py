"""MXFP8 vs bf16 grouped GEMM throughput on one B200 (same box, interleaved runs).

Mixtral-shape expert GEMMs: 8 experts x 4096 rows, h = 4096, m = 14336.
  fc1 (+SwiGLU): 2 * R * h * 2m FLOP; fc2: 2 * R * m * h FLOP.
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_07685_b200 import gemm  # noqa: E402


def timed(fn, iters=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    dev = torch.device("cuda", 0)
    E, per, h, m = 8, 4096, 4096, 14336
    rows = E * per
    bf = torch.bfloat16
    be = (torch.arange(rows // 128, device=dev, dtype=torch.int32) // (per // 128))
    nmb = torch.tensor([rows // 128], dtype=torch.int32, device=dev)
    x = torch.randn((rows, h), device=dev).to(bf)
    gate = (torch.randn((E, m, h), device=dev) * h ** -0.5).to(bf)
    up = (torch.randn((E, m, h), device=dev) * h ** -0.5).to(bf)
    w2 = (torch.randn((E, h, m), device=dev) * m ** -0.5).to(bf)
    w1 = gemm.interleave_gate_up(gate, up)
    w1mx = gemm.interleave_gate_up_mx(gate, up)
    xq, xsf, _ = gemm.mxfp8_quantize(x)
    w1q, w1sf = gemm.mxfp8_quantize_weight(w1mx)
    w1qw, w1sfw = gemm.mxfp8_quantize_w1(w1, wide=True)
    w2q, w2sf = gemm.mxfp8_quantize_weight(w2)
    fl1 = 2.0 * rows * h * 2 * m
    fl2 = 2.0 * rows * m * h
    out = {}
    st = {}

    def bf_fc1():
        st["pa"] = gemm.fc1_fwd(x, w1, be, nmb, pair=True)

    def mx_fc1():
        st["mx"] = gemm.mxfp8_fc1(xq, xsf, w1q, w1sf, E, be, nmb, m)

    def mx_fc1_pair():
        st["mx"] = gemm.mxfp8_fc1(xq, xsf, w1q, w1sf, E, be, nmb, m, pair=True)

    def mx_fc1_pair_wide():
        st["mxw"] = gemm.mxfp8_fc1(xq, xsf, w1qw, w1sfw, E, be, nmb, m, pair=True, wide=True)

    for _ in range(2):
        for name, fn, fl in (("bf16_fc1", bf_fc1, fl1), ("mxfp8_fc1", mx_fc1, fl1),
                             ("mxfp8_fc1_pair", mx_fc1_pair, fl1),
                             ("mxfp8_fc1_pair_wide", mx_fc1_pair_wide, fl1)):
            ms = timed(fn)
            out[name] = {"ms": round(ms, 3), "TFLOPs": round(fl / ms / 1e9, 1)}
    act = st["pa"][1]
    aq, asf = st["mx"][2], st["mx"][3]
    for _ in range(2):
        for name, fn, fl in (
                ("bf16_fc2", lambda: gemm.fc2_fwd(act, w2, be, nmb, pair=True), fl2),
                ("mxfp8_fc2", lambda: gemm.mxfp8_gemm(aq, asf, w2q, w2sf, E, be, nmb, h), fl2),
                ("mxfp8_fc2_pair", lambda: gemm.mxfp8_gemm(aq, asf, w2q, w2sf, E, be, nmb, h,
                                                           pair=True), fl2),
                ("mxfp8_fc2_pair_wide", lambda: gemm.mxfp8_gemm(aq, asf, w2q, w2sf, E, be, nmb,
                                                                h, pair=True, wide=True), fl2),
                ("mxfp8_quant_x", lambda: gemm.mxfp8_quantize(x), 0.0)):
            ms = timed(fn)
            out[name] = {"ms": round(ms, 3)}
            if fl:
                out[name]["TFLOPs"] = round(fl / ms / 1e9, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
