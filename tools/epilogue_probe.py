"""bf16 grouped GEMM epilogue A/B on one B200: per-thread 16-byte stores (the default
EPI_BF16 path) vs shared-memory staging + one 256-byte TMA bulk store per row half (the
scatter epilogue, here with row_dst pointing at the local output rows).

Mixtral shape: 8 experts x 4096 rows, h = 4096, m = 14336 (fc2 forward, fc1 dgrad).
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
    act = torch.randn((rows, m), device=dev).to(bf)
    d_pre = torch.randn((rows, 2 * m), device=dev).to(bf)
    w1 = (torch.randn((E, 2 * m, h), device=dev) * h ** -0.5).to(bf)
    w2 = (torch.randn((E, h, m), device=dev) * m ** -0.5).to(bf)
    out_a = torch.empty((rows, h), device=dev, dtype=bf)
    out_b = torch.empty((rows, h), device=dev, dtype=bf)
    row_dst = (torch.arange(rows, device=dev, dtype=torch.int64) * (h * 2) + out_b.data_ptr())
    fl2 = 2.0 * rows * m * h
    fl1d = 2.0 * rows * 2 * m * h
    res = {}
    for _ in range(2):
        for name, fn, fl in (
                ("fc2_fwd_stores", lambda: gemm.fc2_fwd(act, w2, be, nmb, out=out_a, pair=True), fl2),
                ("fc2_fwd_bulk", lambda: gemm.fc2_fwd_scatter(act, w2, be, nmb, row_dst, pair=True),
                 fl2),
                ("fc1_dgrad_stores", lambda: gemm.fc1_dgrad(d_pre, w1, be, nmb, out=out_a, pair=True),
                 fl1d),
                ("fc1_dgrad_bulk", lambda: gemm.fc1_dgrad_scatter(d_pre, w1, be, nmb, row_dst,
                                                                  pair=True), fl1d)):
            ms = timed(fn)
            res[name] = {"ms": round(ms, 3), "TFLOPs": round(fl / ms / 1e9, 1)}
    gemm.fc2_fwd(act, w2, be, nmb, out=out_a, pair=True)
    gemm.fc2_fwd_scatter(act, w2, be, nmb, row_dst, pair=True)
    torch.cuda.synchronize()
    res["bulk_equals_stores"] = bool(torch.equal(out_a, out_b))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
