"""NVLink evidence for the EP exchange kernels, in ONE process driving 2 GPUs (so ncu can
profile it: no multi-rank command). GPU 0 plays EP rank 0 of a Mixtral-shape EP=2 layer
(E=8, K=2, h=4096, m=14336, T=16384 tokens per rank):

  * dispatch: moe_ep_dispatch_push stores rank 0's token rows into both ranks' padded expert
    plans -- rows for experts 4..7 go straight into GPU 1's memory over NVLink;
  * return: moe_gg_fc2_fwd_scatter (fc2 of rank 0's experts 0..3) stores each output row into
    its source rank's compact buffer from the GEMM epilogue -- rank 1's rows over NVLink.

Prints exact remote bytes (from the plan) and CUDA-event times; under
  ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,... python tools/nvlink_probe.py
the NVLink TX counters of GPU 0 measure the same transfers.

    python tools/nvlink_probe.py [iters]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_07685_b200 import _lib, gemm, ops  # noqa: E402
from paper_2603_07685_b200.dispatcher import _excl_cumsum, p2p_tables  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
assert torch.cuda.device_count() >= 2, "needs 2 GPUs (gpurun --gpus 2)"
import cuda.bindings.runtime as rt  # noqa: E402

for a, b in ((0, 1), (1, 0)):
    torch.cuda.set_device(a)
    torch.zeros(1, device=f"cuda:{a}")
    err = rt.cudaDeviceEnablePeerAccess(b, 0)[0]
    assert err in (rt.cudaError_t.cudaSuccess,
                   rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled), err
torch.cuda.set_device(0)

E, K, h, m, T, n = 8, 2, 4096, 14336, 16384, 2
el = E // n
bf = torch.bfloat16
d0, d1 = torch.device("cuda:0"), torch.device("cuda:1")
g = torch.Generator(device=d0).manual_seed(0)
w_r = (torch.randn((h, E), device=d0, generator=g) * h ** -0.5).to(bf)
xs = [torch.randn((T, h), device=d0, generator=g).to(bf) for _ in range(n)]
routes = [ops.router_forward(x, w_r, K, "softmax") for x in xs]
counts_all = np.stack([r.counts.cpu().numpy() for r in routes]).astype(np.int64)
align = ops.pick_align(n * T, K, E)
base, rows_all, hp = p2p_tables(counts_all, 0, -1, False, align)
splan = ops.build_plan(routes[0].topk_idx, routes[0].topk_prob, E, -1, False, compact=True)
base_d = torch.from_numpy(base.astype(np.int32)).to(d0)
xp = [torch.zeros((max(rows_all[r], 256), h), dtype=bf, device=d) for r, d in enumerate((d0, d1))]
peers = torch.tensor([t.data_ptr() for t in xp], dtype=torch.int64, device=d0)
stream = torch.cuda.current_stream(d0).cuda_stream


def push():
    _lib.call("moe_ep_dispatch_push", xs[0].data_ptr(), T, K, h, routes[0].topk_idx.data_ptr(),
              splan.inv_map.data_ptr(), base_d.data_ptr(), el, peers.data_ptr(), None, None,
              stream)


# fc2 of rank 0's experts with the row-scatter epilogue returning rows to their source rank
w2 = (torch.randn((el, h, m), device=d0, generator=g) * m ** -0.5).to(bf)
rows_pad = hp.rows_pad
act = torch.randn((max(rows_pad, 256), m), device=d0, generator=g).to(bf)
dst_off = _excl_cumsum(hp.kept, axis=1)[:, 0:el].ravel()
tab = torch.from_numpy(np.concatenate([hp.table.astype(np.int64), hp.block_expert,
                                       [rows_pad // 128], dst_off]).astype(np.int32)).to(d0)
nt, nb = hp.table.size, hp.block_expert.size
table_d, be_d, nmb, dst_off_d = tab[:nt], tab[nt:nt + nb], tab[nt + nb:nt + nb + 1], tab[nt + nb + 1:]
orecv = [torch.zeros((T * K, h), dtype=bf, device=d) for d in (d0, d1)]
orecv_peers = torch.tensor([t.data_ptr() for t in orecv], dtype=torch.int64, device=d0)
row_dst = torch.empty((rows_pad,), dtype=torch.int64, device=d0)
_lib.call("moe_ep_row_dst", table_d.data_ptr(), n, el, rows_pad, dst_off_d.data_ptr(),
          orecv_peers.data_ptr(), h * 2, row_dst.data_ptr(), stream)
pair = align == 256


def scatter():
    gemm.fc2_fwd_scatter(act, w2, be_d, nmb, row_dst, max_rows=act.shape[0], pair=pair)


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize(d0)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize(d0)
    return s.elapsed_time(e) / iters


# correctness of the remote rows: every selection of rank 0 on a rank-1 expert landed on GPU 1
push()
torch.cuda.synchronize(d0)
idx = routes[0].topk_idx.long().cpu().numpy()
inv = splan.inv_map.long().cpu().numpy()
t_sel, k_sel = np.nonzero(idx >= el)
rows_remote = base[idx[t_sel, k_sel]] + inv[t_sel, k_sel]
got = xp[1][torch.from_numpy(rows_remote).to(d1)].to(d0)
assert torch.equal(got, xs[0][torch.from_numpy(t_sel).to(d0)]), "remote rows differ"
sent_remote = int(len(t_sel))
# rows of rank 0's plan whose source is rank 1 (returned over NVLink by the scatter epilogue)
recv_remote = int(hp.recv_splits[1])
ms_push = timeit(push)
ms_scatter = timeit(scatter)
flops = 2.0 * rows_pad * m * h
out = {
    "shape": "Mixtral EP=2 rank 0 (T=16384/rank, E=8, K=2, h=4096, m=14336)",
    "dispatch_push": {"ms": round(ms_push, 4), "remote_rows": sent_remote,
                      "remote_bytes": sent_remote * h * 2,
                      "local_bytes": (int((idx < el).sum())) * h * 2,
                      "nvlink_GBps": round(sent_remote * h * 2 / (ms_push / 1e3) / 1e9, 1)},
    "fc2_fwd_scatter": {"ms": round(ms_scatter, 4), "remote_rows": recv_remote,
                        "remote_bytes": recv_remote * h * 2,
                        "tflops": round(flops / (ms_scatter / 1e3) / 1e12, 1),
                        "nvlink_GBps_if_spread": round(recv_remote * h * 2 / (ms_scatter / 1e3)
                                                       / 1e9, 1)},
}
print(json.dumps(out))
