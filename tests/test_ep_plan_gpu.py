"""Sync-free EP planning on the device (moe_ep_plan_device) against the host restatement
(dispatcher.p2p_tables / ep_host_plan / global_aux): every integer table bit-exact, the aux
loss and its gradient to fp32 rounding. Single GPU: the kernel takes the all-gathered
[counts | mean scores] matrix as input, so no process group is needed."""
import numpy as np
import pytest
import torch

from paper_2603_07685_b200 import _lib, ops
from paper_2603_07685_b200.dispatcher import _excl_cumsum, ep_static_rows, global_aux, p2p_tables

pytestmark = pytest.mark.gpu

CASES = [
    # n, E, T, K, capacity factor, pad, skew
    (2, 8, 512, 2, None, False, 0.0),
    (4, 8, 4096, 2, None, False, 1.0),
    (4, 128, 1024, 8, None, False, 0.5),
    (8, 256, 512, 8, None, False, 0.0),
    (4, 8, 1024, 2, 1.0, True, 1.0),
    (2, 16, 777, 4, 1.25, False, 2.0),
    (4, 32, 300, 4, 0.5, True, 0.0),
]


@pytest.mark.parametrize("case", CASES, ids=[str(i) for i in range(len(CASES))])
def test_device_plan_matches_host(case):
    n, E, T, K, cf, pad, skew = case
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(hash(case) % 2**31)
    logits = rng.normal(size=(n * T, E)) - skew * np.log1p(np.arange(E))
    top = np.argsort(-logits, axis=1, kind="stable")[:, :K]
    counts_all = np.stack([np.bincount(top[s * T:(s + 1) * T].ravel(), minlength=E)
                           for s in range(n)])
    mean_scores = rng.random((n, E)).astype(np.float32)
    g = np.concatenate([counts_all.astype(np.float32), mean_scores], axis=1)
    gathered = torch.from_numpy(g).to(dev)
    cap = -1 if cf is None else -(-int(round(cf * n * T * K)) // E)
    align = ops.pick_align(n * T, K, E)
    el = E // n
    coeff = 1e-2
    for me in range(n):
        rows_cap = ep_static_rows(n, T, K, E, cap, align)
        i32 = dict(dtype=torch.int32, device=dev)
        base = torch.empty((E,), **i32)
        cap_l = torch.empty((E,), **i32)
        table = torch.empty((2 * n * el + 2 * el + 1,), **i32)
        be = torch.full((rows_cap // 128,), -7, **i32)
        meta = torch.empty((3,), **i32)
        dst_off = torch.empty((n * el,), **i32)
        aux = torch.empty((1 + E,), dtype=torch.float32, device=dev)
        status = torch.zeros((1,), **i32)
        _lib.call("moe_ep_plan_device", gathered.data_ptr(), 2 * E, n, E, me, T, K, cap,
                  int(pad), align, coeff, rows_cap, base.data_ptr(), cap_l.data_ptr(),
                  table.data_ptr(), be.data_ptr(), rows_cap // 128, meta.data_ptr(),
                  dst_off.data_ptr(), aux.data_ptr(), aux[1:].data_ptr(), status.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        hb, rows_all, hp = p2p_tables(counts_all, me, cap, pad, align)
        assert status.item() == 0
        assert np.array_equal(base.cpu().numpy(), hb)
        want_cap = hp.cap_local if hp.cap_local is not None else np.full(E, -1)
        assert np.array_equal(cap_l.cpu().numpy(), want_cap)
        assert np.array_equal(table.cpu().numpy(), hp.table)
        nb = hp.rows_pad // 128
        assert list(meta.cpu().numpy()) == [nb, hp.rows_pad, 0]
        assert np.array_equal(be[:nb].cpu().numpy(), hp.block_expert)
        want_dst = _excl_cumsum(hp.kept, axis=1)[:, me * el:(me + 1) * el].ravel()
        assert np.array_equal(dst_off.cpu().numpy(), want_dst)
        assert max(rows_all) <= rows_cap
        av, ag = global_aux(counts_all, mean_scores, T, K, coeff)
        got = aux.cpu().numpy().astype(np.float64)
        assert abs(got[0] - av) <= 1e-5 * max(abs(av), 1e-9)
        np.testing.assert_allclose(got[1:], ag, rtol=1e-6, atol=1e-12)
