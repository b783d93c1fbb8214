"""CPU checks of the loopback EP group's collectives (paper_2603_07685_b200.loopback):
the single-GPU EP tests rely on them behaving like the NCCL group's."""
import torch

from paper_2603_07685_b200.loopback import run_ranks


def test_loopback_collectives_match_semantics():
    n = 3
    dev = torch.device("cpu")

    def body(ep):
        r = ep.rank
        inp = torch.arange(4, dtype=torch.float32) + 10 * r
        out = torch.empty((n, 4))
        ep.all_gather_into_tensor(out, inp)
        t = torch.full((2,), float(r + 1))
        ep.all_reduce(t)
        # rank r sends (s + 1) rows of value 100*r + s to rank s
        in_splits = [s + 1 for s in range(n)]
        send = torch.cat([torch.full((s + 1, 2), 100.0 * r + s) for s in range(n)])
        out_splits = [r + 1] * n
        recv = torch.empty((sum(out_splits), 2))
        ep.all_to_all_single(recv, send, out_splits, in_splits)
        buf, ptrs, h = ep.symm_empty(8, torch.int32, dev)
        buf[:] = r
        ep.all_reduce(torch.zeros(1))  # barrier
        peer = h.get_remote_tensor((r + 1) % n, (8,), torch.int32).clone()
        return out, t, recv, ptrs, peer, buf.data_ptr()

    res = run_ranks(n, body, dev)
    expect_gather = torch.stack([torch.arange(4, dtype=torch.float32) + 10 * s for s in range(n)])
    for r, (out, t, recv, ptrs, peer, own) in enumerate(res):
        assert torch.equal(out, expect_gather)
        assert torch.equal(t, torch.full((2,), float(sum(range(1, n + 1)))))
        exp = torch.cat([torch.full((r + 1, 2), 100.0 * s + r) for s in range(n)])
        assert torch.equal(recv, exp)
        assert ptrs[r] == own and len(set(ptrs)) == n
        assert torch.equal(peer, torch.full((8,), (r + 1) % n, dtype=torch.int32))
