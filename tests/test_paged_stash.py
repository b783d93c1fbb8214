"""Paged Stashing: the oracle (oracle/paged_stash_ref.py) against op sequences replayed
through the reference allocator (tests/golden/stash_golden.npz, planners.py:394-463) and the
reference's own tests (test_planners.py:314-375); the device allocator + copies
(csrc/stash.cu via paper_2603_07685_b200/stash.py) against the same golden sequences, and
stash -> reload byte identity."""
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.paged_stash_ref import PagedStashRef

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "stash_golden.npz")
MAXP = 16


def _replay_oracle(i):
    num_pages, page_size = GOLD[f"{i}/shape"].tolist()
    ps = PagedStashRef(num_pages, page_size)
    out = []
    for kind, layer, tokens in GOLD[f"{i}/ops"].tolist():
        if kind == 0:
            try:
                pages = ps.stash(layer, tokens)
                row = pages + [-1] * (MAXP - len(pages))
            except MemoryError:
                row = [-2] * MAXP
        else:
            ps.reload(layer)
            row = [-1] * MAXP
        out.append(row + [ps.peak_pages_used, ps.free_pages])
    return np.array(out, dtype=np.int64)


def test_oracle_matches_reference_golden():
    for i in range(int(GOLD["n"])):
        assert np.array_equal(_replay_oracle(i), GOLD[f"{i}/res"]), i


def test_oracle_reference_unit_cases():
    ps = PagedStashRef(16, 64)
    assert len(ps.stash(0, 100)) == 2
    ps = PagedStashRef(4, 1)
    assert ps.stash(0, 2) == [0, 1]
    ps.reload(0)  # free list [2, 3, 0, 1]
    assert ps.stash(1, 2) == [2, 3]
    ps = PagedStashRef(2, 64)
    ps.stash(0, 128)
    with pytest.raises(MemoryError, match="pages"):
        ps.stash(1, 1)
    ps = PagedStashRef(4096, 64, worst_case_tokens=4096)
    for layer in range(60):
        ps.stash(layer, 256)
    assert ps.peak_memory_tokens() == 4096 + 60 * 256


@pytest.mark.gpu
def test_device_allocator_matches_reference_golden():
    from paper_2603_07685_b200.stash import PagedStashBuffer

    dev = torch.device("cuda", 0)
    for i in range(int(GOLD["n"])):
        num_pages, page_size = GOLD[f"{i}/shape"].tolist()
        buf = PagedStashBuffer(num_pages, {"x": 16}, page_rows=page_size, max_records=512,
                               max_pages_per_record=MAXP, device=dev)
        dense = torch.zeros((MAXP * page_size, 4), dtype=torch.int32, device=dev)
        failed = set()
        for j, ((kind, layer, tokens), want) in enumerate(zip(GOLD[f"{i}/ops"].tolist(),
                                                              GOLD[f"{i}/res"].tolist())):
            if kind == 0:
                rec = buf.stash(layer, {"x": dense}, rows=tokens)
                r = rec.tolist()
                st = buf.stats()
                if st["last_failed"]:
                    got = [-2] * MAXP
                    buf.release(layer)
                    failed.add(layer)
                else:
                    got = r[1:1 + r[0]] + [-1] * (MAXP - r[0])
            else:
                buf.reload(layer, {"x": dense}, rows=0)
                got = [-1] * MAXP
                st = buf.stats()
            got += [st["peak_pages_used"], st["free_pages"]]
            assert got == want, (i, j, kind, layer, tokens)


@pytest.mark.gpu
def test_device_stash_reload_identity_device_rows():
    from paper_2603_07685_b200.stash import PagedStashBuffer

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(3)
    widths = {"a": 4096 * 2, "b": 3072 * 2}
    buf = PagedStashBuffer(64, widths, page_rows=64, max_records=8, device=dev)
    saved = {}
    for layer, rows in enumerate([700, 64, 1, 1000]):
        a = torch.randn((1024, 4096), generator=g, device=dev).to(torch.bfloat16)
        b = torch.randn((1024, 3072), generator=g, device=dev).to(torch.bfloat16)
        n_dev = torch.tensor([rows], dtype=torch.int32, device=dev)
        buf.stash(layer, {"a": a, "b": b}, rows_dev=n_dev)
        saved[layer] = (a.clone(), b.clone(), rows, n_dev)
    buf.check()
    assert buf.stats()["peak_pages_used"] == sum(-(-r // 64) for r in [700, 64, 1, 1000])
    for layer in [2, 0, 3, 1]:
        a0, b0, rows, n_dev = saved[layer]
        a = torch.zeros_like(a0)
        b = torch.zeros_like(b0)
        buf.reload(layer, {"a": a, "b": b}, rows_dev=n_dev)
        assert torch.equal(a[:rows], a0[:rows]) and torch.equal(b[:rows], b0[:rows])
        assert not a[rows:].any()
    assert buf.stats()["free_pages"] == 64


@pytest.mark.gpu
def test_device_stash_out_of_pages_poisons_reload():
    """A stash that runs out of pages (the reference's MemoryError) records nothing; its
    reload fills the destination rows with NaN instead of leaving stale activations, and
    check() raises MemoryError."""
    from paper_2603_07685_b200.stash import PagedStashBuffer

    dev = torch.device("cuda", 0)
    buf = PagedStashBuffer(4, {"a": 256 * 2}, page_rows=64, device=dev)
    a0 = torch.randn((512, 256), device=dev).to(torch.bfloat16)
    buf.stash(0, {"a": a0}, rows=200)          # 4 pages: fits exactly
    buf.stash(1, {"a": a0}, rows=10)           # no page left: fails
    with pytest.raises(MemoryError, match="out of pages"):
        buf.check()
    a = torch.zeros_like(a0)
    buf.reload(1, {"a": a}, rows=10)
    assert torch.isnan(a[:10].float()).all() and not a[10:].any()
    b = torch.zeros_like(a0)
    buf.reload(0, {"a": b}, rows=200)
    assert torch.equal(b[:200], a0[:200])
    assert buf.stats()["free_pages"] == 4
