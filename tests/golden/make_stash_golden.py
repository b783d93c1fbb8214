"""Golden Paged-Stashing op sequences replayed through the REFERENCE allocator
(pkg/src/moelab/planners.py:394-463).

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_stash_golden.py

Writes tests/golden/stash_golden.npz: per sequence, the pool shape and the ops
(kind 0 = stash(layer, tokens), 1 = reload(layer)) with the reference's outcome: the page ids
returned by stash (padded with -1), -2 for MemoryError, and the peak pages / free pages after
each op.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "stash_golden.npz"
MAXP = 16


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF_SRC))
    from moelab.planners import PagedStash  # noqa: E402 (reference)

    rng = np.random.default_rng(2603)
    g: dict[str, np.ndarray] = {}
    seqs = [(4, 1, 6), (16, 64, 40), (32, 16, 200), (256, 16, 600), (9, 7, 120)]
    g["n"] = np.array(len(seqs))
    for i, (num_pages, page_size, n_ops) in enumerate(seqs):
        ps = PagedStash(num_pages=num_pages, page_size=page_size)
        live: list[int] = []
        nxt = 0
        ops, res = [], []
        for _ in range(n_ops):
            if live and (rng.random() < 0.45 or ps.free_pages < 2):
                layer = live.pop(int(rng.integers(0, len(live))))
                ps.reload(layer)
                ops.append((1, layer, 0))
                res.append([-1] * MAXP + [ps.peak_pages_used, ps.free_pages])
            else:
                tokens = int(rng.integers(1, min(MAXP, num_pages) * page_size + 1))
                try:
                    pages = ps.stash(nxt, tokens, b"")
                    live.append(nxt)
                    row = pages + [-1] * (MAXP - len(pages))
                except MemoryError:
                    row = [-2] * MAXP
                ops.append((0, nxt, tokens))
                nxt += 1
                res.append(row + [ps.peak_pages_used, ps.free_pages])
        g[f"{i}/shape"] = np.array([num_pages, page_size])
        g[f"{i}/ops"] = np.array(ops, dtype=np.int64)
        g[f"{i}/res"] = np.array(res, dtype=np.int64)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({len(seqs)} sequences)")


if __name__ == "__main__":
    main()
