"""Golden ECHO plans from the REFERENCE planner (pkg/src/moelab/planners.py:190-389).

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_echo_golden.py

Writes tests/golden/echo_golden.npz (counts, experts_per_rank, spare slots -> clones,
target, pre/post loads, best-effort flag, placement) for tests/test_echo.py.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "echo_golden.npz"


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF_SRC))
    from moelab.planners import echo_plan, rewrite_routing_counts  # noqa: E402 (reference)

    rng = np.random.default_rng(1234)
    cases = [([10, 2, 2, 2], 1, 1), ([4, 4, 4, 4], 1, 1), ([100, 0, 0, 0], 1, 0),
             ([12, 1, 3, 3, 0, 5], 2, 2), ([40, 1, 1, 1, 1, 1, 1, 2], 1, 1)]
    for _ in range(60):
        ranks = int(rng.integers(2, 7))
        epr = int(rng.integers(1, 4))
        slots = int(rng.integers(0, 4))
        hot = rng.integers(0, 40, size=ranks * epr)
        hot[int(rng.integers(0, ranks * epr))] += int(rng.integers(0, 120))
        cases.append((hot.tolist(), epr, slots))
    for _ in range(10):  # beyond the exact-search limit: FFD only
        cases.append((rng.integers(0, 200, size=16).tolist(), 2, 2))
    g: dict[str, np.ndarray] = {"n": np.array(len(cases))}
    for i, (counts, epr, slots) in enumerate(cases):
        plan = echo_plan(counts, epr, slots)
        place = rewrite_routing_counts(counts, plan, epr)
        g[f"{i}/counts"] = np.array(counts, dtype=np.int64)
        g[f"{i}/epr"] = np.array(epr)
        g[f"{i}/slots"] = np.array(slots)
        g[f"{i}/clones"] = np.array([[c.expert, c.rank, c.tokens] for c in plan.clones],
                                    dtype=np.int64).reshape(-1, 3)
        g[f"{i}/target"] = np.array(plan.target_load)
        g[f"{i}/pre_max"] = np.array(plan.pre_max_load)
        g[f"{i}/post"] = np.array(plan.post_loads, dtype=np.int64)
        g[f"{i}/best_effort"] = np.array(plan.best_effort)
        g[f"{i}/placement"] = np.array(sorted((e, r, v) for (e, r), v in place.items()),
                                       dtype=np.int64).reshape(-1, 3)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({len(cases)} plans)")


if __name__ == "__main__":
    main()
