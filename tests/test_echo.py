"""ECHO hot-expert cloning planner: oracle (oracle/echo_ref.py) and product
(paper_2603_07685_b200/echo.py) against plans produced by the reference itself
(tests/golden/echo_golden.npz, reference planners.py:190-389), the reference's own unit
tests (test_planners.py:173-311), and invariants of the virtual-expert layout."""
import itertools
from pathlib import Path

import numpy as np
import pytest

from oracle import echo_ref as O
from paper_2603_07685_b200 import echo as P

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "echo_golden.npz")
N = int(GOLD["n"])


def clones_of(plan):
    return np.array([[c.expert, c.rank, c.tokens] for c in plan.clones],
                    dtype=np.int64).reshape(-1, 3)


@pytest.mark.parametrize("impl", [O, P], ids=["oracle", "product"])
def test_plans_match_reference_golden(impl):
    for i in range(N):
        counts = GOLD[f"{i}/counts"]
        epr, slots = int(GOLD[f"{i}/epr"]), int(GOLD[f"{i}/slots"])
        plan = impl.echo_plan(counts, epr, slots)
        assert np.array_equal(clones_of(plan), GOLD[f"{i}/clones"]), (i, counts.tolist())
        assert plan.target_load == int(GOLD[f"{i}/target"])
        assert plan.pre_max_load == int(GOLD[f"{i}/pre_max"])
        assert np.array_equal(plan.post_loads, GOLD[f"{i}/post"])
        assert bool(plan.best_effort) == bool(GOLD[f"{i}/best_effort"])


def test_oracle_placement_matches_reference_golden():
    for i in range(N):
        counts = GOLD[f"{i}/counts"].tolist()
        epr, slots = int(GOLD[f"{i}/epr"]), int(GOLD[f"{i}/slots"])
        place = O.rewrite_routing_counts(counts, O.echo_plan(counts, epr, slots), epr)
        got = np.array(sorted((e, r, v) for (e, r), v in place.items())).reshape(-1, 3)
        assert np.array_equal(got, GOLD[f"{i}/placement"])


def test_product_matches_oracle_random():
    rng = np.random.default_rng(99)
    for _ in range(300):
        ranks, epr = int(rng.integers(2, 6)), int(rng.integers(1, 4))
        counts = rng.integers(0, 30, size=ranks * epr)
        counts[int(rng.integers(0, ranks * epr))] += int(rng.integers(0, 90))
        slots = int(rng.integers(0, 4))
        a, b = O.echo_plan(counts, epr, slots), P.echo_plan(counts, epr, slots)
        assert np.array_equal(clones_of(a), clones_of(b))
        assert a.post_loads == b.post_loads and a.best_effort == b.best_effort


# -- the reference's own tests (test_planners.py:173-311), restated ------------------

def test_canonical_example():
    plan = P.echo_plan([10, 2, 2, 2], 1, 1)
    assert plan.clone_count == 3 and plan.post_max_load == 4
    assert sorted((c.expert, c.rank, c.tokens) for c in plan.clones) == [
        (0, 1, 2), (0, 2, 2), (0, 3, 2)]


def test_balanced_is_empty_and_best_effort_flag():
    assert P.echo_plan([4, 4, 4, 4], 1, 1).clone_count == 0
    assert P.echo_plan([100, 0, 0, 0], 1, 0).best_effort
    with pytest.raises(ValueError):
        P.echo_plan([1, 2, 3], 2, 1)
    with pytest.raises(ValueError):
        P.echo_plan([1, 2], 1, -1)


def test_variance_never_increases():
    rng = np.random.default_rng(4)
    for _ in range(200):
        ranks, epr = int(rng.integers(2, 5)), int(rng.integers(1, 3))
        counts = rng.integers(0, 20, size=ranks * epr).tolist()
        plan = P.echo_plan(counts, epr, 2)
        pre = [sum(counts[r * epr:(r + 1) * epr]) for r in range(ranks)]
        assert plan.post_max_load <= max(pre)
        assert np.var(plan.post_loads) <= np.var(pre) + 1e-9


def test_grad_reduce_is_plain_sum():
    rng = np.random.default_rng(5)
    g = rng.normal(size=(3, 3))
    parts = [rng.normal(size=(3, 3)) for _ in range(3)]
    assert np.allclose(O.echo_grad_reduce(parts, g), g + sum(parts))
    assert np.array_equal(O.echo_grad_reduce([np.zeros((3, 3))], g), g)


# -- virtual-expert layout ------------------------------------------------------------

def test_layout_conserves_tokens_and_covers_segments():
    rng = np.random.default_rng(7)
    for _ in range(100):
        n, el, slots = int(rng.integers(2, 5)), int(rng.integers(1, 3)), int(rng.integers(1, 3))
        E = n * el
        counts_all = rng.integers(0, 15, size=(n, E))
        counts_all[:, 0] += rng.integers(0, 40, size=n)  # a hot expert
        plan = P.echo_plan(counts_all.sum(axis=0), el, slots)
        lay = P.echo_layout(counts_all, plan, el, slots)
        el_v = el + slots
        assert lay.counts_v.shape == (n, n * el_v)
        # every source sends all of its rows, split over the expert's segments
        for e in range(E):
            vs = [v for v in lay.seg_v[e] if v >= 0]
            assert lay.counts_v[:, vs].sum(axis=1).tolist() == counts_all[:, e].tolist()
        # post-plan rank loads equal the planner's
        loads = lay.counts_v.sum(axis=0).reshape(n, el_v).sum(axis=1)
        assert loads.tolist() == plan.post_loads
        # each clone slot holds the expert the plan put there
        for c in plan.clones:
            assert c.expert in lay.slot_expert[c.rank].tolist()
        # segments start at 0 and are contiguous, home first
        for e in range(E):
            assert lay.seg_start[e, 0] == 0
            assert lay.seg_v[e, 0] == (e // el) * el_v + e % el


def test_exhaustive_small_minimality():
    """Clone count is minimal (reference test_acceptance.py:373-393 style) on tiny
    instances, by enumeration over per-expert rank subsets."""
    for counts in itertools.product(range(0, 9, 4), repeat=4):
        plan = P.echo_plan(list(counts), 1, 4)
        if plan.best_effort or plan.clone_count == 0:
            continue
        assert plan.clone_count <= sum(1 for c in counts if c > -(-sum(counts) // 4)) * 3
