"""ECHO hot-expert cloning planner — CPU oracle, TEST INFRASTRUCTURE ONLY.

Restates the reference planner (reference pkg/src/moelab/planners.py):
  ExpertClone / EchoPlan           :190-223
  _expert_spillover                :226-240  per-rank overload charged to the rank's
                                             largest experts first
  echo_plan                        :243-290  target = ceil(total / ranks); spare = target -
                                             load; FFD packing; exact refinement for small
                                             instances (<= 12 experts, <= 6 ranks)
  _pack_spillover                  :293-316  first-fit-decreasing, biggest spill takes the
                                             biggest spare (ties: lower rank)
  _exact_min_clones                :319-361  branch and bound, minimal clone count
  rewrite_routing_counts           :364-376  (expert, rank) -> tokens after the plan
  echo_grad_reduce                 :379-387  plain sum of clone gradients into the home
Pinned by tests/test_echo.py against golden plans produced by the reference itself
(tests/golden/make_golden.py -> echo_golden.npz) and the reference's own tests
(test_planners.py:173-311).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Clone:
    expert: int
    rank: int
    tokens: int


@dataclass
class Plan:
    clones: list = field(default_factory=list)
    target_load: int = 0
    pre_max_load: int = 0
    post_loads: list = field(default_factory=list)
    best_effort: bool = False

    @property
    def clone_count(self) -> int:
        return len(self.clones)

    @property
    def post_max_load(self) -> int:
        return max(self.post_loads) if self.post_loads else 0


def rank_loads(counts, epr):
    c = np.asarray(counts, dtype=np.int64).reshape(-1, epr)
    return [int(v) for v in c.sum(axis=1)]


def spillover(counts, epr, target):
    """planners.py:226-240"""
    counts = [int(v) for v in counts]
    out = [0] * len(counts)
    for r, load in enumerate(rank_loads(counts, epr)):
        over = load - target
        ids = sorted(range(r * epr, (r + 1) * epr), key=lambda i: -counts[i])  # stable
        for e in ids:
            if over <= 0:
                break
            out[e] = min(counts[e], over)
            over -= out[e]
    return out


def pack_ffd(spill, spare, slots, epr):
    """planners.py:293-316"""
    spare = list(spare)
    used = [0] * len(spare)
    plan = []
    for e in sorted(range(len(spill)), key=lambda i: -spill[i]):
        need, home = spill[e], e // epr
        while need > 0:
            ok = [r for r in range(len(spare)) if r != home and spare[r] > 0 and used[r] < slots]
            if not ok:
                break
            r = max(ok, key=lambda i: (spare[i], -i))
            take = min(need, spare[r])
            plan.append(Clone(e, r, take))
            spare[r] -= take
            used[r] += 1
            need -= take
    return plan


def exact_min(spill, spare, slots, epr):
    """planners.py:319-361 (depth-first over experts, subsets by increasing size)."""
    hot = [e for e in range(len(spill)) if spill[e] > 0]
    if not hot:
        return []
    best = {"plan": None, "n": float("inf")}
    n_ranks = len(spare)

    def dfs(i, sp, sl, acc):
        if len(acc) >= best["n"]:
            return
        if i == len(hot):
            best["plan"], best["n"] = list(acc), len(acc)
            return
        e = hot[i]
        cand = [r for r in range(n_ranks) if r != e // epr and sp[r] > 0 and sl[r] > 0]
        for size in range(1, len(cand) + 1):
            if len(acc) + size >= best["n"]:
                break
            for subset in itertools.combinations(cand, size):
                if sum(sp[r] for r in subset) < spill[e]:
                    continue
                left, takes = spill[e], []
                for r in sorted(subset, key=lambda q: -sp[q]):
                    t = min(left, sp[r])
                    takes.append((r, t))
                    left -= t
                if left > 0:
                    continue
                for r, t in takes:
                    sp[r] -= t
                    sl[r] -= 1
                    acc.append(Clone(e, r, t))
                dfs(i + 1, sp, sl, acc)
                for r, t in takes:
                    sp[r] += t
                    sl[r] += 1
                    acc.pop()

    dfs(0, list(spare), [slots] * n_ranks, [])
    return best["plan"]


def echo_plan(counts, experts_per_rank: int, spare_slots_per_rank: int,
              exact_limit: int = 12) -> Plan:
    """planners.py:243-290"""
    counts = np.asarray(counts, dtype=np.int64)
    if spare_slots_per_rank < 0:
        raise ValueError("spare slots must be >= 0")
    if len(counts) % experts_per_rank:
        raise ValueError("expert count must be divisible by experts_per_rank")
    epr = experts_per_rank
    loads = rank_loads(counts, epr)
    n_ranks = len(loads)
    target = -(-int(counts.sum()) // n_ranks)
    spill = spillover(counts, epr, target)
    spare = [max(0, target - v) for v in loads]
    best_effort = sum(spill) > sum(spare) or (sum(spill) > 0 and spare_slots_per_rank == 0)
    clones = pack_ffd(spill, spare, spare_slots_per_rank, epr)
    if not best_effort and len(counts) <= exact_limit and n_ranks <= 6:
        ex = exact_min(spill, spare, spare_slots_per_rank, epr)
        if ex is not None and len(ex) < len(clones):
            clones = ex
    post = list(loads)
    for c in clones:
        post[c.rank] += c.tokens
        post[c.expert // epr] -= c.tokens
    return Plan(clones, target, max(loads), post, best_effort)


def rewrite_routing_counts(counts, plan: Plan, experts_per_rank: int) -> dict:
    """planners.py:364-376"""
    out: dict = {}
    moved = [0] * len(counts)
    for c in plan.clones:
        out[(c.expert, c.rank)] = out.get((c.expert, c.rank), 0) + c.tokens
        moved[c.expert] += c.tokens
    for e, v in enumerate(counts):
        key = (e, e // experts_per_rank)
        out[key] = out.get(key, 0) + int(v) - moved[e]
    return out


def echo_grad_reduce(clone_grads, home_grad=None):
    """planners.py:379-387"""
    parts = ([home_grad] if home_grad is not None else []) + list(clone_grads)
    if not parts:
        raise ValueError("nothing to reduce")
    out = parts[0].copy()
    for g in parts[1:]:
        out = out + g
    return out
