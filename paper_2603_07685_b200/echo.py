"""ECHO hot-expert cloning for the EP layer.

Planning is host-side integer logic with the reference's semantics (reference
pkg/src/moelab/planners.py:243-389): tokens above the balanced rank load (ceil of the
mean) are spilled from each overloaded rank's largest experts to clone slots on ranks with
spare capacity, first-fit-decreasing, refined by an exact minimum-clone search on small
instances. Execution maps every (expert, segment) to a *virtual expert* that lives on the
rank serving it:

  * expert e's token copies, in global order (source rank, token) = the oracle's permute
    order, are split into consecutive segments: the home rank keeps the first
    home_n = count - sum(clone tokens), each clone takes the next `tokens` copies;
  * rank r serves el + S virtual experts: its el own experts, then S clone slots; virtual
    expert v = r * (el + S) + group; a clone slot computes with a copy of the home
    expert's weights, and its weight gradient is summed into the home expert's
    (echo_grad_reduce, planners.py:379-387);
  * the device kernels are the ordinary EP kernels run over virtual experts, so rows of
    a segment stay in global order and parity with the single-process oracle holds.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np


@dataclass
class CloneSpec:
    expert: int
    rank: int
    tokens: int


@dataclass
class EchoPlan:
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


class _Planner:
    def __init__(self, counts, epr: int, slots: int):
        self.counts = np.asarray(counts, dtype=np.int64)
        self.epr, self.slots = epr, slots
        self.loads = self.counts.reshape(-1, epr).sum(axis=1)
        self.ranks = len(self.loads)
        self.target = int(-(-int(self.counts.sum()) // self.ranks))
        self.spill = self._spill()
        self.spare = np.maximum(self.target - self.loads, 0)

    def _spill(self):
        spill = np.zeros_like(self.counts)
        for r in range(self.ranks):
            over = int(self.loads[r]) - self.target
            ids = r * self.epr + np.argsort(-self.counts[r * self.epr:(r + 1) * self.epr],
                                            kind="stable")
            for e in ids:
                if over <= 0:
                    break
                spill[e] = min(int(self.counts[e]), over)
                over -= int(spill[e])
        return spill

    def greedy(self):
        spare = self.spare.copy()
        used = np.zeros(self.ranks, dtype=np.int64)
        out = []
        for e in np.argsort(-self.spill, kind="stable"):
            need, home = int(self.spill[e]), int(e) // self.epr
            while need > 0:
                best = -1
                for r in range(self.ranks):  # largest spare, lowest rank on ties
                    if r != home and spare[r] > 0 and used[r] < self.slots:
                        if best < 0 or spare[r] > spare[best]:
                            best = r
                if best < 0:
                    break
                take = min(need, int(spare[best]))
                out.append(CloneSpec(int(e), best, take))
                spare[best] -= take
                used[best] += 1
                need -= take
        return out

    def exact(self):
        hot = [int(e) for e in np.flatnonzero(self.spill > 0)]
        if not hot:
            return []
        state = {"best": None, "n": np.inf}
        spare = [int(v) for v in self.spare]
        slots = [self.slots] * self.ranks

        def place(i, acc):
            if len(acc) >= state["n"]:
                return
            if i == len(hot):
                state["best"], state["n"] = list(acc), len(acc)
                return
            e = hot[i]
            need = int(self.spill[e])
            usable = [r for r in range(self.ranks)
                      if r != e // self.epr and spare[r] > 0 and slots[r] > 0]
            for size in range(1, len(usable) + 1):
                if len(acc) + size >= state["n"]:
                    break
                for combo in itertools.combinations(usable, size):
                    if sum(spare[r] for r in combo) < need:
                        continue
                    rest, takes = need, []
                    for r in sorted(combo, key=lambda q: -spare[q]):
                        t = min(rest, spare[r])
                        takes.append((r, t))
                        rest -= t
                    if rest:
                        continue
                    for r, t in takes:
                        spare[r] -= t
                        slots[r] -= 1
                    place(i + 1, acc + [CloneSpec(e, r, t) for r, t in takes])
                    for r, t in takes:
                        spare[r] += t
                        slots[r] += 1

        place(0, [])
        return state["best"]


def echo_plan(counts, experts_per_rank: int, spare_slots_per_rank: int,
              exact_limit: int = 12) -> EchoPlan:
    """Hot-expert cloning plan (same contract as reference planners.echo_plan)."""
    if spare_slots_per_rank < 0:
        raise ValueError("spare slots must be >= 0")
    if len(counts) % experts_per_rank:
        raise ValueError("expert count must be divisible by experts_per_rank")
    pl = _Planner(counts, experts_per_rank, spare_slots_per_rank)
    total_spill = int(pl.spill.sum())
    best_effort = total_spill > int(pl.spare.sum()) or (
        total_spill > 0 and spare_slots_per_rank == 0)
    clones = pl.greedy()
    if not best_effort and len(pl.counts) <= exact_limit and pl.ranks <= 6:
        ex = pl.exact()
        if ex is not None and len(ex) < len(clones):
            clones = ex
    post = [int(v) for v in pl.loads]
    for c in clones:
        post[c.rank] += c.tokens
        post[c.expert // experts_per_rank] -= c.tokens
    return EchoPlan(clones, pl.target, int(pl.loads.max()), post, best_effort)


@dataclass
class EchoLayout:
    """Virtual-expert layout of one forward (identical on every rank)."""

    slots: int                 # S clone slots per rank
    el_v: int                  # el + S groups per rank
    seg_start: np.ndarray      # [E, NS] global start position of each segment (int32 max pad)
    seg_v: np.ndarray          # [E, NS] virtual expert of each segment (-1 unused)
    counts_v: np.ndarray       # [n, E_v] rows source s sends to virtual expert v
    slot_expert: np.ndarray    # [n, S] global expert held by each clone slot (-1 empty)
    plan: EchoPlan


def echo_layout(counts_all, plan: EchoPlan, el: int, slots: int) -> EchoLayout:
    """Segments and virtual experts from the gathered per-source counts [n, E]."""
    counts_all = np.asarray(counts_all, dtype=np.int64)
    n, E = counts_all.shape
    el_v = el + slots
    total = counts_all.sum(axis=0)
    per_e: list = [[] for _ in range(E)]
    slot_expert = np.full((n, slots), -1, dtype=np.int64)
    used = np.zeros(n, dtype=np.int64)
    for c in plan.clones:
        g = el + int(used[c.rank])
        if used[c.rank] >= slots:
            raise ValueError("plan uses more clone slots than configured")
        slot_expert[c.rank, used[c.rank]] = c.expert
        used[c.rank] += 1
        per_e[c.expert].append((c.rank * el_v + g, c.tokens))
    ns = 1 + max((len(s) for s in per_e), default=0)
    big = np.iinfo(np.int32).max
    seg_start = np.full((E, ns), big, dtype=np.int64)
    seg_v = np.full((E, ns), -1, dtype=np.int64)
    counts_v = np.zeros((n, n * el_v), dtype=np.int64)
    prefix = np.cumsum(counts_all, axis=0) - counts_all        # [n, E] global start per src
    for e in range(E):
        home = e // el
        clone_tokens = sum(t for _, t in per_e[e])
        segs = [(home * el_v + e % el, int(total[e]) - clone_tokens)] + per_e[e]
        start = 0
        for j, (v, cnt) in enumerate(segs):
            seg_start[e, j] = start
            seg_v[e, j] = v
            lo, hi = start, start + cnt
            # rows each source contributes to [lo, hi): its global range intersected
            a = prefix[:, e]
            b = a + counts_all[:, e]
            counts_v[:, v] += np.clip(np.minimum(b, hi) - np.maximum(a, lo), 0, None)
            start = hi
    return EchoLayout(slots, el_v, seg_start, seg_v, counts_v, slot_expert, plan)
