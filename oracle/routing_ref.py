"""CPU oracle for the MoE-layer hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference package's numerics oracle
``moelab.routing`` (reference ``pkg/src/moelab/routing.py``), plus the EP byte
model ``perf.a2a_send_volume`` (``pkg/src/moelab/perf.py:62-70``). Each function
cites the reference lines whose behaviour it restates. The restatement is
vectorised (no per-row Python loops) but keeps the reference's semantics exactly:
W_r is [h, E]; sigmoid scores are normalised over all E; top-k ties go to the
lower expert index; probs are NOT renormalised; selection_bias is added to the
scores; capacity keeps the lowest token indices; phantom rows sit at the end of
each expert block; unpermute sums token copies in expert-ascending order.

Pinning: ``tests/test_oracle.py`` checks every function here against golden
vectors produced by the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/moelab`` in the build container and writes
``tests/golden/routing_golden.npz``), and against the reference's own hand
goldens (reference ``pkg/tests/test_routing.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this module. The product path (``paper_2603_07685_b200``) never does.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np


def ceil_div(a: int, b: int) -> int:
    """reference pkg/src/moelab/model.py:353-354"""
    return -(-a // b)


@dataclass(frozen=True)
class RoutingDecision:
    """reference routing.py:16-39 (same fields, same effective_counts rule)."""

    probs: np.ndarray
    routing_map: np.ndarray
    counts: np.ndarray
    scores: np.ndarray
    dropped: np.ndarray | None = None
    phantom_rows: np.ndarray | None = None

    @property
    def num_tokens(self) -> int:
        return self.routing_map.shape[0]

    @property
    def num_experts(self) -> int:
        return self.routing_map.shape[1]

    def effective_counts(self) -> np.ndarray:
        """routing.py:33-39: selected − dropped + phantom, per expert."""
        kept = self.routing_map if self.dropped is None else (self.routing_map & ~self.dropped)
        eff = kept.sum(axis=0).astype(np.int64)
        if self.phantom_rows is not None:
            eff = eff + np.asarray(self.phantom_rows, dtype=np.int64)
        return eff


@dataclass(frozen=True)
class ExpertParams:
    """routing.py:42-52. w1 ("up") [m,h], w2 [h,m], gate [m,h] per expert (out x in)."""

    w1: list
    w2: list
    gate: list | None = None

    @property
    def num_experts(self) -> int:
        return len(self.w1)


def silu(x):
    """routing.py:55-56"""
    return x * (1.0 / (1.0 + np.exp(-x)))


def expert_activation(params: ExpertParams, expert: int, x_rows):
    """routing.py:59-64: silu(x gate^T) * (x w1^T), or silu(x w1^T) when ungated."""
    up = x_rows @ params.w1[expert].T
    if params.gate is None:
        return silu(up)
    return silu(x_rows @ params.gate[expert].T) * up


def expert_forward(params: ExpertParams, expert: int, x_rows):
    """routing.py:67-68"""
    return expert_activation(params, expert, x_rows) @ params.w2[expert].T


def _scores(logits, score):
    """routing.py:85-93"""
    if score == "softmax":
        z = np.exp(logits - logits.max(axis=1, keepdims=True))
        return z / z.sum(axis=1, keepdims=True)
    if score == "sigmoid":
        s = 1.0 / (1.0 + np.exp(-logits))
        return s / s.sum(axis=1, keepdims=True)
    raise ValueError(f"unknown score function {score!r}")


def topk_lowest_index(values, k):
    """Indices of the k largest entries per row, ties to the lower index
    (routing.py:96-98: stable argsort of -values). Returned ascending by index."""
    order = np.argsort(-values, axis=1, kind="stable")[:, :k]
    return np.sort(order, axis=1)


def route(hidden, w_r, score: str = "softmax", top_k: int = 1, selection_bias=None):
    """routing.py:71-108"""
    logits = hidden @ w_r
    if not np.isfinite(logits).all():
        raise ValueError("router logits are not finite")
    t, e = logits.shape
    if top_k > e:
        raise ValueError(f"top_k={top_k} exceeds num_experts={e}")
    scores = _scores(logits, score)
    select_on = scores if selection_bias is None else scores + selection_bias
    top = topk_lowest_index(select_on, top_k)
    routing_map = np.zeros((t, e), dtype=bool)
    np.put_along_axis(routing_map, top, True, axis=1)
    return RoutingDecision(
        probs=np.where(routing_map, scores, 0.0),
        routing_map=routing_map,
        counts=routing_map.sum(axis=0).astype(np.int64),
        scores=scores,
    )


def aux_loss(decision: RoutingDecision, coeff: float) -> float:
    """routing.py:111-120: coeff * E * sum_i f_i P_i, f = counts / sum(map)."""
    total = max(int(decision.routing_map.sum()), 1)
    f = decision.counts / total
    p = decision.scores.mean(axis=0)
    return float(coeff * decision.num_experts * np.dot(f, p))


def aux_loss_grad_wr(hidden, w_r, top_k: int, coeff: float, score: str = "softmax"):
    """routing.py:123-137 (softmax only; f treated as constant)."""
    d = route(hidden, w_r, score=score, top_k=top_k)
    if score != "softmax":
        raise NotImplementedError("analytic gradient implemented for softmax scoring")
    t, e = d.scores.shape
    g = coeff * e * (d.counts / max(int(d.routing_map.sum()), 1)) / t  # dL/ds_ti, per i
    s = d.scores
    dl = s * (g[None, :] - (s * g[None, :]).sum(axis=1, keepdims=True))
    return hidden.T @ dl


def auxfree_bias_update(counts, bias, step: float):
    """routing.py:140-146"""
    if step <= 0:
        raise ValueError("step must be > 0")
    return bias + step * np.sign(counts.mean() - counts)


def _row_id_map(decision: RoutingDecision) -> np.ndarray:
    """routing.py:155-163 (vectorised): expert-major, ascending token within an
    expert, dropped slots skipped, phantom rows (-1) appended per expert."""
    kept = decision.routing_map if decision.dropped is None else (
        decision.routing_map & ~decision.dropped)
    blocks = []
    for e in range(decision.num_experts):
        src = np.flatnonzero(kept[:, e]).astype(np.int64)
        blocks.append(src)
        if decision.phantom_rows is not None and int(decision.phantom_rows[e]) > 0:
            blocks.append(np.full(int(decision.phantom_rows[e]), -1, dtype=np.int64))
    return np.concatenate(blocks) if blocks else np.zeros(0, dtype=np.int64)


def permute(tokens, decision: RoutingDecision):
    """routing.py:149-168"""
    row_id_map = _row_id_map(decision)
    out = np.zeros((len(row_id_map), tokens.shape[1]), dtype=tokens.dtype)
    real = row_id_map >= 0
    out[real] = tokens[row_id_map[real]]
    return out, row_id_map


def unpermute_sum(rows, row_id_map, num_tokens: int):
    """routing.py:171-177: out[src] += rows[r] in row order (expert-ascending per
    token). np.add.at accumulates unbuffered in index order, matching the loop."""
    out = np.zeros((num_tokens, rows.shape[1]), dtype=rows.dtype)
    real = row_id_map >= 0
    np.add.at(out, row_id_map[real], rows[real])
    return out


def expert_slices(decision: RoutingDecision):
    """routing.py:180-186"""
    counts = decision.effective_counts()
    starts = np.concatenate([[0], np.cumsum(counts)])
    return [(e, slice(int(starts[e]), int(starts[e + 1]))) for e in range(len(counts))]


def _row_probs(decision, row_id_map):
    """prob of each permuted row (0 for phantom rows), expert taken from its block."""
    p = np.zeros(len(row_id_map), dtype=decision.probs.dtype)
    for e, sl in expert_slices(decision):
        src = row_id_map[sl]
        real = src >= 0
        idx = np.arange(sl.start, sl.stop)[real]
        p[idx] = decision.probs[src[real], e]
    return p


def combine_standard(tokens, decision: RoutingDecision, params: ExpertParams):
    """routing.py:189-201: weight expert outputs by p, then unpermute-sum."""
    permuted, row_id_map = permute(tokens, decision)
    out_rows = np.zeros_like(permuted)
    for e, sl in expert_slices(decision):
        if sl.stop > sl.start:
            out_rows[sl] = expert_forward(params, e, permuted[sl])
    real = row_id_map >= 0
    out_rows[real] *= _row_probs(decision, row_id_map)[real, None]
    return unpermute_sum(out_rows, row_id_map, decision.num_tokens)


def combine_mem_efficient(tokens, decision: RoutingDecision, params: ExpertParams):
    """routing.py:204-223: p absorbed into the activation before fc2."""
    permuted, row_id_map = permute(tokens, decision)
    width = params.w2[0].shape[0]
    rows = np.zeros((len(row_id_map), width), dtype=tokens.dtype)
    probs = _row_probs(decision, row_id_map)
    for e, sl in expert_slices(decision):
        if sl.stop <= sl.start:
            continue
        acts = expert_activation(params, e, permuted[sl])
        src = row_id_map[sl]
        acts = np.where((src >= 0)[:, None], acts * probs[sl, None], acts)
        rows[sl] = acts @ params.w2[e].T
    # phantom rows are not scattered back (routing.py:219-222)
    return unpermute_sum(rows, row_id_map, decision.num_tokens)


def expert_capacity(capacity_factor: float, tokens: int, top_k: int, num_experts: int) -> int:
    """routing.py:250-251"""
    return ceil_div(int(round(capacity_factor * tokens * top_k)), num_experts)


def apply_capacity(decision: RoutingDecision, capacity_factor: float, pad: bool = False):
    """routing.py:226-247: keep the first C selections of each expert by token index."""
    if capacity_factor <= 0:
        raise ValueError("capacity_factor must be > 0")
    t = decision.num_tokens
    k = int(round(decision.routing_map.sum() / max(t, 1)))
    cap = expert_capacity(capacity_factor, t, k, decision.num_experts)
    # rank of each selection within its expert column, in token order
    rank = np.cumsum(decision.routing_map, axis=0) - 1
    dropped = decision.routing_map & (rank >= cap)
    phantom = None
    if pad:
        phantom = (cap - np.minimum(decision.routing_map.sum(axis=0), cap)).astype(np.int64)
    return replace(decision, dropped=dropped, phantom_rows=phantom)


def moe_output_with_residual(tokens, decision: RoutingDecision, params: ExpertParams):
    """routing.py:254-262: fully dropped tokens pass through on the residual."""
    out = combine_standard(tokens, decision, params)
    if decision.dropped is not None:
        alive = (decision.routing_map & ~decision.dropped).any(axis=1)
        out[~alive] += tokens[~alive]
    return out


def latent_moe_forward(x, w_down, w_up, experts: ExpertParams, decision: RoutingDecision,
                       shared: ExpertParams | None = None):
    """routing.py:265-279"""
    out = combine_standard(x @ w_down.T, decision, experts) @ w_up.T
    if shared is not None:
        for j in range(shared.num_experts):
            out = out + expert_forward(shared, j, x)
    return out


def upcycle(dense_w1, dense_w2, granularity: int, duplication: int, dense_gate=None):
    """routing.py:282-309 (init-only; oracle-only)."""
    inter, h = dense_w1.shape
    if inter % granularity != 0:
        raise ValueError(f"intermediate dim {inter} not divisible by granularity {granularity}")
    shard = inter // granularity
    n = granularity * duplication
    idx = [slice(g * shard, (g + 1) * shard) for g in range(granularity)] * duplication
    params = ExpertParams(
        w1=[dense_w1[s].copy() for s in idx],
        w2=[dense_w2[:, s] * n for s in idx],
        gate=[dense_gate[s].copy() for s in idx] if dense_gate is not None else None,
    )
    return params, np.zeros((h, n))


def routing_map_pad(decision: RoutingDecision, multiple: int, num_filler_tokens=None):
    """routing.py:312-325 (uses raw routing_map counts; replaces phantom_rows)."""
    if multiple < 1:
        raise ValueError("multiple must be >= 1")
    needed = (-decision.routing_map.sum(axis=0)) % multiple
    if num_filler_tokens is not None and needed.max(initial=0) > num_filler_tokens:
        raise ValueError(
            f"insufficient filler capacity: need {int(needed.max())} rows per "
            f"expert, have {num_filler_tokens}")
    return replace(decision, phantom_rows=needed.astype(np.int64))


def a2a_send_volume(tokens: int, top_k: int, hidden: int, ep: int, width: float = 2.0) -> float:
    """reference pkg/src/moelab/perf.py:62-70: per-GPU bytes of one all-to-all."""
    if ep < 1:
        raise ValueError("ep must be >= 1")
    return tokens * top_k * hidden * width * (ep - 1) / ep


def expert_rank(expert: int, num_experts: int, ep: int) -> int:
    """EP placement e -> rank e // (E/EP) (reference planners.py:299,
    tests/test_perf.py:27-33)."""
    return expert // (num_experts // ep)
