"""Device-side building blocks of the MoE layer, one thin wrapper per C-ABI call.

Everything here enqueues work on torch's current CUDA stream through
``libmoe_b200.so``; nothing synchronises with the host unless a function's
docstring says so. Reference anchors (pkg/src/moelab/routing.py) are given per
function; the kernels cite them line by line.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import torch

from . import _lib, gemm

SCORE_FN = {"softmax": 0, "sigmoid": 1}
ALIGN = 128
ROUTER_NPAD = 256  # router logits GEMM N tile


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _p(t):
    return None if t is None else t.data_ptr()


def ceil_to(a: int, b: int) -> int:
    return -(-a // b) * b


# ---------------------------------------------------------------------------- router

@dataclass
class RouterOut:
    logits: torch.Tensor       # [ceil128(T), Epad] fp32 (rows >= T, cols >= E unused)
    topk_idx: torch.Tensor     # [T, K] int32, ascending expert
    topk_prob: torch.Tensor    # [T, K] fp32, unbiased score of the selection
    counts: torch.Tensor       # [E] int32 (pre-drop)
    aux: torch.Tensor          # [] fp32 device scalar, aux_loss(coeff)
    aux_grad: torch.Tensor     # [E] fp32, d aux / d s_te = coeff*E*f_e/T
    mean_scores: torch.Tensor  # [E] fp32, P_e
    status: torch.Tensor       # [1] int32, bit0 = non-finite logits
    scores: torch.Tensor | None = None  # [T, E] fp32 when requested
    w_r: torch.Tensor | None = None     # [h, E] bf16: set on the small-E path (backward operand)


# Small-E CUDA-core router (moe_router_fused + CUDA-core backward) instead of the tcgen05
# logits / gradient GEMMs padded to 256 columns. Correct (tests/test_router_gpu.py) but measured
# SLOWER on B200 (tools/router_probe.py, profiles/r02_router_probe.txt: Mixtral shape fwd+bwd
# chain 289 us vs 244 us): the x . W_r product at E = 8 is ~32 FLOP per x element over three
# passes, which is CUDA-core instruction bound, while the padded tensor-core tiles stay near
# the HBM floor. Opt-in with MOE_ROUTER_SMALL=1.
ROUTER_SMALL = os.environ.get("MOE_ROUTER_SMALL", "0") == "1"


def router_small(num_experts: int, hidden: int) -> bool:
    """True when the small-E CUDA-core router is enabled (ROUTER_SMALL) and eligible
    (E <= 16, W_r^T fits shared memory); else the tcgen05 logits GEMM path runs."""
    return ROUTER_SMALL and bool(_lib.query("moe_router_small_ok", num_experts, hidden))


def stage_router(w_r: torch.Tensor):
    """Per-forward router-weight operands: (W_r^T padded, W_r padded) for the tcgen05 path,
    (None, None) on the small-E path (which reads W_r [h, E] as is)."""
    h, e = w_r.shape
    if router_small(e, h):
        return None, None
    return stage_router_weight(w_r)


def stage_router_weight(w_r: torch.Tensor, want_t=True, want_pad=True):
    """W_r [h, E] bf16 -> (W_r^T zero-padded [1, Epad, h], W_r zero-padded [1, h, Epad])."""
    h, e = w_r.shape
    epad = ceil_to(e, ROUTER_NPAD)
    wt = torch.empty((1, epad, h), dtype=torch.bfloat16, device=w_r.device) if want_t else None
    wp = torch.empty((1, h, epad), dtype=torch.bfloat16, device=w_r.device) if want_pad else None
    _lib.call("moe_stage_router_weight", w_r.data_ptr(), h, e, epad, _p(wt), _p(wp), _stream())
    return wt, wp


def router_forward(x: torch.Tensor, w_r: torch.Tensor, top_k: int, score: str = "softmax",
                   selection_bias: torch.Tensor | None = None, coeff: float = 0.0,
                   want_scores: bool = False, w_r_t: torch.Tensor | None = None) -> RouterOut:
    """route() (routing.py:71-108) + aux_loss() (:111-120) on the device.

    logits = x @ W_r on the tcgen05 GEMM (fp32 accumulate), then a warp-per-token
    score / top-k / statistics kernel. No host sync.
    """
    t, h = x.shape
    e = w_r.shape[1]
    dev = x.device
    if w_r_t is None and router_small(e, h):
        return _router_forward_small(x, w_r, top_k, score, selection_bias, coeff, want_scores)
    if w_r_t is None:
        w_r_t, _ = stage_router_weight(w_r, want_pad=False)
    epad = w_r_t.shape[1]
    rows = max(ceil_to(t, ALIGN), ALIGN)
    nmb = torch.full((1,), rows // ALIGN, dtype=torch.int32, device=dev)
    be = torch.zeros((rows // ALIGN,), dtype=torch.int32, device=dev)
    logits = torch.empty((rows, epad), dtype=torch.float32, device=dev)
    if t > 0:
        gemm.gemm_f32(x, w_r_t, be, nmb, out=logits, max_rows=rows)
    topk_idx = torch.empty((t, top_k), dtype=torch.int32, device=dev)
    topk_prob = torch.empty((t, top_k), dtype=torch.float32, device=dev)
    counts = torch.empty((e,), dtype=torch.int32, device=dev)
    npart = _lib.query("moe_router_num_partials", t)
    partials = torch.empty((max(npart, 1), e), dtype=torch.float32, device=dev)
    status = torch.empty((1,), dtype=torch.int32, device=dev)
    scores = torch.empty((t, e), dtype=torch.float32, device=dev) if want_scores else None
    bias = None
    if selection_bias is not None:
        bias = selection_bias.to(device=dev, dtype=torch.float32).contiguous()
    _lib.call("moe_router_topk", logits.data_ptr(), epad, t, e, top_k, SCORE_FN[score], _p(bias),
              topk_idx.data_ptr(), topk_prob.data_ptr(), _p(scores), counts.data_ptr(),
              partials.data_ptr(), status.data_ptr(), _stream())
    aux = torch.empty((), dtype=torch.float32, device=dev)
    aux_grad = torch.empty((e,), dtype=torch.float32, device=dev)
    mean_scores = torch.empty((e,), dtype=torch.float32, device=dev)
    _lib.call("moe_router_finalize", counts.data_ptr(), partials.data_ptr(), t, top_k, e,
              float(coeff), aux.data_ptr(), aux_grad.data_ptr(), mean_scores.data_ptr(), _stream())
    return RouterOut(logits, topk_idx, topk_prob, counts, aux, aux_grad, mean_scores, status,
                     scores)


def _router_forward_small(x, w_r, top_k, score, selection_bias, coeff, want_scores):
    """route() + aux_loss() for E <= 16: one kernel computes the logits (CUDA cores, x read
    once), scores, top-k, counts and score partials (moe_router_fused)."""
    t, h = x.shape
    e = w_r.shape[1]
    dev = x.device
    w_r = w_r.to(torch.bfloat16).contiguous()
    logits = torch.empty((t, e), dtype=torch.float32, device=dev)
    topk_idx = torch.empty((t, top_k), dtype=torch.int32, device=dev)
    topk_prob = torch.empty((t, top_k), dtype=torch.float32, device=dev)
    counts = torch.empty((e,), dtype=torch.int32, device=dev)
    npart = _lib.query("moe_router_num_partials", t)
    partials = torch.empty((max(npart, 1), e), dtype=torch.float32, device=dev)
    status = torch.empty((1,), dtype=torch.int32, device=dev)
    scores = torch.empty((t, e), dtype=torch.float32, device=dev) if want_scores else None
    bias = None
    if selection_bias is not None:
        bias = selection_bias.to(device=dev, dtype=torch.float32).contiguous()
    _lib.call("moe_router_fused", x.data_ptr(), t, h, w_r.data_ptr(), e, top_k, SCORE_FN[score],
              _p(bias), logits.data_ptr(), topk_idx.data_ptr(), topk_prob.data_ptr(),
              _p(scores), counts.data_ptr(), partials.data_ptr(), status.data_ptr(), _stream())
    aux = torch.empty((), dtype=torch.float32, device=dev)
    aux_grad = torch.empty((e,), dtype=torch.float32, device=dev)
    mean_scores = torch.empty((e,), dtype=torch.float32, device=dev)
    _lib.call("moe_router_finalize", counts.data_ptr(), partials.data_ptr(), t, top_k, e,
              float(coeff), aux.data_ptr(), aux_grad.data_ptr(), mean_scores.data_ptr(), _stream())
    return RouterOut(logits, topk_idx, topk_prob, counts, aux, aux_grad, mean_scores, status,
                     scores, w_r)


def _router_backward_small(x, r: RouterOut, dprob, score, aux_g, want_dx=True):
    t, h = x.shape
    e = r.counts.shape[0]
    k = r.topk_idx.shape[1]
    dev = x.device
    dl = torch.empty((t, e), dtype=torch.float32, device=dev)
    _lib.call("moe_router_bwd_f32", r.logits.data_ptr(), r.logits.shape[1], t, e, k,
              SCORE_FN[score], r.topk_idx.data_ptr(), dprob.data_ptr(), _p(aux_g),
              dl.data_ptr(), _stream())
    ws = torch.empty((max(int(_lib.query("moe_router_wgrad_small_ws", t, h, e)), 1),),
                     dtype=torch.float32, device=dev)
    dw = torch.empty((h, e), dtype=torch.float32, device=dev)
    _lib.call("moe_router_wgrad_small", x.data_ptr(), t, h, dl.data_ptr(), e, ws.data_ptr(),
              dw.data_ptr(), _stream())
    dx = None
    if want_dx:
        dx = torch.empty((t, h), dtype=torch.bfloat16, device=dev)
        _lib.call("moe_router_dx_small", dl.data_ptr(), t, e, r.w_r.data_ptr(), h, dx.data_ptr(),
                  _stream())
    return dw, dx


def router_backward(x: torch.Tensor, w_r_pad: torch.Tensor | None, r: RouterOut,
                    dprob: torch.Tensor, score: str,
                    aux_scale: float | torch.Tensor | None = 1.0, num_splits: int = 8):
    """Router backward (aux part = routing.py:123-137).

    Returns (dW_r [h, E] fp32, dX_router [>= T, h] bf16 or None).
    aux_scale multiplies the aux-loss gradient (the upstream grad of the aux output).
    w_r_pad: the staged [h, 256k] router weight of the tcgen05 path (None on the small-E path,
    which uses r.w_r).
    """
    if r.w_r is not None:
        aux_g = None
        if aux_scale is not None:
            aux_g = r.aux_grad if (isinstance(aux_scale, float) and aux_scale == 1.0) else (
                r.aux_grad * aux_scale)
        return _router_backward_small(x, r, dprob, score, aux_g)
    t, h = x.shape
    e = r.counts.shape[0]
    k = r.topk_idx.shape[1]
    epad = r.logits.shape[1]
    rows = r.logits.shape[0]
    dev = x.device
    dl = torch.empty((rows, epad), dtype=torch.bfloat16, device=dev)
    aux_g = None
    if aux_scale is not None:
        aux_g = r.aux_grad if (isinstance(aux_scale, float) and aux_scale == 1.0) else (
            r.aux_grad * aux_scale)
    _lib.call("moe_router_bwd", r.logits.data_ptr(), epad, t, e, k, SCORE_FN[score],
              r.topk_idx.data_ptr(), dprob.data_ptr(), _p(aux_g), dl.data_ptr(), epad, _stream())
    if t == 0:
        return torch.zeros((h, e), dtype=torch.float32, device=dev), None
    # dW_r = x^T dl : split-K over token chunks (multiples of 64 rows), fixed-order reduce
    splits = max(1, min(num_splits, -(-t // 64)))
    chunk = ceil_to(-(-t // splits), 64)
    # chunk * splits >= ceil64(t), so the clamp makes the last offset exactly ceil64(t);
    # built on the device (no host->device scalar copy, hence no stream sync)
    offs_t = (torch.arange(splits + 1, dtype=torch.int32, device=dev) * chunk).clamp_(
        max=ceil_to(t, 64))
    parts = gemm.wgrad_f32(x, dl, offs_t, splits, max_rows=t)
    dw = torch.empty((h, e), dtype=torch.float32, device=dev)
    _lib.call("moe_reduce_groups_f32", parts.data_ptr(), splits, h, epad, e, dw.data_ptr(),
              _stream())
    # dX_router = dl @ W_r^T  (fc2-shaped GEMM: K = Epad, N = h)
    nmb = torch.full((1,), rows // ALIGN, dtype=torch.int32, device=dev)
    be = torch.zeros((rows // ALIGN,), dtype=torch.int32, device=dev)
    dx = gemm.fc2_fwd(dl, w_r_pad, be, nmb)
    return dw, dx


# ---------------------------------------------------------------------------- plan

@dataclass
class Plan:
    """Padded dispatch plan (permute() routing.py:149-168 + apply_capacity() :226-247)."""

    T: int
    K: int
    E: int
    capacity: int      # -1 = dropless
    pad: bool
    max_rows: int
    meta: torch.Tensor          # [3] int32: num_m_blocks, padded rows, compact rows
    off_pad: torch.Tensor       # [E+1]
    off_c: torch.Tensor         # [E+1]
    kept: torch.Tensor          # [E]
    eff: torch.Tensor           # [E]
    counts: torch.Tensor        # [E] (pre-drop)
    block_expert: torch.Tensor  # [max_rows/128]
    inv_map: torch.Tensor       # [T, K] dest row or -1 (dropped)
    row_src: torch.Tensor       # [max_rows] source token or -1
    row_prob: torch.Tensor      # [max_rows] fp32
    status: torch.Tensor        # [1] bit1 = overflow of max_rows
    align: int = ALIGN          # expert block alignment (256: CTA-pair GEMM engine)

    @property
    def num_m_blocks(self) -> torch.Tensor:
        return self.meta[0:1]

    @property
    def pair(self) -> bool:
        return self.align == 2 * ALIGN


def plan_max_rows(T: int, K: int, E: int, capacity: int = -1, pad: bool = False,
                  align: int = ALIGN) -> int:
    """Static upper bound of the padded plan's rows (buffer sizing, no host sync)."""
    if capacity < 0:
        bound = T * K + E * (align - 1)
    elif pad:
        bound = E * ceil_to(capacity, align)
    else:
        bound = min(T * K, E * capacity) + E * (align - 1)
    return max(ceil_to(bound, align), align)


def pick_align(T: int, K: int, E: int) -> int:
    """256-row expert blocks (CTA-pair GEMM engine) when experts are large enough that the
    extra padding is negligible; 128 otherwise (e.g. DeepSeek-shape at EP=1, ~128 rows).
    MOE_B200_ALIGN=128|256 overrides (A/B measurements)."""
    forced = os.environ.get("MOE_B200_ALIGN")
    if forced:
        return int(forced)
    return 2 * ALIGN if T * K >= 8 * 2 * ALIGN * E else ALIGN


def build_plan(topk_idx: torch.Tensor, topk_prob: torch.Tensor | None, E: int,
               capacity: int = -1, pad: bool = False, max_rows: int | None = None,
               phantom: torch.Tensor | None = None, phantom_max: int = 0,
               cap_e: torch.Tensor | None = None, compact: bool = False,
               align: int = ALIGN) -> Plan:
    """phantom: optional device int32 [E] extra zero rows per expert (routing_map_pad);
    phantom_max bounds it for buffer sizing. cap_e: optional device int32 [E] per-expert
    capacity (EP global-position drops). compact: no 128-row alignment (EP send layout)."""
    t, k = topk_idx.shape
    dev = topk_idx.device
    if max_rows is None:
        if compact:
            max_rows = max(t * k, 1)
        else:
            max_rows = (plan_max_rows(t, k, E, capacity, pad, align)
                        + ceil_to(E * phantom_max, align))
    i32 = dict(dtype=torch.int32, device=dev)
    meta = torch.empty((3,), **i32)
    off_pad = torch.empty((E + 1,), **i32)
    off_c = torch.empty((E + 1,), **i32)
    kept = torch.empty((E,), **i32)
    eff = torch.empty((E,), **i32)
    counts = torch.empty((E,), **i32)
    block_expert = None if compact else torch.empty((max_rows // ALIGN,), **i32)
    inv_map = torch.empty((t, k), **i32)
    row_src = torch.empty((max_rows,), **i32)
    row_prob = torch.empty((max_rows,), dtype=torch.float32, device=dev)
    ws = torch.empty((max(int(_lib.query("moe_permute_workspace_ints", t, k, E)), 1),), **i32)
    status = torch.empty((1,), **i32)
    _lib.call("moe_permute_plan", topk_idx.data_ptr(), _p(topk_prob), t, k, E, int(capacity),
              _p(cap_e), int(bool(pad)), _p(phantom), 1 if compact else align, max_rows,
              meta.data_ptr(), off_pad.data_ptr(), off_c.data_ptr(), kept.data_ptr(),
              eff.data_ptr(), counts.data_ptr(), _p(block_expert), inv_map.data_ptr(),
              row_src.data_ptr(), row_prob.data_ptr(), ws.data_ptr(), status.data_ptr(),
              _stream())
    return Plan(t, k, E, int(capacity), bool(pad), max_rows, meta, off_pad, off_c, kept, eff,
                counts, block_expert, inv_map, row_src, row_prob, status,
                1 if compact else align)


def compact_row_id_map(plan: Plan, n_compact: int | None = None):
    """Oracle-layout row_id_map (int64) + compact->padded index. Syncs if n_compact is None."""
    if n_compact is None:
        n_compact = int(plan.meta[2].item())
    dev = plan.meta.device
    rmap = torch.empty((n_compact,), dtype=torch.int64, device=dev)
    c2p = torch.empty((n_compact,), dtype=torch.int32, device=dev)
    if n_compact:
        _lib.call("moe_permute_compact_map", plan.meta.data_ptr(), plan.off_c.data_ptr(),
                  plan.off_pad.data_ptr(), plan.E, plan.row_src.data_ptr(), rmap.data_ptr(),
                  c2p.data_ptr(), n_compact, _stream())
    return rmap, c2p


def permute_gather(x: torch.Tensor, plan: Plan, out: torch.Tensor | None = None):
    t, h = x.shape
    if out is None:
        out = torch.empty((plan.max_rows, h), dtype=x.dtype, device=x.device)
    _lib.call("moe_permute_gather", x.data_ptr(), t, plan.K, h, plan.inv_map.data_ptr(),
              plan.row_src.data_ptr(), plan.meta.data_ptr(), out.data_ptr(), _stream())
    return out


def zero_pad_rows(rows: torch.Tensor, plan: Plan):
    _lib.call("moe_zero_pad_rows", plan.meta.data_ptr(), plan.row_src.data_ptr(), rows.shape[1],
              rows.data_ptr(), _stream())


def gather_rows(src: torch.Tensor, index: torch.Tensor, n: int | None = None,
                n_dev: torch.Tensor | None = None, out: torch.Tensor | None = None):
    """out[r] = src[index[r]] (zero where index < 0)."""
    if out is None:
        out = torch.empty((index.shape[0], src.shape[1]), dtype=src.dtype, device=src.device)
    _lib.call("moe_gather_rows", src.data_ptr(), src.shape[1], index.data_ptr(), _p(n_dev),
              int(index.shape[0] if n is None else n), out.data_ptr(), _stream())
    return out


def combine(rows: torch.Tensor, plan: Plan, weights: torch.Tensor | None,
            resid: torch.Tensor | None = None, extra: torch.Tensor | None = None,
            extra2: torch.Tensor | None = None, out: torch.Tensor | None = None):
    """y[t] = sum_k w[t,k] rows[inv[t,k]] (+resid if all dropped) (+extra) (+extra2)."""
    h = rows.shape[1]
    if out is None:
        out = torch.empty((plan.T, h), dtype=rows.dtype, device=rows.device)
    _lib.call("moe_combine", rows.data_ptr(), plan.T, plan.K, h, plan.inv_map.data_ptr(),
              _p(weights), _p(resid), _p(extra), _p(extra2), out.data_ptr(), _stream())
    return out


def combine_backward(dy: torch.Tensor, plan: Plan, o_rows: torch.Tensor | None,
                     prob: torch.Tensor | None, d_rows: torch.Tensor | None = None):
    """d_rows[dest] = p * dY[t]; dprob[t,k] = <dY[t], O[dest]> (standard combine)."""
    h = dy.shape[1]
    if d_rows is None:
        d_rows = torch.empty((plan.max_rows, h), dtype=dy.dtype, device=dy.device)
    zero_pad_rows(d_rows, plan)
    dprob = torch.empty((plan.T, plan.K), dtype=torch.float32, device=dy.device)
    _lib.call("moe_combine_bwd", dy.data_ptr(), _p(o_rows), plan.T, plan.K, h,
              plan.inv_map.data_ptr(), _p(prob), d_rows.data_ptr(),
              dprob.data_ptr() if o_rows is not None else None, _stream())
    return d_rows, dprob


def dprob_from_partials(plan: Plan, partial: torch.Tensor):
    dprob = torch.empty((plan.T, plan.K), dtype=torch.float32, device=partial.device)
    _lib.call("moe_dprob_from_partials", plan.inv_map.data_ptr(), plan.T * plan.K,
              partial.data_ptr(), partial.shape[1], dprob.data_ptr(), _stream())
    return dprob
