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
    w_pad: torch.Tensor | None = None   # [1, h, KPAD] bf16: set on the tensor-core (tc) path
    path: str = "gemm"                  # "tc" (default), "gemm" (256-padded), "small"


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


# Small-N tensor-core router (csrc/router_tc.cu): the logits GEMM with N = E padded to 16
# and route() fused into its epilogue, and the weight gradient on the same small-N tile. The
# default for K <= 8 and h % 128 == 0; MOE_ROUTER_TC=0 selects the round-1 chain (logits
# GEMM padded to 256 columns + warp-per-token top-k) for A/B measurements.
ROUTER_TC = os.environ.get("MOE_ROUTER_TC", "1") != "0"


def router_tc(num_experts: int, hidden: int, top_k: int) -> bool:
    return (ROUTER_TC and 1 <= num_experts <= 256 and 1 <= top_k <= min(8, num_experts)
            and hidden >= 128 and hidden % 128 == 0)


_TC_STAGE: dict = {}


def tc_kpad(e: int) -> int:
    """Router dX GEMM K (= the row stride of the row-major dlogits): E rounded up to 64 when the
    weight gradient runs on the small-N tile (E <= 32), else to 256 (the grouped-K split GEMM
    the larger-E backward uses needs N % 256 == 0)."""
    return ceil_to(e, 64) if e <= 32 else ceil_to(e, ROUTER_NPAD)


def stage_router_tc(w_r: torch.Tensor):
    """W_r [h, E] -> (W_r^T [1, NPAD, h], W_r [1, h, KPAD]) zero-padded bf16 for the small-N
    router (NPAD = moe_router_tc_npad(E), KPAD = E rounded up to 64: the dX GEMM's K).

    Cached on the tensor object and its version counter (an in-place optimizer update bumps
    it), so repeated forwards with unchanged weights stage nothing; never cached while a CUDA
    graph is being captured (a replay must re-stage weights updated in place)."""
    h, e = w_r.shape
    capturing = torch.cuda.is_current_stream_capturing()
    key = id(w_r)
    if not capturing:
        hit = _TC_STAGE.get(key)
        if (hit is not None and hit[0]() is w_r and hit[1] == w_r._version
                and hit[2] == w_r.data_ptr()):
            return hit[3], hit[4]
    npad = int(_lib.query("moe_router_tc_npad", e))
    kpad = tc_kpad(e)
    w_r = w_r.contiguous() if w_r.dtype == torch.bfloat16 else w_r.to(torch.bfloat16)
    wt = torch.empty((1, npad, h), dtype=torch.bfloat16, device=w_r.device)
    wp = torch.empty((1, h, kpad), dtype=torch.bfloat16, device=w_r.device)
    _lib.call("moe_stage_router_weight", w_r.data_ptr(), h, e, npad, wt.data_ptr(), None,
              _stream())
    _lib.call("moe_stage_router_weight", w_r.data_ptr(), h, e, kpad, None, wp.data_ptr(),
              _stream())
    if not capturing:
        import weakref

        try:
            ref = weakref.ref(w_r)
        except TypeError:
            return wt, wp
        if len(_TC_STAGE) > 16:
            _TC_STAGE.clear()
        _TC_STAGE[key] = (ref, w_r._version, w_r.data_ptr(), wt, wp)
    return wt, wp


def stage_router(w_r: torch.Tensor):
    """Per-forward router-weight operands of the round-1 tcgen05 chain: (W_r^T padded,
    W_r padded); (None, None) on the small-E and the small-N tensor-core paths (which stage
    their own operands inside router_forward)."""
    h, e = w_r.shape
    if router_small(e, h) or (ROUTER_TC and 1 <= e <= 256 and h % 128 == 0 and h >= 128):
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
    if router_tc(e, h, top_k):
        return _router_forward_tc(x, w_r, top_k, score, selection_bias, coeff, want_scores)
    if w_r_t is None and router_small(e, h):
        return _router_forward_small(x, w_r, top_k, score, selection_bias, coeff, want_scores)
    w_pad = None
    if w_r_t is None or w_r_t.shape[1] != ceil_to(e, ROUTER_NPAD):
        w_r_t, w_pad = stage_router_weight(w_r)
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
                     scores, w_pad=w_pad)


def _router_forward_tc(x, w_r, top_k, score, selection_bias, coeff, want_scores):
    """route() + aux_loss() on the small-N tensor-core router: one GEMM launch whose epilogue
    scores, selects and counts, then the finalize (moe_router_tc_fwd). No host sync."""
    t, h = x.shape
    e = w_r.shape[1]
    dev = x.device
    w_t, w_pad = stage_router_tc(w_r)
    x = x.contiguous()
    logits = torch.empty((t, e), dtype=torch.float32, device=dev)
    topk_idx = torch.empty((t, top_k), dtype=torch.int32, device=dev)
    topk_prob = torch.empty((t, top_k), dtype=torch.float32, device=dev)
    counts = torch.empty((e,), dtype=torch.int32, device=dev)
    ws = torch.empty((max(int(_lib.query("moe_router_tc_fwd_ws", t, h, e)), 1),),
                     dtype=torch.float32, device=dev)
    status = torch.empty((1,), dtype=torch.int32, device=dev)
    scores = torch.empty((t, e), dtype=torch.float32, device=dev) if want_scores else None
    bias = None
    if selection_bias is not None:
        bias = selection_bias.to(device=dev, dtype=torch.float32).contiguous()
    aux = torch.empty((), dtype=torch.float32, device=dev)
    aux_grad = torch.empty((e,), dtype=torch.float32, device=dev)
    mean_scores = torch.empty((e,), dtype=torch.float32, device=dev)
    _lib.call("moe_router_tc_fwd", x.data_ptr(), t, h, w_t.data_ptr(), e, top_k,
              SCORE_FN[score], _p(bias), float(coeff), logits.data_ptr(), topk_idx.data_ptr(),
              topk_prob.data_ptr(), _p(scores), counts.data_ptr(), ws.data_ptr(),
              status.data_ptr(), aux.data_ptr(), aux_grad.data_ptr(), mean_scores.data_ptr(),
              _stream())
    return RouterOut(logits, topk_idx, topk_prob, counts, aux, aux_grad, mean_scores, status,
                     scores, w_pad=w_pad, path="tc")


def _router_backward_tc(x, r: RouterOut, dprob, score, aux_g, want_dx=True,
                        num_splits: int = 8):
    """Router backward of the tensor-core router: the score Jacobian (moe_router_bwd2 on the
    compact logits), dW_r = x^T dl and the router dX = dl . W_r^T (expert GEMM engine, K =
    tc_kpad(E)). dW_r runs on the small-N tile for E <= 32 (split-K, fixed-order sum); for
    larger E the grouped-K split GEMM with N padded to 256 measured faster (Qwen3 shape
    67 + 12 us vs 105 us, tools/router_bench.py), so that E uses it."""
    t, h = x.shape
    e = r.counts.shape[0]
    k = r.topk_idx.shape[1]
    dev = x.device
    npad = int(_lib.query("moe_router_tc_npad", e))
    kpad = r.w_pad.shape[2]
    rows = max(ceil_to(t, ALIGN), ALIGN)
    small = e <= 32
    dl = (torch.empty((rows, kpad), dtype=torch.bfloat16, device=dev)
          if (want_dx or not small) else None)
    ldt = max(ceil_to(t, 8), 8)
    dlt = torch.empty((npad, ldt), dtype=torch.bfloat16, device=dev) if small else None
    _lib.call("moe_router_bwd2", r.logits.data_ptr(), e, t, e, k, SCORE_FN[score],
              r.topk_idx.data_ptr(), dprob.data_ptr(), _p(aux_g), _p(dl), kpad,
              _p(dlt), ldt, npad, _stream())
    dw = torch.empty((h, e), dtype=torch.float32, device=dev)
    if small:
        ws = torch.empty((max(int(_lib.query("moe_router_tc_wgrad_ws", t, h, e)), 1),),
                         dtype=torch.float32, device=dev)
        _lib.call("moe_router_tc_wgrad", x.contiguous().data_ptr(), t, h, dlt.data_ptr(), ldt,
                  e, ws.data_ptr(), dw.data_ptr(), _stream())
    elif t > 0:
        splits = max(1, min(num_splits, -(-t // 64)))
        chunk = ceil_to(-(-t // splits), 64)
        offs_t = (torch.arange(splits + 1, dtype=torch.int32, device=dev) * chunk).clamp_(
            max=ceil_to(t, 64))
        parts = gemm.wgrad_f32(x, dl, offs_t, splits, max_rows=t)
        _lib.call("moe_reduce_groups_f32", parts.data_ptr(), splits, h, kpad, e, dw.data_ptr(),
                  _stream())
    else:
        dw.zero_()
    dx = None
    if want_dx and t > 0:
        nmb = torch.full((1,), rows // ALIGN, dtype=torch.int32, device=dev)
        be = torch.zeros((rows // ALIGN,), dtype=torch.int32, device=dev)
        dx = gemm.fc2_fwd(dl, r.w_pad, be, nmb)
    return dw, dx


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
                     scores, w_r, path="small")


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
    if r.path in ("tc", "small"):
        aux_g = None
        if aux_scale is not None:
            aux_g = r.aux_grad if (isinstance(aux_scale, float) and aux_scale == 1.0) else (
                r.aux_grad * aux_scale)
        if r.path == "tc":
            return _router_backward_tc(x, r, dprob, score, aux_g)
        return _router_backward_small(x, r, dprob, score, aux_g)
    if w_r_pad is None:
        w_r_pad = r.w_pad
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
    # split units (build_plan(split=True)): a 128-row aligned plan whose grouped GEMMs run
    # each expert's 256-row pairs on the CTA-pair engine and its odd last 128-row block on
    # the 1-CTA engine (moe_split_units table, passed as the GEMMs' `units`)
    units: torch.Tensor | None = None

    @property
    def num_m_blocks(self) -> torch.Tensor:
        return self.meta[0:1]

    @property
    def pair(self) -> bool:
        return self.align == 2 * ALIGN or self.units is not None


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


# Split units for the pair engine (Plan.units): on by default; MOE_B200_SPLIT_UNITS=0 keeps
# the 256-row aligned plan (A/B)
SPLIT_UNITS = os.environ.get("MOE_B200_SPLIT_UNITS", "1") != "0"
SPLIT_FORCE = os.environ.get("MOE_B200_SPLIT_UNITS", "1") == "2"  # (A/B: ignore the size rule)


def build_plan(topk_idx: torch.Tensor, topk_prob: torch.Tensor | None, E: int,
               capacity: int = -1, pad: bool = False, max_rows: int | None = None,
               phantom: torch.Tensor | None = None, phantom_max: int = 0,
               cap_e: torch.Tensor | None = None, compact: bool = False,
               align: int = ALIGN, split: bool = False) -> Plan:
    """phantom: optional device int32 [E] extra zero rows per expert (routing_map_pad);
    phantom_max bounds it for buffer sizing. cap_e: optional device int32 [E] per-expert
    capacity (EP global-position drops). compact: no 128-row alignment (EP send layout).
    split (with align 256, bf16 expert GEMMs only): build the 128-row aligned plan plus the
    split-unit table instead (half the padding; Plan.units)."""
    t, k = topk_idx.shape
    dev = topk_idx.device
    # measured (profiles/r02_split_units_ab.txt, alternating runs on one box): Mixtral
    # (~4096 rows per expert) 30.85 -> 30.26 ms per step; Qwen3 (~2048 rows per expert, 128
    # experts: ~64 one-block tails per GEMM on the 1-CTA engine) 31.0 -> 31.2 ms. Split
    # where experts hold >= 16 pair units.
    split = (split and SPLIT_UNITS and align == 2 * ALIGN and not compact
             and (SPLIT_FORCE or t * k >= 16 * 2 * ALIGN * E))
    if split:
        align = ALIGN
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
    units = None
    if split:
        cap = max_rows // ALIGN
        units = torch.empty((2 + 2 * cap,), **i32)
        _lib.call("moe_split_units", meta.data_ptr(), block_expert.data_ptr(), off_pad.data_ptr(),
                  cap, units.data_ptr(), _stream())
    return Plan(t, k, E, int(capacity), bool(pad), max_rows, meta, off_pad, off_c, kept, eff,
                counts, block_expert, inv_map, row_src, row_prob, status,
                1 if compact else align, units)


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
