"""Thin torch-facing wrappers over the tcgen05 grouped-GEMM entry points.

All tensors are CUDA tensors; group metadata (``block_expert``, ``num_m_blocks``,
``expert_offsets``) stays on the device, so none of these calls synchronises with
the host. Shapes follow the expert-major, 128-row-padded permuted layout produced
by :mod:`paper_2603_07685_b200.permute`.
"""
from __future__ import annotations

import torch

from . import _lib

BLOCK_M = 128
GATE_UP_BLOCK = 128  # gate/up rows interleave granularity inside the stacked W1


def dprob_partials(m: int) -> int:
    """Per-row dprob partials the fc2-dgrad epilogue writes: one per (256-col tile, epilogue
    column half), as the library was built (moe_gg_dprob_partials)."""
    return int(_lib.query("moe_gg_dprob_partials", m))


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def interleave_gate_up(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    """Stack gate [E,m,h] and up [E,m,h] into W1 [E,2m,h] with 128-row interleave.

    Rows [256j, 256j+128) hold gate rows [128j, 128j+128), the next 128 rows the
    matching up rows, so one 256-wide GEMM N-tile carries both halves of SwiGLU.
    """
    e, m, h = gate.shape
    assert m % GATE_UP_BLOCK == 0, "ffn dim must be a multiple of 128"
    w = torch.empty((e, m // GATE_UP_BLOCK, 2, GATE_UP_BLOCK, h), dtype=gate.dtype,
                    device=gate.device)
    w[:, :, 0] = gate.reshape(e, m // GATE_UP_BLOCK, GATE_UP_BLOCK, h)
    w[:, :, 1] = up.reshape(e, m // GATE_UP_BLOCK, GATE_UP_BLOCK, h)
    return w.reshape(e, 2 * m, h)


def split_gate_up(w1: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Inverse of :func:`interleave_gate_up` (works on gradients too)."""
    e, m2, h = w1.shape
    m = m2 // 2
    v = w1.reshape(e, m // GATE_UP_BLOCK, 2, GATE_UP_BLOCK, h)
    return v[:, :, 0].reshape(e, m, h), v[:, :, 1].reshape(e, m, h)


def deinterleave_cols(preact: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Split an interleaved [rows, 2m] pre-activation into (gate, up) [rows, m] views."""
    r, m2 = preact.shape
    m = m2 // 2
    v = preact.reshape(r, m // GATE_UP_BLOCK, 2, GATE_UP_BLOCK)
    return v[:, :, 0].reshape(r, m), v[:, :, 1].reshape(r, m)


def _wait_args(wait):
    """wait = (src_flag [n] int32, epoch [1] int32 (device), block_need [blocks] int32,
    unit_order [units] int32, status [8] int32): the EP dispatch-overlap arguments of the
    *_ep GEMMs."""
    flag, epoch, need, order, status = wait
    return (flag.data_ptr(), epoch.data_ptr(), need.data_ptr(), _ptr(order), _ptr(status))


def _blocks(num_m_blocks, pair, units):
    """(num_m_blocks-or-unit-table pointer, flags) of a grouped-M call: with a split-unit
    table (ops.Plan.units) the table stands in for num_m_blocks and flags = pair | split."""
    if units is not None:
        return units.data_ptr(), 3
    return num_m_blocks.data_ptr(), int(pair)


def fc1_fwd(xp, w1, block_expert, num_m_blocks, row_prob=None, preact=None, act=None,
            max_rows=None, pair=False, wait=None, units=None):
    a_rows, h = xp.shape
    rows = a_rows if max_rows is None else max_rows
    e, m2, _ = w1.shape
    m = m2 // 2
    if preact is None:
        preact = torch.empty((rows, m2), dtype=torch.bfloat16, device=xp.device)
    if act is None:
        act = torch.empty((rows, m), dtype=torch.bfloat16, device=xp.device)
    nmb, flags = _blocks(num_m_blocks, pair, units)
    args = (xp.data_ptr(), w1.data_ptr(), a_rows, rows, h, m, e, block_expert.data_ptr(),
            nmb, _ptr(row_prob), preact.data_ptr(), act.data_ptr(), flags)
    if wait is None:
        _lib.call("moe_gg_fc1_fwd", *args, _stream())
    else:
        _lib.call("moe_gg_fc1_fwd_ep", *args, *_wait_args(wait), _stream())
    return preact, act


def fc2_fwd(act, w2, block_expert, num_m_blocks, out=None, max_rows=None, pair=False,
            units=None):
    a_rows, m = act.shape
    rows = a_rows if max_rows is None else max_rows
    e, h, _ = w2.shape
    if out is None:
        out = torch.empty((rows, h), dtype=torch.bfloat16, device=act.device)
    nmb, flags = _blocks(num_m_blocks, pair, units)
    _lib.call("moe_gg_fc2_fwd", act.data_ptr(), w2.data_ptr(), a_rows, rows, m, h, e,
              block_expert.data_ptr(), nmb, out.data_ptr(), flags, _stream())
    return out


def fc2_fwd_scatter(act, w2, block_expert, num_m_blocks, row_dst, max_rows=None, pair=False):
    """fc2 forward storing row r at address row_dst[r] (int64 device tensor; 0 = skip)."""
    a_rows, m = act.shape
    rows = a_rows if max_rows is None else max_rows
    e, h, _ = w2.shape
    _lib.call("moe_gg_fc2_fwd_scatter", act.data_ptr(), w2.data_ptr(), a_rows, rows, m, h, e,
              block_expert.data_ptr(), num_m_blocks.data_ptr(), row_dst.data_ptr(), int(pair),
              _stream())


def fc1_dgrad_scatter(d_preact, w1, block_expert, num_m_blocks, row_dst, max_rows=None,
                      pair=False):
    a_rows, m2 = d_preact.shape
    rows = a_rows if max_rows is None else max_rows
    e, _, h = w1.shape
    _lib.call("moe_gg_fc1_dgrad_scatter", d_preact.data_ptr(), w1.data_ptr(), a_rows, rows,
              m2 // 2, h, e, block_expert.data_ptr(), num_m_blocks.data_ptr(),
              row_dst.data_ptr(), int(pair), _stream())


def fc2_dgrad(dout, w2, preact, block_expert, num_m_blocks, row_prob=None, want_dprob=False,
              d_preact=None, max_rows=None, pair=False, part=None, wait=None, units=None):
    """part: optional preallocated [rows, m/256] fp32 dprob partials (implies want_dprob)."""
    a_rows, h = dout.shape
    rows = a_rows if max_rows is None else max_rows
    e, _, m = w2.shape
    if d_preact is None:
        d_preact = torch.empty((rows, 2 * m), dtype=torch.bfloat16, device=dout.device)
    if want_dprob and part is None:
        part = torch.empty((rows, dprob_partials(m)), dtype=torch.float32, device=dout.device)
    nmb, flags = _blocks(num_m_blocks, pair, units)
    args = (dout.data_ptr(), w2.data_ptr(), preact.data_ptr(), a_rows, rows, h, m, e,
            block_expert.data_ptr(), nmb, _ptr(row_prob), d_preact.data_ptr(), _ptr(part),
            flags)
    if wait is None:
        _lib.call("moe_gg_fc2_dgrad", *args, _stream())
    else:
        _lib.call("moe_gg_fc2_dgrad_ep", *args, *_wait_args(wait), _stream())
    return d_preact, part


def fc1_dgrad(d_preact, w1, block_expert, num_m_blocks, out=None, max_rows=None, pair=False,
              units=None):
    a_rows, m2 = d_preact.shape
    rows = a_rows if max_rows is None else max_rows
    e, _, h = w1.shape
    if out is None:
        out = torch.empty((rows, h), dtype=torch.bfloat16, device=d_preact.device)
    nmb, flags = _blocks(num_m_blocks, pair, units)
    _lib.call("moe_gg_fc1_dgrad", d_preact.data_ptr(), w1.data_ptr(), a_rows, rows, m2 // 2, h, e,
              block_expert.data_ptr(), nmb, out.data_ptr(), flags, _stream())
    return out


def wgrad(a, b, expert_offsets, num_experts, out=None, max_rows=None, overlap_prev=False):
    """out[e] = a[rows_e]^T @ b[rows_e] for each expert's padded row range.

    max_rows bounds the rows TMA reads from both operands (beyond it: zeros).
    overlap_prev: programmatic dependent launch; the caller asserts a and b are not written
    by the previous launch on the stream (it then fills that launch's last wave)."""
    rows, M = a.shape
    if max_rows is not None:
        rows = max_rows
    _, N = b.shape
    if out is None:
        out = torch.empty((num_experts, M, N), dtype=torch.bfloat16, device=a.device)
    _lib.call("moe_gg_wgrad_ex", a.data_ptr(), b.data_ptr(), rows, M, N, num_experts,
              expert_offsets.data_ptr(), out.data_ptr(), 1 if overlap_prev else 0, _stream())
    return out


def gemm_f32(a, b, block_expert, num_m_blocks, out=None, max_rows=None):
    a_rows, K = a.shape
    rows = a_rows if max_rows is None else max_rows
    e, N, _ = b.shape
    if out is None:
        out = torch.empty((rows, N), dtype=torch.float32, device=a.device)
    _lib.call("moe_gg_gemm_f32", a.data_ptr(), b.data_ptr(), a_rows, rows, K, N, e,
              block_expert.data_ptr(), num_m_blocks.data_ptr(), out.data_ptr(), _stream())
    return out


def wgrad_f32(a, b, offsets, num_groups, max_rows=None, out=None):
    """Split-K fp32 partials: out[g] = a[off[g]:off[g+1]]^T @ b[...] (rows >= max_rows read 0)."""
    a_rows, M = a.shape
    _, N = b.shape
    rows = a_rows if max_rows is None else max_rows
    if out is None:
        out = torch.empty((num_groups, M, N), dtype=torch.float32, device=a.device)
    _lib.call("moe_gg_wgrad_f32", a.data_ptr(), b.data_ptr(), rows, M, N, num_groups,
              offsets.data_ptr(), out.data_ptr(), _stream())
    return out


# ---------------------------------------------------------------- MXFP8 (csrc/mxfp8.cu,
# csrc/grouped_gemm_mxfp8.cu): 1x32 E8M0-scaled E4M3 operands, block-scaled tcgen05 MMA.

def mxfp8_quantize(x: torch.Tensor, rows_pad: int | None = None, plain: bool = False,
                   w1_m: int = 0):
    """x bf16 [rows, K] -> (codes uint8 [rows_pad, K], tiled scales uint8, plain scales
    uint8 [rows, K/32] or None). Rows past `rows` in the tiled layout read scale 0.
    w1_m: x is a stacked bf16-engine W1 (rows = E * 2m); emit the 64-row interleave."""
    rows, k = x.shape
    rp = rows_pad if rows_pad is not None else -(-rows // 128) * 128
    if rp > rows:
        codes = torch.zeros((rp, k), dtype=torch.uint8, device=x.device)
        sf_t = torch.zeros((rp * k // 32,), dtype=torch.uint8, device=x.device)
    else:
        codes = torch.empty((rp, k), dtype=torch.uint8, device=x.device)
        sf_t = torch.empty((rp * k // 32,), dtype=torch.uint8, device=x.device)
    sf_p = torch.empty((rows, k // 32), dtype=torch.uint8, device=x.device) if plain else None
    _lib.call("moe_mxfp8_quantize", x.data_ptr(), x.stride(0), rows, k, codes.data_ptr(), k,
              _ptr(sf_p), sf_t.data_ptr(), int(w1_m), _stream())
    return codes, sf_t, sf_p


def mxfp8_quantize_t(x: torch.Tensor, plain: bool = False):
    """Transposing quantisation: x [B, R, C] (or [R, C]) bf16 -> (codes [B*C, R], tiled
    scales, plain scales [B*C, R/32] or None), 1x32 blocks along R."""
    x3 = x if x.dim() == 3 else x.unsqueeze(0)
    b, r, c = x3.shape
    codes = torch.empty((b * c, r), dtype=torch.uint8, device=x.device)
    sf_t = torch.empty((b * c * r // 32,), dtype=torch.uint8, device=x.device)
    sf_p = torch.empty((b * c, r // 32), dtype=torch.uint8, device=x.device) if plain else None
    _lib.call("moe_mxfp8_quantize_t", x3.data_ptr(), b, r, c, codes.data_ptr(), sf_t.data_ptr(),
              _ptr(sf_p), _stream())
    return codes, sf_t, sf_p


def mxfp8_quantize_w1(w1: torch.Tensor, wide: bool = False):
    """bf16-engine W1 [E, 2m, h] (128-row gate/up interleave) -> MXFP8 codes/scales for the
    MXFP8 fc1: the narrow (128-wide tile) engine wants 64-row gate/up blocks (re-interleaved
    in the same pass); the wide (256) engine uses the 128-row layout as is."""
    e, m2, h = w1.shape
    codes, sf, _ = mxfp8_quantize(w1.reshape(e * m2, h), w1_m=0 if wide else m2 // 2)
    return codes, sf


def interleave_gate_up_mx(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    """[E, m, h] gate / up -> [E, 2m, h] with 64-row gate/up blocks (the MXFP8 fc1 tile of
    128 columns then holds matching gate and up rows)."""
    e, m, h = gate.shape
    g = gate.reshape(e, m // 64, 64, h)
    u = up.reshape(e, m // 64, 64, h)
    return torch.stack([g, u], dim=2).reshape(e, 2 * m, h).contiguous()


def mxfp8_quantize_weight(w: torch.Tensor):
    """Stacked K-major weights [E, N, K] -> (codes [E*N, K], tiled scales)."""
    e, n, k = w.shape
    codes, sf, _ = mxfp8_quantize(w.reshape(e * n, k))
    return codes, sf


def mxfp8_gemm(aq, sfa, bq, sfb, num_experts, block_expert, num_m_blocks, N,
               out=None, max_rows=None, pair=False, wide=False):
    """out[rows, N] bf16 = dequant(aq) @ dequant(bq_e)^T per 128-row block's expert."""
    a_rows, k = aq.shape
    rows = a_rows if max_rows is None else max_rows
    if out is None:
        out = torch.empty((rows, N), dtype=torch.bfloat16, device=aq.device)
    _lib.call("moe_gg_mxfp8_gemm", aq.data_ptr(), sfa.data_ptr(), a_rows, rows, k, N,
              bq.data_ptr(), sfb.data_ptr(), num_experts, block_expert.data_ptr(),
              num_m_blocks.data_ptr(), out.data_ptr(), int(pair) | (int(wide) << 1), _stream())
    return out


def mxfp8_fc1(xq, sfx, w1q, sfw, num_experts, block_expert, num_m_blocks, m, max_rows=None,
              want_act=True, pair=False, wide=False, want_t=False):
    """fc1 + SwiGLU on MXFP8 operands (w1q from interleave_gate_up_mx). Returns (preact bf16
    [rows, 2m] in the bf16 engine's layout, act bf16 [rows, m] or None, act codes [rows, m],
    act tiled scales) -- the last two are fc2's MXFP8 A operand."""
    a_rows, h = xq.shape
    rows = a_rows if max_rows is None else max_rows
    dev = xq.device
    preact = torch.empty((rows, 2 * m), dtype=torch.bfloat16, device=dev)
    act = torch.empty((rows, m), dtype=torch.bfloat16, device=dev) if want_act else None
    act_q = torch.empty((rows, m), dtype=torch.uint8, device=dev)
    act_sf = torch.zeros((rows * m // 32,), dtype=torch.uint8, device=dev)
    args = (xq.data_ptr(), sfx.data_ptr(), a_rows, rows, h, m, w1q.data_ptr(), sfw.data_ptr(),
            num_experts, block_expert.data_ptr(), num_m_blocks.data_ptr(), preact.data_ptr(),
            _ptr(act), act_q.data_ptr(), act_sf.data_ptr())
    flags = int(pair) | (int(wide) << 1)
    if not want_t:
        _lib.call("moe_gg_mxfp8_fc1", *args, flags, _stream())
        return preact, act, act_q, act_sf
    # act quantised along the token rows ([m, rows] codes): the dW2 operand
    act_t = torch.zeros((m, rows), dtype=torch.uint8, device=dev)
    act_tsf = torch.zeros((m * rows // 32,), dtype=torch.uint8, device=dev)
    _lib.call("moe_gg_mxfp8_fc1_t", *args, act_t.data_ptr(), act_tsf.data_ptr(), flags,
              _stream())
    return preact, act, act_q, act_sf, act_t, act_tsf


def mxfp8_fc2_dgrad(doq, sfd, w2tq, sfw, num_experts, block_expert, num_m_blocks, preact,
                    max_rows=None, pair=False, wide=False, want_t=False):
    """fc2 dgrad + SwiGLU backward on MXFP8 operands. Returns (d_preact bf16 [rows, 2m],
    d_preact codes [rows, 2m], tiled scales) -- the last two are fc1 dgrad's A operand."""
    a_rows, h = doq.shape
    rows = a_rows if max_rows is None else max_rows
    m2 = preact.shape[1]
    dev = doq.device
    d_pre = torch.empty((rows, m2), dtype=torch.bfloat16, device=dev)
    dq = torch.empty((rows, m2), dtype=torch.uint8, device=dev)
    dsf = torch.zeros((rows * m2 // 32,), dtype=torch.uint8, device=dev)
    args = (doq.data_ptr(), sfd.data_ptr(), a_rows, rows, h, m2 // 2, w2tq.data_ptr(),
            sfw.data_ptr(), num_experts, block_expert.data_ptr(), num_m_blocks.data_ptr(),
            preact.data_ptr(), d_pre.data_ptr(), dq.data_ptr(), dsf.data_ptr())
    flags = int(pair) | (int(wide) << 1)
    if not want_t:
        _lib.call("moe_gg_mxfp8_fc2_dgrad", *args, flags, _stream())
        return d_pre, dq, dsf
    dpt = torch.zeros((m2, rows), dtype=torch.uint8, device=dev)
    dptsf = torch.zeros((m2 * rows // 32,), dtype=torch.uint8, device=dev)
    _lib.call("moe_gg_mxfp8_fc2_dgrad_t", *args, dpt.data_ptr(), dptsf.data_ptr(), flags,
              _stream())
    return d_pre, dq, dsf, dpt, dptsf


def mxfp8_wgrad_q(at, asf, bt, bsf, k_off: torch.Tensor, num_experts: int, out=None):
    """Weight gradient from pre-quantised transposed operands (codes [M, K] / [N, K])."""
    m, k = at.shape
    n = bt.shape[0]
    if out is None:
        out = torch.empty((num_experts, m, n), dtype=torch.bfloat16, device=at.device)
    _lib.call("moe_gg_mxfp8_wgrad", at.data_ptr(), asf.data_ptr(), bt.data_ptr(),
              bsf.data_ptr(), k, m, n, num_experts, k_off.data_ptr(), out.data_ptr(),
              int(m % 256 == 0) | (int(n % 256 == 0) << 1), _stream())
    return out


def mxfp8_wgrad(a: torch.Tensor, b: torch.Tensor, k_off: torch.Tensor, num_experts: int,
                out=None):
    """dw[e] = a[rows_e]^T @ b[rows_e] (bf16 [E, M, N]) on MXFP8 operands: a [K, M] and
    b [K, N] (K = padded token rows, k_off multiples of 128) are quantised along K by the
    transposing quantiser, then one grouped-K block-scaled tcgen05 GEMM."""
    k, m = a.shape
    _, n = b.shape
    at, asf, _ = mxfp8_quantize_t(a)
    bt, bsf, _ = mxfp8_quantize_t(b)
    if out is None:
        out = torch.empty((num_experts, m, n), dtype=torch.bfloat16, device=a.device)
    pair = m % 256 == 0
    wide = n % 256 == 0
    _lib.call("moe_gg_mxfp8_wgrad", at.data_ptr(), asf.data_ptr(), bt.data_ptr(),
              bsf.data_ptr(), k, m, n, num_experts, k_off.data_ptr(), out.data_ptr(),
              int(pair) | (int(wide) << 1), _stream())
    return out


# ---- MXFP8 expert-GEMM chain (shared by layer.py at EP = 1 and the EP dispatcher)

def mxfp8_wide(m: int, h: int) -> bool:
    """256-wide N tiles (single TMEM accumulator, 8 epilogue warps) when the shapes allow."""
    return (2 * m) % 256 == 0 and m % 256 == 0 and h % 256 == 0


def mxfp8_experts_fwd(xp, w1, w2, block_expert, num_m_blocks, pair, out=None):
    """fc1 + SwiGLU and fc2 on MXFP8 operands (x rows and weights quantised here, the
    activation re-quantised row-wise in fc1's epilogue for fc2, and along the token rows by
    the transposing quantiser for the dW2 GEMM). Returns (preact bf16, act_t = (codes
    [m, rows], scales), o bf16).

    (The epilogues can also emit the token-row copies directly -- want_t, warp-shuffle block
    amax, bit-exact -- but that measured slower: fc1 5.2 -> 7.9 ms, fc2-dgrad 4.1 -> 10.4 ms
    against 1.4 ms saved in the transposing quantiser.)"""
    e, m2, h = w1.shape
    m = m2 // 2
    wide = mxfp8_wide(m, h)
    xq, xsf, _ = mxfp8_quantize(xp)
    w1q, w1sf = mxfp8_quantize_w1(w1, wide=wide)
    w2q, w2sf = mxfp8_quantize_weight(w2)
    preact, act, aq, asf = mxfp8_fc1(xq, xsf, w1q, w1sf, e, block_expert, num_m_blocks, m,
                                     pair=pair, wide=wide)
    act_t, act_tsf, _ = mxfp8_quantize_t(act)
    o = mxfp8_gemm(aq, asf, w2q, w2sf, e, block_expert, num_m_blocks, h, out=out, pair=pair,
                   wide=wide)
    return preact, (act_t, act_tsf), o


def mxfp8_experts_bwd(d_o, xp, w1, w2, preact, act_t, block_expert, num_m_blocks, k_off,
                      pair, dx_out=None):
    """fc2 dgrad + dSwiGLU, fc1 dgrad and both weight gradients on MXFP8 operands. d_preact
    is re-quantised in fc2-dgrad's epilogue (row-wise for fc1 dgrad, along the token rows for
    dW1). Returns (dxp, dw1, dw2)."""
    e, h, m = w2.shape
    wide = mxfp8_wide(m, h)
    doq, dosf, _ = mxfp8_quantize(d_o)
    w2tq, w2tsf, _ = mxfp8_quantize_t(w2)
    d_pre, dq, dsf = mxfp8_fc2_dgrad(doq, dosf, w2tq, w2tsf, e, block_expert, num_m_blocks,
                                     preact, pair=pair, wide=wide)
    dpt, dptsf, _ = mxfp8_quantize_t(d_pre)
    w1tq, w1tsf, _ = mxfp8_quantize_t(w1)
    dxp = mxfp8_gemm(dq, dsf, w1tq, w1tsf, e, block_expert, num_m_blocks, h, out=dx_out,
                     pair=pair, wide=wide)
    dot, dotsf, _ = mxfp8_quantize_t(d_o)
    dw2 = mxfp8_wgrad_q(dot, dotsf, act_t[0], act_t[1], k_off, e)
    xpt, xptsf, _ = mxfp8_quantize_t(xp)
    dw1 = mxfp8_wgrad_q(dpt, dptsf, xpt, xptsf, k_off, e)
    return dxp, dw1, dw2
