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
EPI_HALVES = 1       # epilogue warps per TMEM lane quarter (csrc/grouped_gemm.cu EPI_WARPS/4)


def dprob_partials(m: int) -> int:
    """Per-row dprob partials the fc2-dgrad epilogue writes: one per (256-col tile, half)."""
    return (m // 256) * EPI_HALVES


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


def fc1_fwd(xp, w1, block_expert, num_m_blocks, row_prob=None, preact=None, act=None,
            max_rows=None, pair=False, wait=None):
    a_rows, h = xp.shape
    rows = a_rows if max_rows is None else max_rows
    e, m2, _ = w1.shape
    m = m2 // 2
    if preact is None:
        preact = torch.empty((rows, m2), dtype=torch.bfloat16, device=xp.device)
    if act is None:
        act = torch.empty((rows, m), dtype=torch.bfloat16, device=xp.device)
    args = (xp.data_ptr(), w1.data_ptr(), a_rows, rows, h, m, e, block_expert.data_ptr(),
            num_m_blocks.data_ptr(), _ptr(row_prob), preact.data_ptr(), act.data_ptr(),
            int(pair))
    if wait is None:
        _lib.call("moe_gg_fc1_fwd", *args, _stream())
    else:
        _lib.call("moe_gg_fc1_fwd_ep", *args, *_wait_args(wait), _stream())
    return preact, act


def fc2_fwd(act, w2, block_expert, num_m_blocks, out=None, max_rows=None, pair=False):
    a_rows, m = act.shape
    rows = a_rows if max_rows is None else max_rows
    e, h, _ = w2.shape
    if out is None:
        out = torch.empty((rows, h), dtype=torch.bfloat16, device=act.device)
    _lib.call("moe_gg_fc2_fwd", act.data_ptr(), w2.data_ptr(), a_rows, rows, m, h, e,
              block_expert.data_ptr(), num_m_blocks.data_ptr(), out.data_ptr(), int(pair),
              _stream())
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
              d_preact=None, max_rows=None, pair=False, part=None, wait=None):
    """part: optional preallocated [rows, m/256] fp32 dprob partials (implies want_dprob)."""
    a_rows, h = dout.shape
    rows = a_rows if max_rows is None else max_rows
    e, _, m = w2.shape
    if d_preact is None:
        d_preact = torch.empty((rows, 2 * m), dtype=torch.bfloat16, device=dout.device)
    if want_dprob and part is None:
        part = torch.empty((rows, dprob_partials(m)), dtype=torch.float32, device=dout.device)
    args = (dout.data_ptr(), w2.data_ptr(), preact.data_ptr(), a_rows, rows, h, m, e,
            block_expert.data_ptr(), num_m_blocks.data_ptr(), _ptr(row_prob),
            d_preact.data_ptr(), _ptr(part), int(pair))
    if wait is None:
        _lib.call("moe_gg_fc2_dgrad", *args, _stream())
    else:
        _lib.call("moe_gg_fc2_dgrad_ep", *args, *_wait_args(wait), _stream())
    return d_preact, part


def fc1_dgrad(d_preact, w1, block_expert, num_m_blocks, out=None, max_rows=None, pair=False):
    a_rows, m2 = d_preact.shape
    rows = a_rows if max_rows is None else max_rows
    e, _, h = w1.shape
    if out is None:
        out = torch.empty((rows, h), dtype=torch.bfloat16, device=d_preact.device)
    _lib.call("moe_gg_fc1_dgrad", d_preact.data_ptr(), w1.data_ptr(), a_rows, rows, m2 // 2, h, e,
              block_expert.data_ptr(), num_m_blocks.data_ptr(), out.data_ptr(), int(pair),
              _stream())
    return out


def wgrad(a, b, expert_offsets, num_experts, out=None, max_rows=None):
    """out[e] = a[rows_e]^T @ b[rows_e] for each expert's padded row range.

    max_rows bounds the rows TMA reads from both operands (beyond it: zeros)."""
    rows, M = a.shape
    if max_rows is not None:
        rows = max_rows
    _, N = b.shape
    if out is None:
        out = torch.empty((num_experts, M, N), dtype=torch.bfloat16, device=a.device)
    _lib.call("moe_gg_wgrad", a.data_ptr(), b.data_ptr(), rows, M, N, num_experts,
              expert_offsets.data_ptr(), out.data_ptr(), _stream())
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
