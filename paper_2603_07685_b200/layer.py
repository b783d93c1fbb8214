"""Autograd MoE layer (router -> permute -> grouped-GEMM SwiGLU -> combine), EP = 1.

The reference has no layer class and no backward: its forward is the
function chain route() -> apply_capacity() -> combine_standard() /
combine_mem_efficient() -> moe_output_with_residual() (pkg/src/moelab/routing.py
:71-108, :226-247, :189-223, :254-262) plus aux_loss() (:111-120). This module runs
that chain on the device kernels and implements its exact gradient (SURVEY
Appendix C), with the loss convention L = <dY, y> + daux * aux.

Megatron names are used for the modules: ``TopKRouter``,
``GroupedMLP`` and ``MoELayer``; the expert-parallel dispatcher lives in
:mod:`paper_2603_07685_b200.dispatcher`.

No host synchronisation happens in forward or backward at EP = 1.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import torch

from . import gemm, ops

# weight gradients as programmatic dependent launches behind the data-gradient GEMMs
# (MOE_B200_WGRAD_PDL=0: plain launches, for A/B)
OVERLAP_WGRAD = os.environ.get("MOE_B200_WGRAD_PDL", "1") != "0"


@dataclass(frozen=True)
class MoEConfig:
    num_experts: int
    top_k: int
    hidden: int
    ffn_hidden: int
    score: str = "softmax"            # "softmax" | "sigmoid"
    aux_loss_coeff: float = 0.0       # --moe-aux-loss-coeff
    capacity_factor: float | None = None   # --moe-expert-capacity-factor
    pad_to_capacity: bool = False     # --moe-pad-expert-input-to-capacity
    mem_efficient: bool = False       # combine_mem_efficient (prob folded into act)
    shared_ffn_hidden: int = 0        # DeepSeek shared expert width (0 = none)
    # expert GEMMs: "bf16", or "mxfp8" (the paper's Blackwell recipe, 1x32 E8M0 blocks,
    # quant.py:62-64; block-scaled tcgen05 MMA) for all six: forward fc1/fc2, the
    # data-gradient GEMMs (operands re-quantised in the producing epilogues, weights
    # transposed-quantised along the dgrad K) and the weight-gradient GEMMs (activations and
    # gradients transposed-quantised along the token rows, the reference's column twin).
    precision: str = "bf16"
    # raise the reference's ValueError("router logits are not finite") (routing.py:80-81) when
    # a token's router logits are NaN / inf. Costs one host sync per forward, so it is off by
    # default; the kernels stay memory-safe either way (non-finite keys select valid experts)
    check_finite: bool = False

    def capacity(self, num_tokens: int) -> int:
        """expert_capacity() routing.py:250-251 (k = top_k since every token selects K)."""
        if self.capacity_factor is None:
            return -1
        return -(-int(round(self.capacity_factor * num_tokens * self.top_k)) // self.num_experts)


class _MoEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w_r, w1, w2, sel_bias, w1s, w2s, cfg: MoEConfig):
        t, h = x.shape
        e = cfg.num_experts
        w_r_t, w_r_pad = ops.stage_router(w_r)
        r = ops.router_forward(x, w_r, cfg.top_k, cfg.score, sel_bias, cfg.aux_loss_coeff,
                               w_r_t=w_r_t)
        if cfg.check_finite and int(r.status.item()) & 1:
            raise ValueError("router logits are not finite")
        cap = cfg.capacity(t)
        plan = ops.build_plan(r.topk_idx, r.topk_prob, e, cap, cfg.pad_to_capacity,
                              align=ops.pick_align(t, cfg.top_k, e),
                              split=cfg.precision == "bf16")
        xp = ops.permute_gather(x, plan)
        row_prob = plan.row_prob if cfg.mem_efficient else None
        act_t = None
        if cfg.precision == "mxfp8":
            preact, act_t, o = gemm.mxfp8_experts_fwd(xp, w1, w2, plan.block_expert,
                                                      plan.num_m_blocks, plan.pair)
            act = None  # the weight gradient reads the token-row quantised copy
        else:
            preact, act = gemm.fc1_fwd(xp, w1, plan.block_expert, plan.num_m_blocks, row_prob,
                                       pair=plan.pair, units=plan.units)
            o = gemm.fc2_fwd(act, w2, plan.block_expert, plan.num_m_blocks, pair=plan.pair,
                             units=plan.units)
        shared = shared_expert_forward(x, w1s, w2s) if w1s is not None else None
        y = ops.combine(o, plan, None if cfg.mem_efficient else r.topk_prob,
                        resid=x if cap >= 0 else None,
                        extra=shared[-1] if shared is not None else None)
        ctx.cfg = cfg
        ctx.plan = plan
        ctx.r = r
        ctx.act_t = act_t
        ctx.shared = shared[:-1] if shared is not None else None
        ctx.save_for_backward(x, w_r_pad, w1, w2, xp, preact, act, o, w1s, w2s)
        return y, r.aux

    @staticmethod
    def backward(ctx, dy, daux):
        cfg, plan, r = ctx.cfg, ctx.plan, ctx.r
        x, w_r_pad, w1, w2, xp, preact, act, o, w1s, w2s = ctx.saved_tensors
        e = cfg.num_experts
        dy = dy.contiguous()
        if cfg.mem_efficient:
            d_o, _ = ops.combine_backward(dy, plan, None, None)
            d_pre, part = gemm.fc2_dgrad(d_o, w2, preact, plan.block_expert, plan.num_m_blocks,
                                         row_prob=plan.row_prob, want_dprob=True,
                                         pair=plan.pair, units=plan.units)
            dprob = ops.dprob_from_partials(plan, part)
        else:
            d_o, dprob = ops.combine_backward(dy, plan, o, r.topk_prob)
            if cfg.precision != "mxfp8":
                d_pre, _ = gemm.fc2_dgrad(d_o, w2, preact, plan.block_expert,
                                          plan.num_m_blocks, pair=plan.pair, units=plan.units)
        if cfg.precision == "mxfp8":
            dxp, dw1, dw2 = gemm.mxfp8_experts_bwd(d_o, xp, w1, w2, preact, ctx.act_t,
                                                   plan.block_expert, plan.num_m_blocks,
                                                   plan.off_pad, plan.pair)
        else:
            # each weight gradient reads nothing the data-gradient GEMM launched just before
            # it writes (dW2: d_O, act; dW1: d_pre, xp), so it is launched to overlap that
            # GEMM's last wave (programmatic dependent launch)
            dw2 = gemm.wgrad(d_o, act, plan.off_pad, e, overlap_prev=OVERLAP_WGRAD)
            dxp = gemm.fc1_dgrad(d_pre, w1, plan.block_expert, plan.num_m_blocks,
                                 pair=plan.pair, units=plan.units)
            dw1 = gemm.wgrad(d_pre, xp, plan.off_pad, e, overlap_prev=OVERLAP_WGRAD)
        aux_scale = None if daux is None else daux.float()
        dw_r, dx_router = ops.router_backward(x, w_r_pad, r, dprob, cfg.score,
                                              aux_scale=aux_scale)
        dx_shared = dw1s = dw2s = None
        if ctx.shared is not None:
            dx_shared, dw1s, dw2s = shared_expert_backward(x, dy, w1s, w2s, ctx.shared)
        cap = cfg.capacity(x.shape[0])
        dx = ops.combine(dxp, plan, None, resid=dy if cap >= 0 else None, extra=dx_router,
                         extra2=dx_shared)
        return (dx, dw_r.to(torch.bfloat16), dw1, dw2, None, dw1s, dw2s, None)


def shared_expert_forward(x, w1s, w2s):
    """DeepSeek shared expert (latent_moe_forward's shared term, routing.py:276-278): a dense
    SwiGLU MLP on every token, run as a 1-group grouped GEMM. Returns saved state + output."""
    t = x.shape[0]
    rows = ops.ceil_to(max(t, 1), ops.ALIGN)
    nmb = torch.full((1,), rows // ops.ALIGN, dtype=torch.int32, device=x.device)
    be = torch.zeros((rows // ops.ALIGN,), dtype=torch.int32, device=x.device)
    pre_s, act_s = gemm.fc1_fwd(x, w1s, be, nmb, max_rows=rows)
    o_s = gemm.fc2_fwd(act_s, w2s, be, nmb)
    return pre_s, act_s, nmb, be, rows, o_s


def shared_expert_backward(x, dy, w1s, w2s, saved):
    pre_s, act_s, nmb, be, rows = saved
    t = x.shape[0]
    d_pre_s, _ = gemm.fc2_dgrad(dy, w2s, pre_s, be, nmb, max_rows=rows)
    dx_s = gemm.fc1_dgrad(d_pre_s, w1s, be, nmb)
    offs = torch.arange(2, dtype=torch.int32, device=x.device) * ops.ceil_to(t, 64)
    # rows >= t read as zero (TMA bound = t)
    dw2s = gemm.wgrad(dy, act_s, offs, 1, max_rows=t)
    dw1s = gemm.wgrad(d_pre_s, x, offs, 1, max_rows=t)
    return dx_s, dw1s, dw2s


def moe_forward(x, w_r, w1, w2, cfg: MoEConfig, selection_bias=None, w1_shared=None,
                w2_shared=None):
    """Functional MoE layer: returns (y [T,h] bf16, aux [] fp32). Differentiable."""
    if cfg.precision not in ("bf16", "mxfp8"):
        raise ValueError(f"unknown precision {cfg.precision!r}")
    if cfg.precision == "mxfp8" and cfg.mem_efficient:
        raise ValueError("mxfp8 experts use the standard combine")
    return _MoEFunction.apply(x, w_r, w1, w2, selection_bias, w1_shared, w2_shared, cfg)


class TopKRouter(torch.nn.Module):
    """Router weights W_r [h, E] (reference layout, routing.py:79) + aux-free bias buffer."""

    def __init__(self, cfg: MoEConfig, device=None, dtype=torch.bfloat16):
        super().__init__()
        self.cfg = cfg
        self.weight = torch.nn.Parameter(
            torch.empty((cfg.hidden, cfg.num_experts), device=device, dtype=dtype))
        self.register_buffer("selection_bias", None)

    def reset_parameters(self, generator=None):
        with torch.no_grad():
            self.weight.normal_(0.0, self.cfg.hidden ** -0.5, generator=generator)


class GroupedMLP(torch.nn.Module):
    """Stacked SwiGLU experts: w1 [E, 2m, h] (gate/up 128-row interleave), w2 [E, h, m]."""

    def __init__(self, num_experts, hidden, ffn_hidden, device=None, dtype=torch.bfloat16):
        super().__init__()
        self.w1 = torch.nn.Parameter(
            torch.empty((num_experts, 2 * ffn_hidden, hidden), device=device, dtype=dtype))
        self.w2 = torch.nn.Parameter(
            torch.empty((num_experts, hidden, ffn_hidden), device=device, dtype=dtype))

    def reset_parameters(self, generator=None):
        h, m = self.w2.shape[1], self.w2.shape[2]
        with torch.no_grad():
            self.w1.normal_(0.0, h ** -0.5, generator=generator)
            self.w2.normal_(0.0, m ** -0.5, generator=generator)

    @classmethod
    def from_gate_up(cls, gate, up, w2):
        mlp = cls.__new__(cls)
        torch.nn.Module.__init__(mlp)
        mlp.w1 = torch.nn.Parameter(gemm.interleave_gate_up(gate, up))
        mlp.w2 = torch.nn.Parameter(w2.contiguous())
        return mlp


class MoELayer(torch.nn.Module):
    """Megatron-style MoE layer on one GPU (EP = 1); returns (y, aux_loss)."""

    def __init__(self, cfg: MoEConfig, device=None, dtype=torch.bfloat16):
        super().__init__()
        self.cfg = cfg
        self.router = TopKRouter(cfg, device, dtype)
        self.experts = GroupedMLP(cfg.num_experts, cfg.hidden, cfg.ffn_hidden, device, dtype)
        self.shared_experts = None
        if cfg.shared_ffn_hidden:
            self.shared_experts = GroupedMLP(1, cfg.hidden, cfg.shared_ffn_hidden, device, dtype)

    def reset_parameters(self, generator=None):
        self.router.reset_parameters(generator)
        self.experts.reset_parameters(generator)
        if self.shared_experts is not None:
            self.shared_experts.reset_parameters(generator)

    def forward(self, x):
        s = self.shared_experts
        return moe_forward(x, self.router.weight, self.experts.w1, self.experts.w2, self.cfg,
                           self.router.selection_bias,
                           None if s is None else s.w1, None if s is None else s.w2)
