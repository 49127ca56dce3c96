"""Tape integration: the SLA2 forward + backward as one autograd node.

Mirrors Tape::sla2_attention (tape.hpp:263-286): the forward is smooth_k -> block_scores ->
hard_topk -> sla2_forward_blockwise (one device call, `forward`), and the node's backward is
sla2_backward (attention.hpp:610-809) through the device kernels of backward.cu, accumulating
dq, dk, dv and drho; the router projections are constants of the node (hard top-k blocks the
gradient into them by construction, tape.hpp:260-262). `SLA2Attention` is the per-head layer
of model.hpp:265-268 (router projections and mixing logits per head).

The device backward is the fp32 path (d <= 128, bk <= 64, bq <= 64 or 128): this node takes fp32 tensors."""
from __future__ import annotations

import torch

from . import ContractError, forward, sla2_backward


class SLA2AttentionFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, rho, proj_q, proj_k, k_percent, bq, bk, smooth):
        if q.dtype != torch.float32:
            raise ContractError("SLA2AttentionFunction: fp32 tensors (the device backward is fp32)")
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        out, mask, saved = forward(q, k, v, proj_q.contiguous(), proj_k.contiguous(), rho.contiguous(),
                                   k_percent=k_percent, bq=bq, bk=bk, smooth=smooth, return_mask=True, saved=True)
        ctx.save_for_backward(q, k, v, rho, mask, saved["o_s"], saved["o_l"], saved["big_l"])
        ctx.cfg = (bq, bk, smooth)
        ctx.mark_non_differentiable(mask)
        return out, mask

    @staticmethod
    def backward(ctx, g_out, g_mask):
        q, k, v, rho, mask, o_s, o_l, big_l = ctx.saved_tensors
        bq, bk, smooth = ctx.cfg
        g = sla2_backward(q, k, v, g_out.contiguous(), rho, mask, {"o_s": o_s, "o_l": o_l, "big_l": big_l},
                          bq=bq, bk=bk, smooth=smooth)
        drho = g["drho"].sum(dim=0)  # rho is per head, shared over the batch (model.hpp:38-39)
        return g["dq"], g["dk"], g["dv"], drho, None, None, None, None, None, None


def sla2_attention(q, k, v, rho, proj_q, proj_k, *, k_percent=10.0, bq=64, bk=64, smooth=True):
    """Differentiable SLA2 attention, q/k/v [B,H,N,d] fp32 on the GPU, rho [H,tm], proj [H,d,d].
    Returns (out, mask)."""
    return SLA2AttentionFunction.apply(q, k, v, rho, proj_q, proj_k, k_percent, bq, bk, smooth)


class SLA2Attention(torch.nn.Module):
    """Per-head SLA2 attention layer (model.hpp:265-268): learnable mixing logits rho [H, tm]
    (stage-2 / QAT fine-tuning trains them together with the upstream q, k, v), router
    projections as buffers (identity + noise init as test_gradients.cpp:143-149)."""

    def __init__(self, heads, seq_len, head_dim, *, bq=64, bk=64, k_percent=10.0, smooth=True, device="cuda",
                 seed=0):
        super().__init__()
        gen = torch.Generator().manual_seed(seed)
        tm = -(-seq_len // bq)
        eye = torch.eye(head_dim)[None]
        self.rho = torch.nn.Parameter((torch.rand((heads, tm), generator=gen) * 2 - 1).to(device))
        self.register_buffer("proj_q", (eye + 0.05 * torch.randn((heads, head_dim, head_dim), generator=gen)).to(device))
        self.register_buffer("proj_k", (eye + 0.05 * torch.randn((heads, head_dim, head_dim), generator=gen)).to(device))
        self.cfg = dict(k_percent=k_percent, bq=bq, bk=bk, smooth=smooth)
        self.last_mask = None

    def forward(self, q, k, v):
        out, mask = sla2_attention(q, k, v, self.rho, self.proj_q, self.proj_k, **self.cfg)
        self.last_mask = mask
        return out
