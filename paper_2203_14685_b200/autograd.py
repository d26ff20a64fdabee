"""torch.autograd wrappers of the routing path: each
forward step of Algorithm 1 paired with its adjoint kernel,
so an MoE layer built on these trains through torch autograd.

    w  = gate_weights(logits, gate, routing_out)   # Eq. 1 weights, routing kept
    xd = dispatch(x, r)                            # Layout_Transform
    ...                                            # AllToAll + experts (caller)
    y  = combine(back, w, r)                       # Reverse_Layout_Transform

Backward: combine -> moe_reverse_layout_backward (d_back, d_weight);
dispatch -> moe_layout_backward (dx); gate_weights -> moe_gate_backward
(d_logits).  The routing (ids, slots, drops) is piecewise constant in its
inputs and carries no gradient.  Argument marshalling only: every gradient is
computed by libmoe_b200's kernels.
"""
from __future__ import annotations

from typing import List

import torch

from .api import Gate, Routing, gate_backward, layout, layout_backward, reverse_layout, \
    reverse_layout_backward


class _GateWeights(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits: torch.Tensor, g: Gate, out: List[Routing]):
        r = g(logits.detach())
        out.append(r)
        ctx.r = r
        ctx.save_for_backward(logits)
        return r.weight

    @staticmethod
    def backward(ctx, d_weight):
        (logits,) = ctx.saved_tensors
        return gate_backward(logits.detach(), ctx.r, d_weight.contiguous()), None, None


class _Dispatch(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x: torch.Tensor, r: Routing):
        ctx.r = r
        return layout(x.detach(), r)

    @staticmethod
    def backward(ctx, d_dispatch):
        return layout_backward(d_dispatch.contiguous(), ctx.r), None


class _Combine(torch.autograd.Function):
    @staticmethod
    def forward(ctx, back: torch.Tensor, weight: torch.Tensor, r: Routing):
        if weight.data_ptr() != r.weight.data_ptr():
            raise ValueError("combine: weight must be the routing's weight tensor")
        ctx.r = r
        ctx.save_for_backward(back)
        return reverse_layout(back.detach(), r)

    @staticmethod
    def backward(ctx, dy):
        (back,) = ctx.saved_tensors
        d_back, d_w = reverse_layout_backward(dy.contiguous(), back.detach().contiguous(), ctx.r)
        return d_back.view_as(back), d_w, None


def gate_weights(logits: torch.Tensor, g: Gate, routing_out: List[Routing]) -> torch.Tensor:
    """Eq. 1 weights [S,k] (differentiable w.r.t. logits); the Routing of the
    call is appended to routing_out."""
    return _GateWeights.apply(logits, g, routing_out)


def dispatch(x: torch.Tensor, r: Routing) -> torch.Tensor:
    """Layout_Transform [S,d] -> [E,cap,d] (differentiable w.r.t. x)."""
    return _Dispatch.apply(x, r)


def combine(back: torch.Tensor, weight: torch.Tensor, r: Routing) -> torch.Tensor:
    """Weighted Reverse_Layout_Transform [E,cap,d] -> [S,d] (differentiable
    w.r.t. back and weight; weight must be r.weight, e.g. from gate_weights)."""
    return _Combine.apply(back, weight, r)
