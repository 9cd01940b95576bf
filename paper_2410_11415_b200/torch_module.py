"""Torch surface of the B200 evaluator: an autograd Function and nn.Module.

The reference package has no torch (pkg/pyproject.toml:10); its paper's
library exposes circuits as torch modules. This module gives
the same shape of API on top of the device plan:

    layer = CircuitModule(tc, semiring="log")      # tc: TensorizedCircuit
    roots = layer(log_weights)                      # [B, K] cuda -> [B, R]
    loss = -roots[torch.arange(B), labels].mean()
    loss.backward()                                 # d loss / d log_weights via libklay

Forward runs klay_forward with the trace retained; backward runs
klay_backward with seed = grad_output, i.e. exactly the reference's
backward(tc, trace, seed) (engine.py:307-355): gradient of
sum_r seed[:, r] * root_r with respect to the input slots (log domain:
d log-root / d log-weight). The Boolean and max-product semirings are
forward-only, as in the reference (evaluate_semiring, engine.py:285-304).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .engine import EvalError, device_plan

_CODES = {"real": _lib.KLAY_REAL, "log": _lib.KLAY_LOG, "bool": _lib.KLAY_BOOL,
          "maxprod": _lib.KLAY_MAXPROD}


class KlayFunction(torch.autograd.Function):
    """roots = circuit(weights); weights [B, K] float32/float64 on the plan's device."""

    @staticmethod
    def forward(ctx, weights, plan, code, epsilon):
        dt = np.float64 if weights.dtype == torch.float64 else np.float32
        differentiable = code in (_lib.KLAY_REAL, _lib.KLAY_LOG) and weights.requires_grad
        outputs, values = plan.forward(weights.detach(), code, dt, retain=differentiable,
                                       epsilon=epsilon)
        ctx.plan, ctx.code, ctx.dt = plan, code, dt
        ctx.values = values if differentiable else None
        ctx.batch = weights.shape[0]
        return outputs

    @staticmethod
    def backward(ctx, grad_out):
        if ctx.values is None:
            return None, None, None, None
        # the trace stays with ctx (freed with the graph), so backward is
        # reentrant: retain_graph / gradcheck may run it more than once
        grads = ctx.plan.backward(ctx.values, ctx.batch, ctx.code, ctx.dt,
                                  seed=grad_out.contiguous())
        return grads, None, None, None


class CircuitModule(torch.nn.Module):
    """A tensorized circuit as a layer: [B, K] input-slot weights -> [B, R] roots.

    `semiring`: "log" (weights are log-probabilities, outputs log-WMC),
    "real", "bool" or "maxprod". Weights in the semiring's domain, on the
    module's CUDA device; the compute dtype follows the weights (float32 or
    float64)."""

    def __init__(self, tc, semiring: str = "log", epsilon: float = 0.0, device=None):
        super().__init__()
        if semiring not in _CODES:
            raise EvalError(f"unknown semiring {semiring!r}")
        if semiring == "log" and epsilon < 0:
            raise EvalError("epsilon must be >= 0")
        self.tc = tc
        self.semiring = semiring
        self.epsilon = float(epsilon)
        self.plan = device_plan(tc, device)
        self.num_inputs = tc.num_inputs
        self.num_roots = tc.num_roots

    def forward(self, weights: torch.Tensor) -> torch.Tensor:
        if weights.dim() != 2 or weights.shape[1] != self.num_inputs:
            raise EvalError(f"weights must be [batch, {self.num_inputs}], got {tuple(weights.shape)}")
        if weights.dtype not in (torch.float32, torch.float64):
            raise EvalError("weights must be float32 or float64")
        if weights.device != self.plan.device:
            raise EvalError(f"weights on {weights.device}, circuit on {self.plan.device}")
        return KlayFunction.apply(weights.contiguous(), self.plan, _CODES[self.semiring],
                                  self.epsilon)

    def extra_repr(self) -> str:
        return (f"inputs={self.num_inputs}, roots={self.num_roots}, "
                f"layers={len(self.tc.layers)}, semiring={self.semiring}")
