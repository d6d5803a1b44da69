"""Layer sensitivity and adaptive layer budgets (allocation.hpp).

`sensitivity_from_keys` is the reduction of measure_sensitivity
(allocation.hpp:80-100) as the K5 kernel: sigma_l = mean over (kv-head, token)
of cosine(K_full, K_block), zero-norm pairs skipped; s_l = 1 - sigma_l.  The
two model forwards that produce the key states (causal and sink+recent masks,
allocation.hpp:70-72) are the model substrate and are out of scope.

`allocate` / `uniform_allocation` are host code (L scalars), restated from
allocation.hpp:120-207 with the same floating-point sequence so the integer
budgets match the reference exactly.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .context import Context, default_context, ptr
from .errors import Error

_DT = {torch.float32: _lib.EPK_F32, torch.bfloat16: _lib.EPK_BF16, torch.float64: _lib.EPK_F64}


@dataclass
class SensitivityProfile:
    """SensitivityProfile (allocation.hpp:22-32)."""
    sigma: list
    sensitivity: list
    mask_sink: int = 0
    mask_recent: int = 0
    input_id: str = ""
    model_seed: int = 0
    skipped_zero_norm: int = 0

    def layer_count(self) -> int:
        return len(self.sigma)


@dataclass
class BudgetAllocation:
    """BudgetAllocation (allocation.hpp:36-49)."""
    alpha: float = 0.0
    weights: list = field(default_factory=list)
    layer_budgets: list = field(default_factory=list)
    per_head_budget: int = 0

    def layer_count(self) -> int:
        return len(self.layer_budgets)

    def total(self) -> int:
        return int(sum(self.layer_budgets))


def sensitivity_from_keys(k_full: torch.Tensor, k_block: torch.Tensor, sink: int = 0, recent: int = 0,
                          ctx: Context | None = None) -> SensitivityProfile:
    """k_full, k_block: [layers, kv_heads, tokens, head_dim] on the device."""
    if k_full.shape != k_block.shape or k_full.dim() != 4:
        raise Error("measure_sensitivity: key tensors must both be [layers, heads, tokens, dim]")
    if k_full.dtype != k_block.dtype or k_full.dtype not in _DT:
        raise Error("measure_sensitivity: unsupported key dtype")
    ctx = ctx or default_context(k_full.device.index)
    L, H, N, d = k_full.shape
    if N < 2:
        raise Error("measure_sensitivity: need at least 2 calibration tokens")
    sigma = torch.empty(L, dtype=torch.float64, device=k_full.device)
    skipped = torch.empty(1, dtype=torch.int64, device=k_full.device)
    _lib.call("epk_key_cosine_sigma", ctx.handle, ptr(k_full.contiguous()), ptr(k_block.contiguous()),
              _DT[k_full.dtype], L, H, N, d, ptr(sigma), ptr(skipped))
    s = sigma.cpu().tolist()
    return SensitivityProfile(sigma=s, sensitivity=[1.0 - x for x in s], mask_sink=sink, mask_recent=recent,
                              skipped_zero_norm=int(skipped.item()))


def allocate(profile: SensitivityProfile, per_head_budget: int, alpha: float) -> BudgetAllocation:
    """Sharpened proportional allocation with largest-remainder rounding and a
    floor of 1 (allocation.hpp:120-198)."""
    layers = profile.layer_count()
    if layers < 1:
        raise Error("allocate: empty profile")
    if per_head_budget < 1:
        raise Error("allocate: budget must be >= 1")
    if alpha < 0.0:
        raise Error("allocate: alpha must be >= 0")
    powered = [math.pow(max(0.0, float(s)), float(alpha)) for s in profile.sensitivity]
    total = 0.0
    for pw in powered:
        total += pw
    if total <= 0.0:
        weights = [1.0 / float(layers)] * layers
    else:
        weights = [pw / total for pw in powered]
    grand = layers * per_head_budget
    real = [w * float(grand) for w in weights]
    budgets = [int(math.floor(r)) for r in real]
    assigned = sum(budgets)
    order = sorted(range(layers), key=lambda l: (-(real[l] - math.floor(real[l])), l))
    i = 0
    while assigned < grand:
        budgets[order[i % layers]] += 1
        assigned += 1
        i += 1
    for l in range(layers):
        while budgets[l] < 1:
            victim = 0
            for j in range(1, layers):
                if budgets[j] > budgets[victim] or (budgets[j] == budgets[victim] and weights[j] < weights[victim]):
                    victim = j
            if budgets[victim] <= 1:
                raise Error("allocate: cannot satisfy per-layer floor")
            budgets[victim] -= 1
            budgets[l] += 1
    return BudgetAllocation(alpha=alpha, weights=weights, layer_budgets=budgets, per_head_budget=per_head_budget)


def uniform_allocation(layers: int, per_head_budget: int) -> BudgetAllocation:
    """uniform_allocation (allocation.hpp:200-207)."""
    return BudgetAllocation(alpha=0.0, weights=[1.0 / layers] * layers, layer_budgets=[per_head_budget] * layers,
                            per_head_budget=per_head_budget)
