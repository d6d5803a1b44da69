"""One fused block step for all layers: score -> pooled select -> compact
(blockprefill.hpp:420-444), enqueued on the context stream without host
synchronisation (so it can be captured in a CUDA graph)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .context import Context, default_context, ptr
from .kvcache import EpisodeCache, _pins_tensor
from .scoring import AGG, MODES


class StepPlan:
    """Host-side arguments of epk_evict_step, marshalled once and reused."""

    def __init__(self, cache_in: EpisodeCache, cache_out: EpisodeCache, layer_budgets, pinned=None):
        self.a = cache_in.desc()
        self.b = cache_out.desc()
        L = cache_in.layers
        self.budgets = (C.c_int64 * L)(*[int(x) for x in np.broadcast_to(layer_budgets, (L,))])
        self.pins, self.npins = _pins_tensor(pinned, cache_in.device)


def evict_step(cache_in: EpisodeCache, cache_out: EpisodeCache, q_prompt: torch.Tensor, k_prompt: torch.Tensor,
               layer_budgets, pinned=None, aggregation: str = "max", mode: str | None = None, slack: int = 0,
               n_max_per_head: int | None = None, scores: torch.Tensor | None = None,
               kept_per_layer: torch.Tensor | None = None, plan: StepPlan | None = None,
               ctx: Context | None = None) -> None:
    ctx = ctx or default_context(cache_in.device.index)
    if mode is None:
        mode = "tc_bf16" if cache_in.dtype == torch.bfloat16 else "exact_f32"
    if n_max_per_head is None:
        n_max_per_head = int(cache_in.head_len.max().item())
    plan = plan or StepPlan(cache_in, cache_out, layer_budgets, pinned)
    _lib.call("epk_evict_step", ctx.handle, C.byref(plan.a), C.byref(plan.b), ptr(q_prompt), ptr(k_prompt),
              int(q_prompt.shape[1]), int(q_prompt.shape[2]), C.cast(plan.budgets, C.c_void_p), ptr(plan.pins),
              plan.npins, AGG[aggregation], MODES[mode], int(n_max_per_head), int(slack), ptr(scores),
              ptr(kept_per_layer))
