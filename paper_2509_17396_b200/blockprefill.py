"""The bounded block-prefill engine (block_prefill, blockprefill.hpp:92-228).

Per block: append the block's K/V (append_to_cache) -> score the live cache
against the episode's patched prompt -> evict every layer back to its budget,
all on the GPU, ping-ponging between two HBM caches.  The model forward that
produces the block's K/V and the prompt's Q/K is the step BEFORE this path
(toymodel.hpp:228-411, out of scope): a `StateProvider`
supplies those tensors (synthetic in the bench and tests).

Occupancy is sampled after every append, prompt forward and eviction exactly
as the reference does (blockprefill.hpp:389-447), so the reference's
occupancy-trace tests (3,1,4,1,4,1) run unchanged against this engine.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Protocol

import numpy as np
import torch

from .context import default_context
from .errors import DimensionError, Error
from .kvcache import EpisodeCache, compact, select_pooled, append_to_cache
from .scoring import keydiff_scores, score_with_prompt


class StateProvider(Protocol):
    def block_kv(self, start: int, length: int):
        """-> (k [L,H,len,d], v [L,H,len,d], positions [len] int) on the device."""

    def prompt(self, episode_id: int, block_index: int):
        """-> (q [L,Hq,p,d], k_prompt [L,H,p,d]) on the device."""


@dataclass
class BlockPrefillConfig:
    """BlockPrefillConfig (blockprefill.hpp:27-35)."""
    budget_per_head: int = 64
    block_size: int = 16
    scorer: str = "patched"        # patched | keydiff | streaming
    aggregation: str = "max"       # max | avg
    layer_budgets: list | None = None  # BudgetAllocation.layer_budgets, or None for uniform
    streaming_sink: int = 128
    mode: str | None = None        # exact_f32 | tc_bf16 (default by dtype)


@dataclass
class OccupancySample:
    step: int
    kind: str  # append | prompt | evict
    entries_per_layer: list
    prompt_resident_per_layer: list


@dataclass
class PrefillReport:
    """PrefillReport (blockprefill.hpp:42-55)."""
    cache: EpisodeCache
    occupancy: list = field(default_factory=list)
    blocks_processed: int = 0
    evictions_per_block: list = field(default_factory=list)
    prompt_ranges: list = field(default_factory=list)
    layer_budgets: list = field(default_factory=list)

    def total_evictions(self) -> int:
        return int(sum(self.evictions_per_block))

    def append_evict_series(self, layer: int = 0) -> list:
        return [s.entries_per_layer[layer] for s in self.occupancy if s.kind != "prompt"]


def _layer_budgets(layers: int, cfg: BlockPrefillConfig) -> list:
    budgets = [cfg.budget_per_head] * layers
    if cfg.layer_budgets is not None:
        if len(cfg.layer_budgets) != layers:
            raise Error("block_prefill: allocation layer count != model layers")
        if sum(cfg.layer_budgets) != layers * cfg.budget_per_head:
            raise Error("block_prefill: allocation does not target layers * budget")
        budgets = [int(b) for b in cfg.layer_budgets]
    return budgets


def block_prefill(provider: StateProvider, layers: int, q_heads: int, kv_heads: int, head_dim: int,
                  n_tokens: int, config: BlockPrefillConfig, episode_id: int = 0, prompt_len: int | None = None,
                  dtype=torch.bfloat16, device=None) -> PrefillReport:
    """Ingests n_tokens in blocks of config.block_size on the GPU."""
    if n_tokens <= 0:
        raise Error("block_prefill: empty context")
    if config.budget_per_head < 1 or config.block_size < 1:
        raise Error("block_prefill: budget and block size must be >= 1")
    if q_heads % kv_heads != 0:
        raise DimensionError("block_prefill: query heads must be a multiple of kv heads")
    budgets = _layer_budgets(layers, config)
    pins = None
    if config.scorer == "streaming":
        if config.streaming_sink > config.budget_per_head:
            raise Error("block_prefill: streaming sink exceeds budget")
        if config.layer_budgets is not None and any(config.streaming_sink > b for b in budgets):
            raise Error("block_prefill: streaming sink exceeds an allocated layer budget")
        pins = set(range(config.streaming_sink))
    elif config.scorer not in ("patched", "keydiff"):
        raise Error(f"block_prefill: scorer '{config.scorer}' not supported on the GPU path")

    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ctx = default_context(device.index)
    B = config.block_size
    cap = [kv_heads * (b + B) for b in budgets]
    bufs = [EpisodeCache(layers, kv_heads, head_dim, cap, dtype, device) for _ in range(2)]
    cur = 0
    bufs[cur].set_regions(B)
    report = PrefillReport(cache=bufs[cur], layer_budgets=budgets)
    prompt_base = n_tokens  # prompts sit right after the context (blockprefill.hpp:136)
    zeros = [0] * layers
    scores = torch.empty(bufs[0].rows, dtype=torch.float32 if dtype != torch.float64 else torch.float64,
                         device=device)
    for start in range(0, n_tokens, B):
        length = min(B, n_tokens - start)
        block_index = report.blocks_processed
        k_new, v_new, positions = provider.block_kv(start, length)
        append_to_cache(bufs[cur], k_new, v_new, positions, ctx=ctx)
        ctx.poll_error()
        before = bufs[cur].entries_per_layer()
        report.occupancy.append(OccupancySample(len(report.occupancy), "append", before, zeros))
        if config.scorer == "patched":
            q, kp = provider.prompt(episode_id, block_index)
            p = q.shape[2]
            if p == 0:
                raise Error("block_prefill: empty patched prompt")
            report.prompt_ranges.append((prompt_base, p))
            report.occupancy.append(OccupancySample(len(report.occupancy), "prompt", before,
                                                    [kv_heads * p] * layers))
            sc = score_with_prompt(bufs[cur], q, kp, config.aggregation, config.mode, ctx=ctx)
        elif config.scorer == "keydiff":
            sc = keydiff_scores(bufs[cur], ctx=ctx)  # keydiff_scores (scoring.hpp:186-221)
        else:
            sc = bufs[cur].pos.to(torch.float64)  # streaming_scores (blockprefill.hpp:70-82)
        nxt = 1 - cur
        keep = select_pooled(bufs[cur], sc, budgets, pins, synchronous=True, ctx=ctx)
        compact(bufs[cur], keep, bufs[nxt], slack=B, ctx=ctx)
        ctx.poll_error()
        cur = nxt
        after = bufs[cur].entries_per_layer()
        report.evictions_per_block.append(int(sum(before) - sum(after)))
        report.occupancy.append(OccupancySample(len(report.occupancy), "evict", after, zeros))
        report.blocks_processed += 1
    report.cache = bufs[cur]
    return report
