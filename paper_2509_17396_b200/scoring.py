"""Patched-prompt scoring (scoring.hpp:80-128) fused with the prompt's
attention-weight computation (toymodel.hpp:327-391).

The reference computes full attention grids for the prompt rows and then
reduces them (window Max/Avg over prompt rows, max over a kv-head's query
heads, cache columns only).  On the GPU the grid is never materialised:
`score_with_prompt` returns one fp32 score per live cache row directly.

Modes:
  "exact_f32"  CUDA-core fp32, EPK-F32 v1 op order; bit-exact with
               oracle.score_layer_f32 (the parity path).
  "tc_bf16"    tcgen05/TMEM tensor-core kernel on bf16 Q/K with fp32
               accumulation (the throughput path).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .context import Context, default_context, ptr
from .errors import DimensionError, Error
from .kvcache import EpisodeCache

AGG = {"max": _lib.EPK_AGG_MAX, "avg": _lib.EPK_AGG_AVG}
MODES = {"exact_f32": _lib.EPK_SCORE_EXACT_F32, "tc_bf16": _lib.EPK_SCORE_TC_BF16}


def score_with_prompt(cache: EpisodeCache, q_prompt: torch.Tensor, k_prompt: torch.Tensor,
                      aggregation: str = "max", mode: str | None = None, n_max_per_head: int | None = None,
                      out: torch.Tensor | None = None, ctx: Context | None = None) -> torch.Tensor:
    """Scores every live cache row against the patched prompt.

    q_prompt [layers, Hq, p, d], k_prompt [layers, H, p, d] (prompt rows attend
    the whole cache plus prompt rows 0..t).  Returns fp32 [cache.rows]
    (entries of non-live rows are unspecified)."""
    ctx = ctx or default_context(cache.device.index)
    if mode is None:
        mode = "tc_bf16" if cache.dtype == torch.bfloat16 else "exact_f32"
    if q_prompt.dim() != 4 or q_prompt.shape[0] != cache.layers or q_prompt.shape[3] != cache.head_dim:
        raise DimensionError("score_with_prompt: attention grid shape mismatch")
    p = q_prompt.shape[2]
    if p == 0:
        raise Error("score_with_prompt: empty prompt")
    if tuple(k_prompt.shape) != (cache.layers, cache.kv_heads, p, cache.head_dim):
        raise DimensionError("score_with_prompt: attention grid shape mismatch")
    if q_prompt.dtype != cache.dtype or k_prompt.dtype != cache.dtype:
        raise Error("score_with_prompt: prompt dtype must match the cache dtype")
    if n_max_per_head is None:
        n_max_per_head = int(cache.head_len.max().item()) if cache.rows else 0
    out = out if out is not None else torch.empty(cache.rows, dtype=torch.float32, device=cache.device)
    d = cache.desc()
    _lib.call("epk_score", ctx.handle, C.byref(d), ptr(q_prompt.contiguous()), ptr(k_prompt.contiguous()),
              int(q_prompt.shape[1]), int(p), AGG[aggregation], MODES[mode], int(n_max_per_head), ptr(out))
    return out


def score_grids(grids, head_off, q_heads: int, aggregation: str = "max", ctx: Context | None = None) -> np.ndarray:
    """score_with_prompt (scoring.hpp:80) over explicit fp64 attention grids of
    ONE layer: grids[qh] has shape [p, n_h + p].  Returns fp64 scores in
    head-major row order (bit-exact with the reference)."""
    ctx = ctx or default_context()
    head_off = np.asarray(head_off, np.int64)
    H = head_off.size - 1
    if len(grids) == 0 or len(grids) % H != 0:
        raise DimensionError("score_with_prompt: attention grid shape mismatch")
    p = grids[0].shape[0]
    if p == 0:
        raise Error("score_with_prompt: empty prompt")
    G = len(grids) // H
    for qh, g in enumerate(grids):
        h = qh // G
        if g.shape != (p, head_off[h + 1] - head_off[h] + p):
            raise DimensionError("score_with_prompt: attention grid shape mismatch")
    flat = torch.as_tensor(np.concatenate([np.asarray(g, np.float64).ravel() for g in grids]),
                           device=torch.device("cuda", ctx.device))
    out = torch.empty(int(head_off[-1]), dtype=torch.float64, device=flat.device)
    ho = (C.c_int64 * (H + 1))(*head_off.tolist())
    _lib.call("epk_score_grids", ctx.handle, len(grids), H, p, C.cast(ho, C.c_void_p), ptr(flat),
              AGG[aggregation], ptr(out))
    return out.cpu().numpy()


def keydiff_scores(cache: EpisodeCache, out: torch.Tensor | None = None, ctx: Context | None = None) -> torch.Tensor:
    """keydiff_scores (scoring.hpp:186-221): per (layer, kv-head) every live
    entry scores -cosine(key, mean key), 0 on a zero norm.  fp64 [cache.rows]
    in cache row order (gap rows unspecified), bit-exact with the reference;
    feed it to select_pooled + compact like any other score."""
    ctx = ctx or default_context(cache.device.index)
    if cache.dtype not in (torch.bfloat16, torch.float32, torch.float64):
        raise Error("keydiff_scores: cache dtype must be bf16, fp32 or fp64")
    out = out if out is not None else torch.zeros(cache.rows, dtype=torch.float64, device=cache.device)
    d = cache.desc()
    _lib.call("epk_score_keydiff", ctx.handle, C.byref(d), ptr(out))
    return out


def pool_scores(cache: EpisodeCache, scores: torch.Tensor, kernel: int, out: torch.Tensor | None = None,
                ctx: Context | None = None) -> torch.Tensor:
    """Opt-in 1-D max-pool smoothing (north_star; NOT in the reference, whose
    score_with_prompt has no pooling, scoring.hpp:80-128): max over an odd
    `kernel`-row window of each head's live rows (position order), never
    across heads.  epk_pool_scores."""
    ctx = ctx or default_context(cache.device.index)
    if scores.dtype != torch.float32 or scores.numel() < cache.rows:
        raise DimensionError("pool_scores: fp32 scores for every cache row expected")
    out = out if out is not None else torch.empty_like(scores)
    d = cache.desc()
    _lib.call("epk_pool_scores", ctx.handle, C.byref(d), ptr(scores), ptr(out), int(kernel))
    return out


def debug_expf(x: torch.Tensor, ctx: Context | None = None) -> torch.Tensor:
    """The device epk_expf (EPK-F32 v1), for the bitwise parity test."""
    ctx = ctx or default_context(x.device.index)
    x = x.to(torch.float32).contiguous()
    y = torch.empty_like(x)
    _lib.call("epk_debug_expf", ctx.handle, ptr(x), ptr(y), x.numel())
    return y
