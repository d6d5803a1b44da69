"""Episode KV cache resident in HBM, and evict_to_budget on it.

Mirrors kvcache.hpp: the reference keeps, per layer, a list of kv-heads each
holding a position-sorted std::vector<KVEntry> (kvcache.hpp:28-53).  Here a
whole episode lives in one allocation laid out for the GPU:

    k, v      [rows, head_dim]  (bf16, fp32 or fp64)     rows = sum of layer capacities
    pos       [rows] int32
    head_off  [layers, H+1] int32   region of head h (layer-relative rows)
    head_len  [layers, H]   int32   live rows at the start of each region

so a layer's heads are contiguous, per-head counts can be ragged (pooled
eviction makes them uneven), and the slack after each head receives the next
block's append without moving anything.

`evict_to_budget` has two faces:
  * the drop-in (`LayerCache`, `LayerScores`, pinned set) with the reference
    signature, semantics and exceptions (kvcache.hpp:142-201);
  * the device form on an EpisodeCache, used by the block-prefill engine.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .context import Context, default_context, ptr
from .errors import DimensionError, Error

_DT = {torch.float32: _lib.EPK_F32, torch.bfloat16: _lib.EPK_BF16, torch.float64: _lib.EPK_F64}


class EpisodeCache:
    """Layered CSR KV cache for one episode (EpisodicCache, kvcache.hpp:64-95)."""

    def __init__(self, layers: int, kv_heads: int, head_dim: int, capacity, dtype=torch.bfloat16,
                 device: int | str | torch.device = "cuda"):
        cap = np.broadcast_to(np.asarray(capacity, dtype=np.int64), (layers,)).copy()
        self.layers, self.kv_heads, self.head_dim, self.dtype = int(layers), int(kv_heads), int(head_dim), dtype
        self.capacity = cap
        self.layer_base = np.zeros(layers + 1, np.int64)
        self.layer_base[1:] = np.cumsum(cap)
        rows = int(self.layer_base[-1])
        dev = torch.device(device)
        self.device = dev
        self.k = torch.empty(rows, head_dim, dtype=dtype, device=dev)
        self.v = torch.empty(rows, head_dim, dtype=dtype, device=dev)
        self.pos = torch.full((rows,), -1, dtype=torch.int32, device=dev)
        self.head_off = torch.zeros(layers, kv_heads + 1, dtype=torch.int32, device=dev)
        self.head_len = torch.zeros(layers, kv_heads, dtype=torch.int32, device=dev)
        self._lb_c = (C.c_int64 * (layers + 1))(*self.layer_base.tolist())

    @property
    def rows(self) -> int:
        return int(self.layer_base[-1])

    def desc(self) -> _lib.CacheDesc:
        return _lib.CacheDesc(self.layers, self.kv_heads, self.head_dim, _DT[self.dtype], self.k.data_ptr(),
                              self.v.data_ptr(), self.pos.data_ptr(), self.head_off.data_ptr(),
                              self.head_len.data_ptr(), C.cast(self._lb_c, C.c_void_p))

    # ---- layout helpers ----------------------------------------------------
    def set_regions(self, region_rows_per_head) -> None:
        """Empty cache with head h of layer l owning rows [h*R_l, (h+1)*R_l)."""
        r = np.broadcast_to(np.asarray(region_rows_per_head, dtype=np.int64), (self.layers,))
        if np.any(r * self.kv_heads > self.capacity):
            raise Error("set_regions: regions exceed layer capacity")
        off = np.arange(self.kv_heads + 1, dtype=np.int64)[None, :] * r[:, None]
        self.head_off.copy_(torch.from_numpy(off.astype(np.int32)))
        self.head_len.zero_()

    def load_layers(self, per_layer, slack: int = 0) -> None:
        """Fills the cache from host data.  per_layer[l] = (head_counts[H], pos[n], k[n,d], v[n,d]),
        rows head-major and position-sorted within each head; every head is
        followed by `slack` free rows (0: stored dense)."""
        offs = np.zeros((self.layers, self.kv_heads + 1), np.int32)
        lens = np.zeros((self.layers, self.kv_heads), np.int32)
        for l, (counts, pos, k, v) in enumerate(per_layer):
            counts = np.asarray(counts, np.int64)
            n = int(counts.sum())
            if n + slack * self.kv_heads > self.capacity[l]:
                raise Error(f"load_layers: layer {l} has {n} rows (+ slack) > capacity {self.capacity[l]}")
            offs[l, 1:] = np.cumsum(counts + slack)
            lens[l] = counts
            b = int(self.layer_base[l])
            if n:
                dst = np.concatenate([np.arange(offs[l, h], offs[l, h] + counts[h]) for h in range(self.kv_heads)]) + b
                it = torch.as_tensor(dst, device=self.device, dtype=torch.int64)
                self.pos[it] = torch.as_tensor(np.asarray(pos, np.int32), device=self.device)
                self.k[it] = torch.as_tensor(np.asarray(k), device=self.device).to(self.dtype)
                self.v[it] = torch.as_tensor(np.asarray(v), device=self.device).to(self.dtype)
        self.head_off.copy_(torch.from_numpy(offs))
        self.head_len.copy_(torch.from_numpy(lens))

    def layer_view(self, l: int):
        """Host copy of layer l: (head_counts, pos, k, v) with the gaps removed."""
        off = self.head_off[l].cpu().numpy().astype(np.int64)
        ln = self.head_len[l].cpu().numpy().astype(np.int64)
        b = int(self.layer_base[l])
        idx = np.concatenate([np.arange(off[h], off[h] + ln[h]) for h in range(self.kv_heads)]) + b
        it = torch.as_tensor(idx, device=self.device, dtype=torch.int64)
        return ln, self.pos[it].cpu().numpy(), self.k[it].cpu(), self.v[it].cpu()

    def live_rows(self, l: int) -> torch.Tensor:
        """Global row indices of layer l's live entries (head-major)."""
        off = self.head_off[l].cpu().numpy().astype(np.int64)
        ln = self.head_len[l].cpu().numpy().astype(np.int64)
        b = int(self.layer_base[l])
        idx = np.concatenate([np.arange(off[h], off[h] + ln[h]) for h in range(self.kv_heads)]) + b
        return torch.as_tensor(idx, device=self.device, dtype=torch.int64)

    def entries_per_layer(self) -> list[int]:
        return self.head_len.sum(dim=1).cpu().tolist()

    def retained_positions(self) -> list[list[list[int]]]:
        """retained_positions (kvcache.hpp:220-236)."""
        out = []
        for l in range(self.layers):
            ln, pos, _, _ = self.layer_view(l)
            heads, o = [], 0
            for h in range(self.kv_heads):
                heads.append(pos[o:o + ln[h]].tolist())
                o += int(ln[h])
            out.append(heads)
        return out


def _pins_tensor(pinned, device) -> tuple[torch.Tensor | None, int]:
    if not pinned:
        return None, 0
    arr = np.unique(np.asarray(sorted(int(p) for p in pinned), dtype=np.int64))
    if arr.size and (arr.min() < 0 or arr.max() >= 2 ** 31):
        raise Error("pinned positions must fit in int32")
    return torch.as_tensor(arr.astype(np.int32), device=device), int(arr.size)


def select_pooled(cache: EpisodeCache, scores: torch.Tensor, layer_budgets, pinned=None, keep=None,
                  synchronous: bool = True, ctx: Context | None = None) -> torch.Tensor:
    """K2: keep mask (uint8 [rows]) of evict_to_budget's pooled selection."""
    ctx = ctx or default_context(cache.device.index)
    if scores.dtype not in (torch.float32, torch.float64) or scores.numel() < cache.rows:
        raise DimensionError("evict_to_budget: score head count mismatch")
    budgets = (C.c_int64 * cache.layers)(*[int(b) for b in np.broadcast_to(layer_budgets, (cache.layers,))])
    keep = keep if keep is not None else torch.zeros(cache.rows, dtype=torch.uint8, device=cache.device)
    pins, npins = _pins_tensor(pinned, cache.device)
    d = cache.desc()
    _lib.call("epk_select_pooled", ctx.handle, C.byref(d), ptr(scores),
              _lib.EPK_F32 if scores.dtype == torch.float32 else _lib.EPK_F64, C.cast(budgets, C.c_void_p),
              ptr(pins), npins, ptr(keep), None, int(synchronous))
    return keep


def select_per_head(cache: EpisodeCache, scores: torch.Tensor, k_per_layer, ctx: Context | None = None):
    """top_k_indices (numerics.hpp:111-125) applied to every (layer, kv-head)."""
    ctx = ctx or default_context(cache.device.index)
    ks = (C.c_int64 * cache.layers)(*[int(b) for b in np.broadcast_to(k_per_layer, (cache.layers,))])
    keep = torch.zeros(cache.rows, dtype=torch.uint8, device=cache.device)
    d = cache.desc()
    _lib.call("epk_select_per_head", ctx.handle, C.byref(d), ptr(scores),
              _lib.EPK_F32 if scores.dtype == torch.float32 else _lib.EPK_F64, C.cast(ks, C.c_void_p), ptr(keep))
    return keep


def compact(cache: EpisodeCache, keep: torch.Tensor, out: EpisodeCache, slack: int = 0,
            ctx: Context | None = None) -> EpisodeCache:
    """K3: stable gather of the kept rows into `out` (heads followed by `slack` free rows)."""
    ctx = ctx or default_context(cache.device.index)
    a, b = cache.desc(), out.desc()
    _lib.call("epk_compact", ctx.handle, C.byref(a), C.byref(b), ptr(keep), int(slack))
    return out


def append_to_cache(cache: EpisodeCache, k_new: torch.Tensor, v_new: torch.Tensor, positions: torch.Tensor,
                    slack: int = 0, ctx: Context | None = None) -> None:
    """append_to_cache (toymodel.hpp:428-443): k_new/v_new [layers, H, len, d].
    `slack` (> 0) is the gap the caller left after every head; a longer block
    is refused at once."""
    ctx = ctx or default_context(cache.device.index)
    if k_new.shape[:2] != (cache.layers, cache.kv_heads) or k_new.shape[3] != cache.head_dim:
        raise DimensionError("append_to_cache: block shape mismatch")
    d = cache.desc()
    _lib.call("epk_append", ctx.handle, C.byref(d), ptr(k_new.contiguous()), ptr(v_new.contiguous()),
              ptr(positions.to(torch.int32).contiguous()), int(k_new.shape[2]), int(slack))


def evict_device(cache: EpisodeCache, scores: torch.Tensor, layer_budgets, pinned=None,
                 out: EpisodeCache | None = None, slack: int = 0, ctx: Context | None = None) -> EpisodeCache:
    """evict_to_budget for every layer of a device cache -> a fresh compacted cache."""
    ctx = ctx or default_context(cache.device.index)
    keep = select_pooled(cache, scores, layer_budgets, pinned, synchronous=True, ctx=ctx)
    if out is None:
        out = EpisodeCache(cache.layers, cache.kv_heads, cache.head_dim, cache.capacity, cache.dtype, cache.device)
    return compact(cache, keep, out, slack, ctx)


# ---------------------------------------------------------------------------
# Drop-in reference API (kvcache.hpp:28-53,134,142)
# ---------------------------------------------------------------------------

@dataclass
class KVEntry:
    position: int
    key: list = field(default_factory=list)
    value: list = field(default_factory=list)


@dataclass
class LayerCache:
    heads: list
    budget: int = 0

    @staticmethod
    def empty(kv_heads: int, budget: int) -> "LayerCache":
        return LayerCache([[] for _ in range(kv_heads)], budget)

    def entry_count(self) -> int:
        return sum(len(h) for h in self.heads)


def evict_to_budget(cache: LayerCache, scores, pinned=frozenset()) -> LayerCache:
    """Drop-in for epikv::evict_to_budget (kvcache.hpp:142): same arguments
    (per-head position->score maps), same result, same exceptions; computed by
    the K2/K3 kernels in fp64 on the GPU."""
    H = len(cache.heads)
    if len(scores) != H:
        raise DimensionError("evict_to_budget: score head count mismatch")
    limit = H * cache.budget
    if cache.entry_count() <= limit:
        return LayerCache([list(h) for h in cache.heads], cache.budget)
    counts = [len(h) for h in cache.heads]
    pos = np.array([e.position for h in cache.heads for e in h], dtype=np.int64)
    sc = np.empty(pos.size, np.float64)
    i = 0
    for h, entries in enumerate(cache.heads):
        for e in entries:
            if e.position in pinned:
                sc[i] = 0.0
            else:
                try:
                    sc[i] = scores[h][e.position]
                except KeyError:
                    raise DimensionError(f"evict_to_budget: missing score for head {h} position {e.position}")
            i += 1
    if pos.size and pos.max() >= 2 ** 31:
        raise Error("evict_to_budget: positions must fit in int32 on the device path")
    dim = max((len(e.key) for h in cache.heads for e in h), default=0)
    dev = torch.device("cuda", torch.cuda.current_device())
    dc = EpisodeCache(1, H, max(dim, 2), [max(pos.size, 1)], torch.float64, dev)
    kk = np.zeros((pos.size, max(dim, 2)), np.float64)
    vv = np.zeros_like(kk)
    i = 0
    for entries in cache.heads:
        for e in entries:
            kk[i, :len(e.key)] = e.key
            vv[i, :len(e.value)] = e.value
            i += 1
    dc.load_layers([(counts, pos, kk, vv)])
    keep = select_pooled(dc, torch.as_tensor(sc, device=dev), [cache.budget], set(pinned), synchronous=True)
    out_dc = EpisodeCache(1, H, max(dim, 2), [max(pos.size, 1)], torch.float64, dev)
    compact(dc, keep, out_dc, 0)
    default_context(dev.index).poll_error()
    ln, opos, ok, ov = out_dc.layer_view(0)
    out = LayerCache.empty(H, cache.budget)
    src = np.nonzero(keep.cpu().numpy().astype(bool))[0]
    flat = [e for entries in cache.heads for e in entries]
    ok = ok.numpy()
    r = 0
    for h in range(H):
        for _ in range(int(ln[h])):
            e = flat[src[r]]
            # the device-compacted row must be this entry, bit for bit
            if e.position != int(opos[r]) or (dim and not np.array_equal(ok[r, :len(e.key)], np.asarray(e.key))):
                raise Error("evict_to_budget: device compaction mismatch")
            out.heads[h].append(e)
            r += 1
    return out
