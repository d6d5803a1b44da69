"""Episodic cache store (kvcache.hpp:281-429, episodic.hpp:76-99,227-253).

The writer runs on the GPU: `persist` serialises a device-resident
EpisodeCache into the reference's `.epkv` byte stream with one kernel
(`epk_serialize_epkv`, csrc/store.cu: keys/values widened to fp64 exactly, the
reference's field layout), copies the finished bytes into pinned host memory
in one D2H transfer and writes them out -- byte-identical to the reference's
`persist` for the same cache.  `load_cache` parses a `.epkv` file (the
reference's or ours) with vectorised numpy views and uploads it as an
EpisodeCache in one H2D pass.  `CacheStore` mirrors the reference's
directory of `episode_<e>.epkv` files plus `manifest.json`; `route` is
Phase B's query-to-episode routing (cosine to the centroids, ties to the
lower id) with the load-on-switch rule.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .context import Context, default_context, ptr
from .errors import Error, IoError
from .kvcache import EpisodeCache

_MAGIC = b"EPKV"
_VERSION = 1


@dataclass
class CacheMeta:
    """The .epkv header fields beyond the entries (kvcache.hpp:287-299, CacheProvenance)."""
    episode_id: int = 0
    scorer: str = ""
    budget_per_head: int = 0
    layer_budgets: list = field(default_factory=list)
    layer_budget_fields: list = field(default_factory=list)  # LayerCache::budget of every layer


def serialize(cache: EpisodeCache, episode_id: int = 0, scorer: str = "patched", budget_per_head: int = 0,
              layer_budgets=None, ctx: Context | None = None) -> torch.Tensor:
    """The .epkv bytes of `cache` as a pinned host uint8 tensor (persist's
    stream, kvcache.hpp:281-317).  Per-layer budget fields are
    layer_budgets[l] (else budget_per_head)."""
    ctx = ctx or default_context(cache.device.index)
    lb = [int(b) for b in (layer_budgets or [])]
    lb_c = (C.c_int64 * max(1, len(lb)))(*lb) if lb else None
    d = cache.desc()
    off, tot = C.c_int64(0), C.c_int64(0)
    sc = scorer.encode()
    _lib.call("epk_serialize_epkv", ctx.handle, C.byref(d), int(episode_id), sc, int(budget_per_head),
              C.cast(lb_c, C.c_void_p) if lb_c else None, len(lb), None, 0, C.byref(off), C.byref(tot))
    buf = torch.empty(off.value + tot.value + 16, dtype=torch.uint8, device=cache.device)
    _lib.call("epk_serialize_epkv", ctx.handle, C.byref(d), int(episode_id), sc, int(budget_per_head),
              C.cast(lb_c, C.c_void_p) if lb_c else None, len(lb), ptr(buf), buf.numel(), C.byref(off),
              C.byref(tot))
    host = torch.empty(tot.value, dtype=torch.uint8, pin_memory=True)
    host.copy_(buf[off.value:off.value + tot.value], non_blocking=True)
    torch.cuda.current_stream(cache.device).synchronize()
    return host


def persist(cache: EpisodeCache, path, episode_id: int = 0, scorer: str = "patched", budget_per_head: int = 0,
            layer_budgets=None, ctx: Context | None = None) -> int:
    """persist (kvcache.hpp:281): writes the cache; returns the byte count."""
    data = serialize(cache, episode_id, scorer, budget_per_head, layer_budgets, ctx)
    try:
        with open(path, "wb") as f:
            f.write(memoryview(data.numpy()))
    except OSError as e:
        raise IoError(f"persist: cannot open {path}") from e
    return data.numel()


class _Reader:
    def __init__(self, buf: bytes, path):
        self.b, self.p, self.path = buf, 0, path

    def take(self, n: int) -> memoryview:
        if self.p + n > len(self.b):
            raise IoError("cache file truncated")
        v = memoryview(self.b)[self.p:self.p + n]
        self.p += n
        return v

    def u(self, n: int) -> int:
        return int.from_bytes(self.take(n), "little")


def parse(buf: bytes, path="<bytes>"):
    """-> (CacheMeta, per_layer) with per_layer[l] = (head_counts[H], pos[n] int64,
    k[n, d] f64, v[n, d] f64) in head-major, file order (load_cache,
    kvcache.hpp:321-372; fails closed like the reference)."""
    r = _Reader(buf, path)
    if bytes(r.take(4)) != _MAGIC:
        raise IoError(f"load: bad magic in {path}")
    ver = r.u(2)
    if ver != _VERSION:
        raise IoError(f"load: version mismatch in {path} (got {ver}, expected {_VERSION})")
    meta = CacheMeta(episode_id=r.u(8))
    layers = r.u(4)
    r.u(4)  # head count of layer 0 (redundant)
    meta.scorer = bytes(r.take(r.u(4))).decode()
    meta.budget_per_head = r.u(8)
    meta.layer_budgets = [r.u(8) for _ in range(r.u(4))]
    per_layer = []
    for _ in range(layers):
        meta.layer_budget_fields.append(r.u(8))
        heads = r.u(4)
        counts, pos, ks, vs = [], [], [], []
        for _ in range(heads):
            n = r.u(8)
            counts.append(n)
            if n == 0:
                continue
            if r.p + 12 > len(r.b):
                raise IoError("cache file truncated")
            dim = int.from_bytes(r.b[r.p + 8:r.p + 12], "little")
            dt = np.dtype([("pos", "<u8"), ("dim", "<u4"), ("k", "<f8", (dim,)), ("v", "<f8", (dim,))])
            rec = np.frombuffer(r.take(n * dt.itemsize), dtype=dt, count=n)
            if np.any(rec["dim"] != dim):
                raise Error("load: ragged key dimensions are not supported by the device cache")
            pos.append(rec["pos"].astype(np.int64))
            ks.append(rec["k"].reshape(n, dim))
            vs.append(rec["v"].reshape(n, dim))
        dim = ks[0].shape[1] if ks else 0
        per_layer.append((np.array(counts, np.int64),
                          np.concatenate(pos) if pos else np.zeros(0, np.int64),
                          np.concatenate(ks) if ks else np.zeros((0, dim)),
                          np.concatenate(vs) if vs else np.zeros((0, dim))))
    return meta, per_layer


def _parse_header(buf, path) -> CacheMeta:
    r = _Reader(buf, path)
    if bytes(r.take(4)) != _MAGIC:
        raise IoError(f"load: bad magic in {path}")
    if r.u(2) != _VERSION:
        raise IoError(f"load: version mismatch in {path}")
    meta = CacheMeta(episode_id=r.u(8))
    layers = r.u(4)
    r.u(4)
    meta.scorer = bytes(r.take(r.u(4))).decode()
    meta.budget_per_head = r.u(8)
    meta.layer_budgets = [r.u(8) for _ in range(r.u(4))]
    return meta, layers, r.p


def retrieve(path, dtype=torch.bfloat16, device="cuda", slack: int = 0, ctx: Context | None = None):
    """load_cache on the GPU (Phase B "KVs Retrieve"): the file's structure is
    walked on the host through a memory map (epk_epkv_scan touches only the
    header and count fields), the bytes stream from the file into reused
    pinned buffers and across PCIe, and epk_load_epkv narrows every entry into
    a device cache (values must round-trip to `dtype`, like
    load_cache(exact=True)).  -> (EpisodeCache, CacheMeta)."""
    dev = torch.device(device)
    ctx = ctx or default_context(dev.index if dev.index is not None else torch.cuda.current_device())
    try:
        size = os.path.getsize(path)
        mm = np.memmap(path, dtype=np.uint8, mode="r") if size else np.zeros(0, np.uint8)
    except (OSError, ValueError) as e:
        raise IoError(f"load: cannot open {path}") from e
    info = (C.c_int64 * 4)()
    base = C.c_void_p(mm.ctypes.data if size else 0)
    rc = _lib.load().epk_epkv_scan(base, size, C.cast(info, C.c_void_p), None, None)
    if rc != 0:
        raise IoError(_lib.load().epk_last_error().decode())
    L, H, d = int(info[0]), int(info[1]), int(info[2])
    counts = np.zeros(max(1, L * H), np.int64)
    eoff = np.zeros(max(1, L * H), np.int64)
    _lib.call("epk_epkv_scan", base, size, C.cast(info, C.c_void_p), counts.ctypes.data_as(C.c_void_p),
              eoff.ctypes.data_as(C.c_void_p))
    meta, _, _ = _parse_header(bytes(mm[:int(info[3])]), path)
    if L < 1:
        raise Error("load: cache has no layers")
    counts = counts[:L * H].reshape(L, H)
    meta.layer_budget_fields = _layer_budget_fields(mm, int(info[3]), L, H, counts, d)  # kvcache.hpp:304
    del mm
    cap = [int(counts[l].sum()) + slack * H for l in range(L)]
    cache = EpisodeCache(L, H, d, cap, dtype, dev)
    offs = np.zeros((L, H + 1), np.int32)
    offs[:, 1:] = np.cumsum(counts + slack, axis=1)
    cache.head_off.copy_(torch.from_numpy(offs))
    cache.head_len.copy_(torch.from_numpy(counts.astype(np.int32)))
    pad = (-int(eoff[0])) % 4
    dfile = torch.empty(size + pad, dtype=torch.uint8, device=dev)
    try:
        with open(path, "rb", buffering=0) as f:
            _file_to_device(f, size, dfile[pad:])
    except OSError as e:
        raise IoError(f"load: cannot read {path}") from e
    desc = cache.desc()
    _lib.call("epk_load_epkv", ctx.handle, ptr(dfile), pad, eoff.ctypes.data_as(C.c_void_p), C.byref(desc))
    ctx.poll_error()  # fails closed: a value that does not round-trip to dtype
    return cache, meta


_STAGE = []


def _file_to_device(f, size: int, dst: torch.Tensor, chunk: int = 64 << 20) -> None:
    """File bytes -> device through two reused pinned 64 MB buffers: the read
    into one overlaps the DMA out of the other."""
    if not _STAGE:
        _STAGE.extend(torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2))
        _STAGE.extend(torch.cuda.Event() for _ in range(2))
    bufs, evs = _STAGE[:2], _STAGE[2:]
    stream = torch.cuda.current_stream(dst.device)
    used = [False, False]
    for i, a in enumerate(range(0, size, chunk)):
        j = i % 2
        n = min(chunk, size - a)
        if used[j]:
            evs[j].synchronize()
        got = f.readinto(memoryview(bufs[j].numpy())[:n])
        if got != n:
            raise IoError("cache file truncated")
        dst[a:a + n].copy_(bufs[j][:n], non_blocking=True)
        evs[j].record(stream)
        used[j] = True
    for j in range(2):
        if used[j]:
            evs[j].synchronize()


def _layer_budget_fields(hb, at, L, H, counts, d):
    out = []
    for l in range(L):
        out.append(int.from_bytes(bytes(hb[at:at + 8]), "little"))
        at += 12
        for h in range(H):
            at += 8 + int(counts[l, h]) * (12 + 16 * d)
    return out


def load_cache(path, dtype=torch.bfloat16, device="cuda", slack: int = 0, exact: bool = True):
    """load_cache (kvcache.hpp:321): -> (EpisodeCache, CacheMeta).  The fp64
    reals narrow to `dtype`; with exact=True a value that does not round-trip
    raises (a bf16/fp32 cache persisted by `persist` always round-trips).
    Each head gets `slack` free rows after its entries (room for appends).
    Host-side parse (numpy); `retrieve` is the same on the GPU."""
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError as e:
        raise IoError(f"load: cannot open {path}") from e
    meta, per_layer = parse(buf, path)
    if not per_layer:
        raise Error("load: cache has no layers")
    H = len(per_layer[0][0])
    dims = {pl[2].shape[1] for pl in per_layer if pl[2].shape[0]}
    if len(dims) > 1:
        raise Error("load: layers with different key dimensions")
    d = dims.pop() if dims else 1
    cap = [int(pl[0].sum()) + slack * H for pl in per_layer]
    cache = EpisodeCache(len(per_layer), H, d, cap, dtype, device)
    if exact and dtype != torch.float64:
        for _, _, k, v in per_layer:
            for a in (k, v):
                t = torch.as_tensor(a).to(dtype).double().numpy()
                if not np.array_equal(t, a):
                    raise Error(f"load: values are not exactly representable in {dtype}")
    cache.load_layers([(c, p, k, v) for c, p, k, v in per_layer], slack=slack)
    return cache, meta


class CacheStore:
    """Directory of episode_<e>.epkv files plus manifest.json (kvcache.hpp:375-429)."""

    def __init__(self, directory):
        self.dir = str(directory)
        try:
            os.makedirs(self.dir, exist_ok=True)
        except OSError as e:
            raise IoError(f"store: cannot create {self.dir}: {e}") from e

    def episode_path(self, episode_id: int) -> str:
        return os.path.join(self.dir, f"episode_{int(episode_id)}.epkv")

    def save(self, cache: EpisodeCache, episode_id: int, **provenance) -> int:
        return persist(cache, self.episode_path(episode_id), episode_id=episode_id, **provenance)

    def load(self, episode_id: int, **kw):
        path = self.episode_path(episode_id)
        if not os.path.exists(path):
            raise IoError(f"store: unknown episode id {episode_id}")
        return load_cache(path, **kw)

    def stored_bytes(self, episode_id: int) -> int:
        try:
            return os.path.getsize(self.episode_path(episode_id))
        except OSError:
            return 0

    def write_manifest(self, manifest: dict) -> None:
        """manifest.json, dumped with 2-space indent like nlohmann::ordered_json::dump(2)."""
        try:
            with open(os.path.join(self.dir, "manifest.json"), "w") as f:
                f.write(json.dumps(manifest, indent=2, ensure_ascii=False) + "\n")
        except OSError as e:
            raise IoError(f"store: cannot write manifest in {self.dir}") from e

    def read_manifest(self) -> dict:
        try:
            with open(os.path.join(self.dir, "manifest.json")) as f:
                return json.load(f)
        except OSError as e:
            raise IoError(f"store: missing manifest in {self.dir}") from e


def manifest_json(centroids, prompt_turn_spans, prompt_texts, store: CacheStore, scorer: str,
                  budget_per_head: int, layer_budgets, embed_dim: int) -> dict:
    """detail::manifest_json (episodic.hpp:76-99), key order preserved."""
    eps = []
    for e, c in enumerate(centroids):
        eps.append({"id": e, "file": os.path.basename(store.episode_path(e)), "centroid": [float(x) for x in c],
                    "medoid_first_turn": int(prompt_turn_spans[e][0]),
                    "medoid_turn_count": int(prompt_turn_spans[e][1]), "prompt_text": prompt_texts[e]})
    return {"version": 1, "embedder_dim": int(embed_dim), "budget_per_head": int(budget_per_head),
            "scorer": scorer, "layer_budgets": [int(b) for b in layer_budgets], "episodes": eps}


@dataclass
class RouteRecord:
    turn: int
    episode: int
    switched: bool = False
    load_bytes: int = 0


@dataclass
class SessionState:
    """SessionState (episodic.hpp:62-67): the resident episode cache in HBM."""
    resident_id: int | None = None
    resident: EpisodeCache | None = None
    switch_count: int = 0
    route_log: list = field(default_factory=list)


def _seq_dot(a, b) -> float:
    acc = 0.0
    for x, y in zip(a, b):  # sequential, like numerics.hpp:52-70 (built-in sum() is compensated)
        acc += x * y
    return acc


def centroid_similarity(q, c) -> float:
    """centroid_similarity (clustering.hpp:289-294): cosine (numerics.hpp:75-87,
    sequential sums, clamp) or -inf when either vector has zero norm."""
    q = [float(x) for x in np.asarray(q, np.float64).ravel()]
    c = [float(x) for x in np.asarray(c, np.float64).ravel()]
    na, nb = math.sqrt(_seq_dot(q, q)), math.sqrt(_seq_dot(c, c))
    if na == 0.0 or nb == 0.0:
        return -math.inf
    return max(-1.0, min(1.0, _seq_dot(q, c) / (na * nb)))


def route(store: CacheStore, centroids, query_embedding, state: SessionState, **load_kw) -> int:
    """route (episodic.hpp:227-253): the episode whose centroid is most cosine-
    similar to the query (ties to the lower id); its cache is loaded into HBM
    only when it differs from the resident one."""
    best, best_cos = 0, -math.inf
    for e, c in enumerate(centroids):
        s = centroid_similarity(query_embedding, c)
        if s > best_cos:
            best, best_cos = e, s
    rec = RouteRecord(turn=len(state.route_log), episode=best)
    if state.resident_id is None or state.resident_id != best:
        state.resident, _ = store.load(best, **load_kw)
        state.resident_id = best
        rec.switched = True
        rec.load_bytes = store.stored_bytes(best)
        state.switch_count += 1
    state.route_log.append(rec)
    return best
