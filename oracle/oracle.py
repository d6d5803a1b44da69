"""ctypes front-end for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Loads oracle/_build/libepkoracle.so (the plain-C++ restatement in
epk_oracle.cpp) and, when present, oracle/_ref/libepkref.so (the reference
headers compiled in place, ref_shim.cpp).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs import this module; the
product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libepkoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libepkref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile the oracle (and oracle/_ref where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str):
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        lib = _load(ORACLE_SO)
        lib.orc_score_layer_f64.argtypes = [C.c_int] * 4 + [_i64p, _f64p, _f64p, _f64p, C.c_int, _f64p]
        lib.orc_score_layer_f64.restype = None
        lib.orc_score_layer_f32.argtypes = [C.c_int] * 4 + [_i64p, _f32p, _f32p, _f32p, C.c_int, _f32p]
        lib.orc_score_layer_f32.restype = None
        lib.orc_score_layer_f64_mt.argtypes = [C.c_int] * 4 + [_i64p, _f64p, _f64p, _f64p, C.c_int, _f64p, C.c_int]
        lib.orc_score_layer_f64_mt.restype = None
        lib.orc_score_layer_f32_mt.argtypes = [C.c_int] * 4 + [_i64p, _f32p, _f32p, _f32p, C.c_int, _f32p, C.c_int]
        lib.orc_score_layer_f32_mt.restype = None
        lib.orc_prompt_grids_f64.argtypes = [C.c_int] * 4 + [_i64p, _f64p, _f64p, _f64p, _f64p]
        lib.orc_prompt_grids_f64.restype = None
        lib.orc_expf.argtypes = [C.c_float]
        lib.orc_expf.restype = C.c_float
        lib.orc_expf_many.argtypes = [_f32p, C.c_int64, _f32p]
        lib.orc_tree_sum.argtypes = [_f32p, C.c_int64]
        lib.orc_tree_sum.restype = C.c_float
        lib.orc_evict_layer.argtypes = [C.c_int, C.c_int64, _i64p, _i64p, _f64p, _i64p, C.c_int64, _u8p]
        lib.orc_evict_layer.restype = C.c_int
        lib.orc_topk_per_head.argtypes = [C.c_int, C.c_int64, _i64p, _f64p, _u8p]
        lib.orc_kmeans.argtypes = [_f64p, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int64,
                                   _i64p, _f64p, _i64p, _f64p]
        lib.orc_kmeans.restype = C.c_int
        lib.orc_sensitivity.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, _f64p, _f64p, _f64p, _i64p]
        lib.orc_allocate.argtypes = [_f64p, C.c_int, C.c_int64, C.c_double, _i64p, _f64p]
        lib.orc_keydiff_layer.argtypes = [C.c_int, C.c_int, _i64p, _f64p, _f64p]
        lib.orc_keydiff_layer.restype = None
        lib.orc_allocate.restype = C.c_int
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir("/root/reference/proj/include/epikv")


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_score_layer_f64.argtypes = [C.c_int] * 4 + [_i64p, _i64p, _f64p, _f64p, _f64p, C.c_int, _f64p]
        lib.ref_score_layer_f64.restype = C.c_int
        lib.ref_score_grids.argtypes = [C.c_int] * 3 + [_i64p, _i64p, _f64p, C.c_int, _f64p]
        lib.ref_score_grids.restype = C.c_int
        lib.ref_evict_layer.argtypes = [C.c_int, C.c_int64, C.c_int, _i64p, _i64p, C.c_void_p, C.c_void_p,
                                        _f64p, _i64p, C.c_int64, _u8p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]
        lib.ref_evict_layer.restype = C.c_int64
        lib.ref_step_layer_f64.argtypes = [C.c_int] * 4 + [C.c_int64, _i64p, _i64p, _f64p, C.c_void_p,
                                                           C.c_void_p, _f64p, C.c_int, _u8p]
        lib.ref_step_layer_f64.restype = C.c_int64
        lib.ref_top_k_indices.argtypes = [_f64p, C.c_int64, C.c_int64, _i64p]
        lib.ref_top_k_indices.restype = C.c_int64
        lib.ref_cosine.argtypes = [_f64p, _f64p, C.c_int64]
        lib.ref_keydiff_layer.argtypes = [C.c_int, C.c_int, _i64p, _i64p, _f64p, _f64p]
        lib.ref_keydiff_layer.restype = C.c_int
        lib.ref_persist.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, _i64p, C.c_int, C.c_int, C.c_int,
                                    C.c_int, _i64p, _i64p, _f64p, _f64p, _i64p]
        lib.ref_persist.restype = C.c_int64
        lib.ref_load_repersist.argtypes = [C.c_char_p, C.c_char_p]
        lib.ref_load_repersist.restype = C.c_int64
        lib.ref_cosine.restype = C.c_double
        lib.ref_kmeans.argtypes = [_f64p, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int64,
                                   _i64p, _f64p, _i64p, _f64p]
        lib.ref_kmeans.restype = C.c_int
        lib.ref_allocate.argtypes = [_f64p, C.c_int, C.c_int64, C.c_double, _i64p, _f64p]
        lib.ref_allocate.restype = C.c_int
        lib.ref_measure_sensitivity.argtypes = [C.c_int] * 4 + [C.c_uint64, C.c_int64, C.c_uint64,
                                                                C.c_int64, C.c_int64, _f64p, _i64p, _f64p, _f64p]
        lib.ref_measure_sensitivity.restype = C.c_int
        lib.ref_block_prefill.argtypes = [C.c_int] * 4 + [C.c_uint64, C.c_int64, C.c_uint64, C.c_int64,
                                                          C.c_int64, _i64p, C.c_int64, C.c_void_p, _i64p,
                                                          _i64p, _i64p, _i64p, _i64p, _i64p]
        lib.ref_block_prefill.restype = C.c_int
        _ref = lib
    return _ref


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ---------------------------------------------------------------------------
# Oracle restatement (epk_oracle.cpp)
# ---------------------------------------------------------------------------

def score_layer_f64(q, k, kp, head_off, agg_max=True):
    """q [Hq,p,d], k [n,d], kp [Hkv,p,d], head_off [Hkv+1] -> scores [n] (fp64)."""
    hq, p, d = q.shape
    hkv = kp.shape[0]
    out = np.empty(k.shape[0], np.float64)
    orc().orc_score_layer_f64(hq, hkv, d, p, _c(head_off, np.int64), _c(q, np.float64), _c(k, np.float64),
                              _c(kp, np.float64), int(agg_max), out)
    return out


def score_layer_f64_mt(q, k, kp, head_off, agg_max=True, threads=0):
    """score_layer_f64 on `threads` host threads (0: all cores); same bits."""
    hq, p, d = q.shape
    hkv = kp.shape[0]
    out = np.empty(k.shape[0], np.float64)
    orc().orc_score_layer_f64_mt(hq, hkv, d, p, _c(head_off, np.int64), _c(q, np.float64), _c(k, np.float64),
                                 _c(kp, np.float64), int(agg_max), out, int(threads))
    return out


def score_layer_f32_mt(q, k, kp, head_off, agg_max=True, threads=0):
    """score_layer_f32 (EPK-F32 v1) on `threads` host threads; same bits."""
    hq, p, d = q.shape
    hkv = kp.shape[0]
    out = np.empty(k.shape[0], np.float32)
    orc().orc_score_layer_f32_mt(hq, hkv, d, p, _c(head_off, np.int64), _c(q, np.float32), _c(k, np.float32),
                                 _c(kp, np.float32), int(agg_max), out, int(threads))
    return out


def prompt_grids_f64(q, k, kp, head_off):
    """The restated fp64 attention grids: list of Hq arrays [p, n_h + p]."""
    hq, p, d = q.shape
    hkv = kp.shape[0]
    head_off = _c(head_off, np.int64)
    G = hq // hkv
    sizes = [p * (int(head_off[qh // G + 1] - head_off[qh // G]) + p) for qh in range(hq)]
    flat = np.zeros(sum(sizes), np.float64)
    orc().orc_prompt_grids_f64(hq, hkv, d, p, head_off, _c(q, np.float64), _c(k, np.float64), _c(kp, np.float64),
                               flat)
    out, o = [], 0
    for qh, sz in enumerate(sizes):
        out.append(flat[o:o + sz].reshape(p, -1))
        o += sz
    return out


def score_layer_f32(q, k, kp, head_off, agg_max=True):
    hq, p, d = q.shape
    hkv = kp.shape[0]
    out = np.empty(k.shape[0], np.float32)
    orc().orc_score_layer_f32(hq, hkv, d, p, _c(head_off, np.int64), _c(q, np.float32), _c(k, np.float32),
                              _c(kp, np.float32), int(agg_max), out)
    return out


def maxpool_scores(head_off, scores, kernel):
    """Opt-in max-pool smoothing restated (north_star; no reference counterpart):
    per head, pooled[j] = max scores[i] over |i - j| <= kernel // 2 within the
    head (SnapKV's max_pool1d, stride 1, same padding).  TEST INFRASTRUCTURE."""
    head_off = np.asarray(head_off, np.int64)
    s = np.asarray(scores)
    out = np.empty_like(s)
    half = int(kernel) // 2
    for h in range(len(head_off) - 1):
        a, b = int(head_off[h]), int(head_off[h + 1])
        seg = s[a:b]
        n = b - a
        if n == 0:
            continue
        pad = np.concatenate([np.full(half, -np.inf, s.dtype), seg, np.full(half, -np.inf, s.dtype)])
        win = np.lib.stride_tricks.sliding_window_view(pad, 2 * half + 1)
        out[a:b] = win.max(axis=1).astype(s.dtype)
    return out


def expf(x):
    x = _c(x, np.float32).ravel()
    out = np.empty_like(x)
    orc().orc_expf_many(x, x.size, out)
    return out


def tree_sum(e):
    e = _c(e, np.float32)
    return np.float32(orc().orc_tree_sum(e, e.size))


def evict_layer(head_off, pos, scores, budget, pins=()):
    """-> (status, keep[n] bool).  status 0 evicted, 1 under budget, -2 pin overflow."""
    head_off = _c(head_off, np.int64)
    n = int(head_off[-1])
    keep = np.zeros(n, np.uint8)
    pins = _c(np.array(list(pins), dtype=np.int64).reshape(-1), np.int64)
    if pins.size == 0:
        pins = np.zeros(1, np.int64)
        npins = 0
    else:
        npins = pins.size
    st = orc().orc_evict_layer(len(head_off) - 1, int(budget), head_off, _c(pos, np.int64),
                               _c(scores, np.float64), pins, npins, keep)
    return st, keep.astype(bool)


def topk_per_head(head_off, scores, k):
    head_off = _c(head_off, np.int64)
    keep = np.zeros(int(head_off[-1]), np.uint8)
    orc().orc_topk_per_head(len(head_off) - 1, int(k), head_off, _c(scores, np.float64), keep)
    return keep.astype(bool)


def kmeans(points, k, seed, max_iters=64):
    pts = _c(points, np.float64)
    n, dim = pts.shape
    assign = np.zeros(n, np.int64)
    cent = np.zeros((k, dim), np.float64)
    iters = np.zeros(1, np.int64)
    sse = np.zeros(max(max_iters, 1), np.float64)
    rc = orc().orc_kmeans(pts, n, dim, k, seed, max_iters, assign, cent.reshape(-1), iters, sse)
    if rc != 0:
        raise ValueError("kmeans: bad arguments")
    return assign, cent, int(iters[0]), sse[: int(iters[0])]


def sensitivity(kf, kb):
    kf = _c(kf, np.float64)
    kb = _c(kb, np.float64)
    L, H, N, d = kf.shape
    sigma = np.zeros(L, np.float64)
    skipped = np.zeros(1, np.int64)
    orc().orc_sensitivity(L, H, N, d, kf.reshape(-1), kb.reshape(-1), sigma, skipped)
    return sigma, int(skipped[0])


def keydiff_layer(k, head_off):
    """KeyDiff scores of one layer (scoring.hpp:186-221), rows in cache order."""
    k = _c(k, np.float64)
    ho = _c(head_off, np.int64)
    out = np.zeros(k.shape[0], np.float64)
    orc().orc_keydiff_layer(len(ho) - 1, k.shape[1], ho, k.reshape(-1), out)
    return out


def allocate(sens, per_head_budget, alpha):
    sens = _c(sens, np.float64)
    b = np.zeros(sens.size, np.int64)
    w = np.zeros(sens.size, np.float64)
    rc = orc().orc_allocate(sens, sens.size, int(per_head_budget), float(alpha), b, w)
    if rc != 0:
        raise ValueError("allocate: error")
    return b, w


# ---------------------------------------------------------------------------
# Reference (oracle/_ref/libepkref.so)
# ---------------------------------------------------------------------------

def _check(rc):
    if rc < 0:
        raise RefError(int(rc), ref().ref_last_error().decode())
    return rc


def ref_score_layer_f64(q, k, kp, head_off, pos, agg_max=True):
    hq, p, d = q.shape
    hkv = kp.shape[0]
    out = np.empty(k.shape[0], np.float64)
    _check(ref().ref_score_layer_f64(hq, hkv, d, p, _c(head_off, np.int64), _c(pos, np.int64),
                                     _c(q, np.float64), _c(k, np.float64), _c(kp, np.float64),
                                     int(agg_max), out))
    return out


def ref_score_grids(grids, head_off, pos, hq, agg_max=True):
    """grids: list of Hq arrays [p, n_h + p] (fp64)."""
    hkv = len(head_off) - 1
    p = grids[0].shape[0]
    flat = np.concatenate([_c(g, np.float64).ravel() for g in grids])
    out = np.empty(int(head_off[-1]), np.float64)
    _check(ref().ref_score_grids(hq, hkv, p, _c(head_off, np.int64), _c(pos, np.int64), flat,
                                 int(agg_max), out))
    return out


def ref_evict_layer(head_off, pos, scores, budget, pins=(), k=None, v=None):
    """-> (keep[n] bool, per-head counts, compacted (k, v, pos) or None)."""
    head_off = _c(head_off, np.int64)
    hkv = len(head_off) - 1
    n = int(head_off[-1])
    d = 0 if k is None else k.shape[1]
    keep = np.zeros(n, np.uint8)
    counts = np.zeros(hkv, np.int64)
    pins = np.array(list(pins), dtype=np.int64).reshape(-1)
    npins = pins.size
    if npins == 0:
        pins = np.zeros(1, np.int64)
    kk = vv = ko = vo = po = None
    if k is not None:
        kk = _c(k, np.float64)
        vv = _c(v, np.float64)
        ko = np.zeros_like(kk)
        vo = np.zeros_like(vv)
    po = np.zeros(max(n, 1), np.int64)
    total = _check(ref().ref_evict_layer(hkv, int(budget), d, head_off, _c(pos, np.int64), _ptr(kk), _ptr(vv),
                                         _c(scores, np.float64), pins, npins, keep, _ptr(counts), _ptr(ko),
                                         _ptr(vo), _ptr(po)))
    comp = None
    if k is not None:
        comp = (ko[:total], vo[:total], po[:total])
    else:
        comp = (None, None, po[:total])
    return keep.astype(bool), counts, comp


def ref_top_k_indices(scores, k):
    scores = _c(scores, np.float64)
    out = np.zeros(max(scores.size, 1), np.int64)
    m = ref().ref_top_k_indices(scores, scores.size, int(k), out)
    return out[:m]


def ref_keydiff_layer(k, head_off, pos):
    k = _c(k, np.float64)
    ho = _c(head_off, np.int64)
    out = np.zeros(k.shape[0], np.float64)
    _check(ref().ref_keydiff_layer(len(ho) - 1, k.shape[1], ho, _c(pos, np.int64), k.reshape(-1), out))
    return out


def ref_persist(path, per_layer, episode_id=0, scorer="patched", budget_per_head=0, layer_budgets=(),
                layer_budget_fields=None):
    """persist (kvcache.hpp:281) of per_layer[l] = (head_counts, pos, k, v) (fp64)."""
    L = len(per_layer)
    H = len(per_layer[0][0])
    d = per_layer[0][2].shape[1]
    ho, rows = [], 0
    for counts, _, _, _ in per_layer:
        c = np.concatenate([[0], np.cumsum(counts)]) + rows
        ho.append(c)
        rows = int(c[-1])
    pos = np.concatenate([p for _, p, _, _ in per_layer]).astype(np.int64)
    k = np.concatenate([x for _, _, x, _ in per_layer]).astype(np.float64)
    v = np.concatenate([x for _, _, _, x in per_layer]).astype(np.float64)
    lb = _c(np.asarray(list(layer_budgets) or [0], np.int64), np.int64)
    fields = _c(np.asarray(layer_budget_fields if layer_budget_fields is not None else [budget_per_head] * L,
                           np.int64), np.int64)
    n = ref().ref_persist(str(path).encode(), int(episode_id), scorer.encode(), int(budget_per_head), lb,
                          len(list(layer_budgets)), L, H, d, _c(np.concatenate(ho), np.int64), _c(pos, np.int64),
                          _c(k, np.float64), _c(v, np.float64), fields)
    _check(n)
    return int(n)


def ref_load_repersist(src, dst):
    n = ref().ref_load_repersist(str(src).encode(), str(dst).encode())
    _check(n)
    return int(n)


def ref_cosine(a, b):
    return ref().ref_cosine(_c(a, np.float64), _c(b, np.float64), len(a))


def ref_kmeans(points, k, seed, max_iters=64):
    pts = _c(points, np.float64)
    n, dim = pts.shape
    assign = np.zeros(n, np.int64)
    cent = np.zeros((k, dim), np.float64)
    iters = np.zeros(1, np.int64)
    sse = np.zeros(max(max_iters, 1), np.float64)
    _check(ref().ref_kmeans(pts, n, dim, k, seed, max_iters, assign, cent.reshape(-1), iters, sse))
    return assign, cent, int(iters[0]), sse[: int(iters[0])]


def ref_allocate(sens, per_head_budget, alpha):
    sens = _c(sens, np.float64)
    b = np.zeros(sens.size, np.int64)
    w = np.zeros(sens.size, np.float64)
    _check(ref().ref_allocate(sens, sens.size, int(per_head_budget), float(alpha), b, w))
    return b, w


def ref_measure_sensitivity(layers, hq, hkv, d, model_seed, ntok, tok_seed, budget, sink):
    sigma = np.zeros(layers, np.float64)
    skipped = np.zeros(1, np.int64)
    kf = np.zeros((layers, hkv, ntok, d), np.float64)
    kb = np.zeros_like(kf)
    _check(ref().ref_measure_sensitivity(layers, hq, hkv, d, model_seed, ntok, tok_seed, budget, sink,
                                         sigma, skipped, kf.reshape(-1), kb.reshape(-1)))
    return sigma, int(skipped[0]), kf, kb


def ref_block_prefill(layers, hq, hkv, d, model_seed, ntok, tok_seed, budget, block, prompt,
                      layer_budgets=None):
    nblocks_max = (ntok + block - 1) // block
    series = np.zeros(2 * nblocks_max + 2, np.int64)
    ns = np.zeros(1, np.int64)
    ev = np.zeros(nblocks_max + 1, np.int64)
    nb = np.zeros(1, np.int64)
    retained = np.zeros(layers * hkv * (ntok + 1), np.int64)
    counts = np.zeros(layers * hkv, np.int64)
    prompt = _c(prompt, np.int64)
    lb = None if layer_budgets is None else _c(layer_budgets, np.int64)
    _check(ref().ref_block_prefill(layers, hq, hkv, d, model_seed, ntok, tok_seed, budget, block, prompt,
                                   prompt.size, _ptr(lb), series, ns, ev, nb, retained, counts))
    return (series[: int(ns[0])], ev[: int(nb[0])], int(nb[0]),
            counts.reshape(layers, hkv), retained[: int(counts.sum())])
