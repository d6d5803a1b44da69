"""Episode clustering: kmeans (clustering.hpp:148-260) on the GPU.

`kmeans` is the drop-in: same arguments, same result bits (fp64, sequential
distance order, ties to the lower cluster, index-ordered centroid sums, the
reference's mt19937_64 stream for k-means++ seeding and farthest-point repair).

`kmeans_sharded` runs the same algorithm with the points sharded across ranks
of a torch.distributed group (one process per GPU).  Each Lloyd iteration
hands the running centroid sums down an ordered rank chain
(rank r adds its contiguous shard in index order on top of rank r-1's sums),
then broadcasts, so every rank reproduces the single-GPU bits exactly
(SURVEY.md section 8e).  With backend "nccl" the chain runs over NVLink.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .context import Context, default_context, ptr
from .errors import Error


@dataclass
class KMeansResult:
    """KMeansResult (clustering.hpp:124-129)."""
    assignments: list
    centroids: np.ndarray
    iterations: int
    sse_per_iteration: list


def kmeans(points, k: int, seed: int, max_iters: int = 64, ctx: Context | None = None) -> KMeansResult:
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim != 2:
        raise Error("kmeans: points must be a 2-D array")
    n, dim = pts.shape
    if k < 1:
        raise Error("kmeans: cluster count must be >= 1")
    if n < k:
        raise Error(f"kmeans: fewer points ({n}) than clusters ({k})")
    d_pts = torch.as_tensor(pts, device=torch.device("cuda", ctx.device))
    assign = np.zeros(n, np.int64)
    cent = np.zeros((k, dim), np.float64)
    iters = np.zeros(1, np.int64)
    sse = np.zeros(max(max_iters, 1), np.float64)
    _lib.call("epk_kmeans", ctx.handle, ptr(d_pts), n, dim, k, C.c_uint64(seed), max_iters,
              assign.ctypes.data_as(C.c_void_p), cent.ctypes.data_as(C.c_void_p),
              iters.ctypes.data_as(C.c_void_p), sse.ctypes.data_as(C.c_void_p))
    it = int(iters[0])
    return KMeansResult(assign.tolist(), cent, it, sse[:it].tolist())


def kmeans_multi_device(points, k: int, seed: int, max_iters: int = 64, contexts=None) -> KMeansResult:
    """kmeans with the points split in index order over `contexts` (one per
    GPU of this process; a device may repeat): epk_kmeans_sharded, the ordered
    chain over NCCL between distinct devices.  Bit-identical to `kmeans`."""
    contexts = contexts or [default_context()]
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim != 2:
        raise Error("kmeans: points must be a 2-D array")
    n, dim = pts.shape
    S = len(contexts)
    bounds = [n * s // S for s in range(S + 1)]
    shards = [torch.as_tensor(pts[bounds[s]:bounds[s + 1]], device=torch.device("cuda", c.device))
              for s, c in enumerate(contexts)]
    ctxs = (C.c_void_p * S)(*[c.handle.value for c in contexts])
    ptrs = (C.c_void_p * S)(*[s.data_ptr() if s.numel() else 0 for s in shards])
    ns = (C.c_int64 * S)(*[bounds[s + 1] - bounds[s] for s in range(S)])
    assign = np.zeros(n, np.int64)
    cent = np.zeros((k, dim), np.float64)
    iters = np.zeros(1, np.int64)
    sse = np.zeros(max(max_iters, 1), np.float64)
    _lib.call("epk_kmeans_sharded", C.cast(ctxs, C.c_void_p), S, C.cast(ptrs, C.c_void_p), C.cast(ns, C.c_void_p),
              dim, k, C.c_uint64(seed), max_iters, assign.ctypes.data_as(C.c_void_p),
              cent.ctypes.data_as(C.c_void_p), iters.ctypes.data_as(C.c_void_p), sse.ctypes.data_as(C.c_void_p))
    it = int(iters[0])
    return KMeansResult(assign.tolist(), cent, it, sse[:it].tolist())


# ---------------------------------------------------------------------------
# Sharded k-means (points split across ranks)
# ---------------------------------------------------------------------------

class _DeviceShardOps:
    """The per-shard device work of one Lloyd iteration (K4 kernels)."""

    def __init__(self, shard: torch.Tensor, ctx: Context):
        self.x = shard.contiguous()
        self.ctx = ctx

    def sq_dist_to(self, c: torch.Tensor) -> torch.Tensor:
        n, dim = self.x.shape
        a = torch.empty(n, dtype=torch.int64, device=self.x.device)
        d = torch.empty(n, dtype=torch.float64, device=self.x.device)
        _lib.call("epk_kmeans_assign", self.ctx.handle, ptr(self.x), n, dim, ptr(c.contiguous()), 1, ptr(a), ptr(d))
        return d

    def assign(self, cent: torch.Tensor) -> torch.Tensor:
        n, dim = self.x.shape
        a = torch.empty(n, dtype=torch.int64, device=self.x.device)
        _lib.call("epk_kmeans_assign", self.ctx.handle, ptr(self.x), n, dim, ptr(cent), cent.shape[0], ptr(a), None)
        return a

    def sq_dist_assigned(self, cent: torch.Tensor, assign: torch.Tensor) -> torch.Tensor:
        n, dim = self.x.shape
        d = torch.empty(n, dtype=torch.float64, device=self.x.device)
        _lib.call("epk_kmeans_sq_dist", self.ctx.handle, ptr(self.x), n, dim, ptr(cent), ptr(assign), ptr(d))
        return d

    def chain_sums(self, assign: torch.Tensor, k: int, sums: torch.Tensor, counts: torch.Tensor, accumulate: bool):
        n, dim = self.x.shape
        _lib.call("epk_kmeans_partial_sums", self.ctx.handle, ptr(self.x), n, dim, ptr(assign), k, ptr(sums),
                  ptr(counts), int(accumulate))

    def finalize(self, sums: torch.Tensor, counts: torch.Tensor, k: int, dim: int) -> torch.Tensor:
        cent = torch.empty(k, dim, dtype=torch.float64, device=sums.device)
        _lib.call("epk_kmeans_finalize", self.ctx.handle, ptr(sums), ptr(counts), k, dim, ptr(cent))
        return cent


class _HostRng:
    """epikv::Rng (numerics.hpp:146-183): mt19937_64, 53-bit uniform, 128-bit index."""

    def __init__(self, seed: int):
        self._mt = _MT19937_64(seed)

    def uniform(self) -> float:
        return float(self._mt.next() >> 11) * 2.0 ** -53

    def uniform_index(self, n: int) -> int:
        return (self._mt.next() * n) >> 64


class _MT19937_64:
    """std::mt19937_64 (the reference's generator), pure integer arithmetic."""
    _N, _M = 312, 156
    _MATRIX_A = 0xB5026F5AA96619E9
    _UM, _LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
    _MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        self.mt = [0] * self._N
        self.mt[0] = seed & self._MASK
        for i in range(1, self._N):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self._MASK
        self.idx = self._N

    def next(self) -> int:
        if self.idx >= self._N:
            mt, N, M = self.mt, self._N, self._M
            for i in range(N):
                x = (mt[i] & self._UM) | (mt[(i + 1) % N] & self._LM)
                xa = x >> 1
                if x & 1:
                    xa ^= self._MATRIX_A
                mt[i] = mt[(i + M) % N] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self._MASK


def kmeans_sharded(shard: torch.Tensor, shard_start: int, n_total: int, k: int, seed: int, max_iters: int = 64,
                   group=None, ops=None) -> KMeansResult:
    """kmeans with points sharded over the ranks of `group` (contiguous, in
    rank order).  Returns the same KMeansResult on every rank, bit-identical to
    `kmeans` on the concatenated points.  `ops` overrides the per-shard device
    work (tests substitute a CPU implementation to exercise the rank chain
    with the gloo backend)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n, dim = shard.shape
    if k < 1:
        raise Error("kmeans: cluster count must be >= 1")
    if n_total < k:
        raise Error(f"kmeans: fewer points ({n_total}) than clusters ({k})")
    if ops is None:
        ops = _DeviceShardOps(shard, default_context(shard.device.index))
    dev = shard.device
    sizes = torch.zeros(world, dtype=torch.int64, device=dev)
    sizes[rank] = n
    dist.all_reduce(sizes, group=group)
    starts = [0]
    for s in sizes.tolist()[:-1]:
        starts.append(starts[-1] + s)
    if starts[rank] != shard_start or int(sizes.sum()) != n_total:
        raise Error("kmeans_sharded: shards must be contiguous and in rank order")

    def owner(i: int) -> int:
        r = 0
        while r + 1 < world and starts[r + 1] <= i:
            r += 1
        return r

    def fetch_point(i: int) -> torch.Tensor:
        buf = torch.empty(dim, dtype=torch.float64, device=dev)
        r = owner(i)
        if r == rank:
            buf.copy_(shard[i - starts[r]])
        dist.broadcast(buf, src=dist.get_global_rank(group, r) if group is not None else r, group=group)
        return buf

    def gather_all(local: torch.Tensor) -> torch.Tensor:
        parts = [torch.empty(int(s), dtype=local.dtype, device=dev) for s in sizes.tolist()]
        dist.all_gather(parts, local.contiguous(), group=group) if _uniform(sizes) else _gather_ragged(parts, local)
        return torch.cat(parts)

    def _uniform(sz):
        return bool((sz == sz[0]).all())

    def _gather_ragged(parts, local):
        for r, part in enumerate(parts):
            if r == rank:
                part.copy_(local)
            dist.broadcast(part, src=dist.get_global_rank(group, r) if group is not None else r, group=group)

    rng = _HostRng(seed)
    cent = [fetch_point(rng.uniform_index(n_total))]
    best = np.full(n_total, np.inf)
    while len(cent) < k:
        d = gather_all(ops.sq_dist_to(cent[-1].reshape(1, dim))).cpu().numpy()
        best = np.minimum(best, d)
        total = 0.0
        for v in best:
            total += float(v)
        if total > 0.0:
            target = rng.uniform() * total
            acc, chosen = 0.0, n_total - 1
            for i in range(n_total):
                acc += float(best[i])
                if acc > target:
                    chosen = i
                    break
        else:
            chosen = rng.uniform_index(n_total)
        cent.append(fetch_point(chosen))
    centroids = torch.stack(cent)
    assign_all = np.zeros(n_total, np.int64)
    sse_hist = []
    iters = 0
    for it in range(max_iters):
        a_local = ops.assign(centroids)
        a_all = gather_all(a_local).cpu().numpy()
        changed = bool(np.any(a_all != assign_all))
        counts = np.bincount(a_all, minlength=k)
        for c in range(k):
            if counts[c] > 0:
                continue
            a_dev = torch.as_tensor(a_all[starts[rank]:starts[rank] + n], device=dev)
            d = gather_all(ops.sq_dist_assigned(centroids, a_dev)).cpu().numpy()
            victim, worst = 0, -1.0
            for i in range(n_total):
                if counts[a_all[i]] <= 1:
                    continue
                if d[i] > worst:
                    worst, victim = float(d[i]), i
            counts[a_all[victim]] -= 1
            a_all[victim] = c
            counts[c] += 1
            changed = True
        a_dev = torch.as_tensor(a_all[starts[rank]:starts[rank] + n], device=dev)
        # ordered rank chain: rank r continues rank r-1's running sums
        sums = torch.zeros(k, dim, dtype=torch.float64, device=dev)
        cnts = torch.zeros(k, dtype=torch.int64, device=dev)
        if rank > 0:
            src = dist.get_global_rank(group, rank - 1) if group is not None else rank - 1
            dist.recv(sums, src=src, group=group)
            dist.recv(cnts, src=src, group=group)
        ops.chain_sums(a_dev, k, sums, cnts, accumulate=rank > 0)
        if rank < world - 1:
            dst = dist.get_global_rank(group, rank + 1) if group is not None else rank + 1
            dist.send(sums, dst=dst, group=group)
            dist.send(cnts, dst=dst, group=group)
        last = dist.get_global_rank(group, world - 1) if group is not None else world - 1
        dist.broadcast(sums, src=last, group=group)
        dist.broadcast(cnts, src=last, group=group)
        centroids = ops.finalize(sums, cnts, k, dim)
        iters = it + 1
        d = gather_all(ops.sq_dist_assigned(centroids, a_dev)).cpu().numpy()
        sse = 0.0
        for v in d:
            sse += float(v)
        sse_hist.append(sse)
        assign_all = a_all
        if not changed:
            break
    return KMeansResult(assign_all.tolist(), centroids.cpu().numpy(), iters, sse_hist)
