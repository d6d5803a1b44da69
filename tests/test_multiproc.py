"""Multi-process host logic with the gloo backend, world_size 2, on CPU:

* kmeans_sharded: the ordered rank chain (rank r continues rank r-1's
  centroid sums) reproduces the single-process kmeans bits exactly
  (clustering.hpp:234-246 sums in point-index order).  The per-shard device
  work is substituted by a sequential CPU implementation here; on GPUs it is
  the K4 kernels.
* build_episodes: round-robin episode ownership, summaries gathered in
  episode order on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class CpuShardOps:
    """Sequential-order CPU twin of clustering._DeviceShardOps (test only)."""

    def __init__(self, shard):
        self.x = shard.double().numpy()

    @staticmethod
    def _sq(a, b):
        acc = 0.0
        for u, v in zip(a.tolist(), b.tolist()):
            d = u - v
            acc += d * d
        return acc

    def sq_dist_to(self, c):
        c = c.numpy().reshape(-1)
        return torch.tensor([self._sq(p, c) for p in self.x], dtype=torch.float64)

    def assign(self, cent):
        cent = cent.numpy()
        out = []
        for p in self.x:
            best, bd = 0, self._sq(p, cent[0])
            for c in range(1, cent.shape[0]):
                d = self._sq(p, cent[c])
                if d < bd:
                    best, bd = c, d
            out.append(best)
        return torch.tensor(out, dtype=torch.int64)

    def sq_dist_assigned(self, cent, assign):
        cent = cent.numpy()
        return torch.tensor([self._sq(p, cent[a]) for p, a in zip(self.x, assign.tolist())], dtype=torch.float64)

    def chain_sums(self, assign, k, sums, counts, accumulate):
        s = sums.numpy().copy() if accumulate else np.zeros_like(sums.numpy())
        n = counts.numpy().copy() if accumulate else np.zeros_like(counts.numpy())
        for p, a in zip(self.x, assign.tolist()):
            for d in range(self.x.shape[1]):
                s[a, d] = s[a, d] + p[d]
            n[a] += 1
        sums.copy_(torch.from_numpy(s))
        counts.copy_(torch.from_numpy(n))

    def finalize(self, sums, counts, k, dim):
        return sums / counts.double().reshape(-1, 1)


def _kmeans_worker(rank, world, port, pts, k, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_17396_b200.clustering import kmeans_sharded
        n = pts.shape[0]
        bounds = [0, 23, n] if world == 2 else [0, n]  # uneven shards
        lo, hi = bounds[rank], bounds[rank + 1]
        shard = torch.from_numpy(pts[lo:hi])
        r = kmeans_sharded(shard, lo, n, k, seed, ops=CpuShardOps(shard))
        out[rank] = (r.assignments, r.centroids.tolist(), r.iterations, r.sse_per_iteration)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k,seed", [(3, 7), (5, 11)])
def test_kmeans_sharded_chain_bitexact_gloo(orc, k, seed):
    rng = np.random.default_rng(seed)
    pts = rng.standard_normal((60, 4))
    pts[10:14] = pts[3]  # duplicates: exercise ties and possible repairs
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_kmeans_worker, args=(2, _free_port(), pts, k, seed, out), nprocs=2, join=True)
    a, c, it, sse = orc.kmeans(pts, k, seed)
    for rank in range(2):
        ra, rc, rit, rsse = out[rank]
        assert ra == a.tolist()
        assert np.array_equal(np.array(rc), c)
        assert rit == it and np.array_equal(np.array(rsse), sse)


class _FakeReport:
    def __init__(self, e):
        self.blocks_processed = e + 1

        class _C:
            @staticmethod
            def entries_per_layer():
                return [e, 2 * e]
        self.cache = _C()
        self.evictions_per_block = [e] * (e + 1)


def _episodes_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_17396_b200.episodic import build_episodes
        ran = []

        def run(e):
            ran.append(e)
            return _FakeReport(e)

        res = build_episodes(run, 5)
        out[rank] = (ran, [(s.episode_id, s.rank, s.blocks_processed, s.entries_per_layer) for s in res])
    finally:
        dist.destroy_process_group()


def test_build_episodes_round_robin_gloo():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_episodes_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0][0] == [0, 2, 4] and out[1][0] == [1, 3]
    expect = [(e, e % 2, e + 1, [e, 2 * e]) for e in range(5)]
    assert out[0][1] == expect and out[1][1] == expect


def test_assign_episodes():
    from paper_2509_17396_b200.episodic import assign_episodes
    assert assign_episodes(8, 8) == [[i] for i in range(8)]
    assert assign_episodes(4, 2) == [[0, 2], [1, 3]]
    assert assign_episodes(3, 4) == [[0], [1], [2], []]
