"""K4 (k-means) bit-exact vs the reference fixtures/oracle; K5 (sensitivity)
vs the reference's measure_sensitivity; allocate vs the reference."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")


def test_kmeans_golden_bitwise(gpu):
    g = np.load(GOLDEN)
    for i in range(int(g["km_count"])):
        r = gpu.kmeans(g[f"km{i}_pts"], int(g[f"km{i}_k"]), int(g[f"km{i}_seed"]))
        assert r.assignments == g[f"km{i}_assign"].tolist()
        assert np.array_equal(r.centroids, g[f"km{i}_cent"])
        assert r.iterations == int(g[f"km{i}_iters"])
        assert np.array_equal(np.array(r.sse_per_iteration), g[f"km{i}_sse"])


@pytest.mark.parametrize("n,dim,k,seed", [(2048, 256, 4, 1), (2048, 1024, 8, 2), (300, 3, 7, 9)])
def test_kmeans_vs_oracle(gpu, orc, n, dim, k, seed):
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((k, dim)) * 3
    pts = centers[rng.integers(0, k, n)] + rng.standard_normal((n, dim))
    r = gpu.kmeans(pts, k, seed)
    a, c, it, sse = orc.kmeans(pts, k, seed)
    assert r.assignments == a.tolist() and np.array_equal(r.centroids, c) and r.iterations == it
    assert np.array_equal(np.array(r.sse_per_iteration), sse)


def test_kmeans_repair_and_edges(gpu, orc):
    pts = np.repeat(np.random.default_rng(0).standard_normal((3, 4)), 5, axis=0)
    pts = np.concatenate([pts, pts[:1]])
    r = gpu.kmeans(pts, 6, 3)
    a, c, it, sse = orc.kmeans(pts, 6, 3)
    assert r.assignments == a.tolist() and np.array_equal(r.centroids, c)
    with pytest.raises(gpu.Error, match="fewer points"):
        gpu.kmeans(pts[:2], 3, 1)
    with pytest.raises(gpu.Error, match="cluster count"):
        gpu.kmeans(pts, 0, 1)
    one = gpu.kmeans(pts, 1, 4)  # E = 1: the plain mean
    assert np.allclose(one.centroids[0], pts.mean(0))


def test_sensitivity_golden(gpu):
    g = np.load(GOLDEN)
    kf = torch.as_tensor(g["sens_kf"], device="cuda")
    kb = torch.as_tensor(g["sens_kb"], device="cuda")
    prof = gpu.sensitivity_from_keys(kf, kb)
    assert np.array_equal(np.asarray(prof.sigma), g["sens_sigma"])  # bit-exact
    assert prof.skipped_zero_norm == int(g["sens_skipped"])


def test_sensitivity_bf16_large_vs_oracle(gpu, orc):
    torch.manual_seed(0)
    L, H, N, d = 4, 8, 4096, 128
    kf = torch.randn(L, H, N, d, device="cuda").bfloat16()
    kb = (kf.float() + 0.3 * torch.randn_like(kf.float())).bfloat16()
    kb[1, 2, 5] = 0  # a zero-norm pair is skipped
    prof = gpu.sensitivity_from_keys(kf, kb)
    sig, sk = orc.sensitivity(kf.double().cpu().numpy(), kb.double().cpu().numpy())
    assert np.array_equal(np.asarray(prof.sigma), sig) and prof.skipped_zero_norm == sk == 1  # bit-exact


def test_allocate_golden(gpu):
    g = np.load(GOLDEN)
    for i in range(int(g["al_count"])):
        prof = gpu.SensitivityProfile(sigma=[1 - s for s in g[f"al{i}_s"]], sensitivity=g[f"al{i}_s"].tolist())
        a = gpu.allocate(prof, int(g[f"al{i}_M"]), float(g[f"al{i}_alpha"]))
        assert a.layer_budgets == g[f"al{i}_b"].tolist()
        assert a.weights == g[f"al{i}_w"].tolist()
        assert a.total() == len(a.layer_budgets) * int(g[f"al{i}_M"])


def test_kmeans_sharded_device_ops_nccl_world1(gpu, orc):
    """kmeans_sharded through the K4 device ops under a 1-rank NCCL group
    equals the single-GPU kmeans (the N>1 chain is covered with gloo)."""
    import os
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(4)
        pts = rng.standard_normal((500, 64))
        r = gpu.kmeans_sharded(torch.as_tensor(pts, device="cuda"), 0, 500, 6, 9)
        a, c, it, sse = orc.kmeans(pts, 6, 9)
        assert r.assignments == a.tolist() and np.array_equal(r.centroids, c) and r.iterations == it
        assert np.array_equal(np.array(r.sse_per_iteration), sse)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype,L,H,N,d", [(torch.bfloat16, 3, 2, 1000, 128), (torch.float32, 2, 3, 333, 128),
                                           (torch.float64, 2, 1, 77, 128), (torch.float32, 2, 2, 150, 7),
                                           (torch.bfloat16, 1, 1, 2, 8)])
def test_sensitivity_ragged_tiles_and_skips(gpu, orc, dtype, L, H, N, d):
    """The pair tiles (128 / 64 / 32 pairs by dtype, chunk-major over layers)
    and the chain's 1,024-cosine ring slots with partial last tiles, rows not
    16-byte multiples (the direct-read pair kernel), zero-norm pairs skipped
    across tile and slot boundaries: bit-exact vs the oracle."""
    torch.manual_seed(L * 100 + N)
    kf = torch.randn(L, H, N, d, dtype=torch.float64, device="cuda").to(dtype)
    kb = (kf.double() + 0.5 * torch.randn_like(kf.double())).to(dtype)
    kb.view(L, -1, d)[:, ::97] = 0
    kf.view(L, -1, d)[-1, -1] = 0
    prof = gpu.sensitivity_from_keys(kf, kb)
    sig, sk = orc.sensitivity(kf.double().cpu().numpy(), kb.double().cpu().numpy())
    assert np.array_equal(np.asarray(prof.sigma), sig) and prof.skipped_zero_norm == sk


@pytest.mark.parametrize("shards", [1, 2, 3, 5])
def test_kmeans_multi_device_chain(gpu, orc, shards):
    """epk_kmeans_sharded: the ordered chain over `shards` contexts (one GPU,
    device copies between shards) equals kmeans / the oracle bit for bit,
    including an empty shard and the empty-cluster repair."""
    from paper_2509_17396_b200.context import Context
    rng = np.random.default_rng(shards)
    pts = rng.standard_normal((700, 48)) + rng.integers(0, 4, (700, 1))
    ctxs = [Context(0) for _ in range(shards)]
    for k, p in ((5, pts), (6, np.repeat(pts[:4], 3, axis=0))):
        r = gpu.kmeans_multi_device(p, k, 11, contexts=ctxs)
        a, c, it, sse = orc.kmeans(p, k, 11)
        assert r.assignments == a.tolist() and np.array_equal(r.centroids, c) and r.iterations == it
        assert np.array_equal(np.array(r.sse_per_iteration), sse)
    r = gpu.kmeans_multi_device(pts[:3], 3, 2, contexts=ctxs)  # fewer points than shards: empty shards
    a, c, it, sse = orc.kmeans(pts[:3], 3, 2)
    assert r.assignments == a.tolist() and np.array_equal(r.centroids, c)
    for c_ in ctxs:
        c_.close()
