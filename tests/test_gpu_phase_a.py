"""Phase A and Phase B end to end on the GPU (episodic.hpp:108-253, the cfg3
flow at toy size): k-means over segment embeddings -> per-layer budgets from
the key-cosine sensitivity -> one block prefill per episode with its own
prompt and the allocated budgets -> caches persisted to a CacheStore with a
manifest -> queries routed to the nearest centroid, loading a cache only on a
switch.  Every stage is checked against the oracle restatement of the same
stage where one exists (k-means and sensitivity bit-exact, allocation exact);
the per-episode caches must realise the allocated budgets, and block
prefill's chained parity and the store's byte-identity are covered by
test_gpu_blockprefill.py / test_gpu_store.py."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_phase_a_and_b(gpu, orc, tmp_path):
    from tests.test_gpu_blockprefill import SynthProvider
    rng = np.random.default_rng(3)
    E, L, Hq, H, d, n, B, M = 3, 2, 4, 2, 16, 64, 16, 8
    # A1: episodes from segment embeddings
    emb = rng.standard_normal((40, 32))
    km = gpu.kmeans(emb, E, seed=7)
    a, c, it, sse = orc.kmeans(emb, E, 7)
    assert list(km.assignments) == list(a) and np.array_equal(km.centroids, c)
    # A2: layer budgets from the key-cosine sensitivity
    kf = torch.randn(L, H, 48, d, device="cuda", dtype=torch.float64)
    kb = kf + 0.3 * torch.randn_like(kf) * torch.arange(1, L + 1, device="cuda").view(L, 1, 1, 1)
    prof = gpu.sensitivity_from_keys(kf, kb)
    sigma, _ = orc.sensitivity(kf.cpu().numpy(), kb.cpu().numpy())
    assert np.array_equal(np.asarray(prof.sigma), sigma)  # bit-exact
    alloc = gpu.allocate(prof, M, 1.1)
    b_ref, _ = orc.allocate(np.asarray(prof.sensitivity), M, 1.1)
    assert list(alloc.layer_budgets) == list(b_ref) and sum(alloc.layer_budgets) == L * M
    # A3: one block prefill per episode (fp32 parity path), persisted
    store = gpu.CacheStore(tmp_path / "store")
    kept = []
    for e in range(E):
        prov = SynthProvider(L, Hq, H, d, n, 3, seed=100 + e, dtype=torch.float32)
        cfg = gpu.BlockPrefillConfig(M, B, layer_budgets=list(alloc.layer_budgets), mode="exact_f32")
        rep = gpu.block_prefill(prov, L, Hq, H, d, n, cfg, episode_id=e, dtype=torch.float32)
        assert rep.cache.entries_per_layer() == [min(H * b, H * n) for b in alloc.layer_budgets]
        store.save(rep.cache, e, scorer="patched", budget_per_head=M, layer_budgets=list(alloc.layer_budgets))
        kept.append(rep.cache.retained_positions())
    man = gpu.manifest_json(km.centroids, [(0, 1)] * E, [f"episode {e}" for e in range(E)], store, "patched", M,
                            alloc.layer_budgets, emb.shape[1])
    store.write_manifest(man)
    # Phase B: route and load on switch
    state = gpu.SessionState()
    for q, want in [(km.centroids[2], 2), (km.centroids[2] * 3, 2), (km.centroids[0], 0)]:
        assert gpu.route(store, km.centroids, q, state, dtype=torch.float32) == want
    assert state.switch_count == 2
    assert state.resident.retained_positions() == kept[0]
