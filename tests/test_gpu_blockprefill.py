"""The block-prefill engine on the GPU vs the reference's block-loop tests
(test_blockprefill.cpp, acceptance C1/C2) and vs the oracle chained step by
step (fp32 parity path: every block's retained sets bit-exact)."""
import os

import numpy as np
import pytest
import torch

from tests.helpers import random_layer

pytestmark = pytest.mark.gpu


class SynthProvider:
    """Seeded synthetic K/V per token and a fixed patched prompt per episode."""

    def __init__(self, L, Hq, H, d, n, p, seed=0, dtype=torch.float32):
        g = torch.Generator().manual_seed(seed)
        self.k = torch.randn(L, H, n, d, generator=g).to(dtype)
        self.v = torch.randn(L, H, n, d, generator=g).to(dtype)
        self.q = torch.randn(L, Hq, p, d, generator=g).to(dtype)
        self.kp = torch.randn(L, H, p, d, generator=g).to(dtype)
        self.calls = []

    def block_kv(self, start, length):
        sl = slice(start, start + length)
        return (self.k[:, :, sl].cuda(), self.v[:, :, sl].cuda(),
                torch.arange(start, start + length, dtype=torch.int32).cuda())

    def prompt(self, episode_id, block_index):
        self.calls.append((episode_id, block_index))
        return self.q.cuda(), self.kp.cuda()


def test_three_token_blocks_trace_c2(gpu):
    """9 tokens, blocks of 3, budget 1 -> occupancy 3,1,4,1,4,1."""
    prov = SynthProvider(1, 1, 1, 8, 9, 3)
    cfg = gpu.BlockPrefillConfig(budget_per_head=1, block_size=3, mode="exact_f32")
    rep = gpu.block_prefill(prov, 1, 1, 1, 8, 9, cfg, dtype=torch.float32)
    assert rep.append_evict_series(0) == [3, 1, 4, 1, 4, 1]
    assert rep.blocks_processed == 3


def test_golden_traces(gpu):
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz"))
    prov = SynthProvider(2, 4, 2, 8, 120, 3)
    cfg = gpu.BlockPrefillConfig(budget_per_head=8, block_size=16, mode="exact_f32")
    rep = gpu.block_prefill(prov, 2, 4, 2, 8, 120, cfg, dtype=torch.float32)
    assert rep.append_evict_series(0) == g["bp_120_series"].tolist()
    assert rep.evictions_per_block == g["bp_120_evictions"].tolist()
    prov = SynthProvider(2, 2, 1, 8, 64, 3)
    cfg = gpu.BlockPrefillConfig(budget_per_head=8, block_size=16, layer_budgets=[4, 12], mode="exact_f32")
    rep = gpu.block_prefill(prov, 2, 2, 1, 8, 64, cfg, dtype=torch.float32)
    assert rep.cache.entries_per_layer() == g["bp_alloc_counts"].tolist()


def test_under_budget_keeps_whole_context_and_ceiling(gpu):
    prov = SynthProvider(1, 1, 1, 8, 12, 2)
    rep = gpu.block_prefill(prov, 1, 1, 1, 8, 12, gpu.BlockPrefillConfig(16, 4, mode="exact_f32"), dtype=torch.float32)
    assert rep.total_evictions() == 0
    assert rep.cache.retained_positions()[0][0] == list(range(12))
    for n in (1, 15, 16, 17, 33):
        prov = SynthProvider(1, 1, 1, 8, n, 2)
        rep = gpu.block_prefill(prov, 1, 1, 1, 8, n, gpu.BlockPrefillConfig(4, 16, mode="exact_f32"),
                                dtype=torch.float32)
        assert rep.blocks_processed == (n + 15) // 16


def test_bounded_occupancy_and_prompt_positions(gpu):
    for scorer in ("patched", "streaming"):
        prov = SynthProvider(2, 4, 2, 16, 120, 5)
        cfg = gpu.BlockPrefillConfig(8, 16, scorer=scorer, streaming_sink=4, mode="exact_f32")
        rep = gpu.block_prefill(prov, 2, 4, 2, 16, 120, cfg, dtype=torch.float32)
        limit = 2 * (8 + 16)
        for s in rep.occupancy:
            assert all(e <= limit for e in s.entries_per_layer)
        assert all(e <= 2 * 8 for e in rep.cache.entries_per_layer())
        for heads in rep.cache.retained_positions():
            for ps in heads:
                assert all(p < 120 for p in ps)
        if scorer == "streaming":
            # sink + most recent positions (streaming_retention, scoring.hpp:132-148)
            for heads in rep.cache.retained_positions():
                allp = sorted(set(p for ps in heads for p in ps))
                assert set(range(4)) <= set(allp)


def test_error_paths(gpu):
    prov = SynthProvider(2, 2, 1, 8, 8, 2)
    with pytest.raises(gpu.Error, match="empty context"):
        gpu.block_prefill(prov, 2, 2, 1, 8, 0, gpu.BlockPrefillConfig(4, 4), dtype=torch.float32)
    with pytest.raises(gpu.Error, match="allocation layer count"):
        gpu.block_prefill(prov, 2, 2, 1, 8, 8, gpu.BlockPrefillConfig(4, 4, layer_budgets=[4, 4, 4]),
                          dtype=torch.float32)
    with pytest.raises(gpu.Error, match="sink exceeds budget"):
        gpu.block_prefill(prov, 2, 2, 1, 8, 8, gpu.BlockPrefillConfig(4, 4, scorer="streaming", streaming_sink=5),
                          dtype=torch.float32)


def test_chained_episode_bitexact_vs_oracle(gpu, orc):
    """Every block step of a 2-layer episode equals the oracle's chain (fp32
    scores -> evict_to_budget) -- retained positions and K rows."""
    L, Hq, H, d, n, p, M, B = 2, 6, 2, 32, 160, 8, 20, 24
    prov = SynthProvider(L, Hq, H, d, n, p, seed=3)
    cfg = gpu.BlockPrefillConfig(M, B, mode="exact_f32")
    rep = gpu.block_prefill(prov, L, Hq, H, d, n, cfg, dtype=torch.float32)
    # oracle chain
    for l in range(L):
        heads = [np.zeros(0, np.int64) for _ in range(H)]
        for start in range(0, n, B):
            length = min(B, n - start)
            heads = [np.concatenate([hp, np.arange(start, start + length)]) for hp in heads]
            ho = np.concatenate([[0], np.cumsum([len(hp) for hp in heads])])
            pos = np.concatenate(heads)
            k = np.concatenate([prov.k[l, h, heads[h]].numpy() for h in range(H)])
            s = orc.score_layer_f32(prov.q[l].numpy(), k, prov.kp[l].numpy(), ho, True)
            _, keep = orc.evict_layer(ho, pos, s.astype(np.float64), M)
            heads = [heads[h][keep[ho[h]:ho[h + 1]]] for h in range(H)]
        assert rep.cache.retained_positions()[l] == [hp.tolist() for hp in heads]
