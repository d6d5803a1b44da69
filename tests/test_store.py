"""The .epkv reader and Phase B routing helpers on the host (no GPU): files
written by the reference's own persist (kvcache.hpp:281) parse back to the
same data; truncation / bad magic / version mismatch fail closed like
load_cache (kvcache.hpp:321-372); centroid_similarity matches the reference's
cosine.  The GPU writer is checked byte for byte in test_gpu_store.py."""
import os

import numpy as np
import pytest

from paper_2509_17396_b200 import store
from paper_2509_17396_b200.errors import IoError


def _layers(rng, L, H, d, counts):
    out = []
    for l in range(L):
        c = np.asarray(counts[l], np.int64)
        n = int(c.sum())
        pos = np.concatenate([np.sort(rng.choice(1000, int(x), replace=False)) for x in c]).astype(np.int64)
        out.append((c, pos, rng.standard_normal((n, d)), rng.standard_normal((n, d))))
    return out


def test_parse_reference_files(ref, tmp_path):
    rng = np.random.default_rng(3)
    for i, (L, H, d, counts) in enumerate([(2, 3, 4, [[3, 0, 2], [1, 1, 1]]), (1, 1, 128, [[40]]),
                                           (3, 2, 16, [[0, 0], [5, 7], [2, 0]])]):
        pl = _layers(rng, L, H, d, counts)
        path = tmp_path / f"r{i}.epkv"
        n = ref.ref_persist(path, pl, episode_id=7 + i, scorer="patched", budget_per_head=9,
                            layer_budgets=[4] * L, layer_budget_fields=[4 + l for l in range(L)])
        assert n == os.path.getsize(path)
        meta, per = store.parse(path.read_bytes(), path)
        assert (meta.episode_id, meta.scorer, meta.budget_per_head) == (7 + i, "patched", 9)
        assert meta.layer_budgets == [4] * L and meta.layer_budget_fields == [4 + l for l in range(L)]
        for (c, p, k, v), (c2, p2, k2, v2) in zip(pl, per):
            assert np.array_equal(c, c2) and np.array_equal(p, p2)
            if len(p):
                assert np.array_equal(k, k2) and np.array_equal(v, v2)


def test_parse_fails_closed(ref, tmp_path):
    rng = np.random.default_rng(4)
    path = tmp_path / "a.epkv"
    ref.ref_persist(path, _layers(rng, 1, 2, 8, [[3, 4]]), budget_per_head=4)
    b = path.read_bytes()
    for cut in (3, 10, 40, len(b) - 1):
        with pytest.raises(IoError, match="truncated|bad magic"):
            store.parse(b[:cut])
    with pytest.raises(IoError, match="bad magic"):
        store.parse(b"EPKX" + b[4:])
    with pytest.raises(IoError, match="version mismatch"):
        store.parse(b[:4] + (2).to_bytes(2, "little") + b[6:])


def test_golden_epkv_fixture():
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz"))
    meta, per = store.parse(g["epkv_bytes"].tobytes())
    assert meta.episode_id == 5 and meta.scorer == "keydiff"
    for l, (c, p, k, v) in enumerate(per):
        assert np.array_equal(c, g[f"epkv_counts{l}"]) and np.array_equal(p, g[f"epkv_pos{l}"])
        assert np.array_equal(k, g[f"epkv_k{l}"]) and np.array_equal(v, g[f"epkv_v{l}"])


def test_centroid_similarity_matches_reference_cosine(ref):
    rng = np.random.default_rng(5)
    for _ in range(50):
        a, b = rng.standard_normal(64), rng.standard_normal(64)
        assert store.centroid_similarity(a, b) == ref.ref_cosine(a, b)
    assert store.centroid_similarity(np.zeros(8), np.ones(8)) == -np.inf
