"""Seeded synthetic inputs shared by the CPU and GPU tests."""
import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float32 (exactly representable)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def random_layer(rng, H, counts, d, pos_space=None, dtype=np.float64):
    """One layer: head-major rows, strictly increasing positions per head."""
    counts = np.asarray(counts, np.int64)
    head_off = np.zeros(H + 1, np.int64)
    head_off[1:] = np.cumsum(counts)
    n = int(head_off[-1])
    pos = []
    for c in counts:
        space = pos_space or max(int(c) * 3, 8)
        pos.append(np.sort(rng.choice(space, int(c), replace=False)))
    pos = np.concatenate(pos).astype(np.int64) if n else np.zeros(0, np.int64)
    k = rng.standard_normal((n, d)).astype(dtype)
    v = rng.standard_normal((n, d)).astype(dtype)
    return head_off, pos, k, v


def quantised_scores(rng, n, levels=4):
    """Coarse score grid forcing ties (test_kvcache.cpp:131-133)."""
    return rng.integers(0, levels, n).astype(np.float64)


def composite_topk(head_off, pos, scores, budget, pins=()):
    """Independent brute force (test_kvcache.cpp:29-59): keep pins, then sort by
    (-score, position, head) and keep until the layer limit."""
    H = len(head_off) - 1
    keep = np.zeros(len(pos), bool)
    rows = []
    pinned_live = 0
    for h in range(H):
        for r in range(head_off[h], head_off[h + 1]):
            if pos[r] in pins:
                keep[r] = True
                pinned_live += 1
            else:
                rows.append((-scores[r], pos[r], h, r))
    limit = H * budget
    if len(pos) <= limit:
        return np.ones(len(pos), bool)
    rows.sort()
    for i in range(max(0, limit - pinned_live)):
        if i < len(rows):
            keep[rows[i][3]] = True
    return keep
