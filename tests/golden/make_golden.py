"""Generates tests/golden/golden_v1.npz from the UNMODIFIED reference
(oracle/_ref/libepkref.so, built from /root/reference by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures travel with the repo, so the oracle and the GPU path stay pinned
to the reference on machines without /root/reference.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.helpers import quantised_scores, random_layer  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")


def main():
    g = {}
    rng = np.random.default_rng(20261017)
    # eviction instances (kvcache.hpp:142) incl. ties and pins
    for i in range(40):
        H = int(rng.integers(1, 5))
        counts = rng.integers(0, 12, H)
        ho, pos, k, v = random_layer(rng, H, counts, 2, pos_space=16)
        sc = quantised_scores(rng, len(pos), int(rng.integers(2, 6)))
        budget = int(rng.integers(1, 6))
        pins = np.array([0], np.int64) if i % 3 == 0 and H * budget >= H else np.zeros(0, np.int64)
        try:
            keep, hc, _ = O.ref_evict_layer(ho, pos, sc, budget, set(pins.tolist()))
            status = 0
        except O.RefError:
            keep, status = np.zeros(len(pos), bool), -2
        g[f"ev{i}_head_off"], g[f"ev{i}_pos"], g[f"ev{i}_scores"] = ho, pos, sc
        g[f"ev{i}_budget"], g[f"ev{i}_pins"], g[f"ev{i}_keep"], g[f"ev{i}_status"] = budget, pins, keep, status
    g["ev_count"] = 40
    # patched-prompt scores (score_with_prompt over the restated grids)
    shapes = [(6, 2, 16, 5, [13, 9]), (4, 4, 8, 3, [5, 0, 7, 2]), (24, 8, 64, 8, [20] * 8), (2, 1, 32, 1, [33])]
    for i, (hq, H, d, p, counts) in enumerate(shapes):
        ho, pos, k, _ = random_layer(rng, H, counts, d)
        q = rng.standard_normal((hq, p, d))
        kp = rng.standard_normal((H, p, d))
        for agg in (1, 0):
            g[f"sc{i}_{agg}_scores"] = O.ref_score_layer_f64(q, k, kp, ho, pos, bool(agg))
        g[f"sc{i}_q"], g[f"sc{i}_k"], g[f"sc{i}_kp"], g[f"sc{i}_head_off"], g[f"sc{i}_pos"] = q, k, kp, ho, pos
    g["sc_count"] = len(shapes)
    # kmeans
    for i, (n, dim, k, seed) in enumerate([(200, 8, 4, 7), (96, 16, 8, 3), (30, 4, 30, 9), (50, 5, 1, 2)]):
        pts = rng.standard_normal((n, dim))
        a, c, it, sse = O.ref_kmeans(pts, k, seed)
        g[f"km{i}_pts"], g[f"km{i}_k"], g[f"km{i}_seed"] = pts, k, seed
        g[f"km{i}_assign"], g[f"km{i}_cent"], g[f"km{i}_iters"], g[f"km{i}_sse"] = a, c, it, sse
    g["km_count"] = 4
    # allocate
    for i in range(20):
        L = int(rng.integers(1, 29))
        s = rng.random(L) * (rng.random(L) > 0.1)
        M = int(rng.integers(1, 9000))
        alpha = float(rng.choice([0.0, 1.0, 1.1, 2.0]))
        b, w = O.ref_allocate(s, M, alpha)
        g[f"al{i}_s"], g[f"al{i}_M"], g[f"al{i}_alpha"], g[f"al{i}_b"], g[f"al{i}_w"] = s, M, alpha, b, w
    g["al_count"] = 20
    # sensitivity (measure_sensitivity on a seeded toy model)
    sig, sk, kf, kb = O.ref_measure_sensitivity(3, 4, 2, 8, 3, 48, 5, 16, 4)
    g["sens_sigma"], g["sens_skipped"], g["sens_kf"], g["sens_kb"] = sig, sk, kf, kb
    # block_prefill occupancy traces
    series, ev, nb, counts, _ = O.ref_block_prefill(1, 1, 1, 8, 3, 9, 2, 1, 3, [7, 21, 42])
    g["bp_c2_series"], g["bp_c2_evictions"] = series, ev
    series, ev, nb, counts, _ = O.ref_block_prefill(2, 2, 1, 8, 3, 64, 17, 8, 16, [7, 21, 42], [4, 12])
    g["bp_alloc_counts"] = counts.sum(axis=1)
    series, ev, nb, counts, _ = O.ref_block_prefill(2, 4, 2, 8, 3, 120, 5, 8, 16, [7, 21, 42])
    g["bp_120_series"], g["bp_120_evictions"], g["bp_120_counts"] = series, ev, counts
    # KeyDiff scores (keydiff_scores, scoring.hpp:186), own RNG stream: ragged
    # heads, an empty head, a zero key, a zero-anchor head
    krng = np.random.default_rng(186)
    for i, (d, counts) in enumerate([(8, [5, 0, 9, 3]), (16, [40, 33]), (128, [64, 1, 17]), (4, [6, 6])]):
        ho, pos, k, _ = random_layer(krng, len(counts), counts, d)
        if i == 0:
            k[2] = 0.0
        if i == 3:
            k[6:12] = 0.0
        g[f"kd{i}_head_off"], g[f"kd{i}_pos"], g[f"kd{i}_k"] = ho, pos, k
        g[f"kd{i}_scores"] = O.ref_keydiff_layer(k, ho, pos)
    g["kd_count"] = 4
    # a .epkv file written by the reference's persist (kvcache.hpp:281)
    import tempfile
    erng = np.random.default_rng(281)
    pl = []
    for l, counts in enumerate([[3, 0, 2], [1, 4, 1]]):
        c = np.asarray(counts, np.int64)
        n = int(c.sum())
        pos = np.concatenate([np.sort(erng.choice(100, int(x), replace=False)) for x in c]).astype(np.int64)
        pl.append((c, pos, erng.standard_normal((n, 8)), erng.standard_normal((n, 8))))
        g[f"epkv_counts{l}"], g[f"epkv_pos{l}"], g[f"epkv_k{l}"], g[f"epkv_v{l}"] = pl[-1]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "e.epkv")
        O.ref_persist(path, pl, episode_id=5, scorer="keydiff", budget_per_head=3, layer_budgets=[2, 4],
                      layer_budget_fields=[2, 4])
        g["epkv_bytes"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    np.savez_compressed(OUT, **g)
    print(OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
