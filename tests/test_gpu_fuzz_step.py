"""Randomised shapes through the DEFAULT block step (epk_evict_step, tensor-core
mode: P1 -> lse merge -> P2 with fused histograms -> threshold select +
compaction plan -> gather), each case checked against the CPU oracle:

* scores within 1e-4 relative of the fp64 restatement (oracle.score_layer_f64_mt,
  pinned to the reference by tests/test_oracle_vs_ref.py), Max or Avg;
* the selection + compaction bit-exact with evict_to_budget (kvcache.hpp:142-201;
  oracle/_ref where the reference tree exists, else the pinned restatement) on
  the step's OWN scores: per-head kept counts, retained positions in order,
  compacted K / V rows and the output head layout (heads followed by `slack`
  free rows).

Shapes drawn per case: layers 1-3, KV heads {1, 2, 4, 8}, query group 1-8,
prompt length 1-256 with G*p <= 2048 (1-16 query chunks: resident and streamed
P2 queries, 1-4 P1 chunk groups), ragged live counts per head (0 .. 3,000,
head regions with gaps), per-layer budgets from 0 to above the live count,
slack 0-300.  Seeds are fixed, so a failure names its case."""
import numpy as np
import pytest
import torch

from tests.helpers import bf16_round

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-4
D = 128


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    L = int(rng.integers(1, 4))
    H = int(rng.choice([1, 2, 4, 8, 8]))
    G = int(rng.integers(1, 9))
    p = int(rng.integers(1, min(256, 2048 // G) + 1))
    slack = int(rng.integers(0, 301))
    agg = "max" if seed % 3 else "avg"
    layers = []
    for _ in range(L):
        counts = rng.integers(0, 3001, H)
        if rng.random() < 0.3:
            counts[rng.integers(0, H)] = 0  # an empty head
        gaps = rng.integers(0, 64, H)  # rows between head regions (not live)
        live = int(counts.sum())
        r = rng.random()
        budget = 0 if r < 0.1 else (int(counts.max()) + 5 if r < 0.2 else int(rng.integers(1, max(2, live // H + 1))))
        layers.append((counts, gaps, budget))
    return rng, L, H, G, p, slack, agg, layers


@pytest.mark.timeout(900)
@pytest.mark.parametrize("seed", range(24))
def test_default_step_random_shapes_vs_oracle(gpu, orc, seed):
    from paper_2509_17396_b200.step import evict_step
    rng, L, H, G, p, slack, agg, layers = _case(seed)
    Hq = H * G
    # input cache: head h of layer l at an offset with a gap after every head
    caps, offs, host = [], [], []
    for counts, gaps, _ in layers:
        off = np.concatenate([[0], np.cumsum(counts + gaps)]).astype(np.int64)
        offs.append(off)
        caps.append(int(off[-1]) + 1)
    cin = gpu.EpisodeCache(L, H, D, caps, torch.bfloat16, "cuda")
    kept_rows = []
    for l, (counts, gaps, budget) in enumerate(layers):
        n = int(counts.sum())
        pos = np.concatenate([np.sort(rng.choice(1 << 20, c, replace=False)) for c in counts]).astype(np.int64)
        k = bf16_round(rng.standard_normal((n, D)).astype(np.float32))
        v = bf16_round(rng.standard_normal((n, D)).astype(np.float32))
        host.append((pos, k, v))
        b = int(cin.layer_base[l])
        rows = np.concatenate([np.arange(offs[l][h], offs[l][h] + counts[h]) for h in range(H)]).astype(np.int64) + b
        it = torch.as_tensor(rows, device="cuda")
        cin.k[it] = torch.as_tensor(k, device="cuda").bfloat16()
        cin.v[it] = torch.as_tensor(v, device="cuda").bfloat16()
        cin.pos[it] = torch.as_tensor(pos.astype(np.int32), device="cuda")
        cin.head_off[l] = torch.as_tensor(offs[l][:H + 1].astype(np.int32), device="cuda")
        cin.head_len[l] = torch.as_tensor(counts.astype(np.int32), device="cuda")
        kept_rows.append(min(n, H * budget))
    q = bf16_round(rng.standard_normal((L, Hq, p, D)).astype(np.float32))
    kp = bf16_round(rng.standard_normal((L, H, p, D)).astype(np.float32))
    out_caps = [H * (max(1, b) + slack) + kr + 1 for (_, _, b), kr in zip(layers, kept_rows)]
    cout = gpu.EpisodeCache(L, H, D, out_caps, torch.bfloat16, "cuda")
    scores = torch.zeros(cin.rows, dtype=torch.float32, device="cuda")
    kept = torch.zeros(L, dtype=torch.int32, device="cuda")
    n_max = max(int(c.max()) for c, _, _ in layers)
    evict_step(cin, cout, torch.as_tensor(q, device="cuda").bfloat16(), torch.as_tensor(kp, device="cuda").bfloat16(),
               [b for _, _, b in layers], aggregation=agg, mode="tc_bf16", slack=slack, n_max_per_head=max(n_max, 1),
               scores=scores, kept_per_layer=kept)
    torch.cuda.synchronize()
    gpu.default_context(0).poll_error()
    assert kept.cpu().tolist() == kept_rows
    use_ref = orc.ref_available()
    out_off, out_len, out_pos = cout.head_off.cpu().numpy(), cout.head_len.cpu().numpy(), cout.pos.cpu().numpy()
    for l, (counts, gaps, budget) in enumerate(layers):
        pos, k, v = host[l]
        ho = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        b = int(cin.layer_base[l])
        rows = np.concatenate([np.arange(offs[l][h], offs[l][h] + counts[h]) for h in range(H)]).astype(np.int64)
        s = scores[b:b + caps[l]].cpu().numpy()[rows].astype(np.float64)
        if len(pos):
            ref64 = orc.score_layer_f64_mt(q[l].astype(np.float64), k.astype(np.float64), kp[l].astype(np.float64),
                                           ho, agg == "max")
            rel = np.abs(s - ref64) / ref64
            assert rel.max() < SCORE_RTOL, (seed, l, rel.max())
        if use_ref:
            keep, cnt, _ = orc.ref_evict_layer(ho, pos, s, budget)
        else:
            _, keep = orc.evict_layer(ho, pos, s, budget)
            cnt = np.array([keep[ho[h]:ho[h + 1]].sum() for h in range(H)])
        keep = keep.astype(bool)
        exp_pos = [pos[ho[h]:ho[h + 1]][keep[ho[h]:ho[h + 1]]].tolist() for h in range(H)]
        assert out_len[l].tolist() == [int(c) for c in cnt], (seed, l)
        ob = int(cout.layer_base[l])
        assert [out_pos[ob + out_off[l, h]:ob + out_off[l, h] + out_len[l, h]].tolist() for h in range(H)] == \
            exp_pos, (seed, l)
        # output layout: heads in order, each followed by `slack` free rows
        exp_off = np.concatenate([[0], np.cumsum(np.asarray(cnt, np.int64) + slack)])
        assert out_off[l].tolist() == exp_off.tolist(), (seed, l)
        src = torch.as_tensor(rows[keep] + b, device="cuda")
        dst = cout.live_rows(l) if keep.any() else None
        if dst is not None:
            assert torch.equal(cout.k[dst].view(torch.int16), cin.k[src].view(torch.int16)), (seed, l)
            assert torch.equal(cout.v[dst].view(torch.int16), cin.v[src].view(torch.int16)), (seed, l)
    print(f"fuzz case {seed}: L={L} H={H} G={G} p={p} slack={slack} agg={agg} budgets={[b for _, _, b in layers]} "
          f"live={[int(c.sum()) for c, _, _ in layers]} ({'oracle/_ref' if use_ref else 'restatement'})")
