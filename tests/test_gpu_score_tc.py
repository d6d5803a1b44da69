"""K1 (tcgen05/TMEM tensor-core scorer, bf16 inputs, fp32 accumulate) vs
the oracle on the same bf16-rounded inputs.

Tolerances (north_star): the bf16 tensor-core path must give retained-set
overlap >= 99.9% per block step on identical cache state.  The scores
themselves are checked at 1e-4 relative against the fp64 restatement
(products of bf16 values are exact in fp32; the residual is fp32
accumulation order plus ex2/lg2.approx, measured ~1e-6)."""
import numpy as np
import pytest
import torch

from tests.helpers import bf16_round, random_layer

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-4
OVERLAP_MIN = 0.999


def _run(epk, layers, qs, kps, agg="max", mode="tc_bf16"):
    H = len(layers[0][0]) - 1
    cap = [int(ho[-1]) + 1 for ho, _, _, _ in layers]
    dt = torch.bfloat16 if mode == "tc_bf16" else torch.float32
    c = epk.EpisodeCache(len(layers), H, 128, cap, dt, "cuda")
    c.load_layers([(np.diff(ho), pos, k, v) for ho, pos, k, v in layers])
    q = torch.as_tensor(np.stack(qs), device="cuda").to(dt)
    kp = torch.as_tensor(np.stack(kps), device="cuda").to(dt)
    sc = epk.score_with_prompt(c, q, kp, agg, mode=mode).cpu().numpy()
    return c, [sc[int(c.layer_base[l]):int(c.layer_base[l]) + len(layers[l][1])] for l in range(len(layers))]


def _inputs(rng, L, Hq, H, p, counts):
    layers, qs, kps = [], [], []
    for _ in range(L):
        ho, pos, k, v = random_layer(rng, H, counts, 128, dtype=np.float32)
        layers.append((ho, pos, bf16_round(k), bf16_round(v)))
        qs.append(bf16_round(rng.standard_normal((Hq, p, 128)).astype(np.float32)))
        kps.append(bf16_round(rng.standard_normal((H, p, 128)).astype(np.float32)))
    return layers, qs, kps


@pytest.mark.parametrize("agg", ["max", "avg"])
@pytest.mark.parametrize("cfg", [
    (1, 3, 1, 128, [1000]),           # one head, G*p = 384 (3 query chunks, resident)
    (2, 24, 8, 64, [300] * 8),        # Llama GQA, p = 64
    (1, 4, 4, 1, [0, 129, 5, 256]),   # p = 1, empty head, partial tiles
    (1, 12, 2, 200, [700, 333]),      # two prompt tiles, G*p = 1200 (streamed Q)
    (1, 28, 4, 128, [2100, 1900, 17, 4096]),  # Qwen GQA (G = 7, NQ = 7)
    (1, 16, 2, 256, [600, 450]),      # the kernel's prompt limits: p = 256, G*p = 2048 (NQ = 16, streamed)
])
def test_tc_scores_vs_fp64_oracle(gpu, orc, cfg, agg):
    L, Hq, H, p, counts = cfg
    rng = np.random.default_rng(sum(counts) + p + Hq)
    layers, qs, kps = _inputs(rng, L, Hq, H, p, counts)
    _, got = _run(gpu, layers, qs, kps, agg)
    for l, (ho, pos, k, v) in enumerate(layers):
        if len(pos) == 0:
            continue
        exp = orc.score_layer_f64(qs[l].astype(np.float64), k.astype(np.float64), kps[l].astype(np.float64), ho,
                                  agg == "max")
        rel = np.abs(got[l].astype(np.float64) - exp) / exp
        assert rel.max() < SCORE_RTOL, (l, rel.max())


def test_tc_retained_overlap_cfg2_layer(gpu, orc):
    """cfg2 layer shape (8 heads x 10,240 live entries, G = 3, p = 128, M = 8,192):
    the bf16 tensor-core selection keeps >= 99.9% of the fp64 oracle's set."""
    rng = np.random.default_rng(2)
    layers, qs, kps = _inputs(rng, 1, 24, 8, 128, [10240] * 8)
    c, got = _run(gpu, layers, qs, kps)
    ho, pos, k, v = layers[0]
    # fp64 reference scores via the exact GPU path on the same values is
    # too slow to restate on CPU at this size; use the fp32 parity kernel
    # (bit-exact with the oracle, within 1e-5 of fp64) as the reference.
    _, ref32 = _run(gpu, layers, qs, kps, mode="exact_f32")
    rel = np.abs(got[0] - ref32[0]) / ref32[0]
    assert rel.max() < SCORE_RTOL, rel.max()
    M = 8192
    _, keep_ref = orc.evict_layer(ho, pos, ref32[0].astype(np.float64), M)
    _, keep_tc = orc.evict_layer(ho, pos, got[0].astype(np.float64), M)
    inter = np.logical_and(keep_ref, keep_tc).sum()
    recall = inter / keep_ref.sum()
    assert recall >= OVERLAP_MIN, recall


def test_tc_fused_step_overlap(gpu, orc):
    """The whole tensor-core step (score -> select -> compact) against the
    oracle chain on the same state: retained overlap >= 99.9% per layer."""
    from paper_2509_17396_b200.step import evict_step
    rng = np.random.default_rng(4)
    L, Hq, H, p, M = 3, 24, 8, 128, 1024
    layers, qs, kps = _inputs(rng, L, Hq, H, p, [1280] * H)
    cap = [int(ho[-1]) + 256 * H for ho, _, _, _ in layers]
    cin = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    cin.load_layers([(np.diff(ho), pos, k, v) for ho, pos, k, v in layers])
    cout = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    evict_step(cin, cout, torch.as_tensor(np.stack(qs), device="cuda").bfloat16(),
               torch.as_tensor(np.stack(kps), device="cuda").bfloat16(), [M] * L, slack=256)
    for l, (ho, pos, k, v) in enumerate(layers):
        s = orc.score_layer_f64(qs[l].astype(np.float64), k.astype(np.float64), kps[l].astype(np.float64), ho, True)
        _, keep = orc.evict_layer(ho, pos, s, M)
        got = cout.retained_positions()[l]
        ref = [pos[ho[h]:ho[h + 1]][keep[ho[h]:ho[h + 1]]].tolist() for h in range(H)]
        inter = sum(len(set(a) & set(b)) for a, b in zip(got, ref))
        assert sum(len(a) for a in got) == H * M
        assert inter / (H * M) >= OVERLAP_MIN


@pytest.mark.timeout(300)
def test_tc_scorer_deterministic_at_scale_nq4(gpu):
    """Regression for the P1 TMEM-slot protocol (three epilogue job groups):
    Llama-3.1-8B grouping (G = 4, p = 128 -> four query chunks), 24 layers of
    8 x 10,240 rows, scored repeatedly: every run finishes and gives the same
    bits (a slot waited on by two warps once aliased mbarrier phases here)."""
    L, Hq, H, p, n = 24, 32, 8, 128, 10240
    c = gpu.EpisodeCache(L, H, 128, [n * H] * L, torch.bfloat16, "cuda")
    c.set_regions(n)
    c.head_len.fill_(n)
    g = torch.Generator(device="cuda").manual_seed(3)
    c.k.copy_(torch.randn(c.rows, 128, device="cuda", generator=g).bfloat16())
    q = torch.randn(L, Hq, p, 128, device="cuda", generator=g).bfloat16()
    kp = torch.randn(L, H, p, 128, device="cuda", generator=g).bfloat16()
    ref = gpu.score_with_prompt(c, q, kp, "max", mode="tc_bf16").clone()
    assert torch.isfinite(ref).all() and (ref > 0).all() and (ref <= 1.0 + 1e-6).all()
    for _ in range(6):
        again = gpu.score_with_prompt(c, q, kp, "max", mode="tc_bf16")
        assert torch.equal(again.view(torch.int32), ref.view(torch.int32))


def test_grouped_step_equals_single_group(gpu):
    """epk_evict_step with layer groups (P1 once, then per group P2 -> select
    -> compaction on the side stream) gives the same bits as one group."""
    from paper_2509_17396_b200.step import evict_step
    rng = np.random.default_rng(9)
    L, Hq, H, p, M = 5, 24, 8, 128, 700
    counts = [[900, 800, 1000, 0, 950, 870, 1200, 640]] * L
    layers, qs, kps = [], [], []
    for l in range(L):
        ho, pos, k, v = random_layer(rng, H, counts[l], 128, dtype=np.float32)
        layers.append((ho, pos, bf16_round(k), bf16_round(v)))
        qs.append(bf16_round(rng.standard_normal((Hq, p, 128)).astype(np.float32)))
        kps.append(bf16_round(rng.standard_normal((H, p, 128)).astype(np.float32)))
    cap = [int(ho[-1]) + 128 * H for ho, _, _, _ in layers]
    cin = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
    cin.load_layers([(np.diff(ho), pos, k, v) for ho, pos, k, v in layers])
    q = torch.as_tensor(np.stack(qs), device="cuda").bfloat16()
    kp = torch.as_tensor(np.stack(kps), device="cuda").bfloat16()
    ctx = gpu.default_context(0)
    outs = []
    for group in (0, 2):
        ctx.set_option(layer_group=group, overlap=True)
        cout = gpu.EpisodeCache(L, H, 128, cap, torch.bfloat16, "cuda")
        sc = torch.zeros(cin.rows, dtype=torch.float32, device="cuda")
        evict_step(cin, cout, q, kp, [M] * L, mode="tc_bf16", slack=128, scores=sc, ctx=ctx)
        torch.cuda.synchronize()
        ctx.poll_error()
        outs.append((cout, sc))
    ctx.set_option(layer_group=0)
    (a, sa), (b, sb) = outs
    for l in range(L):
        lo, hi = int(cin.layer_base[l]), int(cin.layer_base[l]) + int(np.sum(counts[l]))
        assert torch.equal(sa[lo:hi].view(torch.int32), sb[lo:hi].view(torch.int32)), l
    assert torch.equal(a.head_off, b.head_off) and torch.equal(a.head_len, b.head_len)
    for l in range(L):
        ra, rb = a.live_rows(l), b.live_rows(l)
        assert torch.equal(a.pos[ra], b.pos[rb])
        assert torch.equal(a.k[ra].view(torch.int16), b.k[rb].view(torch.int16))
        assert torch.equal(a.v[ra].view(torch.int16), b.v[rb].view(torch.int16))


def test_tc_chained_episode_overlap_reported(gpu, orc):
    """the bf16 path chained over a whole episode, against the
    fp64 oracle chained on its own decisions.  Swaps compound across steps, so
    the end-of-episode overlap is REPORTED (printed) and only loosely gated;
    the per-step gate (>= 99.9 % on identical state) is the test above."""
    from tests.test_gpu_blockprefill import SynthProvider
    L, Hq, H, d, n, B, M, p = 1, 24, 8, 128, 8 * 512, 512, 1024, 64
    prov = SynthProvider(L, Hq, H, d, n, p, seed=11, dtype=torch.bfloat16)
    rep = gpu.block_prefill(prov, L, Hq, H, d, n, gpu.BlockPrefillConfig(M, B), dtype=torch.bfloat16)
    got = rep.cache.retained_positions()[0]
    k = prov.k[0].double().numpy()
    q = prov.q[0].double().numpy()
    kp = prov.kp[0].double().numpy()
    state = [[] for _ in range(H)]
    for start in range(0, n, B):
        for h in range(H):
            state[h] += list(range(start, min(n, start + B)))
        ho = np.concatenate([[0], np.cumsum([len(s) for s in state])])
        pos = np.concatenate([np.array(s, np.int64) for s in state])
        kk = np.concatenate([k[h, state[h]] for h in range(H)])
        sc = orc.score_layer_f64(q, kk, kp, ho, True)
        st, keep = orc.evict_layer(ho, pos, sc, M)
        assert st >= 0
        state = [pos[ho[h]:ho[h + 1]][keep[ho[h]:ho[h + 1]]].tolist() for h in range(H)]
    a = {(h, x) for h in range(H) for x in got[h]}
    b = {(h, x) for h in range(H) for x in state[h]}
    jac = len(a & b) / len(a | b)
    rec = len(a & b) / len(b)
    print(f"chained bf16 vs fp64 oracle over {n // B} blocks: Jaccard {jac:.4f}, recall {rec:.4f}")
    assert len(a) == len(b) == H * M
    assert rec >= 0.95
