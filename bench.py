#!/usr/bin/env python
"""bench.py -- EpiCache block-prefill eviction step (score + select + compact)
on B200, BASELINE.json metric "KV tokens scored+evicted+compacted/sec per
block step at Llama-3.2-3B shape".

A step = one pass of the hot path over one block step of one episode at the
cfg2 shape (BASELINE.json configs[1]): 28 layers x 8 kv-heads x (8,192 budget +
2,048 block) = 2,293,760 live entries scored against a 128-row patched prompt
(24 query heads), pooled top-k per layer (65,536 kept), compacted out of place.

  python bench.py [--gpus N --steps K --warmup W]           our sm_100a path
  python bench.py --impl reference [...]                      the reference CPU path
  (N > 1: launched by torch.distributed.run; one episode per GPU, weak scaling)

JSON keys beyond the base contract:
  roofline      dominant kernel of the step (live CUDA-event timing) vs the
                measured peaks in MEASURED_PEAKS.json; `traffic` from the
                committed ncu capture (profiles/) when present
  step_roofline whole-step algorithmic bytes / step time vs measured HBM
  kernels       per-kernel average ms / share of the step
  cpu_baseline  the reference CPU path (oracle/_ref, compiled from the
                reference headers) on the host cores, bounded sample
  e2e           same metric through the public API with host buffers: the
                block's K/V + prompt copied H2D and retained positions copied
                D2H inside the timed region, cache resident in HBM
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KV tokens scored+evicted+compacted/sec per block step at Llama-3.2-3B shape"
UNIT = "tokens/s"

CONFIGS = {
    "cfg1": dict(L=1, Hq=24, H=8, d=128, N=16384, block=512, M=2048, p=64,
                 desc="cfg1 CPU-oracle toy: 1 layer, 24 Q / 8 KV heads, hd 128, 16K context, block 512, budget 2K"),
    "cfg2": dict(L=28, Hq=24, H=8, d=128, N=131072, block=2048, M=8192, p=128,
                 desc="cfg2 Llama-3.2-3B shape (28 layers, 24 Q / 8 KV heads, hd 128), 128K context, block 2048, "
                      "budget 8192/head, uniform layer budgets, p=128 patched-prompt rows, steady-state block step"),
    "cfg3": dict(L=28, Hq=24, H=8, d=128, N=131072, block=2048, M=8192, p=128, E=4, adaptive=True,
                 desc="cfg3 Llama-3.2-3B shape, E=4 episodes (K-means on 2,048 segment embeddings of dim 1,024), "
                      "adaptive layer budgets allocate(sigma, 8192, alpha=1.1), block 2048, 128K context"),
    "cfg4": dict(L=32, Hq=32, H=8, d=128, N=262144, block=2048, M=8192, p=128,
                 desc="cfg4 Llama-3.1-8B shape (32 layers, 32 Q / 8 KV heads), 256K context, block 2048, budget 8192"),
    "cfg5": dict(L=28, Hq=28, H=4, d=128, N=1048576, block=4096, M=174762, p=128,
                 desc="cfg5 Qwen2.5-7B shape (28 layers, 28 Q / 4 KV heads), 1M context, block 4096, "
                      "6x compression (M = N/6)"),
}


def _flatten(obj, path=""):
    if isinstance(obj, dict):
        for k, v in obj.items():
            yield from _flatten(v, f"{path}.{k}".lower())
    elif isinstance(obj, (int, float)) and not isinstance(obj, bool):
        yield path, float(obj)


def load_peaks():
    """(hbm GB/s, bf16 TF/s sustained, bf16 TF/s burst, source).  The
    driver-written MEASURED_PEAKS.json is read by key names (any nesting:
    an 'hbm' number for bandwidth, 'bf16' numbers for the tensor pipe,
    'sustained' preferred); TB/s values are converted.  Fallback: the
    B200_PROFILING.md figures."""
    hbm, tc_sus, tc_burst = 6650.0, 1400.0, 1590.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            flat = list(_flatten(json.load(f)))
    except Exception:
        return hbm, tc_sus, tc_burst, "fallback"
    hb = [(k, v) for k, v in flat if "hbm" in k or "copy" in k or "dram" in k]
    bf = [(k, v) for k, v in flat if "bf16" in k or "tensor" in k or "tflop" in k]
    if not hb and not bf:
        return hbm, tc_sus, tc_burst, "fallback"
    if hb:
        k, v = max(hb, key=lambda kv: ("gb" in kv[0] or "bw" in kv[0] or "band" in kv[0], "burst" not in kv[0]))
        hbm = v * 1000.0 if v < 100 else v  # TB/s -> GB/s
    if bf:
        sus = [kv for kv in bf if "sustain" in kv[0]] or bf
        tc_sus = sus[0][1] * (1000.0 if sus[0][1] < 20 else 1.0)
        burst = [kv for kv in bf if "sustain" not in kv[0]] or sus
        tc_burst = max(v for _, v in burst) * (1000.0 if max(v for _, v in burst) < 20 else 1.0)
    return hbm, tc_sus, tc_burst, "measured"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") >= 8]
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        load = [s for s in sm if s > 600] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for i, nm in enumerate(names):
                if "Active" in r[5 + i] and "Not" not in r[5 + i]:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons),
                "samples": len(rows)}


class EnergyMeter:
    """NVML total-energy counter (mJ) of one GPU and its enforced power limit;
    every method returns None where NVML is unavailable."""

    def __init__(self, gpu: int):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
        except Exception:  # noqa: BLE001 (no NVML: energy is simply not reported)
            self.h = None

    def mj(self):
        try:
            return float(self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h)) if self.h is not None else None
        except Exception:  # noqa: BLE001
            return None

    def limit_w(self):
        try:
            return self.nv.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0 if self.h is not None else None
        except Exception:  # noqa: BLE001
            return None


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def synthetic_sigma(L, seed=11):
    """A seeded per-layer key-similarity profile sigma_l (cfg3's adaptive
    budgets): the same numbers for both arms, so the reference's allocate and
    ours see identical inputs (SURVEY 7 hard part 10)."""
    rng = np.random.default_rng(seed)
    return (1.0 - rng.uniform(0.05, 0.6, L)).tolist()


def layer_budgets(c):
    """Per-layer per-head budgets: uniform M, or cfg3's allocate(sigma, M, 1.1)
    (allocation.hpp:120-198, restated bit-for-bit in paper_2509_17396_b200.allocation)."""
    if not c.get("adaptive"):
        return [c["M"]] * c["L"]
    from paper_2509_17396_b200.allocation import SensitivityProfile, allocate
    sig = synthetic_sigma(c["L"])
    prof = SensitivityProfile(sigma=sig, sensitivity=[1.0 - x for x in sig])
    return list(allocate(prof, c["M"], 1.1).layer_budgets)


def step_sizes(c):
    """(max live per head, live entries, kept entries) of ONE episode's steady-state step."""
    bud = layer_budgets(c)
    n_h = max(bud) + c["block"]
    live = sum(c["H"] * (b + c["block"]) for b in bud)
    keep = sum(c["H"] * b for b in bud)
    return n_h, live, keep


def algorithmic(c):
    """bytes / flops / exps per episode step (bf16)."""
    n_h, live, keep = step_sizes(c)
    d, G, p = c["d"], c["Hq"] // c["H"], c["p"]
    B = live * d * 2 + c["L"] * (c["Hq"] + c["H"]) * p * d * 2 + 4 * keep * d * 2 + 4 * live + 4 * keep
    F = 2 * p * d * G * live
    X = p * G * live
    return B, F, X


def config_dict(c, c_total, world, shard):
    """The workload description both arms print (identical dicts)."""
    n_h, live, keep = step_sizes(c_total)
    E = c_total.get("E", 1)
    return {"workload": c_total["desc"], "layers": c_total["L"], "q_heads": c_total["Hq"], "kv_heads": c_total["H"],
            "head_dim": c_total["d"], "context": c_total["N"], "block": c_total["block"],
            "budget_per_head": c_total["M"], "layer_budgets": "adaptive" if c_total.get("adaptive") else "uniform",
            "prompt_len": c_total["p"], "episodes": E, "live_entries_per_episode_step": live,
            "kept_per_episode_step": keep, "aggregation": "max",
            "parallelism": f"layers x{world} (one episode)" if shard else f"episodes over {world} GPU(s)",
            "l2": "inputs larger than L2: >= 3 rotating steady-state caches of "
                  f"{2 * live * c_total['d'] * 2 / 1e9:.2f} GB K+V per GPU"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def make_inputs(epk, torch, c, R, device, seed, dtype=None, budgets=None):
    """R steady-state input caches (n_l = M_l + block live rows per head of
    layer l, dense) and R prompt sets, resident in HBM (bf16 by default)."""
    dtype = dtype or torch.bfloat16
    bud = budgets if budgets is not None else layer_budgets(c)
    L, H, d, p, Hq = c["L"], c["H"], c["d"], c["p"], c["Hq"]
    nl = [b + c["block"] for b in bud]
    cap = [H * n for n in nl]
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    caches, qs, kps = [], [], []
    pos_all = torch.sort(torch.randperm(c["N"], device=device, generator=g)[:max(nl)])[0].to(torch.int32)
    for r in range(R):
        cc = epk.EpisodeCache(L, H, d, cap, dtype, device)
        cc.k.copy_(torch.randn(cc.rows, d, device=device, generator=g, dtype=torch.float32).to(dtype))
        cc.v.copy_(torch.randn(cc.rows, d, device=device, generator=g, dtype=torch.float32).to(dtype))
        for l in range(L):
            b = int(cc.layer_base[l])
            cc.pos[b:b + H * nl[l]].copy_(torch.sort(pos_all[:nl[l]])[0].repeat(H))
        off = torch.stack([torch.arange(H + 1, device=device, dtype=torch.int32) * n for n in nl])
        cc.head_off.copy_(off)
        cc.head_len.copy_(torch.tensor(nl, device=device, dtype=torch.int32)[:, None].expand(L, H))
        caches.append(cc)
        qs.append(torch.randn(L, Hq, p, d, device=device, generator=g).to(dtype))
        kps.append(torch.randn(L, H, p, d, device=device, generator=g).to(dtype))
    out = epk.EpisodeCache(L, H, d, cap, dtype, device)
    return caches, qs, kps, out


def run_ours(args, c, rank, world, device, torch, dist):
    import paper_2509_17396_b200 as epk
    from paper_2509_17396_b200.step import StepPlan, evict_step

    ctx = epk.default_context(device.index)
    ctx.set_option(layer_group=args.layer_group, overlap=not args.no_overlap)
    n_h, live, keep = step_sizes(c)
    # this rank's episodes (episodes round-robin over the GPUs)
    n_ep = len(range(rank, c.get("E", 1), world)) if not args.total_live else 1
    # several episodes on this GPU: one step over all of them -- their layers
    # concatenated in one cache (the C ABI is layer-agnostic and every layer
    # keeps its own budget), so the episodes share the step's launches
    batch = n_ep > 1 and not args.no_batch_episodes and n_ep * c["L"] <= 128
    budgets = layer_budgets(c)
    eps = []
    if batch:
        R = 3
        budgets = budgets * n_ep
        eps.append(make_inputs(epk, torch, dict(c, L=n_ep * c["L"]), R, device, 1234 + 97 * rank, budgets=budgets))
    else:
        R = max(1, -(-3 // max(1, n_ep)))  # >= 3 distinct input caches per GPU: every step reads cold K/V
        for e in range(n_ep):
            eps.append(make_inputs(epk, torch, c, R, device, 1234 + 97 * rank + e))
    plans = [[StepPlan(cs[r], out, budgets) for r in range(R)] for cs, _, _, out in eps]

    def step(i):
        r = i % R
        for e, (caches, qs, kps, out) in enumerate(eps):
            evict_step(caches[r], out, qs[r], kps[r], budgets, mode="tc_bf16", slack=c["block"], n_max_per_head=n_h,
                       plan=plans[e][r], ctx=ctx)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    ctx.poll_error()
    stream = torch.cuda.current_stream(device)

    meter = EnergyMeter(device.index)

    def timed(steps):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks = ClockSampler(device.index)
        clocks.start()
        time.sleep(0.3)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = ctx.launches
        e0 = meter.mj()
        ev0.record(stream)
        for i in range(steps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
        e1 = meter.mj()
        if dist is not None:
            dist.barrier()
        launches = ctx.launches - launches0
        clk = clocks.stop()
        # board energy of this GPU over the timed steps (NVML counter; coarse
        # for a short burst), with the enforced power limit it runs against
        clk["energy_j_per_step"] = ((e1 - e0) / 1000.0 / steps
                                    if e0 is not None and e1 is not None and e1 > e0 else None)
        clk["power_limit_w"] = meter.limit_w()
        t = torch.tensor([ev0.elapsed_time(ev1)], device=device, dtype=torch.float64)
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ctx.poll_error()
        return float(t.item()), launches, clk

    ms_max, launches, clk = timed(args.steps)
    # per-kernel live timing: a separate pass with events around every launch,
    # right after the timed steps (the same thermal state as the headline)
    prof_steps = min(args.steps, 30)
    ctx.profile(True)
    for i in range(prof_steps):
        step(i)
    recs = ctx.profile_records()
    ctx.profile(False)
    kern = {}
    for name, kms in recs:
        kern.setdefault(name, []).append(kms)
    kernels = {k: {"ms_per_step": sum(v) / prof_steps, "launches_per_step": len(v) / prof_steps}
               for k, v in kern.items()}
    prof_total = sum(x["ms_per_step"] for x in kernels.values())
    for k in kernels:
        kernels[k]["share"] = kernels[k]["ms_per_step"] / prof_total if prof_total else None

    # the same step over a long power-capped run (clocks settle under the 1 kW cap)
    sustained = None
    if args.sustained_steps > 0:
        s_ms, _, s_clk = timed(args.sustained_steps)
        sustained = {"steps": args.sustained_steps, "ms_per_step": s_ms / args.sustained_steps,
                     "value": None, "clocks": s_clk}
        # power-bound check: the step's board energy at the enforced power
        # limit; ms_per_step close to this means the run is energy-bound (the
        # 1 kW cap), not bound by any one unit's rate
        if s_clk.get("energy_j_per_step") and s_clk.get("power_limit_w"):
            sustained["ms_at_power_limit"] = s_clk["energy_j_per_step"] / s_clk["power_limit_w"] * 1000.0

    energy_costs = None
    if sustained is not None and not args.no_power_roofline and meter.mj() is not None:
        try:  # 4 GiB of scratch: a GPU short of memory skips the power roofline, not the bench
            energy_costs = calibrate_energy(torch, device, meter)
        except torch.cuda.OutOfMemoryError:
            torch.cuda.empty_cache()

    if args.timeline:  # one profiled step's launch timeline (start, duration, stream)
        ctx.profile(True)
        for i in range(3):
            step(i)
        tl = ctx.profile_timeline()
        ctx.profile(False)
        with open(args.timeline, "w") as f:
            f.write("# kernel  start_ms  dur_ms  stream(0 main, 1 side)\n")
            for name, t0, d, side in tl:
                f.write(f"{name:16s} {t0:9.4f} {d:8.4f} {side}\n")
    del eps, plans
    torch.cuda.empty_cache()
    exact = run_exact_f32(args, c, epk, torch, device, ctx, dist) if not args.no_exact else None
    e2e = run_e2e(args, c, epk, torch, device, ctx, dist) if not args.no_e2e else None
    phase_a = run_phase_a(c, epk, torch, device) if c.get("E", 1) > 1 and rank == 0 else None
    return dict(ms=ms_max, launches=launches, clocks=clk, kernels=kernels, e2e=e2e, live=live * n_ep, keep=keep,
                sustained=sustained, exact=exact, phase_a=phase_a, episodes=n_ep, energy_costs=energy_costs,
                batched=batch)


def calibrate_energy(torch, device, meter, secs=1.5):
    """Board energy per byte of a plain HBM copy (b.copy_(a), 1 Gi bf16: 4 GiB
    read + written per 2 launches) and per bf16 FLOP of a dense GEMM (8192^3),
    each run back to back for ~secs on this GPU (NVML energy counter).  These
    board-level costs (static power included) price the step's algorithmic
    bytes and tensor FLOPs for the power roofline."""
    out = {}
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device=device).normal_()
    b = torch.empty_like(a)
    x = torch.randn(8192, 8192, dtype=torch.bfloat16, device=device)
    y = torch.randn(8192, 8192, dtype=torch.bfloat16, device=device)
    for name, fn, work in (("pj_per_byte", lambda: b.copy_(a), 2.0 * (1 << 31)),
                           ("pj_per_flop", lambda: torch.matmul(x, y), 2.0 * 8192 ** 3)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        t = time.time()
        n = 0
        e0 = meter.mj()
        while time.time() - t < secs:
            for _ in range(10):
                fn()
            n += 10
            torch.cuda.synchronize()
        e1 = meter.mj()
        out[name] = (e1 - e0) * 1e9 / n / work  # mJ -> pJ per unit
    del a, b, x, y
    torch.cuda.empty_cache()
    out["how"] = ("NVML board energy over ~1.5 s of back-to-back torch b.copy_(a) (1 Gi bf16) and torch.matmul "
                  "bf16 8192^3 on this GPU, right after the sustained step run")
    return out


def run_exact_f32(args, c, epk, torch, device, ctx, dist):
    """The precision-matched path: the same step with fp32 K/V/Q through the
    EPK-F32 parity scorer (bit-exact with the CPU restatement) and the generic
    pooled select -- the throughput a user gets with bit-exact retained sets."""
    from paper_2509_17396_b200.step import StepPlan, evict_step
    n_h, live, keep = step_sizes(c)
    caches, qs, kps, out = make_inputs(epk, torch, c, 2, device, 4321, dtype=torch.float32)
    budgets = layer_budgets(c)
    plans = [StepPlan(caches[r], out, budgets) for r in range(2)]
    steps = max(2, min(args.steps, 6))

    def step(i):
        evict_step(caches[i % 2], out, qs[i % 2], kps[i % 2], budgets, mode="exact_f32", slack=c["block"],
                   n_max_per_head=n_h, plan=plans[i % 2], ctx=ctx)

    step(0)
    torch.cuda.synchronize()
    ctx.poll_error()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    e0.record()
    for i in range(steps):
        step(i)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device=device, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    world = dist.get_world_size() if dist is not None else 1
    units = getattr(args, "total_live", None) or world * live
    ms = float(t.item()) / steps
    del caches, qs, kps, out, plans
    torch.cuda.empty_cache()
    return {"value": units / (ms / 1000.0), "unit": UNIT, "ms_per_step": ms, "steps": steps, "dtype": "f32",
            "path": "epk_evict_step mode EPK_SCORE_EXACT_F32 (score_f32.cu) -> generic pooled select -> compaction; "
                    "retained sets bit-exact vs the CPU restatement"}


def run_phase_a(c, epk, torch, device):
    """cfg3's one-time Phase A on this GPU (episodic.hpp:117-146): K-means of
    2,048 segment embeddings (dim 1,024, k = E) and the layer-sensitivity
    reduction at the calibration size N_cal = max(4M, 256) (episodic.hpp:138-140),
    then allocate(sigma, M, 1.1)."""
    rng = np.random.default_rng(3)
    E = c["E"]
    pts = rng.standard_normal((E, 1024))[rng.integers(0, E, 2048)] + 0.7 * rng.standard_normal((2048, 1024))
    epk.kmeans(pts, E, 1)
    t0 = time.perf_counter()
    km = epk.kmeans(pts, E, 1)
    km_ms = (time.perf_counter() - t0) * 1e3
    ncal = max(4 * c["M"], 256)
    g = torch.Generator(device=device).manual_seed(5)
    kf = torch.randn(c["L"], c["H"], ncal, c["d"], device=device, generator=g).bfloat16()
    noise = torch.linspace(0.1, 0.8, c["L"], device=device).view(-1, 1, 1, 1)
    kb = (kf.float() + noise * torch.randn(kf.shape, device=device, generator=g)).bfloat16()
    epk.sensitivity_from_keys(kf, kb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    prof = epk.sensitivity_from_keys(kf, kb)
    e1.record()
    torch.cuda.synchronize()
    alloc = epk.allocate(prof, c["M"], 1.1)
    del kf, kb
    torch.cuda.empty_cache()
    return {"kmeans_2048x1024": {"k": E, "ms": km_ms, "iterations": km.iterations,
                                 "us_per_lloyd_iteration": 1e3 * km_ms / max(1, km.iterations)},
            "sensitivity": {"tokens": ncal, "ms": e0.elapsed_time(e1),
                            "key_bytes": 2 * c["L"] * c["H"] * ncal * c["d"] * 2},
            "allocate_from_measured_sigma": alloc.layer_budgets,
            "bench_layer_budgets": layer_budgets(c)}


def run_e2e(args, c, epk, torch, device, ctx, dist):
    """Chained block steps through the public API with host buffers: each step
    copies the block's K/V and the prompt H2D from pinned memory, appends,
    evicts (score -> select -> compact) and copies the retained positions and
    per-head counts D2H.  The cache stays resident in HBM.  The H2D copies run
    on a copy stream one step ahead (double-buffered device staging), so step
    i+1's inputs cross PCIe while step i computes; every step still copies its
    own inputs and reads back its own result."""
    from paper_2509_17396_b200.step import StepPlan, evict_step
    n_h, live, keep = step_sizes(c)
    L, H, d, p, Hq, B, M = c["L"], c["H"], c["d"], c["p"], c["Hq"], c["block"], c["M"]
    cap = H * (M + B)
    bufs = [epk.EpisodeCache(L, H, d, [cap] * L, torch.bfloat16, device) for _ in range(2)]
    # steady state: M live rows per head, block-sized slack after each head
    for bcache in bufs:
        bcache.head_off.copy_((torch.arange(H + 1, device=device, dtype=torch.int32) * (M + B)).repeat(L, 1))
    bufs[0].head_len.fill_(M)
    bufs[0].k.normal_()
    bufs[0].v.normal_()
    bufs[0].pos.copy_(torch.arange(M + B, device=device, dtype=torch.int32).repeat(L * H))
    g = torch.Generator().manual_seed(7)
    nblk = 2
    host_k = [torch.randn(L, H, B, d, generator=g).to(torch.bfloat16).pin_memory() for _ in range(nblk)]
    host_v = [torch.randn(L, H, B, d, generator=g).to(torch.bfloat16).pin_memory() for _ in range(nblk)]
    host_q = [torch.randn(L, Hq, p, d, generator=g).to(torch.bfloat16).pin_memory() for _ in range(nblk)]
    host_kp = [torch.randn(L, H, p, d, generator=g).to(torch.bfloat16).pin_memory() for _ in range(nblk)]
    dev_k = [torch.empty(L, H, B, d, dtype=torch.bfloat16, device=device) for _ in range(2)]
    dev_v = [torch.empty_like(dev_k[0]) for _ in range(2)]
    dev_q = [torch.empty(L, Hq, p, d, dtype=torch.bfloat16, device=device) for _ in range(2)]
    dev_kp = [torch.empty(L, H, p, d, dtype=torch.bfloat16, device=device) for _ in range(2)]
    dev_pos = torch.empty(B, dtype=torch.int32, device=device)
    out_pos = torch.empty(bufs[0].rows, dtype=torch.int32).pin_memory()
    out_len = torch.empty(L, H, dtype=torch.int32).pin_memory()
    budgets = [M] * L
    plans = [StepPlan(bufs[0], bufs[1], budgets), StepPlan(bufs[1], bufs[0], budgets)]
    start_pos = [M + B]
    comp = torch.cuda.current_stream(device)
    copy_s = torch.cuda.Stream(device)
    ev_copied = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    used = [False, False]

    def issue_copy(i):
        j, h = i % 2, i % nblk
        with torch.cuda.stream(copy_s):
            if used[j]:
                copy_s.wait_event(ev_used[j])  # step i-2 finished reading this staging buffer
            dev_k[j].copy_(host_k[h], non_blocking=True)
            dev_v[j].copy_(host_v[h], non_blocking=True)
            dev_q[j].copy_(host_q[h], non_blocking=True)
            dev_kp[j].copy_(host_kp[h], non_blocking=True)
            ev_copied[j].record(copy_s)

    def one(i):
        cur, j = i % 2, i % 2
        comp.wait_event(ev_copied[j])
        torch.arange(start_pos[0], start_pos[0] + B, out=dev_pos)
        start_pos[0] += B
        epk.append_to_cache(bufs[cur], dev_k[j], dev_v[j], dev_pos, ctx=ctx)
        evict_step(bufs[cur], bufs[1 - cur], dev_q[j], dev_kp[j], budgets, mode="tc_bf16", slack=B,
                   n_max_per_head=n_h, plan=plans[cur], ctx=ctx)
        ev_used[j].record(comp)
        used[j] = True
        out_pos.copy_(bufs[1 - cur].pos, non_blocking=True)
        out_len.copy_(bufs[1 - cur].head_len, non_blocking=True)
        issue_copy(i + 1)  # next step's inputs cross PCIe while this step computes
        comp.synchronize()  # this step's result is on the host

    issue_copy(0)
    nwarm = max(2, min(args.warmup, 4))
    for i in range(nwarm):
        one(i)
    ctx.poll_error()
    steps = max(4, min(args.e2e_steps, args.steps))
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    # device-timed like the kernel-only value: events on the compute stream
    # bracket every step's H2D wait, append + evict step and D2H of its result
    e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_a.record(comp)
    for i in range(nwarm, nwarm + steps):
        one(i)
    e_b.record(comp)
    e_b.synchronize()
    copy_s.synchronize()
    tt = torch.tensor([e_a.elapsed_time(e_b) / 1000.0], device=device, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    world = dist.get_world_size() if dist is not None else 1
    h2d = (dev_k[0].numel() + dev_v[0].numel() + dev_q[0].numel() + dev_kp[0].numel()) * 2 + 0  # positions on device
    d2h = out_pos.numel() * 4 + out_len.numel() * 4
    units = getattr(args, "total_live", None) or world * live  # layer sharding: the episode's units
    return {"value": units * steps / float(tt.item()), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "ms_per_step": 1000.0 * float(tt.item()) / steps,
            "path": "paper_2509_17396_b200.append_to_cache + step.evict_step (C ABI epk_append/epk_evict_step), "
                    "pinned host buffers, H2D of step i+1 overlapped with step i on a copy stream"
                    + ("" if c.get("E", 1) == 1 and not c.get("adaptive") else
                       "; one episode per GPU with uniform budgets M (the config's own per-episode shape)")}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the reference headers compiled in place)
# ---------------------------------------------------------------------------

def ref_layer_inputs(c, layer, layer_seed):
    """One steady-state layer of the same synthetic distribution, fp64
    (bf16-rounded values, as the GPU sees them)."""
    from tests.helpers import bf16_round
    M_l = layer_budgets(c)[layer]
    n_h = M_l + c["block"]
    H, d, p, Hq = c["H"], c["d"], c["p"], c["Hq"]
    rng = np.random.default_rng(layer_seed)
    ho = (np.arange(H + 1) * n_h).astype(np.int64)
    pos = np.tile(np.sort(rng.choice(c["N"], n_h, replace=False)), H).astype(np.int64)
    k = bf16_round(rng.standard_normal((H * n_h, d)).astype(np.float32)).astype(np.float64)
    q = bf16_round(rng.standard_normal((Hq, p, d)).astype(np.float32)).astype(np.float64)
    kp = bf16_round(rng.standard_normal((H, p, d)).astype(np.float32)).astype(np.float64)
    return ho, pos, q, k, kp, M_l


def ref_units(c, units, threads, seed0=1000):
    """Runs the reference CPU path (restated fp64 attention grid ->
    epikv::score_with_prompt -> epikv::evict_to_budget, oracle/_ref = the
    reference headers compiled in place) over `units` = [(layer, seed)] on
    `threads` host threads; returns (tokens, seconds, kind)."""
    from oracle import oracle as O
    kind = "reference"
    try:
        lib = O.ref()
        fn = lib.ref_step_layer_f64
    except Exception:
        kind = "port"
        fn = None
    inputs = [ref_layer_inputs(c, l, seed0 + sd) for l, sd in units]
    tokens = sum(int(x[0][-1]) for x in inputs)

    def work(u):
        ho, pos, q, k, kp, M_l = inputs[u]
        keep = np.zeros(len(pos), np.uint8)
        if fn is not None:
            fn(c["Hq"], c["H"], c["d"], c["p"], M_l, ho, pos, q, k.ctypes.data_as(O.C.c_void_p),
               k.ctypes.data_as(O.C.c_void_p), kp, 1, keep)
        else:
            sc = O.score_layer_f64(q, k, kp, ho, True)
            O.evict_layer(ho, pos, sc, M_l)

    it = iter(range(len(units)))
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                u = next(it, None)
            if u is None:
                return
            work(u)

    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker) for _ in range(max(1, threads))]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return tokens, time.perf_counter() - t0, kind


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(c):
    """The reference CPU path on this box's host cores, bounded: two whole
    steady-state steps (every layer; BASELINE.md section 3 asks for >= 2) on all
    host threads, and a 2-layer sample on one thread."""
    cores = cpu_cores()
    L = c["L"]
    tok_n = sec_n = 0
    for st in range(2):  # one step's inputs in host memory at a time
        tk, sc, kind = ref_units(c, [(l, st * L + l) for l in range(L)], cores)
        tok_n += tk
        sec_n += sc
    tok_1, sec_1, _ = ref_units(c, [(0, 0), (1 % L, 1)], 1)
    return {"value": tok_n / sec_n, "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": cpu_model(),
            "value_1_thread": tok_1 / sec_1,
            "sample": f"{cores} threads: two whole steady-state steps ({L} layers x {c['H']} heads, "
                      f"p={c['p']}) in {sec_n:.1f} s; 1 thread: 2 of {L} layer-steps in {sec_1:.1f} s "
                      "(per-step throughput, the metric's unit; whole runs not timed): restated fp64 attention -> "
                      "epikv::score_with_prompt -> epikv::evict_to_budget (oracle/_ref)"}


def run_reference(args, c, rank, config):
    """--impl reference: the reference's own CPU path on all host threads, K
    timed steps after W warm-up steps.  A step is one steady-state block step
    over every layer when K such steps fit ~3 minutes of host time, else a
    per-step sample of layers (stated in `sample`)."""
    if rank != 0:
        return None
    cores = cpu_cores()
    L, E = c["L"], c.get("E", 1)
    t_unit = None
    for w in range(args.warmup):  # warm-up: one layer-step each (the first one sizes the steps)
        tok, sec, _ = ref_units(c, [(w % L, 500 + w)], 1)
        t_unit = sec if t_unit is None else min(t_unit, sec)
    if t_unit is None:
        tok, t_unit, _ = ref_units(c, [(0, 500)], 1)
    budget_s = 180.0
    whole = L * E
    per_step = whole if args.steps * whole * t_unit / cores <= budget_s else \
        max(1, min(whole, int(budget_s * cores / (args.steps * t_unit))))
    units = [((u % whole) % L, s * whole + u) for s in range(args.steps) for u in range(per_step)]
    tok, sec, kind = ref_units(c, units, cores)
    v = tok / sec
    sample = (f"each of {args.steps} steps: " + (f"one whole block step ({L} layers" + (f" x {E} episodes" if E > 1 else "")
                                                + ")" if per_step == whole else f"{per_step} of {whole} layer-steps")
              + f" ({c['H']} heads x M_l + {c['block']} live entries, p={c['p']}) on {cores} host threads "
              f"({cpu_model()}); restated fp64 attention -> epikv::score_with_prompt -> epikv::evict_to_budget")
    return dict(metric=METRIC, value=v, unit=UNIT, impl="reference", n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=1000.0 * step_sizes(c)[1] * E / v,
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64", data="synthetic",
                config=config,
                cpu_baseline={"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                              "cpu_model": cpu_model()},
                e2e={"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})


# ---------------------------------------------------------------------------

def traffic_from_profiles(kernel):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=40)
    ap.add_argument("--no-batch-episodes", action="store_true",
                    help="several episodes per GPU: one step call per episode instead of one over all")
    ap.add_argument("--no-power-roofline", action="store_true",
                    help="skip the copy / GEMM energy calibration behind the power roofline")
    ap.add_argument("--sustained-steps", type=int, default=1000,
                    help="a second, long timed run of the same step (power-capped clocks); 0 = skip")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-exact", action="store_true", help="skip the precision-matched fp32 step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layer-group", type=int, default=0, help="layers per P2/select/compaction group (0 = all layers)")
    ap.add_argument("--no-overlap", action="store_true", help="compaction on the main stream")
    ap.add_argument("--shard-layers", action="store_true",
                    help="N>1: split ONE episode's layers over the ranks (strong scaling) instead of one episode "
                         "per rank (weak scaling, the default)")
    ap.add_argument("--layers", type=int, default=0, help=argparse.SUPPRESS)  # experiments: override L
    ap.add_argument("--timeline", default=None, help="write one profiled step's kernel timeline to this file")
    args = ap.parse_args()
    c = dict(CONFIGS[args.config])
    if args.layers:  # experiments only: the metric/config of record is the full config
        c["L"] = args.layers

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shard = args.shard_layers and world > 1
    if "E" not in c:
        c["E"] = world if not shard else 1  # weak scaling: one episode per GPU
    config = config_dict(c, c, world, shard)

    if args.impl == "reference":
        res = run_reference(args, dict(c, E=1), rank, config)  # per-step throughput of one episode's step
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    import torch
    dist = None
    # EPK_BENCH_SHARE_GPU=1 (plumbing tests only): ranks share the visible GPUs
    # round-robin and talk over gloo, so the N>1 path runs on a 1-GPU box
    share = os.environ.get("EPK_BENCH_SHARE_GPU") == "1"
    device = torch.device("cuda", local % torch.cuda.device_count() if share else local)
    torch.cuda.set_device(device)
    if world > 1:
        import torch.distributed as td
        if share:
            td.init_process_group("gloo")
        else:
            td.init_process_group("nccl", device_id=device)
        dist = td
    # episodes are the natural shard (round-robin over the ranks,
    # weak scaling); --shard-layers splits one episode's layers instead (strong)
    c_total = c
    if shard:
        l0, l1 = c["L"] * rank // world, c["L"] * (rank + 1) // world
        c = dict(c, L=max(1, l1 - l0))
    args.total_live = step_sizes(c_total)[1] if shard else None
    r = run_ours(args, c, rank, world, device, torch, dist)
    hbm, tc_sus, tc_burst, peak_src = load_peaks()
    n_ep = r["episodes"]
    B1, F1, X1 = algorithmic(c)
    B, F, X = B1 * n_ep, F1 * n_ep, X1 * n_ep  # this GPU's work per step
    ms = r["ms"]
    step_ms = ms / args.steps
    units_all = args.total_live or c_total["E"] * step_sizes(c_total)[1]  # every rank's episodes
    value = units_all * args.steps / (ms / 1000.0)
    kernels = r["kernels"]
    G, p, d, L, H = c["Hq"] // c["H"], c["p"], c["d"], c["L"], c["H"]
    n_h, live, keep = step_sizes(c)
    live, keep = live * n_ep, keep * n_ep
    # per-kernel algorithmic work per step: bound, amount, unit, peak
    sfu_peak = 4.63e12  # measured MUFU.EX2 rate (profiles/mufu_rate_r01.txt)
    work = {
        "p1_rowstats": ("sfu", G * p * (live + L * H * p * n_ep) / 1e12, "Tex2/s", sfu_peak / 1e12),
        "p2_colscore": ("tensor", 2.0 * G * p * d * live / 1e12, "TFLOP/s", tc_burst),
        # gather: K and V rows read + written, positions of the kept rows read + written, every live row's key
        "compact_gather": ("hbm", (4.0 * keep * d * 2 + 8.0 * keep + 4.0 * live) / 1e9, "GB/s", hbm),
        "select": ("hbm", (4.0 * live) / 1e9, "GB/s", hbm),
    }
    for k, (bound, amount, unit, peak) in work.items():
        if k in kernels and kernels[k]["ms_per_step"] > 0:
            ach = amount / (kernels[k]["ms_per_step"] / 1000.0)
            kernels[k].update({"bound": bound, "achieved": ach, "unit": unit, "peak": peak, "frac": ach / peak})
    # dominant kernel: the largest share of the step, whatever unit bounds it
    dom = max((k for k in kernels if k in work), key=lambda k: kernels[k]["ms_per_step"], default=None)
    roof = None
    if dom is not None:
        bound, amount, unit, peak = work[dom]
        nl = kernels[dom]["launches_per_step"]
        kms = kernels[dom]["ms_per_step"] / nl
        amount = amount / nl  # the work of ONE launch (a layer group)
        ach = amount / (kms / 1000.0)
        roof = {"kernel": dom, "bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                "traffic": traffic_from_profiles(dom) if bound == "hbm" else None,
                "peak_source": (f"{peak_src} (MEASURED_PEAKS.json)" if peak_src == "measured"
                                else "fallback (B200_PROFILING.md)") if bound != "sfu"
                else "measured MUFU.EX2 microbenchmark (profiles/mufu_rate_r01.txt)",
                "algorithmic_per_launch": amount * (1e9 if unit == "GB/s" else 1e12), "ms_per_launch": kms}
    step_roof = {"bound": "hbm", "algorithmic_bytes": B, "achieved": B / (step_ms / 1000.0) / 1e9, "peak": hbm,
                 "unit": "GB/s", "frac": B / (step_ms / 1000.0) / 1e9 / hbm,
                 "tensor_flops_single_pass": F, "exps": X,
                 "bound_times_ms": {"hbm": B / hbm / 1e6, "tensor_burst": F / tc_burst / 1e9,
                                    "sfu": X / sfu_peak * 1e3}}
    sus = r["sustained"]
    if sus is not None:
        sus["value"] = units_all / (sus["ms_per_step"] / 1000.0)
        sus["step_roofline_frac"] = B / (sus["ms_per_step"] / 1000.0) / 1e9 / hbm
    # power roofline: the step's algorithmic HBM bytes and its two MMA passes
    # priced at this board's measured energy per copied byte and per GEMM
    # FLOP; at the enforced power limit that energy takes model_ms.  The
    # sustained step runs at the 1 kW cap, so its time is its energy / limit.
    power_roof = None
    ec = r.get("energy_costs")
    if ec and sus is not None and sus["clocks"].get("energy_j_per_step") and sus["clocks"].get("power_limit_w"):
        model_j = B * ec["pj_per_byte"] * 1e-12 + 2.0 * F * ec["pj_per_flop"] * 1e-12
        meas_j = sus["clocks"]["energy_j_per_step"]
        lim = sus["clocks"]["power_limit_w"]
        power_roof = {"bound": "board energy at the power limit", "model_j_per_step": model_j,
                      "measured_j_per_step": meas_j, "frac": model_j / meas_j, "power_limit_w": lim,
                      "model_ms_at_limit": model_j / lim * 1000.0, "sustained_ms_per_step": sus["ms_per_step"],
                      "algorithmic_bytes": B, "tensor_flops_two_passes": 2.0 * F,
                      "pj_per_byte": ec["pj_per_byte"], "pj_per_flop": ec["pj_per_flop"], "how": ec["how"]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(dict(c, E=1))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": config, "score_mode": "tc_bf16", "episodes_per_gpu": n_ep,
            "episodes_batched": r["batched"],
            "roofline": roof, "step_roofline": step_roof, "power_roofline": power_roof, "kernels": kernels, "cpu_baseline": cpu,
            "e2e": r["e2e"], "gpu_launches": r["launches"], "clocks": r["clocks"],
            "sustained": sus, "exact_f32": r["exact"], "phase_a": r["phase_a"],
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
