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
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def step_sizes(c):
    n_h = c["M"] + c["block"]
    live = c["L"] * c["H"] * n_h
    keep = c["L"] * c["H"] * c["M"]
    return n_h, live, keep


def algorithmic(c):
    """bytes / flops / exps per step (bf16)."""
    n_h, live, keep = step_sizes(c)
    d, G, p = c["d"], c["Hq"] // c["H"], c["p"]
    B = live * d * 2 + c["L"] * (c["Hq"] + c["H"]) * p * d * 2 + 4 * keep * d * 2 + 4 * live + 4 * keep
    F = 2 * p * d * G * live
    X = p * G * live
    return B, F, X


def make_inputs(epk, torch, c, R, device, seed):
    """R steady-state input caches (n_h = M + block live rows per head, dense)
    and R prompt sets, bf16, resident in HBM."""
    n_h, live, keep = step_sizes(c)
    L, H, d, p, Hq = c["L"], c["H"], c["d"], c["p"], c["Hq"]
    cap = H * n_h
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    caches, qs, kps = [], [], []
    pos_head = torch.sort(torch.randperm(c["N"], device=device, generator=g)[:n_h])[0].to(torch.int32)
    for r in range(R):
        cc = epk.EpisodeCache(L, H, d, [cap] * L, torch.bfloat16, device)
        cc.k.copy_(torch.randn(cc.rows, d, device=device, generator=g, dtype=torch.float32).to(torch.bfloat16))
        cc.v.copy_(torch.randn(cc.rows, d, device=device, generator=g, dtype=torch.float32).to(torch.bfloat16))
        cc.pos.copy_(pos_head.repeat(L * H))
        off = (torch.arange(H + 1, device=device, dtype=torch.int32) * n_h).repeat(L, 1)
        cc.head_off.copy_(off)
        cc.head_len.fill_(n_h)
        caches.append(cc)
        qs.append(torch.randn(L, Hq, p, d, device=device, generator=g).to(torch.bfloat16))
        kps.append(torch.randn(L, H, p, d, device=device, generator=g).to(torch.bfloat16))
    out = epk.EpisodeCache(L, H, d, [cap] * L, torch.bfloat16, device)
    return caches, qs, kps, out


def run_ours(args, c, rank, world, device, torch, dist):
    import paper_2509_17396_b200 as epk
    from paper_2509_17396_b200.step import StepPlan, evict_step

    ctx = epk.default_context(device.index)
    ctx.set_option(layer_group=args.layer_group, overlap=not args.no_overlap)
    n_h, live, keep = step_sizes(c)
    R = 3
    caches, qs, kps, out = make_inputs(epk, torch, c, R, device, 1234 + rank)
    budgets = [c["M"]] * c["L"]
    plans = [StepPlan(caches[r], out, budgets) for r in range(R)]

    def step(i):
        r = i % R
        evict_step(caches[r], out, qs[r], kps[r], budgets, mode="tc_bf16", slack=c["block"], n_max_per_head=n_h,
                   plan=plans[r], ctx=ctx)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    ctx.poll_error()
    stream = torch.cuda.current_stream(device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(device.index)
    clocks.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    ev0.record(stream)
    for i in range(args.steps):
        step(i)
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    launches = ctx.launches - launches0
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device=device, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ctx.poll_error()

    # per-kernel live timing: a separate pass with events around every launch
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
    e2e = run_e2e(args, c, epk, torch, device, ctx, dist) if not args.no_e2e else None
    return dict(ms=ms_max, launches=launches, clocks=clk, kernels=kernels, e2e=e2e, live=live, keep=keep)


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
                    "pinned host buffers, H2D of step i+1 overlapped with step i on a copy stream"}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the reference headers compiled in place)
# ---------------------------------------------------------------------------

def ref_layer_inputs(c, layer_seed):
    """One steady-state layer of the same synthetic distribution, fp64
    (bf16-rounded values, as the GPU sees them)."""
    from tests.helpers import bf16_round
    n_h, _, _ = step_sizes(c)
    H, d, p, Hq = c["H"], c["d"], c["p"], c["Hq"]
    rng = np.random.default_rng(layer_seed)
    ho = (np.arange(H + 1) * n_h).astype(np.int64)
    pos = np.tile(np.sort(rng.choice(c["N"], n_h, replace=False)), H).astype(np.int64)
    k = bf16_round(rng.standard_normal((H * n_h, d)).astype(np.float32)).astype(np.float64)
    q = bf16_round(rng.standard_normal((Hq, p, d)).astype(np.float32)).astype(np.float64)
    kp = bf16_round(rng.standard_normal((H, p, d)).astype(np.float32)).astype(np.float64)
    return ho, pos, q, k, kp


def ref_sample(c, units, threads):
    """Runs `units` layer-steps of the reference CPU path (restated attention
    grid -> epikv::score_with_prompt -> epikv::evict_to_budget) on `threads`
    host threads; returns (tokens, seconds, kind)."""
    from oracle import oracle as O
    kind = "reference"
    try:
        lib = O.ref()
        fn = lib.ref_step_layer_f64
    except Exception:
        kind = "port"
        fn = None
    inputs = [ref_layer_inputs(c, 1000 + u) for u in range(units)]
    n_h, _, _ = step_sizes(c)
    tokens = units * c["H"] * n_h
    results = [None] * units

    def work(u):
        ho, pos, q, k, kp = inputs[u]
        keep = np.zeros(len(pos), np.uint8)
        if fn is not None:
            rc = fn(c["Hq"], c["H"], c["d"], c["p"], c["M"], ho, pos, q, k.ctypes.data_as(O.C.c_void_p),
                    k.ctypes.data_as(O.C.c_void_p), kp, 1, keep)
            results[u] = int(rc)
        else:
            s = O.score_layer_f64(q, k, kp, ho, True)
            results[u] = O.evict_layer(ho, pos, s, c["M"])[0]

    t0 = time.perf_counter()
    ths = []
    it = iter(range(units))
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                u = next(it, None)
            if u is None:
                return
            work(u)

    for _ in range(threads):
        th = threading.Thread(target=worker)
        th.start()
        ths.append(th)
    for th in ths:
        th.join()
    return tokens, time.perf_counter() - t0, kind


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, c, rank):
    if rank != 0:
        return None
    cores = cpu_cores()
    units = min(c["L"], cores)
    for _ in range(min(args.warmup, 1)):
        ref_sample(c, min(units, 2), min(units, 2))
    steps = max(1, min(args.steps, 3))
    rates = []
    kind = "reference"
    for _ in range(steps):
        tok, sec, kind = ref_sample(c, units, units)
        rates.append(tok / sec)
    v = float(np.median(rates))
    sample = (f"{units} of {c['L']} layers of one steady-state cfg block step ({c['H']} heads x "
              f"{c['M'] + c['block']} live entries each, p={c['p']}), one layer per host thread, "
              f"{steps} step(s); attention restated in fp64 -> epikv::score_with_prompt -> epikv::evict_to_budget")
    return dict(metric=METRIC, value=v, unit=UNIT, impl="reference", n_gpus=args.gpus, steps=steps,
                warmup=min(args.warmup, 1), ms_per_step=1000.0 * c["L"] * c["H"] * (c["M"] + c["block"]) / v,
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64", data="synthetic",
                config={"workload": c["desc"], "layers": c["L"], "q_heads": c["Hq"], "kv_heads": c["H"],
                        "head_dim": c["d"], "block": c["block"], "budget_per_head": c["M"], "prompt_len": c["p"]},
                cpu_baseline={"value": v, "unit": UNIT, "cores": units, "kind": kind, "sample": sample},
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
    ap.add_argument("--no-e2e", action="store_true")
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

    if args.impl == "reference":
        res = run_reference(args, c, rank)
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
    # episodes are the natural shard (one per rank, weak scaling);
    # --shard-layers splits one episode's layers instead (strong scaling)
    shard = args.shard_layers and world > 1
    c_total = c
    if shard:
        l0, l1 = c["L"] * rank // world, c["L"] * (rank + 1) // world
        c = dict(c, L=max(1, l1 - l0))
    args.total_live = step_sizes(c_total)[1] if shard else None
    r = run_ours(args, c, rank, world, device, torch, dist)
    hbm, tc_sus, tc_burst, peak_src = load_peaks()
    B, F, X = algorithmic(c)  # per GPU
    ms = r["ms"]
    step_ms = ms / args.steps
    value = (args.total_live or world * r["live"]) * args.steps / (ms / 1000.0)
    # dominant kernel (largest share of the step) and its roofline
    kernels = r["kernels"]
    G, p, d, L, H = c["Hq"] // c["H"], c["p"], c["d"], c["L"], c["H"]
    n_h, live, keep = step_sizes(c)
    # per-kernel algorithmic work per step: bound, amount, unit, peak
    sfu_peak = 4.63e12  # measured MUFU.EX2 rate (profiles/mufu_rate_r01.txt)
    work = {
        "p1_rowstats": ("sfu", G * p * (live + L * H * p) / 1e12, "Tex2/s", sfu_peak / 1e12),
        "p2_colscore": ("tensor", 2.0 * G * p * d * live / 1e12, "TFLOP/s", tc_sus),
        "compact_gather": ("hbm", (4.0 * keep * d * 2 + 8.0 * keep + live) / 1e9, "GB/s", hbm),
        "select": ("hbm", (4.0 * live) / 1e9, "GB/s", hbm),
        "compact_count": ("hbm", (4.0 * live + live) / 1e9, "GB/s", hbm),
    }
    for k, (bound, amount, unit, peak) in work.items():
        if k in kernels and kernels[k]["ms_per_step"] > 0:
            ach = amount / (kernels[k]["ms_per_step"] / 1000.0)
            kernels[k].update({"bound": bound, "achieved": ach, "unit": unit, "peak": peak, "frac": ach / peak})
    dom = max((k for k in kernels if k in work and work[k][0] in ("hbm", "tensor")),
              key=lambda k: kernels[k]["ms_per_step"], default=None)
    roof = None
    if dom is not None:
        bound, amount, unit, peak = work[dom]
        nl = kernels[dom]["launches_per_step"]
        kms = kernels[dom]["ms_per_step"] / nl
        amount = amount / nl  # the work of ONE launch (a layer group)
        ach = amount / (kms / 1000.0)
        roof = {"kernel": dom, "bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                "traffic": traffic_from_profiles(dom), "peak_source": f"{peak_src} (MEASURED_PEAKS.json)"
                if peak_src == "measured" else "fallback (B200_PROFILING.md)",
                "algorithmic_per_launch": amount * (1e9 if unit == "GB/s" else 1e12), "ms_per_launch": kms}
    step_roof = {"bound": "hbm", "algorithmic_bytes": B, "achieved": B / (step_ms / 1000.0) / 1e9, "peak": hbm,
                 "unit": "GB/s", "frac": B / (step_ms / 1000.0) / 1e9 / hbm,
                 "tensor_flops_single_pass": F, "exps": X,
                 "bound_times_ms": {"hbm": B / hbm / 1e6, "tensor": F / tc_sus / 1e9}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        units = min(4, L)
        tok, sec, kind = ref_sample(c, units, units)
        cpu = {"value": tok / sec, "unit": UNIT, "cores": units, "kind": kind,
               "sample": f"{units} layer-steps of the cfg shape ({H} heads x {n_h} live entries, p={p}), "
                         f"one per host thread: fp64 attention restatement -> epikv::score_with_prompt -> "
                         f"epikv::evict_to_budget (oracle/_ref)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": c["desc"], "layers": c_total["L"], "q_heads": c["Hq"], "kv_heads": H, "head_dim": d,
                       "context": c["N"], "block": c["block"], "budget_per_head": c["M"], "prompt_len": p,
                       "live_entries_per_step": step_sizes(c_total)[1], "kept_per_step": step_sizes(c_total)[2],
                       "score_mode": "tc_bf16", "aggregation": "max",
                       "episodes_per_gpu": 1 if not shard else 1.0 / world,
                       "parallelism": f"layers x{world} (one episode)" if shard else f"episodes x{world}",
                       "l2": "inputs larger than L2: 3 rotating steady-state caches of "
                             f"{2 * live * d * 2 / 1e9:.2f} GB K+V each"},
            "roofline": roof, "step_roofline": step_roof, "kernels": kernels, "cpu_baseline": cpu,
            "e2e": r["e2e"], "gpu_launches": r["launches"], "clocks": r["clocks"],
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
