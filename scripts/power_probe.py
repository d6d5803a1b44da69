"""Power / clock / energy of the cfg2 step and of its parts (NVML), on the box.

Each mode runs back to back for ~SECS seconds on the same resident inputs
(three rotating caches, as bench.py):
  step    epk_evict_step (P1 -> bias -> P2 -> threshold select -> gather)
  score   epk_score (P1 -> bias -> P2 only)
  gather  epk_compact with a fixed keep mask (79 % kept: count -> plan -> gather)
  copy    torch b.copy_(a), 1 Gi bf16 (2 GiB of HBM traffic): board pJ per byte moved
  gemm    torch.matmul bf16 8192^3: board pJ per FLOP
and reports ms per iteration, mean board power, energy per iteration (NVML
total-energy counter), median SM clock and the throttle reasons seen.
Usage: python scripts/power_probe.py [modes...]"""
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pynvml  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_17396_b200 as epk  # noqa: E402
from paper_2509_17396_b200.step import StepPlan, evict_step  # noqa: E402

SECS = float(os.environ.get("SECS", "3"))
REASONS = {
    "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
    "hw_power_brake_slowdown": 0x80,
}


def main(modes):
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    c = dict(bench.CONFIGS["cfg2"])
    if os.environ.get("PROBE_LAYERS"):  # e.g. 4: one step's K (84 MB) stays in L2 between P1 and P2
        c["L"] = int(os.environ["PROBE_LAYERS"])
    dev = torch.device("cuda:0")
    ctx = epk.default_context(0)
    n_h, live, keep_n = bench.step_sizes(c)
    caches, qs, kps, out = bench.make_inputs(epk, torch, c, 3, dev, 1234)
    budgets = bench.layer_budgets(c)
    plans = [StepPlan(caches[r], out, budgets) for r in range(3)]
    scores = torch.empty(caches[0].rows, dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev).manual_seed(7)
    keeps = []
    for r in range(3):  # 79 % of the live rows (the output layers hold 80 % + slack); keep[] must be 0 on gap rows
        live_mask = torch.zeros(caches[r].rows, dtype=torch.bool, device=dev)
        for l in range(caches[r].layers):
            live_mask[caches[r].live_rows(l)] = True
        keeps.append(((torch.rand(caches[r].rows, generator=g, device=dev) < 0.79) & live_mask).to(torch.uint8))

    ca = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev).normal_() if "copy" in modes else None
    cb = torch.empty_like(ca) if ca is not None else None
    ga = torch.randn(8192, 8192, dtype=torch.bfloat16, device=dev) if "gemm" in modes else None
    gb = torch.randn(8192, 8192, dtype=torch.bfloat16, device=dev) if "gemm" in modes else None
    work = {"copy": ("pj_per_byte", 2.0 * (1 << 31)), "gemm": ("pj_per_flop", 2.0 * 8192 ** 3)}

    def run(mode, i):
        r = i % 3
        if mode == "copy":
            cb.copy_(ca)
            return
        if mode == "gemm":
            torch.matmul(ga, gb)
            return
        if mode == "step":
            evict_step(caches[r], out, qs[r], kps[r], budgets, mode="tc_bf16", slack=c["block"], n_max_per_head=n_h,
                       plan=plans[r], ctx=ctx)
        elif mode == "score":
            epk.score_with_prompt(caches[r], qs[r], kps[r], n_max_per_head=n_h, out=scores, ctx=ctx)
        elif mode == "gather":
            epk.compact(caches[r], keeps[r], out, slack=c["block"], ctx=ctx)

    res = {}
    for mode in modes:
        for i in range(10):
            run(mode, i)
        torch.cuda.synchronize()
        # calibrate the iteration count to ~SECS seconds
        t = time.time()
        for i in range(20):
            run(mode, i)
        torch.cuda.synchronize()
        per = (time.time() - t) / 20
        n = max(20, int(SECS / per))
        samples = []
        stop = threading.Event()

        def sampler():
            while not stop.is_set():
                try:
                    samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
                except pynvml.NVMLError:
                    pass
                time.sleep(0.02)

        th = threading.Thread(target=sampler, daemon=True)
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        th.start()
        ev0.record(torch.cuda.current_stream())
        t0 = time.time()
        for i in range(n):
            run(mode, i)
        ev1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        t1 = time.time()
        e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        stop.set()
        th.join()
        ms = ev0.elapsed_time(ev1) / n
        clocks = sorted(s[0] for s in samples[len(samples) // 4:]) or [0]
        watts = [s[1] for s in samples[len(samples) // 4:]] or [0]
        reasons = sorted({k for s in samples for k, b in REASONS.items() if s[2] & b})
        res[mode] = dict(layers=c["L"], iters=n, ms_per_iter=round(ms, 4), wall_s=round(t1 - t0, 2),
                         energy_mj_per_iter=round((e1 - e0) / n, 3), mean_w=round(sum(watts) / len(watts), 1),
                         sm_mhz_median=clocks[len(clocks) // 2], sm_mhz_min=clocks[0], reasons=reasons)
        if mode in work:
            res[mode][work[mode][0]] = round((e1 - e0) / n * 1e9 / work[mode][1], 3)
            res[mode]["rate_per_s"] = work[mode][1] / (ms / 1000.0)
        ctx.poll_error()  # a flagged (skipped) layer would make the timing meaningless
        print(mode, json.dumps(res[mode]), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1:] or ["step", "score", "gather"])
