"""bench.py host helpers (no GPU): the MEASURED_PEAKS.json reader and the
algorithmic byte / flop / exp counts of SURVEY 8(d)."""
import json
import os

import pytest

import bench


def test_peaks_fallback_and_parsing(tmp_path, monkeypatch):
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    assert bench.load_peaks() == (6650.0, 1400.0, 1590.0, "fallback")
    for doc in ({"hbm_copy_gbs": 6550.0, "bf16_dense_tflops": {"burst": 1641.0, "sustained": 1407.0}},
                {"hbm_tbs": 6.55, "bf16_tflops_sustained": 1407.0, "bf16_tflops": 1641.0}):
        with open(os.path.join(tmp_path, "MEASURED_PEAKS.json"), "w") as f:
            json.dump(doc, f)
        assert bench.load_peaks() == (6550.0, 1407.0, 1641.0, "measured")
    with open(os.path.join(tmp_path, "MEASURED_PEAKS.json"), "w") as f:
        f.write("{not json")
    assert bench.load_peaks()[3] == "fallback"


def test_algorithmic_counts_cfg2():
    B, F, X = bench.algorithmic(bench.CONFIGS["cfg2"])
    assert B == 2512125952  # 2.512 GB per cfg2 step
    assert F == pytest.approx(225.5e9, rel=1e-3) and X == pytest.approx(881e6, rel=1e-3)
    n_h, live, keep = bench.step_sizes(bench.CONFIGS["cfg2"])
    assert (n_h, live, keep) == (10240, 2293760, 1835008)


def test_cfg3_adaptive_budgets_and_config_dicts():
    """cfg3's adaptive budgets are allocate(sigma, 8192, 1.1) on the shared
    synthetic profile -- Sigma M_l = L * M exactly -- and both arms print the
    same config dict."""
    c3 = dict(bench.CONFIGS["cfg3"])
    bud = bench.layer_budgets(c3)
    assert len(bud) == 28 and sum(bud) == 28 * 8192 and len(set(bud)) > 1 and min(bud) >= 1
    n_h, live, keep = bench.step_sizes(c3)
    assert keep == 8 * 28 * 8192 and live == keep + 28 * 8 * 2048 and n_h == max(bud) + 2048
    a = bench.config_dict(c3, c3, 1, False)
    assert a == bench.config_dict(dict(c3), dict(c3), 1, False) and a["layer_budgets"] == "adaptive"
    assert bench.cpu_model()


def test_reference_arm_sizes_steps(monkeypatch):
    """The reference arm keeps the driver's --steps / --warmup and shrinks each
    step to a layer sample only when whole steps would not fit ~3 minutes."""
    calls = []

    def fake_units(c, units, threads, seed0=1000):
        calls.append((len(units), threads))
        return 81920 * len(units), 3.4 * len(units) / threads, "reference"

    monkeypatch.setattr(bench, "ref_units", fake_units)
    monkeypatch.setattr(bench, "cpu_cores", lambda: 16)

    class A:
        steps, warmup, gpus = 20, 5, 1

    c = dict(bench.CONFIGS["cfg2"], E=1)
    res = bench.run_reference(A, c, 0, bench.config_dict(c, c, 1, False))
    assert res["steps"] == 20 and res["warmup"] == 5 and res["impl"] == "reference"
    assert calls[-1][0] == 20 * 28  # whole steps fit: 20 x 28 layer-steps
    A.steps = 1000
    res = bench.run_reference(A, c, 0, bench.config_dict(c, c, 1, False))
    assert res["steps"] == 1000 and calls[-1][0] < 1000 * 28 and "layer-steps" in res["cpu_baseline"]["sample"]
