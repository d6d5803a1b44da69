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
