"""bench.py host logic that needs no GPU: the roofline peak taken from the
driver-written MEASURED_PEAKS.json (any of its HBM spellings), else the
documented fallback."""
from __future__ import annotations

import json

import bench


def test_peak_fallback_and_measured_spellings(tmp_path, monkeypatch):
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    assert bench.peaks() == (6650.0, "fallback")
    for doc, want in (({"hbm_gbs": 6549.8, "bf16_tflops": 2100.0}, 6549.8),
                      ({"hbm": {"sustained_gbs": 6400.0, "burst_gbs": 7100.0}}, 7100.0),
                      ({"hbm_copy_gbs": 6600.0}, 6600.0)):
        (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps(doc))
        assert bench.peaks() == (want, "measured")
    (tmp_path / "MEASURED_PEAKS.json").write_text("not json")
    assert bench.peaks() == (6650.0, "fallback")
