"""bench.py's contract pieces that need no GPU: the default line's metric is
BASELINE.json's, both arms report one config dict, the byte model of the
roofline (f64 and the fused f32 solve), and the single-GPU-only f32 option."""
import argparse
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def _args(**kw):
    d = dict(n=512, contrast=100.0, axes="xyz", rtol=1e-6, field="balls", precision="f64")
    d.update(kw)
    return argparse.Namespace(**d)


def test_default_metric_is_baselines():
    base = json.loads((ROOT / "BASELINE.json").read_text())
    assert bench.metric_for(_args()) == bench.METRIC
    assert base["metric"].startswith("PCG time-to-solution") and bench.METRIC.startswith("PCG time-to-solution")
    assert "512" in base["metric"] and "512^3" in bench.METRIC


def test_config_names_the_workload():
    c = bench.bench_config(_args())
    assert "BASELINE config 4" in c["workload"] and "f64" in c["workload"] and "L2" in c["l2"]
    c32 = bench.bench_config(_args(precision="f32"))
    assert "f32" in c32["workload"] and "config 4" not in c32["workload"]
    assert "precision f32" in bench.metric_for(_args(precision="f32"))


def test_byte_model():
    b = bench.bytes_per_cell(True, True)
    assert b == {"stencil": 17, "update_fwd2d": 32, "fwd2d": 16, "zsolve": 16, "inv2d": 24}
    assert bench.bytes_per_cell(True, False)["stencil"] == 40
    b32 = bench.bytes_per_cell(True, True, 4)
    assert b32["stencil"] == 9 and b32["update_fwd2d"] == 16 and b32["zsolve"] == 8 and b32["inv2d"] == 12
    assert sum(b[k] for k in ("stencil", "update_fwd2d", "zsolve", "inv2d")) == 89


def test_f32_is_single_gpu(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py", "--precision", "f32", "--slab"])
    with pytest.raises(SystemExit, match="single-GPU"):
        bench.main()
