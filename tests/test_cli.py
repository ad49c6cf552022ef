"""`etc generate` / `etc solve` on the GPU backend:
the reference CLI's flags, report schema, residual CSV and exit codes
(cli.py:165-186, 300-323; pipeline.py:250-295).  CPU tests cover parsing,
the error paths and the report document; the gpu ones solve a
reference-written file and compare with the reference CLI's own artifacts
(tests/golden/cli_ball8_*, make_golden_cli.py)."""

import csv
import json
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2404_02433_b200.cli import main, report_to_dict  # noqa: E402
from paper_2404_02433_b200.grid import Axis, BoundaryConfig, GridSpec  # noqa: E402
from paper_2404_02433_b200.reference import ReferenceParams  # noqa: E402

GOLD = Path(__file__).parent / "golden"


def test_usage_and_file_errors(tmp_path):
    assert main(["solve", str(GOLD / "ball8.vox"), "--frobnicate"]) == 2
    assert main(["frobnicate"]) == 2
    assert main(["solve", str(tmp_path / "missing.vox")]) == 3
    bad = tmp_path / "bad.vox"
    bad.write_bytes(b"NOTAVOX!" + (GOLD / "ball8.vox").read_bytes()[8:])
    assert main(["solve", str(bad)]) == 3


def test_report_document_matches_reference_schema():
    ref = json.loads((GOLD / "cli_ball8_report.json").read_text())
    rp = ReferenceParams(*[ref["ref_params"][k] for k in ("kx", "ky", "kz", "kin", "kout", "lambda_lo",
                                                           "lambda_hi")])
    rep = SimpleNamespace(preconditioner="fct", ref_params=rp, iterations=10, converged=True,
                          kappa_eff=1.0, prep_seconds=0.0, exec_seconds=0.0, precision="f64", l2_error=None)
    doc = report_to_dict(rep, {"input": "x"}, GridSpec(8, 8, 8), BoundaryConfig(Axis("x"), 1.0, 0.0), 1e-8)
    assert set(doc) == set(ref)
    assert set(doc["grid"]) == set(ref["grid"]) and set(doc["boundary"]) == set(ref["boundary"])
    assert set(doc["ref_params"]) == set(ref["ref_params"])


@pytest.mark.gpu
def test_solve_matches_reference_cli(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rep_path, hist_path = tmp_path / "r.json", tmp_path / "h.csv"
    rc = main(["solve", str(GOLD / "ball8.vox"), "--rtol", "1e-8", "--axis", "x", "--report", str(rep_path),
               "--history", str(hist_path)])
    assert rc == 0
    got, want = json.loads(rep_path.read_text()), json.loads((GOLD / "cli_ball8_report.json").read_text())
    for key in ("boundary", "grid", "precision", "precond", "rtol", "converged", "iterations"):
        assert got[key] == want[key], key
    assert got["ref_params"] == pytest.approx(want["ref_params"], rel=1e-15)
    assert abs(got["kappa_eff"] - want["kappa_eff"]) <= 1e-8 * want["kappa_eff"]
    h = np.array([float(r["relres"]) for r in csv.DictReader(open(hist_path))])
    w = np.array([float(r["relres"]) for r in csv.DictReader(open(GOLD / "cli_ball8_history.csv"))])
    big = w > 1e-2  # 1e-8 while relres > 1e-2
    assert len(h) == len(w) and np.all(np.abs(h[big] - w[big]) <= 1e-8 * w[big])
    # SSOR runs through the plugin composition (exit 0); a configuration
    # error maps to exit 2 (cli.py:309-323)
    assert main(["solve", str(GOLD / "ball8.vox"), "--precond", "ssor", "--omega", "1.2"]) == 0
    assert main(["solve", str(GOLD / "ball8.vox"), "--precond", "ssor", "--omega", "2.5"]) == 2


@pytest.mark.gpu
def test_generate_round_trip(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "c.vox"
    assert main(["generate", "--config", "center-ball", "--n", "8", "--kappa-inc", "10", "-o", str(out)]) == 0
    assert out.read_bytes() == (GOLD / "ball8.vox").read_bytes()
