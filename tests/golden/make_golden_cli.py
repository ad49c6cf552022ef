"""The reference CLI's artifacts for `etc solve tests/golden/ball8.vox
--rtol 1e-8` (cli.py:165-186; report schema pipeline.py:250-295).  Imports
/root/reference (build container only).

    python tests/golden/make_golden_cli.py
"""
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from etchomo.cli import main  # noqa: E402

here = Path(__file__).resolve().parent
rc = main(["solve", str(here / "ball8.vox"), "--rtol", "1e-8", "--axis", "x", "--report",
           str(here / "cli_ball8_report.json"), "--history", str(here / "cli_ball8_history.csv")])
print("rc", rc)
