"""ETCVOX01 files written by the reference (write_vox, grid.py:322-332):
center ball 8^3 contrast 10 in f64 and f32.  Imports /root/reference
(build container only).

    python tests/golden/make_golden_vox.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import etchomo as E  # noqa: E402

here = Path(__file__).resolve().parent
f = E.gen_center_ball(8, 10.0)
E.write_vox(f, here / "ball8.vox")
E.write_vox(f.astype(np.float32), here / "ball8_f32.vox")
