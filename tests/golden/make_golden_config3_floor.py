"""Rounding floor of the config-3 cases: at contrast 1000
finite-precision CG makes valid float64 implementations drift apart below
relres ~1e-2, so GPU-vs-reference is judged against the spread of two other
CPU implementations of the same algorithm: the oracle (numpy/pocketfft
association) and the perturbed oracle (reversed stencil association,
bottom-up z elimination, exactly rounded dots).  Writes
tests/golden/solves_config3_floor.json (iterations, kappa_eff, history of
both per case of solves_config3.json).  CPU only (no reference import).

    python tests/golden/make_golden_config3_floor.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import etc_oracle as O  # noqa: E402

HERE = Path(__file__).resolve().parent
cases = json.loads((HERE / "solves_config3.json").read_text())
out = []
for c in cases:
    n = c["n"]
    if c["kind"] == "fibres":
        fd = c["field"]
        k = O.fibres(n, fd["count"], fd["r_min"], fd["r_max"], fd["kappa_fib"], fd["seed"], fd["axis"])
        kx = ky = kz = k
    else:
        kx, ky, kz = O.channels(8, n // 8, 3.0)
    row = dict(kind=c["kind"], n=n, axis=c["axis"], precond=c["precond"], rtol=c["rtol"])
    for tag, pert in (("oracle", False), ("perturbed", True)):
        t0 = time.time()
        r = O.homogenize(kx, ky, kz, (n, n, n, 1.0, 1.0, 1.0), c["axis"], 1.0, 0.0, c["rtol"], workers=8,
                         perturbed=pert, precond=c["precond"])
        row[tag] = dict(iterations=r["iterations"], converged=bool(r["converged"]), kappa_eff=r["kappa_eff"],
                        history=r["history"])
        print(c["kind"], n, c["axis"], c["precond"], tag, r["iterations"], c["iterations"],
              f"{abs(r['kappa_eff'] - c['kappa_eff']) / c['kappa_eff']:.2e}", f"{time.time() - t0:.1f}s", flush=True)
    out.append(row)
    (HERE / "solves_config3_floor.json").write_text(json.dumps(out) + "\n")
