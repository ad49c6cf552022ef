"""Reference solves for BASELINE config 3 (fibre-reinforced RVE, contrast
1000, FCT against the Jacobi / unpreconditioned baselines).

The reference has no fibre generator, so the same array is fed to both
sides: the documented aligned-fibre field (grid.gen_fibres, FIBRE_PRESET:
24 cylinders along z, r 0.04-0.08, kappa_fib 1000, PCG64 seed 5), built on
the host by the oracle's restatement of the device generator (the GPU tests
check the two are bit-identical).  Also the reference's own orthotropic
channel lattice at psi = 3 (Diag(8, 125, 1000) channels in Diag(0.01, 0.1,
1)).  FCT solves at 128^3 (the largest size the CPU reaches in minutes),
rtol 1e-9 (kappa parity judged at a tight tolerance at
contrast 1000); Jacobi and none at 64^3, rtol 1e-8, reference max_iter 1024.

Imports /root/reference (build container only); writes
tests/golden/solves_config3.json.

    python tests/golden/make_golden_config3.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
import etchomo as E  # noqa: E402

from oracle import etc_oracle as O  # noqa: E402

FIB = dict(count=24, r_min=0.04, r_max=0.08, kappa_fib=1000.0, seed=5, axis="z")

CASES = [
    # kind, n, axis, precond, rtol
    ("fibres", 128, "z", "fct", 1e-9),
    ("fibres", 128, "x", "fct", 1e-9),
    ("channels", 128, "z", "fct", 1e-9),
    ("channels", 128, "y", "fct", 1e-9),
    ("fibres", 64, "z", "fct", 1e-8),
    ("fibres", 64, "z", "jacobi", 1e-8),
    ("fibres", 64, "z", "none", 1e-8),
    ("channels", 64, "z", "fct", 1e-8),
    ("channels", 64, "z", "jacobi", 1e-8),
    ("channels", 64, "z", "none", 1e-8),
]


def field(kind, n):
    if kind == "fibres":
        k = O.fibres(n, FIB["count"], FIB["r_min"], FIB["r_max"], FIB["kappa_fib"], FIB["seed"], FIB["axis"])
        k = np.ascontiguousarray(k).reshape(-1)
        return E.OrthotropicField(E.GridSpec(n, n, n), k, k, k)
    return E.gen_channels(8, n // 8, 3.0)


out = []
for kind, n, ax, pc, rtol in CASES:
    t0 = time.time()
    rep = E.homogenize(field(kind, n), E.BoundaryConfig(E.Axis(ax), 1.0, 0.0), rtol, precond=pc)
    out.append(dict(kind=kind, n=n, axis=ax, precond=pc, rtol=rtol, iterations=rep.iterations,
                    converged=rep.converged, kappa_eff=rep.kappa_eff, history=rep.relative_residuals,
                    refs=rep.ref_params.as_dict(), wall=time.time() - t0,
                    field=(dict(FIB) if kind == "fibres" else dict(cells_per_period=8, periods=n // 8, psi=3.0))))
    print(kind, n, ax, pc, rtol, rep.iterations, rep.converged, repr(rep.kappa_eff), f"{time.time() - t0:.1f}s",
          flush=True)
    (Path(__file__).resolve().parent / "solves_config3.json").write_text(json.dumps(out, indent=1) + "\n")
