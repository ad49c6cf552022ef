"""Reference homogenize() runs with the SSOR preconditioner tag
(pipeline.py:114-132, preconditioner.py:285-321) for the device SSOR sweeps.
Imports /root/reference (build container only); writes
tests/golden/solves_ssor.json.

    python tests/golden/make_golden_ssor.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import etchomo as E  # noqa: E402

CASES = [(16, 10.0, "z", "ssor", 1e-8), (16, 100.0, "x", "ssor:1.5", 1e-8), (24, 100.0, "y", "ssor:0.8", 1e-7),
         (20, 1000.0, "z", "ssor:1.2", 1e-6)]
out = []
for n, C, ax, tag, rtol in CASES:
    f = E.gen_random_balls(n, 40, 0.05, 0.15, C, 11)
    rep = E.homogenize(f, E.BoundaryConfig(E.Axis(ax), 1.0, 0.0), rtol, precond=tag)
    out.append(dict(n=n, kappa=C, axis=ax, precond=tag, rtol=rtol, iterations=rep.iterations,
                    converged=rep.converged, kappa_eff=rep.kappa_eff, history=rep.relative_residuals,
                    preconditioner=rep.preconditioner))
    print(n, C, ax, tag, rep.iterations, repr(rep.kappa_eff), rep.preconditioner, flush=True)
(Path(__file__).resolve().parent / "solves_ssor.json").write_text(json.dumps(out, indent=1) + "\n")
