"""Reference solves with the Jacobi and identity preconditioners
(precond="jacobi" | "none", pipeline.py:114-132; preconditioner.py:324-338),
the SURVEY 8(f) row-1 baselines.  Unpreconditioned CG runs hundreds of
iterations and its kappa_eff at a loose rtol is rounding-sensitive (the
perturbed oracle moves it by up to 1e-5), so the "none" cases are run to a
tight rtol where kappa_eff is converged.  Imports /root/reference (build container
only); writes tests/golden/solves_precond.json.

    python tests/golden/make_golden_precond.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import etchomo as E  # noqa: E402

CASES = [
    # kind, n, contrast, axis, rtol, precond
    ("random-a", 16, 100.0, "z", 1e-6, "jacobi"),
    ("random-a", 16, 100.0, "z", 1e-10, "none"),
    ("random-a", 24, 10.0, "x", 1e-8, "jacobi"),
    ("random-a", 24, 10.0, "y", 1e-10, "none"),
    ("random-a", 32, 1000.0, "z", 1e-6, "jacobi"),
    ("center-ball", 16, 0.01, "z", 1e-7, "jacobi"),
    ("center-ball", 20, 1000.0, "x", 1e-9, "none"),
]

pr = E.RANDOM_BALL_PRESETS["a"]
out = []
for kind, n, c, ax, rtol, pc in CASES:
    if kind == "random-a":
        field = E.gen_random_balls(n, pr["count"], pr["r_min"], pr["r_max"], c, pr["seed"])
    else:
        field = E.gen_center_ball(n, c)
    rep = E.homogenize(field, E.BoundaryConfig(E.Axis(ax), 1.0, 0.0), rtol, precond=pc)
    out.append(dict(kind=kind, n=n, kappa=c, axis=ax, rtol=rtol, precond=pc, iterations=rep.iterations,
                    converged=rep.converged, kappa_eff=rep.kappa_eff, history=rep.relative_residuals,
                    preconditioner=rep.preconditioner))
    print(kind, n, c, ax, rtol, pc, rep.iterations, repr(rep.kappa_eff), flush=True)
path = Path(__file__).resolve().parent / "solves_precond.json"
path.write_text(json.dumps(out, indent=1) + "\n")
