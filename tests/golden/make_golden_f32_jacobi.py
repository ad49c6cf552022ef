"""Reference single-precision solves with the Jacobi and SSOR preconditioners
(homogenize(..., precond=..., precision="f32"), pipeline.py:135-175 with
preconditioner.py:324-329 / the SSOR sweeps), and the float64 solve of the
same problem.  Imports /root/reference (build container only); writes
tests/golden/solves_f32_jacobi.json.

    python tests/golden/make_golden_f32_jacobi.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import etchomo as E  # noqa: E402

CASES = [
    # kind, n, contrast, axis, rtol, precond
    ("random-a", 32, 100.0, "z", 1e-5, "jacobi"),
    ("random-a", 24, 10.0, "x", 1e-6, "jacobi"),
    ("center-ball", 20, 100.0, "y", 1e-5, "jacobi"),
    ("random-a", 16, 10.0, "z", 1e-5, "ssor:1.5"),
]

pr = E.RANDOM_BALL_PRESETS["a"]
out = []
for kind, n, c, ax, rtol, pc in CASES:
    if kind == "random-a":
        field = E.gen_random_balls(n, pr["count"], pr["r_min"], pr["r_max"], c, pr["seed"])
    else:
        field = E.gen_center_ball(n, c)
    bc = E.BoundaryConfig(E.Axis(ax), 1.0, 0.0)
    rep = E.homogenize(field, bc, rtol, precond=pc, precision="f32")
    r64 = E.homogenize(field, bc, rtol, precond=pc, precision="f64")
    out.append(dict(kind=kind, n=n, kappa=c, axis=ax, rtol=rtol, precond=pc, iterations=rep.iterations,
                    converged=rep.converged, kappa_eff=rep.kappa_eff, history=rep.relative_residuals,
                    precision=rep.precision, refs=None, f64_iterations=r64.iterations, f64_kappa_eff=r64.kappa_eff))
    print(kind, n, c, ax, rtol, pc, rep.iterations, repr(rep.kappa_eff), r64.iterations, repr(r64.kappa_eff),
          flush=True)
(Path(__file__).resolve().parent / "solves_f32_jacobi.json").write_text(json.dumps(out, indent=1) + "\n")
