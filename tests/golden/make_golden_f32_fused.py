"""Reference single-precision solves on grids the fused float32 path takes
(square power-of-two planes N >= 128, nz = 32 L with L in {4, 8, 16}):
homogenize(..., precision="f32") of the reference (pipeline.py:147-160) on a
two-phase field (random-ball preset a), a centre ball, an orthotropic channel
lattice (few anisotropic phases) and the smooth manufactured field (every
cell its own conductivity: the stored-face stencil), with the float64 solve of
the same problem.  Imports /root/reference (build container only); writes
tests/golden/solves_f32_fused.json.

    python tests/golden/make_golden_f32_fused.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import etchomo as E  # noqa: E402

CASES = [
    # kind, n, contrast, axis, rtol
    ("random-a", 128, 100.0, "z", 1e-6),
    ("random-a", 128, 100.0, "x", 1e-6),
    ("center-ball", 128, 10.0, "y", 1e-6),
    ("channels", 128, 3.0, "z", 1e-6),
    ("smooth", 128, 0.0, "x", 1e-6),
    ("random-a", 256, 100.0, "z", 1e-6),
]

pr = E.RANDOM_BALL_PRESETS["a"]
out = []
for kind, n, c, ax, rtol in CASES:
    if kind == "random-a":
        field = E.gen_random_balls(n, pr["count"], pr["r_min"], pr["r_max"], c, pr["seed"])
    elif kind == "center-ball":
        field = E.gen_center_ball(n, c)
    elif kind == "channels":
        field = E.gen_channels(8, n // 8, c)
    else:
        field = E.gen_smooth_problem(n)[0]
    bc = E.BoundaryConfig(E.Axis(ax), 1.0, 0.0)
    rep = E.homogenize(field, bc, rtol, precision="f32")
    r64 = E.homogenize(field, bc, rtol, precision="f64")
    out.append(dict(kind=kind, n=n, kappa=c, axis=ax, rtol=rtol, precond="fct", iterations=rep.iterations,
                    converged=rep.converged, kappa_eff=rep.kappa_eff, history=rep.relative_residuals,
                    precision=rep.precision, refs=rep.ref_params.as_dict() if rep.ref_params else None,
                    f64_iterations=r64.iterations, f64_kappa_eff=r64.kappa_eff))
    print(kind, n, c, ax, rtol, rep.iterations, repr(rep.kappa_eff), r64.iterations, repr(r64.kappa_eff),
          flush=True)
    path = Path(__file__).resolve().parent / "solves_f32_fused.json"
    path.write_text(json.dumps(out, indent=1) + "\n")
