"""512^3 reference solves (random-a preset geometry, contrast 100, rtol 1e-6),
one direction per invocation; ~26 min and ~19 GB RSS each on the build host.

    python tests/golden/make_golden_512.py x y z
Appends to tests/golden/solves_512.json.  Imports /root/reference (build
container only)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import etchomo as E  # noqa: E402

path = Path(__file__).resolve().parent / "solves_512.json"
have = json.loads(path.read_text()) if path.exists() else []
pr = E.RANDOM_BALL_PRESETS["a"]
t0 = time.perf_counter()
field = E.gen_random_balls(512, pr["count"], pr["r_min"], pr["r_max"], 100.0, pr["seed"])
gen = time.perf_counter() - t0
for ax in sys.argv[1:]:
    if any(c["axis"] == ax for c in have):
        continue
    t0 = time.perf_counter()
    rep = E.homogenize(field, E.BoundaryConfig(E.Axis(ax), 1.0, 0.0), 1e-6)
    case = dict(kind="random-a", n=512, kappa=100.0, axis=ax, rtol=1e-6, iterations=rep.iterations,
                converged=rep.converged, kappa_eff=rep.kappa_eff, history=rep.relative_residuals,
                refs=rep.ref_params.as_dict(), prep_seconds=rep.prep_seconds,
                exec_seconds=rep.exec_seconds, gen_seconds=gen, wall=time.perf_counter() - t0)
    have.append(case)
    path.write_text(json.dumps(have, indent=1) + "\n")
    print(ax, rep.iterations, repr(rep.kappa_eff), case["wall"], flush=True)
