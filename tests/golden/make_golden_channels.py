"""Reference solves on the orthotropic channel lattice (gen_channels,
grid.py:287-319; the SURVEY 8(d) config-3 proxy and Appendix A's channel
rows): Diag(2^psi, 5^psi, 10^psi) channels in a Diag(0.01, 0.1, 1) matrix,
ref_mode "opt" and "one".  Imports /root/reference (build container only);
writes tests/golden/solves_channels.json.

    python tests/golden/make_golden_channels.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import etchomo as E  # noqa: E402

CASES = [
    # cells_per_period, periods, psi, axis, rtol, ref_mode, precond
    (8, 2, 1.0, "z", 1e-8, "opt", "fct"),
    (8, 2, 2.0, "x", 1e-8, "one", "fct"),
    (8, 4, 1.0, "z", 1e-5, "opt", "fct"),
    (8, 4, 3.0, "y", 1e-6, "opt", "fct"),
    (16, 2, 2.0, "z", 1e-6, "one", "fct"),
    (8, 8, 1.0, "z", 1e-5, "opt", "fct"),
    (8, 8, 1.0, "z", 1e-5, "one", "fct"),
    (8, 2, 2.0, "z", 1e-7, "opt", "jacobi"),
]

out = []
for cpp, per, psi, ax, rtol, mode, pc in CASES:
    field = E.gen_channels(cpp, per, psi)
    rep = E.homogenize(field, E.BoundaryConfig(E.Axis(ax), 1.0, 0.0), rtol, ref_mode=mode, precond=pc)
    out.append(dict(kind="channels", cells_per_period=cpp, periods=per, psi=psi, n=cpp * per, axis=ax,
                    rtol=rtol, ref_mode=mode, precond=pc, iterations=rep.iterations, converged=rep.converged,
                    kappa_eff=rep.kappa_eff, history=rep.relative_residuals, refs=rep.ref_params.as_dict()))
    print(cpp, per, psi, ax, rtol, mode, pc, rep.iterations, repr(rep.kappa_eff), flush=True)
path = Path(__file__).resolve().parent / "solves_channels.json"
path.write_text(json.dumps(out, indent=1) + "\n")

# the generator itself, bit for bit (16^3, psi = 1.5)
import numpy as np  # noqa: E402

f = E.gen_channels(8, 2, 1.5)
np.savez_compressed(Path(__file__).resolve().parent / "channels_8x2.npz", kx=np.asarray(f.kx),
                    ky=np.asarray(f.ky), kz=np.asarray(f.kz))
