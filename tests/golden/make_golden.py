"""Generate the committed golden fixtures from the REFERENCE implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py            # small fixtures (~1 min)
    python tests/golden/make_golden.py --big      # + 128^3 three-direction solve

Writes tests/golden/kernels.npz (per-kernel input/output vectors on the
reference's own test shapes) and tests/golden/solves.json (iteration counts,
kappa_eff and residual histories of reference homogenize() runs).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent

# shapes (nx, ny, nz) used by the reference tests: test_tpfa.py:107 symmetry
# shapes, test_transforms.py parity sizes, criterion-3 style ragged grids
KERNEL_SHAPES = [(5, 4, 3), (8, 8, 8), (17, 9, 5), (1, 6, 4), (7, 6, 1), (2, 1, 3),
                 (1, 1, 1), (33, 17, 9), (16, 16, 16), (32, 8, 12), (64, 64, 8)]


def kernels(E):
    out = {}
    for nx, ny, nz in KERNEL_SHAPES:
        tag = f"{nx}x{ny}x{nz}"
        rng = np.random.default_rng(nx * 10000 + ny * 100 + nz)
        grid = E.GridSpec(nx, ny, nz, 1.0 + 0.25 * (nx % 3), 1.0, 0.5 + 0.5 * (nz % 2))
        k = np.exp(rng.uniform(-np.log(50.0), np.log(50.0), (3, grid.n_cells)))
        field = E.OrthotropicField(grid, *k)
        sys_ = E.build_system(field, E.BoundaryConfig(E.Axis.Z, 1.0, 0.0))
        u = rng.standard_normal(grid.n_cells)
        st = E.coefficient_stats(sys_)
        refs = E.solve_reference_lp(st)
        plan = E.FctPlan(nx, ny, nz)
        fwd, _ = plan.forward(u.reshape(grid.shape))
        bwd, _ = plan.backward(u.reshape(grid.shape))
        fac = E.build_tridiag(grid, refs)
        thom = E.thomas_solve_batch(fac, u.copy())
        pre = E.FctPreconditioner(grid, refs)(u)
        out[f"{tag}/grid"] = np.array([nx, ny, nz, grid.lx, grid.ly, grid.lz])
        out[f"{tag}/k"] = k
        out[f"{tag}/u"] = u
        out[f"{tag}/Au"] = E.apply_operator(sys_, u)
        out[f"{tag}/b"] = E.build_rhs(sys_)
        out[f"{tag}/stats"] = np.array([v for pair in st.groups().values() for v in pair])
        out[f"{tag}/refs"] = np.array(list(refs.as_dict().values()))
        out[f"{tag}/fwd"] = fwd.reshape(-1)
        out[f"{tag}/bwd"] = bwd.reshape(-1)
        out[f"{tag}/thomas"] = thom.reshape(-1)
        out[f"{tag}/precond"] = pre
    np.savez_compressed(HERE / "kernels.npz", **out)
    print("kernels.npz:", len(out), "arrays")


def solve_cases(big: bool):
    cases = []
    for n, C, axes, rtol in [(16, 10.0, "xyz", 1e-6), (24, 100.0, "xyz", 1e-6),
                             (32, 1000.0, "z", 1e-6), (64, 10.0, "z", 1e-6),
                             (64, 100.0, "xyz", 1e-6)]:
        for ax in axes:
            cases.append(dict(kind="random-a", n=n, kappa=C, axis=ax, rtol=rtol))
    for C in (0.01, 10.0, 100.0, 1000.0):
        for rtol in (1e-5, 1e-7, 1e-9):
            cases.append(dict(kind="center-ball", n=32, kappa=C, axis="z", rtol=rtol))
    if big:
        for ax in "xyz":
            cases.append(dict(kind="random-a", n=128, kappa=100.0, axis=ax, rtol=1e-6))
    return cases


def solves(E, big: bool):
    preset = E.RANDOM_BALL_PRESETS["a"]
    path = HERE / "solves.json"
    have = json.loads(path.read_text()) if path.exists() else []
    done = {(c["kind"], c["n"], c["kappa"], c["axis"], c["rtol"]) for c in have}
    fields = {}
    for case in solve_cases(big):
        key = (case["kind"], case["n"], case["kappa"], case["axis"], case["rtol"])
        if key in done:
            continue
        fk = (case["kind"], case["n"], case["kappa"])
        if fk not in fields:
            if case["kind"] == "random-a":
                fields[fk] = E.gen_random_balls(case["n"], preset["count"], preset["r_min"],
                                                preset["r_max"], case["kappa"], preset["seed"])
            else:
                fields[fk] = E.gen_center_ball(case["n"], case["kappa"])
        t0 = time.perf_counter()
        rep = E.homogenize(fields[fk], E.BoundaryConfig(E.Axis(case["axis"]), 1.0, 0.0),
                           case["rtol"])
        case = dict(case, iterations=rep.iterations, converged=rep.converged,
                    kappa_eff=rep.kappa_eff, history=rep.relative_residuals,
                    refs=rep.ref_params.as_dict(), seconds=time.perf_counter() - t0)
        print(key, rep.iterations, repr(rep.kappa_eff), f"{case['seconds']:.1f}s", flush=True)
        have.append(case)
        path.write_text(json.dumps(have, indent=1) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    import etchomo as E

    kernels(E)
    solves(E, args.big)


if __name__ == "__main__":
    main()
