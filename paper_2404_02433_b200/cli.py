"""`etc generate` / `etc solve` with the GPU backend.

Same flags, report JSON schema (`report_to_dict`, pipeline.py:250-280),
residual CSV (`write_history`, pipeline.py:290-295) and exit codes as the
reference CLI (cli.py:1-5, 165-186, 300-323): 0 success, 1 non-convergence
or breakdown, 2 usage / configuration error, 3 I/O or file-format error.
The study subcommands (convergence, compare, channels, precision, bench)
and the verification-suite runner are experiment drivers around the hot
path and stay with the reference.

    python -m paper_2404_02433_b200 generate --config random-balls --preset a --n 128 -o f.vox
    python -m paper_2404_02433_b200 solve f.vox --axis z --rtol 1e-6 --report r.json --history h.csv
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from .grid import (
    RANDOM_BALL_PRESETS,
    Axis,
    BoundaryConfig,
    ConfigError,
    VoxFormatError,
    gen_center_ball,
    gen_channels,
    gen_random_balls,
    read_vox,
    write_vox,
)
from .solver import PcgBreakdownError, homogenize


def _positive_int(text: str) -> int:
    value = int(text)
    if value <= 0:
        raise argparse.ArgumentTypeError(f"expected a positive integer, got {text}")
    return value


def make_field(generator: str, params: dict):
    """pipeline.make_field (pipeline.py:219-247) on the device generators."""
    if generator == "center-ball":
        return gen_center_ball(params.get("n", 64), params.get("kappa_inc", 10.0))
    if generator == "random-balls":
        preset = params.get("preset")
        merged = dict(RANDOM_BALL_PRESETS[preset]) if preset else {}
        merged.update({k: v for k, v in params.items() if k != "preset"})
        return gen_random_balls(merged.get("n", 64), merged["count"], merged["r_min"], merged["r_max"],
                                merged.get("kappa_inc", 10.0), merged.get("seed", 0))
    if generator == "channels":
        return gen_channels(params.get("cells_per_period", 8), params.get("periods", 8), params.get("psi", 1.0))
    raise ConfigError(f"unknown generator {generator!r}")


def report_to_dict(report, config: dict, grid, boundary: BoundaryConfig, rtol: float) -> dict:
    """The reference's report document, key for key (pipeline.py:250-280)."""
    doc = {
        "config": config,
        "grid": {"nx": grid.nx, "ny": grid.ny, "nz": grid.nz, "lx": grid.lx, "ly": grid.ly, "lz": grid.lz},
        "boundary": {"axis": Axis(boundary.axis).value, "p_in": boundary.p_in, "p_out": boundary.p_out},
        "precond": report.preconditioner,
        "ref_params": report.ref_params.as_dict() if report.ref_params else None,
        "rtol": rtol,
        "iterations": report.iterations,
        "converged": report.converged,
        "kappa_eff": report.kappa_eff,
        "prep_seconds": report.prep_seconds,
        "exec_seconds": report.exec_seconds,
        "precision": report.precision,
    }
    if getattr(report, "l2_error", None) is not None:
        doc["l2_error"] = report.l2_error
    return doc


def write_report(path, doc: dict) -> None:
    Path(path).parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=2, sort_keys=True)
        fh.write("\n")


def write_history(path, residuals) -> None:
    Path(path).parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w") as fh:
        fh.write("iter,relres\n")
        for i, res in enumerate(residuals):
            fh.write(f"{i},{res!r}\n")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="etc", description="Effective thermal conductivity of voxel RVEs "
                                     "on the GPU (finite-volume discretization + cosine-transform preconditioned CG).")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("generate", help="write a generated RVE to a voxel file")
    p.add_argument("--config", choices=["center-ball", "random-balls", "channels"], required=True)
    p.add_argument("--n", type=_positive_int, action="append")
    p.add_argument("--kappa-inc", type=float, default=10.0)
    p.add_argument("--count", type=_positive_int, default=40)
    p.add_argument("--r-min", type=float, default=0.05)
    p.add_argument("--r-max", type=float, default=0.15)
    p.add_argument("--psi", type=float, action="append")
    p.add_argument("--periods", type=_positive_int, default=8)
    p.add_argument("--seed", type=int, default=11)
    p.add_argument("--preset", choices=sorted(RANDOM_BALL_PRESETS), default=None)
    p.add_argument("-o", dest="output", required=True, help="output .vox path")
    p.add_argument("--precision", choices=["f64", "f32"], default="f64")

    p = sub.add_parser("solve", help="homogenize one voxel file")
    p.add_argument("input", help="input .vox path")
    p.add_argument("--axis", choices=["x", "y", "z"], default="z")
    p.add_argument("--p-in", type=float, default=1.0)
    p.add_argument("--p-out", type=float, default=0.0)
    p.add_argument("--rtol", type=float, default=1e-9)
    p.add_argument("--max-iter", type=_positive_int, default=1024)
    p.add_argument("--ref", choices=["opt", "one"], default="opt")
    p.add_argument("--precision", choices=["f64", "f32"], default="f64")
    p.add_argument("--threads", type=int, default=0, help="accepted for compatibility (host BLAS is not used)")
    p.add_argument("--precond", choices=["fct", "ssor", "jacobi", "none"], default="fct")
    p.add_argument("--omega", type=float, default=1.0)
    p.add_argument("--report", default=None, help="write the JSON report here")
    p.add_argument("--history", default=None, help="write the residual CSV here")
    return parser


def _generator_params(args) -> dict:
    n = (args.n or [64])[0]
    if args.config == "center-ball":
        return {"n": n, "kappa_inc": args.kappa_inc}
    if args.config == "random-balls":
        if args.preset:
            return {"preset": args.preset, "n": n}
        return {"n": n, "count": args.count, "r_min": args.r_min, "r_max": args.r_max,
                "kappa_inc": args.kappa_inc, "seed": args.seed}
    return {"cells_per_period": (args.n or [8])[0], "periods": args.periods, "psi": (args.psi or [1.0])[0]}


def cmd_generate(args) -> int:
    import numpy as np

    field = make_field(args.config, _generator_params(args))
    write_vox(field, args.output, dtype=np.float32 if args.precision == "f32" else np.float64)
    print(f"wrote {args.output}")
    return 0


def cmd_solve(args) -> int:
    field = read_vox(args.input)
    boundary = BoundaryConfig(Axis(args.axis), args.p_in, args.p_out)
    report = homogenize(field, boundary, args.rtol, args.precond, args.ref, args.precision, args.omega,
                        args.max_iter)
    doc = report_to_dict(report, {"input": str(args.input)}, field.grid, boundary, args.rtol)
    if args.report:
        write_report(args.report, doc)
    if args.history:
        write_history(args.history, report.relative_residuals)
    print(json.dumps({"kappa_eff": report.kappa_eff, "iterations": report.iterations,
                      "converged": report.converged}))
    return 0 if report.converged else 1


_HANDLERS = {"generate": cmd_generate, "solve": cmd_solve}


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code in (0, None) else 2
    try:
        return _HANDLERS[args.command](args)
    except ConfigError as exc:
        print(f"etc: configuration error: {exc}", file=sys.stderr)
        return 2
    except PcgBreakdownError as exc:
        print(f"etc: solver breakdown: {exc}", file=sys.stderr)
        return 1
    except VoxFormatError as exc:
        print(f"etc: file format error: {exc}", file=sys.stderr)
        return 3
    except OSError as exc:
        print(f"etc: i/o error: {exc}", file=sys.stderr)
        return 3
    except ValueError as exc:
        print(f"etc: invalid configuration: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    raise SystemExit(main())
