"""Host-side pieces of the FCT preconditioner that are O(1) or O(nx+ny+nz):
coefficient-statistics record, the closed-form min-max LP for the reference
constants, and the eigen-weight / z-chain tables.  They stay on the host
(north star: "the LP choice of homogeneous reference parameters stays on the
host because it is tiny"); the O(N) statistics reduction itself runs on the
device (etc_coefficient_stats).

Reference: /root/reference/pkg/src/etchomo/preconditioner.py:26-212.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .grid import ConfigError


@dataclass(frozen=True)
class CoefficientStats:
    """Extremes of the scaled face transmissibilities (preconditioner.py:26-55)."""

    kx_min: float
    kx_max: float
    ky_min: float
    ky_max: float
    kz_min: float
    kz_max: float
    kin_min: float
    kin_max: float
    kout_min: float
    kout_max: float

    def __post_init__(self):
        for lo, hi in self.groups().values():
            if not (0.0 < lo <= hi) or not math.isfinite(hi):
                raise ConfigError("stats must satisfy 0 < min <= max < inf")

    def groups(self) -> dict:
        return {
            "x": (self.kx_min, self.kx_max),
            "y": (self.ky_min, self.ky_max),
            "z": (self.kz_min, self.kz_max),
            "in": (self.kin_min, self.kin_max),
            "out": (self.kout_min, self.kout_max),
        }


@dataclass(frozen=True)
class ReferenceParams:
    """Five reference constants + spectral bounds (preconditioner.py:58-91)."""

    kx_ref: float
    ky_ref: float
    kz_ref: float
    kin_ref: float
    kout_ref: float
    lambda_lo: float = 1.0
    lambda_hi: float = 1.0

    def __post_init__(self):
        for name in ("kx_ref", "ky_ref", "kz_ref", "kin_ref", "kout_ref"):
            if getattr(self, name) <= 0.0:
                raise ConfigError(f"{name} must be positive")
        if not (0.0 < self.lambda_lo <= self.lambda_hi):
            raise ConfigError("need 0 < lambda_lo <= lambda_hi")

    @property
    def objective(self) -> float:
        return self.lambda_hi / self.lambda_lo

    def as_dict(self) -> dict:
        return {
            "kx": self.kx_ref, "ky": self.ky_ref, "kz": self.kz_ref,
            "kin": self.kin_ref, "kout": self.kout_ref,
            "lambda_lo": self.lambda_lo, "lambda_hi": self.lambda_hi,
        }

    def constants(self) -> tuple:
        return (self.kx_ref, self.ky_ref, self.kz_ref, self.kin_ref, self.kout_ref)


def _bounds(stats: CoefficientStats, refs: dict) -> tuple[float, float]:
    g = stats.groups()
    lo = min(mn / refs[d] for d, (mn, _) in g.items())
    hi = max(mx / refs[d] for d, (_, mx) in g.items())
    return lo, hi


def solve_reference_lp(stats: CoefficientStats) -> ReferenceParams:
    """Optimum of  min (hi - lo) s.t. c_d + lo <= log min_d, c_d + hi >= log max_d:
    the per-group geometric mean attains the bound max_d log(max_d/min_d)
    (preconditioner.py:117-130)."""
    refs = {d: math.sqrt(mn * mx) for d, (mn, mx) in stats.groups().items()}
    lo, hi = _bounds(stats, refs)
    return ReferenceParams(refs["x"], refs["y"], refs["z"], refs["in"], refs["out"], lo, hi)


def ones_reference(stats: CoefficientStats | None = None) -> ReferenceParams:
    """All-ones constants (preconditioner.py:133-140)."""
    if stats is None:
        return ReferenceParams(1.0, 1.0, 1.0, 1.0, 1.0)
    lo, hi = _bounds(stats, {d: 1.0 for d in ("x", "y", "z", "in", "out")})
    return ReferenceParams(1.0, 1.0, 1.0, 1.0, 1.0, lo, hi)


def eigen_weights(n: int) -> np.ndarray:
    """2 (1 - cos(q pi / n)): eigenvalues of the Neumann chain (preconditioner.py:186-187)."""
    return 2.0 * (1.0 - np.cos(np.arange(n) * np.pi / n))


def z_chain_diagonal(nz: int, refs: ReferenceParams) -> np.ndarray:
    """Diagonal of the z-chain with the two Dirichlet layers (preconditioner.py:192-199)."""
    zd = np.full(nz, 2.0 * refs.kz_ref)
    if nz == 1:
        zd[0] = 0.0
    else:
        zd[0] = refs.kz_ref
        zd[-1] = refs.kz_ref
    zd[0] += 2.0 * refs.kin_ref
    zd[-1] += 2.0 * refs.kout_ref
    return zd


def check_pivots(nz: int, z_diag: np.ndarray, refs: ReferenceParams, dtype=np.float64) -> None:
    """Raise FloatingPointError exactly when the reference's non-pivoting
    elimination would (preconditioner.py:229-244).  Every plane shift is
    >= 0 (shift(0,0) = 0) and the pivots grow with the shift, so the
    zero-shift column carries the smallest pivots; replay it on the host,
    in the solve's dtype (z_diag and off cast as TridiagFactors does,
    preconditioner.py:189-199)."""
    dt = np.dtype(dtype).type
    z_diag = np.asarray(z_diag).astype(dt)
    off = dt(-refs.kz_ref)
    d0 = z_diag[0] + dt(0.0)
    if d0 <= 0:
        raise FloatingPointError("non-positive pivot in tridiagonal solve")
    if nz == 1:
        return
    upper = off / d0
    for k in range(1, nz):
        denom = (z_diag[k] + dt(0.0)) - off * upper
        if denom <= 0:
            raise FloatingPointError(f"non-positive pivot in tridiagonal solve at layer {k}")
        upper = off / denom
