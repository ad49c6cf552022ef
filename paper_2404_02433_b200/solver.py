"""Host orchestration of the device solve: the drop-in `homogenize()`.

Mirrors the reference pipeline (/root/reference/pkg/src/etchomo/pipeline.py:135-175):
permute -> scale -> faces -> statistics -> LP -> preconditioner setup -> rhs ->
PCG -> outflow flux -> kappa_eff, with the same arguments, validation errors,
exception types and SolveReport fields.  Everything O(N) runs in the CUDA
extension (libetc_b200.so) through the C ABI; the host keeps only the O(1)
LP and the O(nx+ny+nz) tables.
"""

from __future__ import annotations

import ctypes as C
import time
import weakref
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _native
from .grid import Axis, BoundaryConfig, ConfigError, GridSpec, OrthotropicField, axis_index
from .reference import (
    CoefficientStats,
    ReferenceParams,
    check_pivots,
    eigen_weights,
    ones_reference,
    solve_reference_lp,
    z_chain_diagonal,
)

_PRECISIONS = ("f64", "f32")


class PcgBreakdownError(RuntimeError):
    """Loss of positive definiteness mid-iteration (reference krylov.py:12-17)."""

    def __init__(self, message: str, iteration: int):
        super().__init__(f"{message} at iteration {iteration}")
        self.iteration = iteration


_BREAKDOWN_MSG = {
    1: "operator inner product lost positivity",
    2: "residual is not finite",
    3: "preconditioned inner product not positive",
}


@dataclass
class SolveReport:
    """Outcome of one solve (reference krylov.py:20-33)."""

    iterations: int
    converged: bool
    relative_residuals: list = dc_field(default_factory=list)
    kappa_eff: float | None = None
    prep_seconds: float = 0.0
    exec_seconds: float = 0.0
    precision: str = "f64"
    preconditioner: str = "fct"
    ref_params: ReferenceParams | None = None
    l2_error: float | None = None
    device_ms: float = 0.0


def _torch():
    import torch

    return torch


def _stream_handle(device_index: int) -> int:
    torch = _torch()
    return torch.cuda.current_stream(device_index).cuda_stream


def _check(rc: int, what: str) -> None:
    if rc == _native.ETC_OK:
        return
    msg = f"{what}: {_native.last_error()}"
    if rc == _native.ETC_CONFIG:
        raise ConfigError(msg)
    if rc == _native.ETC_PIVOT:
        raise FloatingPointError(msg)
    raise RuntimeError(msg)


class DevicePlan:
    """One device workspace for one original-orientation grid (owns ~8-12
    vectors of nx*ny*nz float64 on the GPU).  Not re-entrant."""

    def __init__(self, grid: GridSpec, device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise _native.NativeUnavailable("no CUDA device visible: the solver has no CPU path")
        self.lib = _native.lib()
        self.grid = grid
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self._h = C.c_void_p()
        with torch.cuda.device(self.device):
            stream = _stream_handle(self.device.index)
            _check(self.lib.etc_plan_create(C.byref(self._h), grid.nx, grid.ny, grid.nz,
                                            float(grid.lx), float(grid.ly), float(grid.lz), stream),
                   "etc_plan_create")
        self._field_key = None
        self._keepalive = None
        self.precision = "f64"
        self.canonical = None
        self.axis = None
        self._fin = weakref.finalize(self, self.lib.etc_plan_destroy, self._h)

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        self._fin()

    @property
    def handle(self):
        return self._h

    @property
    def device_bytes(self) -> int:
        return int(self.lib.etc_plan_device_bytes(self._h))

    # -- field -------------------------------------------------------------
    def load_field(self, fld: OrthotropicField, force: bool = False) -> None:
        arrs = (fld.kx, fld.ky, fld.kz)
        key = (id(fld), tuple(id(a) for a in arrs),
               tuple(getattr(a, "_version", 0) for a in arrs))
        if not force and key == self._field_key:
            return
        torch = _torch()
        ptrs = []
        keep = []
        on_dev = fld.on_device
        for a in arrs:
            if on_dev:
                if a.device != self.device:
                    a = a.to(self.device)
                if a.dtype != torch.float64:  # float32 fields widen exactly (the f32 solve casts back)
                    a = a.to(torch.float64)
                keep.append(a)
                ptrs.append(a.data_ptr())
            else:
                if a.dtype != np.float64:
                    a = a.astype(np.float64)
                keep.append(a)
                ptrs.append(a.ctypes.data)
        # identical arrays -> identical pointers -> stored once
        with torch.cuda.device(self.device):
            _check(self.lib.etc_load_field(self._h, ptrs[0], ptrs[1], ptrs[2], 1 if on_dev else 0),
                   "etc_load_field")
        # host buffers must outlive the async copy; the keyed objects
        # themselves are kept too, so their ids cannot be reused by another
        # field while this key is current (a converted copy alone would not
        # pin them)
        self._keepalive = (fld, arrs, keep)
        self._field_key = key
        self.axis = None

    def select_axis(self, axis) -> GridSpec:
        dims = (C.c_int * 3)()
        lens = (C.c_double * 3)()
        _check(self.lib.etc_select_axis(self._h, axis_index(axis), dims, lens), "etc_select_axis")
        self.axis = Axis(axis)
        self.canonical = GridSpec(dims[0], dims[1], dims[2], lens[0], lens[1], lens[2])
        return self.canonical

    def coefficient_stats(self) -> CoefficientStats:
        out = (C.c_double * 10)()
        _check(self.lib.etc_coefficient_stats(self._h, out), "etc_coefficient_stats")
        return CoefficientStats(*[float(v) for v in out])

    def set_reference(self, refs: ReferenceParams) -> None:
        g = self.canonical
        wx = eigen_weights(g.nx)
        wy = eigen_weights(g.ny)
        zd = z_chain_diagonal(g.nz, refs)
        check_pivots(g.nz, zd, refs, np.float32 if self.precision == "f32" else np.float64)
        r5 = (C.c_double * 5)(*refs.constants())
        dp = _native._DP
        _check(self.lib.etc_set_reference(self._h, r5, wx.ctypes.data_as(dp), wy.ctypes.data_as(dp),
                                          zd.ctypes.data_as(dp)), "etc_set_reference")

    # -- solve -------------------------------------------------------------
    def solve(self, p_in: float, p_out: float, rtol: float, max_iter: int):
        info = _native.SolveInfo()
        hist = np.empty(max_iter + 1, dtype=np.float64)
        rc = self.lib.etc_solve(self._h, float(p_in), float(p_out), float(rtol), int(max_iter),
                                C.byref(info), hist.ctypes.data_as(_native._DP))
        history = [float(v) for v in hist[: info.iterations + 1]]
        if rc == _native.ETC_BREAKDOWN:
            raise PcgBreakdownError(_BREAKDOWN_MSG.get(info.breakdown_kind, "breakdown"),
                                    info.breakdown_iter)
        _check(rc, "etc_solve")
        return info, history

    def set_precision(self, precision: str) -> None:
        """Arithmetic of the next stats / solve: "f64" | "f32" (pipeline.py:147-160)."""
        _check(self.lib.etc_set_precision(self._h, 32 if precision == "f32" else 64), "etc_set_precision")
        self.precision = precision

    def keep_solution(self, keep: bool) -> None:
        _check(self.lib.etc_keep_solution(self._h, 1 if keep else 0), "etc_keep_solution")

    def set_precond(self, kind: str) -> None:
        """Preconditioner plugin of the next solves: "fct" | "jacobi" | "none"."""
        _check(self.lib.etc_set_precond(self._h, _native.PRECOND_KINDS[kind]), "etc_set_precond")

    def solution(self):
        torch = _torch()
        g = self.canonical
        out = torch.empty(g.n_cells, dtype=torch.float64, device=self.device)
        _check(self.lib.etc_get_solution(self._h, out.data_ptr(), 1), "etc_get_solution")
        return out


# plans are reused across calls on the same grid (allocation of ~10 vectors
# per call would dominate small solves)
_PLANS: dict = {}


def get_plan(grid: GridSpec, device=None) -> DevicePlan:
    torch = _torch()
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (grid.nx, grid.ny, grid.nz, float(grid.lx), float(grid.ly), float(grid.lz), dev.index)
    plan = _PLANS.get(key)
    if plan is None:
        plan = DevicePlan(grid, dev)
        _PLANS[key] = plan
    return plan


def release_plans() -> None:
    for p in _PLANS.values():
        p.close()
    _PLANS.clear()


def _parse_precond(tag: str, default_omega: float) -> tuple[str, float]:
    """Preconditioner plugin tags (reference pipeline.py:114-122)."""
    if tag.startswith("ssor"):
        omega = default_omega
        if ":" in tag:
            omega = float(tag.split(":", 1)[1])
        return "ssor", omega
    if tag in ("fct", "jacobi", "none"):
        return tag, default_omega
    raise ConfigError(f"unknown preconditioner tag {tag!r}")


def _field_device(fld) -> str | None:
    if getattr(fld, "on_device", False):
        return str(fld.kx.device)
    return None


def _as_field(fld) -> OrthotropicField:
    """Accept this package's field or any duck-typed one (e.g. etchomo's)."""
    if isinstance(fld, OrthotropicField):
        return fld
    g = fld.grid
    grid = GridSpec(int(g.nx), int(g.ny), int(g.nz), float(g.lx), float(g.ly), float(g.lz))
    return OrthotropicField(grid, fld.kx, fld.ky, fld.kz, validate=False)


def homogenize(
    field,
    boundary: BoundaryConfig,
    rtol: float = 1e-9,
    precond: str = "fct",
    ref_mode: str = "opt",
    precision: str = "f64",
    omega: float = 1.0,
    max_iter: int = 1024,
    device=None,
) -> SolveReport:
    """Effective conductivity along `boundary.axis` (reference pipeline.py:135-175).

    Same signature and report as the reference; the whole O(N) path runs on
    the GPU.  `field` arrays may be host numpy arrays (copied to the device
    once per field and cached) or CUDA float64 tensors (used in place)."""
    return _homogenize(field, boundary, rtol, precond, ref_mode, precision, omega, max_iter, device,
                       keep_solution=False)[0]


def homogenize_with_solution(field, boundary: BoundaryConfig, rtol: float = 1e-9, ref_mode: str = "opt",
                             max_iter: int = 1024, device=None, precond: str = "fct"):
    """homogenize() that also returns the full potential p (canonical,
    z-oriented layout) as a CUDA tensor, like the reference's pcg()
    (krylov.py:91).  Costs one extra vector read+write per iteration."""
    return _homogenize(field, boundary, rtol, precond, ref_mode, "f64", 1.0, max_iter, device,
                       keep_solution=True)


def _homogenize(field, boundary, rtol, precond, ref_mode, precision, omega, max_iter, device, keep_solution):
    if precision not in _PRECISIONS:
        raise ConfigError(f"precision must be f64 or f32, got {precision!r}")
    if ref_mode not in ("opt", "one"):
        raise ConfigError(f"ref mode must be opt or one, got {ref_mode!r}")
    kind, omega = _parse_precond(precond, omega)
    if kind == "ssor":
        if keep_solution:
            raise ConfigError("the full-solution mode runs the fused preconditioners (fct | jacobi | none)")
        return _homogenize_composed(field, boundary, rtol, kind, ref_mode, precision, omega, max_iter,
                                    device), None
    if precision == "f32" and keep_solution:
        raise ConfigError("the full-solution mode runs in f64")
    if rtol <= 0.0:
        raise ValueError("rtol must be positive")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    fld = _as_field(field)
    torch = _torch()

    plan = get_plan(fld.grid, device if device is not None else _field_device(fld))
    with torch.cuda.device(plan.device):
        t0 = time.perf_counter()
        plan.load_field(fld)
        plan.select_axis(boundary.axis)
        plan.set_precision(precision)
        stats = plan.coefficient_stats()
        refs = solve_reference_lp(stats) if ref_mode == "opt" else ones_reference(stats)
        plan.set_reference(refs)
        plan.keep_solution(keep_solution)
        plan.set_precond(kind)
        prep = time.perf_counter() - t0
        t1 = time.perf_counter()
        info, history = plan.solve(boundary.p_in, boundary.p_out, rtol, max_iter)
        exec_s = time.perf_counter() - t1
        sol = plan.solution() if keep_solution else None
    rep = SolveReport(
        iterations=int(info.iterations),
        converged=bool(history[-1] <= rtol),
        relative_residuals=history,
        kappa_eff=float(info.kappa_eff),
        prep_seconds=prep,
        exec_seconds=exec_s,
        precision=precision,
        preconditioner=kind,
        ref_params=refs,
        device_ms=float(info.device_ms),
    )
    return rep, sol


def _homogenize_composed(field, boundary, rtol, kind, ref_mode, precision, omega, max_iter, device):
    """homogenize() composed from the operator-plugin layer, statement for
    statement the reference pipeline (pipeline.py:153-175): permute, build,
    stats, LP, preconditioner, rhs, pcg over device tensors, flux, kappa.
    Used for the preconditioners the fused solve does not carry (ssor)."""
    from . import plugin

    if rtol <= 0.0:
        raise ValueError("rtol must be positive")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    fld = _as_field(field)
    torch = _torch()
    dev = torch.device(device) if device is not None else (fld.kx.device if fld.on_device else
                                                           torch.device("cuda", torch.cuda.current_device()))
    with torch.cuda.device(dev):
        t0 = time.perf_counter()
        dt = np.float32 if precision == "f32" else np.float64
        arrs = [plugin._to_dev(a, dt) for a in (fld.kx, fld.ky, fld.kz)]
        work = plugin.axis_permute(OrthotropicField(fld.grid, *arrs, validate=False), boundary.axis)
        canon = BoundaryConfig(Axis.Z, boundary.p_in, boundary.p_out)
        sys = plugin.build_system(work, canon)
        stats = plugin.coefficient_stats(sys)
        refs = solve_reference_lp(stats) if ref_mode == "opt" else ones_reference(stats)
        if kind == "ssor":
            apply_m = plugin.SsorPreconditioner(sys, omega)
        elif kind == "fct":
            apply_m = plugin.FctPreconditioner(sys.grid, refs, dt)
        elif kind == "jacobi":
            apply_m = plugin.JacobiPreconditioner(sys)
        else:
            apply_m = plugin.identity_apply
        b = plugin.build_rhs(sys)
        prep = time.perf_counter() - t0
        t1 = time.perf_counter()
        solution, report = plugin.pcg(lambda u: plugin.apply_operator(sys, u), apply_m, b, rtol, max_iter)
        flux = plugin.reconstruct_boundary_flux(sys, solution)
        report.kappa_eff = plugin.effective_conductivity(sys, flux)
        report.exec_seconds = time.perf_counter() - t1
    report.prep_seconds = prep
    report.precision = precision
    report.preconditioner = f"ssor:{omega:g}" if kind == "ssor" else kind
    report.ref_params = refs
    return report


def effective_tensor(field, rtol: float = 1e-9, p_in: float = 1.0, p_out: float = 0.0,
                     ref_mode: str = "opt", max_iter: int = 1024, device=None, axes="xyz",
                     precond: str = "fct", precision: str = "f64"):
    """Diagonal effective-conductivity tensor from one solve per load
    direction (the reference composes it from three homogenize() calls,
    pkg/tests/test_pipeline.py:54-58).  The field is uploaded once."""
    reports = {}
    for ax in axes:
        reports[ax] = homogenize(field, BoundaryConfig(Axis(ax), p_in, p_out), rtol, precond,
                                 ref_mode, precision, 1.0, max_iter, device)
    kappa = np.array([reports[a].kappa_eff if a in reports else np.nan for a in "xyz"])
    return kappa, reports
