"""Failure paths of the fused device solve (etc_solve's device-resident Ctl):
PcgBreakdownError for a non-finite residual, an operator that loses
positivity and a preconditioner that loses positivity (reference
krylov.py:60-88), each checked against the reference semantics run by the
plugin layer's host-driven pcg on the same operator and preconditioner
(plugin.pcg restates krylov.py:36-91 statement for statement); and the
non-positive pivot FloatingPointError (preconditioner.py:229-244) of the
host replay used by the fused solve against the device Thomas kernel.

The coefficient statistics reject such fields before a solve
(CoefficientStats: 0 < min <= max < inf), exactly as the reference's do, so
these tests drive the plan through the C ABI: load the field unvalidated,
set the reference constants directly, solve."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2404_02433_b200 as P  # noqa: E402
from paper_2404_02433_b200 import _native, plugin as E  # noqa: E402
from paper_2404_02433_b200.reference import check_pivots, eigen_weights, z_chain_diagonal  # noqa: E402
from paper_2404_02433_b200.solver import DevicePlan  # noqa: E402

ONES = P.ReferenceParams(1.0, 1.0, 1.0, 1.0, 1.0)


def _plan(k, n, zdiag=None, precond="fct"):
    g = P.GridSpec(n, n, n)
    fld = P.OrthotropicField(g, k, k, k, validate=False)
    plan = DevicePlan(g)
    plan.load_field(fld, force=True)
    plan.select_axis(P.Axis.Z)
    plan.set_precision("f64")
    plan.set_precond(precond)
    plan.keep_solution(False)
    if zdiag is None:
        plan.set_reference(ONES)
    else:  # crafted z-chain straight through the ABI (the host LP never builds one)
        wx, wy = eigen_weights(n), eigen_weights(n)
        r5 = (C.c_double * 5)(*ONES.constants())
        dp = _native._DP
        z = np.ascontiguousarray(zdiag, dtype=np.float64)
        rc = plan.lib.etc_set_reference(plan.handle, r5, wx.ctypes.data_as(dp), wy.ctypes.data_as(dp),
                                        z.ctypes.data_as(dp))
        assert rc == 0, _native.last_error()
    return plan, fld


def _reference_semantics(fld, precond, zscale=1.0):
    """The same solve through plugin.pcg (reference krylov.py order of checks)."""
    sys_ = _system(fld)
    if precond == "fct":
        m = E.FctPreconditioner(fld.grid, ONES)
        apply_m = (lambda r: zscale * m(r)) if zscale != 1.0 else m
    else:
        apply_m = E.identity_apply
    return E.pcg(lambda u: E.apply_operator(sys_, u), apply_m, E.build_rhs(sys_), 1e-10)


def _system(fld):
    # build_system validates faces (strictly positive); the breakdown fields
    # need the raw faces, so assemble through the device kernels unvalidated
    g = fld.grid
    s = E.build_system(P.OrthotropicField(g, np.ones(g.n_cells), np.ones(g.n_cells), np.ones(g.n_cells)),
                       P.BoundaryConfig(P.Axis.Z, 1.0, 0.0))
    sx, sy, sz = E.scale_field(fld)
    nx, ny, nz = g.nx, g.ny, g.nz

    def harm(a, b):
        return 2.0 * a * b / (a + b)

    return E.DiscreteSystem(g, harm(sx[:, :, :-1], sx[:, :, 1:]), harm(sy[:, :-1], sy[:, 1:]),
                            harm(sz[:-1], sz[1:]), 2.0 * sz[0], 2.0 * sz[-1], s.boundary, validate=False)


def test_nonfinite_residual_breakdown():
    """A NaN cell makes q, alpha and the residual NaN: 'residual is not
    finite' at iteration 1 (krylov.py:80-81)."""
    n = 16
    k = np.ones(n ** 3)
    k[(n // 2) * n * n + 3 * n + 5] = np.nan
    plan, fld = _plan(k, n)
    with pytest.raises(P.PcgBreakdownError, match="not finite") as dev:
        plan.solve(1.0, 0.0, 1e-10, 100)
    with pytest.raises(P.PcgBreakdownError, match="not finite") as ref:
        _reference_semantics(fld, "fct")
    assert dev.value.iteration == ref.value.iteration == 1


def test_operator_loses_positivity():
    """All conductivities negative: A is negative definite, q.w < 0 on the
    first iteration -> 'operator inner product lost positivity' at 1
    (krylov.py:72-75)."""
    n = 16
    k = -np.ones(n ** 3)
    plan, fld = _plan(k, n)
    with pytest.raises(P.PcgBreakdownError, match="operator inner product") as dev:
        plan.solve(1.0, 0.0, 1e-10, 100)
    with pytest.raises(P.PcgBreakdownError, match="operator inner product") as ref:
        _reference_semantics(fld, "fct")
    assert dev.value.iteration == ref.value.iteration == 1


def test_operator_breakdown_unpreconditioned():
    n = 12
    plan, fld = _plan(-np.ones(n ** 3), n, precond="none")
    with pytest.raises(P.PcgBreakdownError, match="operator inner product") as dev:
        plan.solve(1.0, 0.0, 1e-10, 100)
    with pytest.raises(P.PcgBreakdownError) as ref:
        _reference_semantics(fld, "none")
    assert dev.value.iteration == ref.value.iteration == 1


def test_preconditioner_loses_positivity():
    """A z-chain shifted far negative makes every mode's block negative
    definite: r.z < 0 at iteration 0 (krylov.py:65-67)."""
    n = 16
    zd = z_chain_diagonal(n, ONES) - 1e3
    plan, fld = _plan(np.ones(n ** 3), n, zdiag=zd)
    with pytest.raises(P.PcgBreakdownError, match="preconditioned inner product") as dev:
        plan.solve(1.0, 0.0, 1e-10, 100)
    assert dev.value.iteration == 0
    # reference semantics: any negative definite M^-1 breaks down at 0
    with pytest.raises(P.PcgBreakdownError) as ref:
        _reference_semantics(P.OrthotropicField(P.GridSpec(n, n, n), np.ones(n ** 3), np.ones(n ** 3),
                                                np.ones(n ** 3)), "fct", zscale=-1.0)
    assert ref.value.iteration == 0


def test_breakdown_leaves_plan_usable():
    """After a breakdown the same plan solves a valid field normally (the
    device Ctl is re-initialised by the next etc_solve)."""
    n = 16
    plan, _ = _plan(-np.ones(n ** 3), n)
    with pytest.raises(P.PcgBreakdownError):
        plan.solve(1.0, 0.0, 1e-10, 100)
    fld = P.gen_random_balls(n, 40, 0.05, 0.15, 10.0, 11)
    plan.load_field(fld, force=True)
    plan.select_axis(P.Axis.Z)
    refs = P.solve_reference_lp(plan.coefficient_stats())
    plan.set_reference(refs)
    info, hist = plan.solve(1.0, 0.0, 1e-8, 200)
    ref = P.homogenize(fld, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-8)
    assert info.iterations == ref.iterations and hist == ref.relative_residuals


@pytest.mark.parametrize("layer", [0, 1, 5, 15])
def test_pivot_error_host_replay_matches_device_thomas(layer):
    """The fused solve replays the zero-shift column on the host
    (reference.check_pivots); the device Thomas kernel of the plugin layer
    checks every column.  A crafted z-chain with a non-positive pivot at
    `layer` raises FloatingPointError naming that layer in both."""
    n = 16
    zd = z_chain_diagonal(n, ONES).copy()
    zd[layer] = -3.0
    with pytest.raises(FloatingPointError) as host:
        check_pivots(n, zd, ONES)
    fac = E.build_tridiag(P.GridSpec(4, 4, n), ONES)
    fac.z_diag = zd.astype(fac.dtype)
    fac._dev = None
    with pytest.raises(FloatingPointError) as dev:
        E.thomas_solve_batch(fac, np.ones((n, 4, 4)))
    if layer == 0:
        assert "layer" not in str(host.value) and "layer" not in str(dev.value)
    else:
        assert f"layer {layer}" in str(host.value) and f"layer {layer}" in str(dev.value)
