"""etchomo.preconditioner facade (reference preconditioner.py)."""

from ..plugin import (  # noqa: F401
    FctPreconditioner,
    JacobiPreconditioner,
    SsorPreconditioner,
    TridiagFactors,
    build_tridiag,
    coefficient_stats,
    fct_precond_apply,
    identity_apply,
    jacobi_apply,
    reference_system,
    ssor_apply,
    thomas_solve_batch,
)
from ..reference import CoefficientStats, ReferenceParams, ones_reference, solve_reference_lp  # noqa: F401
