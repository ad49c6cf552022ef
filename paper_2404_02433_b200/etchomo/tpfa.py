"""etchomo.tpfa facade (reference tpfa.py)."""

from ..plugin import (  # noqa: F401
    DENSE_GUARD,
    DiscreteSystem,
    add_source,
    apply_operator,
    assemble_dense,
    assemble_sparse,
    build_rhs,
    build_system,
    effective_conductivity,
    l2_error_midpoint,
    operator_diagonal,
    reconstruct_boundary_flux,
    scale_field,
)
