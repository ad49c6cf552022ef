"""B200-native effective-thermal-conductivity solver (arXiv 2404.02433).

Drop-in for the reference `etchomo.homogenize()` path: a voxel conductivity
field goes in, kappa_eff and the PCG residual history come out.  The O(N)
work runs in hand-written sm_100a CUDA kernels (libetc_b200.so, C ABI in
include/etc_b200.h); there is no CPU fallback.
"""

from .grid import (
    Axis,
    BoundaryConfig,
    ConfigError,
    GridSpec,
    OrthotropicField,
    FIBRE_PRESET,
    RANDOM_BALL_PRESETS,
    draw_balls,
    draw_fibres,
    gen_center_ball,
    gen_channels,
    gen_fibres,
    gen_random_balls,
    linear_index,
    read_vox,
    VoxFormatError,
    write_vox,
)
from .reference import (
    CoefficientStats,
    ReferenceParams,
    eigen_weights,
    ones_reference,
    solve_reference_lp,
    z_chain_diagonal,
)
from .solver import (
    DevicePlan,
    PcgBreakdownError,
    SolveReport,
    effective_tensor,
    get_plan,
    homogenize,
    homogenize_with_solution,
    release_plans,
)
from .operators import DeviceSystem
from ._native import NativeUnavailable
# the reference's operator-plugin layer under its own names (plugin.py;
# reference __init__.py:9-71)
from .plugin import (
    DiscreteSystem,
    FctPlan,
    FctPreconditioner,
    JacobiPreconditioner,
    SlabBuffer,
    TridiagFactors,
    add_source,
    apply_operator,
    assemble_dense,
    axis_permute,
    build_rhs,
    build_system,
    build_tridiag,
    coefficient_stats,
    condition_estimate,
    dct1d_ref_backward,
    dct1d_ref_forward,
    dense_solve,
    effective_conductivity,
    fct_backward_batch,
    fct_forward_batch,
    fct_pre_permute,
    fct_precond_apply,
    identity_apply,
    jacobi_apply,
    l2_error_midpoint,
    operator_diagonal,
    pcg,
    reconstruct_boundary_flux,
    reference_system,
    scale_field,
    ssor_apply,
    thomas_solve_batch,
)
from .grid import gen_smooth_problem

__version__ = "0.1.0"
