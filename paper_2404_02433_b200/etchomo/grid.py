"""etchomo.grid facade (reference grid.py): the data model, with the
generators returning host fields like the reference's."""

from ..grid import (  # noqa: F401
    Axis,
    BoundaryConfig,
    ConfigError,
    GridSpec,
    OrthotropicField,
    RANDOM_BALL_PRESETS,
    VoxFormatError,
    gen_smooth_problem,
    linear_index,
    read_vox,
    write_vox,
)
from .. import grid as _g


def gen_random_balls(n, count, r_min, r_max, kappa_inc, seed):
    """Reference grid.py:244-275 (voxelised on the GPU, returned on the host)."""
    return _g.gen_random_balls(n, count, r_min, r_max, kappa_inc, seed, as_numpy=True)


def gen_center_ball(n, kappa_inc):
    """Reference grid.py:230-241 (voxelised on the GPU, returned on the host)."""
    return _g.gen_center_ball(n, kappa_inc, as_numpy=True)


def gen_channels(cells_per_period, periods, psi):
    """Reference grid.py:287-319 (built on the GPU, returned on the host)."""
    return _g.gen_channels(cells_per_period, periods, psi, as_numpy=True)
