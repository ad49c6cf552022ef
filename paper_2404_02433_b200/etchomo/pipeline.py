"""etchomo.pipeline facade (reference pipeline.py): the drop-in homogenize
(the fused device solve) and axis_permute."""

from ..plugin import axis_permute  # noqa: F401
from ..solver import homogenize  # noqa: F401
