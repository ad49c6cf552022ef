"""etchomo.krylov facade (reference krylov.py)."""

from ..plugin import condition_estimate, dense_solve, pcg  # noqa: F401
from ..solver import PcgBreakdownError, SolveReport  # noqa: F401
