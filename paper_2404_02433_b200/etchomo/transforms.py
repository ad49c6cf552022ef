"""etchomo.transforms facade (reference transforms.py)."""

from ..plugin import (  # noqa: F401
    FctPlan,
    SlabBuffer,
    dct1d_ref_backward,
    dct1d_ref_forward,
    fct_backward_batch,
    fct_forward_batch,
    fct_pre_permute,
)
