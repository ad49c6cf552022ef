"""Operator-level device entry points: the plugin callables the reference's
`pcg` consumes (krylov.py:36-42) — the stencil `apply_operator`
(tpfa.py:110-131) and the `FctPreconditioner` (preconditioner.py:273-282) —
plus the transform and tridiagonal stages (transforms.py:83-133,
preconditioner.py:215-250).  Each maps a length-N float64 vector (CUDA
tensor, or numpy array copied to the device) to a NEW vector, like the
reference callables.
"""

from __future__ import annotations

import numpy as np

from .grid import Axis, BoundaryConfig, ConfigError
from .reference import ReferenceParams, ones_reference, solve_reference_lp
from .solver import _as_field, _check, _torch, get_plan


class DeviceSystem:
    """Canonical (z-oriented) system of one field on the GPU."""

    def __init__(self, field, boundary: BoundaryConfig | None = None, ref_mode: str = "opt",
                 refs: ReferenceParams | None = None, device=None):
        fld = _as_field(field)
        self.boundary = boundary or BoundaryConfig(Axis.Z, 1.0, 0.0)
        self.plan = get_plan(fld.grid, device)
        self.plan.load_field(fld, force=True)
        self.grid = self.plan.select_axis(self.boundary.axis)
        self.plan.set_precision("f64")  # the operator-level entry points are float64
        self.stats = self.plan.coefficient_stats()
        if refs is None:
            refs = solve_reference_lp(self.stats) if ref_mode == "opt" else ones_reference(self.stats)
        self.refs = refs
        self.plan.set_reference(refs)
        self.device = self.plan.device

    # -- helpers -------------------------------------------------------------
    def _in(self, u):
        torch = _torch()
        if isinstance(u, np.ndarray):
            u = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64)).to(self.device)
        u = u.reshape(-1)
        if u.numel() != self.grid.n_cells:
            raise ValueError(f"vector has {u.numel()} entries, expected {self.grid.n_cells}")
        if u.dtype != torch.float64:
            raise ConfigError("vectors must be float64")
        return u.contiguous()

    def _new(self):
        torch = _torch()
        return torch.empty(self.grid.n_cells, dtype=torch.float64, device=self.device)

    def _run(self, fn, *args):
        torch = _torch()
        with torch.cuda.device(self.device):
            _check(fn(self.plan.handle, *args), fn.__name__)

    # -- operators -------------------------------------------------------------
    def apply_operator(self, u):
        u = self._in(u)
        out = self._new()
        self._run(self.plan.lib.etc_apply_operator, u.data_ptr(), out.data_ptr())
        return out

    def precondition(self, r):
        r = self._in(r)
        out = self._new()
        self._run(self.plan.lib.etc_apply_precond, r.data_ptr(), out.data_ptr())
        return out

    __call__ = precondition

    def dct2_xy(self, u):
        u = self._in(u)
        out = self._new()
        self._run(self.plan.lib.etc_dct2_xy, u.data_ptr(), out.data_ptr())
        return out

    def dct3_xy(self, c):
        c = self._in(c)
        out = self._new()
        self._run(self.plan.lib.etc_dct3_xy, c.data_ptr(), out.data_ptr())
        return out

    def thomas(self, x):
        out = self._in(x).clone()
        self._run(self.plan.lib.etc_thomas, out.data_ptr())
        return out

    def build_rhs(self):
        out = self._new()
        self._run(self.plan.lib.etc_build_rhs, float(self.boundary.p_in), float(self.boundary.p_out),
                  out.data_ptr())
        return out
