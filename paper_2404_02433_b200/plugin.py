"""The reference's operator-plugin layer on the GPU, under its own names.

`homogenize()` (solver.py) is the fused hot path.  This module is the
lower-level API of the reference package (/root/reference/pkg/src/etchomo/
__init__.py:9-71) that user code composes by hand: `build_system` /
`DiscreteSystem` / `apply_operator` (tpfa.py), `FctPreconditioner` /
`thomas_solve_batch` / `coefficient_stats` (preconditioner.py), `FctPlan` /
`fct_forward_batch` (transforms.py) and `pcg(apply_A, apply_M_inv, b, ...)`
(krylov.py:36-91).  Same signatures, argument meaning, return values and
exceptions; every O(N) operation runs in libetc_b200.so (etc_plugin.cu for the
stateless kernels, the plan-based transform and preconditioner entry points
of etc_b200.cu) and there is no CPU path.

Array convention (what makes it a drop-in): an operation returns the array
type it was given.  numpy in -> the data is copied to the device, computed
there, and a numpy array comes back (the reference's own tests run this way);
a CUDA tensor in -> a CUDA tensor out, no host traffic.  Inputs are never
mutated (the reference's ownership rule); outputs are fresh.
dtype float64 or float32 is threaded through exactly as the reference does.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native
from .grid import Axis, BoundaryConfig, ConfigError, GridSpec, OrthotropicField
from .reference import (
    CoefficientStats,
    ReferenceParams,
    eigen_weights,
    ones_reference,
    solve_reference_lp,
    z_chain_diagonal,
)

DENSE_GUARD = 4096  # tpfa.py:15


# ---------------------------------------------------------------------------
# array plumbing (host <-> device, dtype, stream)
# ---------------------------------------------------------------------------
def _torch():
    import torch

    return torch


def _lib():
    return _native.lib()


def _is_tensor(a) -> bool:
    return type(a).__module__.startswith("torch")


def _device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise _native.NativeUnavailable("no CUDA device visible: the plugin layer has no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _stream(dev=None) -> int:
    torch = _torch()
    return torch.cuda.current_stream(dev).cuda_stream


def _np_dtype(a) -> np.dtype:
    if _is_tensor(a):
        return np.dtype(str(a.dtype).replace("torch.", ""))
    return np.asarray(a).dtype


def _prec(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return 0
    if dt == np.float32:
        return 1
    raise ConfigError(f"arrays must be float64 or float32, got {dt}")


def _tdtype(dtype):
    torch = _torch()
    return torch.float64 if np.dtype(dtype) == np.float64 else torch.float32


def _to_dev(a, dtype=None):
    """Flat contiguous CUDA tensor view/copy of `a` (numpy, list or tensor)."""
    torch = _torch()
    if _is_tensor(a):
        t = a
        if t.device.type != "cuda":
            t = t.to(_device())
        if dtype is not None and t.dtype != _tdtype(dtype):
            t = t.to(_tdtype(dtype))
        return t.reshape(-1).contiguous()
    arr = np.asarray(a)
    if dtype is not None:
        arr = arr.astype(dtype, copy=False)
    elif arr.dtype not in (np.float64, np.float32):
        arr = arr.astype(np.float64)
    arr = np.ascontiguousarray(arr).reshape(-1)
    if not arr.flags.writeable:  # frozen field arrays: torch wants a writable buffer
        arr = arr.copy()
    return torch.from_numpy(arr).to(_device())


def _empty(n, dtype):
    torch = _torch()
    return torch.empty(int(n), dtype=_tdtype(dtype), device=_device())


def _back(t, like_numpy: bool, shape=None):
    """Result in the caller's array type."""
    if like_numpy:
        out = t.cpu().numpy()
        return out.reshape(shape) if shape is not None else out
    return t.reshape(shape) if shape is not None else t


def _ptr(t) -> int:
    return t.data_ptr()


def _ck(rc: int, what: str) -> None:
    if rc == _native.ETC_OK:
        return
    lib = _lib()
    msg = (lib.etc_op_last_error() or b"").decode() or (lib.etc_last_error() or b"").decode()
    if rc == _native.ETC_CONFIG:
        raise ConfigError(f"{what}: {msg}")
    if rc == _native.ETC_PIVOT:
        raise FloatingPointError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


class _Scratch:
    """Per-device reduction scratch (partials + outputs), grown on demand."""

    _bufs: dict = {}

    @classmethod
    def get(cls, n: int):
        torch = _torch()
        dev = _device()
        need = int(_lib().etc_op_reduce_parts(int(max(n, 1)))) + 8
        buf = cls._bufs.get(dev.index)
        if buf is None or buf.numel() < need:
            buf = torch.empty(need, dtype=torch.float64, device=dev)
            cls._bufs[dev.index] = buf
        return buf


def _reduce(kind: int, a, b=None) -> list:
    """Deterministic device reductions (float64 accumulation): kind 0 a.b,
    1 (a.b, a.a, b.b), 2 sum(a)."""
    n = a.numel()
    buf = _Scratch.get(n)
    out = buf[-8:]
    _ck(_lib().etc_op_dots(_prec(_np_dtype(a)), kind, n, _ptr(a), _ptr(b) if b is not None else _ptr(a),
                            _ptr(buf), _ptr(out), _stream()), "etc_op_dots")
    vals = out[: 3 if kind == 1 else 1].cpu().tolist()
    return vals


def _round(v: float, dtype) -> float:
    """A float64 sum as numpy reports it for the array dtype (float32 dots
    come back as float32 numbers)."""
    return float(np.float32(v)) if np.dtype(dtype) == np.float32 else float(v)


# ---------------------------------------------------------------------------
# tpfa.py: scale_field, DiscreteSystem, build_system, apply_operator, ...
# ---------------------------------------------------------------------------
def scale_field(field: OrthotropicField):
    """Per-cell scaled coefficients k/h^2, one (nz, ny, nx) array per axis
    (tpfa.py:19-26): a division by dtype(h)**2, on the device."""
    g = field.grid
    dt = _np_dtype(field.kx)
    numpy_in = not _is_tensor(field.kx)
    out = []
    for comp, h in (("kx", g.hx), ("ky", g.hy), ("kz", g.hz)):
        k = _to_dev(getattr(field, comp), dt)
        h2 = float(dt.type(h) ** 2)
        s = _empty(g.n_cells, dt)
        _ck(_lib().etc_op_scale(_prec(dt), g.n_cells, _ptr(k), h2, _ptr(s), _stream()), "etc_op_scale")
        out.append(_back(s, numpy_in, g.shape))
    return tuple(out)


class DiscreteSystem:
    """Assembled transmissibilities of the canonical z-oriented problem
    (tpfa.py:33-88): tx (nx-1)*ny*nz, ty nx*(ny-1)*nz, tz nx*ny*(nz-1),
    t_in / t_out nx*ny, flat x-fastest, strictly positive.  The arrays are
    numpy or CUDA tensors (the type the system was built from); a device copy
    of the faces is kept for the kernels."""

    __slots__ = ("grid", "tx", "ty", "tz", "t_in", "t_out", "boundary", "_dev")

    def __init__(self, grid, tx, ty, tz, t_in, t_out, boundary, validate: bool = True):
        self.grid = grid
        arrs = []
        for a in (tx, ty, tz, t_in, t_out):
            arrs.append(a.reshape(-1).contiguous() if _is_tensor(a) else np.ascontiguousarray(a).reshape(-1))
        self.tx, self.ty, self.tz, self.t_in, self.t_out = arrs
        self.boundary = boundary
        self._dev = None
        nx, ny, nz = grid.nx, grid.ny, grid.nz
        sizes = {
            "tx": (self.tx, (nx - 1) * ny * nz),
            "ty": (self.ty, nx * (ny - 1) * nz),
            "tz": (self.tz, nx * ny * (nz - 1)),
            "t_in": (self.t_in, nx * ny),
            "t_out": (self.t_out, nx * ny),
        }
        for name, (arr, want) in sizes.items():
            size = arr.numel() if _is_tensor(arr) else arr.size
            if size != want:
                raise ConfigError(f"{name} has {size} entries, expected {want}")
        if validate:
            for name, (arr, want) in sizes.items():
                if not want:
                    continue
                if _is_tensor(arr):
                    torch = _torch()
                    bad = (not bool(torch.isfinite(arr).all())) or bool((arr <= 0).any())
                else:
                    bad = (not np.all(np.isfinite(arr))) or bool(np.any(arr <= 0))
                if bad:
                    raise ConfigError(f"{name} must be strictly positive")

    @property
    def dtype(self) -> np.dtype:
        return _np_dtype(self.tx)

    @property
    def on_device(self) -> bool:
        return _is_tensor(self.tx)

    def faces_x(self):
        g = self.grid
        return self.tx.reshape(g.nz, g.ny, g.nx - 1)

    def faces_y(self):
        g = self.grid
        return self.ty.reshape(g.nz, g.ny - 1, g.nx)

    def faces_z(self):
        g = self.grid
        return self.tz.reshape(g.nz - 1, g.ny, g.nx)

    def layer_in(self):
        g = self.grid
        return self.t_in.reshape(g.ny, g.nx)

    def layer_out(self):
        g = self.grid
        return self.t_out.reshape(g.ny, g.nx)

    def device_faces(self):
        """(tx, ty, tz, t_in, t_out) as CUDA tensors (copied once for numpy systems)."""
        if self._dev is None:
            dt = self.dtype
            torch = _torch()
            faces = []
            for a in (self.tx, self.ty, self.tz, self.t_in, self.t_out):
                t = _to_dev(a, dt)
                if t.numel() == 0:  # a valid pointer for empty face groups
                    t = torch.zeros(1, dtype=t.dtype, device=t.device)
                faces.append(t)
            self._dev = tuple(faces)
        return self._dev


def build_system(field: OrthotropicField, boundary: BoundaryConfig) -> DiscreteSystem:
    """Assemble the canonical system (tpfa.py:91-107): harmonic faces
    ((2a)*b)/(a+b) and t_in/t_out = 2 s_z, built on the device from the
    scaled coefficients (bitwise numpy's)."""
    if Axis(boundary.axis) is not Axis.Z:
        raise ConfigError("build_system expects axis z; permute the field first (pipeline.axis_permute)")
    g = field.grid
    dt = _np_dtype(field.kx)
    numpy_in = not _is_tensor(field.kx)
    nx, ny, nz = g.nx, g.ny, g.nz
    s = []
    for comp, h in (("kx", g.hx), ("ky", g.hy), ("kz", g.hz)):
        k = _to_dev(getattr(field, comp), dt)
        out = _empty(g.n_cells, dt)
        _ck(_lib().etc_op_scale(_prec(dt), g.n_cells, _ptr(k), float(dt.type(h) ** 2), _ptr(out), _stream()),
            "etc_op_scale")
        s.append(out)
    sizes = ((nx - 1) * ny * nz, nx * (ny - 1) * nz, nx * ny * (nz - 1), nx * ny, nx * ny)
    faces = [_empty(max(m, 1), dt) for m in sizes]
    _ck(_lib().etc_op_faces(_prec(dt), nx, ny, nz, *[_ptr(a) for a in s], *[_ptr(f) for f in faces], _stream()),
        "etc_op_faces")
    faces = [f[:m] for f, m in zip(faces, sizes)]
    out = [_back(f, numpy_in) for f in faces]
    sys = DiscreteSystem(g, *out, boundary, validate=False)
    sys._dev = tuple(f if f.numel() else _empty(1, dt) for f in faces)
    return sys


def _vec(sys, u, what="vector"):
    g = sys.grid
    n = u.numel() if _is_tensor(u) else np.asarray(u).size
    if n != g.n_cells:
        raise ValueError(f"{what} has {n} entries, expected {g.n_cells}")
    return _to_dev(u, sys.dtype)


def apply_operator(sys: DiscreteSystem, u):
    """Matrix-free stencil product (tpfa.py:110-131), bitwise numpy's."""
    g = sys.grid
    numpy_in = not _is_tensor(u)
    ud = _vec(sys, u)
    out = _empty(g.n_cells, sys.dtype)
    _ck(_lib().etc_op_stencil(_prec(sys.dtype), g.nx, g.ny, g.nz, *[_ptr(f) for f in sys.device_faces()],
                              _ptr(ud), _ptr(out), _stream()), "etc_op_stencil")
    return _back(out, numpy_in)


def operator_diagonal(sys: DiscreteSystem):
    """Diagonal of the stencil (tpfa.py:134-147)."""
    g = sys.grid
    out = _empty(g.n_cells, sys.dtype)
    _ck(_lib().etc_op_diagonal(_prec(sys.dtype), g.nx, g.ny, g.nz, *[_ptr(f) for f in sys.device_faces()],
                               _ptr(out), _stream()), "etc_op_diagonal")
    return _back(out, not sys.on_device)


def build_rhs(sys: DiscreteSystem, dirichlet_in=None, dirichlet_out=None):
    """Right-hand side carrying the Dirichlet data (tpfa.py:150-167): the
    boundary config's constants, or (ny, nx) planes of face samples."""
    g = sys.grid
    dt = sys.dtype
    plane = g.nx * g.ny

    def side(v, default):
        if v is None:
            return None, float(dt.type(default))
        if np.isscalar(v) or (not _is_tensor(v) and np.asarray(v).ndim == 0):
            return None, float(dt.type(v))
        a = _to_dev(v, dt)
        if a.numel() != plane:
            a = _to_dev(np.broadcast_to(np.asarray(v if not _is_tensor(v) else v.cpu()), (g.ny, g.nx)), dt)
        return a, 0.0

    pin_a, pin = side(dirichlet_in, sys.boundary.p_in)
    pout_a, pout = side(dirichlet_out, sys.boundary.p_out)
    out = _empty(g.n_cells, dt)
    t = sys.device_faces()
    _ck(_lib().etc_op_rhs(_prec(dt), g.nx, g.ny, g.nz, _ptr(t[3]), _ptr(t[4]),
                          _ptr(pin_a) if pin_a is not None else None, pin,
                          _ptr(pout_a) if pout_a is not None else None, pout, _ptr(out), _stream()), "etc_op_rhs")
    return _back(out, not sys.on_device)


def add_source(sys: DiscreteSystem, b, source):
    """b + midpoint source samples (tpfa.py:170-178).  The sampler is a
    user callable of host coordinates; the sum runs on the device."""
    X, Y, Z = cell_centers(sys.grid)
    samples = np.asarray(source(X, Y, Z), dtype=sys.dtype)
    if not np.all(np.isfinite(samples)):
        raise ValueError("source sampler returned non-finite values")
    numpy_in = not _is_tensor(b)
    bd = _vec(sys, b, "rhs")
    sd = _to_dev(samples, sys.dtype)
    out = _empty(sys.grid.n_cells, sys.dtype)
    _ck(_lib().etc_op_elementwise(_prec(sys.dtype), 2, sys.grid.n_cells, _ptr(bd), _ptr(sd), _ptr(out), _stream()),
        "etc_op_elementwise")
    return _back(out, numpy_in)


def cell_centers(grid: GridSpec):
    """Coordinate arrays (X, Y, Z), each (nz, ny, nx) (grid.py:84-90)."""
    cx = (np.arange(grid.nx) + 0.5) * grid.hx
    cy = (np.arange(grid.ny) + 0.5) * grid.hy
    cz = (np.arange(grid.nz) + 0.5) * grid.hz
    Z, Y, X = np.meshgrid(cz, cy, cx, indexing="ij")
    return X, Y, Z


def reconstruct_boundary_flux(sys: DiscreteSystem, p, side: str = "out"):
    """Unscaled z-flux through the Dirichlet faces (tpfa.py:234-251)."""
    if side not in ("in", "out"):
        raise ValueError(f"side must be 'in' or 'out', got {side!r}")
    g = sys.grid
    dt = sys.dtype
    numpy_in = not _is_tensor(p)
    pd = _vec(sys, p, "potential")
    out = _empty(g.nx * g.ny, dt)
    t = sys.device_faces()
    layer = t[4] if side == "out" else t[3]
    pval = float(dt.type(sys.boundary.p_out if side == "out" else sys.boundary.p_in))
    _ck(_lib().etc_op_flux(_prec(dt), g.nx, g.ny, g.nz, _ptr(layer), float(dt.type(g.hz)), _ptr(pd), pval,
                           1 if side == "out" else 0, _ptr(out), _stream()), "etc_op_flux")
    return _back(out, numpy_in)


def effective_conductivity(sys: DiscreteSystem, fluxes) -> float:
    """kappa_eff = l_z sum(flux) / (nx ny (p_in - p_out)) (tpfa.py:254-258),
    the flux sum a float64 device reduction."""
    g = sys.grid
    f = _to_dev(fluxes)
    total = _reduce(2, f)[0]
    drop = sys.boundary.p_in - sys.boundary.p_out
    return float(g.lz * total / (g.nx * g.ny * drop))


def l2_error_midpoint(grid: GridSpec, p, exact) -> float:
    """Midpoint-quadrature L2 distance between a cell vector and a sampler
    (tpfa.py:261-265); the squared sum is a device reduction."""
    X, Y, Z = cell_centers(grid)
    pd = _to_dev(p, np.float64)
    diff = _empty(grid.n_cells, np.float64)
    neg = _to_dev(-np.asarray(exact(X, Y, Z), dtype=np.float64))  # p - e as p + (-e), exact negation
    _ck(_lib().etc_op_elementwise(0, 2, grid.n_cells, _ptr(pd), _ptr(neg), _ptr(diff), _stream()),
        "etc_op_elementwise")
    ss = _reduce(0, diff, diff)[0]
    return float(math.sqrt(ss * grid.hx * grid.hy * grid.hz))


def assemble_dense(sys: DiscreteSystem):
    """Explicit symmetric matrix of the stencil (tpfa.py:181-205; small-grid
    verification helper), filled on the device in np.add.at's accumulation order."""
    g = sys.grid
    n = g.n_cells
    if n > DENSE_GUARD:
        raise ValueError(f"dense assembly capped at {DENSE_GUARD} cells, got {n}")
    torch = _torch()
    t = [_to_dev(f, np.float64) if f.numel() else torch.zeros(1, dtype=torch.float64, device=_device())
         for f in sys.device_faces()]
    mat = torch.empty(n * n, dtype=torch.float64, device=_device())
    _ck(_lib().etc_op_dense(g.nx, g.ny, g.nz, *[_ptr(f) for f in t], _ptr(mat), _stream()), "etc_op_dense")
    return _back(mat, not sys.on_device, (n, n))


def assemble_sparse(sys: DiscreteSystem):
    """CSR form of the operator (tpfa.py:208-231), a host scipy structure
    built from the device-assembled dense matrix (verification sizes) or, above
    the dense guard, from the face arrays."""
    import scipy.sparse as sp

    g = sys.grid
    n = g.n_cells
    if n <= DENSE_GUARD:
        mat = assemble_dense(sys)
        mat = mat.cpu().numpy() if _is_tensor(mat) else mat
        return sp.csr_matrix(mat)
    idx = np.arange(n).reshape(g.shape)
    host = [f.cpu().numpy() if _is_tensor(f) else f for f in (sys.tx, sys.ty, sys.tz)]
    diag = operator_diagonal(sys)
    diag = diag.cpu().numpy() if _is_tensor(diag) else diag
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [diag]
    for (left, right), t in (((idx[:, :, :-1], idx[:, :, 1:]), host[0]), ((idx[:, 1:, :], idx[:, :-1, :]), host[1]),
                             ((idx[1:], idx[:-1]), host[2])):
        rows += [left.ravel(), right.ravel()]
        cols += [right.ravel(), left.ravel()]
        vals += [-t, -t]
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()


# ---------------------------------------------------------------------------
# pipeline.py: axis_permute
# ---------------------------------------------------------------------------
def axis_permute(field: OrthotropicField, axis) -> OrthotropicField:
    """Swap the requested axis with z (pipeline.py:87-111): X does
    swapaxes(0, 2) and kx <-> kz, Y swapaxes(0, 1) and ky <-> kz.  The
    transposes run on the device."""
    axis = Axis(axis)
    if axis is Axis.Z:
        return field
    g = field.grid
    dt = _np_dtype(field.kx)
    numpy_in = not _is_tensor(field.kx)

    def swap(a, ax):
        src = _to_dev(a, dt)
        dst = _empty(g.n_cells, dt)
        _ck(_lib().etc_op_permute(_prec(dt), g.nx, g.ny, g.nz, ax, _ptr(src), _ptr(dst), _stream()),
            "etc_op_permute")
        return _back(dst, numpy_in)

    if axis is Axis.X:
        new_grid = GridSpec(g.nz, g.ny, g.nx, g.lz, g.ly, g.lx)
        return OrthotropicField(new_grid, swap(field.kz, 0), swap(field.ky, 0), swap(field.kx, 0))
    new_grid = GridSpec(g.nx, g.nz, g.ny, g.lx, g.lz, g.ly)
    return OrthotropicField(new_grid, swap(field.kx, 1), swap(field.kz, 1), swap(field.ky, 1))


# ---------------------------------------------------------------------------
# preconditioner.py
# ---------------------------------------------------------------------------
def coefficient_stats(sys: DiscreteSystem) -> CoefficientStats:
    """Exact extremes of the stored transmissibilities (preconditioner.py:94-108):
    device min/max; an empty face group gives (1, 1); in/out use t/2."""
    torch = _torch()
    mm = torch.empty(2, dtype=torch.int64, device=_device())
    faces = sys.device_faces()
    sizes = (sys.tx, sys.ty, sys.tz, sys.t_in, sys.t_out)
    vals = []
    for gi, (f, a) in enumerate(zip(faces, sizes)):
        n = a.numel() if _is_tensor(a) else a.size
        if n == 0:
            vals += [1.0, 1.0]
            continue
        out = (C.c_double * 2)()
        _ck(_lib().etc_op_minmax(_prec(sys.dtype), n, _ptr(f), _ptr(mm), out, _stream()), "etc_op_minmax")
        lo, hi = float(out[0]), float(out[1])
        if gi >= 3:  # t_in / 2.0, t_out / 2.0 in the array dtype (exact halving)
            lo, hi = float(sys.dtype.type(lo) / sys.dtype.type(2.0)), float(sys.dtype.type(hi) / sys.dtype.type(2.0))
        vals += [lo, hi]
    return CoefficientStats(*vals)


def reference_system(grid: GridSpec, refs: ReferenceParams, boundary: BoundaryConfig | None = None,
                     dtype=np.float64) -> DiscreteSystem:
    """The reference operator as a stencil system (preconditioner.py:143-164)."""
    if boundary is None:
        boundary = BoundaryConfig(Axis.Z, 1.0, 0.0)
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    dt = np.dtype(dtype)
    return DiscreteSystem(grid, np.full((nx - 1) * ny * nz, refs.kx_ref, dtype=dt),
                          np.full(nx * (ny - 1) * nz, refs.ky_ref, dtype=dt),
                          np.full(nx * ny * (nz - 1), refs.kz_ref, dtype=dt),
                          np.full(nx * ny, 2.0 * refs.kin_ref, dtype=dt),
                          np.full(nx * ny, 2.0 * refs.kout_ref, dtype=dt), boundary)


class TridiagFactors:
    """Per-mode tridiagonal data (preconditioner.py:167-209): eigen weights
    2(1 - cos(q pi/N)), plane_shift = w_x kx_ref + w_y ky_ref in float64 cast
    to dtype, the z-chain diagonal and off = -kz_ref.  Host tables (O(nx ny +
    nz)), mirrored on the device on first use."""

    __slots__ = ("grid", "refs", "dtype", "weights_x", "weights_y", "plane_shift", "z_diag", "off", "_dev")

    def __init__(self, grid: GridSpec, refs: ReferenceParams, dtype=np.float64):
        self.grid = grid
        self.refs = refs
        self.dtype = np.dtype(dtype)
        self.weights_x = eigen_weights(grid.nx)
        self.weights_y = eigen_weights(grid.ny)
        shift = self.weights_x[None, :] * refs.kx_ref + self.weights_y[:, None] * refs.ky_ref
        self.plane_shift = shift.astype(self.dtype)
        self.z_diag = z_chain_diagonal(grid.nz, refs).astype(self.dtype)
        self.off = self.dtype.type(-refs.kz_ref)
        self._dev = None

    def device_tables(self):
        if self._dev is None:
            self._dev = (_to_dev(self.plane_shift, self.dtype), _to_dev(self.z_diag, self.dtype))
        return self._dev

    def dense_block(self, i: int, j: int) -> np.ndarray:
        """Explicit (nz, nz) matrix of one transformed mode (test helper)."""
        nz = self.grid.nz
        t = np.diag(self.z_diag.astype(np.float64).copy())
        t += np.diag(np.full(nz - 1, float(self.off)), 1)
        t += np.diag(np.full(nz - 1, float(self.off)), -1)
        t += float(self.plane_shift[j, i]) * np.eye(nz)
        return t


def build_tridiag(grid: GridSpec, refs: ReferenceParams, dtype=np.float64) -> TridiagFactors:
    return TridiagFactors(grid, refs, dtype)


def thomas_solve_batch(factors: TridiagFactors, rhs, overwrite: bool = False):
    """Every (i', j') z-column against its tridiagonal block
    (preconditioner.py:215-250): one device thread per column, the
    reference's elimination elementwise (bitwise), FloatingPointError on a
    non-positive pivot."""
    g = factors.grid
    dt = factors.dtype
    numpy_in = not _is_tensor(rhs)
    if not numpy_in and overwrite and rhs.dtype == _tdtype(dt) and rhs.is_contiguous() and rhs.is_cuda:
        x = rhs.reshape(-1)  # in place, as overwrite=True asks
    else:
        x = _to_dev(rhs, dt)
        if not numpy_in and x.data_ptr() == rhs.data_ptr():
            x = x.clone()  # never mutate the caller's tensor unless asked
    shift, zd = factors.device_tables()
    upper = _empty(max((g.nz - 1) * g.nx * g.ny, 1), dt)
    torch = _torch()
    bad_dev = torch.empty(1, dtype=torch.int32, device=_device())
    bad = C.c_int(-1)
    rc = _lib().etc_op_thomas(_prec(dt), g.nx, g.ny, g.nz, _ptr(shift), _ptr(zd), float(factors.off), _ptr(x),
                              _ptr(upper), _ptr(bad_dev), C.byref(bad), _stream())
    if rc == _native.ETC_PIVOT:
        if bad.value <= 0:
            raise FloatingPointError("non-positive pivot in tridiagonal solve")
        raise FloatingPointError(f"non-positive pivot in tridiagonal solve at layer {bad.value}")
    _ck(rc, "etc_op_thomas")
    shape = rhs.shape if not _is_tensor(rhs) else tuple(rhs.shape)
    if numpy_in:
        out = x.cpu().numpy().reshape(shape)
        if overwrite:
            np.copyto(rhs, out.astype(rhs.dtype, copy=False))
            return rhs
        return out
    return x.reshape(shape)


class _BarePlan:
    """A geometry-only device plan (etc_plan_bare) with transform tables and
    reference constants set: what FctPlan and FctPreconditioner drive."""

    def __init__(self, nx: int, ny: int, nz: int, refs: ReferenceParams | None):
        import weakref

        torch = _torch()
        self.lib = _lib()
        self.device = _device()
        self.h = C.c_void_p()
        with torch.cuda.device(self.device):
            _ck(self.lib.etc_plan_create(C.byref(self.h), nx, ny, nz, 1.0, 1.0, 1.0, _stream()), "etc_plan_create")
        self._fin = weakref.finalize(self, self.lib.etc_plan_destroy, self.h)
        _ck(self.lib.etc_plan_bare(self.h), "etc_plan_bare")
        refs = refs or ReferenceParams(1.0, 1.0, 1.0, 1.0, 1.0)
        wx, wy = eigen_weights(nx), eigen_weights(ny)
        zd = z_chain_diagonal(nz, refs)
        dp = _native._DP
        r5 = (C.c_double * 5)(*refs.constants())
        _ck(self.lib.etc_set_reference(self.h, r5, wx.ctypes.data_as(dp), wy.ctypes.data_as(dp),
                                       zd.ctypes.data_as(dp)), "etc_set_reference")


# ---------------------------------------------------------------------------
# transforms.py: FctPlan, SlabBuffer, fct_forward_batch, fct_backward_batch
# ---------------------------------------------------------------------------
def _halving_order(n: int) -> np.ndarray:
    """Even indices ascending, then odd indices descending (transforms.py:41-43)."""
    return np.concatenate([np.arange(0, n, 2), np.arange(1, n, 2)[::-1]])


def fct_pre_permute(v, out=None):
    """Four-quadrant even/odd reshuffle of one (ny, nx) slice (transforms.py:46-53):
    a pure gather (numpy or device indexing)."""
    ny, nx = v.shape
    if _is_tensor(v):
        torch = _torch()
        oy = torch.as_tensor(_halving_order(ny), device=v.device)
        ox = torch.as_tensor(_halving_order(nx), device=v.device)
        g = v.index_select(0, oy).index_select(1, ox)
        if out is None:
            return g
        out.copy_(g)
        return out
    gathered = np.asarray(v)[np.ix_(_halving_order(ny), _halving_order(nx))]
    if out is None:
        return gathered
    out[...] = gathered
    return out


def dct1d_ref_forward(u):
    """Direct-summation forward transform (transforms.py:24-30; the O(N^2)
    verification helper), a cosine-table product on the device."""
    torch = _torch()
    numpy_in = not _is_tensor(u)
    x = _to_dev(u, np.float64)
    n = x.numel()
    i = torch.arange(n, dtype=torch.float64, device=x.device)
    table = torch.cos(math.pi * (2 * i[None, :] + 1) * i[:, None] / (2 * n))
    return _back(table @ x, numpy_in)


def dct1d_ref_backward(uh):
    """Direct-summation backward transform (transforms.py:33-38)."""
    torch = _torch()
    numpy_in = not _is_tensor(uh)
    x = _to_dev(uh, np.float64)
    n = x.numel()
    i = torch.arange(n, dtype=torch.float64, device=x.device)
    w = torch.where(i == 0, 0.5, 1.0)
    table = torch.cos(math.pi * (2 * i[:, None] + 1) * i[None, :] / (2 * n))
    return _back((2.0 / n) * (table @ (w * x)), numpy_in)


class FctPlan:
    """Transform tables for one slab shape (transforms.py:56-133) on the
    device.  forward / backward map a (nz, ny, nx) array to a new one and
    return (out, None): the half spectrum of the reference's numpy path is an
    internal stage of the fused plane kernels and is not materialised."""

    def __init__(self, nx: int, ny: int, nz: int, dtype=np.float64):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.dtype = np.dtype(dtype)
        _prec(self.dtype)
        self.half = ny // 2 + 1
        self.order_x = _halving_order(nx)
        self.order_y = _halving_order(ny)
        self._plan = None

    def spectrum_shape(self) -> tuple[int, int, int]:
        return (self.nz, self.half, self.nx)

    def _bare(self):
        if self._plan is None:
            self._plan = _BarePlan(self.nx, self.ny, self.nz, None)
        return self._plan

    def _run(self, data, inverse: bool):
        numpy_in = not _is_tensor(data)
        shape = (self.nz, self.ny, self.nx)
        x = _to_dev(data, self.dtype)
        if x.numel() != self.nx * self.ny * self.nz:
            raise ValueError(f"slab has {x.numel()} entries, expected {self.nx * self.ny * self.nz}")
        out = _empty(x.numel(), self.dtype)
        bp = self._bare()
        if self.dtype == np.float64:
            fn = bp.lib.etc_dct3_xy if inverse else bp.lib.etc_dct2_xy
        else:
            fn = bp.lib.etc_dct3_xy_f32 if inverse else bp.lib.etc_dct2_xy_f32
        _ck(fn(bp.h, _ptr(x), _ptr(out)), fn.__name__)
        return _back(out, numpy_in, shape), None

    def forward(self, data):
        return self._run(data, False)

    def backward(self, coeff):
        return self._run(coeff, True)


class SlabBuffer:
    """A (nz, ny, nx) slab bound to a plan (transforms.py:136-163); `data` is
    a numpy array or a CUDA tensor."""

    __slots__ = ("plan", "data", "spectrum")

    def __init__(self, plan: FctPlan, data=None):
        self.plan = plan
        shape = (plan.nz, plan.ny, plan.nx)
        if data is None:
            data = np.zeros(shape, dtype=plan.dtype)
        elif _is_tensor(data):
            data = data.reshape(shape)
        else:
            data = np.ascontiguousarray(data, dtype=plan.dtype).reshape(shape)
        self.data = data
        self.spectrum = None

    @property
    def nx(self) -> int:
        return self.plan.nx

    @property
    def ny(self) -> int:
        return self.plan.ny

    @property
    def nz(self) -> int:
        return self.plan.nz


def fct_forward_batch(buf: SlabBuffer) -> SlabBuffer:
    """Forward-transform every k-slice (transforms.py:166-170)."""
    buf.data, buf.spectrum = buf.plan.forward(buf.data)
    return buf


def fct_backward_batch(buf: SlabBuffer) -> SlabBuffer:
    """Backward-transform every k-slice (transforms.py:173-177)."""
    buf.data, buf.spectrum = buf.plan.backward(buf.data)
    return buf


class FctPreconditioner:
    """z = A_ref^-1 r (preconditioner.py:273-282): 2-D DCT-II per z-plane,
    per-mode z-solve, 2-D DCT-III, in the device plan's fused kernels."""

    def __init__(self, grid: GridSpec, refs: ReferenceParams, dtype=np.float64):
        self.grid = grid
        self.refs = refs
        self.dtype = np.dtype(dtype)
        _prec(self.dtype)
        self.factors = build_tridiag(grid, refs, dtype)
        from .reference import check_pivots

        check_pivots(grid.nz, z_chain_diagonal(grid.nz, refs), refs, self.dtype)
        self._plan = _BarePlan(grid.nx, grid.ny, grid.nz, refs)

    def __call__(self, r):
        numpy_in = not _is_tensor(r)
        n = self.grid.n_cells
        x = _to_dev(r, self.dtype)
        if x.numel() != n:
            raise ValueError(f"vector has {x.numel()} entries, expected {n}")
        out = _empty(n, self.dtype)
        bp = self._plan
        fn = bp.lib.etc_apply_precond if self.dtype == np.float64 else bp.lib.etc_apply_precond_f32
        _ck(fn(bp.h, _ptr(x), _ptr(out)), fn.__name__)
        return _back(out, numpy_in)


def fct_precond_apply(factors: TridiagFactors, r, plan: FctPlan | None = None, buf: SlabBuffer | None = None):
    """Inverse reference operator (preconditioner.py:253-266)."""
    return FctPreconditioner(factors.grid, factors.refs, factors.dtype)(r)


class JacobiPreconditioner:
    """r * (1/diag A) (preconditioner.py:324-330)."""

    def __init__(self, sys: DiscreteSystem):
        d = _to_dev(operator_diagonal(sys), sys.dtype)
        self._dtype = sys.dtype
        self._inv = _empty(d.numel(), sys.dtype)
        _ck(_lib().etc_op_elementwise(_prec(sys.dtype), 1, d.numel(), _ptr(d), _ptr(d), _ptr(self._inv), _stream()),
            "etc_op_elementwise")

    def __call__(self, r):
        numpy_in = not _is_tensor(r)
        x = _to_dev(r, self._dtype)
        out = _empty(x.numel(), self._dtype)
        _ck(_lib().etc_op_elementwise(_prec(self._dtype), 0, x.numel(), _ptr(x), _ptr(self._inv), _ptr(out),
                                      _stream()), "etc_op_elementwise")
        return _back(out, numpy_in)


def jacobi_apply(sys: DiscreteSystem, r):
    return JacobiPreconditioner(sys)(r)


def identity_apply(r):
    """identity_apply (preconditioner.py:337-338): a copy."""
    if _is_tensor(r):
        return r.clone()
    return np.array(r, copy=True)


class SsorPreconditioner:
    """Symmetric over-relaxation (preconditioner.py:285-321): y = (L +
    D/w)^-1 r, y *= diag, y = (U + D/w)^-1 y, y *= (2 - w)/w, in float64
    whatever the system dtype (the reference factors the float64 sparse
    matrix), cast back on return.  The triangular sweeps run on the device
    level-scheduled over hyperplanes (etc_op_ssor)."""

    def __init__(self, sys: DiscreteSystem, omega: float = 1.0):
        if not 0.0 < omega < 2.0:
            raise ConfigError(f"omega must lie in (0, 2), got {omega}")
        self.omega = float(omega)
        self._sys = sys
        self._dtype = sys.dtype
        torch = _torch()
        self._faces = [(_to_dev(f, np.float64) if f.numel() else torch.zeros(1, dtype=torch.float64,
                                                                             device=_device()))
                       for f in sys.device_faces()]
        d = operator_diagonal(DiscreteSystem(sys.grid, *[f[: n] for f, n in zip(self._faces, self._sizes(sys))],
                                             sys.boundary, validate=False))
        self._diag = _to_dev(d, np.float64)

    @staticmethod
    def _sizes(sys):
        g = sys.grid
        nx, ny, nz = g.nx, g.ny, g.nz
        return ((nx - 1) * ny * nz, nx * (ny - 1) * nz, nx * ny * (nz - 1), nx * ny, nx * ny)

    def __call__(self, r):
        g = self._sys.grid
        numpy_in = not _is_tensor(r)
        x = _to_dev(r, np.float64)
        if x.numel() != g.n_cells:
            raise ValueError(f"vector has {x.numel()} entries, expected {g.n_cells}")
        out = _empty(g.n_cells, np.float64)
        f = self._faces
        _ck(_lib().etc_op_ssor(g.nx, g.ny, g.nz, _ptr(f[0]), _ptr(f[1]), _ptr(f[2]), _ptr(self._diag), self.omega,
                               _ptr(x), _ptr(out), _stream()), "etc_op_ssor")
        if self._dtype != np.float64:
            out = out.to(_tdtype(self._dtype))
        return _back(out, numpy_in)


def ssor_apply(sys: DiscreteSystem, omega: float, r):
    """One-shot SSOR application (preconditioner.py:324-327)."""
    return SsorPreconditioner(sys, omega)(r)


# ---------------------------------------------------------------------------
# krylov.py: pcg, dense_solve, condition_estimate
# ---------------------------------------------------------------------------
def pcg(apply_A, apply_M_inv, b, rtol: float, max_iter: int = 1024):
    """Conjugate gradients on A p = b with a fixed SPD preconditioner
    (krylov.py:36-91, Alg. 1 statement for statement).  The vector algebra
    runs in fused device kernels (p += alpha w with r -= alpha z and |r|^2
    in one pass; w = z + beta w; deterministic float64 dots); the scalars are
    host floats, as in the reference.  The callables map a vector to a NEW
    vector of b's array type: numpy b -> numpy vectors (host round trips
    around each callable), CUDA-tensor b -> tensors (no host traffic)."""
    if rtol <= 0.0:
        raise ValueError("rtol must be positive")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    from .solver import PcgBreakdownError, SolveReport

    numpy_in = not _is_tensor(b)
    dt = _np_dtype(b) if not numpy_in else np.asarray(b).dtype
    if dt not in (np.float64, np.float32):
        dt = np.dtype(np.float64)
    prec = _prec(dt)
    eps = float(np.finfo(dt).eps)
    bd = _to_dev(b, dt)
    n = bd.numel()
    lib = _lib()
    buf = _Scratch.get(n)
    torch = _torch()

    def call(fn, v):
        if numpy_in:
            return _to_dev(fn(v.cpu().numpy()), dt)  # a fresh device copy
        out = fn(v)
        return out.clone() if out is v else _to_dev(out, dt)

    def norm(sq: float) -> float:
        return float(np.sqrt(np.float32(sq))) if dt == np.float32 else math.sqrt(sq)

    rb = _reduce(0, bd, bd)[0]
    norm_b = norm(rb)
    p = torch.zeros(n, dtype=_tdtype(dt), device=bd.device)
    if norm_b == 0.0:
        return _back(p, numpy_in, np.shape(b) if numpy_in else None), SolveReport(0, True, [0.0])
    r = bd.clone()
    z = call(apply_M_inv, r)
    w = z.clone()
    rho = _round(_reduce(0, r, z)[0], dt)
    if rho <= 0.0:
        raise PcgBreakdownError("preconditioned inner product not positive", 0)
    history = [norm(_reduce(0, r, r)[0]) / norm_b]
    iteration = 0
    out = buf[-8:]
    while history[-1] > rtol and iteration < max_iter:
        z = call(apply_A, w)
        zw, zz, ww = _reduce(1, z, w)
        zw = _round(zw, dt)
        if zw <= 100.0 * eps * norm(zz) * norm(ww):
            raise PcgBreakdownError("operator inner product lost positivity", iteration + 1)
        alpha = rho / zw
        _ck(lib.etc_op_pcg_update(prec, n, float(dt.type(alpha)), _ptr(p), _ptr(w), _ptr(r), _ptr(z), _ptr(buf),
                                  _ptr(out), _stream()), "etc_op_pcg_update")
        relres = norm(float(out[0].item())) / norm_b
        if not np.isfinite(relres):
            raise PcgBreakdownError("residual is not finite", iteration + 1)
        history.append(relres)
        iteration += 1
        if relres <= rtol:
            break
        z = call(apply_M_inv, r)
        rho_next = _round(_reduce(0, r, z)[0], dt)
        if rho_next <= 0.0:
            raise PcgBreakdownError("preconditioned inner product not positive", iteration)
        _ck(lib.etc_op_xpby(prec, n, _ptr(z), float(dt.type(rho_next / rho)), _ptr(w), _stream()), "etc_op_xpby")
        rho = rho_next
    return _back(p, numpy_in, np.shape(b) if numpy_in else None), SolveReport(iteration, history[-1] <= rtol,
                                                                                history)


def dense_solve(mat, b):
    """Direct Cholesky solve of a dense SPD system (krylov.py:94-105; verification helper),
    cuSOLVER through torch.linalg on the device."""
    torch = _torch()
    numpy_in = not _is_tensor(b)
    m = _to_dev(mat, np.float64)
    k = int(round(math.sqrt(m.numel())))
    if k > 4096:
        raise ValueError("dense solves capped at 4096 unknowns")
    m = m.reshape(k, k)
    L, info = torch.linalg.cholesky_ex(m)
    if int(info.item()) != 0:
        raise ValueError(f"matrix is not positive definite: leading minor {int(info.item())} not positive")
    x = torch.cholesky_solve(_to_dev(b, np.float64).reshape(k, 1), L).reshape(-1)
    return _back(x, numpy_in)


def condition_estimate(mat, mat_ref=None):
    """Extreme eigenvalues and condition number of a dense SPD matrix or of
    the pencil (mat, mat_ref) (krylov.py:108-125; verification helper), cuSOLVER eigvalsh
    on the device (the pencil through the reference matrix's Cholesky factor)."""
    torch = _torch()
    m = _to_dev(mat, np.float64)
    k = int(round(math.sqrt(m.numel())))
    if k > 4096:
        raise ValueError("eigen estimates capped at 4096 unknowns")
    m = m.reshape(k, k)
    if mat_ref is None:
        vals = torch.linalg.eigvalsh(m)
    else:
        ref = _to_dev(mat_ref, np.float64).reshape(k, k)
        L, info = torch.linalg.cholesky_ex(ref)
        if int(info.item()) != 0:
            raise ValueError("reference matrix is singular or indefinite")
        y = torch.linalg.solve_triangular(L, m, upper=False)
        c = torch.linalg.solve_triangular(L, y.T, upper=False)
        vals = torch.linalg.eigvalsh(0.5 * (c + c.T))
    lam_min, lam_max = float(vals[0]), float(vals[-1])
    return lam_min, lam_max, lam_max / lam_min


__all__ = [
    "DiscreteSystem", "FctPlan", "FctPreconditioner", "JacobiPreconditioner", "SlabBuffer", "SsorPreconditioner",
    "TridiagFactors", "add_source", "apply_operator", "assemble_dense", "assemble_sparse", "axis_permute",
    "build_rhs", "build_system", "build_tridiag", "cell_centers", "coefficient_stats", "condition_estimate",
    "dct1d_ref_backward", "dct1d_ref_forward", "dense_solve", "effective_conductivity", "fct_backward_batch",
    "fct_forward_batch", "fct_pre_permute", "fct_precond_apply", "identity_apply", "jacobi_apply",
    "l2_error_midpoint", "operator_diagonal", "pcg", "reconstruct_boundary_flux", "reference_system",
    "scale_field", "ssor_apply", "thomas_solve_batch",
]
