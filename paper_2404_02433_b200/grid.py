"""Input contract of the solve: grid, conductivity field, boundary config.

Same names, invariants and error behaviour as the reference data model
(/root/reference/pkg/src/etchomo/grid.py:24-175), so user code written
against `etchomo` constructs the same objects here.  Differences: field
arrays may also be CUDA tensors (float64), which keeps the field resident on
the device across solves; and the two inclusion generators voxelise on the
GPU (grid.py:230-275 membership test, bit-identical) instead of the host.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import struct
from pathlib import Path

import numpy as np


class ConfigError(ValueError):
    """Contract violation of a parameter (reference grid.py:24-25)."""


class Axis(str, Enum):
    X = "x"
    Y = "y"
    Z = "z"


_AXIS_INDEX = {Axis.X: 0, Axis.Y: 1, Axis.Z: 2}


def axis_index(axis) -> int:
    return _AXIS_INDEX[Axis(axis)]


@dataclass(frozen=True)
class GridSpec:
    """Cell counts and edge lengths (reference grid.py:42-90)."""

    nx: int
    ny: int
    nz: int
    lx: float = 1.0
    ly: float = 1.0
    lz: float = 1.0

    def __post_init__(self):
        for name in ("nx", "ny", "nz"):
            n = getattr(self, name)
            if not isinstance(n, (int, np.integer)) or n < 1:
                raise ConfigError(f"{name} must be a positive integer, got {n!r}")
        for name in ("lx", "ly", "lz"):
            length = float(getattr(self, name))
            if not np.isfinite(length) or length <= 0.0:
                raise ConfigError(f"{name} must be positive and finite, got {length!r}")

    @property
    def hx(self) -> float:
        return self.lx / self.nx

    @property
    def hy(self) -> float:
        return self.ly / self.ny

    @property
    def hz(self) -> float:
        return self.lz / self.nz

    @property
    def shape(self) -> tuple[int, int, int]:
        return (self.nz, self.ny, self.nx)

    @property
    def n_cells(self) -> int:
        return self.nx * self.ny * self.nz

    def cell_centers(self):
        """Coordinate arrays (X, Y, Z), each shaped (nz, ny, nx) (grid.py:84-90)."""
        cx = (np.arange(self.nx) + 0.5) * self.hx
        cy = (np.arange(self.ny) + 0.5) * self.hy
        cz = (np.arange(self.nz) + 0.5) * self.hz
        Z, Y, X = np.meshgrid(cz, cy, cx, indexing="ij")
        return X, Y, Z


def linear_index(i: int, j: int, k: int, grid: GridSpec) -> int:
    """x-fastest flat offset (reference grid.py:93-99)."""
    if not (0 <= i < grid.nx and 0 <= j < grid.ny and 0 <= k < grid.nz):
        raise IndexError(f"cell ({i}, {j}, {k}) outside grid {grid.nx}x{grid.ny}x{grid.nz}")
    return (k * grid.ny + j) * grid.nx + i


def _is_tensor(a) -> bool:
    return type(a).__module__.startswith("torch")


class OrthotropicField:
    """Per-cell (kx, ky, kz), strictly positive and finite (reference
    grid.py:102-159).  Arrays are flat x-fastest numpy arrays (frozen
    read-only) or contiguous float64 CUDA tensors.  Passing the same array
    object for all three components marks the field isotropic: it is then
    stored once on the device."""

    __slots__ = ("grid", "kx", "ky", "kz")

    def __init__(self, grid: GridSpec, kx, ky, kz, validate: bool = True):
        self.grid = grid
        src = (kx, ky, kz)
        out = []
        cache = {}
        for name, arr in zip(("kx", "ky", "kz"), src):
            if id(arr) in cache:
                out.append(cache[id(arr)])
                continue
            if _is_tensor(arr):
                a = arr.reshape(-1)
                if a.dtype.__str__() not in ("torch.float64", "torch.float32"):
                    raise ConfigError(f"{name}: CUDA fields must be float64 or float32")
                if not a.is_contiguous():
                    a = a.contiguous()
                if a.numel() != grid.n_cells:
                    raise ConfigError(f"{name} has {a.numel()} entries, expected {grid.n_cells}")
                if validate:
                    import torch

                    if not bool(torch.isfinite(a).all()) or bool((a <= 0).any()):
                        raise ConfigError(f"{name} must be strictly positive and finite")
            else:
                a = np.ascontiguousarray(arr).reshape(-1)
                if a.size != grid.n_cells:
                    raise ConfigError(f"{name} has {a.size} entries, expected {grid.n_cells}")
                if a.dtype not in (np.float64, np.float32):
                    a = a.astype(np.float64)
                if validate and (not np.all(np.isfinite(a)) or np.any(a <= 0.0)):
                    raise ConfigError(f"{name} must be strictly positive and finite")
                a.setflags(write=False)
            cache[id(arr)] = a
            out.append(a)
        dts = {str(a.dtype) for a in out}
        if len(dts) != 1:
            raise ConfigError("kx, ky, kz must share one scalar dtype")
        self.kx, self.ky, self.kz = out

    @property
    def dtype(self):
        return self.kx.dtype

    @property
    def on_device(self) -> bool:
        return _is_tensor(self.kx)

    @property
    def isotropic_storage(self) -> bool:
        return self.kx is self.ky and self.ky is self.kz

    def cube(self, component: str):
        return getattr(self, component).reshape(self.grid.shape)

    def astype(self, dtype) -> "OrthotropicField":
        """The field cast to float32 / float64 (grid.py:139-148)."""
        dtype = np.dtype(dtype)
        if dtype == np.dtype(str(self.dtype).replace("torch.", "")):
            return self
        if self.on_device:
            import torch

            td = torch.float32 if dtype == np.float32 else torch.float64
            return OrthotropicField(self.grid, self.kx.to(td), self.ky.to(td), self.kz.to(td), validate=False)
        return OrthotropicField(self.grid, self.kx.astype(dtype), self.ky.astype(dtype), self.kz.astype(dtype))

    def __eq__(self, other) -> bool:
        if not isinstance(other, OrthotropicField) or other.grid != self.grid:
            return False

        def host(a):
            return a.cpu().numpy() if _is_tensor(a) else a

        return all(np.array_equal(host(getattr(self, c)), host(getattr(other, c))) for c in ("kx", "ky", "kz"))

    __hash__ = None


@dataclass(frozen=True)
class BoundaryConfig:
    """Dirichlet axis and potentials (reference grid.py:162-175)."""

    axis: Axis
    p_in: float
    p_out: float

    def __post_init__(self):
        if not (np.isfinite(self.p_in) and np.isfinite(self.p_out)):
            raise ConfigError("p_in and p_out must be finite")
        if self.p_in == self.p_out:
            raise ConfigError("p_in must differ from p_out")


# ----------------------------------------------------------------------------
# inclusion generators, voxelised on the GPU (reference grid.py:230-284)
# ----------------------------------------------------------------------------

RANDOM_BALL_PRESETS = {
    "a": dict(count=40, r_min=0.05, r_max=0.15, kappa_inc=10.0, seed=11),
    "b": dict(count=80, r_min=0.04, r_max=0.10, kappa_inc=10.0, seed=23),
    "c": dict(count=16, r_min=0.10, r_max=0.20, kappa_inc=10.0, seed=37),
}


def draw_balls(count: int, r_min: float, r_max: float, seed: int) -> np.ndarray:
    """(count, 4) array of (cx, cy, cz, r): per ball three uniform center
    coordinates then one radius draw from PCG64(seed) (grid.py:266-272)."""
    rng = np.random.default_rng(np.uint64(seed))
    out = np.empty((count, 4))
    for b in range(count):
        out[b, :3] = rng.random(3)
        out[b, 3] = r_min + (r_max - r_min) * rng.random()
    return out


def _voxelize(n: int, balls: np.ndarray, kappa_inc: float, device, as_numpy: bool):
    import torch

    from . import _native

    dev = torch.device(device if device is not None else "cuda")
    out = torch.empty(n * n * n, dtype=torch.float64, device=dev)
    balls = np.ascontiguousarray(balls, dtype=np.float64)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = _native.lib().etc_voxelize_balls(
            out.data_ptr(), n, balls.ctypes.data_as(_native._DP), balls.shape[0],
            float(kappa_inc), stream)
    if rc != 0:
        raise RuntimeError(f"voxeliser failed: {_native.last_error()}")
    grid = GridSpec(n, n, n)
    k = out.cpu().numpy() if as_numpy else out
    return OrthotropicField(grid, k, k, k, validate=False)


def gen_random_balls(n: int, count: int, r_min: float, r_max: float, kappa_inc: float,
                     seed: int, device=None, as_numpy: bool = False) -> OrthotropicField:
    """Random isotropic ball pack (reference grid.py:244-275), same PCG64
    draw order and membership test; cells voxelised on the GPU."""
    if n < 2:
        raise ConfigError("random-balls needs n >= 2")
    if count < 1:
        raise ConfigError("count must be >= 1")
    if not (0.0 < r_min <= r_max < 0.5):
        raise ConfigError("radii must satisfy 0 < r_min <= r_max < 1/2")
    if kappa_inc <= 0.0:
        raise ConfigError("kappa_inc must be positive")
    return _voxelize(n, draw_balls(count, r_min, r_max, seed), kappa_inc, device, as_numpy)


def gen_center_ball(n: int, kappa_inc: float, device=None, as_numpy: bool = False) -> OrthotropicField:
    """Ball of radius 1/4 at the cube center (reference grid.py:230-241)."""
    if n < 2:
        raise ConfigError("center-ball needs n >= 2")
    if kappa_inc <= 0.0:
        raise ConfigError("kappa_inc must be positive")
    return _voxelize(n, np.array([[0.5, 0.5, 0.5, 0.25]]), kappa_inc, device, as_numpy)


def gen_smooth_problem(n: int):
    """Smooth manufactured problem on the unit cube (reference grid.py:182-227):
    K = Diag(cos(pi y) + 2, 2 e^z, 3 cos(pi x) + 4) at cell centres, exact
    p = cos(pi x) cos(pi y) e^z and its source f = -div(K grad p).  Returns
    (field, exact, source); the field is host data (a verification input, not
    a benchmark one), the two samplers are vectorised numpy callables."""
    if n < 2:
        raise ConfigError("smooth problem needs n >= 2")
    grid = GridSpec(n, n, n)
    X, Y, Z = grid.cell_centers()
    field = OrthotropicField(grid, np.cos(np.pi * Y) + 2.0, 2.0 * np.exp(Z), 3.0 * np.cos(np.pi * X) + 4.0)

    def exact(x, y, z):
        return np.cos(np.pi * x) * np.cos(np.pi * y) * np.exp(z)

    def source(x, y, z):
        cc = np.cos(np.pi * x) * np.cos(np.pi * y)
        return (np.pi ** 2 * (np.cos(np.pi * y) + 2.0) * cc * np.exp(z)
                + 2.0 * np.pi ** 2 * cc * np.exp(2.0 * z)
                - (3.0 * np.cos(np.pi * x) + 4.0) * cc * np.exp(z))

    return field, exact, source


# ----------------------------------------------------------------------------
# SURVEY 8(d) config 3 inputs: the reference's orthotropic channel lattice and
# a documented aligned-fibre generator (the reference has none)
# ----------------------------------------------------------------------------

FIBRE_PRESET = dict(count=24, r_min=0.04, r_max=0.08, kappa_fib=1000.0, seed=5, axis="z")


def draw_fibres(count: int, r_min: float, r_max: float, seed: int) -> np.ndarray:
    """(count, 3) array of (c1, c2, r): per fibre two uniform centre
    coordinates (the two transverse axes, increasing axis order) then one
    radius draw from PCG64(seed) -- the ball generator's draw order
    (grid.py:266-272) with the axial coordinate dropped."""
    rng = np.random.default_rng(np.uint64(seed))
    out = np.empty((count, 3))
    for f in range(count):
        out[f, :2] = rng.random(2)
        out[f, 2] = r_min + (r_max - r_min) * rng.random()
    return out


def gen_fibres(n: int, count: int, r_min: float, r_max: float, kappa_fib: float, seed: int,
               axis="z", device=None, as_numpy: bool = False) -> OrthotropicField:
    """Unidirectional fibre composite: `count` parallel cylinders through the
    whole unit cube along `axis` (radii uniform in [r_min, r_max], centres
    uniform, overlaps allowed), conductivity kappa_fib inside and 1 in the
    matrix; isotropic per phase.  Deterministic in `seed`.  Cell centres and
    the membership test ((d1*d1) + (d2*d2)) <= r*r follow the ball
    voxeliser (grid.py:86-88, 273).  Voxelised on the GPU."""
    import torch

    from . import _native

    if n < 2:
        raise ConfigError("fibres need n >= 2")
    if count < 1:
        raise ConfigError("count must be >= 1")
    if not (0.0 < r_min <= r_max < 0.5):
        raise ConfigError("radii must satisfy 0 < r_min <= r_max < 1/2")
    if kappa_fib <= 0.0:
        raise ConfigError("kappa_fib must be positive")
    ax = axis_index(axis)
    fib = np.ascontiguousarray(draw_fibres(count, r_min, r_max, seed))
    dev = torch.device(device if device is not None else "cuda")
    out = torch.empty(n * n * n, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = _native.lib().etc_voxelize_fibres(out.data_ptr(), n, fib.ctypes.data_as(_native._DP), count,
                                                float(kappa_fib), ax, stream)
    if rc != 0:
        raise RuntimeError(f"fibre voxeliser failed: {_native.last_error()}")
    k = out.cpu().numpy() if as_numpy else out
    return OrthotropicField(GridSpec(n, n, n), k, k, k, validate=False)


def gen_channels(cells_per_period: int, periods: int, psi: float, device=None,
                 as_numpy: bool = False) -> OrthotropicField:
    """Periodic lattice of three orthogonal square channels (reference
    grid.py:287-319): Diag(2^psi, 5^psi, 10^psi) in the band [3/8, 5/8) of
    each period in two transverse axes, Diag(0.01, 0.1, 1) elsewhere.  Built
    on the GPU."""
    import torch

    from . import _native

    if cells_per_period < 8 or cells_per_period % 8 != 0:
        raise ConfigError("cells_per_period must be a positive multiple of 8")
    if periods < 1:
        raise ConfigError("periods must be >= 1")
    if psi <= 0.0:
        raise ConfigError("psi must be positive")
    n = cells_per_period * periods
    dev = torch.device(device if device is not None else "cuda")
    k = [torch.empty(n * n * n, dtype=torch.float64, device=dev) for _ in range(3)]
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = _native.lib().etc_fill_channels(k[0].data_ptr(), k[1].data_ptr(), k[2].data_ptr(), cells_per_period,
                                              periods, 2.0 ** psi, 5.0 ** psi, 10.0 ** psi, stream)
    if rc != 0:
        raise RuntimeError(f"channel generator failed: {_native.last_error()}")
    if as_numpy:
        k = [t.cpu().numpy() for t in k]
    return OrthotropicField(GridSpec(n, n, n), k[0], k[1], k[2], validate=False)


# ----------------------------------------------------------------------------
# ETCVOX01 container (reference grid.py:18-21, 28-34, 322-371)
# ----------------------------------------------------------------------------

VOX_MAGIC = b"ETCVOX01"
_VOX_HEADER = struct.Struct("<8s3I3dB")  # magic, nx ny nz, lx ly lz, dtype code
_VOX_DTYPE_BY_CODE = {0: np.dtype("<f8"), 1: np.dtype("<f4")}


class VoxFormatError(ValueError):
    """Malformed ETCVOX payload; carries the byte offset of the defect."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (byte offset {offset})")
        self.offset = offset


def write_vox(field, destination, dtype=np.float64) -> None:
    """Serialise a field (host arrays or CUDA tensors) to the single-file
    little-endian ETCVOX container: header, then kx, ky, kz."""
    dt = np.dtype(dtype)
    code = {np.dtype(np.float64): 0, np.dtype(np.float32): 1}[dt]
    g = field.grid
    with open(Path(destination), "wb") as fh:
        fh.write(_VOX_HEADER.pack(VOX_MAGIC, g.nx, g.ny, g.nz, g.lx, g.ly, g.lz, code))
        for a in (field.kx, field.ky, field.kz):
            if _is_tensor(a):
                a = a.detach().cpu().numpy()
            fh.write(np.ascontiguousarray(a, dtype=_VOX_DTYPE_BY_CODE[code]).tobytes())


def read_vox(source, device=None) -> OrthotropicField:
    """Parse an ETCVOX container with the reference's checks and error
    offsets (truncated header, bad magic, unknown dtype code, bad dimensions,
    payload size, first non-positive or non-finite entry).  f32 payloads are
    widened to f64 (exact).  device: also place the arrays on that CUDA
    device (one H2D copy; the solver then uses them in place)."""
    raw = Path(source).read_bytes()
    if len(raw) < _VOX_HEADER.size:
        raise VoxFormatError("truncated header", len(raw))
    magic, nx, ny, nz, lx, ly, lz, code = _VOX_HEADER.unpack_from(raw, 0)
    if magic != VOX_MAGIC:
        raise VoxFormatError(f"bad magic {magic!r}", 0)
    if code not in _VOX_DTYPE_BY_CODE:
        raise VoxFormatError(f"unknown dtype code {code}", _VOX_HEADER.size - 1)
    try:
        grid = GridSpec(int(nx), int(ny), int(nz), lx, ly, lz)
    except ConfigError as exc:
        raise VoxFormatError(f"bad dimensions: {exc}", 8) from exc
    scalar = _VOX_DTYPE_BY_CODE[code]
    count = grid.nx * grid.ny * grid.nz
    expected = _VOX_HEADER.size + 3 * count * scalar.itemsize
    if len(raw) != expected:
        raise VoxFormatError(f"payload holds {len(raw)} bytes, expected {expected}", min(len(raw), expected))
    arrays = []
    for idx, name in enumerate(("kx", "ky", "kz")):
        start = _VOX_HEADER.size + idx * count * scalar.itemsize
        a = np.frombuffer(raw, dtype=scalar, count=count, offset=start)
        bad = ~(np.isfinite(a) & (a > 0))
        if np.any(bad):
            first = int(np.argmax(bad))
            raise VoxFormatError(f"non-positive {name} entry at cell {first}", start + first * scalar.itemsize)
        arrays.append(a.astype(np.float64))
    if device is not None:
        import torch

        arrays = [torch.from_numpy(a).to(device) for a in arrays]
    return OrthotropicField(grid, *arrays, validate=False)
