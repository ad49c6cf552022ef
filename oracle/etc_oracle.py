"""CPU ORACLE — test infrastructure only, never the product path.

A plain-numpy restatement of the reference `etchomo` hot path (arXiv 2404.02433,
`/root/reference/pkg/src/etchomo`): TPFA stencil, reference-medium (FCT)
preconditioner, PCG (Alg. 1) and the homogenize() orchestration.  It is used
by `tests/` as the checker, by `__graft_entry__.smoke()` as the checker, and
by `bench.py` as the CPU baseline ("kind": "port").  Nothing in
`paper_2404_02433_b200/` imports it.

Parity pinning: the functions below were validated against the reference
itself (imported from /root/reference in the build container) by
`tests/golden/make_golden.py`, which wrote the committed fixtures in
`tests/golden/`; `tests/test_oracle_golden.py` re-checks the oracle against
those fixtures and against the reference's own known-answer values
(two-cell matrix, harmonic 2/101, DCT [2,0] / [1, sqrt(2)/2], impulse 1/4, ...).

Array convention (reference `grid.py:1-7`): cell (i, j, k) lives at flat index
(k*ny + j)*nx + i, i.e. a C-ordered (nz, ny, nx) cube.
"""

from __future__ import annotations

import math

import numpy as np

try:  # multithreaded pocketfft for the CPU baseline; same transform family as numpy.fft
    import scipy.fft as _sfft
except Exception:  # pragma: no cover
    _sfft = None

# ----------------------------------------------------------------------------
# discretization (reference tpfa.py)
# ----------------------------------------------------------------------------


def scale(k: np.ndarray, h: float) -> np.ndarray:
    """k / h^2 with h^2 formed as dtype(h)**2 and a true division (tpfa.py:19-26)."""
    return k / (k.dtype.type(h) ** 2)


def harmonic(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Face transmissibility ((2a)*b)/(a+b), a = lower cell (tpfa.py:29-30)."""
    return 2.0 * a * b / (a + b)


def faces(sx, sy, sz):
    """Interior faces and the two Dirichlet layers (tpfa.py:91-107).

    Returns tx (nz,ny,nx-1), ty (nz,ny-1,nx), tz (nz-1,ny,nx), t_in, t_out (ny,nx)."""
    tx = harmonic(sx[:, :, :-1], sx[:, :, 1:])
    ty = harmonic(sy[:, :-1, :], sy[:, 1:, :])
    tz = harmonic(sz[:-1, :, :], sz[1:, :, :])
    return tx, ty, tz, 2.0 * sz[0], 2.0 * sz[-1]


def stencil(fc, u: np.ndarray, reverse: bool = False) -> np.ndarray:
    """Matrix-free 7-point operator, same per-cell association order as
    tpfa.py:110-131: +fx(i-1/2) -fx(i+1/2) +fy.. -fy.. +fz.. -fz.., then the
    Dirichlet layers.  reverse=True accumulates z, y, x instead (the
    "perturbed oracle" of SURVEY.md 8(c): same maths, other rounding)."""
    tx, ty, tz, t_in, t_out = fc
    nz, ny, nx = u.shape
    out = np.zeros_like(u)
    order = ((tx, 2), (ty, 1), (tz, 0))
    for t, axis in (order[::-1] if reverse else order):
        if u.shape[axis] < 2:
            continue
        hi = [slice(None)] * 3
        lo = [slice(None)] * 3
        hi[axis] = slice(1, None)
        lo[axis] = slice(None, -1)
        hi, lo = tuple(hi), tuple(lo)
        f = t * (u[hi] - u[lo])
        out[hi] += f
        out[lo] -= f
    out[0] += t_in * u[0]
    out[-1] += t_out * u[-1]
    return out


def rhs(fc, shape, p_in: float, p_out: float) -> np.ndarray:
    """b = t_in*p_in on k=0 plus t_out*p_out on k=nz-1 (tpfa.py:150-167)."""
    _, _, _, t_in, t_out = fc
    b = np.zeros(shape, dtype=t_in.dtype)
    b[0] = t_in * p_in
    b[-1] += t_out * p_out
    return b


def outflow_kappa(fc, p: np.ndarray, grid, p_in: float, p_out: float) -> float:
    """kappa_eff from the outflow-face fluxes (tpfa.py:234-258)."""
    nx, ny, nz, lx, ly, lz = grid
    t_out = fc[4]
    hz = t_out.dtype.type(lz / nz)
    flux = t_out * hz * (p[-1] - t_out.dtype.type(p_out))
    return float(lz * np.sum(flux, dtype=np.float64) / (nx * ny * (p_in - p_out)))


# ----------------------------------------------------------------------------
# reference constants (reference preconditioner.py:94-140)
# ----------------------------------------------------------------------------

GROUPS = ("x", "y", "z", "in", "out")


def stats(fc) -> dict:
    """Exact extremes per direction group; an empty group is (1, 1) (:94-108)."""
    tx, ty, tz, t_in, t_out = fc
    out = {}
    for name, arr in zip(GROUPS, (tx, ty, tz, t_in / 2.0, t_out / 2.0)):
        out[name] = (1.0, 1.0) if arr.size == 0 else (float(arr.min()), float(arr.max()))
    return out


def reference_constants(st: dict, mode: str = "opt") -> dict:
    """Closed-form min-max LP (:117-130) or all-ones (:133-140), with the bounds."""
    if mode == "opt":
        refs = {d: math.sqrt(lo * hi) for d, (lo, hi) in st.items()}
    else:
        refs = {d: 1.0 for d in GROUPS}
    lam_lo = min(st[d][0] / refs[d] for d in GROUPS)
    lam_hi = max(st[d][1] / refs[d] for d in GROUPS)
    return dict(refs, lambda_lo=lam_lo, lambda_hi=lam_hi)


def tables(nx: int, ny: int, nz: int, refs: dict, dtype=np.float64):
    """Eigen-weights, per-mode plane shift and z-chain diagonal (:167-199)."""
    wx = 2.0 * (1.0 - np.cos(np.arange(nx) * np.pi / nx))
    wy = 2.0 * (1.0 - np.cos(np.arange(ny) * np.pi / ny))
    shift = (wx[None, :] * refs["x"] + wy[:, None] * refs["y"]).astype(dtype)
    zd = np.full(nz, 2.0 * refs["z"])
    if nz == 1:
        zd[0] = 0.0
    else:
        zd[0] = refs["z"]
        zd[-1] = refs["z"]
    zd[0] += 2.0 * refs["in"]
    zd[-1] += 2.0 * refs["out"]
    return wx, wy, shift, zd.astype(dtype), dtype(-refs["z"])


# ----------------------------------------------------------------------------
# cosine transforms (reference transforms.py:9-15 conventions; Makhoul per axis)
# ----------------------------------------------------------------------------


def _order(n: int) -> np.ndarray:
    return np.concatenate([np.arange(0, n, 2), np.arange(n - 1 - (n % 2), 0, -2)])


def _rfft(x, axis, workers):
    if workers and _sfft is not None:
        return _sfft.rfft(x, axis=axis, workers=workers)
    return np.fft.rfft(x, axis=axis)


def _irfft(x, n, axis, workers):
    if workers and _sfft is not None:
        return _sfft.irfft(x, n=n, axis=axis, workers=workers)
    return np.fft.irfft(x, n=n, axis=axis)


def dct2(v: np.ndarray, axis: int, workers: int = 0) -> np.ndarray:
    """Unnormalised DCT-II along one axis: sum_i v[i] cos(pi (2i+1) q / 2N)."""
    n = v.shape[axis]
    w = np.take(v, _order(n), axis=axis)
    half = _rfft(w, axis, workers)  # W[0..n//2]
    q = np.arange(n)
    src = np.where(q <= n // 2, q, n - q)
    sgn = np.where(q <= n // 2, 1.0, -1.0)
    full = np.take(half, src, axis=axis)
    bshape = [1] * v.ndim
    bshape[axis] = n
    c = np.cos(np.pi * q / (2 * n)).reshape(bshape)
    s = (np.sin(np.pi * q / (2 * n)) * sgn).reshape(bshape)
    return c * full.real + s * full.imag


def dct3(c: np.ndarray, axis: int, workers: int = 0) -> np.ndarray:
    """Inverse of dct2 (reference transforms.py:12-13 normalisation)."""
    n = c.shape[axis]
    h = n // 2 + 1
    q = np.arange(h)
    bshape = [1] * c.ndim
    bshape[axis] = h
    cq = np.take(c, q, axis=axis)
    mirror = np.take(c, (n - q) % n, axis=axis) * (q > 0).reshape(bshape)
    tw = np.exp(1j * np.pi * q / (2 * n)).reshape(bshape)
    spec = tw * (cq - 1j * mirror)
    w = _irfft(spec, n, axis, workers)
    out = np.empty_like(c)
    idx = [slice(None)] * c.ndim
    idx[axis] = _order(n)
    out[tuple(idx)] = w
    return out


def fct_forward(u: np.ndarray, workers: int = 0) -> np.ndarray:
    """Plane-wise 2-D DCT-II over (x, y) of an (nz, ny, nx) cube (transforms.py:83-104)."""
    return dct2(dct2(u, 2, workers), 1, workers)


def fct_backward(c: np.ndarray, workers: int = 0) -> np.ndarray:
    """Exact inverse of fct_forward (transforms.py:108-133)."""
    return dct3(dct3(c, 1, workers), 2, workers)


def thomas(shift, zd, off, x: np.ndarray) -> np.ndarray:
    """Per-mode non-pivoting elimination along z (preconditioner.py:215-250).

    Raises FloatingPointError on a non-positive pivot, like the reference."""
    x = x.copy()
    nz = x.shape[0]
    d0 = zd[0] + shift
    if np.any(d0 <= 0):
        raise FloatingPointError("non-positive pivot in tridiagonal solve")
    if nz == 1:
        x[0] /= d0
        return x
    cp = np.empty((nz - 1,) + shift.shape, dtype=x.dtype)
    cp[0] = off / d0
    x[0] = x[0] / d0
    for k in range(1, nz):
        den = (zd[k] + shift) - off * cp[k - 1]
        if np.any(den <= 0):
            raise FloatingPointError(f"non-positive pivot in tridiagonal solve at layer {k}")
        if k < nz - 1:
            cp[k] = off / den
        x[k] = (x[k] - off * x[k - 1]) / den
    for k in range(nz - 2, -1, -1):
        x[k] -= cp[k] * x[k + 1]
    return x


def thomas_bottom_up(shift, zd, off, x: np.ndarray) -> np.ndarray:
    """Same per-mode solve eliminating from the last layer upwards: a valid
    second elimination order (perturbed oracle; no pivot checks)."""
    return thomas(shift, zd[::-1].copy(), off, x[::-1])[::-1].copy()


def precond(tab, r: np.ndarray, workers: int = 0, reverse: bool = False) -> np.ndarray:
    """z = B T F r (preconditioner.py:253-282)."""
    _, _, shift, zd, off = tab
    solve = thomas_bottom_up if reverse else thomas
    return fct_backward(solve(shift, zd, off, fct_forward(r, workers)), workers)


def _dct_tables(n: int):
    i = np.arange(n)
    fwd = np.cos(np.pi * (2 * i[None, :] + 1) * i[:, None] / (2 * n))  # uh = C u (transforms.py:9-15)
    w = np.where(i == 0, 0.5, 1.0)
    bwd = (2.0 / n) * np.cos(np.pi * (2 * i[:, None] + 1) * i[None, :] / (2 * n)) * w[None, :]
    return fwd, bwd


def precond_matmul(tab, r: np.ndarray) -> np.ndarray:
    """z = B T F r with the cosine transforms as dense matrix products (the
    direct sums of transforms.py:24-38, BLAS-ordered): a third valid
    rounding of the same preconditioner, independent of any FFT, used to
    measure the implementation spread at contrast 1000."""
    _, _, shift, zd, off = tab
    nz, ny, nx = r.shape
    fx, bx = _dct_tables(nx)
    fy, by = _dct_tables(ny)
    t = np.einsum("pj,kjq->kpq", fy, np.einsum("qi,kji->kjq", fx, r, optimize=True), optimize=True)
    t = thomas(shift, zd, off, t)
    return np.einsum("jp,kpi->kji", by, np.einsum("iq,kpq->kpi", bx, t, optimize=True), optimize=True)


# ----------------------------------------------------------------------------
# PCG (reference krylov.py:36-91, Alg. 1)
# ----------------------------------------------------------------------------


class Breakdown(RuntimeError):
    def __init__(self, message, iteration):
        super().__init__(f"{message} at iteration {iteration}")
        self.iteration = iteration


def _fsum_dot(a, b):
    return math.fsum((a * b).tolist())


def _fsum_norm(a):
    return math.sqrt(math.fsum((a * a).tolist()))


def pcg(apply_a, apply_m, b: np.ndarray, rtol: float, max_iter: int = 1024, exact_dots: bool = False):
    """Returns (p, iterations, history).  Same update order and stop tests as
    krylov.py:56-91: p0 = 0, relres checked after the r update, M applied only
    when not yet converged.  exact_dots=True uses exactly rounded dots/norms
    (perturbed oracle)."""
    dot = _fsum_dot if exact_dots else (lambda x, y: float(np.dot(x, y)))
    nrm = _fsum_norm if exact_dots else (lambda x: float(np.linalg.norm(x)))
    if rtol <= 0.0:
        raise ValueError("rtol must be positive")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    eps = float(np.finfo(b.dtype).eps)
    nb = nrm(b)
    p = np.zeros_like(b)
    if nb == 0.0:
        return p, 0, [0.0]
    r = b.copy()
    z = apply_m(r)
    w = z.copy()
    rho = dot(r, z)
    if rho <= 0.0:
        raise Breakdown("preconditioned inner product not positive", 0)
    hist = [nrm(r) / nb]
    it = 0
    one = b.dtype.type
    while hist[-1] > rtol and it < max_iter:
        q = apply_a(w)
        qw = dot(q, w)
        if qw <= 100.0 * eps * nrm(q) * nrm(w):
            raise Breakdown("operator inner product lost positivity", it + 1)
        alpha = rho / qw
        p += one(alpha) * w
        r -= one(alpha) * q
        rel = nrm(r) / nb
        if not np.isfinite(rel):
            raise Breakdown("residual is not finite", it + 1)
        hist.append(rel)
        it += 1
        if rel <= rtol:
            break
        z = apply_m(r)
        rho_new = dot(r, z)
        if rho_new <= 0.0:
            raise Breakdown("preconditioned inner product not positive", it)
        w = z + one(rho_new / rho) * w
        rho = rho_new
    return p, it, hist


# ----------------------------------------------------------------------------
# orchestration (reference pipeline.py:87-175)
# ----------------------------------------------------------------------------


def permute(kx, ky, kz, grid, axis: str):
    """Swap `axis` with z (pipeline.py:87-111); cubes are (nz, ny, nx)."""
    nx, ny, nz, lx, ly, lz = grid
    if axis == "z":
        return kx, ky, kz, grid
    if axis == "x":
        sw = lambda a: np.ascontiguousarray(np.swapaxes(a, 0, 2))
        return sw(kz), sw(ky), sw(kx), (nz, ny, nx, lz, ly, lx)
    if axis == "y":
        sw = lambda a: np.ascontiguousarray(np.swapaxes(a, 0, 1))
        return sw(kx), sw(kz), sw(ky), (nx, nz, ny, lx, lz, ly)
    raise ValueError(axis)


def operator_diagonal(fc, shape) -> np.ndarray:
    """Diagonal of the 7-point operator, numpy accumulation order of
    tpfa.py:134-147 (x faces from the left then the right, then y, z, then the
    two Dirichlet layers)."""
    tx, ty, tz, tin, tout = fc
    d = np.zeros(shape)
    d[:, :, 1:] += tx
    d[:, :, :-1] += tx
    d[:, 1:, :] += ty
    d[:, :-1, :] += ty
    d[1:, :, :] += tz
    d[:-1, :, :] += tz
    d[0] += tin
    d[-1] += tout
    return d


def jacobi_inverse_diagonal(fc, shape) -> np.ndarray:
    """JacobiPreconditioner._inv_diag = 1.0 / operator_diagonal (preconditioner.py:324-330)."""
    return 1.0 / operator_diagonal(fc, shape)


def homogenize(kx, ky, kz, grid, axis="z", p_in=1.0, p_out=0.0, rtol=1e-9,
               ref_mode="opt", max_iter=1024, workers: int = 0, perturbed: bool = False,
               precond: str = "fct", dct: str = "fft") -> dict:
    """kx, ky, kz: (nz, ny, nx) cubes; grid = (nx, ny, nz, lx, ly, lz).
    perturbed=True: reversed stencil association, bottom-up z elimination and
    exactly rounded dots (same algorithm, different rounding).
    dct="matmul": the preconditioner's cosine transforms as dense matrix
    products instead of FFTs (precond_matmul).
    precond: "fct" (the FCT preconditioner), "jacobi" (r * 1/diag(A),
    preconditioner.py:324-330) or "none" (a copy of r, :337-338), selected as
    pipeline.py:114-132 does."""
    precond_fct = globals()["precond"]
    kx, ky, kz, g = permute(kx, ky, kz, grid, axis)
    nx, ny, nz, lx, ly, lz = g
    s = (scale(kx, lx / nx), scale(ky, ly / ny), scale(kz, lz / nz))
    fc = faces(*s)
    st = stats(fc)
    refs = reference_constants(st, ref_mode)
    tab = tables(nx, ny, nz, refs, kx.dtype.type)
    b = rhs(fc, kx.shape, p_in, p_out).reshape(-1)
    shape = kx.shape
    if precond == "fct" and dct == "matmul":
        apply_m = lambda r: precond_matmul(tab, r.reshape(shape)).reshape(-1)  # noqa: E731
    elif precond == "fct":
        apply_m = lambda r: precond_fct(tab, r.reshape(shape), workers, perturbed).reshape(-1)  # noqa: E731
    elif precond == "jacobi":
        invd = jacobi_inverse_diagonal(fc, shape).reshape(-1)
        apply_m = lambda r: r * invd  # noqa: E731
    elif precond == "none":
        apply_m = lambda r: r.copy()  # noqa: E731
    else:
        raise ValueError(f"unknown preconditioner {precond!r}")
    p, it, hist = pcg(
        lambda u: stencil(fc, u.reshape(shape), perturbed).reshape(-1),
        apply_m, b, rtol, max_iter, exact_dots=perturbed,
    )
    kappa = outflow_kappa(fc, p.reshape(shape), g, p_in, p_out)
    return {"iterations": it, "converged": hist[-1] <= rtol, "history": hist,
            "kappa_eff": kappa, "refs": refs, "stats": st}


# ----------------------------------------------------------------------------
# inputs (reference grid.py:230-284) — bounding-box voxelisation, bit-identical
# membership test ((dx^2 + dy^2) + dz^2 <= r*r)
# ----------------------------------------------------------------------------

RANDOM_BALL_PRESETS = {
    "a": dict(count=40, r_min=0.05, r_max=0.15, seed=11),
    "b": dict(count=80, r_min=0.04, r_max=0.10, seed=23),
    "c": dict(count=16, r_min=0.10, r_max=0.20, seed=37),
}


def ball_list(count, r_min, r_max, seed):
    """Centers then radius per ball from a PCG64 stream (grid.py:266-272)."""
    rng = np.random.default_rng(np.uint64(seed))
    out = []
    for _ in range(count):
        cx, cy, cz = rng.random(3)
        r = r_min + (r_max - r_min) * rng.random()
        out.append((float(cx), float(cy), float(cz), float(r)))
    return out


def random_balls(n, count, r_min, r_max, kappa_inc, seed) -> np.ndarray:
    h = 1.0 / n
    c = (np.arange(n) + 0.5) * h
    inside = np.zeros((n, n, n), dtype=bool)
    for cx, cy, cz, r in ball_list(count, r_min, r_max, seed):
        rr = r * r
        lo = lambda m: max(0, int(math.floor((m - r) / h)) - 1)
        hi = lambda m: min(n, int(math.ceil((m + r) / h)) + 2)
        i0, i1, j0, j1, k0, k1 = lo(cx), hi(cx), lo(cy), hi(cy), lo(cz), hi(cz)
        dx = (c[i0:i1] - cx) ** 2
        dy = (c[j0:j1] - cy) ** 2
        dz = (c[k0:k1] - cz) ** 2
        d = (dx[None, None, :] + dy[None, :, None]) + dz[:, None, None]
        inside[k0:k1, j0:j1, i0:i1] |= d <= rr
    return np.where(inside, float(kappa_inc), 1.0)


def center_ball(n, kappa_inc) -> np.ndarray:
    h = 1.0 / n
    c = (np.arange(n) + 0.5) * h
    d = ((c[None, None, :] - 0.5) ** 2 + (c[None, :, None] - 0.5) ** 2) + (c[:, None, None] - 0.5) ** 2
    return np.where(d <= 0.25 ** 2, float(kappa_inc), 1.0)


def channels(cells_per_period: int, periods: int, psi: float):
    """gen_channels (grid.py:287-319): returns (kx, ky, kz) cubes."""
    cpp = cells_per_period
    n = cpp * periods
    local = np.arange(n) % cpp
    band = (local >= 3 * cpp // 8) & (local < 5 * cpp // 8)
    bi, bj, bk = band[None, None, :], band[None, :, None], band[:, None, None]
    ch = (bj & bk) | (bi & bk) | (bi & bj)
    return (np.where(ch, 2.0 ** psi, 0.01), np.where(ch, 5.0 ** psi, 0.1), np.where(ch, 10.0 ** psi, 1.0))


def fibres(n, count, r_min, r_max, kappa_fib, seed, axis="z") -> np.ndarray:
    """The aligned-fibre generator (paper_2404_02433_b200.grid.gen_fibres; no
    reference counterpart): PCG64 draws (c1, c2, r) per fibre, cell centres
    (i+0.5)*h, membership ((d1*d1) + (d2*d2)) <= r*r."""
    rng = np.random.default_rng(np.uint64(seed))
    fib = []
    for _ in range(count):
        c = rng.random(2)
        fib.append((c[0], c[1], r_min + (r_max - r_min) * rng.random()))
    h = 1.0 / n
    x = (np.arange(n) + 0.5) * h
    ax = "xyz".index(axis)
    # transverse coordinates in increasing axis order, broadcast to (k, j, i)
    grids = {0: x[None, None, :], 1: x[None, :, None], 2: x[:, None, None]}
    u, v = [grids[a] for a in range(3) if a != ax]
    inside = np.zeros((n, n, n), dtype=bool)
    for c1, c2, r in fib:
        du, dv = u - c1, v - c2
        inside |= (du * du + dv * dv) <= r * r
    return np.where(inside, kappa_fib, 1.0)
