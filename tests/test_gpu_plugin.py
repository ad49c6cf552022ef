"""The operator-plugin layer (paper_2404_02433_b200.plugin, reference names)
on the GPU: the properties the reference's own unit tests pin
(pkg/tests/test_tpfa.py, test_transforms.py, test_preconditioner.py,
test_krylov.py), restated against the package, plus bit-exactness against
the reference's outputs in tests/golden/kernels.npz and numpy <-> CUDA-tensor
agreement.  (The reference's test files themselves were run once through the
etchomo alias: profiles/r02/reference_unit_tests_via_alias.log.)

Tolerances follow the reference tests: elementwise kernels bit-exact (numpy
order, no FMA contraction), transforms 1e-12 of max, solves as stated."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2404_02433_b200 as P  # noqa: E402
from paper_2404_02433_b200 import plugin as E  # noqa: E402
from paper_2404_02433_b200.etchomo import alias  # noqa: E402

BZ = P.BoundaryConfig(P.Axis.Z, 1.0, 0.0)


def field_const(nx, ny, nz, kx=1.0, ky=1.0, kz=1.0, lengths=(1.0, 1.0, 1.0)):
    g = P.GridSpec(nx, ny, nz, *lengths)
    n = g.n_cells
    return P.OrthotropicField(g, np.full(n, kx), np.full(n, ky), np.full(n, kz))


def field_rand(rng, nx, ny, nz, contrast=10.0, dtype=np.float64):
    g = P.GridSpec(nx, ny, nz)
    k = np.exp(rng.uniform(-np.log(contrast), np.log(contrast), (3, g.n_cells)))
    return P.OrthotropicField(g, *(k.astype(dtype)))


def golden_field(data, tag):
    nx, ny, nz, lx, ly, lz = data[f"{tag}/grid"]
    g = P.GridSpec(int(nx), int(ny), int(nz), float(lx), float(ly), float(lz))
    return P.OrthotropicField(g, *data[f"{tag}/k"])


# ---------------------------------------------------------------- bitwise --
def test_bitwise_against_reference_outputs(golden_kernels):
    """apply_operator, build_rhs, coefficient_stats and thomas_solve_batch
    reproduce the reference's arrays bit for bit; the transforms and the
    preconditioner to 1e-12 / 1e-11 (their FFT association differs)."""
    data, shapes = golden_kernels
    for tag in shapes:
        f = golden_field(data, tag)
        sys_ = E.build_system(f, BZ)
        u = data[f"{tag}/u"]
        assert np.array_equal(E.apply_operator(sys_, u), data[f"{tag}/Au"]), tag
        assert np.array_equal(E.build_rhs(sys_), data[f"{tag}/b"]), tag
        st = E.coefficient_stats(sys_)
        assert np.array_equal([v for pr in st.groups().values() for v in pr], data[f"{tag}/stats"]), tag
        refs = E.solve_reference_lp(st)
        fac = E.build_tridiag(f.grid, refs)
        assert np.array_equal(E.thomas_solve_batch(fac, u).reshape(-1), data[f"{tag}/thomas"]), tag
        plan = E.FctPlan(f.grid.nx, f.grid.ny, f.grid.nz)
        cube = u.reshape(f.grid.shape)
        for got, key in ((plan.forward(cube)[0], "fwd"), (plan.backward(cube)[0], "bwd")):
            want = data[f"{tag}/{key}"]
            assert np.max(np.abs(got.reshape(-1) - want)) <= 1e-12 * max(np.max(np.abs(want)), 1e-300), (tag, key)
        pre = E.FctPreconditioner(f.grid, refs)(u)
        want = data[f"{tag}/precond"]
        assert np.max(np.abs(pre - want)) <= 1e-11 * np.max(np.abs(want)), tag


def test_tensor_in_tensor_out_matches_numpy():
    rng = np.random.default_rng(21)
    f = field_rand(rng, 12, 10, 9, 40.0)
    sys_np = E.build_system(f, BZ)
    ft = P.OrthotropicField(f.grid, *[torch.from_numpy(np.array(a)).cuda() for a in (f.kx, f.ky, f.kz)])
    sys_t = E.build_system(ft, BZ)
    assert torch.is_tensor(sys_t.tx) and sys_t.tx.is_cuda
    assert np.array_equal(sys_t.tx.cpu().numpy(), sys_np.tx)
    u = rng.standard_normal(f.grid.n_cells)
    out_t = E.apply_operator(sys_t, torch.from_numpy(u).cuda())
    assert torch.is_tensor(out_t) and np.array_equal(out_t.cpu().numpy(), E.apply_operator(sys_np, u))
    refs = E.solve_reference_lp(E.coefficient_stats(sys_t))
    m = E.FctPreconditioner(f.grid, refs)
    b = E.build_rhs(sys_t)
    p_t, rep_t = E.pcg(lambda v: E.apply_operator(sys_t, v), m, b, 1e-10)
    p_n, rep_n = E.pcg(lambda v: E.apply_operator(sys_np, v), m, E.build_rhs(sys_np), 1e-10)
    assert torch.is_tensor(p_t) and isinstance(p_n, np.ndarray)
    assert rep_t.relative_residuals == rep_n.relative_residuals
    assert np.array_equal(p_t.cpu().numpy(), p_n)


def test_inputs_not_mutated():
    rng = np.random.default_rng(3)
    f = field_rand(rng, 6, 5, 4)
    sys_ = E.build_system(f, BZ)
    u = rng.standard_normal(f.grid.n_cells)
    keep = u.copy()
    E.apply_operator(sys_, u)
    fac = E.build_tridiag(f.grid, E.solve_reference_lp(E.coefficient_stats(sys_)))
    E.thomas_solve_batch(fac, u)
    E.FctPreconditioner(f.grid, fac.refs)(u)
    assert np.array_equal(u, keep)
    ut = torch.from_numpy(keep.copy()).cuda()
    E.thomas_solve_batch(fac, ut)
    assert np.array_equal(ut.cpu().numpy(), keep)
    E.thomas_solve_batch(fac, ut, overwrite=True)  # asked for: solved in place
    assert not np.array_equal(ut.cpu().numpy(), keep)


# ------------------------------------------------------------------- tpfa --
def test_scale_field():
    sx, sy, sz = E.scale_field(field_const(3, 3, 3, lengths=(3.0, 3.0, 3.0)))
    assert np.all(sx == 1.0) and np.all(sy == 1.0) and np.all(sz == 1.0)
    assert np.all(E.scale_field(field_const(2, 2, 2, kz=4.0))[2] == 16.0)
    f = field_rand(np.random.default_rng(1), 3, 4, 5)
    g = P.OrthotropicField(f.grid, 2.5 * f.kx, 2.5 * f.ky, 2.5 * f.kz)
    for a, b in zip(E.scale_field(g), E.scale_field(f)):
        np.testing.assert_allclose(a, 2.5 * b, rtol=1e-15)


def test_build_system_values_and_contract():
    n = 4
    s = E.build_system(field_const(n, n, n), BZ)
    for arr, v in ((s.tx, n * n), (s.ty, n * n), (s.tz, n * n), (s.t_in, 2 * n * n), (s.t_out, 2 * n * n)):
        assert np.all(arr == v)
    g = P.GridSpec(2, 1, 1, 2.0, 1.0, 1.0)
    s = E.build_system(P.OrthotropicField(g, [0.01, 1.0], [1.0, 1.0], [1.0, 1.0]), BZ)
    assert s.tx[0] == pytest.approx(2.0 / 101.0, rel=1e-14)
    with pytest.raises(P.ConfigError):
        E.build_system(field_const(2, 2, 2), P.BoundaryConfig(P.Axis.X, 1.0, 0.0))
    with pytest.raises(P.ConfigError):
        E.DiscreteSystem(g, np.array([-1.0]), np.zeros(0), np.zeros(0), np.ones(2), np.ones(2), BZ)
    with pytest.raises(P.ConfigError):
        E.DiscreteSystem(g, np.ones(2), np.zeros(0), np.zeros(0), np.ones(2), np.ones(2), BZ)


def test_harmonic_faces_between_neighbours():
    f = field_rand(np.random.default_rng(2), 5, 4, 3, contrast=100.0)
    s = E.build_system(f, BZ)
    sx = E.scale_field(f)[0]
    lo, hi = np.minimum(sx[:, :, :-1], sx[:, :, 1:]).ravel(), np.maximum(sx[:, :, :-1], sx[:, :, 1:]).ravel()
    assert np.all(s.tx >= lo - 1e-14) and np.all(s.tx <= hi + 1e-14) and np.all(s.tx <= 2 * lo + 1e-14)


def two_cell():
    return E.build_system(field_const(1, 1, 2, lengths=(1.0, 1.0, 2.0)), BZ)


def test_operator_small_cases():
    s = two_cell()
    np.testing.assert_array_equal(E.apply_operator(s, np.array([1.0, 0.0])), [3.0, -1.0])
    np.testing.assert_array_equal(E.apply_operator(s, np.array([0.0, 1.0])), [-1.0, 3.0])
    np.testing.assert_array_equal(E.assemble_dense(s), [[3.0, -1.0], [-1.0, 3.0]])
    with pytest.raises(ValueError):
        E.apply_operator(s, np.ones(3))
    f = field_rand(np.random.default_rng(3), 4, 3, 5)
    s = E.build_system(f, BZ)
    out = E.apply_operator(s, np.full(f.grid.n_cells, 2.5)).reshape(f.grid.shape)
    sz = E.scale_field(f)[2]
    np.testing.assert_allclose(out[0], 2 * sz[0] * 2.5, rtol=1e-13)
    np.testing.assert_allclose(out[-1], 2 * sz[-1] * 2.5, rtol=1e-13)
    np.testing.assert_allclose(out[1:-1], 0.0, atol=1e-11)


@pytest.mark.parametrize("dims", [(5, 4, 3), (8, 8, 8), (17, 9, 5), (1, 6, 4), (3, 1, 7), (1, 1, 1)])
def test_operator_symmetric_positive(dims):
    rng = np.random.default_rng(sum(dims) * 7)
    s = E.build_system(field_rand(rng, *dims, contrast=50.0), BZ)
    n = int(np.prod(dims))
    u, w = rng.standard_normal(n), rng.standard_normal(n)
    au, aw = E.apply_operator(s, u), E.apply_operator(s, w)
    assert abs(np.dot(au, w) - np.dot(u, aw)) <= 1e-13 * np.linalg.norm(au) * np.linalg.norm(w)
    mat = E.assemble_dense(s)
    assert np.array_equal(mat, mat.T)
    assert np.linalg.eigvalsh(mat)[0] > 0.0
    np.testing.assert_allclose(E.operator_diagonal(s), np.diag(mat), rtol=0, atol=0)
    np.testing.assert_allclose(E.assemble_sparse(s).toarray(), mat)
    for j in rng.choice(n, size=min(n, 6), replace=False):
        e = np.zeros(n)
        e[j] = 1.0
        np.testing.assert_allclose(mat[:, j], E.apply_operator(s, e), atol=1e-14)


def test_dense_guard():
    with pytest.raises(ValueError):
        E.assemble_dense(E.build_system(field_const(17, 17, 17), BZ))


def test_rhs_and_linear_profile():
    n = 4
    s = E.build_system(field_const(n, n, n), BZ)
    b = E.build_rhs(s).reshape(n, n, n)
    assert np.all(b[0] == 32.0) and np.all(b[1:] == 0.0)
    n = 6
    s = E.build_system(field_const(n, n, n), BZ)
    b = E.build_rhs(s)
    prof = 1.0 - (np.arange(n) + 0.5) / n
    p = np.broadcast_to(prof[:, None, None], (n, n, n)).reshape(-1)
    assert np.linalg.norm(E.apply_operator(s, p) - b) <= 1e-12 * np.linalg.norm(b)
    # face-sampled Dirichlet planes (tpfa.py:150-167)
    pin = np.linspace(0.5, 1.5, n * n).reshape(n, n)
    b2 = E.build_rhs(s, dirichlet_in=pin, dirichlet_out=0.25).reshape(n, n, n)
    np.testing.assert_array_equal(b2[0], s.layer_in() * pin)
    np.testing.assert_array_equal(b2[-1], s.layer_out() * 0.25)


def test_sources_and_l2():
    s = E.build_system(field_const(3, 3, 3), BZ)
    b = E.build_rhs(s)
    assert np.array_equal(E.add_source(s, b, lambda x, y, z: np.zeros_like(x)), b)
    np.testing.assert_allclose(E.add_source(s, b, lambda x, y, z: np.ones_like(x)) - b, 1.0)
    g = P.GridSpec(4, 4, 4)
    X, Y, Z = g.cell_centers()
    assert E.l2_error_midpoint(g, (X + 2 * Y - Z).reshape(-1), lambda x, y, z: x + 2 * y - z) == 0.0
    g = P.GridSpec(5, 5, 5)
    assert E.l2_error_midpoint(g, np.full(g.n_cells, 0.25), lambda x, y, z: np.zeros_like(x)) == pytest.approx(0.25)


def test_fluxes_and_effective_conductivity():
    s = E.build_system(field_const(3, 3, 3), BZ)
    np.testing.assert_allclose(E.reconstruct_boundary_flux(s, np.zeros(27), side="out"), 0.0)
    with pytest.raises(ValueError):
        E.reconstruct_boundary_flux(s, np.zeros(27), side="up")
    n = 5
    s = E.build_system(field_const(n, n, n), BZ)
    p = E.dense_solve(E.assemble_dense(s), E.build_rhs(s))
    np.testing.assert_allclose(E.reconstruct_boundary_flux(s, p, side="out"), 1.0, rtol=1e-12)
    np.testing.assert_allclose(E.reconstruct_boundary_flux(s, p, side="in"), 1.0, rtol=1e-12)
    s = E.build_system(field_const(4, 4, 4, kx=2.0, ky=5.0, kz=3.25), BZ)
    p = E.dense_solve(E.assemble_dense(s), E.build_rhs(s))
    assert E.effective_conductivity(s, E.reconstruct_boundary_flux(s, p)) == pytest.approx(3.25, abs=1e-12)
    layers = np.array([1.0, 2.0, 0.5, 4.0, 1.5, 3.0])
    g = P.GridSpec(3, 3, layers.size)
    ones = np.ones(g.n_cells)
    s = E.build_system(P.OrthotropicField(g, ones, ones, np.repeat(layers, 9)), BZ)
    p = E.dense_solve(E.assemble_dense(s), E.build_rhs(s))
    keff = E.effective_conductivity(s, E.reconstruct_boundary_flux(s, p))
    assert keff == pytest.approx(layers.size / np.sum(1.0 / layers), rel=1e-10)
    rng = np.random.default_rng(10)
    for _ in range(3):
        s = E.build_system(field_rand(rng, 6, 5, 7, contrast=30.0), BZ)
        p = E.dense_solve(E.assemble_dense(s), E.build_rhs(s))
        fin = E.reconstruct_boundary_flux(s, p, side="in").sum()
        fout = E.reconstruct_boundary_flux(s, p, side="out").sum()
        assert abs(fin - fout) <= 1e-10 * abs(fout)


def test_smooth_problem_pcg_matches_dense():
    field, exact, source = P.gen_smooth_problem(6)
    s = E.build_system(field, BZ)
    X, Y, _ = field.grid.cell_centers()
    b = E.build_rhs(s, dirichlet_in=exact(X[0], Y[0], 0.0), dirichlet_out=exact(X[0], Y[0], 1.0))
    b = E.add_source(s, b, source)
    direct = E.dense_solve(E.assemble_dense(s), b)
    m = E.FctPreconditioner(field.grid, E.solve_reference_lp(E.coefficient_stats(s)))
    it, rep = E.pcg(lambda v: E.apply_operator(s, v), m, b, 1e-12)
    assert rep.converged
    assert np.linalg.norm(it - direct) <= 1e-9 * np.linalg.norm(direct)


def test_axis_permute_matches_numpy_swapaxes():
    rng = np.random.default_rng(4)
    f = field_rand(rng, 5, 3, 4)
    fx = E.axis_permute(f, P.Axis.X)
    assert fx.grid == P.GridSpec(4, 3, 5, 1.0, 1.0, 1.0)
    assert np.array_equal(fx.cube("kz"), np.swapaxes(f.cube("kx"), 0, 2))
    assert np.array_equal(fx.cube("kx"), np.swapaxes(f.cube("kz"), 0, 2))
    fy = E.axis_permute(f, P.Axis.Y)
    assert fy.grid == P.GridSpec(5, 4, 3, 1.0, 1.0, 1.0)
    assert np.array_equal(fy.cube("kz"), np.swapaxes(f.cube("ky"), 0, 1))
    assert np.array_equal(fy.cube("ky"), np.swapaxes(f.cube("kz"), 0, 1))
    assert E.axis_permute(f, P.Axis.Z) is f


# ------------------------------------------------------------- transforms --
def _ref2d(v):
    ny, nx = v.shape
    out = np.stack([E.dct1d_ref_forward(v[j]) for j in range(ny)])
    return np.stack([E.dct1d_ref_forward(out[:, i]) for i in range(nx)], axis=1)


def test_dct1d_direct_sums():
    np.testing.assert_allclose(E.dct1d_ref_forward([1.0, 1.0]), [2.0, 0.0], atol=1e-15)
    np.testing.assert_allclose(E.dct1d_ref_forward([1.0, 0.0]), [1.0, math.sqrt(2.0) / 2.0], rtol=1e-15)
    for n in (1, 2, 3, 5, 8, 17):
        u = np.random.default_rng(n).standard_normal(n)
        np.testing.assert_allclose(E.dct1d_ref_backward(E.dct1d_ref_forward(u)), u, atol=1e-13)


def test_pre_permute():
    assert np.array_equal(E.fct_pre_permute(np.array([[4.2]])), [[4.2]])
    assert np.array_equal(E.fct_pre_permute(np.array([[1.0, 2.0, 3.0, 4.0]])), [[1.0, 3.0, 4.0, 2.0]])
    v = np.random.default_rng(0).standard_normal((5, 7))
    assert sorted(v.ravel()) == sorted(E.fct_pre_permute(v).ravel())
    out = np.empty_like(v)
    assert E.fct_pre_permute(v, out) is out and np.array_equal(out, E.fct_pre_permute(v))
    vt = torch.from_numpy(v).cuda()
    assert np.array_equal(E.fct_pre_permute(vt).cpu().numpy(), E.fct_pre_permute(v))


def test_forward_batch_properties():
    plan = E.FctPlan(6, 4, 2)
    buf = E.SlabBuffer(plan, np.full((2, 4, 6), 3.0))
    E.fct_forward_batch(buf)
    assert buf.data[0, 0, 0] == pytest.approx(72.0, rel=1e-13)
    mask = np.ones((2, 4, 6), dtype=bool)
    mask[:, 0, 0] = False
    assert np.max(np.abs(buf.data[mask])) <= 1e-12 * 72.0
    rng = np.random.default_rng(3)
    sl = rng.standard_normal((3, 5, 4))
    whole = E.SlabBuffer(E.FctPlan(4, 5, 3), sl.copy())
    E.fct_forward_batch(whole)
    one = E.FctPlan(4, 5, 1)
    for k in range(3):
        single = E.SlabBuffer(one, sl[k:k + 1].copy())
        E.fct_forward_batch(single)
        assert np.array_equal(whole.data[k], single.data[0])
    a, b = E.SlabBuffer(E.FctPlan(4, 5, 3), sl.copy()), E.SlabBuffer(E.FctPlan(4, 5, 3), sl[::-1].copy())
    E.fct_forward_batch(a)
    E.fct_forward_batch(b)
    assert np.array_equal(a.data[::-1], b.data)


@pytest.mark.parametrize("nx", [1, 2, 5, 8])
@pytest.mark.parametrize("ny", [1, 3, 4, 9])
def test_transform_pair_against_direct_sums(nx, ny):
    rng = np.random.default_rng(nx * 100 + ny)
    v = rng.standard_normal((2, ny, nx))
    buf = E.SlabBuffer(E.FctPlan(nx, ny, 2), v.copy())
    E.fct_forward_batch(buf)
    for k in range(2):
        want = _ref2d(v[k])
        assert np.max(np.abs(buf.data[k] - want)) <= 1e-12 * max(np.max(np.abs(want)), 1e-30)
    E.fct_backward_batch(buf)
    assert np.max(np.abs(buf.data - v)) <= 1e-12 * np.max(np.abs(v))


def test_backward_direct_sum_and_impulse():
    buf = E.SlabBuffer(E.FctPlan(2, 2, 1), np.array([[[1.0, 0.0], [0.0, 0.0]]]))
    E.fct_backward_batch(buf)
    np.testing.assert_allclose(buf.data, 0.25, rtol=1e-14)
    coeff = np.random.default_rng(7).standard_normal((1, 5, 4))
    buf = E.SlabBuffer(E.FctPlan(4, 5, 1), coeff.copy())
    E.fct_backward_batch(buf)
    stage = np.stack([E.dct1d_ref_backward(row) for row in coeff[0]])
    want = np.stack([E.dct1d_ref_backward(stage[:, i]) for i in range(4)], axis=1)
    np.testing.assert_allclose(buf.data[0], want, atol=1e-13)


@pytest.mark.parametrize("shape", [(6, 5), (7, 4), (1, 3), (8, 8)])
def test_parseval(shape):
    ny, nx = shape
    rng = np.random.default_rng(ny * 10 + nx)
    r, z = rng.standard_normal((1, ny, nx)), rng.standard_normal((1, ny, nx))
    plan = E.FctPlan(nx, ny, 1)
    br, bz = E.SlabBuffer(plan, r.copy()), E.SlabBuffer(plan, z.copy())
    E.fct_forward_batch(br)
    E.fct_forward_batch(bz)
    ax, ay = np.where(np.arange(nx) == 0, 0.5, 1.0), np.where(np.arange(ny) == 0, 0.5, 1.0)
    spec = 4.0 / (nx * ny) * np.sum(ay[:, None] * ax[None, :] * br.data[0] * bz.data[0])
    assert spec == pytest.approx(np.sum(r * z), rel=1e-11)


def test_float32_plan_round_trip():
    v = np.random.default_rng(9).standard_normal((3, 16, 16)).astype(np.float32)
    plan = E.FctPlan(16, 16, 3, dtype=np.float32)
    fwd, _ = plan.forward(v)
    assert fwd.dtype == np.float32
    want = np.stack([_ref2d(v[k].astype(np.float64)) for k in range(3)])
    assert np.max(np.abs(fwd - want)) <= 1e-5 * np.max(np.abs(want))
    back, _ = plan.backward(fwd)
    assert np.max(np.abs(back - v)) <= 1e-5 * np.max(np.abs(v))


# --------------------------------------------------------- preconditioner --
def test_coefficient_stats():
    s = E.coefficient_stats(E.build_system(field_const(4, 4, 4), BZ))
    for lo, hi in s.groups().values():
        assert lo == hi == 16.0
    rng = np.random.default_rng(11)
    f = field_rand(rng, 4, 4, 4, contrast=100.0)
    s = E.coefficient_stats(E.build_system(f, BZ))
    sx, sy, sz = E.scale_field(f)

    def h(a, b):
        return 2.0 / (1.0 / a + 1.0 / b)

    fx, fy, fz = h(sx[:, :, :-1], sx[:, :, 1:]), h(sy[:, :-1], sy[:, 1:]), h(sz[:-1], sz[1:])
    for (lo, hi), arr in zip((s.groups()[k] for k in "xyz"), (fx, fy, fz)):
        assert lo == pytest.approx(arr.min(), rel=1e-14) and hi == pytest.approx(arr.max(), rel=1e-14)
    assert s.kin_min == pytest.approx(sz[0].min(), rel=1e-14) and s.kout_max == pytest.approx(sz[-1].max(),
                                                                                                 rel=1e-14)
    mir = P.OrthotropicField(f.grid, *(f.cube(c)[:, :, ::-1].copy() for c in ("kx", "ky", "kz")))
    assert E.coefficient_stats(E.build_system(mir, BZ)) == s
    # degenerate axes give the neutral group (preconditioner.py:94-98)
    s1 = E.coefficient_stats(E.build_system(field_const(1, 3, 3), BZ))
    assert s1.kx_min == s1.kx_max == 1.0


def test_thomas_matches_dense_and_pivots():
    g = P.GridSpec(3, 2, 5)
    refs = P.ReferenceParams(1.3, 0.7, 2.0, 0.9, 1.1)
    fac = E.build_tridiag(g, refs)
    rhs = np.random.default_rng(5).standard_normal(g.shape)
    x = E.thomas_solve_batch(fac, rhs)
    for j in range(g.ny):
        for i in range(g.nx):
            np.testing.assert_allclose(x[:, j, i], np.linalg.solve(fac.dense_block(i, j), rhs[:, j, i]),
                                       rtol=1e-12, atol=1e-14)
    bad = E.build_tridiag(g, refs)
    bad.z_diag = bad.z_diag.copy()
    bad.z_diag[2] = -50.0
    bad._dev = None
    with pytest.raises(FloatingPointError, match="layer 2"):
        E.thomas_solve_batch(bad, rhs)
    bad.z_diag[0] = -50.0
    bad._dev = None
    with pytest.raises(FloatingPointError):
        E.thomas_solve_batch(bad, rhs)


def test_fct_preconditioner_exact_for_reference_operator():
    rng = np.random.default_rng(14)
    g = P.GridSpec(6, 5, 7, 1.0, 0.8, 1.3)
    refs = P.ReferenceParams(1.5, 0.6, 2.5, 1.1, 0.8)
    rsys = E.reference_system(g, refs)
    m = E.FctPreconditioner(g, refs)
    r = rng.standard_normal(g.n_cells)
    back = E.apply_operator(rsys, m(r))
    assert np.max(np.abs(back - r)) <= 1e-11 * np.max(np.abs(r))
    fac = E.build_tridiag(g, refs)
    np.testing.assert_allclose(E.fct_precond_apply(fac, r), m(r), rtol=0, atol=0)


def test_reference_bounds_condition_number():
    rng = np.random.default_rng(15)
    s = E.build_system(field_rand(rng, 3, 3, 3, contrast=20.0), BZ)
    st = E.coefficient_stats(s)
    refs = E.solve_reference_lp(st)
    a = E.assemble_dense(s)
    aref = E.assemble_dense(E.reference_system(s.grid, refs))
    lo, hi, cond = E.condition_estimate(a, aref)
    assert lo >= refs.lambda_lo * (1 - 1e-9) and hi <= refs.lambda_hi * (1 + 1e-9)
    assert cond <= refs.objective * (1 + 1e-9)
    assert E.condition_estimate(a, a)[2] == pytest.approx(1.0, rel=1e-10)
    with pytest.raises(ValueError):
        E.condition_estimate(np.eye(3), np.zeros((3, 3)))


def test_jacobi_identity_ssor():
    rng = np.random.default_rng(16)
    s = E.build_system(field_rand(rng, 4, 3, 5, contrast=10.0), BZ)
    r = rng.standard_normal(s.grid.n_cells)
    np.testing.assert_array_equal(E.jacobi_apply(s, r), r * (1.0 / E.operator_diagonal(s)))
    c = E.identity_apply(r)
    assert c is not r and np.array_equal(c, r)
    mat = E.assemble_dense(s)
    d = np.diag(np.diag(mat))
    for omega in (0.7, 1.0, 1.4):
        lo, up = np.tril(mat, -1) + d / omega, np.triu(mat, 1) + d / omega
        m = (omega / (2.0 - omega)) * lo @ np.linalg.inv(d) @ up
        np.testing.assert_allclose(E.ssor_apply(s, omega, r), np.linalg.solve(m, r), rtol=1e-10)
    with pytest.raises(P.ConfigError):
        E.SsorPreconditioner(s, 2.0)
    b = E.build_rhs(s)
    _, rep = E.pcg(lambda v: E.apply_operator(s, v), E.SsorPreconditioner(s, 1.0), b, 1e-10)
    assert rep.converged


# ----------------------------------------------------------------- krylov --
def test_pcg_one_iteration_cases():
    s = E.build_system(field_const(1, 1, 1), BZ)
    b = np.array([3.0])
    p, rep = E.pcg(lambda u: E.apply_operator(s, u), E.identity_apply, b, 1e-12)
    assert rep.converged and rep.iterations == 1
    np.testing.assert_allclose(E.apply_operator(s, p), b, rtol=1e-14)
    s = E.build_system(field_const(6, 5, 4, kx=2.0, ky=3.0, kz=0.7), BZ)
    m = E.FctPreconditioner(s.grid, E.solve_reference_lp(E.coefficient_stats(s)))
    _, rep = E.pcg(lambda u: E.apply_operator(s, u), m, E.build_rhs(s), 1e-12)
    assert rep.converged and rep.iterations == 1 and rep.relative_residuals[-1] <= 1e-14


def test_pcg_contract():
    p, rep = E.pcg(lambda u: u, E.identity_apply, np.zeros(5), 1e-10)
    assert rep.converged and rep.iterations == 0 and np.all(p == 0.0) and rep.relative_residuals == [0.0]
    with pytest.raises(ValueError):
        E.pcg(lambda u: u, E.identity_apply, np.ones(2), -1.0)
    with pytest.raises(ValueError):
        E.pcg(lambda u: u, E.identity_apply, np.ones(2), 1e-9, max_iter=0)
    rng = np.random.default_rng(1)
    s = E.build_system(field_rand(rng, 6, 6, 6, contrast=100.0), BZ)
    _, rep = E.pcg(lambda u: E.apply_operator(s, u), E.identity_apply, E.build_rhs(s), 1e-12, max_iter=3)
    assert not rep.converged and rep.iterations == 3 and len(rep.relative_residuals) == 4
    s = E.build_system(field_rand(np.random.default_rng(0), 5, 5, 5, contrast=20.0), BZ)
    m = E.FctPreconditioner(s.grid, E.solve_reference_lp(E.coefficient_stats(s)))
    _, rep = E.pcg(lambda u: E.apply_operator(s, u), m, E.build_rhs(s), 1e-9)
    assert rep.converged and rep.iterations == len(rep.relative_residuals) - 1
    assert rep.relative_residuals[0] == pytest.approx(1.0) and rep.relative_residuals[-1] <= 1e-9
    hist = [E.pcg(lambda u: E.apply_operator(s, u), E.FctPreconditioner(s.grid, m.refs), E.build_rhs(s),
                  1e-10)[1].relative_residuals for _ in range(2)]
    assert hist[0] == hist[1]


def test_pcg_breakdowns():
    """PcgBreakdownError on an indefinite operator or preconditioner
    (krylov.py:66-88; reference test_krylov.py:76-86)."""
    mat = np.diag([1.0, -1.0])
    with pytest.raises(P.PcgBreakdownError) as err:
        E.pcg(lambda u: mat @ u, E.identity_apply, np.array([1.0, 1.0]), 1e-12)
    assert err.value.iteration >= 0
    minv = np.diag([1.0, -4.0])
    with pytest.raises(P.PcgBreakdownError) as err:
        E.pcg(lambda u: u, lambda r: minv @ r, np.array([0.1, 1.0]), 1e-12)
    assert err.value.iteration == 0


def test_pcg_float32_and_dense():
    f = P.gen_center_ball(16, 10.0, as_numpy=True).astype(np.float32)
    s = E.build_system(f, BZ)
    m = E.FctPreconditioner(s.grid, E.solve_reference_lp(E.coefficient_stats(s)), dtype=np.float32)
    b = E.build_rhs(s)
    assert b.dtype == np.float32
    p, rep = E.pcg(lambda u: E.apply_operator(s, u), m, b, 1e-6)
    assert p.dtype == np.float32 and rep.converged and np.all(np.isfinite(p))
    np.testing.assert_allclose(E.dense_solve(np.array([[3.0, -1.0], [-1.0, 3.0]]), np.array([2.0, 2.0])),
                               [1.0, 1.0], rtol=1e-14)
    with pytest.raises(ValueError):
        E.dense_solve(np.diag([1.0, -2.0]), np.ones(2))
    s = E.build_system(field_rand(np.random.default_rng(3), 5, 5, 5, contrast=100.0), BZ)
    b = E.build_rhs(s)
    direct = E.dense_solve(E.assemble_dense(s), b)
    m = E.FctPreconditioner(s.grid, E.solve_reference_lp(E.coefficient_stats(s)))
    it, rep = E.pcg(lambda u: E.apply_operator(s, u), m, b, 1e-10)
    assert rep.converged and np.linalg.norm(it - direct) <= 1e-8 * np.linalg.norm(direct)


def test_homogenize_composed_matches_fused():
    """homogenize(precond='ssor') runs the plugin composition (pipeline.py:153-175);
    the same composition with fct agrees with the fused device solve."""
    from paper_2404_02433_b200.solver import _homogenize_composed

    f = P.gen_random_balls(20, 40, 0.05, 0.15, 100.0, 11)
    b = P.BoundaryConfig(P.Axis.Y, 1.0, 0.0)
    fused = P.homogenize(f, b, 1e-9)
    comp = _homogenize_composed(f, b, 1e-9, "fct", "opt", "f64", 1.0, 1024, None)
    assert comp.iterations == fused.iterations
    assert abs(comp.kappa_eff - fused.kappa_eff) <= 1e-10 * fused.kappa_eff
    ss = P.homogenize(f, b, 1e-9, precond="ssor:1.3")
    assert ss.converged and ss.preconditioner == "ssor:1.3"
    assert abs(ss.kappa_eff - fused.kappa_eff) <= 1e-6 * fused.kappa_eff


def test_etchomo_alias_namespace():
    import sys

    alias("etchomo_under_test")
    mod = sys.modules["etchomo_under_test"]
    for name in ("homogenize", "pcg", "build_system", "apply_operator", "FctPreconditioner", "thomas_solve_batch",
                 "FctPlan", "SlabBuffer", "coefficient_stats", "build_rhs", "reconstruct_boundary_flux",
                 "effective_conductivity", "scale_field", "axis_permute", "DiscreteSystem", "PcgBreakdownError"):
        assert hasattr(mod, name), name
    assert sys.modules["etchomo_under_test.tpfa"].apply_operator is E.apply_operator
