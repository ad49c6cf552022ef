"""Multi-process (world_size 2 and 4, gloo, CPU) tests of the z-slab
decomposition's host logic: torch.distributed collectives as used by
paper_2404_02433_b200.dist, and a full distributed solve whose per-rank
stages are the CPU restatement in tests/cpu_slab_ops.py.  The GPU twin
(production kernels, virtual ranks) is tests/test_gpu_dist.py."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, size, port):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=size)


def _primitives(rank, size, port, q):
    try:
        _init(rank, size, port)
        from paper_2404_02433_b200.dist import TorchComm

        comm = TorchComm()
        t = torch.tensor([rank + 1.0, -rank, 2.0 * rank])
        comm.allreduce(t)
        ok = torch.allclose(t, torch.tensor([size * (size + 1) / 2, -size * (size - 1) / 2, size * (size - 1.0)]))
        m = torch.tensor([float(rank)])
        comm.allreduce(m, "max")
        ok &= m.item() == size - 1
        # all-to-all: block r of rank s lands at block s of rank r (pencil contract)
        inp = torch.arange(4 * size, dtype=torch.float64) + 100 * rank
        out = torch.empty_like(inp)
        comm.alltoall(out, inp)
        want = torch.cat([torch.arange(4 * rank, 4 * rank + 4, dtype=torch.float64) + 100 * s for s in range(size)])
        ok &= torch.equal(out, want)
        # neighbour planes
        lo, hi = torch.full((3,), 10.0 * rank), torch.full((3,), 10.0 * rank + 1)
        rl, rh = torch.full((3,), -1.0), torch.full((3,), -1.0)
        comm.neighbours(lo, hi, rl, rh)
        if rank > 0:
            ok &= bool(torch.all(rl == 10.0 * (rank - 1) + 1))
        if rank < size - 1:
            ok &= bool(torch.all(rh == 10.0 * (rank + 1)))
        q.put((rank, bool(ok), None))
    except Exception as exc:  # pragma: no cover
        q.put((rank, False, repr(exc)))
    finally:
        if td.is_initialized():
            td.destroy_process_group()


def _solve(rank, size, port, q, n, C, axis, fused=False, zsolve="pencil"):
    try:
        _init(rank, size, port)
        from cpu_slab_ops import CpuSlabOps
        from oracle import etc_oracle as O
        from paper_2404_02433_b200.dist import TorchComm, slab_bounds, slab_solve

        comm = TorchComm()
        k = O.random_balls(n, 40, 0.05, 0.15, C, 11)
        kx, ky, kz, g = O.permute(k, k, k, (n, n, n, 1.0, 1.0, 1.0), axis)
        k0, nzl = slab_bounds(g[2], size, rank)
        sl = lambda a: torch.from_numpy(np.ascontiguousarray(a[k0:k0 + nzl]).reshape(-1))
        ops = CpuSlabOps(g[0], g[1], g[2], k0, nzl, size, rank, g[3], g[4], g[5], fused=fused)
        t = sl(kx)
        rep = slab_solve(ops, comm, t, t, t, g, 1.0, 0.0, 1e-8, zsolve=zsolve)
        q.put((rank, (rep.iterations, rep.kappa_eff, rep.relative_residuals), None))
    except Exception as exc:  # pragma: no cover
        import traceback

        q.put((rank, None, traceback.format_exc()))
    finally:
        if td.is_initialized():
            td.destroy_process_group()


def _spawn(fn, size, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, size, port, q) + args) for r in range(size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(res, key=lambda x: x[0])


@pytest.mark.parametrize("size", [2, 4])
def test_comm_primitives(size):
    for rank, ok, err in _spawn(_primitives, size):
        assert ok, (rank, err)


@pytest.mark.parametrize("size,n,C,axis,fused,zsolve", [(2, 16, 100.0, "z", False, "pencil"),
                                                        (4, 16, 10.0, "x", False, "pencil"),
                                                        (2, 24, 100.0, "y", False, "pencil"),
                                                        (2, 16, 100.0, "z", True, "pencil"),
                                                        (4, 16, 10.0, "y", True, "pencil"),
                                                        (2, 16, 100.0, "z", True, "spike"),
                                                        (4, 16, 100.0, "x", False, "spike"),
                                                        (4, 24, 10.0, "y", True, "spike")])
def test_slab_solve_matches_single_process(size, n, C, axis, fused, zsolve):
    sys.path.insert(0, str(ROOT))
    from oracle import etc_oracle as O

    k = O.random_balls(n, 40, 0.05, 0.15, C, 11)
    ref = O.homogenize(k, k, k, (n, n, n, 1.0, 1.0, 1.0), axis, 1.0, 0.0, 1e-8)
    res = _spawn(_solve, size, n, C, axis, fused, zsolve)
    for rank, out, err in res:
        assert err is None, err
        it, kappa, hist = out
        assert it == ref["iterations"], (rank, it, ref["iterations"])
        assert abs(kappa - ref["kappa_eff"]) <= 1e-10 * abs(ref["kappa_eff"])
        h, s = np.array(hist), np.array(ref["history"])
        big = s > 1e-2
        assert np.all(np.abs(h[big] - s[big]) <= 1e-10 * s[big])
    assert all(out == res[0][1] for _, out, _ in res)  # every rank reports the same solve


def _transpose(rank, size, port, q, dims):
    try:
        _init(rank, size, port)
        from paper_2404_02433_b200.dist import TorchComm, canonical_slabs, slab_bounds

        comm = TorchComm()
        nx, ny, nz = dims
        rng = np.random.default_rng(7)
        cubes = [rng.standard_normal((nz, ny, nx)) for _ in range(3)]
        k0, nzl = slab_bounds(nz, size, rank)
        local = tuple(torch.from_numpy(np.ascontiguousarray(c[k0:k0 + nzl])) for c in cubes)
        grid = (nx, ny, nz, 1.0, 2.0, 3.0)
        ok, msg = True, []
        for axis in "xyz":
            (kx, ky, kz), cg = canonical_slabs(local, grid, axis, comm)
            # the reference permutation (pipeline.py:87-111) of the whole cube, this rank's planes
            if axis == "x":
                want = [np.swapaxes(c, 0, 2) for c in (cubes[2], cubes[1], cubes[0])]
                wg = (nz, ny, nx, 3.0, 2.0, 1.0)
            elif axis == "y":
                want = [np.swapaxes(c, 0, 1) for c in (cubes[0], cubes[2], cubes[1])]
                wg = (nx, nz, ny, 1.0, 3.0, 2.0)
            else:
                want, wg = cubes, grid
            c0, cl = slab_bounds(wg[2], size, rank)
            for got, w in zip((kx, ky, kz), want):
                ok &= np.array_equal(got.numpy(), np.ascontiguousarray(w[c0:c0 + cl]).reshape(-1))
            ok &= cg == wg
            iso = canonical_slabs((local[0],) * 3, grid, axis, comm)[0]
            ok &= iso[0] is iso[1] and iso[1] is iso[2]
            msg.append((axis, ok))
        q.put((rank, bool(ok), None if ok else repr(msg)))
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, False, traceback.format_exc()))
    finally:
        if td.is_initialized():
            td.destroy_process_group()


@pytest.mark.parametrize("size,dims", [(2, (4, 6, 8)), (4, (8, 4, 12)), (2, (6, 2, 4))])
def test_distributed_axis_permute(size, dims):
    """canonical_slabs: the x / y axis permutation of a z-slab-distributed
    field as one all-to-all (no rank holds the whole field) equals the
    reference's swapaxes of the whole cube, rank by rank (anisotropic and
    isotropic fields)."""
    for rank, ok, err in _spawn(_transpose, size, dims):
        assert ok, (rank, err)
