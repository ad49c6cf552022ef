"""The peer-memory exchange across processes (CUDA IPC): two ranks as two
processes sharing one GPU, host plumbing over gloo (scalar all-reduces,
handle exchange), every data exchange through the fused kernels' peer stores
into IPC-opened buffers.  The ranks' kernels never wait on one another
inside a kernel (the barriers are host-side), so one device hosts both."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, size, port, n, q, zsolve="pencil", p2p=True):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as td

        torch.cuda.set_device(0)
        td.init_process_group("gloo", rank=rank, world_size=size)
        import paper_2404_02433_b200 as P
        from paper_2404_02433_b200 import dist

        f = P.gen_random_balls(n, 40, 0.05, 0.15, 100.0, 11)
        k0, nzl = dist.slab_bounds(n, size, rank)
        k = f.kx.reshape(n, n, n)[k0:k0 + nzl].contiguous().reshape(-1)
        ops = dist.CudaSlabOps(n, n, n, k0, nzl, size, rank, 1.0, 1.0, 1.0)
        comm = dist.TorchComm()
        rep = dist.slab_solve(ops, comm, k, k, k, (n, n, n, 1.0, 1.0, 1.0), 1.0, 0.0, 1e-8,
                              p2p=p2p, zsolve=zsolve)
        q.put((rank, (rep.iterations, rep.kappa_eff, rep.relative_residuals,
                      ops.p2p_ok() or zsolve == "spike"), None))
        td.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("zsolve,p2p", [("pencil", True), ("spike", False), ("spike", True)])
def test_two_processes_peer_exchange_over_ipc(zsolve, p2p):
    """pencil: the peer-memory exchange over IPC; spike: the substructured
    z-solve with its end values all-gathered by TorchComm (gloo), or (p2p)
    stored by k_zsub_ends into both ranks' IPC-opened end-value buffers."""
    import torch.multiprocessing as mp

    sys.path.insert(0, str(ROOT))
    import paper_2404_02433_b200 as P

    n, size = 128, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, size, port, n, q, zsolve, p2p)) for r in range(size)]
    for p in procs:
        p.start()
    res = []
    for _ in procs:
        res.append(q.get(timeout=300))
        assert res[-1][2] is None, res[-1][2]
    res.sort(key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for rank, out, err in res:
        assert err is None, err
    single = P.homogenize(P.gen_random_balls(n, 40, 0.05, 0.15, 100.0, 11),
                          P.BoundaryConfig(P.Axis("z"), 1.0, 0.0), 1e-8)
    for rank, (it, kappa, hist, ok) in [(r, o) for r, o, _ in res]:
        assert ok, "peer exchange not available for this geometry"
        assert it == single.iterations
        assert abs(kappa - single.kappa_eff) <= 1e-9 * abs(single.kappa_eff)
        h, s = np.array(hist), np.array(single.relative_residuals)
        big = s > 1e-2
        assert np.all(np.abs(h[big] - s[big]) <= 1e-8 * s[big])
    assert res[0][1][2] == res[1][1][2]  # both ranks report the same history
