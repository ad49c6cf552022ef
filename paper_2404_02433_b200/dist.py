"""Multi-GPU z-slab decomposition of the solve.

The canonical grid nx*ny*nzg is split into P equal z-slabs, one per rank.
All the arithmetic runs in the same sm_100a kernels as the single-GPU path;
this module is the host side of the exchange steps:

* s and z halo planes: one plane each way to the z-neighbours (send/recv).
  s moves once per solve, z once per iteration, after the inverse transform.
* The per-mode z-solve runs on a z-pencil. The all-to-all turns the slab
  (nzl, ny, nx) into the pencil (nzg, ny/P, nx) and back.
* Three scalar all-reduces per iteration ({q.w, q.q, w.w}, r.r, r.z) feed the
  device-side finalisation of Alg. 1 (krylov.py:70-90). It stays
  bit-for-bit the single-GPU logic, in `k_finalize`.
* One min/max all-reduce of the coefficient statistics per solve; the LP and
  the tables stay on the host (preconditioner.py:117-199).

`slab_solve` is written against two small interfaces:

* `comm`: `TorchComm` over torch.distributed (NCCL across GPUs, gloo in tests),
  or `ThreadComm` (P virtual ranks in one process, threads + barriers, used to
  test the partitioned algebra on one GPU).
* `ops`: `CudaSlabOps` is the product, a thin wrapper of the C ABI
  `etc_slab_*`. Tests substitute a CPU restatement to check the decomposition
  with gloo.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native
from .reference import (
    CoefficientStats,
    check_pivots,
    eigen_weights,
    ones_reference,
    solve_reference_lp,
    z_chain_diagonal,
)
from .solver import PcgBreakdownError, SolveReport, _BREAKDOWN_MSG, _check, _torch

FIN_STENCIL, FIN_NORMB, FIN_UPDATE, FIN_THOMAS = 0, 1, 2, 3
(SLAB_FACES, SLAB_STATS, SLAB_NORMB, SLAB_FINALIZE, SLAB_STENCIL, SLAB_UPDATE, SLAB_PACK,
 SLAB_ZSOLVE, SLAB_UNPACK, SLAB_INVERSE, SLAB_PUPDATE, SLAB_FLUX,
 SLAB_ZSUB_TABS, SLAB_ZSUB_ENDS, SLAB_ZSUB_SOLVE) = range(15)


def slab_bounds(nzg: int, size: int, rank: int) -> tuple[int, int]:
    """Planes [k0, k0+nzl) of rank `rank` (equal slabs; P | nzg)."""
    if nzg % size:
        raise ValueError(f"nz={nzg} must be divisible by the number of ranks {size}")
    nzl = nzg // size
    return rank * nzl, nzl


# ----------------------------------------------------------------------------
# communicators
# ----------------------------------------------------------------------------


class TorchComm:
    """torch.distributed (NCCL on GPUs, gloo on CPU); collectives are
    stream-ordered with the caller's current stream."""

    def __init__(self, group=None):
        import torch.distributed as td

        self.td = td
        self.group = group
        self.rank = td.get_rank(group)
        self.size = td.get_world_size(group)

    def allreduce(self, t, op: str = "sum"):
        ops = {"sum": self.td.ReduceOp.SUM, "min": self.td.ReduceOp.MIN, "max": self.td.ReduceOp.MAX}
        self.td.all_reduce(t, op=ops[op], group=self.group)

    def _gloo_cuda(self, t) -> bool:
        """gloo moves host memory only: CUDA tensors are staged through the host"""
        return t.is_cuda and self.td.get_backend(self.group) == "gloo"

    def alltoall(self, out, inp):
        if self._gloo_cuda(inp):
            host = out.cpu()
            self.td.all_to_all_single(host, inp.cpu(), group=self.group)
            out.copy_(host)
            return
        self.td.all_to_all_single(out, inp, group=self.group)

    def allgather(self, out, inp):
        """out = [rank 0's inp, rank 1's inp, ...]"""
        n = inp.numel()
        if self._gloo_cuda(inp):
            host = out.cpu()
            self.td.all_gather([host[r * n:(r + 1) * n] for r in range(self.size)], inp.cpu(), group=self.group)
            out.copy_(host)
            return
        self.td.all_gather_into_tensor(out[:n * self.size], inp, group=self.group)

    def barrier(self):
        # peer stores were issued on the current stream: complete them first
        # (a gloo barrier is host-side)
        _torch().cuda.current_stream().synchronize()
        self.td.barrier(group=self.group)

    def peer_access_ok(self) -> bool:
        """Whether this rank's device can map every other visible device's
        memory (the precondition of the peer-store paths)."""
        torch = _torch()
        me, n = torch.cuda.current_device(), torch.cuda.device_count()
        return all(torch.cuda.can_device_access_peer(me, d) for d in range(n) if d != me)

    def share_pointers(self, ops, ptrs):
        """Every rank's device pointers `ptrs` as pointers valid in this
        process: own ones as they are, the peers' opened through CUDA IPC
        (handle of the plan allocation + byte offset)."""
        mine = [ops.ipc_handle(p) for p in ptrs]
        allh = [None] * self.size
        self.td.all_gather_object(allh, mine, group=self.group)
        out = []
        for r, hs in enumerate(allh):
            if r == self.rank:
                out.append(list(ptrs))
            else:
                out.append([_ipc_open(h, off) for h, off in hs])
        return out

    def neighbours(self, lo, hi, recv_lo, recv_hi):
        """send lo -> rank-1 (its upper halo), hi -> rank+1 (its lower halo);
        receive rank-1's hi into recv_lo and rank+1's lo into recv_hi."""
        td, r, p = self.td, self.rank, self.size
        if self._gloo_cuda(lo):
            hl, hh, rl, rh = lo.cpu(), hi.cpu(), recv_lo.cpu(), recv_hi.cpu()
            self.neighbours(hl, hh, rl, rh)
            recv_lo.copy_(rl)
            recv_hi.copy_(rh)
            return
        ops = []
        if r > 0:
            ops += [td.P2POp(td.isend, lo, r - 1, self.group), td.P2POp(td.irecv, recv_lo, r - 1, self.group)]
        if r < p - 1:
            ops += [td.P2POp(td.isend, hi, r + 1, self.group), td.P2POp(td.irecv, recv_hi, r + 1, self.group)]
        if ops:
            for req in td.batch_isend_irecv(ops):
                req.wait()


_IPC_OPEN = {}


def _ipc_open(handle: bytes, offset: int) -> int:
    """Open a peer's allocation once per process; base + offset."""
    base = _IPC_OPEN.get(handle)
    if base is None:
        ptr = C.c_void_p()
        _check(_native.lib().etc_ipc_open(C.c_char_p(handle), C.byref(ptr)), "etc_ipc_open")
        base = _IPC_OPEN[handle] = int(ptr.value)
    return base + offset


def release_ipc() -> None:
    """Close every peer allocation this process opened (they pin the peers'
    memory); call when the plans that used them are released."""
    lib = _native.lib()
    for base in _IPC_OPEN.values():
        lib.etc_ipc_close(C.c_void_p(base))
    _IPC_OPEN.clear()


class _ThreadHub:
    def __init__(self, size: int):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots: list = [None] * size


class ThreadComm:
    """P virtual ranks in one process (one thread each), sharing one device:
    exchanges are device copies between the ranks' buffers.  Used to run the
    partitioned algebra of the z-slab solve on a single GPU."""

    def __init__(self, hub: _ThreadHub, rank: int):
        self.hub = hub
        self.rank = rank
        self.size = hub.size

    @staticmethod
    def make(size: int):
        hub = _ThreadHub(size)
        return [ThreadComm(hub, r) for r in range(size)]

    def _sync(self):
        torch = _torch()
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self.hub.barrier.wait()

    def barrier(self):
        self._sync()

    def share_pointers(self, ops, ptrs):
        """One process: the ranks' device pointers are valid as they are."""
        self.hub.slots[self.rank] = list(ptrs)
        self._sync()
        out = [list(x) for x in self.hub.slots]
        self._sync()
        return out

    def allreduce(self, t, op: str = "sum"):
        self.hub.slots[self.rank] = t
        self._sync()
        acc = self.hub.slots[0].clone()
        for other in self.hub.slots[1:]:
            if op == "sum":
                acc = acc + other
            elif op == "min":
                acc = acc.minimum(other)
            else:
                acc = acc.maximum(other)
        self._sync()
        t.copy_(acc)
        self._sync()

    def alltoall(self, out, inp):
        self.hub.slots[self.rank] = inp
        self._sync()
        n = inp.numel() // self.size
        for s in range(self.size):
            out[s * n:(s + 1) * n].copy_(self.hub.slots[s][self.rank * n:(self.rank + 1) * n])
        self._sync()

    def allgather(self, out, inp):
        self.hub.slots[self.rank] = inp
        self._sync()
        n = inp.numel()
        for s in range(self.size):
            out[s * n:(s + 1) * n].copy_(self.hub.slots[s])
        self._sync()

    def neighbours(self, lo, hi, recv_lo, recv_hi):
        self.hub.slots[self.rank] = (lo, hi)
        self._sync()
        if self.rank > 0:
            recv_lo.copy_(self.hub.slots[self.rank - 1][1])
        if self.rank < self.size - 1:
            recv_hi.copy_(self.hub.slots[self.rank + 1][0])
        self._sync()


# ----------------------------------------------------------------------------
# device ops: the C ABI etc_slab_*
# ----------------------------------------------------------------------------


class CudaSlabOps:
    """One rank's slab plan in libetc_b200.so."""

    def __init__(self, nx, ny, nzg, k0, nzl, size, rank, lx, ly, lz, device=None):
        torch = _torch()
        self.lib = _native.lib()
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.nx, self.ny, self.nzg, self.k0, self.nzl = nx, ny, nzg, k0, nzl
        self.size, self.rank = size, rank
        self._h = C.c_void_p()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device).cuda_stream
            _check(self.lib.etc_slab_create(C.byref(self._h), nx, ny, nzg, k0, nzl, size, rank,
                                            float(lx), float(ly), float(lz), stream), "etc_slab_create")
        self._fin = weakref.finalize(self, self.lib.etc_plan_destroy, self._h)
        self._keep = None

    def _t(self, n):
        torch = _torch()
        return torch.empty(n, dtype=torch.float64, device=self.device)

    def new(self, n):
        return self._t(n)

    def load(self, kx, ky, kz):
        self._keep = (kx, ky, kz)
        _check(self.lib.etc_slab_load(self._h, kx.data_ptr(), ky.data_ptr(), kz.data_ptr(), 1), "etc_slab_load")

    def get_plane(self, which, plane):
        out = self._t(self.nx * self.ny)
        _check(self.lib.etc_slab_plane(self._h, which, plane, out.data_ptr(), 1), "etc_slab_plane")
        return out

    def set_plane(self, which, plane, t):
        _check(self.lib.etc_slab_plane(self._h, which, plane, t.data_ptr(), 0), "etc_slab_plane")

    def run(self, stage, arg=0, ext=None):
        _check(self.lib.etc_slab_run(self._h, stage, arg, ext.data_ptr() if ext is not None else None),
               "etc_slab_run")

    def stats(self):
        out = self._t(10)
        self.run(SLAB_STATS, 0, out)
        return out

    def set_reference(self, refs, wx, wy, zd):
        r5 = (C.c_double * 5)(*refs.constants())
        dp = _native._DP
        _check(self.lib.etc_set_reference(self._h, r5, wx.ctypes.data_as(dp), wy.ctypes.data_as(dp),
                                          zd.ctypes.data_as(dp)), "etc_set_reference")

    def init(self, p_in, p_out, rtol, max_iter, xbuf):
        _check(self.lib.etc_slab_init(self._h, float(p_in), float(p_out), float(rtol), int(max_iter),
                                      xbuf.data_ptr()), "etc_slab_init")

    def fused(self) -> bool:
        return bool(self.lib.etc_slab_fused(self._h))

    # -- peer exchange (fused all-to-all over peer memory) ---------------------
    def p2p_ok(self) -> bool:
        return bool(self.lib.etc_slab_p2p_ok(self._h))

    def xbuf(self, which: int) -> int:
        ptr = C.c_void_p()
        _check(self.lib.etc_slab_xbuf(self._h, which, C.byref(ptr)), "etc_slab_xbuf")
        return int(ptr.value)

    def plane_ptr(self, which: int, plane: int) -> int:
        ptr = C.c_void_p()
        _check(self.lib.etc_slab_plane_ptr(self._h, which, plane, C.byref(ptr)), "etc_slab_plane_ptr")
        return int(ptr.value)

    def ipc_handle(self, ptr: int):
        buf = C.create_string_buffer(64)
        off = C.c_size_t()
        _check(self.lib.etc_ipc_handle(self._h, C.c_void_p(ptr), buf, C.byref(off)), "etc_ipc_handle")
        return bytes(buf.raw), int(off.value)

    def set_ends_peers(self, ptrs):
        """Peer end-value buffers for k_zsub_ends (None: back to the all-gather)."""
        if ptrs is None:
            _check(self.lib.etc_slab_set_ends_peers(self._h, None), "etc_slab_set_ends_peers")
            return
        arr = C.c_void_p * len(ptrs)
        _check(self.lib.etc_slab_set_ends_peers(self._h, arr(*ptrs)), "etc_slab_set_ends_peers")

    def set_peers(self, recv_ptrs, back_ptrs):
        """Peer pencil / return buffers (None: the all-to-all path)."""
        if recv_ptrs is None or back_ptrs is None:
            _check(self.lib.etc_slab_set_peers(self._h, None, None), "etc_slab_set_peers")
            return
        arr = C.c_void_p * len(recv_ptrs)
        _check(self.lib.etc_slab_set_peers(self._h, arr(*recv_ptrs), arr(*back_ptrs)), "etc_slab_set_peers")

    def plane_view(self, which: int, plane: int):
        """A zero-copy float64 tensor over one plane of the plan's buffer
        `which` (planes -1 and nzl are the halos): collectives read and
        write the plan's planes in place, no staging copies."""
        key = (which, plane)
        views = self.__dict__.setdefault("_views", {})
        if key not in views:
            torch = _torch()
            ptr = self.plane_ptr(which, plane)
            n = self.nx * self.ny

            class _Plane:  # __cuda_array_interface__ carrier (the memory is the plan's)
                __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                            "strides": None}

            views[key] = torch.as_tensor(_Plane(), device=self.device)
        return views[key]

    def put_plane(self, which: int, plane: int, dst_ptr: int):
        """Copy this rank's plane into a (peer) device address."""
        _check(self.lib.etc_slab_plane(self._h, which, plane, C.c_void_p(dst_ptr), 1), "etc_slab_plane")

    def status(self, max_iter):
        info = _native.SolveInfo()
        hist = np.empty(max_iter + 1, dtype=np.float64)
        _check(self.lib.etc_slab_status(self._h, C.byref(info), hist.ctypes.data_as(_native._DP)),
               "etc_slab_status")
        return info, [float(v) for v in hist[: info.iterations + 1]]


# ----------------------------------------------------------------------------
# the distributed solve
# ----------------------------------------------------------------------------


@dataclass
class SlabResult:
    report: SolveReport
    rank: int
    size: int


def _exchange_planes(ops, comm, which: int, nzl: int):
    """One halo plane each way: my first plane -> the lower neighbour's upper
    halo, my last plane -> the upper neighbour's lower halo, sent and
    received in place through views of the plan's planes."""
    if comm.size == 1:
        return
    if hasattr(ops, "plane_view"):
        comm.neighbours(ops.plane_view(which, 0), ops.plane_view(which, nzl - 1), ops.plane_view(which, -1),
                        ops.plane_view(which, nzl))
        return
    lo = ops.get_plane(which, 0)
    hi = ops.get_plane(which, nzl - 1)
    recv_lo = ops.new(lo.numel())
    recv_hi = ops.new(hi.numel())
    comm.neighbours(lo, hi, recv_lo, recv_hi)
    if comm.rank > 0:
        ops.set_plane(which, -1, recv_lo)
    if comm.rank < comm.size - 1:
        ops.set_plane(which, nzl, recv_hi)


def _next_check(it: int, history: list, rtol: float, cap: int = 16) -> int:
    """Iteration of the next host status read.  The device stops itself
    (Ctl.done; every stage kernel early-exits), so the host only needs to
    notice: predict the iteration that reaches rtol from the recent
    geometric residual rate and look again there (at most `cap` later)."""
    h = [v for v in history if v > 0.0]
    if len(h) < 3 or h[-1] <= rtol:
        return it + 1
    span = min(len(h) - 1, 8)
    rate = (h[-1] / h[-1 - span]) ** (1.0 / span)
    if not (0.0 < rate < 1.0):
        return it + 4
    need = np.log(rtol / h[-1]) / np.log(rate)
    return it + int(max(1, min(cap, np.floor(need))))


def slab_solve(ops, comm, kx, ky, kz, grid, p_in=1.0, p_out=0.0, rtol=1e-9, ref_mode="opt",
               max_iter=1024, check_every=None, p2p=None, zsolve=None) -> SolveReport:
    """PCG on this rank's z-slab of the canonical field (kx, ky, kz: local
    planes, x-fastest).  grid = (nx, ny, nzg, lx, ly, lz), the canonical
    global grid.  Every rank returns the same report.

    p2p (default: ETC_P2P=1 in the environment): the pencil all-to-alls are
    fused into the producing kernels over peer memory (the forward transform
    stores into the destination ranks' pencil buffers, the z-solve into the
    owners' return buffers; halo planes are stored into the neighbours' halo
    planes), where the plan supports it (etc_slab_p2p_ok) and the comm can
    share device pointers (same process, or CUDA IPC).

    zsolve (default: ETC_ZSOLVE in the environment, else "pencil"): "pencil"
    moves the spectrum through two all-to-alls so that every z-column is
    solved whole on one rank; "spike" solves each rank's block of every
    column in place (substructured tridiagonal): the ranks
    exchange only the two end values of their block solutions per column
    (an all-gather of 2·nx·ny doubles per rank) and every rank solves the
    small reduced system of the block-boundary unknowns."""
    nx, ny, nzg, lx, ly, lz = grid
    nzl = nzg // comm.size
    if zsolve is None:
        import os

        zsolve = os.environ.get("ETC_ZSOLVE", "pencil")
    if zsolve not in ("pencil", "spike"):
        raise ValueError(f"zsolve must be 'pencil' or 'spike', not {zsolve!r}")
    spike = zsolve == "spike"
    spike_p2p = False
    if spike:
        if p2p is None:
            import os

            p2p = os.environ.get("ETC_P2P", "0") == "1"
        # the end values go to the peers by stores from k_zsub_ends (no all-gather)
        spike_p2p = bool(p2p) and hasattr(comm, "share_pointers") and hasattr(ops, "set_ends_peers")
        if p2p and comm.size > 1:  # every rank must agree (else the collectives mismatch and hang)
            t = ops.new(1)
            t.fill_(float(spike_p2p and getattr(comm, "peer_access_ok", lambda: True)()))
            comm.allreduce(t, "min")
            spike_p2p = bool(float(t.cpu().item()) > 0.5)
        p2p = False
    iso = kx is ky and ky is kz
    ops.load(kx, ky, kz)
    if p2p is None:
        import os

        p2p = os.environ.get("ETC_P2P", "0") == "1"
    use_p2p = bool(p2p) and hasattr(comm, "share_pointers") and hasattr(ops, "p2p_ok") and ops.p2p_ok()
    if p2p and comm.size > 1:  # every rank must agree
        t = ops.new(1)
        t.fill_(float(use_p2p))
        comm.allreduce(t, "min")
        use_p2p = bool(float(t.cpu().item()) > 0.5)
    # plans are cached across solves: peer tables a previous solve installed
    # must not leak into this one's mode (the kernels would store into the
    # peers' buffers and skip the local ones)
    if not use_p2p and hasattr(ops, "set_peers"):
        ops.set_peers(None, None)
    if not spike_p2p and hasattr(ops, "set_ends_peers"):
        ops.set_ends_peers(None)
    if use_p2p:
        # [pencil, return, s_x, s_y, s_z, w] (plane 0) of every rank
        table = comm.share_pointers(ops, [ops.xbuf(0), ops.xbuf(1), ops.plane_ptr(0, 0), ops.plane_ptr(1, 0),
                                          ops.plane_ptr(2, 0), ops.plane_ptr(4, 0)])
        ops.set_peers([t[0] for t in table], [t[1] for t in table])
        pbytes = nx * ny * 8
        slot = {0: 2, 1: 3, 2: 4, 4: 5}

        def put_halos(whiches):
            for which in whiches:
                if comm.rank > 0:  # my first plane -> the lower neighbour's upper halo (plane nzl)
                    ops.put_plane(which, 0, table[comm.rank - 1][slot[which]] + nzl * pbytes)
                if comm.rank < comm.size - 1:  # my last plane -> the upper neighbour's lower halo (plane -1)
                    ops.put_plane(which, nzl - 1, table[comm.rank + 1][slot[which]] - pbytes)
            comm.barrier()

        put_halos((2,) if iso else (0, 1, 2))
    else:
        for which in ((2,) if iso else (0, 1, 2)):
            _exchange_planes(ops, comm, which, nzl)
    ops.run(SLAB_FACES)
    st = ops.stats()
    lo, hi = st[0::2].clone(), st[1::2].clone()
    comm.allreduce(lo, "min")
    comm.allreduce(hi, "max")
    vals = np.empty(10)
    vals[0::2] = lo.cpu().numpy()
    vals[1::2] = hi.cpu().numpy()
    # empty groups (no faces along an axis of length 1) -> (1, 1) (preconditioner.py:94-98)
    for g, n in ((0, nx), (1, ny), (2, nzg)):
        if n < 2:
            vals[2 * g], vals[2 * g + 1] = 1.0, 1.0
    stats = CoefficientStats(*[float(v) for v in vals])
    refs = solve_reference_lp(stats) if ref_mode == "opt" else ones_reference(stats)
    wx, wy, zd = eigen_weights(nx), eigen_weights(ny), z_chain_diagonal(nzg, refs)
    check_pivots(nzg, zd, refs)
    ops.set_reference(refs, wx, wy, zd)
    if spike:
        ops.run(SLAB_ZSUB_TABS)  # every block's spike end values (matrix only, once per solve)

    xbuf = ops.new(8)
    xbuf.zero_()
    nloc = nx * ny * nzl
    send = ops.new(nloc)
    recv = ops.new(nloc)

    # fused path (square power-of-two planes): the inverse stage builds the
    # search direction w itself, so the w halo planes move instead of z
    fused = ops.fused()

    # on the fused path the forward transform writes its spectrum straight
    # into the all-to-all send buffer and the inverse reads it back from there
    # (pack / unpack fused into the transforms)
    spec = None if (use_p2p or spike) else (send if fused else None)
    if spike:
        ends = ops.new(2 * nx * ny)
        ends_all = ops.new(2 * nx * ny * comm.size)
        if spike_p2p:
            table = comm.share_pointers(ops, [ops.xbuf(2)])
            ops.set_ends_peers([t[0] for t in table])
            fence = ops.new(1)

    def zsolve_and_back(first):
        if spike:
            if spike_p2p:
                ops.run(SLAB_ZSUB_ENDS, 0, None)        # stored into every rank's end-value buffer
                comm.allreduce(fence)                   # ... a one-element all-reduce is the barrier
                ops.run(SLAB_ZSUB_SOLVE, 0, None)
            else:
                ops.run(SLAB_ZSUB_ENDS, 0, ends)        # g_first, g_last of the local block solves
                comm.allgather(ends_all, ends)
                ops.run(SLAB_ZSUB_SOLVE, 0, ends_all)   # reduced system, then the coupled block solve
            comm.allreduce(xbuf[4:5])
            ops.run(SLAB_FINALIZE, FIN_THOMAS)
            ops.run(SLAB_INVERSE, 1 if first else 2, None)
            _exchange_planes(ops, comm, 4 if fused else 3, nzl)
            return
        if use_p2p:
            # the forward stage stored the spectrum into the peers' pencil
            # buffers; the scalar all-reduce after it was the barrier
            ops.run(SLAB_ZSOLVE, 0, None)  # own pencil buffer -> the owners' return buffers
            comm.allreduce(xbuf[4:5])      # ... and the barrier before the inverse reads them
            ops.run(SLAB_FINALIZE, FIN_THOMAS)
            ops.run(SLAB_INVERSE, 1 if first else 2, None)
            put_halos((4,))
            return
        if not fused:
            ops.run(SLAB_PACK, 0, send)
        if comm.size == 1:  # one rank: the pencil is the slab, the all-to-alls are identities
            ops.run(SLAB_ZSOLVE, 0, send)
        else:
            comm.alltoall(recv, send)
            ops.run(SLAB_ZSOLVE, 0, recv)
            comm.alltoall(send, recv)
        if not fused:
            ops.run(SLAB_UNPACK, 0, send)
        comm.allreduce(xbuf[4:5])
        ops.run(SLAB_FINALIZE, FIN_THOMAS)
        ops.run(SLAB_INVERSE, 1 if first else 2, spec)
        _exchange_planes(ops, comm, 4 if fused else 3, nzl)

    ops.init(p_in, p_out, rtol, max_iter, xbuf)
    ops.run(SLAB_NORMB, 0, spec)
    comm.allreduce(xbuf[3:4])
    ops.run(SLAB_FINALIZE, FIN_NORMB)
    zsolve_and_back(True)
    it = 0
    done = False
    # the host reads the device state only where convergence is predicted
    # (check_every: a fixed period instead); in between it enqueues the next
    # iterations' stages and collectives without waiting, and after the
    # device has set Ctl.done the stage kernels return at once
    nxt = 1
    while not done and it < max_iter:
        it += 1
        ops.run(SLAB_STENCIL, it)
        comm.allreduce(xbuf[0:3])
        ops.run(SLAB_FINALIZE, FIN_STENCIL)
        ops.run(SLAB_UPDATE, 0, spec)
        comm.allreduce(xbuf[3:4])
        ops.run(SLAB_FINALIZE, FIN_UPDATE)
        zsolve_and_back(False)
        if it >= nxt or it == max_iter:
            info, hist = ops.status(max_iter)
            done = info.pad_ != 0
            nxt = it + check_every if check_every else _next_check(it, hist, rtol)
    info, history = ops.status(max_iter)
    if info.status:
        raise PcgBreakdownError(_BREAKDOWN_MSG.get(info.breakdown_kind, "breakdown"), info.breakdown_iter)
    ops.run(SLAB_PUPDATE, info.iterations)
    fbuf = ops.new(1)
    ops.run(SLAB_FLUX, 0, fbuf)
    comm.allreduce(fbuf)
    flux = float(fbuf.cpu().item())
    kappa = lz * flux / (nx * ny * (p_in - p_out))
    return SolveReport(iterations=int(info.iterations), converged=bool(history[-1] <= rtol),
                       relative_residuals=history, kappa_eff=kappa, ref_params=refs)


def virtual_slab_solve(field_cube, grid, nranks: int, p_in=1.0, p_out=0.0, rtol=1e-9, ref_mode="opt",
                       max_iter=1024, device=None, p2p=None, zsolve=None) -> list:
    """Run the z-slab solve with `nranks` virtual ranks on one GPU (threads +
    device copies stand in for NCCL); field_cube: canonical (nzg, ny, nx)
    CUDA tensor (isotropic field).  Returns every rank's report."""
    torch = _torch()
    nx, ny, nzg, lx, ly, lz = grid
    comms = ThreadComm.make(nranks)
    out: list = [None] * nranks
    errs: list = []
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())

    def worker(r):
        try:
            torch.cuda.set_device(dev)
            k0, nzl = slab_bounds(nzg, nranks, r)
            k = field_cube[k0:k0 + nzl].contiguous().reshape(-1)
            ops = CudaSlabOps(nx, ny, nzg, k0, nzl, nranks, r, lx, ly, lz, dev)
            out[r] = slab_solve(ops, comms[r], k, k, k, grid, p_in, p_out, rtol, ref_mode, max_iter, p2p=p2p,
                                zsolve=zsolve)
        except BaseException as exc:  # surface worker failures
            errs.append(exc)
            comms[r].hub.barrier.abort()

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    return out


# ----------------------------------------------------------------------------
# public multi-GPU entry point
# ----------------------------------------------------------------------------

_OPS_CACHE: dict = {}


def release_slab_plans() -> None:
    """Drop the cached rank plans and close the peer allocations they opened."""
    _OPS_CACHE.clear()
    release_ipc()


def _transpose_slab(local, axis: str, comm, nx: int, ny: int, nz: int):
    """axis_permute (pipeline.py:87-111) of a z-slab-distributed cube as one
    all-to-all: `local` is this rank's original planes [k0, k0+nzl) as an
    (nzl, ny, nx) CUDA tensor; returns its slab of the canonical cube for
    `axis` (x: canonical (nz', ny', nx') = (nx, ny, nz); y: (ny, nz, nx)),
    planes [r m, (r+1) m) with m = nx / P (x) or ny / P (y).  No rank ever
    holds more than its slab (plus the send / receive blocks)."""
    P, nzl = comm.size, nz // comm.size
    if axis == "x":
        m = nx // P
        send = local.permute(2, 1, 0).contiguous()            # [x][y][z_l]: destination-major blocks
        recv = torch_empty_like_flat(send)
        comm.alltoall(recv, send.reshape(-1))
        return recv.reshape(P, m, ny, nzl).permute(1, 2, 0, 3).reshape(m, ny, nz).contiguous()
    m = ny // P
    send = local.permute(1, 0, 2).contiguous()                # [y][z_l][x]
    recv = torch_empty_like_flat(send)
    comm.alltoall(recv, send.reshape(-1))
    return recv.reshape(P, m, nzl, nx).permute(1, 0, 2, 3).reshape(m, nz, nx).contiguous()


def torch_empty_like_flat(t):
    return _torch().empty(t.numel(), dtype=t.dtype, device=t.device)


def canonical_slabs(local, grid, axis: str, comm):
    """This rank's slab of the canonical field for `axis` from its slab of the
    ORIGINAL field (kx, ky, kz as (nzl, ny, nx) tensors; kx is ky is kz marks
    an isotropic field, moved once).  Returns ((kx', ky', kz') flat, the
    canonical grid)."""
    nx, ny, nz, lx, ly, lz = grid
    kx, ky, kz = local
    iso = kx is ky and ky is kz
    if axis == "z":
        flat = [a.reshape(-1) for a in (kx, ky, kz)]
        return (flat[0], flat[0], flat[0]) if iso else tuple(flat), grid
    if (nx if axis == "x" else ny) % comm.size:
        raise ValueError(f"{'nx' if axis == 'x' else 'ny'} must be divisible by the number of ranks")
    tr = lambda a: _transpose_slab(a, axis, comm, nx, ny, nz).reshape(-1)  # noqa: E731
    if axis == "x":
        cgrid = (nz, ny, nx, lz, ly, lx)
        if iso:
            t = tr(kx)
            return (t, t, t), cgrid
        return (tr(kz), tr(ky), tr(kx)), cgrid
    cgrid = (nx, nz, ny, lx, lz, ly)
    if iso:
        t = tr(kx)
        return (t, t, t), cgrid
    return (tr(kx), tr(kz), tr(ky)), cgrid


def effective_tensor_dist_slab(local, grid, comm=None, rtol: float = 1e-9, p_in: float = 1.0, p_out: float = 0.0,
                               ref_mode: str = "opt", max_iter: int = 1024, axes: str = "xyz", device=None,
                               zsolve=None):
    """Multi-GPU effective tensor from distributed input: each rank passes
    only its z-slab of the original field (`local` = (kx, ky, kz), each an
    (nz/P, ny, nx) CUDA tensor, the same object three times for an isotropic
    field) and the global grid (nx, ny, nz, lx, ly, lz).  Load directions
    x and y are permuted by an all-to-all transpose of the slabs
    (canonical_slabs), so no rank holds the whole field.  Returns
    (kappa[3], {axis: SolveReport}) on every rank."""
    torch = _torch()
    comm = comm or TorchComm()
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    reports = {}
    for ax in axes:
        (kx, ky, kz), cgrid = canonical_slabs(local, grid, ax, comm)
        nx, ny, nzg = cgrid[:3]
        k0, nzl = slab_bounds(nzg, comm.size, comm.rank)
        key = (cgrid, comm.rank, comm.size, dev.index)
        ops = _OPS_CACHE.get(key)
        if ops is None:
            ops = CudaSlabOps(nx, ny, nzg, k0, nzl, comm.size, comm.rank, cgrid[3], cgrid[4], cgrid[5], dev)
            _OPS_CACHE[key] = ops
        reports[ax] = slab_solve(ops, comm, kx, ky, kz, cgrid, p_in, p_out, rtol, ref_mode, max_iter,
                                 zsolve=zsolve)
    kappa = np.array([reports[a].kappa_eff if a in reports else np.nan for a in "xyz"])
    return kappa, reports


def effective_tensor_dist(field, comm=None, rtol: float = 1e-9, p_in: float = 1.0, p_out: float = 0.0,
                          ref_mode: str = "opt", max_iter: int = 1024, axes: str = "xyz", device=None,
                          zsolve=None):
    """Multi-GPU effective_tensor from a field every rank can see (host numpy
    or CUDA tensors): each rank takes its z-slab of the original field (one
    copy of 1/P of it) and hands it to effective_tensor_dist_slab."""
    torch = _torch()
    from .solver import _as_field

    comm = comm or TorchComm()
    fld = _as_field(field)
    g = fld.grid
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    k0, nzl = slab_bounds(g.nz, comm.size, comm.rank)

    def slab(a):
        part = a.reshape(g.nz, g.ny, g.nx)[k0:k0 + nzl]
        if isinstance(part, np.ndarray):
            # a z-slab of a C-ordered cube is contiguous: upload it in place
            # (pinned host memory stays a DMA source), no host-side copy
            import warnings

            with warnings.catch_warnings():
                warnings.simplefilter("ignore", UserWarning)  # frozen (read-only) field arrays
                part = torch.from_numpy(np.ascontiguousarray(part))
            out = torch.empty(part.shape, dtype=part.dtype, device=dev)
            out.copy_(part)
            return out
        return part.to(dev).contiguous()

    iso = fld.kx is fld.ky and fld.ky is fld.kz
    local = (slab(fld.kx),) * 3 if iso else tuple(slab(a) for a in (fld.kx, fld.ky, fld.kz))
    return effective_tensor_dist_slab(local, (g.nx, g.ny, g.nz, g.lx, g.ly, g.lz), comm, rtol, p_in, p_out,
                                      ref_mode, max_iter, axes, dev, zsolve)
