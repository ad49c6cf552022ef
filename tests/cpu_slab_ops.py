"""CPU restatement of the z-slab stages (TEST INFRASTRUCTURE ONLY).

Implements the `ops` interface that `paper_2404_02433_b200.dist.slab_solve`
drives. Each method does in numpy exactly what the matching `etc_slab_run` stage
does on the GPU. It lets the host-side decomposition run over a real gloo
process group on CPU:

* halo planes, pencil all-to-all, scalar all-reduces;
* device-side finalisation order and the stop logic.

The test compares the result with the single-process oracle.
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np
import torch

from oracle import etc_oracle as O

EPS = 2.220446049250313e-16


class CpuSlabOps:
    def __init__(self, nx, ny, nzg, k0, nzl, size, rank, lx, ly, lz, fused=False):
        self.nx, self.ny, self.nzg, self.k0, self.nzl = nx, ny, nzg, k0, nzl
        self.size, self.rank = size, rank
        self.lx, self.ly, self.lz = lx, ly, lz
        self.s = None
        self.ctl = None
        self._fused = fused  # the inverse builds w (etc_slab_fused)

    def fused(self):
        return self._fused

    # -- buffers ------------------------------------------------------------
    def new(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def load(self, kx, ky, kz):
        nzl, ny, nx = self.nzl, self.ny, self.nx
        h = (self.lx / nx, self.ly / ny, self.lz / self.nzg)
        self.s = []
        for a, k in enumerate((kx, ky, kz)):
            ext = np.zeros((nzl + 2, ny, nx))
            ext[1:-1] = O.scale(k.numpy().reshape(nzl, ny, nx), h[a])
            self.s.append(ext)
        self.z = np.zeros((nzl + 2, ny, nx))
        self.w = [np.zeros((nzl + 2, ny, nx)), np.zeros((nzl + 2, ny, nx))]
        self.wf = np.zeros((nzl + 2, ny, nx))  # fused path: the search direction, with halos

    def _buf(self, which):
        return self.s[which] if which <= 2 else (self.z if which == 3 else self.wf)

    def get_plane(self, which, plane):
        return torch.from_numpy(self._buf(which)[plane + 1].reshape(-1).copy())

    def set_plane(self, which, plane, t):
        self._buf(which)[plane + 1] = t.numpy().reshape(self.ny, self.nx)

    # -- stages ---------------------------------------------------------------
    def _kg(self, k):
        return self.k0 + k

    def run(self, stage, arg=0, ext=None):
        getattr(self, "_stage%d" % stage)(arg, ext)

    def _stage0(self, arg, ext):  # faces
        sx, sy, sz = self.s
        self.tx = O.harmonic(sx[1:-1, :, :-1], sx[1:-1, :, 1:])
        self.ty = O.harmonic(sy[1:-1, :-1, :], sy[1:-1, 1:, :])
        # tz[k] (k = -1..nzl-1): face between local planes k and k+1
        self.tz = O.harmonic(sz[:-1], sz[1:])

    def stats(self):
        nzl = self.nzl
        out = np.array([np.inf, 0.0] * 5)

        def upd(g, arr):
            if arr.size:
                out[2 * g] = min(out[2 * g], arr.min())
                out[2 * g + 1] = max(out[2 * g + 1], arr.max())

        upd(0, self.tx)
        upd(1, self.ty)
        owned = [k for k in range(nzl) if self._kg(k) + 1 < self.nzg]
        if owned:
            upd(2, self.tz[np.array(owned) + 1])
        if self.k0 == 0:
            upd(3, self.s[2][1])
        if self.k0 + nzl == self.nzg:
            upd(4, self.s[2][nzl])
        return torch.from_numpy(out)

    def set_reference(self, refs, wx, wy, zd):
        self.refs = refs
        self.shift = wx[None, :] * refs.kx_ref + wy[:, None] * refs.ky_ref
        self.zd = zd
        self.off = -refs.kz_ref

    def init(self, p_in, p_out, rtol, max_iter, xbuf):
        self.ctl = SimpleNamespace(rho=0.0, alpha=0.0, beta=0.0, norm_b=0.0, rtol=rtol, it=0, max_iter=max_iter,
                                   done=0, status=0, bd_iter=0, bd_kind=0, converged=0)
        self.hist = [0.0] * (max_iter + 1)
        self.xbuf = xbuf
        self.p_in, self.p_out = p_in, p_out
        nzl = self.nzl
        sz = self.s[2][1:-1]
        self.r = np.zeros((nzl, self.ny, self.nx))
        if self.k0 == 0:
            self.r[0] = (2.0 * sz[0]) * p_in
        if self.k0 + nzl == self.nzg:
            self.r[-1] += (2.0 * sz[-1]) * p_out
        self.p = np.zeros_like(self.r)

    def _pack(self, ext):
        nyl = self.ny // self.size
        blocks = [self.t[:, r * nyl:(r + 1) * nyl, :] for r in range(self.size)]
        ext.copy_(torch.from_numpy(np.concatenate([b.reshape(-1) for b in blocks])))

    def _unpack(self, ext):
        nyl = self.ny // self.size
        a = ext.numpy().reshape(self.size, self.nzl, nyl, self.nx)
        self.t = np.concatenate([a[s] for s in range(self.size)], axis=1)

    def _stage2(self, arg, ext):  # ||b|| + first transform (fused: written packed into ext)
        self.xbuf[3] = float(np.sum(self.r * self.r))
        self.t = O.fct_forward(self.r)
        if ext is not None:
            self._pack(ext)

    def _stage3(self, stage, ext):  # finalize
        c, x = self.ctl, self.xbuf.numpy()
        if c.done and stage != 1:
            return
        if stage == 0:
            if x[0] <= 100.0 * EPS * math.sqrt(x[1]) * math.sqrt(x[2]):
                c.status, c.bd_kind, c.bd_iter, c.done = 1, 1, c.it + 1, 1
            c.alpha = c.rho / x[0]
        elif stage == 1:
            c.norm_b = math.sqrt(x[3])
            self.hist[0] = 1.0 if c.norm_b != 0.0 else 0.0
            if c.norm_b == 0.0:
                c.converged, c.done = 1, 1
        elif stage == 2:
            rel = math.sqrt(x[3]) / c.norm_b
            if not math.isfinite(rel):
                c.status, c.bd_kind, c.bd_iter, c.done = 1, 2, c.it + 1, 1
                return
            c.it += 1
            self.hist[c.it] = rel
            if rel <= c.rtol:
                c.converged, c.done = 1, 1
        else:
            rz = x[4] * 4.0 / (self.nx * self.ny)
            if c.it == 0:
                if rz <= 0.0:
                    c.status, c.bd_kind, c.bd_iter, c.done = 1, 3, 0, 1
                c.rho = rz
            else:
                if rz <= 0.0:
                    c.status, c.bd_kind, c.bd_iter, c.done = 1, 3, c.it, 1
                else:
                    c.beta = rz / c.rho
                    c.rho = rz
                if c.it >= c.max_iter:
                    c.done = 1

    def _stage4(self, it, ext):  # stencil (+ previous p update, dots)
        c = self.ctl
        if c.done:
            return
        if self._fused:
            u = self.wf
        else:
            wn, wo = self.w[it & 1], self.w[(it - 1) & 1]
            if it == 1:
                wn[:] = self.z
            else:
                wn[:] = self.z + c.beta * wo
                kl = self.nzg - 1 - self.k0
                if 0 <= kl < self.nzl:
                    self.p[kl] = self.p[kl] + c.alpha * wo[kl + 1]
            u = wn
        nzl = self.nzl
        q = np.zeros((nzl, self.ny, self.nx))
        core = u[1:-1]
        for t, axis in ((self.tx, 2), (self.ty, 1)):
            hi = [slice(None)] * 3
            lo = [slice(None)] * 3
            hi[axis] = slice(1, None)
            lo[axis] = slice(None, -1)
            f = t * (core[tuple(hi)] - core[tuple(lo)])
            q[tuple(hi)] += f
            q[tuple(lo)] -= f
        for k in range(nzl):
            kg = self._kg(k)
            if kg > 0:
                q[k] += self.tz[k] * (u[k + 1] - u[k])
            if kg + 1 < self.nzg:
                q[k] -= self.tz[k + 1] * (u[k + 2] - u[k + 1])
            if kg == 0:
                q[k] += (2.0 * self.s[2][k + 1]) * u[k + 1]
            if kg == self.nzg - 1:
                q[k] += (2.0 * self.s[2][k + 1]) * u[k + 1]
        self.q = q
        self.xbuf[0] = float(np.sum(q * core))
        self.xbuf[1] = float(np.sum(q * q))
        self.xbuf[2] = float(np.sum(core * core))

    def _stage5(self, arg, ext):  # r -= alpha q; ||r||; transform (fused: written packed into ext)
        if self.ctl.done:
            return
        self.r = self.r - self.ctl.alpha * self.q
        self.xbuf[3] = float(np.sum(self.r * self.r))
        self.t = O.fct_forward(self.r)
        if ext is not None:
            self._pack(ext)

    def _stage6(self, arg, ext):  # pack
        self._pack(ext)

    def _stage7(self, arg, ext):  # z-solve on the pencil
        if self.ctl.done:
            return
        nyl = self.ny // self.size
        pen = ext.numpy().reshape(self.nzg, nyl, self.nx)
        j0 = self.rank * nyl
        shift = self.shift[j0:j0 + nyl]
        x = O.thomas(shift, self.zd, self.off, pen)
        ax = np.where(np.arange(self.nx) == 0, 0.5, 1.0)
        ay = np.where(np.arange(j0, j0 + nyl) == 0, 0.5, 1.0)
        self.xbuf[4] = float(np.sum(ay[:, None] * ax[None, :] * pen * x))
        ext.copy_(torch.from_numpy(x.reshape(-1)))

    def _stage8(self, arg, ext):  # unpack
        self._unpack(ext)

    def _stage9(self, arg, ext):  # inverse transform (fused: builds w, arg 1 first / 2 update; reads ext)
        c = self.ctl
        if c.done:
            return
        if ext is not None:
            self._unpack(ext)
        self.z[1:-1] = O.fct_backward(self.t)
        if self._fused:
            if arg == 1:
                self.wf[1:-1] = self.z[1:-1]
            else:
                kl = self.nzg - 1 - self.k0
                if 0 <= kl < self.nzl:
                    self.p[kl] = self.p[kl] + c.alpha * self.wf[kl + 1]
                self.wf[1:-1] = self.z[1:-1] + c.beta * self.wf[1:-1]

    def _stage10(self, it, ext):  # final p update on the outflow plane
        kl = self.nzg - 1 - self.k0
        w = self.wf if self._fused else self.w[it & 1]
        if it >= 1 and 0 <= kl < self.nzl:
            self.p[kl] = self.p[kl] + self.ctl.alpha * w[kl + 1]

    def _stage11(self, arg, ext):  # outflow flux
        kl = self.nzg - 1 - self.k0
        hz = self.lz / self.nzg
        s = 0.0
        if 0 <= kl < self.nzl:
            tout = 2.0 * self.s[2][kl + 1]
            s = float(np.sum((tout * hz) * (self.p[kl] - self.p_out)))
        ext[0] = s

    # -- substructured ("spike") z-solve: stages 12-14 -----------------------
    def _diag(self, kg):
        return self.zd[kg] + self.shift

    def _stage12(self, arg, ext):  # spike end values of every block (matrix only)
        m, P, off = self.nzl, self.size, self.off
        self.sp = []
        for p in range(P):
            r = 1.0 / self._diag(p * m)
            y = r.copy()  # forward elimination of e_0
            for k in range(1, m):
                r = 1.0 / (self._diag(p * m + k) - off * off * r)
                y = -off * y * r
            rb = 1.0 / self._diag(p * m + m - 1)
            for k in range(m - 2, -1, -1):
                rb = 1.0 / (self._diag(p * m + k) - off * off * rb)
            # V = A_p^-1 (off e_0), W = A_p^-1 (off e_last): first/last entries
            self.sp.append((off * rb, off * y, off * r))  # V_f, V_l (= W_f), W_l

    def _block_solve(self, d, top, bot):
        """A_p x = d - off top e_0 - off bot e_last (top-down elimination)."""
        m, off, k0 = self.nzl, self.off, self.k0
        d = d.copy()
        d[0] = d[0] - off * top
        d[m - 1] = d[m - 1] - off * bot
        rp = np.empty_like(d)
        rp[0] = 1.0 / self._diag(k0)
        d[0] = d[0] * rp[0]
        for k in range(1, m):
            rp[k] = 1.0 / (self._diag(k0 + k) - off * off * rp[k - 1])
            d[k] = (d[k] - off * d[k - 1]) * rp[k]
        for k in range(m - 2, -1, -1):
            d[k] = d[k] - off * rp[k] * d[k + 1]
        return d

    def _stage13(self, arg, ext):  # g = A_p^-1 t: first and last values -> ext
        if self.ctl.done:
            return
        g = self._block_solve(self.t, 0.0, 0.0)
        ext.copy_(torch.from_numpy(np.concatenate([g[0].reshape(-1), g[-1].reshape(-1)])))

    def _stage14(self, arg, ext):  # reduced system of the block-boundary values, coupled block solve
        if self.ctl.done:
            return
        P, me, plane = self.size, self.rank, self.nx * self.ny
        e = ext.numpy().reshape(P, 2, self.ny, self.nx)
        top = np.zeros((self.ny, self.nx))
        bot = np.zeros((self.ny, self.nx))
        if P > 1:
            n = 2 * (P - 1)  # unknowns b_0, a_1, b_1, a_2, ..., b_{P-2}, a_{P-1}
            M = np.zeros((self.ny, self.nx, n, n))
            rhs = np.zeros((self.ny, self.nx, n))
            for p in range(P - 1):
                vf, vl, wl = self.sp[p]
                M[..., 2 * p, 2 * p] = 1.0  # b_p + V_l(p) b_{p-1} + W_l(p) a_{p+1} = g_l(p)
                if p > 0:
                    M[..., 2 * p, 2 * p - 2] = vl
                M[..., 2 * p, 2 * p + 1] = wl
                rhs[..., 2 * p] = e[p, 1]
                vf1, vl1, _ = self.sp[p + 1]  # a_{p+1} + V_f(p+1) b_p + W_f(p+1) a_{p+2} = g_f(p+1)
                M[..., 2 * p + 1, 2 * p + 1] = 1.0
                M[..., 2 * p + 1, 2 * p] = vf1
                if p + 1 < P - 1:
                    M[..., 2 * p + 1, 2 * p + 3] = vl1
                rhs[..., 2 * p + 1] = e[p + 1, 0]
            sol = np.linalg.solve(M, rhs[..., None])[..., 0]
            if me > 0:
                top = sol[..., 2 * (me - 1)]
            if me < P - 1:
                bot = sol[..., 2 * me + 1]
        x = self._block_solve(self.t, top, bot)
        ax = np.where(np.arange(self.nx) == 0, 0.5, 1.0)
        ay = np.where(np.arange(self.ny) == 0, 0.5, 1.0)
        self.xbuf[4] = float(np.sum(ay[:, None] * ax[None, :] * self.t * x))
        self.t = x

    def status(self, max_iter):
        c = self.ctl
        info = SimpleNamespace(iterations=c.it, converged=c.converged, status=c.status, breakdown_iter=c.bd_iter,
                               breakdown_kind=c.bd_kind, pad_=c.done)
        return info, [float(v) for v in self.hist[:c.it + 1]]
