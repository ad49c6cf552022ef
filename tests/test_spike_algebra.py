"""CPU check of the substructured ("spike") z-solve algebra that the CUDA
stages SLAB_ZSUB_TABS/ENDS/REDUCE/SOLVE implement: on the
per-mode tridiagonal T of preconditioner.py:184-250 (diag z_diag + shift,
couplings off), split into P row blocks, the spike end values, the 2x2
block elimination of the reduced system (k_zsub_reduce<P>) and the coupled
block solves reproduce the whole-column Thomas solve (oracle.thomas)."""

import numpy as np
import pytest

from oracle import etc_oracle as O


def _blocks_solve(zd, shift, off, d, P):
    nz = zd.size
    m = nz // P
    diag = zd + shift
    A = np.diag(diag) + np.diag(np.full(nz - 1, off), 1) + np.diag(np.full(nz - 1, off), -1)
    Vf, Vl, Wl, gf, gl = (np.zeros(P) for _ in range(5))
    for p in range(P):
        Ap = A[p * m:(p + 1) * m, p * m:(p + 1) * m]
        inv = np.linalg.inv(Ap)
        Vf[p], Vl[p], Wl[p] = off * inv[0, 0], off * inv[m - 1, 0], off * inv[m - 1, m - 1]
        g = np.linalg.solve(Ap, d[p * m:(p + 1) * m])
        gf[p], gl[p] = g[0], g[-1]
    # k_zsub_reduce<P>: z_p = (b_p, a_{p+1}); D_p = [[1, W_l(p)], [V_f(p+1), 1]],
    # L_p = V_l(p) on z_{p-1}[0], U_p = V_l(p+1) on z_{p+1}[1]
    NB = P - 1
    X, y = [None] * NB, [None] * NB
    for p in range(NB):
        D = np.array([[1.0, Wl[p]], [Vf[p + 1], 1.0]])
        r = np.array([gl[p], gf[p + 1]])
        if p > 0:
            D[0, 1] -= Vl[p] * X[p - 1][0, 1] * Vl[p]
            r[0] -= Vl[p] * (X[p - 1][0] @ y[p - 1])
        X[p], y[p] = np.linalg.inv(D), r
    z = [None] * NB
    for p in range(NB - 1, -1, -1):
        h = y[p].copy()
        if p < NB - 1:
            h[1] -= Vl[p + 1] * z[p + 1][1]
        z[p] = X[p] @ h
    x = np.empty(nz)
    for p in range(P):  # k_zsub_solve: A_p x = d - off b_{p-1} e_0 - off a_{p+1} e_{m-1}
        rhs = d[p * m:(p + 1) * m].copy()
        if p > 0:
            rhs[0] -= off * z[p - 1][0]
        if p < P - 1:
            rhs[-1] -= off * z[p][1]
        x[p * m:(p + 1) * m] = np.linalg.solve(A[p * m:(p + 1) * m, p * m:(p + 1) * m], rhs)
    return x


@pytest.mark.parametrize("P,m", [(2, 8), (3, 5), (4, 16), (8, 4), (8, 1), (5, 2)])
@pytest.mark.parametrize("shift", [0.0, 0.37, 25.0])
def test_spike_blocks_match_whole_column(P, m, shift):
    rng = np.random.default_rng(P * 100 + m)
    kz = 1.3
    nz = P * m
    zd = np.full(nz, 2.0 * kz)
    zd[0] += 2.0 * kz  # Dirichlet faces at both ends (z_diag, preconditioner.py:192-199)
    zd[-1] += 2.0 * kz
    d = rng.normal(size=nz)
    ref = O.thomas(np.array(shift), zd, -kz, d.reshape(nz, 1))[:, 0]
    x = _blocks_solve(zd, shift, -kz, d, P)
    assert np.allclose(x, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
