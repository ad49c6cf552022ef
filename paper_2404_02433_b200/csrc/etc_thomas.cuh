// etc_thomas.cuh — register-staged z-solves of the FCT preconditioner
// (thomas_solve_batch, reference /root/reference/pkg/src/etchomo/
// preconditioner.py:215-250): the runtime-size k_thomas, the exact-fit
// partition solver k_thomas_x and its two-warp variant k_thomas_x2 (the TMA
// kernel is etc_zsolve.cuh).  Included by etc_b200.cu (one translation unit).
#pragma once

// ---- per-mode tridiagonal solve along z (preconditioner.py:215-250).
// Column (j', i') has diagonal z_diag[k] + shift(j',i') and off-diagonals
// -kz_ref.  A group of Q lanes owns one column; lane q owns rows
// [qL, qL+L): rows 0..L-2 are its interior block, row L-1 a separator (the
// last lane has none).  Local block elimination (reciprocal pivots kept in
// registers, values in shared memory) + spike end values give a tridiagonal
// Schur system on the Q-1 separators, solved by parallel cyclic reduction
// over warp shuffles; one more sweep applies the separator coupling.  PCG mode
// also accumulates r.z = 4/(nx ny) sum a_x a_y R^ Z^ from the untouched
// right-hand side tile F and the solution tile X (Parseval, reference
// test_transforms.py:160-176) and finalises beta (krylov.py:85-90).
// branch-free reciprocal of a positive normal pivot: MUFU seed + two Newton
// steps (~1 ulp; the z-solve is not bit-matched to the reference anyway, and
// the IEEE slow-path branch of __drcp_rn costs more than the whole row update)
__device__ __forceinline__ double rcp_fast(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ float rcp_fast(float d) { return __frcp_rn(d); }

// column stride of the z-solve tiles (doubles).  Lane chunks of L values are
// padded to L+1 (odd: conflict-free per-lane sweeps).  For the coalesced tile
// load (a warp covers 32/C rows x C columns) the stride is chosen so the
// lanes of a warp hit each 8-byte bank pair at most twice: = 4 mod 16 when
// C = 8 (4 rows x 8 columns), odd otherwise.
constexpr int thomas_cs(int L, int Q) {
  return (256 / Q == 8) ? ((Q * (L + 1) + 15) / 16) * 16 + 4 : ((Q * (L + 1)) | 1);
}

template <int L, int Q>
__global__ void __launch_bounds__(256, 3) k_thomas(Geom g, double* t, const double* __restrict__ wx,
                                                   const double* __restrict__ wy, double zd0, double zdi, double zdl,
                                                   double kxr, double kyr, double off, Ctl* ctl, double* partials,
                                                   unsigned* counter, int pcg) {
  if (pcg && ctl->done) return;
  extern __shared__ double tile[];
  constexpr int C = 256 / Q;
  constexpr int cs = thomas_cs(L, Q);
  double* F = tile;
  double* X = tile + C * cs;
  const long long plane = g.plane;
  const int nz = g.nz;
  const int rows = Q * L;
  const long long ntiles = (plane + C - 1) / C;
  const int c = threadIdx.x / Q, q = threadIdx.x % Q;
  // z-chain diagonal (TridiagFactors.z_diag, preconditioner.py:192-199)
  auto zdiag = [&](int k) -> double { return k == 0 ? zd0 : (k == nz - 1 ? zdl : zdi); };
  const bool has_sep = q < Q - 1;
  const int nb = has_sep ? L - 1 : L;
  const int k0 = q * L;
  double dot = 0.0;
  auto lo = [&](int k) -> double { return (k >= 1 && k < nz) ? off : 0.0; };
  auto up = [&](int k) -> double { return (k + 1 < nz) ? off : 0.0; };
  for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const long long c0 = tl * C;
    for (int e = threadIdx.x; e < rows * C; e += blockDim.x) {
      const int k = e / C, cc = e - k * C;
      const long long col = c0 + cc;
      F[cc * cs + (k / L) * (L + 1) + (k % L)] = (k < nz && col < plane) ? t[(long long)k * plane + col] : 0.0;
    }
    __syncthreads();
    const long long col = c0 + c;
    const bool valid = col < plane;
    const int ip = valid ? (int)(col % g.nx) : 0;
    const int jp = valid ? (int)(col / g.nx) + g.jofs : 0;  // global mode row (z-pencils)
    const double shift = __dadd_rn(__dmul_rn(wx[ip], kxr), __dmul_rn(wy[jp], kyr));
    const double* myf = F + c * cs + q * (L + 1);
    double* my = X + c * cs + q * (L + 1);
    double rcp[L];
    // local forward elimination (no coupling to the row above the block)
    double xp = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) {
      if (i < nb) {
        const int k = k0 + i;
        const double b = k < nz ? zdiag(k) + shift : 1.0;
        if (i == 0) {
          rcp[0] = rcp_fast(b);
          xp = myf[0] * rcp[0];
        } else {
          const double lk = lo(k);
          rcp[i] = rcp_fast(b - lk * (up(k - 1) * rcp[i - 1]));
          xp = (myf[i] - lk * xp) * rcp[i];
        }
        my[i] = xp;
      } else {
        rcp[i] = 0.0;
      }
    }
    // end values of g = T^-1 f, U = T^-1 e_first, V = T^-1 e_last
    const double g_last = xp;
    const double v_last = has_sep ? rcp[L - 2] : rcp[L - 1];
    double gacc = g_last, mu = 1.0, vprod = v_last;
#pragma unroll
    for (int i = L - 2; i >= 0; --i) {
      if (i < nb - 1) {
        const int k = k0 + i;
        const double cpi = up(k) * rcp[i];
        gacc = my[i] - cpi * gacc;
        mu = 1.0 + cpi * lo(k + 1) * rcp[i + 1] * mu;
        vprod = -cpi * vprod;
      }
    }
    const double g_first = gacc, u_first = rcp[0] * mu, v_first = vprod;
    const double lo_first = lo(k0), up_last = up(k0 + nb - 1);
    // separator equations (Schur complement on the separators)
    const double n_gf = __shfl_down_sync(0xffffffffu, g_first, 1, Q);
    const double n_uf = __shfl_down_sync(0xffffffffu, u_first, 1, Q);
    const double n_vf = __shfl_down_sync(0xffffffffu, v_first, 1, Q);
    const double n_ul = __shfl_down_sync(0xffffffffu, up_last, 1, Q);
    double a = 0.0, b = 1.0, cc = 0.0, d = 0.0;
    if (has_sep) {
      const int ks = k0 + L - 1;
      const double los = lo(ks), ups = up(ks);
      const double bs = ks < nz ? zdiag(ks) + shift : 1.0;
      a = -los * lo_first * v_first;
      b = bs - los * up_last * v_last - ups * ups * n_uf;
      cc = -ups * n_ul * n_vf;
      d = myf[L - 1] - los * g_last - ups * n_gf;
    }
    for (int dd = 1; dd < Q; dd <<= 1) {
      double am = __shfl_up_sync(0xffffffffu, a, dd, Q), bm = __shfl_up_sync(0xffffffffu, b, dd, Q);
      double cm = __shfl_up_sync(0xffffffffu, cc, dd, Q), dm = __shfl_up_sync(0xffffffffu, d, dd, Q);
      double ap = __shfl_down_sync(0xffffffffu, a, dd, Q), bp = __shfl_down_sync(0xffffffffu, b, dd, Q);
      double cp = __shfl_down_sync(0xffffffffu, cc, dd, Q), dp = __shfl_down_sync(0xffffffffu, d, dd, Q);
      if (q < dd) { am = 0.0; bm = 1.0; cm = 0.0; dm = 0.0; }
      if (q + dd >= Q) { ap = 0.0; bp = 1.0; cp = 0.0; dp = 0.0; }
      const double k1 = a * rcp_fast(bm), k2 = cc * rcp_fast(bp);
      const double na = -am * k1, nc = -cp * k2;
      const double nbv = b - cm * k1 - ap * k2, nd = d - dm * k1 - dp * k2;
      a = na; b = nbv; cc = nc; d = nd;
    }
    const double S = d / b;
    double Sm = __shfl_up_sync(0xffffffffu, S, 1, Q);
    if (q == 0) Sm = 0.0;
    // couple the block to its separators: forward sweep of the end
    // corrections, then the backward substitution
    const double eta0 = -lo_first * Sm;
    const double etaL = has_sep ? -up_last * S : 0.0;
    double h = (eta0 + (nb == 1 ? etaL : 0.0)) * rcp[0];
    my[0] += h;
#pragma unroll
    for (int i = 1; i < L; ++i) {
      if (i < nb) {
        h = ((i == nb - 1 ? etaL : 0.0) - lo(k0 + i) * h) * rcp[i];
        my[i] += h;
      }
    }
    double xn = my[nb - 1];
#pragma unroll
    for (int i = L - 2; i >= 0; --i) {
      if (i < nb - 1) {
        xn = my[i] - up(k0 + i) * rcp[i] * xn;
        my[i] = xn;
      }
    }
    if (has_sep) my[L - 1] = S;
    if (pcg && valid) {
      double s = 0.0;
      for (int i = 0; i < L; ++i) s = fma(myf[i], my[i], s);
      dot = fma((ip == 0 ? 0.5 : 1.0) * (jp == 0 ? 0.5 : 1.0), s, dot);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * C; e += blockDim.x) {
      const int k = e / C, c2 = e - k * C;
      const long long cl = c0 + c2;
      if (k < nz && cl < plane) t[(long long)k * plane + cl] = X[c2 * cs + (k / L) * (L + 1) + (k % L)];
    }
    __syncthreads();
  }
  if (pcg) {
    double v[1] = {dot};
    const double scale = 4.0 / ((double)g.nx * (double)g.nyg);
    grid_sum_finalize<1>(v, partials, counter, [&](double (&tt)[1]) {
      if (ctl->dist)
        ctl->xbuf[4] = tt[0];
      else
        fin_thomas(ctl, tt[0] * scale);
    });
  }
}

// ---- exact-fit z-solve (nz == 32*L, the case of every power-of-two grid):
// the same partition algorithm as k_thomas with every in-block coupling the
// constant -kz_ref and only two special diagonals (z_diag[0] in lane 0's first
// row, z_diag[nz-1] in lane 31's last row), so the sweeps carry no per-row
// selects.  One warp per column, 8 columns per CTA.

template <int L, int C = 8>
__global__ void __launch_bounds__(32 * C, 16 / C) k_thomas_x(Geom g, double* t, const double* __restrict__ wx,
                                                     const double* __restrict__ wy, double zd0, double zdi,
                                                     double zdl, double kxr, double kyr, double off, Ctl* ctl,
                                                     double* partials, unsigned* counter, int pcg,
                                                     double* const* zpeers, int me, int nranks) {
  if (pcg && ctl->done) return;
  extern __shared__ double tile[];
  constexpr int Q = 32, NT = 32 * C;
  constexpr int cs = thomas_cs(L, Q);
  constexpr int rows = Q * L;
  double* F = tile;
  double* X = tile + C * cs;
  const long long plane = g.plane;
  const long long ntiles = (plane + C - 1) / C;
  const int c = threadIdx.x >> 5, q = threadIdx.x & 31;
  const bool last = (q == Q - 1);
  const double off2 = off * off;
  double dot = 0.0;
  // the next tile's loads are issued before the current tile's solve and land
  // in registers while it computes (software pipelining across tiles)
  constexpr int PER = rows * C / NT;  // elements per thread per tile
  double pre[PER];
  auto fetch = [&](long long tl) {
    const long long c0 = tl * C;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int e = threadIdx.x + m * NT;
      const int k = e / C, cc = e % C;
      const long long col = c0 + cc;
      pre[m] = (tl < ntiles && col < plane) ? t[(long long)k * plane + col] : 0.0;
    }
  };
  fetch(blockIdx.x);
  for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const long long c0 = tl * C;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int e = threadIdx.x + m * NT;
      const int k = e / C, cc = e % C;
      F[cc * cs + (k / L) * (L + 1) + (k % L)] = pre[m];
    }
    __syncthreads();
    fetch(tl + gridDim.x);
    const long long col = c0 + c;
    const bool valid = col < plane;
    const int ip = valid ? (int)(col % g.nx) : 0;
    const int jp = valid ? (int)(col / g.nx) + g.jofs : 0;  // global mode row (z-pencils)
    const double shift = __dadd_rn(__dmul_rn(wx[ip], kxr), __dmul_rn(wy[jp], kyr));
    const double B = zdi + shift;
    const double b0 = (q == 0 ? zd0 : zdi) + shift;
    const double bl = (last ? zdl : zdi) + shift;  // row L-1 of lane 31 (its own last block row)
    const double* myf = F + c * cs + q * (L + 1);
    double* rcp = X + c * cs + q * (L + 1);  // reciprocal pivots in shared memory, values in registers
    double my[L];
    // local forward elimination; rows 0..L-2 for every lane, row L-1 only in lane 31
    double xp;
    rcp[0] = rcp_fast(L == 1 ? bl : b0);
    xp = myf[0] * rcp[0];
    my[0] = xp;
#pragma unroll
    for (int i = 1; i < L - 1; ++i) {
      rcp[i] = rcp_fast(B - off2 * rcp[i - 1]);
      xp = (myf[i] - off * xp) * rcp[i];
      my[i] = xp;
    }
    if (L > 1) {
      rcp[L - 1] = last ? rcp_fast(bl - off2 * rcp[L - 2]) : 0.0;
      if (last) {
        xp = (myf[L - 1] - off * xp) * rcp[L - 1];
        my[L - 1] = xp;
      }
    }
    // spike end values; nb = L-1 (separator lanes) or L (lane 31)
    const double g_last = xp;
    const double v_last = last ? rcp[L - 1] : (L > 1 ? rcp[L - 2] : rcp[0]);
    double gacc = g_last, mu = 1.0, vprod = v_last;
    if (L > 1 && last) {  // row L-2 against row L-1 (lane 31 only)
      const double cpi = off * rcp[L - 2];
      gacc = my[L - 2] - cpi * gacc;
      mu = 1.0 + cpi * off * rcp[L - 1] * mu;
      vprod = -cpi * vprod;
    }
#pragma unroll
    for (int i = L - 3; i >= 0; --i) {
      const double cpi = off * rcp[i];
      gacc = my[i] - cpi * gacc;
      mu = 1.0 + cpi * off * rcp[i + 1] * mu;
      vprod = -cpi * vprod;
    }
    const double g_first = gacc, u_first = rcp[0] * mu, v_first = vprod;
    const double lo_first = (q == 0) ? 0.0 : off, up_last = last ? 0.0 : off;
    const double n_gf = __shfl_down_sync(0xffffffffu, g_first, 1);
    const double n_uf = __shfl_down_sync(0xffffffffu, u_first, 1);
    const double n_vf = __shfl_down_sync(0xffffffffu, v_first, 1);
    const double n_ul = __shfl_down_sync(0xffffffffu, up_last, 1);
    double a = 0.0, b = 1.0, cc = 0.0, d = 0.0;
    if (!last) {  // separator row qL+L-1: interior row, couplings off on both sides
      a = -off * lo_first * v_first;
      b = B - off * up_last * v_last - off2 * n_uf;
      cc = -off * n_ul * n_vf;
      d = myf[L - 1] - off * g_last - off * n_gf;
    }
#pragma unroll
    for (int dd = 1; dd < Q; dd <<= 1) {
      double am = __shfl_up_sync(0xffffffffu, a, dd), bm = __shfl_up_sync(0xffffffffu, b, dd);
      double cm = __shfl_up_sync(0xffffffffu, cc, dd), dm = __shfl_up_sync(0xffffffffu, d, dd);
      double ap = __shfl_down_sync(0xffffffffu, a, dd), bp = __shfl_down_sync(0xffffffffu, b, dd);
      double cp = __shfl_down_sync(0xffffffffu, cc, dd), dp = __shfl_down_sync(0xffffffffu, d, dd);
      if (q < dd) { am = 0.0; bm = 1.0; cm = 0.0; dm = 0.0; }
      if (q + dd >= Q) { ap = 0.0; bp = 1.0; cp = 0.0; dp = 0.0; }
      const double k1 = a * rcp_fast(bm), k2 = cc * rcp_fast(bp);
      const double na = -am * k1, nc = -cp * k2;
      const double nbv = b - cm * k1 - ap * k2, nd = d - dm * k1 - dp * k2;
      a = na; b = nbv; cc = nc; d = nd;
    }
    const double S = d / b;
    double Sm = __shfl_up_sync(0xffffffffu, S, 1);
    if (q == 0) Sm = 0.0;
    // separator coupling: forward sweep of the end corrections, then back substitution
    const double eta0 = -lo_first * Sm;
    const double etaL = last ? 0.0 : -off * S;
    if (L == 1) {
      if (last) my[0] += eta0 * rcp[0];
    } else {
      double h = eta0 * rcp[0];
      my[0] += h;
#pragma unroll
      for (int i = 1; i < L - 1; ++i) {
        h = ((i == L - 2 && !last ? etaL : 0.0) - off * h) * rcp[i];
        my[i] += h;
      }
      if (L == 2 && !last) my[0] += etaL * rcp[0];  // single-row block: both ends hit row 0
      if (last) {
        h = (0.0 - off * h) * rcp[L - 1];
        my[L - 1] += h;
      }
      double xn = last ? my[L - 1] : my[L - 2];
      if (last) {
        xn = my[L - 2] - off * rcp[L - 2] * xn;
        my[L - 2] = xn;
      }
#pragma unroll
      for (int i = L - 3; i >= 0; --i) {
        xn = my[i] - off * rcp[i] * xn;
        my[i] = xn;
      }
    }
    if (!last) my[L - 1] = S;
    __syncwarp();
    if (pcg && valid) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < L; ++i) s = fma(myf[i], my[i], s);
      dot = fma((ip == 0 ? 0.5 : 1.0) * (jp == 0 ? 0.5 : 1.0), s, dot);
    }
    {
      double* xo = X + c * cs + q * (L + 1);  // the pivots are dead: the values take their place
#pragma unroll
      for (int i = 0; i < L; ++i) xo[i] = my[i];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * C; e += NT) {
      const int k = e / C, c2 = e % C;
      const long long cl = c0 + c2;
      if (cl < plane) {
        const double v = X[c2 * cs + (k / L) * (L + 1) + (k % L)];
        if (zpeers) {  // row k belongs to rank k / nzl: its return buffer, block of this rank
          const int nzl = rows / nranks, s = k / nzl;
          zpeers[s][(long long)(me * nzl + k - s * nzl) * plane + cl] = v;
        } else {
          t[(long long)k * plane + cl] = v;
        }
      }
    }
    __syncthreads();
  }
  if (zpeers) __threadfence_system();
  if (pcg) {
    double v[1] = {dot};
    const double scale = 4.0 / ((double)g.nx * (double)g.nyg);
    grid_sum_finalize<1>(v, partials, counter, [&](double (&tt)[1]) {
      if (ctl->dist)
        ctl->xbuf[4] = tt[0];
      else
        fin_thomas(ctl, tt[0] * scale);
    });
  }
}

// nz = 64 L (1024 for L = 16): two warps per column, so every lane keeps the
// nz = 512 kernel's 16 rows; the separator system has 63 unknowns and its PCR
// levels exchange through shared memory instead of warp shuffles.
template <int L, int C>
__global__ void __launch_bounds__(64 * C, 1) k_thomas_x2(Geom g, double* t, const double* __restrict__ wx,
                                                     const double* __restrict__ wy, double zd0, double zdi,
                                                     double zdl, double kxr, double kyr, double off, Ctl* ctl,
                                                     double* partials, unsigned* counter, int pcg) {
  if (pcg && ctl->done) return;
  extern __shared__ double tile[];
  constexpr int Q = 64, NT = 64 * C;  // two warps per column, C columns per tile
  constexpr int cs = thomas_cs(L, Q);
  constexpr int rows = Q * L;
  double* F = tile;
  double* X = tile + C * cs;
  const long long plane = g.plane;
  const long long ntiles = (plane + C - 1) / C;
  const int c = threadIdx.x >> 6, q = threadIdx.x & 63;
  // lane exchange across the column's two warps (neighbours, PCR levels)
  __shared__ double xs[4][C][Q];
  const bool last = (q == Q - 1);
  const double off2 = off * off;
  double dot = 0.0;
  // the next tile's loads are issued before the current tile's solve and land
  // in registers while it computes (software pipelining across tiles)
  constexpr int PER = rows * C / NT;  // elements per thread per tile
  double pre[PER];
  auto fetch = [&](long long tl) {
    const long long c0 = tl * C;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int e = threadIdx.x + m * NT;
      const int k = e / C, cc = e % C;
      const long long col = c0 + cc;
      pre[m] = (tl < ntiles && col < plane) ? t[(long long)k * plane + col] : 0.0;
    }
  };
  fetch(blockIdx.x);
  for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const long long c0 = tl * C;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int e = threadIdx.x + m * NT;
      const int k = e / C, cc = e % C;
      F[cc * cs + (k / L) * (L + 1) + (k % L)] = pre[m];
    }
    __syncthreads();
    fetch(tl + gridDim.x);
    const long long col = c0 + c;
    const bool valid = col < plane;
    const int ip = valid ? (int)(col % g.nx) : 0;
    const int jp = valid ? (int)(col / g.nx) + g.jofs : 0;  // global mode row (z-pencils)
    const double shift = __dadd_rn(__dmul_rn(wx[ip], kxr), __dmul_rn(wy[jp], kyr));
    const double B = zdi + shift;
    const double b0 = (q == 0 ? zd0 : zdi) + shift;
    const double bl = (last ? zdl : zdi) + shift;  // row L-1 of lane 31 (its own last block row)
    const double* myf = F + c * cs + q * (L + 1);
    double* my = X + c * cs + q * (L + 1);
    double rcp[L];
    // local forward elimination; rows 0..L-2 for every lane, row L-1 only in lane 31
    double xp;
    rcp[0] = rcp_fast(L == 1 ? bl : b0);
    xp = myf[0] * rcp[0];
    my[0] = xp;
#pragma unroll
    for (int i = 1; i < L - 1; ++i) {
      rcp[i] = rcp_fast(B - off2 * rcp[i - 1]);
      xp = (myf[i] - off * xp) * rcp[i];
      my[i] = xp;
    }
    if (L > 1) {
      rcp[L - 1] = last ? rcp_fast(bl - off2 * rcp[L - 2]) : 0.0;
      if (last) {
        xp = (myf[L - 1] - off * xp) * rcp[L - 1];
        my[L - 1] = xp;
      }
    }
    // spike end values; nb = L-1 (separator lanes) or L (lane 31)
    const double g_last = xp;
    const double v_last = last ? rcp[L - 1] : (L > 1 ? rcp[L - 2] : rcp[0]);
    double gacc = g_last, mu = 1.0, vprod = v_last;
    if (L > 1 && last) {  // row L-2 against row L-1 (lane 31 only)
      const double cpi = off * rcp[L - 2];
      gacc = my[L - 2] - cpi * gacc;
      mu = 1.0 + cpi * off * rcp[L - 1] * mu;
      vprod = -cpi * vprod;
    }
#pragma unroll
    for (int i = L - 3; i >= 0; --i) {
      const double cpi = off * rcp[i];
      gacc = my[i] - cpi * gacc;
      mu = 1.0 + cpi * off * rcp[i + 1] * mu;
      vprod = -cpi * vprod;
    }
    const double g_first = gacc, u_first = rcp[0] * mu, v_first = vprod;
    const double lo_first = (q == 0) ? 0.0 : off, up_last = last ? 0.0 : off;
    xs[0][c][q] = g_first;
    xs[1][c][q] = u_first;
    xs[2][c][q] = v_first;
    xs[3][c][q] = up_last;
    __syncthreads();
    const int qn = q + 1 < Q ? q + 1 : q;
    const double n_gf = xs[0][c][qn], n_uf = xs[1][c][qn], n_vf = xs[2][c][qn], n_ul = xs[3][c][qn];
    __syncthreads();
    double a = 0.0, b = 1.0, cc = 0.0, d = 0.0;
    if (!last) {  // separator row qL+L-1: interior row, couplings off on both sides
      a = -off * lo_first * v_first;
      b = B - off * up_last * v_last - off2 * n_uf;
      cc = -off * n_ul * n_vf;
      d = myf[L - 1] - off * g_last - off * n_gf;
    }
#pragma unroll
    for (int dd = 1; dd < Q; dd <<= 1) {
      xs[0][c][q] = a;
      xs[1][c][q] = b;
      xs[2][c][q] = cc;
      xs[3][c][q] = d;
      __syncthreads();
      const int qm = q >= dd ? q - dd : q, qp = q + dd < Q ? q + dd : q;
      double am = xs[0][c][qm], bm = xs[1][c][qm], cm = xs[2][c][qm], dm = xs[3][c][qm];
      double ap = xs[0][c][qp], bp = xs[1][c][qp], cp = xs[2][c][qp], dp = xs[3][c][qp];
      __syncthreads();
      if (q < dd) { am = 0.0; bm = 1.0; cm = 0.0; dm = 0.0; }
      if (q + dd >= Q) { ap = 0.0; bp = 1.0; cp = 0.0; dp = 0.0; }
      const double k1 = a * rcp_fast(bm), k2 = cc * rcp_fast(bp);
      const double na = -am * k1, nc = -cp * k2;
      const double nbv = b - cm * k1 - ap * k2, nd = d - dm * k1 - dp * k2;
      a = na; b = nbv; cc = nc; d = nd;
    }
    const double S = d / b;
    xs[0][c][q] = S;
    __syncthreads();
    double Sm = q ? xs[0][c][q - 1] : 0.0;
    // separator coupling: forward sweep of the end corrections, then back substitution
    const double eta0 = -lo_first * Sm;
    const double etaL = last ? 0.0 : -off * S;
    if (L == 1) {
      if (last) my[0] += eta0 * rcp[0];
    } else {
      double h = eta0 * rcp[0];
      my[0] += h;
#pragma unroll
      for (int i = 1; i < L - 1; ++i) {
        h = ((i == L - 2 && !last ? etaL : 0.0) - off * h) * rcp[i];
        my[i] += h;
      }
      if (L == 2 && !last) my[0] += etaL * rcp[0];  // single-row block: both ends hit row 0
      if (last) {
        h = (0.0 - off * h) * rcp[L - 1];
        my[L - 1] += h;
      }
      double xn = my[last ? L - 1 : L - 2];
      if (last) {
        xn = my[L - 2] - off * rcp[L - 2] * xn;
        my[L - 2] = xn;
      }
#pragma unroll
      for (int i = L - 3; i >= 0; --i) {
        xn = my[i] - off * rcp[i] * xn;
        my[i] = xn;
      }
    }
    if (!last) my[L - 1] = S;
    if (pcg && valid) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < L; ++i) s = fma(myf[i], my[i], s);
      dot = fma((ip == 0 ? 0.5 : 1.0) * (jp == 0 ? 0.5 : 1.0), s, dot);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * C; e += NT) {
      const int k = e / C, c2 = e % C;
      const long long cl = c0 + c2;
      if (cl < plane) t[(long long)k * plane + cl] = X[c2 * cs + (k / L) * (L + 1) + (k % L)];
    }
    __syncthreads();
  }
  if (pcg) {
    double v[1] = {dot};
    const double scale = 4.0 / ((double)g.nx * (double)g.nyg);
    grid_sum_finalize<1>(v, partials, counter, [&](double (&tt)[1]) {
      if (ctl->dist)
        ctl->xbuf[4] = tt[0];
      else
        fin_thomas(ctl, tt[0] * scale);
    });
  }
}
