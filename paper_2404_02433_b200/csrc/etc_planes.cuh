// etc_planes.cuh — the 2-D DCT-II / DCT-III plane transforms of the FCT
// preconditioner (FctPlan.forward / backward, reference
// /root/reference/pkg/src/etchomo/transforms.py:83-133): runtime-size and
// compile-time line FFTs, the paired-item row / column chunks, the cluster
// kernels (k_fwd_c2 / k_inv_c2) and the decoupled persistent kernels
// (k_fwd_q / k_inv_q).  Included by etc_b200.cu (one translation unit).
#pragma once

// ---- plane transforms as thread-block clusters.  A cluster of CL CTAs owns
// one z-plane at a time: phase X transforms its share of the rows (lines along
// x), a cluster barrier (release/acquire) publishes them, phase Y transforms
// its share of the columns (lines along y) reading the phase-X output back
// through L2 (__ldcg).  The intermediate is overwritten in place by phase Y, so
// DRAM sees one read and one write per element per 2-D transform.
// Twiddles live in shared memory.

template <class T>
struct PlaneTabsT {
  const C2<T> *twx, *ex, *twy, *ey;  // global copies
};
using PlaneTabs = PlaneTabsT<double>;

struct SmemTabs {
  double2 *twx, *ex, *twy, *ey, *A, *B;
};

__device__ __forceinline__ SmemTabs carve(double2* sm, const Geom& g, const PlaneTabs& T, int px, int py) {
  SmemTabs s;
  const int nx = g.nx, ny = g.ny;
  s.twx = sm;
  s.ex = s.twx + nx;
  s.twy = s.ex + nx;
  s.ey = s.twy + ny;
  s.A = s.ey + ny;
  const int buf = max(px * nx, py * (ny + 1));
  s.B = s.A + buf;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) {
    s.twx[i] = T.twx[i];
    s.ex[i] = T.ex[i];
  }
  for (int i = threadIdx.x; i < ny; i += blockDim.x) {
    s.twy[i] = T.twy[i];
    s.ey[i] = T.ey[i];
  }
  __syncthreads();
  return s;
}

// DCT-II recombination of pair-packed spectra: line (2f + odd) at index kk
__device__ __forceinline__ double dct2_out(const double2* Z, int nn, int kk, int odd, double2 E) {
  const double2 a = Z[kk];
  const double2 b = Z[kk ? nn - kk : 0];
  return odd ? 0.5 * (E.x * (a.y + b.y) - E.y * (a.x - b.x)) : 0.5 * (E.x * (a.x + b.x) + E.y * (a.y - b.y));
}

// DCT-III pre-twiddle: V[k] = e^{+i pi k/2N} (C[k] - i C[N-k]) for both packed
// lines, Z = V1 + i V2
__device__ __forceinline__ double2 dct3_pre(const double2* A, int nn, int kk, double2 E) {
  const double2 a = A[kk];
  const double2 b = kk ? A[nn - kk] : make_double2(0.0, 0.0);
  const double v1r = E.x * a.x + E.y * b.x, v1i = E.y * a.x - E.x * b.x;
  const double v2r = E.x * a.y + E.y * b.y, v2i = E.y * a.y - E.x * b.y;
  return make_double2(v1r - v2i, v1i + v2r);
}

// Forward 2-D DCT-II of every z-plane.  MODE 0: src -> dst.  MODE 1: r = b:
// transform plus ||b|| (krylov.py:57-68).  MODE 2: r -= alpha q, ||r||
// (krylov.py:76-84), transform of r written over q (dst == q).
template <int MODE>
__global__ void __launch_bounds__(256) k_fwd(Geom g, int px, int py, const double* src, double* dst, double* r,
                                             const double* q, Ctl* ctl, double* partials, unsigned* counter,
                                             PlaneTabs T, double* hist) {
  if (MODE != 0 && ctl->done) return;
  extern __shared__ double2 smem_c[];
  const SmemTabs S = carve(smem_c, g, T, px, py);
  const int nx = g.nx, ny = g.ny;
  const unsigned crank = cluster_ctarank(), csize = cluster_nctarank();
  const unsigned cid = cluster_id_x(), ncl = ncluster_x();
  const double alpha = (MODE == 2) ? ctl->alpha : 0.0;
  const int rows_per = (ny + csize - 1) / csize;
  const int jr0 = min(ny, (int)crank * rows_per), jr1 = min(ny, jr0 + rows_per);
  const int cols_per = (nx + csize - 1) / csize;
  const int cc0 = min(nx, (int)crank * cols_per), cc1 = min(nx, cc0 + cols_per);
  const int pitchy = ny + 1;
  double rr = 0.0;
  for (long long kz = cid; kz < g.nz; kz += ncl) {
    const long long pb = kz * g.plane;
    // ---- phase X: rows [jr0, jr1)
    for (int j0 = jr0; j0 < jr1; j0 += 2 * px) {
      const int nrow = min(2 * px, jr1 - j0);
      const int tile = 2 * px * nx;
      for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        const int lr = e / nx, i = e - lr * nx;
        double v = 0.0;
        if (lr < nrow) {
          const long long idx = pb + (long long)(j0 + lr) * nx + i;
          if (MODE == 2) {
            v = __dsub_rn(r[idx], __dmul_rn(alpha, q[idx]));
            r[idx] = v;
            rr = fma(v, v, rr);
          } else {
            v = src[idx];
            if (MODE == 1) rr = fma(v, v, rr);
          }
        }
        reinterpret_cast<double*>(&S.A[(lr >> 1) * nx + makhoul_pos(i, nx)])[lr & 1] = v;
      }
      __syncthreads();
      const double2* Z = fft_lines(S.A, S.B, px, nx, nx, S.twx, -1.0);
      for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        const int lr = e / nx, kk = e - lr * nx;
        if (lr < nrow) dst[pb + (long long)(j0 + lr) * nx + kk] = dct2_out(Z + (lr >> 1) * nx, nx, kk, lr & 1, S.ex[kk]);
      }
      __syncthreads();
    }
    cluster_barrier();
    // ---- phase Y: columns [cc0, cc1), lines along y read back through L2
    for (int c0 = cc0; c0 < cc1; c0 += 2 * py) {
      const int ncol = min(2 * py, cc1 - c0);
      const int w2 = 2 * py;
      for (int e = threadIdx.x; e < ny * w2; e += blockDim.x) {
        const int j = e / w2, c = e - j * w2;
        const double v = c < ncol ? __ldcg(dst + pb + (long long)j * nx + c0 + c) : 0.0;
        reinterpret_cast<double*>(&S.A[(c >> 1) * pitchy + makhoul_pos(j, ny)])[c & 1] = v;
      }
      __syncthreads();
      const double2* Z = fft_lines(S.A, S.B, py, ny, pitchy, S.twy, -1.0);
      for (int e = threadIdx.x; e < ny * w2; e += blockDim.x) {
        const int j = e / w2, c = e - j * w2;
        if (c < ncol) dst[pb + (long long)j * nx + c0 + c] = dct2_out(Z + (c >> 1) * pitchy, ny, j, c & 1, S.ey[j]);
      }
      __syncthreads();
    }
  }
  if (MODE != 0) {
    double v[1] = {rr};
    grid_sum_finalize<1>(v, partials, counter, [&](double (&t)[1]) {
      if (ctl->dist)
        ctl->xbuf[3] = t[0];
      else if (MODE == 1)
        fin_normb(ctl, t[0], hist);
      else
        fin_update(ctl, t[0], hist);
    });
  }
}

// Inverse 2-D transform (DCT-III with the 2/N weights, transforms.py:108-133):
// phase Y reads src (spectral) and writes dst, phase X finishes dst in place.
template <bool PCG>
__global__ void __launch_bounds__(256) k_inv(Geom g, int px, int py, const double* src, double* dst, const Ctl* ctl,
                                             PlaneTabs T) {
  if (PCG && ctl->done) return;
  extern __shared__ double2 smem_c[];
  const SmemTabs S = carve(smem_c, g, T, px, py);
  const int nx = g.nx, ny = g.ny;
  const unsigned crank = cluster_ctarank(), csize = cluster_nctarank();
  const unsigned cid = cluster_id_x(), ncl = ncluster_x();
  const int rows_per = (ny + csize - 1) / csize;
  const int jr0 = min(ny, (int)crank * rows_per), jr1 = min(ny, jr0 + rows_per);
  const int cols_per = (nx + csize - 1) / csize;
  const int cc0 = min(nx, (int)crank * cols_per), cc1 = min(nx, cc0 + cols_per);
  const int pitchy = ny + 1;
  const bool p2x = (nx & (nx - 1)) == 0, p2y = (ny & (ny - 1)) == 0;
  const double ivx = 1.0 / nx, ivy = 1.0 / ny;
  for (long long kz = cid; kz < g.nz; kz += ncl) {
    const long long pb = kz * g.plane;
    // ---- phase Y
    for (int c0 = cc0; c0 < cc1; c0 += 2 * py) {
      const int ncol = min(2 * py, cc1 - c0);
      const int w2 = 2 * py;
      for (int e = threadIdx.x; e < ny * w2; e += blockDim.x) {
        const int j = e / w2, c = e - j * w2;
        const double v = c < ncol ? src[pb + (long long)j * nx + c0 + c] : 0.0;
        reinterpret_cast<double*>(&S.A[(c >> 1) * pitchy + j])[c & 1] = v;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < py * ny; e += blockDim.x) {
        const int f = e / ny, kk = e - f * ny;
        S.B[f * pitchy + kk] = dct3_pre(S.A + f * pitchy, ny, kk, S.ey[kk]);
      }
      __syncthreads();
      const double2* Z = fft_lines(S.B, S.A, py, ny, pitchy, S.twy, 1.0);
      for (int e = threadIdx.x; e < ny * w2; e += blockDim.x) {
        const int j = e / w2, c = e - j * w2;
        if (c >= ncol) continue;
        const double2 zz = Z[(c >> 1) * pitchy + makhoul_pos(j, ny)];
        const double v = (c & 1) ? zz.y : zz.x;
        dst[pb + (long long)j * nx + c0 + c] = p2y ? v * ivy : v / ny;
      }
      __syncthreads();
    }
    cluster_barrier();
    // ---- phase X
    for (int j0 = jr0; j0 < jr1; j0 += 2 * px) {
      const int nrow = min(2 * px, jr1 - j0);
      const int tile = 2 * px * nx;
      for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        const int lr = e / nx, i = e - lr * nx;
        const double v = lr < nrow ? __ldcg(dst + pb + (long long)(j0 + lr) * nx + i) : 0.0;
        reinterpret_cast<double*>(&S.A[(lr >> 1) * nx + i])[lr & 1] = v;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < px * nx; e += blockDim.x) {
        const int f = e / nx, kk = e - f * nx;
        S.B[f * nx + kk] = dct3_pre(S.A + f * nx, nx, kk, S.ex[kk]);
      }
      __syncthreads();
      const double2* Z = fft_lines(S.B, S.A, px, nx, nx, S.twx, 1.0);
      for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        const int lr = e / nx, i = e - lr * nx;
        if (lr >= nrow) continue;
        const double2 zz = Z[(lr >> 1) * nx + makhoul_pos(i, nx)];
        const double v = (lr & 1) ? zz.y : zz.x;
        dst[pb + (long long)(j0 + lr) * nx + i] = p2x ? v * ivx : v / nx;
      }
      __syncthreads();
    }
  }
}

// ===========================================================================
// compile-time specialised plane transforms for square power-of-two planes
// (nx = ny = N, the canonical shape of every cubic RVE).  256 threads; a
// chunk is LN = 2048/N complex lines (= 2*LN real lines, pair-packed).
// Radix-8 Stockham with the first pass fed straight from global memory (the
// Makhoul even/odd gather folded into the load addresses) and the last pass
// drained straight to registers; only the middle passes go through the
// padded in-place shared buffer.  Twiddle powers w^r are formed in registers
// from one table read.  All index math is shifts.
// ===========================================================================
__device__ __forceinline__ int padi(int i) { return i + (i >> 3); }
// line pitch of the padded buffer, offset so that the lines a quarter-warp
// touches in the column phase (mapping f = tid % LN: 8/LN rows x LN lines, or
// 8 lines) fall on distinct 16-byte bank groups
template <int N>
constexpr int ct_pitch() {
  return N + N / 8 + ((2048 / N) >= 8 ? 1 : 8 / (2048 / N));
}

// twiddle powers t^1..t^(R-1) applied to v[1..R-1] (s < 0: forward)
template <int R>
__device__ __forceinline__ void twiddle_pow(double2 (&v)[R], double2 t1, double s) {
  if (s > 0) t1.y = -t1.y;
  double2 t = t1;
#pragma unroll
  for (int r = 1; r < R; ++r) {
    v[r] = cmul(v[r], t);
    if (r + 1 < R) t = cmul(t, t1);
  }
}

// per-pass twiddle tables: the pass that starts at NS (radix R) owns NS*(R-1)
// entries [k][r-1] = w_{NS R}^{k r} (forward sign), read with 16-byte loads
template <int N>
constexpr int ct_radix(int ns) {
  return (ns * 8 >= N) ? 8 : ((N / ns / 8) >= 8 ? 8 : N / ns / 8);
}
template <int N>
constexpr int ct_tw_off(int NS) {
  int off = 0, ns = 8;
  while (ns < NS) {
    off += ns * (ct_radix<N>(ns) - 1);
    ns *= ct_radix<N>(ns);
  }
  return off;
}
template <int N>
constexpr int ct_tw_size() {
  return ct_tw_off<N>(N);
}

// Only w^k, w^2k and w^4k are read from the table; the other powers are
// products of those (at most two roundings more than a table entry), which
// takes four of the seven shared-memory reads per radix-8 item off the LSU
// pipe, the transforms' bottleneck.
template <int R, class C, class S>
__device__ __forceinline__ void twiddle_tab(C (&v)[R], const C* tt, S s) {
  C t[8];
  t[1] = tt[0];
  if constexpr (R >= 4) {
    t[2] = tt[1];
    t[3] = cmul(t[1], t[2]);
  }
  if constexpr (R == 8) {
    t[4] = tt[3];
    t[5] = cmul(t[1], t[4]);
    t[6] = cmul(t[2], t[4]);
    t[7] = cmul(t[3], t[4]);
  }
#pragma unroll
  for (int r = 1; r < R; ++r) {
    C w = t[r];
    if (s > 0) w.y = -w.y;
    v[r] = cmul(v[r], w);
  }
}

// Lines are independent through every pass, so the N/8 threads of one line
// synchronise only among themselves (named barrier, or warp-sync below 32
// threads): the LN line groups of a CTA drift apart and overlap one
// another's global-memory latency with arithmetic.
template <int N, bool G = true>
__device__ __forceinline__ void line_sync(int f) {
  constexpr int TT = N / 8;
  if constexpr (!G) {
    __syncthreads();
  } else if constexpr (TT >= 32) {
    asm volatile("bar.sync %0, %1;" ::"r"(f + 1), "n"(TT) : "memory");
  } else {
    const unsigned lane = threadIdx.x & 31;
    __syncwarp(((1u << TT) - 1u) << (lane & ~(unsigned)(TT - 1)));
  }
}

// middle pass (smem in place): radix R, IPT = 8/R work items per thread, all
// in the thread's own line
template <int N, int R, int NS, int LN, bool G>
__device__ __forceinline__ void ct_mid(double2* buf, const double2* tw2, double s) {
  constexpr int T = N / R;
  constexpr int TT = N / 8;
  constexpr int IPT = T / TT;
  constexpr int PITCH = ct_pitch<N>();
  constexpr int TOFF = ct_tw_off<N>(NS);
  const int f = threadIdx.x / TT, jt = threadIdx.x % TT;
  double2 v[IPT][R];
  int base[IPT], jj[IPT];
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int j = jt + it * TT;
    base[it] = f * PITCH;
    jj[it] = j;
#pragma unroll
    for (int r = 0; r < R; ++r) v[it][r] = buf[base[it] + padi(j + r * T)];
    twiddle_tab<R>(v[it], tw2 + TOFF + (j % NS) * (R - 1), s);
    dft_small<R>(v[it], s);
  }
  line_sync<N, G>(f);
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int j = jj[it], k = j % NS;
    const int idxD = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[base[it] + padi(idxD + r * NS)] = v[it][r];
  }
  line_sync<N, G>(f);
}

template <int N, int NS, int LN, bool G>
__device__ __forceinline__ void ct_mids(double2* buf, const double2* tw2, double s) {
  if constexpr (NS * 8 < N) {
    constexpr int R = ct_radix<N>(NS);
    ct_mid<N, R, NS, LN, G>(buf, tw2, s);
    ct_mids<N, NS * R, LN, G>(buf, tw2, s);
  }
}

// full line FFT for the item (line f, j in [0, N/8)): v holds w[j + r N/8] on
// entry (first-pass inputs) and Z[j + r N/8] on exit (natural order)
// G: the calling thread's (f, j) is (tid / (N/8), tid % (N/8)) and the line
// groups may synchronise independently; otherwise whole-CTA barriers
template <int N, int LN, bool G>
__device__ __forceinline__ void ct_line_fft(double2 (&v)[8], int f, int j, double2* buf, const double2* tw2, double s) {
  constexpr int PITCH = ct_pitch<N>();
  constexpr int T = N / 8;
  dft_small<8>(v, s);  // first pass, NS = 1: no twiddles
#pragma unroll
  for (int r = 0; r < 8; ++r) buf[f * PITCH + padi(8 * j + r)] = v[r];
  line_sync<N, G>(f);
  ct_mids<N, 8, LN, G>(buf, tw2, s);
  // last pass, NS = N/8: k = j, outputs at j + r*T
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = buf[f * PITCH + padi(j + r * T)];
  twiddle_tab<8>(v, tw2 + ct_tw_off<N>(N / 8) + j * 7, s);
  dft_small<8>(v, s);
}

// Makhoul twiddle E[j + r N/8] = E[j] * exp(i pi r / 16): one table read per
// item instead of eight
template <class Cp>
__device__ __forceinline__ Cp ct_e(Cp ej, int r) {
  using T = decltype(ej.x);
  constexpr double C[8] = {1.0, 0.9807852804032304, 0.9238795325112867, 0.8314696123025452,
                           0.7071067811865476, 0.5555702330196022, 0.3826834323650898, 0.19509032201612828};
  if (r == 0) return ej;
  return cmul(ej, mkc((T)C[r], (T)C[8 - r]));
}

__device__ __forceinline__ int ct_order(int m, int n) { return (m < (n >> 1)) ? 2 * m : 2 * n - 1 - 2 * m; }

// DCT-II recombination of the pair-packed spectrum: lines (even, odd) at k
template <class C>
__device__ __forceinline__ C dct2_pair(C a, C b, C E) {
  using T = decltype(a.x);
  return mkc((T)0.5 * (E.x * (a.x + b.x) + E.y * (a.y - b.y)), (T)0.5 * (E.x * (a.y + b.y) - E.y * (a.x - b.x)));
}

// DCT-III pre-twiddle of both packed lines: c = (C1[m], C2[m]), d = (C1[N-m], C2[N-m])
template <class C>
__device__ __forceinline__ C dct3_pair(C c, C d, C E) {
  const auto v1r = E.x * c.x + E.y * d.x, v1i = E.y * c.x - E.x * d.x;
  const auto v2r = E.x * c.y + E.y * d.y, v2i = E.y * c.y - E.x * d.y;
  return mkc(v1r - v2i, v1i + v2r);
}

template <int N, class T = double>
struct CtSmem {
  C2<T> *tw, *e, *buf;
};

// shared layout: per-pass twiddle tables | Makhoul twiddles e[N] | line buffer
template <int N, class T = double>
__device__ __forceinline__ CtSmem<N, T> ct_carve(C2<T>* sm, const C2<T>* twg, const C2<T>* eg) {
  CtSmem<N, T> S;
  constexpr int TWN = (ct_tw_size<N>() + 1) & ~1;
  S.tw = sm;
  S.e = sm + TWN;
  S.buf = sm + TWN + N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) S.e[i] = eg[i];
  // pass tables from the global table twg[m] = exp(-2 pi i m / N)
  int ns = 8;
#pragma unroll 1
  while (ns < N) {
    const int R = ct_radix<N>(ns), ts = N / (ns * R), off = ct_tw_off<N>(ns);
    for (int e = threadIdx.x; e < ns * (R - 1); e += blockDim.x) {
      const int k = e / (R - 1), r = e % (R - 1) + 1;
      S.tw[off + e] = twg[(k * r * ts) % N];
    }
    ns *= R;
  }
  __syncthreads();
  return S;
}

#ifndef ETC_Q64_MINB
#define ETC_Q64_MINB 2
#endif
#ifndef ETC_Q32_MINB
#define ETC_Q32_MINB 3
#endif
#ifndef ETC_CT_MINB
#define ETC_CT_MINB 2
#endif

// forward 2-D DCT-II, square planes; modes as k_fwd
template <int N, int MODE>
__global__ void __launch_bounds__(256, ETC_CT_MINB) k_fwd_ct(Geom g, const double* src, double* dst, double* r,
                                                   const double* q, Ctl* ctl, double* partials, unsigned* counter,
                                                   PlaneTabs T, double* hist) {
  if (MODE != 0 && ctl->done) return;
  constexpr int LN = 2048 / N, PITCH = ct_pitch<N>(), ROWS = 2 * LN, TT = N / 8;
  extern __shared__ double2 smem_c[];
  const CtSmem<N> S = ct_carve<N>(smem_c, T.twx, T.ex);
  const unsigned crank = cluster_ctarank(), csize = cluster_nctarank();
  const unsigned cid = cluster_id_x(), ncl = ncluster_x();
  const double alpha = (MODE == 2) ? ctl->alpha : 0.0;
  const int per = N / csize;  // rows (phase X) / columns (phase Y) per CTA
  const int a0 = crank * per;
  double rr = 0.0;
  // phase-X inputs of the next chunk are fetched into registers while the
  // current chunk is transformed (the last chunk prefetches the next plane)
  const int fx = threadIdx.x / TT, jx = threadIdx.x % TT;
  double xa[8], xb[8], ya[8], yb[8];
  auto fetch = [&](long long kz, int j0) {
    const long long r0 = kz * (long long)N * N + (long long)(j0 + 2 * fx) * N;
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) {
      const int i = ct_order(jx + r8 * TT, N);
      if (MODE == 2) {
        xa[r8] = r[r0 + i];
        xb[r8] = r[r0 + N + i];
        ya[r8] = q[r0 + i];
        yb[r8] = q[r0 + N + i];
      } else {
        xa[r8] = src[r0 + i];
        xb[r8] = src[r0 + N + i];
      }
    }
  };
  if (cid < g.nz) fetch(cid, a0);
  for (long long kz = cid; kz < g.nz; kz += ncl) {
    const long long pb = kz * (long long)N * N;
    // ---- phase X: rows [a0, a0+per), ROWS at a time; item (f, j) = (tid/TT, tid%TT)
    for (int j0 = a0; j0 < a0 + per; j0 += ROWS) {
      const int f = fx, j = jx;
      const long long r0 = pb + (long long)(j0 + 2 * f) * N;
      double2 v[8];
#pragma unroll
      for (int rr8 = 0; rr8 < 8; ++rr8) {
        const int i = ct_order(j + rr8 * TT, N);
        double a = xa[rr8], b = xb[rr8];
        if (MODE == 2) {
          a = __dsub_rn(a, __dmul_rn(alpha, ya[rr8]));
          b = __dsub_rn(b, __dmul_rn(alpha, yb[rr8]));
          r[r0 + i] = a;
          r[r0 + N + i] = b;
          rr = fma(a, a, fma(b, b, rr));
        } else if (MODE == 1) {
          rr = fma(a, a, fma(b, b, rr));
        }
        v[rr8] = make_double2(a, b);
      }
      if (j0 + ROWS < a0 + per)
        fetch(kz, j0 + ROWS);
      else if (kz + ncl < g.nz)
        fetch(kz + ncl, a0);
      ct_line_fft<N, LN, true>(v, f, j, S.buf, S.tw, -1.0);
      line_sync<N>(f);
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8) S.buf[f * PITCH + padi(j + r8 * TT)] = v[r8];
      line_sync<N>(f);
      const double2 ej = S.e[j];
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8) {
        const int m = j + r8 * TT;
        const double2 o = dct2_pair(v[r8], S.buf[f * PITCH + padi((N - m) & (N - 1))], ct_e(ej, r8));
        dst[r0 + m] = o.x;
        dst[r0 + N + m] = o.y;
      }
      line_sync<N>(f);
    }
    cluster_barrier();
    // ---- phase Y: columns [a0, a0+per), ROWS at a time; item (f, j) = (tid%LN, tid/LN)
    for (int c0 = a0; c0 < a0 + per; c0 += ROWS) {
      const int f = threadIdx.x % LN, j = threadIdx.x / LN;
      const long long cb = pb + c0 + 2 * f;
      double2 v[8];
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8)
        v[r8] = __ldcg(reinterpret_cast<const double2*>(dst + cb + (long long)ct_order(j + r8 * TT, N) * N));
      ct_line_fft<N, LN, false>(v, f, j, S.buf, S.tw, -1.0);
      __syncthreads();
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8) S.buf[f * PITCH + padi(j + r8 * TT)] = v[r8];
      __syncthreads();
      const double2 ej = S.e[j];
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8) {
        const int m = j + r8 * TT;
        *reinterpret_cast<double2*>(dst + cb + (long long)m * N) =
            dct2_pair(v[r8], S.buf[f * PITCH + padi((N - m) & (N - 1))], ct_e(ej, r8));
      }
      __syncthreads();
    }
  }
  if (MODE != 0) {
    double vv[1] = {rr};
    grid_sum_finalize<1>(vv, partials, counter, [&](double (&t)[1]) {
      if (ctl->dist)
        ctl->xbuf[3] = t[0];
      else if (MODE == 1)
        fin_normb(ctl, t[0], hist);
      else
        fin_update(ctl, t[0], hist);
    });
  }
}

// inverse 2-D transform, square planes: phase X (rows of src, DRAM) then
// phase Y (columns of dst, back through L2), finishing dst in place
template <int N, bool PCG>
__global__ void __launch_bounds__(256, ETC_CT_MINB) k_inv_ct(Geom g, const double* src, double* dst, const Ctl* ctl,
                                                   PlaneTabs T) {
  if (PCG && ctl->done) return;
  constexpr int LN = 2048 / N, ROWS = 2 * LN, TT = N / 8;
  constexpr double IV = 1.0 / N;
  extern __shared__ double2 smem_c[];
  const CtSmem<N> S = ct_carve<N>(smem_c, T.twx, T.ex);
  const unsigned crank = cluster_ctarank(), csize = cluster_nctarank();
  const unsigned cid = cluster_id_x(), ncl = ncluster_x();
  const int per = N / csize;
  const int a0 = crank * per;
  const int fx = threadIdx.x / TT, jx = threadIdx.x % TT;
  double xc[8], xd[8], yc[8], yd[8];
  auto fetch = [&](long long kz, int j0) {
    const long long r0 = kz * (long long)N * N + (long long)(j0 + 2 * fx) * N;
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) {
      const int m = jx + r8 * TT;
      xc[r8] = src[r0 + m];
      yc[r8] = src[r0 + N + m];
      xd[r8] = m ? src[r0 + N - m] : 0.0;
      yd[r8] = m ? src[r0 + 2 * N - m] : 0.0;
    }
  };
  for (long long kz = cid; kz < g.nz; kz += ncl) {
    const long long pb = kz * (long long)N * N;
    fetch(kz, a0);
    // ---- phase X
    for (int j0 = a0; j0 < a0 + per; j0 += ROWS) {
      const int f = fx, j = jx;
      const long long r0 = pb + (long long)(j0 + 2 * f) * N;
      double2 v[8];
      const double2 ej = S.e[j];
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8)
        v[r8] = dct3_pair(make_double2(xc[r8], yc[r8]), make_double2(xd[r8], yd[r8]), ct_e(ej, r8));
      if (j0 + ROWS < a0 + per) fetch(kz, j0 + ROWS);
      ct_line_fft<N, LN, true>(v, f, j, S.buf, S.tw, 1.0);
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8) {
        const int i = ct_order(j + r8 * TT, N);
        dst[r0 + i] = v[r8].x * IV;
        dst[r0 + N + i] = v[r8].y * IV;
      }
      line_sync<N>(f);
    }
    cluster_barrier();
    // ---- phase Y (next chunk's columns prefetched during the current one)
    const int fy = threadIdx.x % LN, jy = threadIdx.x / LN;
    double2 pc[8], pd[8];
    auto fetchy = [&](int c0) {
      const long long cb = pb + c0 + 2 * fy;
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8) {
        const int m = jy + r8 * TT;
        pc[r8] = __ldcg(reinterpret_cast<const double2*>(dst + cb + (long long)m * N));
        pd[r8] = m ? __ldcg(reinterpret_cast<const double2*>(dst + cb + (long long)(N - m) * N))
                   : make_double2(0.0, 0.0);
      }
    };
    fetchy(a0);
    for (int c0 = a0; c0 < a0 + per; c0 += ROWS) {
      const int f = fy, j = jy;
      const long long cb = pb + c0 + 2 * f;
      double2 v[8];
      const double2 ej = S.e[j];
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8) v[r8] = dct3_pair(pc[r8], pd[r8], ct_e(ej, r8));
      if (c0 + ROWS < a0 + per) fetchy(c0 + ROWS);
      __syncthreads();  // the line's columns are read before any is rewritten
      ct_line_fft<N, LN, false>(v, f, j, S.buf, S.tw, 1.0);
#pragma unroll
      for (int r8 = 0; r8 < 8; ++r8) {
        const double2 w = v[r8];
        *reinterpret_cast<double2*>(dst + cb + (long long)ct_order(j + r8 * TT, N) * N) =
            make_double2(w.x * IV, w.y * IV);
      }
      __syncthreads();
    }
  }
}

// ===========================================================================
// Paired-item plane transforms (square N >= 128).  Each thread owns TWO
// radix-8 items of its line, chosen so that every value an item needs from
// its mirror item lives in the same thread:
//   * the Makhoul gather w[m] = v[2m] / w[N-1-m] = v[2m+1] pairs item j with
//     item N/8-1-j: one 16-byte load (v[2m], v[2m+1]) feeds both, so phase X
//     reads and the r -= alpha q update are fully vectorised and coalesced;
//   * the DCT-II recombination (and the DCT-III pre-twiddle) couples Z[m]
//     with Z[N-m], i.e. item j with item N/8-j: the mirror is in registers,
//     with no shared-memory round trip.
// A line has TPL = N/16 threads, a chunk LPC = 4096/N lines.  In phase X the
// line's threads are contiguous (one warp for N = 512), so the line
// synchronises by itself; phase Y interleaves lines across lanes for
// coalesced column access and synchronises the CTA.
// ===========================================================================
// threads per CTA of the paired-item transforms: 256 (2 CTAs/SM) up to
// N = 512; at N = 1024 512 threads at 1 CTA/SM, so that fewer 8 MB planes
// are in flight and the phase-X intermediate stays in L2 (1024^3: fwd
// 15.0 -> 11.0 ms, inv 14.4 -> 10.3 ms)
template <int N>
constexpr int c2_nt() { return N >= 1024 ? 512 : 256; }
template <int N>
constexpr int c2_lpc() { return c2_nt<N>() * 16 / N; }
// line pitch (complex elements): one pad per 8 (padi) plus an offset that
// spreads the lines a quarter-warp touches in the column phase over the
// banks; 8-byte elements (float2) are served per half-warp and need an
// offset of 2 there (a bank model of the passes: excess wavefronts of the
// column phase 2.0 -> 1.03 per access at N = 512)
template <int N, class T = double>
constexpr int c2_pitch() {
  return N + N / 8 + ((sizeof(T) == 4 && N >= 512) ? 2 : (c2_lpc<N>() >= 8 ? 1 : 8 / c2_lpc<N>()));
}

template <int N, bool G>
__device__ __forceinline__ void c2_sync(int f) {
  constexpr int TPL = N / 16;
  if constexpr (!G) {
    __syncthreads();
  } else if constexpr (TPL > 32) {
    asm volatile("bar.sync %0, %1;" ::"r"(f + 1), "n"(TPL) : "memory");
  } else if constexpr (TPL == 32) {
    __syncwarp();
  } else {
    const unsigned lane = threadIdx.x & 31;
    __syncwarp(((1u << TPL) - 1u) << (lane & ~(unsigned)(TPL - 1)));
  }
}

// middle Stockham pass (shared, in place) over the line's T = N/R items
template <int N, int R, int NS, bool G, class C, class S>
__device__ __forceinline__ void c2_mid(C* line, const C* tw2, S s, int f, int t) {
  constexpr int TPL = N / 16, T = N / R, IPT = T / TPL, TOFF = ct_tw_off<N>(NS);
  C v[IPT][R];
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int j = t + it * TPL;
#pragma unroll
    for (int r = 0; r < R; ++r) v[it][r] = line[padi(j + r * T)];
    twiddle_tab<R>(v[it], tw2 + TOFF + (j % NS) * (R - 1), s);
    dft_small<R>(v[it], s);
  }
  c2_sync<N, G>(f);
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int j = t + it * TPL;
    const int idxD = (j / NS) * NS * R + j % NS;
#pragma unroll
    for (int r = 0; r < R; ++r) line[padi(idxD + r * NS)] = v[it][r];
  }
  c2_sync<N, G>(f);
}

template <int N, int NS, bool G, class C, class S>
__device__ __forceinline__ void c2_mids(C* line, const C* tw2, S s, int f, int t) {
  if constexpr (NS * 8 < N) {
    constexpr int R = ct_radix<N>(NS);
    c2_mid<N, R, NS, G>(line, tw2, s, f, t);
    c2_mids<N, NS * R, G>(line, tw2, s, f, t);
  }
}

// whole line FFT for the thread's two first-pass items (ja, jb; inputs
// w[j + r N/8] in a, b) and two last-pass items (ka, kb; outputs Z[k + r N/8]
// returned in a, b).  The caller has synchronised the line since its last
// read of the buffer.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

template <int N, bool G, class Hook = NoHook, class C, class S>
__device__ __forceinline__ void c2_fft(C (&a)[8], C (&b)[8], int ja, int jb, int ka, int kb, C* line, const C* tw2,
                                       S s, int f, int t, Hook before_last = Hook()) {
  constexpr int T = N / 8;
  dft_small<8>(a, s);
  dft_small<8>(b, s);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    line[padi(8 * ja + r)] = a[r];
    line[padi(8 * jb + r)] = b[r];
  }
  c2_sync<N, G>(f);
  c2_mids<N, 8, G>(line, tw2, s, f, t);
  before_last();  // e.g. loads the epilogue's operands while the last pass computes
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    a[r] = line[padi(ka + r * T)];
    b[r] = line[padi(kb + r * T)];
  }
  twiddle_tab<8>(a, tw2 + ct_tw_off<N>(T) + ka * 7, s);
  twiddle_tab<8>(b, tw2 + ct_tw_off<N>(T) + kb * 7, s);
  dft_small<8>(a, s);
  dft_small<8>(b, s);
}

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }

// L2 eviction hints: streamed operands (read or written once here) go
// evict-first, the phase-X intermediate that phase Y re-reads evict-last
#ifndef ETC_L2HINTS
#define ETC_L2HINTS 1
#endif

__device__ __forceinline__ unsigned long long pol_first() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_last() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ double2 ld2h(const double* p, unsigned long long pol) {
  if (!ETC_L2HINTS) return ld2(p);
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldh(const double* p, unsigned long long pol) {
  if (!ETC_L2HINTS) return *p;
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st2h(double* p, double2 v, unsigned long long pol) {
  if (!ETC_L2HINTS) {
    *reinterpret_cast<double2*>(p) = v;
    return;
  }
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void sth(double* p, double v, unsigned long long pol) {
  if (!ETC_L2HINTS) {
    *p = v;
    return;
  }
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// the same for the float32 path's pairs
__device__ __forceinline__ float2 ld2h(const float* p, unsigned long long pol) {
  if (!ETC_L2HINTS || pol == 0) return ld2(p);
  float2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ldh(const float* p, unsigned long long pol) {
  if (!ETC_L2HINTS || pol == 0) return *p;
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st2h(float* p, float2 v, unsigned long long pol) {
  if (!ETC_L2HINTS || pol == 0) {
    *reinterpret_cast<float2*>(p) = v;
    return;
  }
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void sth(float* p, float v, unsigned long long pol) {
  if (!ETC_L2HINTS || pol == 0) {
    *p = v;
    return;
  }
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ int g_phmask = 0;  // ETC_PHMASK (measurement only): 1 skips phase Y, 2 skips phase X of the plane transforms
__device__ int g_wpf = 2;  // w_old L2 prefetch in the inverse: 0 off, 1 evict_last, 2 evict_normal (default), 3 plain
__device__ __forceinline__ double2 ld2cg(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }
__device__ __forceinline__ float2 ld2cg(const float* p) { return __ldcg(reinterpret_cast<const float2*>(p)); }
__device__ __forceinline__ void st2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
// one pair of consecutive elements into shared memory (16 bytes of double, 8 of float)
__device__ __forceinline__ void cp_pair(double* smem, const double* gmem) { cp_async16(smem, gmem); }
__device__ __forceinline__ void cp_pair(float* smem, const float* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---- paired-item plane transforms, per chunk.  A chunk is 2*LPC rows
// (phase X: one line of TPL contiguous threads per row pair) or 2*LPC columns
// (phase Y: LPC lines interleaved across lanes).  The cluster kernels
// (k_fwd_c2 / k_inv_c2) run a plane's row chunks, a cluster barrier, then its
// column chunks; the decoupled kernels (k_fwd_q / k_inv_q) run the same chunks
// as independent tasks.

// forward phase X, rows [p0, p0 + 2 LPC) of plane pb: MODE 2 updates r -= alpha q
// (and accumulates |r|^2), MODE 1 accumulates |src|^2; row DCT-II into dst
template <int N, int MODE, class T = double>
__device__ __forceinline__ void fwd_rows(const CtSmem<N, T>& S, long long pb, int p0, const T* src, T* dst, T* r,
                                         const T* q, T alpha, double& rr, unsigned long long PF,
                                         unsigned long long PL) {
  using C = C2<T>;
  constexpr int TT = N / 8, TPL = N / 16, PITCH = c2_pitch<N, T>();
  const int f = threadIdx.x / TPL, t = threadIdx.x % TPL, tq = TT - 1 - t;
  const int ka = t, kb = t ? TT - t : TT / 2;  // last-pass (mirror) items t, TT-t (0: 0, TT/2)
  C* line = S.buf + f * PITCH;
  const C ea = S.e[ka], eb = S.e[kb];
  const long long ra = pb + (long long)(p0 + 2 * f) * N, rb = ra + N;
  C va[8], vb[8];
  // MODE 2: the q row pair goes to this line's shared buffer by cp.async
  // (each thread stages exactly the 16-byte pieces it reads back) while r
  // loads into registers, so both streams are in flight at once without
  // holding 64 doubles of loads in registers
  T* qs = reinterpret_cast<T*>(line);  // [row a | row b], 2 N elements (< the padded line)
  if (MODE == 2) {
    c2_sync<N, true>(f);  // previous chunk's last-pass reads of this line are done
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int m1 = 2 * (t + k * TT), m2 = 2 * (tq + k * TT);
      cp_pair(qs + m1, q + ra + m1);
      cp_pair(qs + N + m1, q + rb + m1);
      cp_pair(qs + m2, q + ra + m2);
      cp_pair(qs + N + m2, q + rb + m2);
    }
    cp_async_commit();
  }
  C rv[16];
  if (MODE == 2) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int m1 = 2 * (t + k * TT), m2 = 2 * (tq + k * TT);
      rv[4 * k + 0] = ld2h(r + ra + m1, PF);
      rv[4 * k + 1] = ld2h(r + rb + m1, PF);
      rv[4 * k + 2] = ld2h(r + ra + m2, PF);
      rv[4 * k + 3] = ld2h(r + rb + m2, PF);
    }
    cp_async_wait_all();
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int m1 = 2 * (t + k * TT), m2 = 2 * (tq + k * TT);
    C A1, B1, A2, B2;  // rows a/b at m1, m2
    if (MODE == 2) {
      A1 = rv[4 * k + 0];
      B1 = rv[4 * k + 1];
      A2 = rv[4 * k + 2];
      B2 = rv[4 * k + 3];
      const C qa1 = ld2(qs + m1), qb1 = ld2(qs + N + m1);
      const C qa2 = ld2(qs + m2), qb2 = ld2(qs + N + m2);
      auto upd = [&](C& x, C y) {
        x.x = sub_rn(x.x, mul_rn(alpha, y.x));
        x.y = sub_rn(x.y, mul_rn(alpha, y.y));
      };
      upd(A1, qa1);
      upd(B1, qb1);
      upd(A2, qa2);
      upd(B2, qb2);
      st2h(r + ra + m1, A1, PF);
      st2h(r + rb + m1, B1, PF);
      st2h(r + ra + m2, A2, PF);
      st2h(r + rb + m2, B2, PF);
    } else {
      A1 = ld2h(src + ra + m1, PF);
      B1 = ld2h(src + rb + m1, PF);
      A2 = ld2h(src + ra + m2, PF);
      B2 = ld2h(src + rb + m2, PF);
    }
    if (MODE != 0) {
      const double a1x = A1.x, a1y = A1.y, b1x = B1.x, b1y = B1.y;
      const double a2x = A2.x, a2y = A2.y, b2x = B2.x, b2y = B2.y;
      rr = fma(a1x, a1x, fma(a1y, a1y, rr));
      rr = fma(b1x, b1x, fma(b1y, b1y, rr));
      rr = fma(a2x, a2x, fma(a2y, a2y, rr));
      rr = fma(b2x, b2x, fma(b2y, b2y, rr));
    }
    va[k] = mkc(A1.x, B1.x);
    vb[7 - k] = mkc(A1.y, B1.y);
    vb[k] = mkc(A2.x, B2.x);
    va[7 - k] = mkc(A2.y, B2.y);
  }
  c2_sync<N, true>(f);  // previous chunk's last-pass reads are done
  c2_fft<N, true>(va, vb, t, tq, ka, kb, line, S.tw, (T)-1, f, t);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const C ma = t ? vb[7 - k] : va[(8 - k) & 7];
    const C mb = t ? va[7 - k] : vb[7 - k];
    const C oa = dct2_pair(va[k], ma, ct_e(ea, k));
    const C ob = dct2_pair(vb[k], mb, ct_e(eb, k));
    sth(dst + ra + ka + k * TT, oa.x, PL);
    sth(dst + rb + ka + k * TT, oa.y, PL);
    sth(dst + ra + kb + k * TT, ob.x, PL);
    sth(dst + rb + kb + k * TT, ob.y, PL);
  }
}

// forward phase Y, columns [c0, c0 + 2 LPC) of plane kz (base pb): column DCT-II
// of the phase-X output in dst, written in place (or, pk != null, into the
// pencil all-to-all's send layout / the peers' pencil buffers)
template <int N, class T = double>
__device__ __forceinline__ void fwd_cols(const CtSmem<N, T>& S, const Geom& g, long long kz, long long pb, int c0,
                                         T* dst, T* pk, int nyl, T* const* peers, int me, unsigned long long PF) {
  using C = C2<T>;
  constexpr int TT = N / 8, LPC = c2_lpc<N>(), PITCH = c2_pitch<N, T>();
  constexpr int EPL = 128 / sizeof(T);  // elements per 128-byte line
  const int f = threadIdx.x % LPC, t = threadIdx.x / LPC, tq = TT - 1 - t;
  const int ka = t, kb = t ? TT - t : TT / 2;
  C* line = S.buf + f * PITCH;
  const C ea = S.e[ka], eb = S.e[kb];
  const long long cb = pb + c0 + 2 * f;
  C va[8], vb[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long m1 = 2 * (t + k * TT), m2 = 2 * (tq + k * TT);
    va[k] = ld2cg(dst + cb + m1 * N);
    vb[7 - k] = ld2cg(dst + cb + (m1 + 1) * N);
    vb[k] = ld2cg(dst + cb + m2 * N);
    va[7 - k] = ld2cg(dst + cb + (m2 + 1) * N);
  }
  __syncthreads();  // every line's columns are read, previous chunk drained
  if (pk) {
    // the spectrum goes to the send buffer, so this chunk's phase-X
    // lines in dst are dead: drop them from L2 instead of writing back
    constexpr int CW = 2 * LPC;
    if constexpr (CW >= EPL) {
      for (int e = threadIdx.x; e < N * (CW / EPL); e += c2_nt<N>())
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(dst + pb + c0 + (e % (CW / EPL)) * EPL +
                                                             (long long)(e / (CW / EPL)) * N)
                     : "memory");
    }
  }
  c2_fft<N, false>(va, vb, t, tq, ka, kb, line, S.tw, (T)-1, f, t);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const C ma = t ? vb[7 - k] : va[(8 - k) & 7];
    const C mb = t ? va[7 - k] : vb[7 - k];
    // spectral row m of column pair cb (or its slot in the pencil send buffer)
    auto outp = [&](int m) -> T* {
      if (pk) {  // nyl is a power of two (etc_slab_fused): shifts, not divisions
        const int sh = __ffs(nyl) - 1, rk = m >> sh, jl = m & (nyl - 1);
        if (peers)  // destination rank rk's pencil buffer, block of this (source) rank
          return peers[rk] + ((long long)(me * g.nz + kz) * nyl + jl) * N + c0 + 2 * f;
        return pk + ((long long)(rk * g.nz + kz) * nyl + jl) * N + c0 + 2 * f;
      }
      return dst + cb + (long long)m * N;
    };
    st2h(outp(ka + k * TT), dct2_pair(va[k], ma, ct_e(ea, k)), PF);
    st2h(outp(kb + k * TT), dct2_pair(vb[k], mb, ct_e(eb, k)), PF);
  }
}

template <int MODE, class T = double>
__device__ __forceinline__ void fwd_finish(double rr, Ctl* ctl, double* partials, unsigned* counter, double* hist) {
  if (MODE != 0) {
    double vv[1] = {rr};
    grid_sum_finalize<1>(vv, partials, counter, [&](double (&t)[1]) {
      if (ctl->dist)
        ctl->xbuf[3] = t[0];
      else if constexpr (sizeof(T) == 4) {
        if (MODE == 1)
          fin_normb32(ctl, t[0], hist);
        else
          fin_update32(ctl, t[0], hist);
      } else if (MODE == 1)
        fin_normb(ctl, t[0], hist);
      else
        fin_update(ctl, t[0], hist);
    });
  }
}

// forward 2-D DCT-II, square planes, paired items; modes as k_fwd
template <int N, int MODE>
__global__ void __launch_bounds__(c2_nt<N>(), 512 / c2_nt<N>()) k_fwd_c2(Geom g, const double* src, double* dst, double* r,
                                                   const double* q, Ctl* ctl, double* partials, unsigned* counter,
                                                   PlaneTabs T, double* hist, double* pk, int nyl,
                                                   double* const* peers, int me) {
  if (MODE != 0 && ctl->done) return;
  constexpr int LPC = c2_lpc<N>();
  extern __shared__ double2 smem_c[];
  const CtSmem<N> S = ct_carve<N>(smem_c, T.twx, T.ex);
  const unsigned crank = cluster_ctarank(), csize = cluster_nctarank();
  const unsigned cid = cluster_id_x(), ncl = ncluster_x();
  const double alpha = (MODE == 2) ? ctl->alpha : 0.0;
  const int per = N / csize;  // rows (phase X) / columns (phase Y) per CTA
  const int a0 = crank * per;
  double rr = 0.0;
  const unsigned long long PF = pol_first(), PL = pol_last();
  for (long long kz = cid; kz < g.nz; kz += ncl) {
    const long long pb = kz * (long long)N * N;
    if (!(g_phmask & 2))
      for (int p0 = a0; p0 < a0 + per; p0 += 2 * LPC) fwd_rows<N, MODE>(S, pb, p0, src, dst, r, q, alpha, rr, PF, PL);
    cluster_barrier();
    if (!(g_phmask & 1)) {
      for (int c0 = a0; c0 < a0 + per; c0 += 2 * LPC) fwd_cols<N>(S, g, kz, pb, c0, dst, pk, nyl, peers, me, PF);
      __syncthreads();
    }
  }
  if (peers) __threadfence_system();  // peer stores ordered before the host-side barrier
  fwd_finish<MODE>(rr, ctl, partials, counter, hist);
}

// inverse phase X, spectral rows [p0, p0 + 2 LPC) of plane kz: DCT-III
// pre-twiddle and row FFT, scaled, into dst (the phase-X scratch)

// the DCT-III pre-twiddle of both packed lines of a thread's two items
template <class C>
__device__ __forceinline__ void dct3_pre(C (&va)[8], C (&vb)[8], int t, C ea, C eb) {
  C oa[8], ob[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const C da = t ? vb[7 - k] : (k ? va[8 - k] : mkc(decltype(ea.x)(0), decltype(ea.x)(0)));
    const C db = t ? va[7 - k] : vb[7 - k];
    oa[k] = dct3_pair(va[k], da, ct_e(ea, k));
    ob[k] = dct3_pair(vb[k], db, ct_e(eb, k));
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    va[k] = oa[k];
    vb[k] = ob[k];
  }
}

template <int N, class T = double>
__device__ __forceinline__ void inv_rows(const CtSmem<N, T>& S, const Geom& g, long long kz, long long pb, int p0,
                                         const T* src, T* dst, const T* pk, int nyl, unsigned long long PF,
                                         unsigned long long PL) {
  using C = C2<T>;
  constexpr int TT = N / 8, TPL = N / 16, PITCH = c2_pitch<N, T>();
  constexpr T IV = (T)(1.0 / N);
  const int f = threadIdx.x / TPL, t = threadIdx.x % TPL, tq = TT - 1 - t;
  const int ja = t, jb = t ? TT - t : TT / 2;  // first-pass (mirror) items; last-pass (store) items t, TT-1-t
  C* line = S.buf + f * PITCH;
  const C ea = S.e[ja], eb = S.e[jb];
  const long long ra = pb + (long long)(p0 + 2 * f) * N, rb = ra + N;
  // the spectrum's rows: plane layout, or the pencil buffer's blocks
  const T* sa = src + ra;
  if (pk) {
    const int row = p0 + 2 * f, rk = row >> (__ffs(nyl) - 1), jl = row & (nyl - 1);
    sa = pk + ((long long)(rk * g.nz + kz) * nyl + jl) * N;
  }
  const T* sb = sa + N;  // nyl is even: the pair never straddles a block
  C va[8], vb[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    va[k] = mkc(ldh(sa + ja + k * TT, PF), ldh(sb + ja + k * TT, PF));
    vb[k] = mkc(ldh(sa + jb + k * TT, PF), ldh(sb + jb + k * TT, PF));
  }
  dct3_pre(va, vb, t, ea, eb);
  c2_sync<N, true>(f);
  c2_fft<N, true>(va, vb, ja, jb, t, tq, line, S.tw, (T)1, f, t);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int m1 = 2 * (t + k * TT), m2 = 2 * (tq + k * TT);
    st2h(dst + ra + m1, mkc(va[k].x * IV, vb[7 - k].x * IV), PL);
    st2h(dst + rb + m1, mkc(va[k].y * IV, vb[7 - k].y * IV), PL);
    st2h(dst + ra + m2, mkc(vb[k].x * IV, va[7 - k].x * IV), PL);
    st2h(dst + rb + m2, mkc(vb[k].y * IV, va[7 - k].y * IV), PL);
  }
}

// inverse phase Y, columns [c0, c0 + 2 LPC) of plane kz: column FFT of the
// phase-X scratch; WM 0 writes z over dst, WM 1 w = z, WM 2 p += alpha w_old
// (planes p_plane / all) and w = z + beta w_old in place
template <int N, int WM, class T = double>
__device__ __forceinline__ void inv_cols(const CtSmem<N, T>& S, long long kz, long long pb, int c0, T* dst, T* w,
                                         T* p, int p_plane, T alpha, T beta, int wpf, unsigned long long PF) {
  using C = C2<T>;
  constexpr int TT = N / 8, LPC = c2_lpc<N>(), PITCH = c2_pitch<N, T>();
  constexpr int EPL = 128 / sizeof(T);  // elements per 128-byte line
  constexpr T IV = (T)(1.0 / N);
  const int f = threadIdx.x % LPC, t = threadIdx.x / LPC, tq = TT - 1 - t;
  const int ja = t, jb = t ? TT - t : TT / 2;
  C* line = S.buf + f * PITCH;
  const C ea = S.e[ja], eb = S.e[jb];
  const long long cb = pb + c0 + 2 * f;
  C va[8], vb[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    va[k] = ld2cg(dst + cb + (long long)(ja + k * TT) * N);
    vb[k] = ld2cg(dst + cb + (long long)(jb + k * TT) * N);
  }
  dct3_pre(va, vb, t, ea, eb);
  __syncthreads();  // columns read before any is rewritten, previous chunk drained
  if constexpr (WM != 0) {
    // the scratch rows of this chunk (one 128-byte line per row) are dead
    // now: drop them from L2 instead of letting them be written back
    // (only when the chunk owns whole lines: the chunks of a plane are
    // independent tasks, so a line shared with another chunk may still be unread)
    constexpr int CW = 2 * LPC;  // chunk width in elements
    if constexpr (CW >= EPL) {
      for (int e = threadIdx.x; e < N * (CW / EPL); e += c2_nt<N>())
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(dst + pb + c0 + (e % (CW / EPL)) * EPL +
                                                             (long long)(e / (CW / EPL)) * N)
                     : "memory");
    }
  }
  if constexpr (WM == 2) {
    // w_old rows of this chunk (one 128-byte line per row at N = 512)
    // start moving to L2 now; the last pass's loads then hit L2
    constexpr int CW = 2 * LPC, NLN = (CW + EPL - 1) / EPL;
    for (int e = threadIdx.x; e < N * NLN; e += c2_nt<N>()) {
      const T* a_ = w + pb + c0 + (e % NLN) * EPL + (long long)(e / NLN) * N;
      if (wpf == 1)
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a_));
      else if (wpf == 2)
        asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(a_));
      else if (wpf == 3)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a_));
    }
  }
  C wo[16];  // WM = 2: w_old at the 16 outputs, loaded during the last pass
  auto ldw = [&]() {
    if constexpr (WM == 2) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long long m1 = 2 * (t + k * TT), m2 = 2 * (tq + k * TT);
        wo[4 * k + 0] = ld2h(w + cb + m1 * N, PF);
        wo[4 * k + 1] = ld2h(w + cb + (m1 + 1) * N, PF);
        wo[4 * k + 2] = ld2h(w + cb + m2 * N, PF);
        wo[4 * k + 3] = ld2h(w + cb + (m2 + 1) * N, PF);
      }
    }
  };
  c2_fft<N, false>(va, vb, ja, jb, t, tq, line, S.tw, (T)1, f, t, ldw);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long m1 = 2 * (t + k * TT), m2 = 2 * (tq + k * TT);
    const C a = va[k], b = vb[7 - k], c = vb[k], d = va[7 - k];
    if constexpr (WM == 0) {
      st2(dst + cb + m1 * N, mkc(a.x * IV, a.y * IV));
      st2(dst + cb + (m1 + 1) * N, mkc(b.x * IV, b.y * IV));
      st2(dst + cb + m2 * N, mkc(c.x * IV, c.y * IV));
      st2(dst + cb + (m2 + 1) * N, mkc(d.x * IV, d.y * IV));
    } else {
      const bool pk = (WM == 2) && (p_plane == -1 || kz == p_plane);
      auto put = [&](long long o, C zv, C wo) {
        zv = mkc(mul_rn(zv.x, IV), mul_rn(zv.y, IV));
        if constexpr (WM == 2) {
          if (pk) {
            const C pv = ld2(p + o);
            st2(p + o, mkc(add_rn(pv.x, mul_rn(alpha, wo.x)), add_rn(pv.y, mul_rn(alpha, wo.y))));
          }
          zv = mkc(add_rn(zv.x, mul_rn(beta, wo.x)), add_rn(zv.y, mul_rn(beta, wo.y)));
        }
        st2h(w + o, zv, PF);
      };
      put(cb + m1 * N, a, wo[4 * k + 0]);
      put(cb + (m1 + 1) * N, b, wo[4 * k + 1]);
      put(cb + m2 * N, c, wo[4 * k + 2]);
      put(cb + (m2 + 1) * N, d, wo[4 * k + 3]);
    }
  }
}

// inverse 2-D transform, square planes, paired items.
// WM = 0: dst = M^-1 applied in place (phase Y rewrites the phase-X output).
// WM = 1, 2 (the solve's fused search-direction update): phase X writes its
// output to dst (scratch); phase Y writes the new search direction instead of
// z, w = z (WM = 1, first iteration) or, WM = 2, p += alpha w_old on the
// planes the solve keeps (p_plane; -1 all) and w = z + beta w_old in place,
// so z never reaches HBM (krylov.py:70-76 order of operations).
template <int N, bool PCG, int WM = 0>
__global__ void __launch_bounds__(c2_nt<N>(), 512 / c2_nt<N>()) k_inv_c2(Geom g, const double* src, double* dst, const Ctl* ctl,
                                                   PlaneTabs T, double* w, double* p, int p_plane,
                                                   const double* pk, int nyl) {
  if (PCG && ctl->done) return;
  const double beta = (WM == 2) ? ctl->beta : 0.0, alpha = (WM == 2) ? ctl->alpha : 0.0;
  constexpr int LPC = c2_lpc<N>();
  extern __shared__ double2 smem_c[];
  const CtSmem<N> S = ct_carve<N>(smem_c, T.twx, T.ex);
  const unsigned crank = cluster_ctarank(), csize = cluster_nctarank();
  const unsigned cid = cluster_id_x(), ncl = ncluster_x();
  const int per = N / csize;
  const int a0 = crank * per;
  const unsigned long long PF = pol_first(), PL = pol_last();
  const int wpf = g_wpf;
  for (long long kz = cid; kz < g.nz; kz += ncl) {
    const long long pb = kz * (long long)N * N;
    if (!(g_phmask & 2))
      for (int p0 = a0; p0 < a0 + per; p0 += 2 * LPC) inv_rows<N>(S, g, kz, pb, p0, src, dst, pk, nyl, PF, PL);
    cluster_barrier();
    if (!(g_phmask & 1)) {
      for (int c0 = a0; c0 < a0 + per; c0 += 2 * LPC)
        inv_cols<N, WM>(S, kz, pb, c0, dst, w, p, p_plane, alpha, beta, wpf, PF);
      __syncthreads();
    }
  }
}

// ---- decoupled plane transforms (single GPU, plane layout): the row chunks
// and column chunks of every plane are independent tasks of one persistent
// grid, with no cluster barrier.  Round r issues the row tasks of plane r and
// the column tasks of plane r - D; CTA b takes tasks b, b + G, b + 2G, ...
// (static, so the reductions are deterministic).  A column task waits until
// every line of its plane has been published by its row task's line group
// (a per-plane counter reset before the launch, release / acquire at gpu
// scope), so consecutive row tasks need no CTA barrier and the warps drift.  Every task a CTA waits on sits at an earlier step of
// some CTA's sequence (D * tasks-per-round >= G), so all co-resident CTAs make
// progress.  The row and column work of different planes and CTAs now overlap
// on every SM instead of meeting at a cluster barrier per plane.
struct QSched {
  unsigned* cnt;        // per-plane published row tasks (monotonic)
  unsigned target;      // epoch * row tasks per plane
  int depth;            // D: planes between a plane's row tasks and its column tasks
  int cta_pub;          // 1: a row task publishes its LPC lines at once after a CTA barrier
};

// a row task's line group publishes its line: the group synchronises (its
// stores are issued and ordered), its first thread releases one count
template <int N>
__device__ __forceinline__ void q_publish_line(unsigned* c) {
  constexpr int TPL = N / 16;
  c2_sync<N, true>(threadIdx.x / TPL);
  if (threadIdx.x % TPL == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
}
template <int N>
__device__ __forceinline__ void q_publish(const QSched& qs, long long kz) {
  if (qs.cta_pub) {
    __syncthreads();
    if (threadIdx.x == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(qs.cnt + kz), "r"((unsigned)c2_lpc<N>())
                   : "memory");
  } else {
    q_publish_line<N>(qs.cnt + kz);
  }
}
__device__ __forceinline__ void q_await(const unsigned* c, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
      if ((int)(v - target) >= 0) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// task t -> (is_column, plane, chunk); false past the last task
template <int N>
__device__ __forceinline__ bool q_task(long long t, long long nz, int depth, bool& col, long long& kz, int& chunk) {
  constexpr int XT = N / (2 * c2_lpc<N>());  // chunks per plane and phase
  const long long round = t / (2 * XT);
  const int within = (int)(t - round * 2 * XT);
  col = within >= XT;
  chunk = within - (col ? XT : 0);
  kz = col ? round - depth : round;
  return round < nz + depth;
}

// minimum CTAs per SM of the decoupled transforms: float halves the line
// buffers and the items' registers
template <int N, class T>
constexpr int q_minb() { return sizeof(T) == 8 ? ETC_Q64_MINB * 256 / c2_nt<N>() : ETC_Q32_MINB * 256 / c2_nt<N>(); }

template <int N, int MODE, class T = double>
__global__ void __launch_bounds__(c2_nt<N>(), q_minb<N, T>())
    k_fwd_q(Geom g, const T* src, T* dst, T* r, const T* q, Ctl* ctl, double* partials, unsigned* counter,
            PlaneTabsT<T> Tb, double* hist, T* pk, int nyl, QSched qs) {
  if (MODE != 0 && ctl->done) return;
  constexpr int LPC = c2_lpc<N>(), XT = N / (2 * LPC);
  extern __shared__ __align__(16) unsigned char smem_q[];
  const CtSmem<N, T> S = ct_carve<N, T>(reinterpret_cast<C2<T>*>(smem_q), Tb.twx, Tb.ex);
  const T alpha = (MODE == 2) ? (T)ctl->alpha : (T)0;
  double rr = 0.0;
  // float32: plain loads and stores (policy 0) instead of the L2 eviction
  // hints, in both transforms (fwd 0.514 -> 0.530, inv 0.597 -> 0.543 ms;
  // float64 keeps the hints: without them fwd 1.034 -> 1.063 ms)
  const unsigned long long PF = sizeof(T) == 4 ? 0ull : pol_first(), PL = sizeof(T) == 4 ? 0ull : pol_last();
  const long long total = (g.nz + qs.depth) * 2LL * XT;
  bool prev_col = true;
  for (long long t = blockIdx.x; t < total; t += gridDim.x) {
    bool col;
    long long kz;
    int chunk;
    q_task<N>(t, g.nz, qs.depth, col, kz, chunk);
    if (kz < 0 || kz >= g.nz) continue;
    const long long pb = kz * (long long)N * N;
    if (!col) {
      // after a column task (lines interleaved across the CTA) every warp must
      // be done with the line buffers; between row tasks each line is one
      // line group's own, so the warps drift apart (fwd_rows syncs the line)
      if (prev_col) __syncthreads();
      fwd_rows<N, MODE, T>(S, pb, chunk * 2 * LPC, src, dst, r, q, alpha, rr, PF, PL);
      q_publish<N>(qs, kz);
    } else {
      q_await(qs.cnt + kz, qs.target);
      fwd_cols<N, T>(S, g, kz, pb, chunk * 2 * LPC, dst, pk, nyl, nullptr, 0, PF);
    }
    prev_col = col;
  }
  fwd_finish<MODE, T>(rr, ctl, partials, counter, hist);
}

template <int N, bool PCG, int WM, class T = double>
__global__ void __launch_bounds__(c2_nt<N>(), q_minb<N, T>())
    k_inv_q(Geom g, const T* src, T* dst, const Ctl* ctl, PlaneTabsT<T> Tb, T* w, T* p, int p_plane, const T* pk,
            int nyl, QSched qs) {
  if (PCG && ctl->done) return;
  constexpr int LPC = c2_lpc<N>(), XT = N / (2 * LPC);
  const T beta = (WM == 2) ? (T)ctl->beta : (T)0, alpha = (WM == 2) ? (T)ctl->alpha : (T)0;
  extern __shared__ __align__(16) unsigned char smem_q[];
  const CtSmem<N, T> S = ct_carve<N, T>(reinterpret_cast<C2<T>*>(smem_q), Tb.twx, Tb.ex);
  // float32: plain loads and stores (see k_fwd_q)
  const unsigned long long PF = sizeof(T) == 4 ? 0ull : pol_first(), PL = sizeof(T) == 4 ? 0ull : pol_last();
  const int wpf = g_wpf;
  const long long total = (g.nz + qs.depth) * 2LL * XT;
  bool prev_col = true;
  for (long long t = blockIdx.x; t < total; t += gridDim.x) {
    bool col;
    long long kz;
    int chunk;
    q_task<N>(t, g.nz, qs.depth, col, kz, chunk);
    if (kz < 0 || kz >= g.nz) continue;
    const long long pb = kz * (long long)N * N;
    if (!col) {
      if (prev_col) __syncthreads();  // see k_fwd_q
      inv_rows<N, T>(S, g, kz, pb, chunk * 2 * LPC, src, dst, pk, nyl, PF, PL);
      q_publish<N>(qs, kz);
    } else {
      q_await(qs.cnt + kz, qs.target);
      inv_cols<N, WM, T>(S, kz, pb, chunk * 2 * LPC, dst, w, p, p_plane, alpha, beta, wpf, PF);
    }
    prev_col = col;
  }
}

// p += alpha w after the last iteration (the stencil of iteration k+1 applies
// iteration k's update; krylov.py:76)
__global__ void k_pupdate(long long n, double* __restrict__ p, const double* __restrict__ w, const Ctl* ctl) {
  const double alpha = ctl->alpha;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
    p[c] = __dadd_rn(p[c], __dmul_rn(alpha, w[c]));
}
