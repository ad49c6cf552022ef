// etc_f32.cuh — the single-precision path (homogenize(..., precision="f32"),
// /root/reference/pkg/src/etchomo/pipeline.py:147-160).  Included at the end of
// etc_b200.cu; selected per plan with etc_set_precision(plan, 32).
//
// What the reference does in f32 (and this file mirrors, op by op):
//   * the field is cast to float32 (pipeline.py:155), s = k / float32(h)**2
//     (tpfa.py:19-26), faces ((2a)b)/(a+b) and the Dirichlet layers 2 s_z in
//     float32 (tpfa.py:29-30, 102-107);
//   * apply_operator in float32 with the numpy association order
//     (tpfa.py:117-130);
//   * the FCT preconditioner: complex64 transforms (transforms.py:83-133),
//     plane shifts and z_diag computed in float64 then cast to float32, the
//     elimination in float32 (preconditioner.py:178-250);
//   * PCG vectors in float32; np.dot / np.linalg.norm return float32 values;
//     the scalars alpha, beta are Python floats cast back to float32 where they
//     scale a vector (krylov.py:56-90), eps = finfo(float32).eps.
// Dots are accumulated here in float64 and rounded to float32 (numpy's sdot
// accumulates in float32; the difference is float32 rounding, which the f32
// parity tolerance covers).
//
// Kernels are one-pass and simple: f32 halves the bytes of every vector, and
// this path is the reference's precision study, not the benchmark.  The 2-D
// transforms run as two line passes (x-lines, then y-lines / the reverse for
// the inverse), each a batch of pair-packed complex lines in shared memory
// (Stockham FFT, radix-4 stages, for power-of-two lengths; direct DFT otherwise); the z-solve
// is the reference's Thomas elimination, one thread per mode column, with the
// elimination coefficients in a scratch vector.

__device__ __forceinline__ float harm32(float a, float b) {
  return __fdiv_rn(__fmul_rn(__fmul_rn(2.0f, a), b), __fadd_rn(a, b));
}

// canonical cell c = (k*ny + j)*nx + i
struct Cell3 {
  int i, j, k;
};
__device__ __forceinline__ Cell3 cell3(const Geom& g, long long c) {
  Cell3 r;
  r.k = (int)(c / g.plane);
  const long long rem = c - (long long)r.k * g.plane;
  r.j = (int)(rem / g.nx);
  r.i = (int)(rem - (long long)r.j * g.nx);
  return r;
}

// faces along canonical axis a from the permuted conductivity kap (float64 as
// loaded): s = float32(k) / h2f, face between c and its + neighbour; on the
// z pass also t_in, t_out = 2 s_z on the two Dirichlet layers
__global__ void k32_faces(Geom g, int a, const double* __restrict__ kap, float h2f, float* __restrict__ face,
                          float* __restrict__ tb) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long step = a == 0 ? 1 : (a == 1 ? (long long)g.nx : g.plane);
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.n; c += stride) {
    const Cell3 p = cell3(g, c);
    const float s = __fdiv_rn((float)kap[c], h2f);
    const bool has = a == 0 ? p.i + 1 < g.nx : (a == 1 ? p.j + 1 < g.ny : p.k + 1 < g.nz);
    face[c] = has ? harm32(s, __fdiv_rn((float)kap[c + step], h2f)) : 0.0f;
    if (a == 2) {
      const long long col = c - (long long)p.k * g.plane;
      if (p.k == 0) tb[col] = __fmul_rn(2.0f, s);
      if (p.k == g.nz - 1) tb[g.plane + col] = __fmul_rn(2.0f, s);
    }
  }
}

// exact min/max of tx, ty, tz, t_in/2, t_out/2 (preconditioner.py:94-108);
// positive floats order like their bit patterns
__global__ void k32_stats(Geom g, const float* __restrict__ tx, const float* __restrict__ ty,
                          const float* __restrict__ tz, const float* __restrict__ tb, unsigned* __restrict__ mm) {
  unsigned lo[5], hi[5];
#pragma unroll
  for (int a = 0; a < 5; ++a) { lo[a] = 0x7f800000u; hi[a] = 0u; }
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.n; c += stride) {
    const Cell3 p = cell3(g, c);
    if (p.i + 1 < g.nx) { const unsigned v = __float_as_uint(tx[c]); lo[0] = min(lo[0], v); hi[0] = max(hi[0], v); }
    if (p.j + 1 < g.ny) { const unsigned v = __float_as_uint(ty[c]); lo[1] = min(lo[1], v); hi[1] = max(hi[1], v); }
    if (p.k + 1 < g.nz) { const unsigned v = __float_as_uint(tz[c]); lo[2] = min(lo[2], v); hi[2] = max(hi[2], v); }
    if (c < g.plane) {
      const unsigned vi = __float_as_uint(__fdiv_rn(tb[c], 2.0f));
      const unsigned vo = __float_as_uint(__fdiv_rn(tb[g.plane + c], 2.0f));
      lo[3] = min(lo[3], vi); hi[3] = max(hi[3], vi);
      lo[4] = min(lo[4], vo); hi[4] = max(hi[4], vo);
    }
  }
#pragma unroll
  for (int a = 0; a < 5; ++a) {
    const unsigned l = __reduce_min_sync(0xffffffffu, lo[a]), h = __reduce_max_sync(0xffffffffu, hi[a]);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(mm + 2 * a, l);
      atomicMax(mm + 2 * a + 1, h);
    }
  }
}

// b = t_in p_in on k = 0, += t_out p_out on k = nz-1 (tpfa.py:150-167); r = b,
// p = 0, ||b|| (krylov.py:57-68)
__global__ void k32_rhs(Geom g, const float* __restrict__ tb, float pin, float pout, float* __restrict__ r,
                        float* __restrict__ p, Ctl* ctl, double* partials, unsigned* counter, double* hist) {
  double rr = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.n; c += stride) {
    const long long k = c / g.plane, col = c - k * g.plane;
    float b = 0.0f;
    if (k == 0) b = __fmul_rn(tb[col], pin);
    if (k == g.nz - 1) b = __fadd_rn(b, __fmul_rn(tb[g.plane + col], pout));
    r[c] = b;
    p[c] = 0.0f;
    rr = fma((double)b, (double)b, rr);
  }
  double v[1] = {rr};
  grid_sum_finalize<1>(v, partials, counter, [&](double (&t)[1]) { fin_normb32(ctl, t[0], hist); });
}

// w = z + float32(beta) w_old (w = z on the first iteration), q = A w in the
// association order of tpfa.py:117-130, dots q.w, q.q, w.w -> alpha
template <bool FIRST>
__global__ void __launch_bounds__(256) k32_stencil(Geom g, int kchunk, const float* __restrict__ tx,
                                                   const float* __restrict__ ty, const float* __restrict__ tz,
                                                   const float* __restrict__ tb, const float* __restrict__ z,
                                                   const float* __restrict__ wold, float* __restrict__ wnew,
                                                   float* __restrict__ q, Ctl* ctl, double* partials,
                                                   unsigned* counter, int pcg) {
  if (pcg && ctl->done) return;
  const float bf = FIRST ? 0.0f : (float)ctl->beta;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long P = g.plane;
  auto W = [&](long long idx) -> float { return FIRST ? z[idx] : __fadd_rn(z[idx], __fmul_rn(bf, wold[idx])); };
  double dqw = 0.0, dqq = 0.0, dww = 0.0;
  // work item = (32x8 column tile, z chunk); each thread marches its column
  const int tx_n = (nx + 31) / 32, ty_n = (ny + 7) / 8, nch = (nz + kchunk - 1) / kchunk;
  const long long work = (long long)tx_n * ty_n * nch;
  for (long long wk = blockIdx.x; wk < work; wk += gridDim.x) {
    const int ch = (int)(wk / ((long long)tx_n * ty_n));
    const int tt = (int)(wk - (long long)ch * tx_n * ty_n);
    const int i = (tt % tx_n) * 32 + (threadIdx.x & 31), j = (tt / tx_n) * 8 + (threadIdx.x >> 5);
    if (i >= nx || j >= ny) continue;
    const int k0 = ch * kchunk, k1 = min(nz, k0 + kchunk);
    const long long col = (long long)j * nx + i;
    // the column's w and tz ride along z in registers (um, u, un; fzm)
    long long c = (long long)k0 * P + col;
    float um = k0 > 0 ? W(c - P) : 0.0f, fzm = k0 > 0 ? tz[c - P] : 0.0f;
    float u = W(c);
    for (int k = k0; k < k1; ++k, c += P) {
      const float un = k + 1 < nz ? W(c + P) : 0.0f;
      const float fz = tz[c];
      float acc = 0.0f;
      if (i > 0) acc = __fadd_rn(acc, __fmul_rn(tx[c - 1], __fsub_rn(u, W(c - 1))));
      if (i + 1 < nx) acc = __fsub_rn(acc, __fmul_rn(tx[c], __fsub_rn(W(c + 1), u)));
      if (j > 0) acc = __fadd_rn(acc, __fmul_rn(ty[c - nx], __fsub_rn(u, W(c - nx))));
      if (j + 1 < ny) acc = __fsub_rn(acc, __fmul_rn(ty[c], __fsub_rn(W(c + nx), u)));
      if (k > 0) acc = __fadd_rn(acc, __fmul_rn(fzm, __fsub_rn(u, um)));
      if (k + 1 < nz) acc = __fsub_rn(acc, __fmul_rn(fz, __fsub_rn(un, u)));
      if (k == 0) acc = __fadd_rn(acc, __fmul_rn(tb[col], u));
      if (k == nz - 1) acc = __fadd_rn(acc, __fmul_rn(tb[P + col], u));
      if (wnew) wnew[c] = u;
      q[c] = acc;
      dqw = fma((double)acc, (double)u, dqw);
      dqq = fma((double)acc, (double)acc, dqq);
      dww = fma((double)u, (double)u, dww);
      um = u;
      u = un;
      fzm = fz;
    }
  }
  if (!pcg) return;
  double v[3] = {dqw, dqq, dww};
  grid_sum_finalize<3>(v, partials, counter, [&](double (&t)[3]) { fin_stencil32(ctl, t[0], t[1], t[2]); });
}

// p += float32(alpha) w, r -= float32(alpha) q, ||r|| (krylov.py:76-84).
// homogenize observes p only through the outflow flux (tpfa.py:234-258), so
// p is updated from cell p0 on: the last plane (as the f64 path does).
__global__ void k32_update(long long n, long long p0, float* __restrict__ p, float* __restrict__ r,
                           const float* __restrict__ w, const float* __restrict__ q, Ctl* ctl, double* partials,
                           unsigned* counter, double* hist) {
  if (ctl->done) return;
  const float af = (float)ctl->alpha;
  double rr = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += stride) {
    if (c >= p0) p[c] = __fadd_rn(p[c], __fmul_rn(af, w[c]));
    const float v = __fsub_rn(r[c], __fmul_rn(af, q[c]));
    r[c] = v;
    rr = fma((double)v, (double)v, rr);
  }
  double v[1] = {rr};
  grid_sum_finalize<1>(v, partials, counter, [&](double (&t)[1]) { fin_update32(ctl, t[0], hist); });
}

// rho = r.z (krylov.py:65-67, 85-90) -> beta
__global__ void k32_rz(long long n, const float* __restrict__ r, const float* __restrict__ z, Ctl* ctl,
                       double* partials, unsigned* counter) {
  if (ctl->done) return;
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += stride)
    s = fma((double)r[c], (double)z[c], s);
  double v[1] = {s};
  grid_sum_finalize<1>(v, partials, counter, [&](double (&t)[1]) { fin_thomas(ctl, f32r(t[0])); });
}

__device__ __forceinline__ float2 c32mul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// One pass of 1-D transforms over the lines of every z-plane along axis AX
// (0: rows along x, 1: columns along y).  A CTA takes 2*LP neighbouring real
// lines of one plane, packed two per complex line.  INV = 0: DCT-II
// (transforms.py:83-104 per axis); INV = 1: the scaled DCT-III
// (transforms.py:108-133 per axis).  tw[m] = exp(-2 pi i m/N) (m < N),
// E[k] = (cos, sin)(pi k/2N): the tables of the float64 path, cast.
// LG > 0: N = 2^LG at compile time (index math in shifts, FFT stages
// unrolled); LG = 0: runtime length (radix-2 if a power of two, else DFT).
__host__ __device__ constexpr int f32_lp_of(int N) { return N >= 4096 ? 1 : (4096 / N > 32 ? 32 : 4096 / N); }

template <int AX, int INV, int LG>
__global__ void __launch_bounds__(256) k32_lines(Geom g, const float* src, float* dst, const float2* __restrict__ tw,
                                                 const float2* __restrict__ E, int LPrt, const Ctl* ctl, int pcg) {
  if (pcg && ctl->done) return;
  extern __shared__ float2 sm32[];
  const int N = LG ? (1 << LG) : (AX == 0 ? g.nx : g.ny);  // line length
  const int LP = LG ? f32_lp_of(1 << LG) : LPrt;
  const int PN = N + 1;                        // padded line pitch (float2)
  const int nl = AX == 0 ? g.ny : g.nx;        // lines per plane
  const int es = AX == 0 ? 1 : g.nx;           // element stride along a line (in-plane: 32-bit)
  const int ls = AX == 0 ? g.nx : 1;           // stride between neighbouring lines
  const bool pow2 = LG ? true : (N & (N - 1)) == 0;
  float2* A = sm32;
  float2* B = sm32 + (size_t)LP * PN;
  const int groups = (nl + 2 * LP - 1) / (2 * LP);
  const long long work = (long long)g.nz * groups;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nel = 2 * LP * N;
  for (long long wk = blockIdx.x; wk < work; wk += gridDim.x) {
    const long long kz = wk / groups;
    const int l0 = (int)(wk - kz * groups) * 2 * LP;
    const int nlines = min(2 * LP, nl - l0);
    const float* sp = src + kz * g.plane + l0 * ls;
    float* dp = dst + kz * g.plane + l0 * ls;
    // ---- load (coalesced: x-lines walk i fastest, y-lines walk the 2LP columns fastest)
    for (int e = tid; e < nel; e += nt) {
      int l, m;
      if (AX == 0) { l = e / N; m = e - l * N; } else { m = e / (2 * LP); l = e - m * (2 * LP); }
      const float v = l < nlines ? sp[l * ls + m * es] : 0.0f;
      if (!INV)  // Makhoul gather: evens ascending, odds descending (transforms.py:41-43)
        reinterpret_cast<float*>(&A[(l >> 1) * PN + makhoul_pos(m, N)])[l & 1] = v;
      else
        reinterpret_cast<float*>(&B[(l >> 1) * PN + m])[l & 1] = v;
    }
    __syncthreads();
    if (INV) {  // DCT-III pre-twiddle of both packed lines: Z = V1 + i V2 (dct3_pre)
      for (int e = tid; e < LP * N; e += nt) {
        const int f = e / N, kk = e - f * N;
        const float2 a = B[f * PN + kk];
        const float2 b = kk ? B[f * PN + N - kk] : make_float2(0.0f, 0.0f);
        const float2 Ek = E[kk];
        const float v1r = Ek.x * a.x + Ek.y * b.x, v1i = Ek.y * a.x - Ek.x * b.x;
        const float v2r = Ek.x * a.y + Ek.y * b.y, v2i = Ek.y * a.y - Ek.x * b.y;
        A[f * PN + kk] = make_float2(v1r - v2i, v1i + v2r);
      }
      __syncthreads();
    }
    // ---- FFT of the LP packed lines in A (natural order in and out);
    // tw is exp(-2 pi i m/N), the inverse uses its conjugate
    float2* Z = A;
    if (LG >= 2) {  // Stockham auto-sort, radix-4 stages (then one radix-2 if LG is odd), ping-pong A <-> B
      float2 *x = A, *y = B;
#pragma unroll
      for (int st = 0; st + 1 < LG; st += 2) {
        const int Ns = 1 << st;
        const int tstep = N / (4 * Ns);
        for (int e = tid; e < LP * (N / 4); e += nt) {
          const int f = e / (N / 4), j = e - f * (N / 4);
          const int k = j & (Ns - 1);
          float2 v[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            v[r] = x[f * PN + j + r * (N / 4)];
            if (r) {
              float2 w = tw[r * k * tstep];
              if (INV) w.y = -w.y;
              v[r] = c32mul(v[r], w);
            }
          }
          // 4-point DFT; forward uses -i, the inverse +i
          const float2 s02 = make_float2(v[0].x + v[2].x, v[0].y + v[2].y);
          const float2 d02 = make_float2(v[0].x - v[2].x, v[0].y - v[2].y);
          const float2 s13 = make_float2(v[1].x + v[3].x, v[1].y + v[3].y);
          const float2 d13 = make_float2(v[1].x - v[3].x, v[1].y - v[3].y);
          const float2 jd = INV ? make_float2(-d13.y, d13.x) : make_float2(d13.y, -d13.x);  // (+-i) d13
          const int d = f * PN + ((j - k) << 2) + k;
          y[d] = make_float2(s02.x + s13.x, s02.y + s13.y);
          y[d + Ns] = make_float2(d02.x + jd.x, d02.y + jd.y);
          y[d + 2 * Ns] = make_float2(s02.x - s13.x, s02.y - s13.y);
          y[d + 3 * Ns] = make_float2(d02.x - jd.x, d02.y - jd.y);
        }
        __syncthreads();
        float2* tmp = x; x = y; y = tmp;
      }
      if (LG & 1) {
        const int Ns = N / 2;
        for (int e = tid; e < LP * (N / 2); e += nt) {
          const int f = e / (N / 2), j = e - f * (N / 2);
          const int k = j & (Ns - 1);
          float2 w = tw[k];
          if (INV) w.y = -w.y;
          const float2 a = x[f * PN + j];
          const float2 t = c32mul(x[f * PN + j + N / 2], w);
          const int d = f * PN + ((j - k) << 1) + k;
          y[d] = make_float2(a.x + t.x, a.y + t.y);
          y[d + Ns] = make_float2(a.x - t.x, a.y - t.y);
        }
        __syncthreads();
        x = y;
      }
      Z = x;
    } else if (pow2) {  // radix-2 Stockham auto-sort, ping-pong A <-> B
      float2 *x = A, *y = B;
#pragma unroll
      for (int st = 0; st < (LG ? LG : 31); ++st) {
        const int Ns = 1 << st;
        if (!LG && Ns >= N) break;
        const int tstep = N / (2 * Ns);
        for (int e = tid; e < LP * (N / 2); e += nt) {
          const int f = e / (N / 2), j = e - f * (N / 2);
          const int k = j & (Ns - 1);
          float2 w = tw[k * tstep];
          if (INV) w.y = -w.y;
          const float2 a = x[f * PN + j];
          const float2 t = c32mul(x[f * PN + j + N / 2], w);
          const int d = f * PN + ((j - k) << 1) + k;
          y[d] = make_float2(a.x + t.x, a.y + t.y);
          y[d + Ns] = make_float2(a.x - t.x, a.y - t.y);
        }
        __syncthreads();
        float2* tmp = x; x = y; y = tmp;
      }
      Z = x;
    } else {  // direct DFT (non-power-of-two lengths)
      for (int e = tid; e < LP * N; e += nt) {
        const int f = e / N, kk = e - f * N;
        float2 acc = make_float2(0.0f, 0.0f);
        for (int m = 0; m < N; ++m) {
          float2 w = tw[(int)(((long long)m * kk) % N)];
          if (INV) w.y = -w.y;
          const float2 t = c32mul(A[f * PN + m], w);
          acc.x += t.x;
          acc.y += t.y;
        }
        B[f * PN + kk] = acc;
      }
      __syncthreads();
      Z = B;
    }
    // ---- store
    for (int e = tid; e < nel; e += nt) {
      int l, m;
      if (AX == 0) { l = e / N; m = e - l * N; } else { m = e / (2 * LP); l = e - m * (2 * LP); }
      if (l >= nlines) continue;
      float v;
      if (!INV) {  // DCT-II recombination of the packed spectra (dct2_out)
        const float2 a = Z[(l >> 1) * PN + m];
        const float2 b = Z[(l >> 1) * PN + (m ? N - m : 0)];
        const float2 Ek = E[m];
        v = (l & 1) ? 0.5f * (Ek.x * (a.y + b.y) - Ek.y * (a.x - b.x))
                    : 0.5f * (Ek.x * (a.x + b.x) + Ek.y * (a.y - b.y));
      } else {
        const float2 zz = Z[(l >> 1) * PN + makhoul_pos(m, N)];
        v = ((l & 1) ? zz.y : zz.x) / (float)N;
      }
      dp[l * ls + m * es] = v;
    }
    __syncthreads();
  }
}

// per-mode z elimination, one thread per (j', i') column, in the order of
// thomas_solve_batch (preconditioner.py:215-250); the shift is formed in
// float64 like TridiagFactors.plane_shift and cast (preconditioner.py:184-189)
__global__ void k32_thomas(Geom g, float* __restrict__ x, float* __restrict__ upper, const double* __restrict__ wx,
                           const double* __restrict__ wy, double kxr, double kyr, float zd0, float zdi, float zdl,
                           float off, const Ctl* ctl, int pcg) {
  if (pcg && ctl->done) return;
  const long long P = g.plane;
  const int nz = g.nz;
  for (long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x; col < P;
       col += (long long)gridDim.x * blockDim.x) {
    const int ip = (int)(col % g.nx), jp = (int)(col / g.nx);
    const float shift = (float)__dadd_rn(__dmul_rn(wx[ip], kxr), __dmul_rn(wy[jp], kyr));
    const float diag0 = __fadd_rn(zd0, shift);
    if (nz == 1) {
      x[col] = __fdiv_rn(x[col], diag0);
      continue;
    }
    float up = __fdiv_rn(off, diag0);
    upper[col] = up;
    float xp = __fdiv_rn(x[col], diag0);
    x[col] = xp;
    // rows are loaded D at a time ahead of the dependent elimination
    constexpr int D = 8;
    for (int k0 = 1; k0 < nz; k0 += D) {
      float xv[D];
#pragma unroll
      for (int u = 0; u < D; ++u) xv[u] = k0 + u < nz ? x[(long long)(k0 + u) * P + col] : 0.0f;
#pragma unroll
      for (int u = 0; u < D; ++u) {
        const int k = k0 + u;
        if (k >= nz) break;
        const long long c = (long long)k * P + col;
        const float denom = __fsub_rn(__fadd_rn(k == nz - 1 ? zdl : zdi, shift), __fmul_rn(off, up));
        if (k < nz - 1) {
          up = __fdiv_rn(off, denom);
          upper[c] = up;
        }
        xp = __fdiv_rn(__fsub_rn(xv[u], __fmul_rn(off, xp)), denom);
        x[c] = xp;
      }
    }
    for (int k0 = nz - 2; k0 >= 0; k0 -= D) {
      float xv[D], uv[D];
#pragma unroll
      for (int u = 0; u < D; ++u) {
        const long long c = (long long)(k0 - u) * P + col;
        xv[u] = k0 - u >= 0 ? x[c] : 0.0f;
        uv[u] = k0 - u >= 0 ? upper[c] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < D; ++u) {
        if (k0 - u < 0) break;
        xp = __fsub_rn(xv[u], __fmul_rn(uv[u], xp));
        x[(long long)(k0 - u) * P + col] = xp;
      }
    }
  }
}

// outflow flux t_out hz (p[nz-1] - p_out) per column in float32
// (tpfa.py:234-251), summed in float64 (tpfa.py:254-258)
__global__ void k32_flux(Geom g, const float* __restrict__ tb, const float* __restrict__ p, float hz, float pout,
                         double* out, double* partials, unsigned* counter) {
  double s = 0.0;
  const long long off = (long long)(g.nz - 1) * g.plane;
  for (long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x; col < g.plane;
       col += (long long)gridDim.x * blockDim.x)
    s += (double)__fmul_rn(__fmul_rn(tb[g.plane + col], hz), __fsub_rn(p[off + col], pout));
  double v[1] = {s};
  grid_sum_finalize<1>(v, partials, counter, [&](double (&t)[1]) { *out = t[0]; });
}

__global__ void k32_tabs(int n, const double2* __restrict__ src, float2* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = make_float2((float)src[i].x, (float)src[i].y);
}

// ---- float32 phase tables (the fused float32 solve's stencil).  The phase
// index is the float64 one (k_phase_index); its float32 scaled coefficient
// s = float32(k) / float32(h)^2 is written per phase by every cell of the
// phase, then every cell is checked against it, so a table is used only if it
// reproduces each float32 face of k32_faces bit for bit.
__global__ void k32_phase_s(long long n, const double* __restrict__ kap, float h2f,
                            const unsigned char* __restrict__ idx, float* __restrict__ stab) {
  // each CTA gathers its phases' values in shared memory and writes each once
  // (every cell storing to the same PH_MAX global words serialises on them)
  __shared__ float sv[PH_MAX];
  __shared__ int seen[PH_MAX];
  if (threadIdx.x < PH_MAX) seen[threadIdx.x] = 0;
  __syncthreads();
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const int p = idx[c];
    if (!seen[p]) {
      sv[p] = __fdiv_rn((float)kap[c], h2f);
      seen[p] = 1;
    }
  }
  __syncthreads();
  if (threadIdx.x < PH_MAX && seen[threadIdx.x]) stab[threadIdx.x] = sv[threadIdx.x];
}
__global__ void k32_phase_check(long long n, const double* __restrict__ kap, float h2f,
                                const unsigned char* __restrict__ idx, const float* __restrict__ stab,
                                int* __restrict__ bad) {
  bool b = false;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
    b |= stab[idx[c]] != __fdiv_rn((float)kap[c], h2f);
  if (b) atomicExch(bad, 1);
}
// faces [ax][a * PH_MAX + b] = harm32(s_a, s_b) (lower cell a, as k32_faces),
// tb[p] = 2 s_z
__global__ void k32_phase_ftab(const float* __restrict__ stab, int m, float* __restrict__ ftab) {
  for (int e = threadIdx.x; e < PH_MAX * PH_MAX; e += blockDim.x) {
    const int a = e / PH_MAX, b = e % PH_MAX;
    const bool ok = a < m && b < m;
    for (int ax = 0; ax < 3; ++ax)
      ftab[ax * PH_MAX * PH_MAX + e] = ok ? harm32(stab[ax * PH_MAX + a], stab[ax * PH_MAX + b]) : 0.0f;
  }
  for (int q = threadIdx.x; q < PH_MAX; q += blockDim.x)
    ftab[3 * PH_MAX * PH_MAX + q] = q < m ? __fmul_rn(2.0f, stab[2 * PH_MAX + q]) : 0.0f;
}

// Jacobi in float32 (JacobiPreconditioner, preconditioner.py:324-329): 1/diag(A)
// in operator_diagonal's accumulation order (tpfa.py:134-147) and an IEEE
// float32 1/d; z = r * (1/diag) with rho = r.z in the same pass
__global__ void k32_jacobi_diag(Geom g, const float* __restrict__ tx, const float* __restrict__ ty,
                                const float* __restrict__ tz, const float* __restrict__ tb, float* __restrict__ invd) {
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long P = g.plane;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.n; c += (long long)gridDim.x * blockDim.x) {
    const long long k = c / P, rem = c - k * P;
    const int j = (int)(rem / nx), i = (int)(rem - (long long)j * nx);
    float d = 0.0f;
    if (i > 0) d = __fadd_rn(d, tx[c - 1]);
    if (i + 1 < nx) d = __fadd_rn(d, tx[c]);
    if (j > 0) d = __fadd_rn(d, ty[c - nx]);
    if (j + 1 < ny) d = __fadd_rn(d, ty[c]);
    if (k > 0) d = __fadd_rn(d, tz[c - P]);
    if (k + 1 < nz) d = __fadd_rn(d, tz[c]);
    if (k == 0) d = __fadd_rn(d, tb[rem]);
    if (k == nz - 1) d = __fadd_rn(d, tb[P + rem]);
    invd[c] = __fdiv_rn(1.0f, d);
  }
}
__global__ void k32_jacobi_rz(long long n, const float* __restrict__ r, const float* __restrict__ invd,
                              float* __restrict__ z, Ctl* ctl, double* partials, unsigned* counter) {
  if (ctl->done) return;
  double s = 0.0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const float v = __fmul_rn(r[c], invd[c]);
    z[c] = v;
    s = fma((double)r[c], (double)v, s);
  }
  double v[1] = {s};
  grid_sum_finalize<1>(v, partials, counter, [&](double (&t)[1]) { fin_thomas(ctl, f32r(t[0])); });
}

// p += float32(alpha) w after the last iteration (krylov.py:76)
__global__ void k32_pupdate(long long n, float* __restrict__ p, const float* __restrict__ w, const Ctl* ctl) {
  const float af = (float)ctl->alpha;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
    p[c] = __fadd_rn(p[c], __fmul_rn(af, w[c]));
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int f32_alloc(etc_plan* pl, float** v, size_t count) {
  double* d = nullptr;
  int rc = dev_alloc(pl, &d, (count + 1) / 2);
  *v = reinterpret_cast<float*>(d);
  return rc;
}

static int f32_buffers(etc_plan* pl) {
  if (pl->v32[0]) return ETC_OK;
  const size_t n = (size_t)pl->n;
  int rc;
  for (int b = 0; b < 10; ++b)  // tx ty tz | p r q z w0 w1 | (unused)
    if (b < 9 && (rc = f32_alloc(pl, &pl->v32[b], n))) return rc;
  if ((rc = f32_alloc(pl, &pl->tb32, 2 * (size_t)pl->nx * pl->ny))) return rc;
  if ((rc = f32_alloc(pl, reinterpret_cast<float**>(&pl->ctab32), 8 * (size_t)pl->maxd))) return rc;
  return ETC_OK;
}

// float32 faces of the current direction from the loaded field
static int f32_faces(etc_plan* pl) {
  if (pl->slab) return fail(ETC_CONFIG, "precision f32 runs on single-GPU plans");
  int rc;
  if ((rc = f32_buffers(pl))) return rc;
  int comp[3] = {0, 1, 2};
  if (pl->axis == 0) { comp[0] = 2; comp[1] = 1; comp[2] = 0; }
  if (pl->axis == 1) { comp[0] = 0; comp[1] = 2; comp[2] = 1; }
  const double h[3] = {pl->lx / pl->nx, pl->ly / pl->ny, pl->lz / pl->nz};
  const Geom g = geom(pl);
  const bool ph = pl->nph > 0 && pl->fast32;
  pl->ph32_ok = false;
  if (ph && !pl->ftab32) {
    if ((rc = f32_alloc(pl, &pl->ftab32, 3 * PH_MAX * PH_MAX + PH_MAX))) return rc;
    if ((rc = f32_alloc(pl, &pl->stab32, 4 * PH_MAX))) return rc;
  }
  int* bad = reinterpret_cast<int*>(pl->stab32 + 3 * PH_MAX);
  if (ph) CK(cudaMemsetAsync(bad, 0, sizeof(int), pl->stream));
  for (int a = 0; a < 3; ++a) {
    // the permuted conductivity (scale 1) into the f64 scratch z, then faces
    if ((rc = scale_into(pl, pl->raw[comp[a]], 1.0, pl->z))) return rc;
    const float hf = (float)h[a];
    const float h2f = hf * hf;  // dtype(h)**2 in float32 (tpfa.py:23-25)
    Tm tm(pl, 6);
    k32_faces<<<grid1d(pl, pl->n), 256, 0, pl->stream>>>(g, a, pl->z, h2f, pl->v32[a], pl->tb32);
    CK(cudaGetLastError());
    if (ph) {
      k32_phase_s<<<grid1d(pl, pl->n), 256, 0, pl->stream>>>(pl->n, pl->z, h2f, pl->pidx, pl->stab32 + a * PH_MAX);
      k32_phase_check<<<grid1d(pl, pl->n), 256, 0, pl->stream>>>(pl->n, pl->z, h2f, pl->pidx,
                                                                  pl->stab32 + a * PH_MAX, bad);
      CK(cudaGetLastError());
    }
  }
  if (ph) {
    k32_phase_ftab<<<1, 256, 0, pl->stream>>>(pl->stab32, pl->nph, pl->ftab32);
    CK(cudaGetLastError());
    int hb = 1;
    CK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    pl->ph32_ok = hb == 0;
  }
  pl->faces32_ok = true;
  return ETC_OK;
}

static int f32_stats(etc_plan* pl, double out[10]) {
  int rc;
  if (!pl->faces32_ok && (rc = f32_faces(pl))) return rc;
  unsigned init[10];
  for (int a = 0; a < 5; ++a) { init[2 * a] = 0x7f800000u; init[2 * a + 1] = 0u; }
  unsigned* mm = reinterpret_cast<unsigned*>(pl->scal);
  CK(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, pl->stream));
  {
    Tm tm(pl, 6);
    k32_stats<<<grid1d(pl, pl->n), 256, 0, pl->stream>>>(geom(pl), pl->v32[0], pl->v32[1], pl->v32[2], pl->tb32, mm);
    CK(cudaGetLastError());
  }
  unsigned res[10];
  CK(cudaMemcpyAsync(res, mm, sizeof(res), cudaMemcpyDeviceToHost, pl->stream));
  CK(cudaStreamSynchronize(pl->stream));
  for (int i = 0; i < 10; ++i) {
    float f;
    std::memcpy(&f, &res[i], sizeof(f));
    out[i] = (double)f;
  }
  if (pl->nx < 2) { out[0] = 1.0; out[1] = 1.0; }
  if (pl->ny < 2) { out[2] = 1.0; out[3] = 1.0; }
  if (pl->nz < 2) { out[4] = 1.0; out[5] = 1.0; }
  return ETC_OK;
}

// line batch size: about 4096 packed complex elements (32 KB) per pass
static int f32_lp(int N) { return f32_lp_of(std::max(1, N)); }

template <int AX, int INV>
static int f32_pass(etc_plan* pl, const float* src, float* dst, int pcg) {
  const Geom g = geom(pl);
  const int N = AX == 0 ? pl->nx : pl->ny, nl = AX == 0 ? pl->ny : pl->nx;
  const int LP = f32_lp(N);
  const size_t smem = 2 * (size_t)LP * (N + 1) * sizeof(float2);
  auto kern = k32_lines<AX, INV, 0>;
  switch (N) {
    case 16: kern = k32_lines<AX, INV, 4>; break;
    case 32: kern = k32_lines<AX, INV, 5>; break;
    case 64: kern = k32_lines<AX, INV, 6>; break;
    case 128: kern = k32_lines<AX, INV, 7>; break;
    case 256: kern = k32_lines<AX, INV, 8>; break;
    case 512: kern = k32_lines<AX, INV, 9>; break;
    case 1024: kern = k32_lines<AX, INV, 10>; break;
    default: break;
  }
  int rc;
  if (smem > 48 * 1024 && (rc = prep_smem(kern, smem))) return rc;
  const long long work = (long long)pl->nz * ((nl + 2 * LP - 1) / (2 * LP));
  const int grid = (int)std::min<long long>(work, (long long)pl->sms * 8);
  const float2* T = pl->ctab32;
  const int M = pl->maxd;
  const float2* tw = AX == 0 ? T : T + M;
  const float2* E = AX == 0 ? T + 2 * M : T + 3 * M;
  Tm tm(pl, INV ? 5 : 2);
  kern<<<grid, 256, smem, pl->stream>>>(g, src, dst, tw, E, LP, pl->ctl, pcg);
  CK(cudaGetLastError());
  return ETC_OK;
}

// z = M^-1 r: forward 2-D DCT of r into t, the z elimination (its
// coefficients in the scratch z), inverse 2-D DCT of t into z
static int f32_precond(etc_plan* pl, const float* r, float* t, float* z, int pcg) {
  int rc;
  if ((rc = f32_pass<0, 0>(pl, r, t, pcg))) return rc;
  if ((rc = f32_pass<1, 0>(pl, t, t, pcg))) return rc;
  {
    const Geom g = geom(pl);
    const int M = pl->maxd;
    Tm tm(pl, 3);
    k32_thomas<<<grid1d(pl, g.plane, 128), 128, 0, pl->stream>>>(
        g, t, z, pl->tabs, pl->tabs + M, pl->refs[0], pl->refs[1], (float)pl->zd3[0], (float)pl->zd3[1],
        (float)pl->zd3[2], (float)(-pl->refs[2]), pl->ctl, pcg);
    CK(cudaGetLastError());
  }
  if ((rc = f32_pass<1, 1>(pl, t, z, pcg))) return rc;
  return f32_pass<0, 1>(pl, z, z, pcg);
}

static int f32_set_reference(etc_plan* pl) {
  int rc;
  if ((rc = f32_buffers(pl))) return rc;
  const int n = 4 * pl->maxd;
  k32_tabs<<<(n + 255) / 256, 256, 0, pl->stream>>>(n, pl->ctab, pl->ctab32);
  CK(cudaGetLastError());
  return ETC_OK;
}

// ---------------------------------------------------------------------------
// the fused float32 solve: the float64 solve's kernels instantiated on float
// (square power-of-two planes, N >= 128, nz = 32 L with L in {4, 8, 16}):
//   k_stencil_pht<N, true, float> (float32 phase tables; k32_stencil with
//     stored float32 faces when the field has more phases): q = A w, dots;
//   k_fwd_q<N, 2, float>: r -= float32(alpha) q, |r|^2, 2-D DCT-II of r;
//   k_zsolve_tma<L, float>: the z elimination on the float32 spectrum with
//     the reference's float32 coefficients, pivots and sweeps in float64
//     registers, r.z by Parseval;
//   k_inv_q<N, true, 2, float>: 2-D DCT-III, w = z + float32(beta) w_old and
//     p += float32(alpha) w_old on the outflow plane.
// The transforms compute in float32 (complex64, as the reference's
// precision study), with the float32 twiddle tables of the line passes.
// ---------------------------------------------------------------------------
static bool fast32_ok(etc_plan* pl) {
  if (!pl->fast32 || pl->precond != ETC_PRECOND_FCT || pl->slab || pl->generic_fft || !pl->qplanes || !pl->ztma)
    return false;
  const Geom g = geom(pl);
  const int N = ct_size(g);
  if (N < 128 || !c2_ok(pl, ct_cfg(pl, g), N)) return false;
  const int Lz = pl->Lz;
  return pl->Qz == 32 && Lz * 32 == g.nz && (Lz == 4 || Lz == 8 || Lz == 16 || (Lz == 32 && pl->z1024tma)) &&
         g.plane % 2 == 0;
}

static PlaneTabsT<float> tabs32(const etc_plan* pl) {
  const int M = pl->maxd;
  PlaneTabsT<float> T;
  T.twx = pl->ctab32;
  T.twy = pl->ctab32 + M;
  T.ex = pl->ctab32 + 2 * M;
  T.ey = pl->ctab32 + 3 * M;
  return T;
}

template <int MODE>
static int f32_fwd(const Launch& L, const float* src, float* dst, float* r, const float* q, unsigned* counter) {
  etc_plan* pl = L.pl;
  Tm tm(pl, MODE == 2 ? 1 : (MODE == 1 ? 6 : 2));
  const PlaneTabsT<float> T = tabs32(pl);
#define ETC_F32_FWD(NN)                                                                                      \
  case NN:                                                                                                   \
    return launch_q<NN, float>(L, k_fwd_q<NN, MODE, float>, L.g, src, dst, r, q, pl->ctl, pl->partials,      \
                               counter, T, pl->hist, (float*)nullptr, 0);
  switch (ct_size(L.g)) {
    ETC_F32_FWD(128)
    ETC_F32_FWD(256)
    ETC_F32_FWD(512)
    ETC_F32_FWD(1024)
  }
#undef ETC_F32_FWD
  return fail(ETC_CONFIG, "fused f32 transform: unsupported plane");
}

template <int WM>
static int f32_inv_w(const Launch& L, const float* src, float* scratch, float* w, float* p) {
  etc_plan* pl = L.pl;
  Tm tm(pl, 5);
  const PlaneTabsT<float> T = tabs32(pl);
  const int p_plane = pl->full_solution ? -1 : L.g.nz - 1;
#define ETC_F32_INV(NN)                                                                                         \
  case NN:                                                                                                      \
    return launch_q<NN, float>(L, k_inv_q<NN, true, WM, float>, L.g, src, scratch, (const Ctl*)pl->ctl, T, w, p, \
                               p_plane, (const float*)nullptr, 0);
  switch (ct_size(L.g)) {
    ETC_F32_INV(128)
    ETC_F32_INV(256)
    ETC_F32_INV(512)
    ETC_F32_INV(1024)
  }
#undef ETC_F32_INV
  return fail(ETC_CONFIG, "fused f32 inverse: unsupported plane");
}

template <int LZ, int TC = ZT_C>
static int f32_zsolve_n(const Launch& L, float* t, unsigned* counter) {
  etc_plan* pl = L.pl;
  const Geom& g = L.g;
  auto enc = tensor_map_encoder();
  if (!enc) return fail(ETC_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)g.plane, (cuuint64_t)g.nz};
  cuuint64_t strides[1] = {(cuuint64_t)g.plane * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)TC, (cuuint32_t)std::min(g.nz, 256)}, es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, t, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return fail(ETC_CUDA, "z-solve tensor map");
  auto kern = k_zsolve_tma<LZ, float, TC>;
  const size_t smem = zt_smem_bytes<LZ, float, TC>();
  int rc;
  if ((rc = prep_smem(kern, smem))) return rc;
  const long long tiles = (g.plane + TC - 1) / TC;
  const int grid = (int)std::max(1LL, std::min(tiles, (long long)pl->sms));
  // the reference's float32 z_diag and off-diagonal (preconditioner.py:178-199)
  auto f = [](double v) { return (double)(float)v; };
  Tm tm(pl, 3);
  kern<<<grid, TC * 32 + 32, smem, pl->stream>>>(g, map, L.wx, L.wy, f(pl->zd3[0]), f(pl->zd3[1]), f(pl->zd3[2]), pl->refs[0],
                                        pl->refs[1], f(-pl->refs[2]), pl->ctl, pl->partials, counter, 1);
  CK(cudaGetLastError());
  return ETC_OK;
}

static int f32_zsolve(const Launch& L, float* t, unsigned* counter) {
  switch (L.pl->Lz) {
    case 4: return f32_zsolve_n<4>(L, t, counter);
    case 8: return f32_zsolve_n<8>(L, t, counter);
    case 16: return f32_zsolve_n<16>(L, t, counter);
    case 32: return f32_zsolve_n<32, 8>(L, t, counter);  // nz = 1024: 8-column tiles
  }
  return fail(ETC_CONFIG, "fused f32 z-solve: unsupported z chunk");
}

// q = A w: the float32 phase tables through the TMA-staged stencil, or the
// stored float32 faces (k32_stencil with w as its direction)
static int f32_stencil_w(const Launch& L, const float* w, float* q, unsigned* counter) {
  etc_plan* pl = L.pl;
  const Geom& g = L.g;
  Tm tm(pl, 0);
  if (pl->nph > 0 && pl->ph32_ok) {
    const bool r4 = pl->phry == 4 && g.nx >= 256;  // 32-row tiles, four rows per thread
    const int RH = r4 ? 32 : 16;
    CUtensorMap mw, mi;
    if (plane_map(&mw, w, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.nx, g.nz, PhaseStageTmaT<float>::WX, RH + 2) &&
        plane_map(&mi, pl->pidx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.nx, g.nz, 64, RH + 2)) {
      const int bx = g.nx / 32, by = g.ny / RH;
      int ks = (int)std::max(1LL, std::min<long long>(g.nz, (2LL * 1024 + bx * by - 1) / (bx * by)));
      const int kchunk = (g.nz + ks - 1) / ks;
      ks = (g.nz + kchunk - 1) / kchunk;
      dim3 grid(bx, by, ks), block(32, 8);
      const size_t sm = ph_ft_bytes<float>() +
                        4 * (r4 ? sizeof(PhaseStageTma34f) : sizeof(PhaseStageTmaT<float>)) +
                        4 * sizeof(unsigned long long);
#define ETC_F32_PHT(NN)                                                                                        \
  case NN: {                                                                                                   \
    auto kern = r4 ? (pl->phcons ? k_stencil_pht<NN, true, float, 4, true> : k_stencil_pht<NN, true, float, 4>) \
                   : k_stencil_pht<NN, true, float>;                                                          \
    int rc_;                                                                                                   \
    if ((rc_ = prep_smem(kern, sm))) return rc_;                                                               \
    kern<<<grid, block, sm, pl->stream>>>(                                                                     \
        g, kchunk, mw, mi, pl->pidx, pl->ftab32, w, q, pl->ctl, pl->partials, counter);                       \
    CK(cudaGetLastError());                                                                                    \
    return ETC_OK;                                                                                             \
  }
      switch (g.nx) {
        ETC_F32_PHT(128)
        ETC_F32_PHT(256)
        ETC_F32_PHT(512)
        ETC_F32_PHT(1024)
      }
#undef ETC_F32_PHT
    }
  }
  if (pl->gen_tma) {  // stored float32 faces through the TMA ring (k_stencil_gt on float)
    constexpr int WX = GenStageTmaT<float>::WX;
    CUtensorMap mw, mx, my, mt;
    if (plane_map(&mw, w, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.nx, g.nz, WX, 18) &&
        plane_map(&mx, pl->v32[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.nx, g.nz, WX, 18) &&
        plane_map(&my, pl->v32[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.nx, g.nz, WX, 18) &&
        plane_map(&mt, pl->v32[2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.nx, g.nz, WX, 18)) {
      const int bx = g.nx / 32, by = g.ny / 16;
      int ks = (int)std::max(1LL, std::min<long long>(g.nz, (2LL * 1024 + bx * by - 1) / (bx * by)));
      const int kchunk = (g.nz + ks - 1) / ks;
      ks = (g.nz + kchunk - 1) / kchunk;
      dim3 grid(bx, by, ks), block(32, 8);
      const size_t sm = 4 * sizeof(GenStageTmaT<float>) + 4 * sizeof(unsigned long long);
#define ETC_F32_GT(NN)                                                                                        \
  case NN: {                                                                                                  \
    auto kern = k_stencil_gt<NN, true, float>;                                                                \
    int rc_;                                                                                                  \
    if ((rc_ = prep_smem(kern, sm))) return rc_;                                                              \
    kern<<<grid, block, sm, pl->stream>>>(g, kchunk, mw, mx, my, mt, w, pl->v32[2], pl->tb32, q, pl->ctl,    \
                                          pl->partials, counter);                                            \
    CK(cudaGetLastError());                                                                                   \
    return ETC_OK;                                                                                            \
  }
      switch (g.nx) {
        ETC_F32_GT(128)
        ETC_F32_GT(256)
        ETC_F32_GT(512)
        ETC_F32_GT(1024)
      }
#undef ETC_F32_GT
    }
  }
  const long long tiles = (long long)((pl->nx + 31) / 32) * ((pl->ny + 7) / 8);
  const int nch = (int)std::max(1LL, std::min<long long>(pl->nz, (long long)pl->sms * 8 / std::max(1LL, tiles)));
  const int kch = (pl->nz + nch - 1) / nch;
  const int GS = (int)std::min<long long>(tiles * ((pl->nz + kch - 1) / kch), (long long)pl->sms * 8);
  k32_stencil<true><<<GS, 256, 0, pl->stream>>>(g, kch, pl->v32[0], pl->v32[1], pl->v32[2], pl->tb32, w, nullptr,
                                                 nullptr, q, pl->ctl, pl->partials, counter, 1);
  CK(cudaGetLastError());
  return ETC_OK;
}

// Alg. 1 on the fused float32 kernels, the float64 solve's stage order
// (etc_solve): ||b|| and the spectrum of r, z-solve, w = z; then per
// iteration q = A w, r / |r| / spectrum, z-solve / r.z, w and p
static int solve32_fused(etc_plan* pl, double p_in, double p_out, double rtol, int max_iter, etc_solve_info* info,
                         double* hist_host) {
  Launch L = mk(pl);
  const Geom& g = L.g;
  float *p = pl->v32[3], *r = pl->v32[4], *q = pl->v32[5], *z = pl->v32[6], *w = pl->v32[7];
  Ctl c;
  std::memset(&c, 0, sizeof(c));
  c.rtol = rtol;
  c.max_iter = max_iter;
  CK(cudaMemcpyAsync(pl->ctl, &c, sizeof(c), cudaMemcpyHostToDevice, pl->stream));
  CK(cudaMemsetAsync(pl->counters, 0, 64 * sizeof(unsigned), pl->stream));
  int rc;
  {
    Tm tm(pl, 6);
    k32_rhs<<<grid1d(pl, pl->n), 256, 0, pl->stream>>>(g, pl->tb32, (float)p_in, (float)p_out, r, p, pl->ctl,
                                                       pl->partials, pl->counters + 3, pl->hist);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(pl->ev0, pl->stream));
  // iteration 0: ||b||, z = M r, rho = r.z, w = z (krylov.py:56-68)
  if ((rc = f32_fwd<1>(L, r, q, nullptr, nullptr, pl->counters + 1))) return rc;
  if ((rc = f32_zsolve(L, q, pl->counters + 2))) return rc;
  if ((rc = f32_inv_w<1>(L, q, z, w, p))) return rc;
  int it = 0;
  bool done = false;
  while (!done && it < max_iter) {
    const int batch = std::min(pl->check_every, max_iter - it);
    for (int b = 0; b < batch; ++b, ++it) {
      if ((rc = f32_stencil_w(L, w, q, pl->counters + 0))) return rc;
      if ((rc = f32_fwd<2>(L, nullptr, q, r, q, pl->counters + 1))) return rc;
      if ((rc = f32_zsolve(L, q, pl->counters + 2))) return rc;
      if ((rc = f32_inv_w<2>(L, q, z, w, p))) return rc;
    }
    CK(cudaMemcpyAsync(pl->ctl_host, pl->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    done = pl->ctl_host->done != 0;
  }
  CK(cudaMemcpyAsync(pl->ctl_host, pl->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, pl->stream));
  CK(cudaStreamSynchronize(pl->stream));
  const Ctl& h = *pl->ctl_host;
  if (h.it >= 1 && !h.status) {  // iteration it's pending p += alpha w
    Tm tm(pl, 6);
    const long long off = pl->full_solution ? 0 : (long long)(pl->nz - 1) * g.plane;
    const long long cnt = pl->full_solution ? pl->n : g.plane;
    k32_pupdate<<<grid1d(pl, cnt), 256, 0, pl->stream>>>(cnt, p + off, w + off, pl->ctl);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(pl->ev1, pl->stream));
  float ms = 0.f;
  CK(cudaEventSynchronize(pl->ev1));
  cudaEventElapsedTime(&ms, pl->ev0, pl->ev1);
  std::memset(info, 0, sizeof(*info));
  info->iterations = h.it;
  info->converged = h.converged;
  info->status = h.status ? ETC_BREAKDOWN : ETC_OK;
  info->breakdown_iter = h.bd_iter;
  info->breakdown_kind = h.bd_kind;
  info->norm_b = h.norm_b;
  info->device_ms = ms;
  if (hist_host) CK(cudaMemcpy(hist_host, pl->hist, (size_t)(h.it + 1) * sizeof(double), cudaMemcpyDeviceToHost));
  if (h.status) return fail(ETC_BREAKDOWN, "PCG breakdown");
  {
    Tm tm(pl, 6);
    const float hzf = (float)(pl->lz / pl->nz);
    k32_flux<<<grid1d(pl, g.plane, 256, 2), 256, 0, pl->stream>>>(g, pl->tb32, p, hzf, (float)p_out, pl->scal + 20,
                                                                  pl->partials, pl->counters + 3);
    CK(cudaGetLastError());
  }
  double fs = 0.0;
  CK(cudaMemcpyAsync(&fs, pl->scal + 20, sizeof(double), cudaMemcpyDeviceToHost, pl->stream));
  CK(cudaStreamSynchronize(pl->stream));
  info->flux_sum = fs;
  info->kappa_eff = pl->lz * fs / ((double)pl->nx * pl->ny * (p_in - p_out));
  return ETC_OK;
}

static int solve32(etc_plan* pl, double p_in, double p_out, double rtol, int max_iter, etc_solve_info* info,
                   double* hist_host) {
  int rc;
  if (!pl->faces32_ok && (rc = f32_faces(pl))) return rc;
  if ((rc = f32_set_reference(pl))) return rc;
  if (fast32_ok(pl)) return solve32_fused(pl, p_in, p_out, rtol, max_iter, info, hist_host);
  const Geom g = geom(pl);
  float *tx = pl->v32[0], *ty = pl->v32[1], *tz = pl->v32[2];
  float *p = pl->v32[3], *r = pl->v32[4], *q = pl->v32[5], *z = pl->v32[6];
  float* w[2] = {pl->v32[7], pl->v32[8]};
  const bool none = pl->precond == ETC_PRECOND_NONE, jac = pl->precond == ETC_PRECOND_JACOBI;
  const int G_ = grid1d(pl, pl->n);
  if (jac) {
    if (!pl->invd32 && (rc = f32_alloc(pl, &pl->invd32, (size_t)pl->n))) return rc;
    Tm tm(pl, 6);
    k32_jacobi_diag<<<grid1d(pl, pl->n), 256, 0, pl->stream>>>(geom(pl), tx, ty, tz, pl->tb32, pl->invd32);
    CK(cudaGetLastError());
  }
  // z = M r and rho = r.z (fct: the line passes and the z elimination, then r.z)
  auto precond_rz = [&]() -> int {
    if (jac) {
      k32_jacobi_rz<<<G_, 256, 0, pl->stream>>>(pl->n, r, pl->invd32, z, pl->ctl, pl->partials, pl->counters + 2);
      CK(cudaGetLastError());
      return ETC_OK;
    }
    int rc_;
    if (!none && (rc_ = f32_precond(pl, r, q, z, 1))) return rc_;
    k32_rz<<<G_, 256, 0, pl->stream>>>(pl->n, r, none ? r : z, pl->ctl, pl->partials, pl->counters + 2);
    CK(cudaGetLastError());
    return ETC_OK;
  };
  Ctl c;
  std::memset(&c, 0, sizeof(c));
  c.rtol = rtol;
  c.max_iter = max_iter;
  CK(cudaMemcpyAsync(pl->ctl, &c, sizeof(c), cudaMemcpyHostToDevice, pl->stream));
  CK(cudaMemsetAsync(pl->counters, 0, 64 * sizeof(unsigned), pl->stream));
  CK(cudaEventRecord(pl->ev0, pl->stream));
  const int G = grid1d(pl, pl->n);
  // stencil: 32x8 column tiles x z chunks, about 8 CTAs per SM
  const long long tiles = (long long)((pl->nx + 31) / 32) * ((pl->ny + 7) / 8);
  const int nch = (int)std::max(1LL, std::min<long long>(pl->nz, (long long)pl->sms * 8 / std::max(1LL, tiles)));
  const int kch = (pl->nz + nch - 1) / nch;
  const int GS = (int)std::min<long long>(tiles * ((pl->nz + kch - 1) / kch), (long long)pl->sms * 8);
  {
    Tm tm(pl, 6);
    k32_rhs<<<G, 256, 0, pl->stream>>>(g, pl->tb32, (float)p_in, (float)p_out, r, p, pl->ctl, pl->partials,
                                       pl->counters + 1, pl->hist);
    CK(cudaGetLastError());
  }
  // iteration 0: z = M r, rho = r.z (krylov.py:63-68)
  const float* zv = none ? r : z;
  if ((rc = precond_rz())) return rc;
  int it = 0;
  bool done = false;
  while (!done && it < max_iter) {
    const int batch = std::min(pl->check_every, max_iter - it);
    for (int b = 0; b < batch; ++b) {
      ++it;
      float* wn = w[it & 1];
      const float* wo = w[(it - 1) & 1];
      {
        Tm tm(pl, 0);
        if (it == 1)
          k32_stencil<true><<<GS, 256, 0, pl->stream>>>(g, kch, tx, ty, tz, pl->tb32, zv, nullptr, wn, q, pl->ctl,
                                                        pl->partials, pl->counters + 0, 1);
        else
          k32_stencil<false><<<GS, 256, 0, pl->stream>>>(g, kch, tx, ty, tz, pl->tb32, zv, wo, wn, q, pl->ctl,
                                                         pl->partials, pl->counters + 0, 1);
        CK(cudaGetLastError());
      }
      {
        Tm tm(pl, 1);
        k32_update<<<G, 256, 0, pl->stream>>>(pl->n, (long long)(pl->nz - 1) * g.plane, p, r, wn, q, pl->ctl,
                                              pl->partials, pl->counters + 1, pl->hist);
        CK(cudaGetLastError());
      }
      if ((rc = precond_rz())) return rc;
    }
    CK(cudaMemcpyAsync(pl->ctl_host, pl->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    done = pl->ctl_host->done != 0;
  }
  CK(cudaEventRecord(pl->ev1, pl->stream));
  CK(cudaMemcpyAsync(pl->ctl_host, pl->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, pl->stream));
  CK(cudaStreamSynchronize(pl->stream));
  const Ctl& h = *pl->ctl_host;
  float ms = 0.f;
  CK(cudaEventSynchronize(pl->ev1));
  cudaEventElapsedTime(&ms, pl->ev0, pl->ev1);
  std::memset(info, 0, sizeof(*info));
  info->iterations = h.it;
  info->converged = h.converged;
  info->status = h.status ? ETC_BREAKDOWN : ETC_OK;
  info->breakdown_iter = h.bd_iter;
  info->breakdown_kind = h.bd_kind;
  info->norm_b = h.norm_b;
  info->device_ms = ms;
  if (hist_host) CK(cudaMemcpy(hist_host, pl->hist, (size_t)(h.it + 1) * sizeof(double), cudaMemcpyDeviceToHost));
  if (h.status) return fail(ETC_BREAKDOWN, "PCG breakdown");
  {
    Tm tm(pl, 6);
    const float hzf = (float)(pl->lz / pl->nz);
    k32_flux<<<grid1d(pl, g.plane, 256, 2), 256, 0, pl->stream>>>(g, pl->tb32, p, hzf, (float)p_out, pl->scal + 20,
                                                                  pl->partials, pl->counters + 3);
    CK(cudaGetLastError());
  }
  double fs = 0.0;
  CK(cudaMemcpyAsync(&fs, pl->scal + 20, sizeof(double), cudaMemcpyDeviceToHost, pl->stream));
  CK(cudaStreamSynchronize(pl->stream));
  info->flux_sum = fs;
  info->kappa_eff = pl->lz * fs / ((double)pl->nx * pl->ny * (p_in - p_out));
  return ETC_OK;
}

extern "C" int etc_set_precision(etc_plan* pl, int bits) {
  if (!pl) return fail(ETC_CONFIG, "null plan");
  if (bits != 32 && bits != 64) return fail(ETC_CONFIG, "precision must be 32 or 64 bits");
  if (bits == 32 && pl->slab) return fail(ETC_CONFIG, "precision f32 runs on single-GPU plans");
  pl->prec32 = bits == 32;
  return ETC_OK;
}

// ---- float32 operator-plugin entry points (the reference's FctPlan /
// FctPreconditioner with dtype=float32, transforms.py:56-61 and
// preconditioner.py:273-282): the same line passes and elimination as the
// f32 solve, on caller vectors.  Need etc_set_reference (field or bare plan).
static int f32_tabs_ready(etc_plan* pl) {
  if (!pl || !pl->have_axis) return fail(ETC_CONFIG, "select an axis first");
  if (!pl->have_ref) return fail(ETC_CONFIG, "set the reference first");
  if (pl->slab) return fail(ETC_CONFIG, "precision f32 runs on single-GPU plans");
  return f32_set_reference(pl);
}

extern "C" int etc_dct2_xy_f32(etc_plan* pl, const float* in, float* out) {
  int rc;
  if ((rc = f32_tabs_ready(pl))) return rc;
  if ((rc = f32_pass<0, 0>(pl, in, out, 0))) return rc;
  return f32_pass<1, 0>(pl, out, out, 0);
}

extern "C" int etc_dct3_xy_f32(etc_plan* pl, const float* in, float* out) {
  int rc;
  if ((rc = f32_tabs_ready(pl))) return rc;
  if ((rc = f32_pass<1, 1>(pl, in, out, 0))) return rc;
  return f32_pass<0, 1>(pl, out, out, 0);
}

extern "C" int etc_apply_precond_f32(etc_plan* pl, const float* r, float* z) {
  int rc;
  if ((rc = f32_tabs_ready(pl))) return rc;
  if (r == z) return fail(ETC_CONFIG, "etc_apply_precond_f32 needs distinct input and output");
  return f32_precond(pl, r, pl->v32[5], z, 0);
}
