// etc_kernels.cuh — shared device definitions of the B200 ETC solver
// (sm_100a, float64): the local geometry (Geom), the device-resident PCG
// state (Ctl), complex helpers, the deterministic block / grid reductions
// with last-CTA finalisation, the small radix-2/4/8 DFTs and the runtime-size
// Stockham line FFT, and the thread-block cluster helpers.
//
// The kernels of one PCG iteration (reference krylov.py:70-90, Alg. 1) live
// in etc_stencil.cuh, etc_planes.cuh and etc_zsolve.cuh (included by
// etc_b200.cu; float instances for precision f32 in etc_f32.cuh):
//   k_stencil_pht / k_stencil_cp : q = A w (tpfa.py:110-131) and q.w, q.q, w.w
//   k_fwd_q (k_fwd_c2 on z-slab ranks with peer stores) : r -= alpha q, |r|^2,
//                 2-D DCT-II of r (transforms.py:83-104, Makhoul)
//   k_zsolve_tma : per-mode tridiagonal solve along z (preconditioner.py:215-250)
//                 with r.z by Parseval
//   k_inv_q (k_inv_c2) : 2-D DCT-III, w = z + beta w_old, p += alpha w_old
// Scalars (alpha, beta, rho, relres, breakdown state) never leave the device:
// the last CTA of every reducing kernel finalises them (deterministic order).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace etc {

constexpr int kThreads = 256;

// Local geometry.  Single-GPU: kg0 = 0, nzg = nz, jofs = 0, nyg = ny.  A z-slab
// rank holds planes [kg0, kg0+nz) of nzg (vectors that need neighbours carry
// one halo plane each side, addressed as local planes -1 and nz); a z-pencil
// holds all nzg planes of rows [jofs, jofs+ny) of nyg.
struct Geom {
  int nx, ny, nz;
  long long plane;  // nx*ny
  long long n;      // nx*ny*nz
  int kg0, nzg;     // global index of local plane 0, global plane count
  int jofs, nyg;    // global index of local row 0, global row count
};

// Device-resident PCG state (one per plan).
struct Ctl {
  double rho, alpha, beta, norm_b, rtol;
  double last_rz, last_qw, last_rr;
  int it, max_iter, done, status, bd_iter, bd_kind, converged, dist;
  // dist != 0: reducing kernels export their totals to xbuf (device, 8
  // doubles) instead of finalising; an all-reduce over ranks and k_finalize
  // complete the stage
  double* xbuf;
};

enum { BD_NONE = 0, BD_OPERATOR = 1, BD_NONFINITE = 2, BD_PRECOND = 3 };

// ---------------------------------------------------------------------------
// complex helpers (double2 for the float64 solve, float2 for precision f32)
// ---------------------------------------------------------------------------
template <class T>
struct Cx;
template <>
struct Cx<double> {
  using type = double2;
};
template <>
struct Cx<float> {
  using type = float2;
};
template <class T>
using C2 = typename Cx<T>::type;  // complex (or pair) of T

__device__ __forceinline__ double2 mkc(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ float2 mkc(float a, float b) { return make_float2(a, b); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * (s*i), s = +-1
__device__ __forceinline__ double2 cmul_si(double2 a, double s) { return make_double2(-s * a.y, s * a.x); }

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmul_si(float2 a, float s) { return make_float2(-s * a.y, s * a.x); }

// correctly rounded scalar ops in the reference's association order
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }

// position of source index i in the Makhoul even/odd reordering
// (evens ascending then odds descending; transforms.py:41-43)
__device__ __forceinline__ int makhoul_pos(int i, int n) { return (i & 1) ? n - ((i + 1) >> 1) : (i >> 1); }

// ---------------------------------------------------------------------------
// deterministic block + grid reductions with last-CTA finalisation
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lin_tid() { return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); }
__device__ __forceinline__ int lin_nthreads() { return blockDim.x * blockDim.y * blockDim.z; }

// Deterministic block sum (fixed shuffle tree); result valid in linear thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  const int tid = lin_tid();
  const int lane = tid & 31, warp = tid >> 5, nw = (lin_nthreads() + 31) >> 5;
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) sm[i * 32 + warp] = v[i];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = lane < nw ? sm[i * 32 + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < NV; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
}

// Every CTA contributes v; the last CTA to arrive reduces all partials in a
// fixed order and thread 0 calls fin(total).  Requires a 1-D grid index.
template <int NV, class F>
__device__ __forceinline__ void grid_sum_finalize(double (&v)[NV], double* partials, unsigned* counter, F fin) {
  __shared__ double sm[NV * 32];
  __shared__ bool last;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
  const int tid = lin_tid();
  block_sum<NV>(v, sm);
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) partials[(size_t)bid * NV + i] = v[i];
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    last = (prev == nb - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.0;
  for (unsigned b = tid; b < nb; b += lin_nthreads())
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] += __ldcg(partials + (size_t)b * NV + i);
  block_sum<NV>(acc, sm);
  if (tid == 0) {
    *counter = 0u;
    fin(acc);
  }
}

// ---------------------------------------------------------------------------
// shared-memory Stockham FFT over a batch of complex lines (radix 8/4/2),
// direct DFT for non-power-of-two lengths.  tw[m] = exp(-2 pi i m / N).
// s = -1 forward, +1 inverse (no 1/N).  Returns the buffer holding the result.
// ---------------------------------------------------------------------------
template <int R, class C, class S>
__device__ __forceinline__ void dft_small(C (&v)[R], S s) {
  if constexpr (R == 2) {
    C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    C t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    C t2 = cadd(v[1], v[3]), t3 = cmul_si(csub(v[1], v[3]), s);
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  } else {
    static_assert(R == 8, "radix 2, 4 or 8");
    const S h = (S)0.70710678118654752440;
    C u[4], d[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      u[m] = cadd(v[m], v[m + 4]);
      d[m] = csub(v[m], v[m + 4]);
    }
    // d[m] *= W^m, W = exp(s 2 pi i / 8)
    d[1] = mkc(h * (d[1].x - s * d[1].y), h * (d[1].y + s * d[1].x));
    d[2] = cmul_si(d[2], s);
    d[3] = mkc(-h * (d[3].x + s * d[3].y), h * (s * d[3].x - d[3].y));
    dft_small<4>(u, s);
    dft_small<4>(d, s);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[2 * q] = u[q];
      v[2 * q + 1] = d[q];
    }
  }
}

template <int R>
__device__ __forceinline__ void stockham_pass(const double2* __restrict__ src, double2* __restrict__ dst, int nlines,
                                              int N, int pitch, int Ns, const double2* __restrict__ tw, double s) {
  const int T = N / R;
  const int total = nlines * T;
  const int tstride = N / (Ns * R);
  for (int w = threadIdx.x; w < total; w += blockDim.x) {
    const int line = w / T;
    const int j = w - line * T;
    const int k = j & (Ns - 1);
    const int base = line * pitch;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[base + j + r * T];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 t = tw[(k * r * tstride) & (N - 1)];
        if (s > 0) t.y = -t.y;
        v[r] = cmul(v[r], t);
      }
    }
    dft_small<R>(v, s);
    const int idxD = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[base + idxD + r * Ns] = v[r];
  }
}

__device__ __forceinline__ double2* fft_lines(double2* A, double2* B, int nlines, int N, int pitch,
                                              const double2* __restrict__ tw, double s) {
  if (N == 1) return A;
  if (N & (N - 1)) {  // direct DFT, O(N^2): small / non-power-of-two lengths
    const int total = nlines * N;
    for (int w = threadIdx.x; w < total; w += blockDim.x) {
      const int line = w / N, kk = w - line * N, base = line * pitch;
      double2 acc = make_double2(0.0, 0.0);
      int idx = 0;
      for (int m = 0; m < N; ++m) {
        double2 t = tw[idx];
        if (s > 0) t.y = -t.y;
        acc = cadd(acc, cmul(A[base + m], t));
        idx += kk;
        if (idx >= N) idx -= N;
      }
      B[base + kk] = acc;
    }
    __syncthreads();
    return B;
  }
  double2* src = A;
  double2* dst = B;
  int Ns = 1;
  while (Ns < N) {
    const int rem = N / Ns;
    if (rem >= 8) {
      stockham_pass<8>(src, dst, nlines, N, pitch, Ns, tw, s);
      Ns *= 8;
    } else if (rem == 4) {
      stockham_pass<4>(src, dst, nlines, N, pitch, Ns, tw, s);
      Ns *= 4;
    } else {
      stockham_pass<2>(src, dst, nlines, N, pitch, Ns, tw, s);
      Ns *= 2;
    }
    __syncthreads();
    double2* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

// ---------------------------------------------------------------------------
// thread-block cluster helpers (sm_90+; B200 portable cluster size <= 8)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_nctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_id_x() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned ncluster_x() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// all threads of all CTAs of the cluster; release/acquire orders the global
// writes of one phase before the reads of the next
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace etc
