// etc_plugin.cu — stateless device kernels behind the reference's
// operator-plugin layer (etchomo tpfa / preconditioner / krylov functions,
// /root/reference/pkg/src/etchomo/__init__.py:9-71).  Unlike the plan-based
// entry points of etc_b200.cu (one field, fused solve), these take the
// reference's own data structures as plain device arrays — the compact face
// arrays of a DiscreteSystem (tpfa.py:33-88), the TridiagFactors tables
// (preconditioner.py:167-212), bare vectors for pcg (krylov.py:36-91) — so any
// system a caller builds (reference_system, hand-made faces) runs on the GPU.
// Every entry point is stream-ordered, takes `prec` (0 float64, 1 float32:
// the reference threads the field dtype through every array) and follows the
// reference's per-element operation order with no FMA contraction, so the
// elementwise results are bitwise numpy's.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstring>
#include <string>

#include "../../include/etc_b200.h"

namespace {

// exact IEEE operations of the element type (no contraction)
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float div_(float a, float b) { return __fdiv_rn(a, b); }

constexpr int NT = 256;

int g_sms = 0;
int nblocks(long long work, int per_sm = 8) {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  long long b = (work + NT - 1) / NT;
  if (b > (long long)g_sms * per_sm) b = (long long)g_sms * per_sm;
  return (int)(b < 1 ? 1 : b);
}

// ---- stencil q = A u over compact faces (apply_operator, tpfa.py:110-131):
// per cell, in numpy's accumulation order: +x(i-1/2) -x(i+1/2) +y(j-1/2)
// -y(j+1/2) +z(k-1/2) -z(k+1/2) (each flux t*(u_hi - u_lo)), then the
// Dirichlet layers t_in*u (k = 0) and t_out*u (k = nz-1).
template <class T>
__global__ void k_op_stencil(int nx, int ny, int nz, const T* __restrict__ tx, const T* __restrict__ ty,
                             const T* __restrict__ tz, const T* __restrict__ tin, const T* __restrict__ tout,
                             const T* __restrict__ u, T* __restrict__ out) {
  const long long n = (long long)nx * ny * nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % nx);
    const long long kj = c / nx;
    const int j = (int)(kj % ny), k = (int)(kj / ny);
    const T v = u[c];
    T acc = T(0);
    if (i > 0) acc = add_(acc, mul_(tx[kj * (nx - 1) + i - 1], sub_(v, u[c - 1])));
    if (i < nx - 1) acc = sub_(acc, mul_(tx[kj * (nx - 1) + i], sub_(u[c + 1], v)));
    const long long fy = ((long long)k * (ny - 1) + j) * nx + i;
    if (j > 0) acc = add_(acc, mul_(ty[fy - nx], sub_(v, u[c - nx])));
    if (j < ny - 1) acc = sub_(acc, mul_(ty[fy], sub_(u[c + nx], v)));
    const long long P = (long long)nx * ny, pc = c - (long long)k * P;
    if (k > 0) acc = add_(acc, mul_(tz[c - P], sub_(v, u[c - P])));
    if (k < nz - 1) acc = sub_(acc, mul_(tz[c], sub_(u[c + P], v)));
    if (k == 0) acc = add_(acc, mul_(tin[pc], v));
    if (k == nz - 1) acc = add_(acc, mul_(tout[pc], v));
    out[c] = acc;
  }
}

// ---- diagonal of the stencil (operator_diagonal, tpfa.py:134-147):
// d[:,:,1:] += tx; d[:,:,:-1] += tx; (y, z likewise); d[0] += t_in; d[-1] += t_out
template <class T>
__global__ void k_op_diag(int nx, int ny, int nz, const T* __restrict__ tx, const T* __restrict__ ty,
                          const T* __restrict__ tz, const T* __restrict__ tin, const T* __restrict__ tout,
                          T* __restrict__ out) {
  const long long n = (long long)nx * ny * nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % nx);
    const long long kj = c / nx;
    const int j = (int)(kj % ny), k = (int)(kj / ny);
    const long long P = (long long)nx * ny, pc = c - (long long)k * P;
    const long long fy = ((long long)k * (ny - 1) + j) * nx + i;
    T d = T(0);
    if (i > 0) d = add_(d, tx[kj * (nx - 1) + i - 1]);
    if (i < nx - 1) d = add_(d, tx[kj * (nx - 1) + i]);
    if (j > 0) d = add_(d, ty[fy - nx]);
    if (j < ny - 1) d = add_(d, ty[fy]);
    if (k > 0) d = add_(d, tz[c - P]);
    if (k < nz - 1) d = add_(d, tz[c]);
    if (k == 0) d = add_(d, tin[pc]);
    if (k == nz - 1) d = add_(d, tout[pc]);
    out[c] = d;
  }
}

// ---- compact faces from the scaled coefficient cubes (build_system,
// tpfa.py:91-107): t = ((2 a) b)/(a + b) with a the lower cell, t_in/t_out = 2 s_z
template <class T>
__global__ void k_op_faces(int nx, int ny, int nz, const T* __restrict__ sx, const T* __restrict__ sy,
                           const T* __restrict__ sz, T* __restrict__ tx, T* __restrict__ ty, T* __restrict__ tz,
                           T* __restrict__ tin, T* __restrict__ tout) {
  const long long n = (long long)nx * ny * nz, P = (long long)nx * ny;
  const T two = T(2);
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % nx);
    const long long kj = c / nx;
    const int j = (int)(kj % ny), k = (int)(kj / ny);
    if (i < nx - 1) {
      const T a = sx[c], b = sx[c + 1];
      tx[kj * (nx - 1) + i] = div_(mul_(mul_(two, a), b), add_(a, b));
    }
    if (j < ny - 1) {
      const T a = sy[c], b = sy[c + nx];
      ty[((long long)k * (ny - 1) + j) * nx + i] = div_(mul_(mul_(two, a), b), add_(a, b));
    }
    if (k < nz - 1) {
      const T a = sz[c], b = sz[c + P];
      tz[c] = div_(mul_(mul_(two, a), b), add_(a, b));
    }
    if (k == 0) tin[c] = mul_(two, sz[c]);
    if (k == nz - 1) tout[c - (long long)k * P] = mul_(two, sz[c]);
  }
}

// ---- s = k / h^2 (scale_field, tpfa.py:19-26; a division, as numpy's)
template <class T>
__global__ void k_op_scale(long long n, const T* __restrict__ k, T h2, T* __restrict__ s) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
    s[c] = div_(k[c], h2);
}

// ---- axis permutation of one (nz, ny, nx) cube (axis_permute, pipeline.py:87-111):
// axis 0 (x): swapaxes(0, 2) -> (nx, ny, nz); axis 1 (y): swapaxes(0, 1) -> (ny, nz, nx)
template <class T>
__global__ void k_op_permute(int nx, int ny, int nz, int axis, const T* __restrict__ src, T* __restrict__ dst) {
  const long long n = (long long)nx * ny * nz;
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n; d += (long long)gridDim.x * blockDim.x) {
    long long s;
    if (axis == 0) {  // dst[i][j][k] (shape nx, ny, nz) = src[k][j][i]
      const int k = (int)(d % nz);
      const long long r = d / nz;
      const int j = (int)(r % ny), i = (int)(r / ny);
      s = ((long long)k * ny + j) * nx + i;
    } else {  // dst[j][k][i] (shape ny, nz, nx) = src[k][j][i]
      const int i = (int)(d % nx);
      const long long r = d / nx;
      const int k = (int)(r % nz), j = (int)(r / nz);
      s = ((long long)k * ny + j) * nx + i;
    }
    dst[d] = src[s];
  }
}

// ---- right-hand side (build_rhs, tpfa.py:150-167): b = 0; b[0] = t_in * p_in;
// b[-1] += t_out * p_out (p_in / p_out: scalars or (ny, nx) planes)
template <class T>
__global__ void k_op_rhs(int nx, int ny, int nz, const T* __restrict__ tin, const T* __restrict__ tout,
                         const T* __restrict__ pin_a, T pin, const T* __restrict__ pout_a, T pout, T* __restrict__ b) {
  const long long n = (long long)nx * ny * nz, P = (long long)nx * ny;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const long long k = c / P, pc = c - k * P;
    T v = T(0);
    if (k == 0) v = mul_(tin[pc], pin_a ? pin_a[pc] : pin);
    if (k == nz - 1) v = add_(v, mul_(tout[pc], pout_a ? pout_a[pc] : pout));
    b[c] = v;
  }
}

// ---- Dirichlet-face fluxes (reconstruct_boundary_flux, tpfa.py:234-251):
// out: (t_out hz)(u[-1] - p_out); in: (t_in hz)(p_in - u[0])
template <class T>
__global__ void k_op_flux(int nx, int ny, int nz, const T* __restrict__ t, T hz, const T* __restrict__ u, T pval,
                          int side_out, T* __restrict__ out) {
  const long long P = (long long)nx * ny;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < P; c += (long long)gridDim.x * blockDim.x) {
    const T th = mul_(t[c], hz);
    out[c] = side_out ? mul_(th, sub_(u[(long long)(nz - 1) * P + c], pval)) : mul_(th, sub_(pval, u[c]));
  }
}

// ---- batched Thomas along z (thomas_solve_batch, preconditioner.py:215-250),
// one thread per (j', i') column, elementwise the reference's vectorised
// elimination: upper[0] = off/d0, x0 /= d0; denom = (z_diag[k] + shift) -
// off*upper[k-1], upper[k] = off/denom, x[k] = (x[k] - off x[k-1])/denom;
// back substitution x[k] -= upper[k] x[k+1].  A non-positive pivot records
// its layer (the smallest over columns) for the host's FloatingPointError.
template <class T>
__global__ void k_op_thomas(int nx, int ny, int nz, const T* __restrict__ shift, const T* __restrict__ zdiag, T off,
                            T* __restrict__ x, T* __restrict__ upper, int* __restrict__ bad) {
  const long long P = (long long)nx * ny;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < P; c += (long long)gridDim.x * blockDim.x) {
    const T sh = shift[c];
    const T d0 = add_(zdiag[0], sh);
    if (d0 <= T(0)) {  // (NaN passes, as np.any(diag0 <= 0) lets it)
      atomicMin(bad, 0);
      continue;
    }
    if (nz == 1) {
      x[c] = div_(x[c], d0);
      continue;
    }
    T up = div_(off, d0);
    upper[c] = up;
    T xp = div_(x[c], d0);
    x[c] = xp;
    for (int k = 1; k < nz; ++k) {
      const T den = sub_(add_(zdiag[k], sh), mul_(off, up));
      if (den <= T(0)) {
        atomicMin(bad, k);
        break;
      }
      if (k < nz - 1) {
        up = div_(off, den);
        upper[(long long)k * P + c] = up;
      }
      xp = div_(sub_(x[(long long)k * P + c], mul_(off, xp)), den);
      x[(long long)k * P + c] = xp;
    }
    for (int k = nz - 2; k >= 0; --k) {
      xp = sub_(x[(long long)k * P + c], mul_(upper[(long long)k * P + c], xp));
      x[(long long)k * P + c] = xp;
    }
  }
}

// ---- elementwise products: out = a * b (Jacobi r * inv_diag), out = 1 / a
template <class T>
__global__ void k_op_mul(long long n, const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
    out[c] = mul_(a[c], b[c]);
}
template <class T>
__global__ void k_op_recip(long long n, const T* __restrict__ a, T* __restrict__ out) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
    out[c] = div_(T(1), a[c]);
}
template <class T>
__global__ void k_op_add(long long n, const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
    out[c] = add_(a[c], b[c]);
}

// ---- deterministic reductions (fixed grid, fixed tree, accumulated in
// float64 whatever the element type): per-block partials, then one block
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int NV>
__device__ __forceinline__ void block_sums(double (&v)[NV], double* out) {
  __shared__ double sm[NV][NT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) sm[i][w] = v[i];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double t = lane < NT / 32 ? sm[i][lane] : 0.0;
      t = warp_sum(t);
      if (lane == 0) out[i] = t;
    }
  }
}
template <int NV>
__global__ void k_op_final(int nparts, const double* __restrict__ parts, double* __restrict__ out) {
  double v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = 0.0;
  for (int b = threadIdx.x; b < nparts; b += NT)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += parts[(size_t)b * NV + i];
  block_sums<NV>(v, out);
}

// dots of two vectors: kind 0: (a.b), 1: (a.b, a.a, b.b), 2: (sum a)
template <class T, int KIND>
__global__ void k_op_dots(long long n, const T* __restrict__ a, const T* __restrict__ b, double* __restrict__ parts) {
  constexpr int NV = KIND == 1 ? 3 : 1;
  double v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = 0.0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const double x = (double)a[c];
    if (KIND == 2) {
      v[0] += x;
    } else {
      const double y = (double)b[c];
      v[0] = fma(x, y, v[0]);
      if (KIND == 1) {
        v[1] = fma(x, x, v[1]);
        v[2] = fma(y, y, v[2]);
      }
    }
  }
  block_sums<NV>(v, parts + (size_t)blockIdx.x * NV);
}

// pcg update (krylov.py:76-77): p += dtype(alpha) w; r -= dtype(alpha) z; -> r.r
template <class T>
__global__ void k_op_pcg_update(long long n, T alpha, T* __restrict__ p, const T* __restrict__ w, T* __restrict__ r,
                                const T* __restrict__ z, double* __restrict__ parts) {
  double v[1] = {0.0};
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    p[c] = add_(p[c], mul_(alpha, w[c]));
    const T rv = sub_(r[c], mul_(alpha, z[c]));
    r[c] = rv;
    v[0] = fma((double)rv, (double)rv, v[0]);
  }
  block_sums<1>(v, parts + blockIdx.x);
}

// w = z + dtype(beta) w (krylov.py:89)
template <class T>
__global__ void k_op_xpby(long long n, const T* __restrict__ z, T beta, T* __restrict__ w) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
    w[c] = add_(z[c], mul_(beta, w[c]));
}

// exact min / max (coefficient_stats, preconditioner.py:94-108): positive
// finite values order like their bit patterns
template <class T>
__global__ void k_op_minmax(long long n, const T* __restrict__ a, unsigned long long* __restrict__ mm) {
  double lo = INFINITY, hi = -INFINITY;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const double x = (double)a[c];
    lo = fmin(lo, x);
    hi = fmax(hi, x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0 && lo <= hi) {  // warps that saw no element stay out
    atomicMin(&mm[0], (unsigned long long)__double_as_longlong(lo));
    atomicMax(&mm[1], (unsigned long long)__double_as_longlong(hi));
  }
}

// dense matrix of the stencil (assemble_dense, tpfa.py:181-205; oracle
// sizes only): diagonal accumulated in np.add.at's order (x faces as the
// left then the right cell, y and z likewise, then the Dirichlet sum)
__global__ void k_op_dense(int nx, int ny, int nz, const double* __restrict__ tx, const double* __restrict__ ty,
                           const double* __restrict__ tz, const double* __restrict__ tin,
                           const double* __restrict__ tout, double* __restrict__ mat) {
  const long long n = (long long)nx * ny * nz, P = (long long)nx * ny;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % nx);
    const long long kj = c / nx;
    const int j = (int)(kj % ny), k = (int)(kj / ny);
    const long long fy = ((long long)k * (ny - 1) + j) * nx + i;
    double d = 0.0;
    // x: couple(idx[:,:,:-1] (left), idx[:,:,1:] (right))
    if (i < nx - 1) { const double t = tx[kj * (nx - 1) + i]; d = __dadd_rn(d, t); mat[c * n + c + 1] = -t; }
    if (i > 0) { const double t = tx[kj * (nx - 1) + i - 1]; d = __dadd_rn(d, t); mat[c * n + c - 1] = -t; }
    // y: couple(idx[:,1:,:] (left), idx[:,:-1,:] (right))
    if (j > 0) { const double t = ty[fy - nx]; d = __dadd_rn(d, t); mat[c * n + c - nx] = -t; }
    if (j < ny - 1) { const double t = ty[fy]; d = __dadd_rn(d, t); mat[c * n + c + nx] = -t; }
    // z: couple(idx[1:] (left), idx[:-1] (right))
    if (k > 0) { const double t = tz[c - P]; d = __dadd_rn(d, t); mat[c * n + c - P] = -t; }
    if (k < nz - 1) { const double t = tz[c]; d = __dadd_rn(d, t); mat[c * n + c + P] = -t; }
    double bnd = 0.0;
    if (k == 0) bnd = __dadd_rn(bnd, tin[c - (long long)k * P]);
    if (k == nz - 1) bnd = __dadd_rn(bnd, tout[c - (long long)k * P]);
    mat[c * n + c] = __dadd_rn(d, bnd);
  }
}

// ---- SSOR apply (SsorPreconditioner.__call__, preconditioner.py:285-321),
// float64: y = (L + D/w)^-1 r; y *= diag; y = (U + D/w)^-1 y; y *= (2-w)/w,
// with L / U the strict triangles of the stencil in natural (x-fastest)
// order.  A cell's lower neighbours (c-1, c-nx, c-P) lie on the previous
// hyperplane i+j+k, so each sweep is level-scheduled over hyperplanes inside
// one CTA (a verification baseline, not a hot kernel).
__global__ void __launch_bounds__(1024) k_op_ssor(int nx, int ny, int nz, const double* __restrict__ tx,
                                                   const double* __restrict__ ty, const double* __restrict__ tz,
                                                   const double* __restrict__ diag, double omega,
                                                   const double* __restrict__ r, double* __restrict__ y) {
  const long long P = (long long)nx * ny;
  const int S = nx + ny + nz - 2;
  const long long lines = (long long)ny * nz;
  for (int s = 0; s < S; ++s) {  // forward: (L + D/w) y = r
    for (long long e = threadIdx.x; e < lines; e += blockDim.x) {
      const int j = (int)(e % ny), k = (int)(e / ny), i = s - j - k;
      if (i < 0 || i >= nx) continue;
      const long long c = (long long)k * P + (long long)j * nx + i;
      double v = r[c];
      if (k > 0) v = __dadd_rn(v, __dmul_rn(tz[c - P], y[c - P]));
      if (j > 0) v = __dadd_rn(v, __dmul_rn(ty[((long long)k * (ny - 1) + j - 1) * nx + i], y[c - nx]));
      if (i > 0) v = __dadd_rn(v, __dmul_rn(tx[((long long)k * ny + j) * (nx - 1) + i - 1], y[c - 1]));
      y[c] = __ddiv_rn(v, __ddiv_rn(diag[c], omega));
    }
    __syncthreads();
  }
  for (long long c = threadIdx.x; c < P * nz; c += blockDim.x) y[c] = __dmul_rn(y[c], diag[c]);
  __syncthreads();
  for (int s = S - 1; s >= 0; --s) {  // backward: (U + D/w) y' = y
    for (long long e = threadIdx.x; e < lines; e += blockDim.x) {
      const int j = (int)(e % ny), k = (int)(e / ny), i = s - j - k;
      if (i < 0 || i >= nx) continue;
      const long long c = (long long)k * P + (long long)j * nx + i;
      double v = y[c];
      if (k < nz - 1) v = __dadd_rn(v, __dmul_rn(tz[c], y[c + P]));
      if (j < ny - 1) v = __dadd_rn(v, __dmul_rn(ty[((long long)k * (ny - 1) + j) * nx + i], y[c + nx]));
      if (i < nx - 1) v = __dadd_rn(v, __dmul_rn(tx[((long long)k * ny + j) * (nx - 1) + i], y[c + 1]));
      y[c] = __ddiv_rn(v, __ddiv_rn(diag[c], omega));
    }
    __syncthreads();
  }
  const double sc = (2.0 - omega) / omega;
  for (long long c = threadIdx.x; c < P * nz; c += blockDim.x) y[c] = __dmul_rn(y[c], sc);
}

thread_local std::string g_perr;
int perr(int code, const std::string& m) {
  g_perr = m;
  return code;
}
#define PCK(x)                                                                            \
  do {                                                                                    \
    cudaError_t e__ = (x);                                                                \
    if (e__ != cudaSuccess) return perr(ETC_CUDA, std::string(#x) + ": " + cudaGetErrorString(e__)); \
  } while (0)

// reductions: parts must hold nblocks(n) * 3 doubles
int reduce_finish(int nb, int nv, double* parts, double* out, cudaStream_t st) {
  if (nv == 1)
    k_op_final<1><<<1, NT, 0, st>>>(nb, parts, out);
  else
    k_op_final<3><<<1, NT, 0, st>>>(nb, parts, out);
  PCK(cudaGetLastError());
  return ETC_OK;
}

}  // namespace

extern "C" {

const char* etc_op_last_error(void) { return g_perr.c_str(); }

int etc_op_reduce_parts(long long n) { return nblocks(n) * 3 + 8; }

int etc_op_stencil(int prec, int nx, int ny, int nz, const void* tx, const void* ty, const void* tz, const void* tin,
                   const void* tout, const void* u, void* out, void* stream) {
  if (nx < 1 || ny < 1 || nz < 1) return perr(ETC_CONFIG, "grid dimensions must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks((long long)nx * ny * nz);
  if (prec == 0)
    k_op_stencil<double><<<grid, NT, 0, st>>>(nx, ny, nz, (const double*)tx, (const double*)ty, (const double*)tz,
                                             (const double*)tin, (const double*)tout, (const double*)u, (double*)out);
  else
    k_op_stencil<float><<<grid, NT, 0, st>>>(nx, ny, nz, (const float*)tx, (const float*)ty, (const float*)tz,
                                            (const float*)tin, (const float*)tout, (const float*)u, (float*)out);
  PCK(cudaGetLastError());
  return ETC_OK;
}

int etc_op_diagonal(int prec, int nx, int ny, int nz, const void* tx, const void* ty, const void* tz,
                    const void* tin, const void* tout, void* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks((long long)nx * ny * nz);
  if (prec == 0)
    k_op_diag<double><<<grid, NT, 0, st>>>(nx, ny, nz, (const double*)tx, (const double*)ty, (const double*)tz,
                                          (const double*)tin, (const double*)tout, (double*)out);
  else
    k_op_diag<float><<<grid, NT, 0, st>>>(nx, ny, nz, (const float*)tx, (const float*)ty, (const float*)tz,
                                         (const float*)tin, (const float*)tout, (float*)out);
  PCK(cudaGetLastError());
  return ETC_OK;
}

int etc_op_faces(int prec, int nx, int ny, int nz, const void* sx, const void* sy, const void* sz, void* tx,
                 void* ty, void* tz, void* tin, void* tout, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks((long long)nx * ny * nz);
  if (prec == 0)
    k_op_faces<double><<<grid, NT, 0, st>>>(nx, ny, nz, (const double*)sx, (const double*)sy, (const double*)sz,
                                           (double*)tx, (double*)ty, (double*)tz, (double*)tin, (double*)tout);
  else
    k_op_faces<float><<<grid, NT, 0, st>>>(nx, ny, nz, (const float*)sx, (const float*)sy, (const float*)sz,
                                          (float*)tx, (float*)ty, (float*)tz, (float*)tin, (float*)tout);
  PCK(cudaGetLastError());
  return ETC_OK;
}

int etc_op_scale(int prec, long long n, const void* k, double h2, void* s, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks(n);
  if (prec == 0)
    k_op_scale<double><<<grid, NT, 0, st>>>(n, (const double*)k, h2, (double*)s);
  else
    k_op_scale<float><<<grid, NT, 0, st>>>(n, (const float*)k, (float)h2, (float*)s);
  PCK(cudaGetLastError());
  return ETC_OK;
}

int etc_op_permute(int prec, int nx, int ny, int nz, int axis, const void* src, void* dst, void* stream) {
  if (axis != 0 && axis != 1) return perr(ETC_CONFIG, "axis must be 0 (x) or 1 (y)");
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks((long long)nx * ny * nz);
  if (prec == 0)
    k_op_permute<double><<<grid, NT, 0, st>>>(nx, ny, nz, axis, (const double*)src, (double*)dst);
  else
    k_op_permute<float><<<grid, NT, 0, st>>>(nx, ny, nz, axis, (const float*)src, (float*)dst);
  PCK(cudaGetLastError());
  return ETC_OK;
}

int etc_op_rhs(int prec, int nx, int ny, int nz, const void* tin, const void* tout, const void* pin_plane,
               double pin, const void* pout_plane, double pout, void* b, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks((long long)nx * ny * nz);
  if (prec == 0)
    k_op_rhs<double><<<grid, NT, 0, st>>>(nx, ny, nz, (const double*)tin, (const double*)tout,
                                         (const double*)pin_plane, pin, (const double*)pout_plane, pout, (double*)b);
  else
    k_op_rhs<float><<<grid, NT, 0, st>>>(nx, ny, nz, (const float*)tin, (const float*)tout, (const float*)pin_plane,
                                        (float)pin, (const float*)pout_plane, (float)pout, (float*)b);
  PCK(cudaGetLastError());
  return ETC_OK;
}

int etc_op_flux(int prec, int nx, int ny, int nz, const void* t_layer, double hz, const void* u, double pval,
                int side_out, void* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks((long long)nx * ny);
  if (prec == 0)
    k_op_flux<double><<<grid, NT, 0, st>>>(nx, ny, nz, (const double*)t_layer, hz, (const double*)u, pval, side_out,
                                          (double*)out);
  else
    k_op_flux<float><<<grid, NT, 0, st>>>(nx, ny, nz, (const float*)t_layer, (float)hz, (const float*)u, (float)pval,
                                         side_out, (float*)out);
  PCK(cudaGetLastError());
  return ETC_OK;
}

// returns ETC_PIVOT with *bad_layer set when a pivot is not positive (synchronises the stream)
int etc_op_thomas(int prec, int nx, int ny, int nz, const void* shift, const void* zdiag, double off, void* x,
                  void* upper, int* bad_dev, int* bad_layer, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks((long long)nx * ny, 16);
  const int big = 0x7fffffff;
  PCK(cudaMemcpyAsync(bad_dev, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  if (prec == 0)
    k_op_thomas<double><<<grid, NT, 0, st>>>(nx, ny, nz, (const double*)shift, (const double*)zdiag, off,
                                            (double*)x, (double*)upper, bad_dev);
  else
    k_op_thomas<float><<<grid, NT, 0, st>>>(nx, ny, nz, (const float*)shift, (const float*)zdiag, (float)off,
                                           (float*)x, (float*)upper, bad_dev);
  PCK(cudaGetLastError());
  int b = big;
  PCK(cudaMemcpyAsync(&b, bad_dev, sizeof(int), cudaMemcpyDeviceToHost, st));
  PCK(cudaStreamSynchronize(st));
  *bad_layer = b == big ? -1 : b;
  if (b != big) return perr(ETC_PIVOT, "non-positive pivot in tridiagonal solve");
  return ETC_OK;
}

// kind: 0 out = a * b, 1 out = 1 / a, 2 out = a + b
int etc_op_elementwise(int prec, int kind, long long n, const void* a, const void* b, void* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks(n);
  if (kind == 0) {
    if (prec == 0) k_op_mul<double><<<grid, NT, 0, st>>>(n, (const double*)a, (const double*)b, (double*)out);
    else k_op_mul<float><<<grid, NT, 0, st>>>(n, (const float*)a, (const float*)b, (float*)out);
  } else if (kind == 1) {
    if (prec == 0) k_op_recip<double><<<grid, NT, 0, st>>>(n, (const double*)a, (double*)out);
    else k_op_recip<float><<<grid, NT, 0, st>>>(n, (const float*)a, (float*)out);
  } else if (kind == 2) {
    if (prec == 0) k_op_add<double><<<grid, NT, 0, st>>>(n, (const double*)a, (const double*)b, (double*)out);
    else k_op_add<float><<<grid, NT, 0, st>>>(n, (const float*)a, (const float*)b, (float*)out);
  } else {
    return perr(ETC_CONFIG, "unknown elementwise kind");
  }
  PCK(cudaGetLastError());
  return ETC_OK;
}

// kind 0: out[0] = a.b; 1: out[0..2] = (a.b, a.a, b.b); 2: out[0] = sum a.
// parts: etc_op_reduce_parts(n) doubles of device scratch; out: device
int etc_op_dots(int prec, int kind, long long n, const void* a, const void* b, double* parts, double* out,
                void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks(n);
#define ETC_DOTS(K)                                                                                        \
  if (prec == 0)                                                                                           \
    k_op_dots<double, K><<<grid, NT, 0, st>>>(n, (const double*)a, (const double*)b, parts);               \
  else                                                                                                     \
    k_op_dots<float, K><<<grid, NT, 0, st>>>(n, (const float*)a, (const float*)b, parts);
  if (kind == 0) { ETC_DOTS(0) } else if (kind == 1) { ETC_DOTS(1) } else if (kind == 2) { ETC_DOTS(2) }
  else return perr(ETC_CONFIG, "unknown reduction kind");
#undef ETC_DOTS
  PCK(cudaGetLastError());
  return reduce_finish(grid, kind == 1 ? 3 : 1, parts, out, st);
}

int etc_op_pcg_update(int prec, long long n, double alpha, void* p, const void* w, void* r, const void* z,
                      double* parts, double* rr_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks(n);
  if (prec == 0)
    k_op_pcg_update<double><<<grid, NT, 0, st>>>(n, alpha, (double*)p, (const double*)w, (double*)r,
                                                (const double*)z, parts);
  else
    k_op_pcg_update<float><<<grid, NT, 0, st>>>(n, (float)alpha, (float*)p, (const float*)w, (float*)r,
                                               (const float*)z, parts);
  PCK(cudaGetLastError());
  return reduce_finish(grid, 1, parts, rr_out, st);
}

int etc_op_xpby(int prec, long long n, const void* z, double beta, void* w, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = nblocks(n);
  if (prec == 0)
    k_op_xpby<double><<<grid, NT, 0, st>>>(n, (const double*)z, beta, (double*)w);
  else
    k_op_xpby<float><<<grid, NT, 0, st>>>(n, (const float*)z, (float)beta, (float*)w);
  PCK(cudaGetLastError());
  return ETC_OK;
}

// exact (min, max) of a positive array; mm: 2 device uint64 (bit patterns)
int etc_op_minmax(int prec, long long n, const void* a, void* mm, double out[2], void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long init[2] = {0x7ff0000000000000ull, 0ull};  // +inf, +0
  PCK(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, st));
  if (n > 0) {
    const int grid = nblocks(n);
    if (prec == 0)
      k_op_minmax<double><<<grid, NT, 0, st>>>(n, (const double*)a, (unsigned long long*)mm);
    else
      k_op_minmax<float><<<grid, NT, 0, st>>>(n, (const float*)a, (unsigned long long*)mm);
    PCK(cudaGetLastError());
  }
  unsigned long long h[2];
  PCK(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, st));
  PCK(cudaStreamSynchronize(st));
  std::memcpy(&out[0], &h[0], 8);
  std::memcpy(&out[1], &h[1], 8);
  return ETC_OK;
}

int etc_op_ssor(int nx, int ny, int nz, const double* tx, const double* ty, const double* tz, const double* diag,
                double omega, const double* r, double* out, void* stream) {
  if (!(omega > 0.0 && omega < 2.0)) return perr(ETC_CONFIG, "omega must lie in (0, 2)");
  cudaStream_t st = (cudaStream_t)stream;
  k_op_ssor<<<1, 1024, 0, st>>>(nx, ny, nz, tx, ty, tz, diag, omega, r, out);
  PCK(cudaGetLastError());
  return ETC_OK;
}

int etc_op_dense(int nx, int ny, int nz, const double* tx, const double* ty, const double* tz, const double* tin,
                 const double* tout, double* mat, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const long long n = (long long)nx * ny * nz;
  PCK(cudaMemsetAsync(mat, 0, (size_t)(n * n) * sizeof(double), st));
  k_op_dense<<<nblocks(n), NT, 0, st>>>(nx, ny, nz, tx, ty, tz, tin, tout, mat);
  PCK(cudaGetLastError());
  return ETC_OK;
}

}  // extern "C"
