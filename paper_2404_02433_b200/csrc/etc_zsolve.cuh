// etc_zsolve.cuh — TMA-fed z-solve of the FCT preconditioner
// (thomas_solve_batch, /root/reference/pkg/src/etchomo/preconditioner.py:215-250),
// included by etc_b200.cu after k_thomas_x (it reuses rcp_fast, the mbarrier
// helpers, fin_thomas and grid_sum_finalize).
//
// Same partition algorithm as k_thomas_x (nz = 32 L rows per column, 32
// blocks of L rows, the last row of blocks 0..30 a separator; local block
// elimination, spike end values, parallel cyclic reduction on the 31
// separators, one coupling sweep), so the solution is bitwise that kernel's.
// What changes is how the data moves:
//   * a tile is 16 consecutive columns x all nz rows, row-major in shared
//     memory exactly as it lies in HBM (128-byte row segments), moved by TMA
//     (cp.async.bulk.tensor.2d) in 16 x min(nz,256) boxes: loads complete on an
//     mbarrier, the solved tile leaves by a TMA store from the same buffer;
//   * a persistent CTA per SM keeps three tile buffers: while it solves tile
//     n, tile n+1 is landing and tile n-1 is draining, so HBM never waits on
//     the solve and no thread issues a global load or store of the vector;
//   * thread (c, q) owns rows [qL, qL+L) of column c: lanes 0-15 of a warp
//     are block 2w, lanes 16-31 block 2w+1, so every warp access to the tile is
//     one 256-byte row pair (two wavefronts, no bank conflicts).  Values and
//     reciprocal pivots stay in registers (2L doubles);
//   * the separator system of column c is solved by warp c after a shared
//     transpose of the blocks' spike end values (lane = block, shuffle PCR).
// PCG mode accumulates r.z = 4/(nx ny) sum a_x a_y R^ Z^ (Parseval,
// reference test_transforms.py:160-176) while the solution overwrites the
// right-hand side, and finalises beta (krylov.py:85-90).
#pragma once

namespace etc {

constexpr int ZT_C = 16;       // columns per tile (one 128-byte row segment)
constexpr int ZT_STAGES = 3;   // tile buffers per CTA
constexpr int ZT_XS = 33;      // padded stride of the per-column exchange rows

// T: the type of the vector and of the elimination (double; float for
// precision f32, which eliminates in float32 as the reference does)
// TC: columns per tile (16, one 128-byte row segment of doubles; 8 for
// nz = 1024, whose 16-column tiles would not fit three stages in shared memory)
template <int L, class T = double, int TC = ZT_C>
constexpr size_t zt_tile_bytes() { return (size_t)32 * L * TC * sizeof(T); }
template <int L, class T = double, int TC = ZT_C>
constexpr size_t zt_smem_bytes() {
  return ZT_STAGES * zt_tile_bytes<L, T, TC>() + (size_t)2 * (2 * L + 7) * TC * sizeof(T) +
         (size_t)3 * TC * ZT_XS * sizeof(T) + 8 * ZT_STAGES;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(map), "r"(x), "r"(y), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(x),
               "r"(y), "r"((unsigned)__cvta_generic_to_shared(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// per-tile column tables, built by the producer warp one tile ahead: the
// reciprocal pivots and spike end values depend on the column's shift only,
// not on the data, so the 16 compute warps never run the pivot recurrence
template <int L, class R = double, int TC = ZT_C>
struct ZtTab {
  R rf[L - 1][TC];  // first block (q = 0): reciprocal pivots of rows 0..L-2
  R ri[L][TC];      // other blocks: rows 0..L-2; [L-1] the last block's row L-1
  // 0 v_last (first block) | 1 u_first 2 v_first 3 v_last (interior blocks) |
  // 4 u_first 5 v_first (last block) | 6 z_diag interior + shift | 7 r.z weight (0: column past the plane)
  R sv[8][TC];
};

// map: 2-D tensor map over t viewed as (nz rows) x (plane columns), box
// ZT_C x BR (BR = min(nz, 256) rows).  Warps 0-15 solve, warp 16 (the
// producer) builds the next tile's tables and drives the TMA ring.
template <int L, class T = double, int TC = ZT_C>
__global__ void __launch_bounds__(TC * 32 + 32, 1)
    k_zsolve_tma(Geom g, const __grid_constant__ CUtensorMap map, const double* __restrict__ wx,
                 const double* __restrict__ wy, double zd0_, double zdi_, double zdl_, double kxr, double kyr, double off_,
                 Ctl* ctl, double* partials, unsigned* counter, int pcg) {
  static_assert(L >= 3, "blocks of at least three rows");
  using R = T;  // float32 solve: the elimination in float32, as the reference's
  const R zd0 = (R)zd0_, zdi = (R)zdi_, zdl = (R)zdl_, off = (R)off_;
  if (pcg && ctl->done) return;
  constexpr int Q = 32, NZ = Q * L, S = ZT_STAGES, BPW = 32 / TC;  // BPW: blocks per compute warp
  constexpr int BR = NZ < 256 ? NZ : 256, NB = NZ / BR;  // TMA boxes per tile
  constexpr unsigned TILE_TX = (unsigned)zt_tile_bytes<L, T, TC>();
  extern __shared__ __align__(128) double zsm[];
  T* tiles = reinterpret_cast<T*>(zsm);                   // S x [NZ][TC]
  ZtTab<L, R, TC>* tab = reinterpret_cast<ZtTab<L, R, TC>*>(tiles + (size_t)S * NZ * TC);  // 2 stages
  R* X = reinterpret_cast<R*>(tab + 2);         // [2][TC][ZT_XS]: g_first, d partial
  R* SX = X + 2 * TC * ZT_XS;                        // [TC][ZT_XS] separator values
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(SX + TC * ZT_XS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool producer = warp == TC;
  const long long plane = g.plane;
  const long long ntiles = (plane + TC - 1) / TC;
  const long long G = gridDim.x;
  const R off2 = off * off;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](long long n) {  // local tile n of this CTA -> stage n % S
    const long long tl = blockIdx.x + n * G;
    if (tl < ntiles) {
      const int s = (int)(n % S);
      mbar_expect_tx(&bar[s], TILE_TX);
#pragma unroll
      for (int b = 0; b < NB; ++b)
        tma_load_2d(tiles + (size_t)s * NZ * TC + (size_t)b * BR * TC, &map, (int)(tl * TC), b * BR, &bar[s]);
    }
  };
  // producer: the tables of local tile n (lane = column c, variant v: 0 first block, 1 the others)
  auto tables = [&](long long n) {
    const long long tl = blockIdx.x + n * G;
    if (tl >= ntiles) return;
    ZtTab<L, R, TC>& Tp = tab[n & 1];
    const int c = lane % TC, v = lane / TC;
    if (v >= 2) return;  // TC = 8: lanes 16-31 idle
    const long long col = tl * TC + c;
    const bool valid = col < plane;
    const unsigned cu = valid ? (unsigned)col : 0u;
    const int ip = (int)(cu % (unsigned)g.nx), jp = (int)(cu / (unsigned)g.nx) + g.jofs;
    // precision f32: the shift is formed in float64 and cast, z_diag + shift
    // and the elimination run in float32 (preconditioner.py:184-250)
    const R shift = (R)__dadd_rn(__dmul_rn(wx[ip], kxr), __dmul_rn(wy[jp], kyr));
    const R B = zdi + shift;
    R r[L];
    r[0] = rcp_fast((v == 0 ? zd0 : zdi) + shift);
#pragma unroll
    for (int i = 1; i < L - 1; ++i) r[i] = rcp_fast(B - off2 * r[i - 1]);
    // spike end values of a block of L-1 rows (first / interior)
    const R v_last = r[L - 2];
    R mu = (R)1, vprod = v_last;
#pragma unroll
    for (int i = L - 3; i >= 0; --i) {
      const R cpi = off * r[i];
      mu = (R)1 + cpi * off * r[i + 1] * mu;
      vprod = -cpi * vprod;
    }
    if (v == 0) {
#pragma unroll
      for (int i = 0; i < L - 1; ++i) Tp.rf[i][c] = r[i];
      Tp.sv[0][c] = v_last;
    } else {
#pragma unroll
      for (int i = 0; i < L - 1; ++i) Tp.ri[i][c] = r[i];
      Tp.sv[1][c] = r[0] * mu;
      Tp.sv[2][c] = vprod;
      Tp.sv[3][c] = v_last;
      // the last block: L rows, row L-1 on z_diag[nz-1]
      const R rl = rcp_fast(zdl + shift - off2 * r[L - 2]);
      Tp.ri[L - 1][c] = rl;
      R mul = (R)1, vpl = rl;
      {
        const R cpi = off * r[L - 2];
        mul = (R)1 + cpi * off * rl * mul;
        vpl = -cpi * vpl;
      }
#pragma unroll
      for (int i = L - 3; i >= 0; --i) {
        const R cpi = off * r[i];
        mul = (R)1 + cpi * off * r[i + 1] * mul;
        vpl = -cpi * vpl;
      }
      Tp.sv[4][c] = r[0] * mul;
      Tp.sv[5][c] = vpl;
      Tp.sv[6][c] = B;
      Tp.sv[7][c] = valid ? (ip == 0 ? 0.5 : 1.0) * (jp == 0 ? 0.5 : 1.0) : 0.0;
    }
  };
  double dot = 0.0;
  if (producer) {
    if (lane == 0) {
      issue(0);
      issue(1);
    }
    tables(0);
    __syncthreads();
    for (long long n = 0;; ++n) {
      const long long tl = blockIdx.x + n * G;
      if (tl >= ntiles) break;
      tables(n + 1);
      __syncthreads();  // tile n solved and written back; tables n+1 ready
      if (lane == 0) {
        const int s = (int)(n % S);
#pragma unroll
        for (int b = 0; b < NB; ++b)
          tma_store_2d(&map, (int)(tl * TC), b * BR, tiles + (size_t)s * NZ * TC + (size_t)b * BR * TC);
        bulk_commit();
        // tile n+2 goes into tile n-1's buffer once that store has read it
        bulk_wait_read<1>();
        issue(n + 2);
      }
    }
    if (lane == 0) bulk_wait_all();
  } else {
    const int c = lane % TC, q = BPW * warp + lane / TC;  // column in tile, block
    const bool last = (q == Q - 1);
    __syncthreads();
    for (long long n = 0;; ++n) {
      const long long tl = blockIdx.x + n * G;
      if (tl >= ntiles) break;
      const int s = (int)(n % S);
      T* tile = tiles + (size_t)s * NZ * TC;
      const ZtTab<L, R, TC>& Tt = tab[n & 1];
      T* myf = tile + (size_t)q * L * TC + c;  // row i of the block at myf[i * TC]
      // reciprocal pivots straight from the table (rows L-1 of the last block
      // continue the interior table); values in registers
      const R* rp = (q == 0) ? &Tt.rf[0][c] : &Tt.ri[0][c];
      // float: the block's reciprocal pivots fit in registers, read once per
      // tile instead of once per sweep (0.340 -> 0.326 ms at 512^3); double
      // keeps them in the table (in registers they spill at the 96-register
      // cap of the 544-thread CTA: 0.451 -> 0.594 ms)
      constexpr bool RREG = sizeof(R) == 4;
      R rcpv[RREG ? L : 1];
      if constexpr (RREG) {
#pragma unroll
        for (int i = 0; i < L; ++i) rcpv[i] = (i < L - 1 || last) ? rp[i * TC] : (R)0;
      }
      auto rcp = [&](int i) -> R {
        if constexpr (RREG)
          return rcpv[i];
        else
          return rp[i * TC];
      };
      R my[L];
      mbar_wait(&bar[s], (unsigned)((n / S) & 1));
      // local forward elimination; rows 0..L-2 in every block, row L-1 only in the last
      R xp = (R)myf[0] * rcp(0);
      my[0] = xp;
#pragma unroll
      for (int i = 1; i < L - 1; ++i) {
        xp = ((R)myf[i * TC] - off * xp) * rcp(i);
        my[i] = xp;
      }
      if (last) {
        xp = ((R)myf[(L - 1) * TC] - off * xp) * rcp(L - 1);
        my[L - 1] = xp;
      }
      // g = block^-1 f at the block's ends
      const R g_last = xp;
      R gacc = g_last;
      if (last) gacc = my[L - 2] - off * rcp(L - 2) * gacc;
#pragma unroll
      for (int i = L - 3; i >= 0; --i) gacc = my[i] - off * rcp(i) * gacc;
      {
        const int xo = c * ZT_XS + q;
        X[xo] = gacc;                                                     // g_first
        if (!last) X[TC * ZT_XS + xo] = (R)myf[(L - 1) * TC] - off * g_last;  // separator rhs minus own coupling
      }
      asm volatile("bar.sync 1, %0;" ::"n"(TC * 32) : "memory");
      {  // warp `warp` solves the separator system of column `warp`, lane = block
        const int cw = warp, qq = lane;
        const int xo = cw * ZT_XS + qq;
        const R lo_first = (qq == 0) ? (R)0 : off, up_last = (qq == Q - 1) ? (R)0 : off;
        const R n_ul = (qq + 1 == Q - 1) ? (R)0 : off;
        R a = (R)0, b = (R)1, cc = (R)0, d = (R)0;
        if (qq < Q - 1) {  // separator row qq L + L-1
          const R v_first = qq == 0 ? (R)0 : Tt.sv[2][cw];
          const R v_l = qq == 0 ? Tt.sv[0][cw] : Tt.sv[3][cw];
          const R n_uf = (qq + 1 == Q - 1) ? Tt.sv[4][cw] : Tt.sv[1][cw];
          const R n_vf = (qq + 1 == Q - 1) ? Tt.sv[5][cw] : Tt.sv[2][cw];
          const R n_gf = X[xo + 1], dpart = X[TC * ZT_XS + xo];
          a = -off * lo_first * v_first;
          b = Tt.sv[6][cw] - off * up_last * v_l - off2 * n_uf;
          cc = -off * n_ul * n_vf;
          d = dpart - off * n_gf;
        }
#pragma unroll
        for (int dd = 1; dd < Q; dd <<= 1) {
          R am = __shfl_up_sync(0xffffffffu, a, dd), bm = __shfl_up_sync(0xffffffffu, b, dd);
          R cm = __shfl_up_sync(0xffffffffu, cc, dd), dm = __shfl_up_sync(0xffffffffu, d, dd);
          R ap = __shfl_down_sync(0xffffffffu, a, dd), bp = __shfl_down_sync(0xffffffffu, b, dd);
          R cp = __shfl_down_sync(0xffffffffu, cc, dd), dp = __shfl_down_sync(0xffffffffu, d, dd);
          if (qq < dd) { am = (R)0; bm = (R)1; cm = (R)0; dm = (R)0; }
          if (qq + dd >= Q) { ap = (R)0; bp = (R)1; cp = (R)0; dp = (R)0; }
          const R k1 = a * rcp_fast(bm), k2 = cc * rcp_fast(bp);
          const R na = -am * k1, nc = -cp * k2;
          const R nbv = b - cm * k1 - ap * k2, nd = d - dm * k1 - dp * k2;
          a = na; b = nbv; cc = nc; d = nd;
        }
        SX[xo] = d / b;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(TC * 32) : "memory");
      const R Sv = SX[c * ZT_XS + q];
      const R Sm = q ? SX[c * ZT_XS + q - 1] : (R)0;
      // separator coupling: forward sweep of the end corrections, then back substitution
      const R lo_first = (q == 0) ? (R)0 : off;
      const R eta0 = -lo_first * Sm;
      const R etaL = last ? (R)0 : -off * Sv;
      {
        R h = eta0 * rcp(0);
        my[0] += h;
#pragma unroll
        for (int i = 1; i < L - 1; ++i) {
          h = ((i == L - 2 && !last ? etaL : (R)0) - off * h) * rcp(i);
          my[i] += h;
        }
        if (last) {
          h = ((R)0 - off * h) * rcp(L - 1);
          my[L - 1] += h;
        }
        R xn = last ? my[L - 1] : my[L - 2];
        if (last) {
          xn = my[L - 2] - off * rcp(L - 2) * xn;
          my[L - 2] = xn;
        }
#pragma unroll
        for (int i = L - 3; i >= 0; --i) {
          xn = my[i] - off * rcp(i) * xn;
          my[i] = xn;
        }
      }
      if (!last) my[L - 1] = Sv;
      // r.z partial and the solution over the right-hand side
      {
        double sacc = 0.0;
#pragma unroll
        for (int i = 0; i < L; ++i) {
          sacc = fma((double)myf[i * TC], (double)my[i], sacc);
          myf[i * TC] = (T)my[i];
        }
        if (pcg) dot = fma((double)Tt.sv[7][c], sacc, dot);
      }
      fence_proxy_async_smem();  // the generic-proxy writes are seen by the TMA store
      __syncthreads();
    }
  }
  if (pcg) {
    double v[1] = {dot};
    const double scale = 4.0 / ((double)g.nx * (double)g.nyg);
    grid_sum_finalize<1>(v, partials, counter, [&](double (&tt)[1]) {
      if (ctl->dist)
        ctl->xbuf[4] = tt[0];
      else if constexpr (sizeof(T) == 4)
        fin_thomas(ctl, f32r(tt[0] * scale));  // np.dot of two float32 vectors
      else
        fin_thomas(ctl, tt[0] * scale);
    });
  }
}

}  // namespace etc
