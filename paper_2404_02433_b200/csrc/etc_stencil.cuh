// etc_stencil.cuh — q = A w on the device (apply_operator, reference
// /root/reference/pkg/src/etchomo/tpfa.py:110-131) and the face
// transmissibilities (tpfa.py:29-30, 91-107): the unfused stencil with the
// search-direction update, the cp.async stencil, the phase detection and
// phase-indexed TMA stencil (k_stencil_pht), the stored-face TMA stencil
// (k_stencil_gt).  Included by etc_b200.cu (one translation unit).
#pragma once

// ---- stencil: w_new = z + beta*w_old (Alg. 1 line `w = z + beta w`) fused with
// q = A w_new and the dots q.w, q.q, w.w (krylov.py:71-74), plus the previous
// iteration's p += alpha w (krylov.py:76).  Per-cell association order of
// tpfa.py:117-130 with no FMA contraction, so q is bitwise the reference
// apply_operator(w).  Faces are the harmonic-mean transmissibilities built
// once per solve by k_faces (bitwise tpfa.py:29-30 / 102-104): tx[c] is the
// face between cell c and c+1 along x, likewise ty, tz.  2.5-D blocking: a
// 32x8 CTA marches along z with the current plane of w and ty in
// double-buffered shared tiles (one-cell halo), plane k+1 prefetched in
// registers; tx(i-1/2) arrives by shuffle, tz(k-1/2) is carried.
template <bool FIRST, bool PCG>
__global__ void __launch_bounds__(256, 4) k_stencil(Geom g, int kchunk, const double* __restrict__ tx,
                                                    const double* __restrict__ ty, const double* __restrict__ tz,
                                                    const double* __restrict__ tb, const double* __restrict__ zv,
                                                    const double* __restrict__ wold, double* __restrict__ wnew,
                                                    double* __restrict__ qout, double* __restrict__ p, int p_plane,
                                                    int halo_wb, Ctl* ctl, double* partials, unsigned* counter) {
  if (PCG && ctl->done) return;
  // iteration k's p += alpha_k w_k rides on iteration k+1's read of w_k;
  // alpha_k is still in ctl (overwritten only by this kernel's last CTA,
  // after every CTA has read it)
  const double alpha_prev = (PCG && !FIRST) ? ctl->alpha : 0.0;
  const double beta = (PCG && !FIRST) ? ctl->beta : 0.0;
  __shared__ double Ut[2][10][34];
  __shared__ double Yt[2][9][32];
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long P = g.plane;
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int i = blockIdx.x * 32 + lx, j = blockIdx.y * 8 + ly;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(nz, k0 + kchunk);
  const bool in = (i < nx && j < ny);
  const int ic = min(i, nx - 1), jc = min(j, ny - 1);
  const long long col = (long long)jc * nx + ic;
  const long long cl = col - (i > 0 ? 1 : 0), cr = (long long)jc * nx + min(i + 1, nx - 1);
  const long long cu = col - (j > 0 ? nx : 0), cd = (long long)min(j + 1, ny - 1) * nx + ic;
  auto W = [&](long long idx) -> double {
    if (FIRST) return zv[idx];
    return __dadd_rn(zv[idx], __dmul_rn(beta, wold[idx]));
  };
  const int kg0 = g.kg0, nzg = g.nzg;  // global plane of local plane 0; global count
  double dqw = 0.0, dqq = 0.0, dww = 0.0;
  if (k0 < k1) {
    double um = 0.0, fzm = 0.0;
    if (kg0 + k0 > 0) {  // local plane k0-1 may be the lower halo (-1)
      um = W((long long)(k0 - 1) * P + col);
      fzm = tz[(long long)(k0 - 1) * P + col];
      if (halo_wb && k0 == 0 && in) wnew[col - P] = um;
    }
    // register pipeline: plane k (c) and k+1 (n)
    long long pk = (long long)k0 * P;
    double zc = zv[pk + col], oc = FIRST ? 0.0 : wold[pk + col];
    double xc = tx[pk + col], yc = ty[pk + col], fzc = tz[pk + col];
    double zn = 0.0, on = 0.0;
    if (kg0 + k0 + 1 < nzg) {
      zn = zv[pk + P + col];
      if (!FIRST) on = wold[pk + P + col];
    }
    for (int k = k0; k < k1; ++k, pk += P) {
      const int buf = k & 1;
      const bool hasp = kg0 + k + 1 < nzg;
      // prefetch plane k+1 coefficients and plane k+2 vectors
      double xn = 0.0, yn = 0.0, fzn = 0.0, z2 = 0.0, o2 = 0.0;
      if (k + 1 < k1) {
        xn = tx[pk + P + col];
        yn = ty[pk + P + col];
        fzn = tz[pk + P + col];
        if (kg0 + k + 2 < nzg) {
          z2 = zv[pk + 2 * P + col];
          if (!FIRST) o2 = wold[pk + 2 * P + col];
        }
      }
      const double uc = FIRST ? zc : __dadd_rn(zc, __dmul_rn(beta, oc));
      const double un = FIRST ? zn : __dadd_rn(zn, __dmul_rn(beta, on));
      Ut[buf][ly + 1][lx + 1] = uc;
      Yt[buf][ly + 1][lx] = yc;
      if (lx == 0) Ut[buf][ly + 1][0] = W(pk + cl);
      if (lx == 31) Ut[buf][ly + 1][33] = W(pk + cr);
      if (ly == 0) {
        Ut[buf][0][lx + 1] = W(pk + cu);
        Yt[buf][0][lx] = ty[pk + cu];
      }
      if (ly == 7) Ut[buf][9][lx + 1] = W(pk + cd);
      double fxm = __shfl_up_sync(0xffffffffu, xc, 1);
      if (lx == 0) fxm = tx[pk + cl];
      __syncthreads();
      double (*U)[34] = Ut[buf];
      if (in) {
        double acc = 0.0;
        if (i > 0) acc = __dadd_rn(acc, __dmul_rn(fxm, __dsub_rn(uc, U[ly + 1][lx])));
        if (i + 1 < nx) acc = __dsub_rn(acc, __dmul_rn(xc, __dsub_rn(U[ly + 1][lx + 2], uc)));
        if (j > 0) acc = __dadd_rn(acc, __dmul_rn(Yt[buf][ly][lx], __dsub_rn(uc, U[ly][lx + 1])));
        if (j + 1 < ny) acc = __dsub_rn(acc, __dmul_rn(yc, __dsub_rn(U[ly + 2][lx + 1], uc)));
        if (kg0 + k > 0) acc = __dadd_rn(acc, __dmul_rn(fzm, __dsub_rn(uc, um)));
        if (hasp) acc = __dsub_rn(acc, __dmul_rn(fzc, __dsub_rn(un, uc)));
        if (kg0 + k == 0) acc = __dadd_rn(acc, __dmul_rn(tb[col], uc));
        if (kg0 + k == nzg - 1) acc = __dadd_rn(acc, __dmul_rn(tb[P + col], uc));
        if (halo_wb && k == nz - 1 && hasp) wnew[pk + P + col] = un;
        if (wnew) wnew[pk + col] = uc;
        qout[pk + col] = acc;
        if (PCG && !FIRST && (p_plane == -1 || k == p_plane))
          p[pk + col] = __dadd_rn(p[pk + col], __dmul_rn(alpha_prev, oc));
        if (PCG) {
          dqw = fma(acc, uc, dqw);
          dqq = fma(acc, acc, dqq);
          dww = fma(uc, uc, dww);
        }
      }
      um = uc;
      fzm = fzc;
      zc = zn; oc = on;
      zn = z2; on = o2;
      xc = xn; yc = yn; fzc = fzn;
    }
  }
  if (PCG) {
    double v[3] = {dqw, dqq, dww};
    grid_sum_finalize<3>(v, partials, counter, [&](double (&t)[3]) {
      if (ctl->dist) {
        ctl->xbuf[0] = t[0];
        ctl->xbuf[1] = t[1];
        ctl->xbuf[2] = t[2];
      } else {
        fin_stencil(ctl, t[0], t[1], t[2]);
      }
    });
  }
}

// ---- cp.async multistage stencil for square power-of-two planes: the same
// arithmetic as k_stencil (bitwise), with plane k+3 streaming into a 4-deep
// shared-memory ring (LDGSTS, 8-byte, halos included) while plane k is
// computed, so each thread keeps ~3 planes of loads in flight without
// holding them in registers.
__device__ __forceinline__ void cp8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory"); }

struct StencilStage {
  double Z[10][34];  // z with a one-cell halo
  double O[10][34];  // w_old with a one-cell halo
  double X[8][33];   // tx, column 0 = face i-1/2 of the first lane
  double Y[9][32];   // ty, row 0 = face j-1/2 of the first row
  double T[8][32];   // tz
};

template <int N, bool FIRST, bool PCG>
__global__ void __launch_bounds__(256, 4) k_stencil_cp(Geom g, int kchunk, const double* __restrict__ tx,
                                                       const double* __restrict__ ty, const double* __restrict__ tz,
                                                       const double* __restrict__ tb, const double* __restrict__ zv,
                                                       const double* __restrict__ wold, double* __restrict__ wnew,
                                                       double* __restrict__ qout, double* __restrict__ p, int p_plane,
                                                       int halo_wb, Ctl* ctl, double* partials, unsigned* counter) {
  if (PCG && ctl->done) return;
  constexpr int S = 4;
  constexpr long long P = (long long)N * N;
  const double alpha_prev = (PCG && !FIRST) ? ctl->alpha : 0.0;
  const double beta = (PCG && !FIRST) ? ctl->beta : 0.0;
  extern __shared__ double smem_d[];
  StencilStage* st = reinterpret_cast<StencilStage*>(smem_d);
  const int nz = g.nz, kg0 = g.kg0, nzg = g.nzg;
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int i = blockIdx.x * 32 + lx, j = blockIdx.y * 8 + ly;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(nz, k0 + kchunk);
  const int col = j * N + i;
  const int dl = (i > 0) ? -1 : 0, dr = (i + 1 < N) ? 1 : 0;
  const int du = (j > 0) ? -N : 0, dd = (j + 1 < N) ? N : 0;
  auto Wv = [&](double z, double o) -> double { return FIRST ? z : __dadd_rn(z, __dmul_rn(beta, o)); };
  auto issue = [&](int k) {
    if (k < k1 + 1 && kg0 + k < nzg) {  // plane k1 (maybe the upper halo) feeds the z+ neighbour of k1-1
      StencilStage& s = st[k % S];
      const long long o = (long long)k * P + col;
      cp8(&s.Z[ly + 1][lx + 1], zv + o);
      if (!FIRST) cp8(&s.O[ly + 1][lx + 1], wold + o);
      if (k < k1) {
        cp8(&s.X[ly][lx + 1], tx + o);
        cp8(&s.Y[ly + 1][lx], ty + o);
        cp8(&s.T[ly][lx], tz + o);
        if (lx == 0) {
          cp8(&s.Z[ly + 1][0], zv + o + dl);
          if (!FIRST) cp8(&s.O[ly + 1][0], wold + o + dl);
          cp8(&s.X[ly][0], tx + o + dl);
        }
        if (lx == 31) {
          cp8(&s.Z[ly + 1][33], zv + o + dr);
          if (!FIRST) cp8(&s.O[ly + 1][33], wold + o + dr);
        }
        if (ly == 0) {
          cp8(&s.Z[0][lx + 1], zv + o + du);
          if (!FIRST) cp8(&s.O[0][lx + 1], wold + o + du);
          cp8(&s.Y[0][lx], ty + o + du);
        }
        if (ly == 7) {
          cp8(&s.Z[9][lx + 1], zv + o + dd);
          if (!FIRST) cp8(&s.O[9][lx + 1], wold + o + dd);
        }
      }
    }
    cp_commit();
  };
  double dqw = 0.0, dqq = 0.0, dww = 0.0;
  if (k0 < k1) {
    double um = 0.0, fzm = 0.0;
    if (kg0 + k0 > 0) {  // local plane k0-1 may be the lower halo (-1)
      const long long o = (long long)(k0 - 1) * P + col;
      um = Wv(zv[o], FIRST ? 0.0 : wold[o]);
      fzm = tz[o];
      if (halo_wb && k0 == 0) wnew[o] = um;
    }
    issue(k0);
    issue(k0 + 1);
    issue(k0 + 2);
    for (int k = k0; k < k1; ++k) {
      cp_wait<1>();  // planes k and k+1 have landed (own copies)
      __syncthreads();
      issue(k + 3);  // refills the slot of plane k-1, read by everyone before the barrier
      const StencilStage& c = st[k % S];
      const StencilStage& nx_ = st[(k + 1) % S];
      const bool hasp = kg0 + k + 1 < nzg;
      const double oc = FIRST ? 0.0 : c.O[ly + 1][lx + 1];
      const double uc = Wv(c.Z[ly + 1][lx + 1], oc);
      double acc = 0.0;
      if (i > 0) acc = __dadd_rn(acc, __dmul_rn(c.X[ly][lx], __dsub_rn(uc, Wv(c.Z[ly + 1][lx], c.O[ly + 1][lx]))));
      if (i + 1 < N)
        acc = __dsub_rn(acc, __dmul_rn(c.X[ly][lx + 1], __dsub_rn(Wv(c.Z[ly + 1][lx + 2], c.O[ly + 1][lx + 2]), uc)));
      if (j > 0) acc = __dadd_rn(acc, __dmul_rn(c.Y[ly][lx], __dsub_rn(uc, Wv(c.Z[ly][lx + 1], c.O[ly][lx + 1]))));
      if (j + 1 < N)
        acc = __dsub_rn(acc, __dmul_rn(c.Y[ly + 1][lx], __dsub_rn(Wv(c.Z[ly + 2][lx + 1], c.O[ly + 2][lx + 1]), uc)));
      if (kg0 + k > 0) acc = __dadd_rn(acc, __dmul_rn(fzm, __dsub_rn(uc, um)));
      const double fzp = c.T[ly][lx];
      if (hasp) {
        const double un = Wv(nx_.Z[ly + 1][lx + 1], FIRST ? 0.0 : nx_.O[ly + 1][lx + 1]);
        acc = __dsub_rn(acc, __dmul_rn(fzp, __dsub_rn(un, uc)));
        if (halo_wb && k == nz - 1) wnew[(long long)nz * P + col] = un;
      }
      if (kg0 + k == 0) acc = __dadd_rn(acc, __dmul_rn(tb[col], uc));
      if (kg0 + k == nzg - 1) acc = __dadd_rn(acc, __dmul_rn(tb[P + col], uc));
      const long long o = (long long)k * P + col;
      if (wnew) wnew[o] = uc;
      qout[o] = acc;
      if (PCG && !FIRST && (p_plane == -1 || k == p_plane)) p[o] = __dadd_rn(p[o], __dmul_rn(alpha_prev, oc));
      if (PCG) {
        dqw = fma(acc, uc, dqw);
        dqq = fma(acc, acc, dqq);
        dww = fma(uc, uc, dww);
      }
      um = uc;
      fzm = fzp;
    }
    cp_wait<0>();
  }
  if (PCG) {
    double v[3] = {dqw, dqq, dww};
    grid_sum_finalize<3>(v, partials, counter, [&](double (&t)[3]) {
      if (ctl->dist) {
        ctl->xbuf[0] = t[0];
        ctl->xbuf[1] = t[1];
        ctl->xbuf[2] = t[2];
      } else {
        fin_stencil(ctl, t[0], t[1], t[2]);
      }
    });
  }
}

// ---- few-phase fields (voxel composites: a handful of distinct
// conductivities).  The scaled coefficients take at most PH_MAX distinct
// (s_x, s_y, s_z) triples; each cell then carries a one-byte phase index and
// every face transmissibility is an entry of a PH_MAX^2 table built with the
// same harm() -- bit-identical to k_faces.  The stencil streams w (8 B),
// the index (1 B) and q (8 B): 17 instead of 40 bytes per cell.
constexpr int PH_MAX = 16;

__device__ __forceinline__ unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }

__device__ __forceinline__ unsigned long long ph_hash(unsigned long long a, unsigned long long b,
                                                      unsigned long long d) {
  unsigned long long h = a * 0x9E3779B97F4A7C15ull;
  h ^= (b + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2)) * 0xBF58476D1CE4E5B9ull;
  h ^= (d + 0x94D049BB133111EBull + (h << 6) + (h >> 2)) * 0x94D049BB133111EBull;
  return h | 1ull;  // 0 marks an empty slot
}

// distinct (s_x, s_y, s_z) triples: each warp dedupes its cells with
// __match_any_sync into a warp-local set, then inserts the set into a global
// table of PH_MAX slots keyed by a 64-bit hash (atomicCAS, lock-free).
// k_phase_index verifies every cell against the stored triples, so a hash
// collision cannot go unnoticed (it reports an overflow and the solve keeps
// the stored faces).
__global__ void k_phase_collect(long long n, const double* __restrict__ s0, const double* __restrict__ s1,
                                const double* __restrict__ s2, unsigned long long* __restrict__ keys,
                                unsigned long long* __restrict__ trip, int* __restrict__ overflow) {
  __shared__ unsigned long long tab[8][PH_MAX][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int cnt = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long span = (n + stride - 1) / stride * stride;  // every lane runs the same trip count
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < span; c += stride) {
    const bool act = c < n;
    const unsigned long long a = act ? dbits(s0[c]) : 0ull, b = act ? dbits(s1[c]) : 0ull,
                             d = act ? dbits(s2[c]) : 0ull;
    bool have = !act;
    for (int p = 0; p < cnt && !have; ++p) have = tab[warp][p][0] == a && tab[warp][p][1] == b && tab[warp][p][2] == d;
    const unsigned grp = __match_any_sync(0xffffffffu, a) & __match_any_sync(0xffffffffu, b) &
                         __match_any_sync(0xffffffffu, d);
    const bool leader = (__ffs(grp) - 1) == lane;
    const unsigned fresh = __ballot_sync(0xffffffffu, leader && !have);
    if (fresh) {
      const int pos = cnt + __popc(fresh & ((1u << lane) - 1u));
      if ((fresh >> lane) & 1u && pos < PH_MAX) {
        tab[warp][pos][0] = a;
        tab[warp][pos][1] = b;
        tab[warp][pos][2] = d;
      }
      cnt += __popc(fresh);
      __syncwarp();
      if (cnt > PH_MAX) {
        if (lane == 0) atomicExch(overflow, 1);
        return;
      }
    }
  }
  if (lane < cnt) {
    const unsigned long long a = tab[warp][lane][0], b = tab[warp][lane][1], d = tab[warp][lane][2];
    const unsigned long long h = ph_hash(a, b, d);
    for (int p = 0; p < PH_MAX; ++p) {
      const unsigned long long old = atomicCAS(keys + p, 0ull, h);
      if (old == 0ull) {
        trip[3 * p] = a;
        trip[3 * p + 1] = b;
        trip[3 * p + 2] = d;
        return;
      }
      if (old == h) return;
    }
    atomicExch(overflow, 1);
  }
}

// per-cell phase index (verified against the stored triples), the face
// tables [a * PH_MAX + b] = harm(s_a, s_b) (lower cell a first, as k_faces)
// and tb[p] = 2 s_z; nph = number of phases, 0 on overflow
__global__ void k_phase_index(long long n, const double* __restrict__ s0, const double* __restrict__ s1,
                              const double* __restrict__ s2, const unsigned long long* __restrict__ keys,
                              const unsigned long long* __restrict__ trip, int* __restrict__ overflow,
                              int* __restrict__ nph, unsigned char* __restrict__ idx, double* __restrict__ ftab) {
  __shared__ unsigned long long t[PH_MAX][3];
  __shared__ int m;
  if (threadIdx.x == 0) {
    int c = 0;
    while (c < PH_MAX && keys[c] != 0ull) ++c;
    m = c;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 3 * m; e += blockDim.x) t[e / 3][e % 3] = trip[e];
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < PH_MAX * PH_MAX; e += blockDim.x) {
      const int a = e / PH_MAX, b = e % PH_MAX;
      const bool ok = a < m && b < m;
      for (int ax = 0; ax < 3; ++ax)
        ftab[ax * PH_MAX * PH_MAX + e] =
            ok ? harm(__longlong_as_double((long long)t[a][ax]), __longlong_as_double((long long)t[b][ax])) : 0.0;
    }
    for (int p = threadIdx.x; p < PH_MAX; p += blockDim.x)
      ftab[3 * PH_MAX * PH_MAX + p] = p < m ? __dmul_rn(2.0, __longlong_as_double((long long)t[p][2])) : 0.0;
    if (threadIdx.x == 0) *nph = m;
  }
  bool bad = false;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const unsigned long long a = dbits(s0[c]), b = dbits(s1[c]), d = dbits(s2[c]);
    int p = -1;
    for (int q = 0; q < m; ++q)
      if (t[q][0] == a && t[q][1] == b && t[q][2] == d) p = q;
    bad |= p < 0;
    idx[c] = (unsigned char)max(p, 0);
  }
  if (bad) atomicExch(overflow, 1);
}

// which phase pairs meet across x, y and z faces, and which phases lie on the
// two Dirichlet layers (the exact coefficient statistics of a few-phase field
// are min/max over those table entries; single-GPU plans)
__global__ void k_phase_pairs(Geom g, const unsigned char* __restrict__ idx, unsigned* __restrict__ masks) {
  __shared__ unsigned sm[3 * 8 + 2];
  for (int e = threadIdx.x; e < 26; e += blockDim.x) sm[e] = 0u;
  __syncthreads();
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long P = g.plane;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long span = (g.n + stride - 1) / stride * stride;  // whole warps to the end (match_any)
  const int lane = threadIdx.x & 31;
  // lanes with the same code are merged first (__match_any_sync): one shared
  // atomic per distinct code per warp instead of one per cell
  auto mark = [&](int code, unsigned* base) {  // code < 0: no face
    const unsigned grp = __match_any_sync(0xffffffffu, code);
    if (code >= 0 && (__ffs(grp) - 1) == lane) atomicOr(&base[code >> 5], 1u << (code & 31));
  };
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < span; c += stride) {
    const bool act = c < g.n;
    const long long cc = act ? c : 0;
    const long long k = cc / P, rem = cc - k * P;
    const int j = (int)(rem / nx), i = (int)(rem - (long long)j * nx);
    const int a = idx[cc];
    mark(act && i + 1 < nx ? a * PH_MAX + idx[cc + 1] : -1, sm);
    mark(act && j + 1 < ny ? a * PH_MAX + idx[cc + nx] : -1, sm + 8);
    mark(act && k + 1 < nz ? a * PH_MAX + idx[cc + P] : -1, sm + 16);
    mark(act && k == 0 ? a : -1, sm + 24);
    mark(act && k == nz - 1 ? a : -1, sm + 25);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 26; e += blockDim.x)
    if (sm[e]) atomicOr(masks + e, sm[e]);
}

// q = A w with the faces looked up from the phase indices (the fused solve's
// stencil for few-phase fields); same arithmetic order as k_stencil_cp.
// The face tables in shared memory: rows padded from PH_MAX to PH_RS doubles
// so the few (a, b) pairs of a warp (a 2x2 block for two phases) fall in
// distinct banks; PH_FT doubles in all (tb follows the three tables)
constexpr int PH_RS = 18, PH_TS = PH_MAX * PH_RS, PH_FT = 3 * PH_TS + PH_MAX;
__host__ __device__ constexpr int ph_slot(int e) {  // global ftab index -> shared slot
  return e < 3 * PH_MAX * PH_MAX ? (e / (PH_MAX * PH_MAX)) * PH_TS + ((e / PH_MAX) % PH_MAX) * PH_RS + e % PH_MAX
                                 : 3 * PH_TS + (e - 3 * PH_MAX * PH_MAX);
}

// Wc / Ic point at the cell in its plane's staged tiles (row pitches WP
// doubles / IP bytes), Wn / In at the same cell of the next plane
template <int N, bool MASK, int WP, int IP, class T>
__device__ __forceinline__ T ph_cell_p(const T* Wc, const unsigned char* Ic, const T* Wn, const unsigned char* In,
                                       const T* FT, int i, int j, bool kin, bool hasp, T uc, int pc, T um, T fzm,
                                       T& fzp, T& un, int& pn) {
  // uc, pc: this cell (carried in registers from the previous plane's
  // z-neighbour load); un, pn: the z+ neighbour, returned for the next plane
  constexpr int T2 = PH_TS, R = PH_RS;
  const T* FX = FT + pc;       // [a][pc]: faces below / left of the cell
  const T* FXr = FT + pc * R;  // [pc][b]: faces above / right
  const T fxm = FX[Ic[-1] * R], fxp = FXr[Ic[1]];
  const T fym = FX[T2 + Ic[-IP] * R], fyp = FXr[T2 + Ic[IP]];
  T acc = 0, t;
  t = add_rn(acc, mul_rn(fxm, sub_rn(uc, Wc[-1])));
  acc = (!MASK || i > 0) ? t : acc;
  t = sub_rn(acc, mul_rn(fxp, sub_rn(Wc[1], uc)));
  acc = (!MASK || i + 1 < N) ? t : acc;
  t = add_rn(acc, mul_rn(fym, sub_rn(uc, Wc[-WP])));
  acc = (!MASK || j > 0) ? t : acc;
  t = sub_rn(acc, mul_rn(fyp, sub_rn(Wc[WP], uc)));
  acc = (!MASK || j + 1 < N) ? t : acc;
  if (kin) acc = add_rn(acc, mul_rn(fzm, sub_rn(uc, um)));
  fzp = 0;
  un = *Wn;
  pn = *In;
  if (hasp) {
    fzp = FXr[2 * T2 + pn];
    acc = sub_rn(acc, mul_rn(fzp, sub_rn(un, uc)));
  }
  return acc;
}

// ---- the same stencil with TMA plane staging: one elected thread moves each
// plane's w tile and phase-index tile into the 4-deep ring with two
// cp.async.bulk.tensor loads that complete on the stage's mbarrier, so the
// consumer warps issue no global loads and no per-thread halo bookkeeping.
// A box's x origin must be 16-byte aligned (an unaligned origin traps with
// an illegal instruction -- measured, profiles/probes/tma_box_probe.log), so
// the tiles are wider than the halo needs (w from i0-2, index from i0-16).
// The origins are also clamped into the grid: on the grid's edge blocks the
// tile shifts inwards and the cells read across the grid edge are in-grid
// neighbours, which the boundary masks drop.
// T = double: w boxes 36 wide from i0-2; T = float (precision f32): 40 wide
// from i0-4 (box origins 16-byte aligned either way)
template <class T, int HB = 18>  // HB: box rows (the tile's rows + 2 halo rows)
struct alignas(128) PhaseStageTmaT {
  static constexpr int WX = sizeof(T) == 8 ? 36 : 40, XO = sizeof(T) == 8 ? 2 : 4;
  T W[HB][WX];                    // w, rows oy .. oy+HB-1, columns ox .. ox+WX-1
  T wpad[64 / sizeof(T)];         // zero: index reads one row above row 0 land here
  unsigned char I[HB][64];        // phase index, rows oy .., bytes oxi .. oxi+63
  unsigned char I18[64];          // zero: index reads one row below row HB-1
  static constexpr unsigned TX = sizeof(T) * HB * WX + HB * 64;  // bytes landing per stage
};
using PhaseStageTma = PhaseStageTmaT<double>;
static_assert(offsetof(PhaseStageTmaT<double>, I) % 128 == 0, "TMA destinations are 128-byte aligned");
static_assert(offsetof(PhaseStageTmaT<float>, I) % 128 == 0, "TMA destinations are 128-byte aligned");
using PhaseStageTma34 = PhaseStageTmaT<double, 34>;
using PhaseStageTma34f = PhaseStageTmaT<float, 34>;
static_assert(offsetof(PhaseStageTma34, I) % 128 == 0, "TMA destinations are 128-byte aligned");
static_assert(offsetof(PhaseStageTma34f, I) % 128 == 0, "TMA destinations are 128-byte aligned");
// shared bytes of the face tables in front of the ring (a 128-byte multiple)
template <class T>
constexpr size_t ph_ft_bytes() { return (PH_FT * sizeof(T) + 127) / 128 * 128; }

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

// CONS: a thread's RY rows are consecutive (rows ly*RY .. ly*RY+RY-1 of the
// tile instead of ly, ly+8, ...), so a row's y neighbours inside the group
// are the neighbouring rows' own values and phases, already in registers,
// and the y face between two of them is looked up once
template <int N, bool PCG = true, class T = double, int RY = 2, bool CONS = false>
__global__ void __launch_bounds__(256, 4)
    k_stencil_pht(Geom g, int kchunk, const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap mi,
                  const unsigned char* __restrict__ pidx, const T* __restrict__ ftab, const T* __restrict__ wv,
                  T* __restrict__ qout, Ctl* ctl, double* partials, unsigned* counter) {
  if (PCG && ctl->done) return;
  constexpr int RH = 8 * RY, HB = RH + 2;  // tile rows; box rows with the halo
  using Stage = PhaseStageTmaT<T, HB>;
  constexpr int S = 4, T2 = PH_TS, WX = Stage::WX, WPD = 64 / sizeof(T);
  constexpr long long P = (long long)N * N;
  extern __shared__ __align__(128) double smem_t[];
  T* FT = reinterpret_cast<T*>(smem_t);  // PH_FT entries, padded to a 128-byte multiple
  Stage* st = reinterpret_cast<Stage*>(reinterpret_cast<unsigned char*>(smem_t) + ph_ft_bytes<T>());
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(st + S);
  const int lx = threadIdx.x, ly = threadIdx.y, tid = ly * 32 + lx;
  for (int e = tid; e < 3 * PH_MAX * PH_MAX + PH_MAX; e += 256) FT[ph_slot(e)] = ftab[e];
  for (int e = tid; e < S * WPD; e += 256) st[e / WPD].wpad[e % WPD] = 0;
  for (int e = tid; e < S * 64; e += 256) st[e / 64].I18[e % 64] = 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nz = g.nz, kg0 = g.kg0, nzg = g.nzg;
  const int i0 = blockIdx.x * 32, i = i0 + lx, j0 = blockIdx.y * RH;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(nz, k0 + kchunk);
  const int kmax = min(k1, nzg - 1 - kg0);
  const int ox = min(max(i0 - Stage::XO, 0), N - WX), oxi = min(max(i0 - 16, 0), N - 64),
            oy = min(max(j0 - 1, 0), N - HB);
  auto issue = [&](int k) {  // planes k0 .. k1 (the last clamped: the z+ neighbour of k1-1)
    if (tid == 0 && k <= k1) {
      const int kk = min(k, kmax), s = k % S;
      mbar_expect_tx(&bar[s], Stage::TX);
      tma_load_3d(&st[s].W[0][0], &mw, ox, oy, kk, &bar[s]);
      tma_load_3d(&st[s].I[0][0], &mi, oxi, oy, kk, &bar[s]);
    }
  };
  double dqw = 0.0, dqq = 0.0, dww = 0.0;
  if (k0 < k1) {
    const bool interior = i0 > 0 && i0 + 32 < N && j0 > 0 && j0 + RH < N;
    T um[RY], fzm[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      um[r] = 0;
      fzm[r] = 0;
      if (kg0 + k0 > 0) {  // plane k0-1 may be the lower halo
        const long long o = (long long)(k0 - 1) * P + (long long)(j0 + (CONS ? ly * RY + r : ly + 8 * r)) * N + i;
        um[r] = wv[o];
        fzm[r] = FT[2 * T2 + pidx[o] * PH_RS + pidx[o + P]];
      }
    }
    issue(k0);
    issue(k0 + 1);
    issue(k0 + 2);
    const int ly0 = CONS ? ly * RY : ly, rs = CONS ? 1 : 8;  // the thread's first row, row step
    const int wo = (j0 + ly0 - oy) * WX + (i - ox), io = (j0 + ly0 - oy) * 64 + (i - oxi);  // cell offsets, r = 0
    T ucur[RY];
    int pcur[RY];
    for (int k = k0; k < k1; ++k) {
      // stage k landed (waited as the z+ plane last time round), stage k+1 now
      mbar_wait(&bar[k % S], ((k - k0) / S) & 1);
      mbar_wait(&bar[(k + 1) % S], ((k + 1 - k0) / S) & 1);
      __syncthreads();  // every warp is done with plane k-1: its stage is refilled
      issue(k + 3);
      const Stage& c = st[k % S];
      const Stage& nx_ = st[(k + 1) % S];
      const bool hasp = kg0 + k + 1 < nzg;
      if (k == k0) {
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          ucur[r] = (&c.W[0][0])[wo + rs * WX * r];
          pcur[r] = (&c.I[0][0])[io + rs * 64 * r];
        }
      }
      if constexpr (CONS) {
        constexpr int R = PH_RS;
        T unext[RY];
        int pnext[RY];
        // the plane's rows; MASK (edge blocks only) applies the boundary masks
        auto rows = [&](auto mk) {
        constexpr bool MASK = decltype(mk)::value;
        T fyprev = 0;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          const int j = j0 + ly0 + r;
          const T* Wc = &c.W[0][0] + wo + WX * r;
          const unsigned char* Ic = &c.I[0][0] + io + 64 * r;
          const T uc = ucur[r];
          const int pc = pcur[r];
          const T* FX = FT + pc;       // [a][pc]
          const T* FXr = FT + pc * R;  // [pc][b]
          const T fxm = FX[Ic[-1] * R], fxp = FXr[Ic[1]];
          const T wup = r == 0 ? Wc[-WX] : ucur[r > 0 ? r - 1 : 0];
          const T fym = r == 0 ? FX[T2 + Ic[-64] * R] : fyprev;
          const T wdn = r == RY - 1 ? Wc[WX] : ucur[r < RY - 1 ? r + 1 : 0];
          const int pdn = r == RY - 1 ? (int)Ic[64] : pcur[r < RY - 1 ? r + 1 : 0];
          const T fyp = FXr[T2 + pdn];
          fyprev = fyp;
          T acc = 0, t;
          t = add_rn(acc, mul_rn(fxm, sub_rn(uc, Wc[-1])));
          acc = (!MASK || i > 0) ? t : acc;
          t = sub_rn(acc, mul_rn(fxp, sub_rn(Wc[1], uc)));
          acc = (!MASK || i + 1 < N) ? t : acc;
          t = add_rn(acc, mul_rn(fym, sub_rn(uc, wup)));
          acc = (!MASK || j > 0) ? t : acc;
          t = sub_rn(acc, mul_rn(fyp, sub_rn(wdn, uc)));
          acc = (!MASK || j + 1 < N) ? t : acc;
          if (kg0 + k > 0) acc = add_rn(acc, mul_rn(fzm[r], sub_rn(uc, um[r])));
          const T un = (&nx_.W[0][0])[wo + WX * r];
          const int pn = (&nx_.I[0][0])[io + 64 * r];
          T fzp = 0;
          if (hasp) {
            fzp = FXr[2 * T2 + pn];
            acc = sub_rn(acc, mul_rn(fzp, sub_rn(un, uc)));
          }
          if (kg0 + k == 0) acc = add_rn(acc, mul_rn(FT[3 * T2 + pc], uc));
          if (kg0 + k == nzg - 1) acc = add_rn(acc, mul_rn(FT[3 * T2 + pc], uc));
          qout[(long long)k * P + (long long)j * N + i] = acc;
          if (PCG) {
            const double a_ = acc, u_ = uc;
            dqw = fma(a_, u_, dqw);
            dqq = fma(a_, a_, dqq);
            dww = fma(u_, u_, dww);
          }
          unext[r] = un;
          pnext[r] = pn;
          um[r] = uc;
          fzm[r] = fzp;
        }
        };
        if (interior)
          rows(std::false_type{});
        else
          rows(std::true_type{});
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          ucur[r] = unext[r];
          pcur[r] = pnext[r];
        }
        continue;
      }
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const int j = j0 + ly0 + rs * r;
        const int w_ = wo + rs * WX * r, i_ = io + rs * 64 * r;
        const T uc = ucur[r];
        const int pc = pcur[r];
        T fzp;
        T acc = interior ? ph_cell_p<N, false, WX, 64>(&c.W[0][0] + w_, &c.I[0][0] + i_, &nx_.W[0][0] + w_,
                                                       &nx_.I[0][0] + i_, FT, i, j, kg0 + k > 0, hasp, uc, pc,
                                                       um[r], fzm[r], fzp, ucur[r], pcur[r])
                         : ph_cell_p<N, true, WX, 64>(&c.W[0][0] + w_, &c.I[0][0] + i_, &nx_.W[0][0] + w_,
                                                      &nx_.I[0][0] + i_, FT, i, j, kg0 + k > 0, hasp, uc, pc,
                                                      um[r], fzm[r], fzp, ucur[r], pcur[r]);
        if (kg0 + k == 0) acc = add_rn(acc, mul_rn(FT[3 * T2 + pc], uc));
        if (kg0 + k == nzg - 1) acc = add_rn(acc, mul_rn(FT[3 * T2 + pc], uc));
        qout[(long long)k * P + (long long)j * N + i] = acc;
        if (PCG) {
          const double a_ = acc, u_ = uc;
          dqw = fma(a_, u_, dqw);
          dqq = fma(a_, a_, dqq);
          dww = fma(u_, u_, dww);
        }
        um[r] = uc;
        fzm[r] = fzp;
      }
    }
  }
  if (!PCG) return;
  double v[3] = {dqw, dqq, dww};
  grid_sum_finalize<3>(v, partials, counter, [&](double (&t)[3]) {
    if (ctl->dist) {
      ctl->xbuf[0] = t[0];
      ctl->xbuf[1] = t[1];
      ctl->xbuf[2] = t[2];
    } else {
      if constexpr (sizeof(T) == 4)
        fin_stencil32(ctl, t[0], t[1], t[2]);
      else
        fin_stencil(ctl, t[0], t[1], t[2]);
    }
  });
}

// ---- q = A w for general fields (stored faces tx, ty, tz; the fused
// solve's stencil when the field has more than PH_MAX phases), staged like
// k_stencil_pht: a 32 x 16 tile, two rows per thread, marching along z with
// plane k+3 streaming into a 4-deep shared ring by TMA -- four 36 x 18 boxes
// per plane (w with its halo, tx, ty, tz; origins 16-byte aligned and clamped
// into the grid) on one mbarrier, so the consumer warps issue no global
// loads.  Arithmetic order of k_stencil_cp (tpfa.py:117-130, no FMA): bitwise.
template <class E>  // element type: boxes 36 (double) or 40 (float) wide
struct alignas(128) GenStageTmaT {  // each box padded to a 128-byte multiple (TMA destinations)
  static constexpr int WX = sizeof(E) == 8 ? 36 : 40, XO = sizeof(E) == 8 ? 2 : 4, PD = 64 / sizeof(E);
  E W[18][WX];
  E pw[PD];
  E X[18][WX];
  E px[PD];
  E Y[18][WX];
  E py[PD];
  E T[18][WX];
  E pt[PD];
  static constexpr unsigned TX = 4 * sizeof(E) * 18 * WX;
};
using GenStageTma = GenStageTmaT<double>;
static_assert(offsetof(GenStageTmaT<double>, X) % 128 == 0 && offsetof(GenStageTmaT<double>, Y) % 128 == 0 &&
                  offsetof(GenStageTmaT<double>, T) % 128 == 0 && sizeof(GenStageTmaT<double>) % 128 == 0,
              "TMA destinations are 128-byte aligned");
static_assert(offsetof(GenStageTmaT<float>, X) % 128 == 0 && offsetof(GenStageTmaT<float>, Y) % 128 == 0 &&
                  offsetof(GenStageTmaT<float>, T) % 128 == 0 && sizeof(GenStageTmaT<float>) % 128 == 0,
              "TMA destinations are 128-byte aligned");

template <int N, bool PCG = true, class E = double>
__global__ void __launch_bounds__(256, 2)
    k_stencil_gt(Geom g, int kchunk, const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap mx,
                 const __grid_constant__ CUtensorMap my, const __grid_constant__ CUtensorMap mt,
                 const E* __restrict__ wv, const E* __restrict__ tz, const E* __restrict__ tb, E* __restrict__ qout,
                 Ctl* ctl, double* partials, unsigned* counter) {
  if (PCG && ctl->done) return;
  constexpr int S = 4, RY = 2, RH = 16;
  constexpr long long P = (long long)N * N;
  extern __shared__ __align__(128) double smem_g[];
  using Stage = GenStageTmaT<E>;
  Stage* st = reinterpret_cast<Stage*>(smem_g);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(st + S);
  const int lx = threadIdx.x, ly = threadIdx.y, tid = ly * 32 + lx;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nz = g.nz, kg0 = g.kg0, nzg = g.nzg;
  const int i0 = blockIdx.x * 32, i = i0 + lx, j0 = blockIdx.y * RH;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(nz, k0 + kchunk);
  const int kmax = min(k1, nzg - 1 - kg0);  // last plane of w read (the z+ neighbour, maybe the upper halo)
  const int ox = min(max(i0 - Stage::XO, 0), N - Stage::WX), oy = min(max(j0 - 1, 0), N - 18);
  auto issue = [&](int k) {  // planes k0 .. k1 (face boxes only below k1)
    if (tid == 0 && k <= k1) {
      const int s = k % S;
      mbar_expect_tx(&bar[s], Stage::TX);
      tma_load_3d(&st[s].W[0][0], &mw, ox, oy, min(k, kmax), &bar[s]);
      const int kf = min(k, k1 - 1);  // the last stage's face boxes are never read: reload a valid plane
      tma_load_3d(&st[s].X[0][0], &mx, ox, oy, kf, &bar[s]);
      tma_load_3d(&st[s].Y[0][0], &my, ox, oy, kf, &bar[s]);
      tma_load_3d(&st[s].T[0][0], &mt, ox, oy, kf, &bar[s]);
    }
  };
  double dqw = 0.0, dqq = 0.0, dww = 0.0;
  if (k0 < k1) {
    E um[RY], fzm[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      um[r] = 0;
      fzm[r] = 0;
      if (kg0 + k0 > 0) {  // plane k0-1 may be the lower halo
        const long long o = (long long)(k0 - 1) * P + (long long)(j0 + ly + 8 * r) * N + i;
        um[r] = wv[o];
        fzm[r] = tz[o];
      }
    }
    issue(k0);
    issue(k0 + 1);
    issue(k0 + 2);
    const int cx = i - ox;  // the cell's column in the boxes
    for (int k = k0; k < k1; ++k) {
      mbar_wait(&bar[k % S], ((k - k0) / S) & 1);
      mbar_wait(&bar[(k + 1) % S], ((k + 1 - k0) / S) & 1);
      __syncthreads();  // every warp is done with plane k-1: its stage is refilled
      issue(k + 3);
      const Stage& c = st[k % S];
      const Stage& nx_ = st[(k + 1) % S];
      const bool hasp = kg0 + k + 1 < nzg;
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const int j = j0 + ly + 8 * r, cy = j - oy;
        const E uc = c.W[cy][cx];
        E acc = 0;
        if (i > 0) acc = add_rn(acc, mul_rn(c.X[cy][cx - 1], sub_rn(uc, c.W[cy][cx - 1])));
        if (i + 1 < N) acc = sub_rn(acc, mul_rn(c.X[cy][cx], sub_rn(c.W[cy][cx + 1], uc)));
        if (j > 0) acc = add_rn(acc, mul_rn(c.Y[cy - 1][cx], sub_rn(uc, c.W[cy - 1][cx])));
        if (j + 1 < N) acc = sub_rn(acc, mul_rn(c.Y[cy][cx], sub_rn(c.W[cy + 1][cx], uc)));
        if (kg0 + k > 0) acc = add_rn(acc, mul_rn(fzm[r], sub_rn(uc, um[r])));
        const E fzp = c.T[cy][cx];
        if (hasp) acc = sub_rn(acc, mul_rn(fzp, sub_rn(nx_.W[cy][cx], uc)));
        const long long col = (long long)j * N + i;
        if (kg0 + k == 0) acc = add_rn(acc, mul_rn(tb[col], uc));
        if (kg0 + k == nzg - 1) acc = add_rn(acc, mul_rn(tb[P + col], uc));
        qout[(long long)k * P + col] = acc;
        if (PCG) {
          const double a_ = acc, u_ = uc;
          dqw = fma(a_, u_, dqw);
          dqq = fma(a_, a_, dqq);
          dww = fma(u_, u_, dww);
        }
        um[r] = uc;
        fzm[r] = fzp;
      }
    }
  }
  if (!PCG) return;
  double v[3] = {dqw, dqq, dww};
  grid_sum_finalize<3>(v, partials, counter, [&](double (&t)[3]) {
    if (ctl->dist) {
      ctl->xbuf[0] = t[0];
      ctl->xbuf[1] = t[1];
      ctl->xbuf[2] = t[2];
    } else if constexpr (sizeof(E) == 4) {
      fin_stencil32(ctl, t[0], t[1], t[2]);
    } else {
      fin_stencil(ctl, t[0], t[1], t[2]);
    }
  });
}

// ---- face transmissibilities, once per solve (tpfa.py:91-107): harmonic
// means ((2a)*b)/(a+b) of the scaled coefficients (lower cell first);
// tb = [t_in plane | t_out plane] = 2 s_z on the first / last layer.
__global__ void k_faces(Geom g, const double* __restrict__ sx, const double* __restrict__ sy,
                        const double* __restrict__ sz, double* __restrict__ tx, double* __restrict__ ty,
                        double* __restrict__ tz, double* __restrict__ tb) {
  // z-slab ranks: sz carries halo planes -1 and nz; tz[-1] (face kg0-1/2) is
  // built too, so the stencil finds both faces of its boundary planes
  const int nx = g.nx, ny = g.ny, nz = g.nz, kg0 = g.kg0, nzg = g.nzg;
  const long long n = g.n, P = g.plane;
  const long long lo = (kg0 > 0) ? -P : 0;
  for (long long c = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const long long k = (c + P) / P - 1, rem = c - k * P;
    const int kg = kg0 + (int)k;
    tz[c] = (kg + 1 < nzg) ? harm(sz[c], sz[c + P]) : 0.0;
    if (k < 0) continue;
    const int j = (int)(rem / nx), i = (int)(rem - (long long)j * nx);
    tx[c] = (i + 1 < nx) ? harm(sx[c], sx[c + 1]) : 0.0;
    ty[c] = (j + 1 < ny) ? harm(sy[c], sy[c + nx]) : 0.0;
    if (kg == 0) tb[rem] = __dmul_rn(2.0, sz[c]);
    if (kg == nzg - 1) tb[P + rem] = __dmul_rn(2.0, sz[c]);
  }
  (void)ny;
}
