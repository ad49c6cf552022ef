/*
 * etc_b200.h — C ABI of the B200-native effective-thermal-conductivity solver
 * (arXiv 2404.02433 reference: /root/reference/pkg/src/etchomo, "etchomo").
 *
 * The reference is pure Python; its hot path is `homogenize()`
 * (pipeline.py:135-175) driving `pcg()` (krylov.py:36-91) with two operator
 * callables: `apply_operator` (tpfa.py:110-131) and `FctPreconditioner`
 * (preconditioner.py:273-282).  This header is the plugin boundary a
 * maintainer binds from Python with ctypes; every entry
 * point below names the reference interface it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or CUDA types in signatures
 *    (`stream` is a cudaStream_t passed as void*; NULL = legacy stream).
 *  - Arrays are float64, x-fastest: cell (i,j,k) at (k*ny + j)*nx + i
 *    (reference grid.py:1-7).
 *  - Return codes: ETC_OK 0; ETC_BREAKDOWN 1 (PcgBreakdownError,
 *    krylov.py:12-17); ETC_CONFIG 2 (ConfigError / ValueError); ETC_CUDA 3;
 *    ETC_PIVOT 4 (FloatingPointError, preconditioner.py:229-244).
 *    etc_last_error() returns a thread-local message for the last failure.
 *  - A plan owns its device workspace and is not re-entrant (one solve at a
 *    time per plan), mirroring SlabBuffer (transforms.py:136-138).
 */
#ifndef ETC_B200_H
#define ETC_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct etc_plan etc_plan;

enum {
  ETC_OK = 0,
  ETC_BREAKDOWN = 1,
  ETC_CONFIG = 2,
  ETC_CUDA = 3,
  ETC_PIVOT = 4
};

/* Preconditioner plugin kinds (reference tags "fct" | "jacobi" | "none",
 * pipeline.py:114-132). */
enum {
  ETC_PRECOND_FCT = 0,    /* FctPreconditioner (preconditioner.py:253-282) */
  ETC_PRECOND_JACOBI = 1, /* JacobiPreconditioner (preconditioner.py:324-330) */
  ETC_PRECOND_NONE = 2    /* identity_apply (preconditioner.py:337-338)    */
};

/* Outcome of one solve (reference SolveReport, krylov.py:20-33). */
typedef struct {
  int iterations;      /* == len(history) - 1                              */
  int converged;       /* history[-1] <= rtol                              */
  int status;          /* ETC_OK or ETC_BREAKDOWN                          */
  int breakdown_iter;  /* PcgBreakdownError.iteration when status == 1     */
  int breakdown_kind;  /* 1 operator, 2 residual not finite, 3 precond     */
  int pad_;
  double kappa_eff;    /* effective_conductivity (tpfa.py:254-258)         */
  double flux_sum;     /* sum of outflow fluxes (tpfa.py:234-251)          */
  double norm_b;       /* ||b||                                            */
  double device_ms;    /* device time of the PCG loop (CUDA events)        */
} etc_solve_info;

const char* etc_last_error(void);
int etc_version(void);

/* Plan for an ORIGINAL-orientation grid nx*ny*nz with edge lengths lx,ly,lz
 * (reference GridSpec, grid.py:42-90).  Allocates the device workspace. */
int etc_plan_create(etc_plan** out, int nx, int ny, int nz,
                    double lx, double ly, double lz, void* stream);
int etc_plan_destroy(etc_plan* plan);
/* Bytes of device memory owned by the plan. */
size_t etc_plan_device_bytes(const etc_plan* plan);

/* Copy the conductivity field (OrthotropicField kx, ky, kz; grid.py:102-159)
 * into plan-owned device storage.  `on_device` != 0: the pointers are device
 * pointers; otherwise host pointers (H2D copies on the plan stream).  When
 * kx == ky == kz (same pointer) the field is stored once. */
int etc_load_field(etc_plan* plan, const double* kx, const double* ky,
                   const double* kz, int on_device);

/* Rotate the loaded field so `axis` (0 x, 1 y, 2 z) becomes canonical z and
 * scale by 1/h^2: replaces axis_permute (pipeline.py:87-111) + scale_field
 * (tpfa.py:19-26).  dims_out/len_out receive the canonical grid. */
int etc_select_axis(etc_plan* plan, int axis, int dims_out[3], double len_out[3]);

/* Exact extremes of the face transmissibilities (coefficient_stats,
 * preconditioner.py:94-108), order x,y,z,in,out as (min,max) pairs. */
int etc_coefficient_stats(etc_plan* plan, double out[10]);

/* Reference constants chosen on the host (solve_reference_lp / ones_reference,
 * preconditioner.py:117-140) and the host-built tables of TridiagFactors
 * (preconditioner.py:178-199): weights_x[nx], weights_y[ny], z_diag[nz]
 * of the canonical grid.  refs = {kx, ky, kz, kin, kout}. */
int etc_set_reference(etc_plan* plan, const double refs[5], const double* weights_x,
                      const double* weights_y, const double* z_diag);

/* Full PCG solve of the canonical system with Dirichlet data p_in/p_out:
 * build_rhs (tpfa.py:150-167) + pcg (krylov.py:36-91) + outflow flux and
 * kappa_eff (tpfa.py:234-258), device-resident.  hist_host (capacity
 * max_iter+1) receives the relative-residual history. */
int etc_solve(etc_plan* plan, double p_in, double p_out, double rtol, int max_iter,
              etc_solve_info* info, double* hist_host);

/* homogenize() only observes the potential p on the outflow plane
 * (reconstruct_boundary_flux, tpfa.py:234-251), so by default the solve
 * updates p on that plane only.  keep != 0 makes etc_solve keep the full
 * solution vector (reference pcg() output, krylov.py:91) for
 * etc_get_solution. */
int etc_keep_solution(etc_plan* plan, int keep);

/* Select the preconditioner of the following etc_solve calls
 * (_make_preconditioner, pipeline.py:125-132): ETC_PRECOND_FCT (default),
 * ETC_PRECOND_JACOBI (r * 1/diag(A), diag in the accumulation order of
 * operator_diagonal, tpfa.py:134-147) or ETC_PRECOND_NONE (z = r).  SSOR
 * (SciPy SuperLU sweeps) is out of scope and has no kind. */
int etc_set_precond(etc_plan* plan, int kind);

/* Arithmetic precision of the following etc_coefficient_stats / etc_solve
 * calls (homogenize's precision="f64" | "f32", pipeline.py:147-160): 64
 * (default) or 32.  At 32 the field is cast to float32 and the faces,
 * operator, transforms, z elimination and PCG vectors are float32, as the
 * reference does with dtype float32; the statistics then come from the
 * float32 faces.  Single-GPU plans; fct, jacobi and none preconditioners
 * (fct on square power-of-two planes with nz = 32 L, L in {4, 8, 16, 32}, runs
 * the float64 solve's fused kernels instantiated on float). */
int etc_set_precision(etc_plan* plan, int bits);

/* Copy the solution vector p of the last solve (canonical layout); requires
 * etc_keep_solution(plan, 1) before the solve. */
int etc_get_solution(etc_plan* plan, double* dst, int dst_on_device);

/* ---- operator-level entry points (device pointers, canonical layout) ---- */
/* apply_operator(sys, u) (tpfa.py:110-131). */
int etc_apply_operator(etc_plan* plan, const double* u, double* out);
/* FctPlan.forward: plane-wise 2-D DCT-II (transforms.py:83-104). */
int etc_dct2_xy(etc_plan* plan, const double* in, double* out);
/* FctPlan.backward: exact inverse (transforms.py:108-133). */
int etc_dct3_xy(etc_plan* plan, const double* in, double* out);
/* thomas_solve_batch on spectral data, in place (preconditioner.py:215-250). */
int etc_thomas(etc_plan* plan, double* inout);
/* FctPreconditioner.__call__ (preconditioner.py:253-282). */
int etc_apply_precond(etc_plan* plan, const double* r, double* z);
/* build_rhs (tpfa.py:150-167). */
int etc_build_rhs(etc_plan* plan, double p_in, double p_out, double* out);

/* Per-kernel device timing for measurement (bench.py): when enabled, every
 * launch is bracketed by CUDA events on the plan stream.  Kernel classes:
 * 0 stencil (+ w update, p update, dots), 1 r update + 2-D DCT-II, 2 plain
 * 2-D DCT-II, 3 z-solve, 4 unused, 5 2-D DCT-III, 6 setup (rhs, ||b|| +
 * first transform, flux, stats, permute/scale, final p update).  Launch counts are kept
 * even when timing is off.  `reset` != 0 clears both after reading. */
int etc_profile(etc_plan* plan, int enable);
int etc_profile_read(etc_plan* plan, double ms[8], long long counts[8], int reset);

/* ---- z-slab ranks of a multi-GPU solve --------------------
 * The canonical (already axis-rotated) grid nx x ny x nzg is split into P
 * equal z-slabs; this plan holds planes [k0, k0+nzl) and, for the z-solve,
 * the pencil of rows [rank*ny/P, (rank+1)*ny/P) over all nzg planes.  The
 * host moves data between ranks (NCCL through torch.distributed): the s and z
 * halo planes (etc_slab_plane), the pencil all-to-all around SLAB_ZSOLVE, and
 * the all-reduce of the 8 scalar partials in `xbuf` before SLAB_FINALIZE.
 * Stages for etc_slab_run: 0 faces, 1 stats (ext = 10 doubles), 2 ||b|| and
 * first transform, 3 finalize (arg: 0 stencil, 1 ||b||, 2 update, 3 z-solve),
 * 4 stencil (arg = iteration), 5 r update + transform, 6 pack (ext = send),
 * 7 z-solve (ext = pencil), 8 unpack (ext = received), 9 inverse transform,
 * 10 final p update (arg = last iteration), 11 outflow flux (ext = 1 double),
 * substructured z-solve instead of 6-8 (replaces the pencil
 * all-to-alls, preconditioner.py:215-250 on each rank's block of rows):
 * 12 spike tables (once per solve, after etc_set_reference; nranks <= 8),
 * 13 block end values g_first/g_last (ext = 2 nx ny doubles, this rank's),
 * 14 reduced system + coupled block solve in place (ext = all ranks' stage-13
 * outputs, all-gathered: nranks x 2 nx ny doubles).
 * Same kernels as the single-GPU path; krylov.py:56-90 semantics. */
int etc_slab_create(etc_plan** out, int nx, int ny, int nzg, int k0, int nzl, int nranks, int rank,
                    double lx, double ly, double lz, void* stream);
int etc_slab_load(etc_plan* plan, const double* kx, const double* ky, const double* kz, int on_device);
/* which: 0..2 s_x,s_y,s_z, 3 z, 4 w (fused path); plane -1..nzl (halo planes -1 and nzl);
 * to_ext != 0 copies plan -> ext, else ext -> plan (device pointers). */
int etc_slab_plane(etc_plan* plan, int which, int plane, double* ext, int to_ext);
int etc_slab_init(etc_plan* plan, double p_in, double p_out, double rtol, int max_iter, double* xbuf);
int etc_slab_run(etc_plan* plan, int stage, int arg, double* ext);
/* ctl state + history; info->pad_ carries the device `done` flag. */
int etc_slab_status(etc_plan* plan, etc_solve_info* info, double* hist_host);

/* 1 if this slab plan runs the fused search-direction path (square
 * power-of-two planes): the inverse stage builds w (arg 1: w = z, arg 2:
 * p += alpha w_old on the outflow plane, w = z + beta w_old), the stencil
 * stage reads w, and the host exchanges w halo planes (etc_slab_plane
 * which = 4) instead of z (which = 3) after the inverse. */
int etc_slab_fused(etc_plan* plan);

/* Peer exchange (fused all-to-all over peer memory): 1 if this slab plan
 * can run it (fused path, exact-fit z-solve on the pencil). */
int etc_slab_p2p_ok(etc_plan* plan);
/* The plan's exchange buffers (device, allocated on first request):
 * which 0 = pencil (recv) buffer, 1 = return buffer (nzl*ny*nx doubles
 * each), 2 = the spike z-solve's end values of all ranks (nranks*2*ny*nx). */
int etc_slab_xbuf(etc_plan* plan, int which, double** out);
/* Every rank's pencil and return buffers as pointers valid in this process
 * (own, same-process, or CUDA-IPC-opened), nranks entries each; NULL turns
 * the peer exchange off.  With peers set, SLAB_NORMB/SLAB_UPDATE store the
 * spectrum into the destination ranks' pencil buffers and SLAB_ZSOLVE stores
 * its rows into the owners' return buffers (no all-to-all); the host's
 * following scalar all-reduce is the barrier. */
int etc_slab_set_peers(etc_plan* plan, double* const* recv_peers, double* const* back_peers);
/* Spike z-solve over peer memory: SLAB_ZSUB_ENDS stores this rank's end
 * values into slot `rank` of every rank's etc_slab_xbuf(plan, 2, ...) buffer
 * (nranks x 2 nx ny doubles; device pointers valid in this process, own or
 * IPC-opened), replacing the host all-gather; SLAB_ZSUB_SOLVE with ext = NULL
 * reads the own buffer.  NULL table: back to the all-gather. */
int etc_slab_set_ends_peers(etc_plan* plan, double* const* ends_peers);
/* Device address of plane `plane` (-1..nzl) of buffer `which` (as
 * etc_slab_plane): the target of the peers' halo-plane stores. */
int etc_slab_plane_ptr(etc_plan* plan, int which, int plane, double** out);
/* CUDA IPC helpers for multi-process ranks: the 64-byte handle of the plan
 * allocation holding dev_ptr and dev_ptr's byte offset in it; open / close a
 * peer's handle (the opened base + offset is the peer's pointer). */
int etc_ipc_handle(etc_plan* plan, const void* dev_ptr, void* handle_out, size_t* offset_out);
int etc_ipc_open(const void* handle_in, void** dev_ptr);
int etc_ipc_close(void* dev_ptr);

/* Voxelise gen_random_balls / gen_center_ball (grid.py:230-275) on the device:
 * balls = count x (cx, cy, cz, r) drawn on the host; out = n^3 cube of
 * kappa_inc inside any ball, 1.0 elsewhere (bit-identical membership test). */
int etc_voxelize_balls(double* out_dev, int n, const double* balls_host, int count,
                       double kappa_inc, void* stream);

/* Aligned-fibre field (no reference generator exists; SURVEY 8(d) config 3
 * asks for a documented deterministic one, see grid.gen_fibres): fibres =
 * count x (c1, c2, r) drawn on the host, cylinders through the whole cube
 * along axis (0 x, 1 y, 2 z); out = kappa_fib inside, 1.0 elsewhere, with
 * the ball voxeliser's cell centres and ((d1*d1) + (d2*d2)) <= r*r test. */
int etc_voxelize_fibres(double* out_dev, int n, const double* fibres_host, int count,
                        double kappa_fib, int axis, void* stream);

/* gen_channels (grid.py:287-319) on the device: n = cells_per_period *
 * periods; (cx, cy, cz) = (2^psi, 5^psi, 10^psi) in the channels,
 * Diag(0.01, 0.1, 1) elsewhere. */
int etc_fill_channels(double* kx_dev, double* ky_dev, double* kz_dev, int cells_per_period, int periods,
                      double cx, double cy, double cz, void* stream);

/* ---------------------------------------------------------------------------
 * Operator-plugin layer (the reference's lower-level exports,
 * __init__.py:9-71), used by paper_2404_02433_b200.plugin.
 * ------------------------------------------------------------------------ */

/* Geometry-only plan (no field): what FctPlan (transforms.py:56-61) and
 * FctPreconditioner (preconditioner.py:273-282) need — etc_set_reference,
 * then etc_dct2_xy / etc_dct3_xy / etc_thomas / etc_apply_precond (and the
 * float32 variants below).  Field entry points fail with ETC_CONFIG. */
int etc_plan_bare(etc_plan* plan);

/* float32 transforms and preconditioner (FctPlan / FctPreconditioner with
 * dtype=float32; the line passes of the f32 solve).  z != r. */
int etc_dct2_xy_f32(etc_plan* plan, const float* in, float* out);
int etc_dct3_xy_f32(etc_plan* plan, const float* in, float* out);
int etc_apply_precond_f32(etc_plan* plan, const float* r, float* z);

/* Stateless kernels on the reference's own data structures (etc_plugin.cu).
 * prec: 0 float64, 1 float32 (every array of the call).  Arrays are device
 * pointers; faces are a DiscreteSystem's compact arrays (tpfa.py:33-88):
 * tx (nx-1)*ny*nz, ty nx*(ny-1)*nz, tz nx*ny*(nz-1), t_in / t_out nx*ny.
 * Elementwise results follow numpy's operation order (bitwise). */
const char* etc_op_last_error(void);
/* doubles of device scratch the reductions below need for n elements */
int etc_op_reduce_parts(long long n);
/* apply_operator (tpfa.py:110-131) */
int etc_op_stencil(int prec, int nx, int ny, int nz, const void* tx, const void* ty, const void* tz,
                   const void* t_in, const void* t_out, const void* u, void* out, void* stream);
/* operator_diagonal (tpfa.py:134-147) */
int etc_op_diagonal(int prec, int nx, int ny, int nz, const void* tx, const void* ty, const void* tz,
                    const void* t_in, const void* t_out, void* out, void* stream);
/* build_system's faces from scale_field's cubes (tpfa.py:91-107) */
int etc_op_faces(int prec, int nx, int ny, int nz, const void* sx, const void* sy, const void* sz, void* tx,
                 void* ty, void* tz, void* t_in, void* t_out, void* stream);
/* scale_field (tpfa.py:19-26): s = k / h2, h2 = dtype(h)**2 */
int etc_op_scale(int prec, long long n, const void* k, double h2, void* s, void* stream);
/* axis_permute of one cube (pipeline.py:87-111): axis 0 swapaxes(0,2), 1 swapaxes(0,1) */
int etc_op_permute(int prec, int nx, int ny, int nz, int axis, const void* src, void* dst, void* stream);
/* build_rhs (tpfa.py:150-167): p_in / p_out planes (ny*nx) or, when NULL, the scalars */
int etc_op_rhs(int prec, int nx, int ny, int nz, const void* t_in, const void* t_out, const void* pin_plane,
               double pin, const void* pout_plane, double pout, void* b, void* stream);
/* reconstruct_boundary_flux (tpfa.py:234-251): side_out 1 "out", 0 "in" */
int etc_op_flux(int prec, int nx, int ny, int nz, const void* t_layer, double hz, const void* u, double pval,
                int side_out, void* out, void* stream);
/* thomas_solve_batch (preconditioner.py:215-250), in place on x; upper:
 * (nz-1)*ny*nx scratch; returns ETC_PIVOT with the first non-positive pivot's
 * layer in *bad_layer (bad_dev: one device int of scratch) */
int etc_op_thomas(int prec, int nx, int ny, int nz, const void* shift, const void* z_diag, double off, void* x,
                  void* upper, int* bad_dev, int* bad_layer, void* stream);
/* kind 0: out = a*b, 1: out = 1/a, 2: out = a+b */
int etc_op_elementwise(int prec, int kind, long long n, const void* a, const void* b, void* out, void* stream);
/* deterministic float64 reductions into out (device): kind 0 a.b, 1 (a.b, a.a, b.b), 2 sum(a) */
int etc_op_dots(int prec, int kind, long long n, const void* a, const void* b, double* parts, double* out,
                void* stream);
/* pcg's update (krylov.py:76-77): p += alpha w; r -= alpha z; *rr_out (device) = r.r */
int etc_op_pcg_update(int prec, long long n, double alpha, void* p, const void* w, void* r, const void* z,
                      double* parts, double* rr_out, void* stream);
/* w = z + beta w (krylov.py:89) */
int etc_op_xpby(int prec, long long n, const void* z, double beta, void* w, void* stream);
/* exact (min, max) of a positive array into out (host; mm: 2 device uint64) */
int etc_op_minmax(int prec, long long n, const void* a, void* mm, double out[2], void* stream);
/* SsorPreconditioner apply (preconditioner.py:285-321), float64: the two
 * triangular sweeps of the stencil in natural order, level-scheduled */
int etc_op_ssor(int nx, int ny, int nz, const double* tx, const double* ty, const double* tz, const double* diag,
                double omega, const double* r, double* out, void* stream);
/* assemble_dense (tpfa.py:181-205), float64, n = nx*ny*nz <= 4096: mat n*n */
int etc_op_dense(int nx, int ny, int nz, const double* tx, const double* ty, const double* tz,
                 const double* t_in, const double* t_out, double* mat, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ETC_B200_H */
