/*
 * mgrit_b200.h -- C ABI of the B200-native MGRIT hot path (libmgrit_b200.so).
 *
 * The reference (mgrit-advection 0.1.0, pure Python + numpy) has no FFI; every
 * entry point below replaces one numpy call site or solver primitive of its
 * time-parallel hot path.  Citations are relative to
 * /root/reference/pkg/src/mgrit_advection/.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers to row-major float64 data with a
 *     row length n_x (one spatial slice per row); strides are in elements.
 *   - Calls are asynchronous on the given cudaStream_t (passed as void*).
 *   - No allocation happens in hot calls except the one-time growth of a step
 *     plan's GMRES workspace (mgb_step_reserve_workspace sizes it up front).
 *   - Return value: MGB_OK or an MGB_ERR_* code; mgb_last_error() gives text.
 *     The Python host maps codes to the reference's exceptions
 *     (ValueError / DimensionMismatchError / SingularOperatorError).
 */
#ifndef MGRIT_B200_H
#define MGRIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGB_OK 0
#define MGB_ERR_INVALID 1     /* ValueError                                   */
#define MGB_ERR_DIMENSION 2   /* DimensionMismatchError (circulant.py:116-118) */
#define MGB_ERR_SINGULAR 3    /* SingularOperatorError (circulant.py:228-234)  */
#define MGB_ERR_CUDA 4        /* CUDA runtime failure                          */
#define MGB_ERR_UNSUPPORTED 5 /* shape/stencil outside the kernel envelope     */

/* One-step operator Phi realised on the device (stepping.py:266-309). */
#define MGB_STEP_STENCIL 0   /* out = sum_k w_k v[i+o_k]; circulant.py:113-124   */
#define MGB_STEP_RK_STAGED 1 /* RK stage sweep, SDIRK stage solves;
                                stepping.py:355-380                            */
#define MGB_STEP_SL_DIRECT 2 /* SL stencil then exact (I - phi D) solve;
                                stepping.py:546-551 (assembled quotient)       */
#define MGB_STEP_SL_GMRES 3  /* SL stencil then capped GMRES on (I - phi D);
                                stepping.py:553-561, circulant.py:262-332      */

typedef struct {
  int32_t kind;     /* MGB_STEP_*                                            */
  int32_t n_x;      /* periodic mesh size                                    */
  int32_t exact;    /* 1: mul-then-add in canonical tap order (bitwise equal
                       to the reference's rolled sums, circulant.py:119-123);
                       0: fused multiply-add                                 */
  int32_t repeat;   /* apply the step this many times (ideal coarse op
                       Phi^m, stepping.py:589-598); 1 otherwise              */
  /* primary stencil: STENCIL -> Phi itself; RK -> (-c L_p); SL_* -> SL step  */
  int32_t n_taps;
  const int64_t* offsets; /* host pointers, canonical order (circulant.py:29-44) */
  const double* weights;
  /* implicit operator: RK -> stage matrix I - gamma(-c L_p); SL_* -> I - phi D */
  int32_t n_taps2;
  const int64_t* offsets2;
  const double* weights2;
  /* Runge-Kutta tableau (row-major stages x stages), RK kind only           */
  int32_t stages;
  int32_t implicit; /* 1: stage solves with the implicit operator (SDIRK)    */
  const double* rk_a;
  const double* rk_b;
  /* GMRES controls (SL_GMRES): relative tolerance and column cap           */
  double gmres_tol;
  int32_t gmres_cap;
} mgb_step_desc;

typedef struct mgb_step mgb_step; /* opaque device plan */

/* Build a device plan for one stepper.  For RK(implicit) and SL_DIRECT the
 * implicit circulant is factorised on the host (spectral factorisation into
 * first/second-order periodic recurrences).  Replaces the host-side assembly
 * in stepping.py:312-314, 504-568 for execution purposes. */
int mgb_step_create(const mgb_step_desc* desc, mgb_step** out);
void mgb_step_destroy(mgb_step* step);
/* Kernel launch geometry chosen for the plan (threads per CTA, points/thread). */
int mgb_step_layout(const mgb_step* step, int32_t* threads, int32_t* points_per_thread,
                    int32_t* smem_bytes);
/* Pre-size the per-CTA GMRES workspace (no-op for other kinds). */
int mgb_step_reserve_workspace(mgb_step* step, void* stream);

/* Interval relaxation: the batched kernel behind f_relax / c_relax /
 * restrict_residual / cpoint_residual_norm and the fused FCF passes
 * (mgrit.py:132-166, 225-247).  Interval k (0 <= k < n_intervals) starts from
 * its C-point row, advances n_fsteps fine steps (F-points k*m+1 .. k*m+n_fsteps)
 * and optionally performs one tail step (C-relaxation or residual). */
typedef struct {
  int64_t n_intervals;
  int64_t k_global0;    /* global index of interval 0 (time sharding)       */
  int32_t m;            /* coarsening factor: row of F-point j is k*m + j    */
  int32_t n_fsteps;     /* fine steps per interval (m-1 for F-relaxation)    */
  const double* c_src;  /* C-point row of interval k: c_src + k*c_stride;
                           NULL -> zero rows                                 */
  int64_t c_stride;
  const double* c_src0; /* overrides the row of global interval 0 if not NULL */
  const double* e;      /* correction e_k added to the C-point for global k>=1
                           (u[m::m] += e[1:], mgrit.py:246); NULL -> none    */
  int64_t e_stride;
  double* c_out;        /* store the (corrected) C-point row; NULL -> none   */
  int64_t c_out_stride;
  double* c_last_out;   /* if not NULL, the last interval also stores the
                           final C-point c_src[n] (+ e[n]), n = n_intervals:
                           the point no interval starts from (mgrit.py:246) */
  double* u;            /* F-point rows u + (k*m+j)*n_x                      */
  int32_t write_f;      /* 0: none, 1: last F-point only, 2: all F-points    */
  const double* g;      /* rhs rows g + row*n_x; NULL -> zero rhs            */
  int32_t tail;         /* 0: none, 1: C-relax (tail_out row k = Phi u_last +
                           g[(k+1)m]), 2: residual r_k = g + Phi u_last - cref */
  double* tail_out;     /* tail row destination: tail_out + k*tail_stride    */
  int64_t tail_stride;
  const double* cref;   /* residual reference C-point: cref + k*cref_stride  */
  int64_t cref_stride;
  const double* cref_e; /* optional correction added to cref (k-th row)      */
  int64_t cref_e_stride;
  double* partials;     /* per-interval sum of squares of the residual row   */
  int32_t* stats_depth; /* SL_GMRES: per-interval GMRES depth of the last solve */
  double* stats_res;    /* SL_GMRES: per-interval relative residual          */
  double* z_out;        /* tail == 2, explicit / staged-RK plans: also store the
                           tail step's value g + Phi u_last (the residual before
                           cref is subtracted) at z_out + k*z_stride: the C-relaxed
                           value c_relax would compute next (mgrit.py:148-149) */
  int64_t z_stride;
} mgb_relax_args;

int mgb_relax(mgb_step* step, const mgb_relax_args* args, void* stream);

/* Deterministic fixed-order sum of n partials into *out (device scalar).
 * Backs np.linalg.norm in cpoint_residual_norm (mgrit.py:164-166). */
int mgb_sum(const double* partials, int64_t n, double* out, void* stream);

/* Strided row copy (any direction, UVA): `rows` rows of `row_bytes` bytes from
 * src (row pitch src_pitch bytes) to dst (pitch dst_pitch), asynchronous on
 * `stream`.  Moves the live rows of a host iterate to the device in one DMA
 * (solve(initial_iterate=<host>), mgrit.py:288-291): only the C-points and
 * the rows before them are read before the first closing F-relaxation
 * rewrites every F-point. */
int mgb_copy_rows(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                  int64_t row_bytes, int64_t rows, void* stream);

/* Diagnostics: launch the FP64 (DFMA) throughput probe used as the FP64
 * roofline denominator by bench.py; *flops_per_launch receives its flop count. */
int mgb_fp64_peak(int64_t iters, double* flops_per_launch, void* stream);

/* Library identification and error text. */
int mgb_version(void);
const char* mgb_last_error(void);
/* Number of kernel launches issued by this process (for bench gpu_launches). */
int64_t mgb_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MGRIT_B200_H */
