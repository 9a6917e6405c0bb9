// mgb_device.cuh -- device side of the B200 MGRIT hot path (sm_100a).
//
// One CTA owns one CF-interval at a time and keeps that interval's periodic
// FP64 slice resident in shared memory for all of its fine steps (the
// reference walks the same steps as batched numpy calls, mgrit.py:132-142).
//
// Data layout of a resident slice (n = T*P points, T owning threads, P points
// per thread, P a power of two <= 16):
//   point i is owned by thread t = i / P as chunk element q = i % P and lives
//   at shared address q*S + t, with S = T + pad chosen so that (a) every
//   stencil / window read (fixed q, consecutive t) and (b) the natural-order
//   row copies to and from HBM are both bank-conflict free.
// Every thread keeps its own chunk in registers; stencil taps read neighbours
// from shared memory; periodic wrap-around is an index wrap on t.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/mgrit_b200.h"

namespace mgb {

// Optional phase timers (trace builds only: -DMGB_CL_TRACE): clock64 deltas of
// thread 0 of block 0, accumulated per phase (one buffer per translation unit).
#ifdef MGB_CL_TRACE
__device__ unsigned long long g_cl_trace[16];
#define CL_TR_INIT long long cl_t0_ = clock64();
#define CL_TR(k)                                                                      \
  if (threadIdx.x == 0 && blockIdx.x == 0) {                                          \
    const long long t_ = clock64();                                                   \
    atomicAdd(&g_cl_trace[k], (unsigned long long)(t_ - cl_t0_));                    \
    cl_t0_ = t_;                                                                      \
  }
#define CL_TR_STEP \
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&g_cl_trace[15], 1ull);
// second timer: first lane of the CTA's last warp (the cluster kernel's scalar warp)
#define CL_TRS_INIT long long cl_s0_ = clock64();
#define CL_TRS(k)                                                                     \
  if (threadIdx.x == blockDim.x - 32 && blockIdx.x == 0) {                            \
    const long long t_ = clock64();                                                   \
    atomicAdd(&g_cl_trace[k], (unsigned long long)(t_ - cl_s0_));                    \
    cl_s0_ = t_;                                                                      \
  }
#else
#define CL_TRS_INIT
#define CL_TRS(k)
#define CL_TR_INIT
#define CL_TR(k)
#define CL_TR_STEP
#endif

constexpr int MAXP = 16;
constexpr int MAX_TAPS = 256;
constexpr int MAX_TAPS2 = 32;
constexpr int MAX_FAC = 8;
constexpr int MAX_ST = 6;
constexpr int LOGT = 11;
constexpr int MAX_CAP = 128;
constexpr int MAX_WIN = 31;  // register-window stencils: span <= 30

enum { K_WIN = 0, K_GEN = 1, K_RK = 2, K_SLD = 3, K_SLG = 4, K_SLGC = 5, K_SLGC1 = 6 };
constexpr int RK_ZSOLVE = 8;  // K_RK NST flag: SDIRK stage values cL y = (y - rhs) / gamma

// One periodic first/second-order recurrence factor of a factorised
// circulant (see bandsolve in mgb_host.cu):
//   y_i = b_i + a1*y_{i-1} + a2*y_{i-2}   (dir = +1; dir = -1 runs i downward)
// Tables are precomputed in long double for the launch geometry (T, P).
struct Factor {
  double a1, a2;
  int dir, win;  // win > 0: carries by windowed look-back over win chunks
  double h1[MAXP], h2[MAXP];  // first row of A^(q+1): response to the carry-in state
  double M[4];                // A^P: chunk transition
  double Mpow[LOGT][4];       // M^(2^k)
  double MR[5][4];            // (M^R)^(2^d), R = ceil(T/32): lane scan multipliers
  double Winv[4];             // (I - M^T)^-1: periodic closure
};

struct StepParams {
  int kind, n, P, T, S, exact, repeat, stages;
  int implicit, nfac, shift, cap;
  int ntap, ntap2, win_lo, win_span;
  int win2_lo, win2_span, win2_ok, win1_ok;  // contiguous stencils: GMRES operator / RK -cL
  int z_solve, zpad_;  // SDIRK: stage value cL y = (y - rhs) / gamma from the stage solve
  double gain_inv, tol, inv_gamma;
  double A[MAX_ST * MAX_ST], b[MAX_ST];
  int tap_off[MAX_TAPS];
  double tap_w[MAX_TAPS];
  int tap2_off[MAX_TAPS2];
  double tap2_w[MAX_TAPS2];
  double win_w[32];
  double win2_w[8];
  Factor fac[MAX_FAC];
};
static_assert(sizeof(StepParams) % 16 == 0, "StepParams must be 16-byte sized");

// Constants of the dedicated SDIRK kernel (relax_rkd_kernel), passed as kernel
// parameters: the parameter space is a constant bank, so factor coefficients,
// carry responses and tableau entries are instruction operands (no shared-memory
// loads, no registers).
constexpr int RKD_MAXF = 3;   // factors of the stage operator
constexpr int RKD_MAXP = 8;   // points per thread
constexpr int RKD_KMAX = 16;  // longest carry window (chunks)
constexpr int WIN_X = 4;      // wrap replica columns of a resident slice (fixed-geometry / SLD kernels)
struct RkdFactor {
  double a1, a2, M[4], h1[RKD_MAXP], h2[RKD_MAXP];
  int dir, win;
};
// factor of the dedicated SL + direct-solve kernel: up to 16 points per thread and
// the tables of the hierarchical scan (slow-decaying factors: win == 0)
struct SldFactor {
  double a1, a2, M[4], h1[16], h2[16];
  double Mpow[10][4];  // M^(2^k): lane scan (k < 5), warp scan (k >= 5)
  double Winv[4];      // (I - M^T)^-1: periodic closure
  int dir, win;
};
struct SldConst {
  SldFactor f[2];
  double gain_inv;
  int nfac, pad_;
};
struct RkdConst {
  RkdFactor f[RKD_MAXF];
  double A[9], b[3], gain_inv, inv_gamma;
  int nfac, pad_;
};

struct RelaxLaunch {
  mgb_relax_args a;
  double* ws;            // GMRES workspace base (slot = blockIdx.x)
  long long ws_slot;     // doubles per slot
  // register-window stencil weights (relax_win_kernel): kernel parameters live in
  // the constant bank, so every tap weight is an instruction operand, not a register
  double win_w[32];
  RkdConst rk;
  SldConst sd;
};

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(a), "r"(parity) : "memory");
  }
}
// TMA bulk copy global -> shared (one instruction, completes tx bytes on `bar`)
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <bool EXACT>
__device__ __forceinline__ double madd(double acc, double w, double v) {
  // EXACT: numpy's `out += w * roll(v)` -- product rounded, then sum rounded.
  if (EXACT) return __dadd_rn(acc, __dmul_rn(w, v));
  return fma(w, v, acc);
}

template <int P>
__device__ __forceinline__ int saddr(int e, int S) {
  return (e & (P - 1)) * S + e / P;
}

template <int P>
__device__ __forceinline__ void load_chunk(const double* __restrict__ src, int t, double (&x)[P]) {
  const double* s = src + (size_t)t * P;
  if constexpr (P % 2 == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(s);
#pragma unroll
    for (int q = 0; q < P / 2; ++q) {
      double2 v = __ldg(s2 + q);
      x[2 * q] = v.x;
      x[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < P; ++q) x[q] = __ldg(s + q);
  }
}

template <int P>
__device__ __forceinline__ void store_chunk(double* dst, int t, const double (&x)[P]) {
  double* d = dst + (size_t)t * P;
  if constexpr (P % 2 == 0) {
    double2* d2 = reinterpret_cast<double2*>(d);
#pragma unroll
    for (int q = 0; q < P / 2; ++q) d2[q] = make_double2(x[2 * q], x[2 * q + 1]);
  } else {
#pragma unroll
    for (int q = 0; q < P; ++q) d[q] = x[q];
  }
}

template <int P>
__device__ __forceinline__ void chunk_to_row(double* row, int t, int S, const double (&x)[P]) {
#pragma unroll
  for (int q = 0; q < P; ++q) row[q * S + t] = x[q];
}

// natural-order copy of the resident slice to HBM (coalesced, streaming:
// F-point rows are not re-read before the next cycle overwrites them)
template <int P>
__device__ __forceinline__ void row_to_global(const double* row, double* dst, int n, int S) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) __stcs(dst + i, row[saddr<P>(i, S)]);
}

struct Ctx {
  const StepParams* sp;
  double* row;
  double* red;   // 2 x 32 reduction slots
  double* bc;    // broadcast scalars
  double* scan;  // 4*T: recurrence carry states
  double* gm;    // GMRES: Hessenberg column + y
  double* ws;    // GMRES: per-CTA global workspace
  int t, T, S, n;
  bool own;
  int parity;
  unsigned phase;  // GMRES stage mbarrier phases
};

// Deterministic block reduction: warp butterfly, one CTA barrier, then every
// warp butterflies the warp partials (lane i holds partial i) -> the same
// summation tree in every warp, bitwise identical result in all threads.
__device__ __forceinline__ double block_sum(Ctx& c, double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* slot = c.red + (c.parity << 5);
  if (lane == 0) slot[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double s;
  if (nw == 8) {  // broadcast reads in lane 0's butterfly order (bitwise the same
                  // sum as the generic path below, without its shuffle chain)
    s = ((slot[0] + slot[4]) + (slot[2] + slot[6])) + ((slot[1] + slot[5]) + (slot[3] + slot[7]));
  } else if (nw == 16) {
    s = (((slot[0] + slot[8]) + (slot[4] + slot[12])) + ((slot[2] + slot[10]) + (slot[6] + slot[14]))) +
        (((slot[1] + slot[9]) + (slot[5] + slot[13])) + ((slot[3] + slot[11]) + (slot[7] + slot[15])));
  } else {
    s = lane < nw ? slot[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1)
      if (o < nw) s += __shfl_xor_sync(0xffffffffu, s, o);  // lanes >= nw hold 0
    s = __shfl_sync(0xffffffffu, s, 0);
  }
  c.parity ^= 1;
  return s;
}

// ---------------------------------------------------------------- stencils

// generic taps (offsets pre-reduced to [0, n)), read from shared memory
template <int P, bool EXACT>
__device__ __forceinline__ void stencil_gen(const Ctx& c, int ntap, const int* off, const double* w,
                                            double (&y)[P]) {
#pragma unroll
  for (int q = 0; q < P; ++q) y[q] = 0.0;
  if (!c.own) return;
  for (int k = 0; k < ntap; ++k) {
    const int o = off[k];
    const double wk = w[k];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const int cq = o + q;
      int tt = c.t + cq / P;
      tt = tt >= c.T ? tt - c.T : tt;
      y[q] = madd<EXACT>(y[q], wk, c.row[(cq & (P - 1)) * c.S + tt]);
    }
  }
}

// contiguous short stencil through a register window: outputs in part-chunks of
// H points from a window of H + SPAN neighbours (reuse factor (SPAN+1)H/(H+SPAN)).
// The whole chunk at once (H = P) for up to 16 points per thread; 8-point parts
// for 32 points per thread (n_x = 16384), whose full window spilled registers.
template <int P, int SPAN, bool EXACT>
__device__ __forceinline__ void stencil_win(const Ctx& c, int tb, int r0, const double (&wd)[SPAN + 1],
                                            double (&y)[P]) {
  if (!c.own) {
#pragma unroll
    for (int q = 0; q < P; ++q) y[q] = 0.0;
    return;
  }
  constexpr int H = P > 16 ? 8 : P;
#pragma unroll
  for (int h = 0; h < P; h += H) {
    double win[H + SPAN];
#pragma unroll
    for (int w = 0; w < H + SPAN; ++w) {
      const int cw = r0 + h + w;
      int tt = tb + cw / P;
      tt = tt >= c.T ? tt - c.T : tt;
      tt = tt >= c.T ? tt - c.T : tt;
      win[w] = c.row[(cw & (P - 1)) * c.S + tt];
    }
#pragma unroll
    for (int q = 0; q < H; ++q) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k <= SPAN; ++k) acc = madd<EXACT>(acc, wd[k], win[q + k]);
      y[h + q] = acc;
    }
  }
}

// ------------------------------------------------ factorised periodic solve

__device__ __forceinline__ void mv2(const double* M, double& x1, double& x2) {
  const double n1 = fma(M[0], x1, M[1] * x2);
  const double n2 = fma(M[2], x1, M[3] * x2);
  x1 = n1;
  x2 = n2;
}

// Carry-state storage for the factor scans: component-split arrays, chunk tl
// at (tl % R) * 33 + tl / R (R = chunks per lane of warp 0): conflict-free for
// warp 0's lane-strided scan, at most 2-way for the chunk-owner writes.
__host__ __device__ __forceinline__ int scan_R(int T) { return T <= 32 ? 1 : (T + 31) >> 5; }
__device__ __forceinline__ int scan_addr(int tl, int R) { return (tl % R) * 33 + tl / R; }
__host__ __device__ __forceinline__ int scan_stride(int T) { return 33 * scan_R(T) + 33; }

// warp 0: carry-in states of all logical chunks for one factor.
__device__ __forceinline__ void lane_scan(const Factor& F, const double* st, double* cin, double* sb,
                                          int T, int lane) {
  const int R = (T + 31) >> 5;
  const int SS = scan_stride(T);
  const int base = lane * R;
  double X1 = 0.0, X2 = 0.0;
  for (int i = 0; i < R; ++i) {
    const int tl = base + i;
    double b1 = 0.0, b2 = 0.0;
    if (tl < T) {
      b1 = st[scan_addr(tl, R)];
      b2 = st[SS + scan_addr(tl, R)];
    }
    mv2(F.M, X1, X2);
    X1 += b1;
    X2 += b2;
  }
  double Y1 = X1, Y2 = X2;
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    const int off = 1 << d;
    double p1 = __shfl_up_sync(0xffffffffu, Y1, off);
    double p2 = __shfl_up_sync(0xffffffffu, Y2, off);
    if (lane >= off) {
      mv2(F.MR[d], p1, p2);
      Y1 += p1;
      Y2 += p2;
    }
  }
  double s1 = __shfl_up_sync(0xffffffffu, Y1, 1);
  double s2 = __shfl_up_sync(0xffffffffu, Y2, 1);
  if (lane == 0) s1 = s2 = 0.0;
  for (int i = 0; i < R; ++i) {
    const int tl = base + i;
    if (tl < T) {
      cin[scan_addr(tl, R)] = s1;
      cin[SS + scan_addr(tl, R)] = s2;
      mv2(F.M, s1, s2);
      s1 += st[scan_addr(tl, R)];
      s2 += st[SS + scan_addr(tl, R)];
      if (tl == T - 1) {  // zero-start end state -> periodic closure
        double w1 = s1, w2 = s2;
        mv2(F.Winv, w1, w2);
        sb[0] = w1;
        sb[1] = w2;
      }
    }
  }
}

struct M2r {
  double a, b, c, d;
};
__device__ __forceinline__ M2r ld_m2(const double* M) { return {M[0], M[1], M[2], M[3]}; }
__device__ __forceinline__ void mv2r(const M2r& M, double& x1, double& x2) {
  const double n1 = fma(M.a, x1, M.b * x2);
  const double n2 = fma(M.c, x1, M.d * x2);
  x1 = n1;
  x2 = n2;
}

// warp 0: TRUE carry-in states (periodic closure included) of all logical
// chunks for one factor; requires T % 32 == 0 or T <= 32 (exact R chunks/lane).
// Transition matrices live in registers for the whole scan.
__device__ __forceinline__ void lane_scan_true(const Factor& F, const double* st, double* cin,
                                               int T, int lane) {
  const int R = T <= 32 ? 1 : (T >> 5);
  const int SS = scan_stride(T);
  const int base = lane * R;
  const M2r M = ld_m2(F.M);
  M2r MR[5];
#pragma unroll
  for (int d = 0; d < 5; ++d) MR[d] = ld_m2(F.MR[d]);
  const M2r W = ld_m2(F.Winv);
  // pass 1: zero-start totals of my R chunks
  double X1 = 0.0, X2 = 0.0;
  for (int i = 0; i < R; ++i) {
    const int tl = base + i;
    const double b1 = tl < T ? st[scan_addr(tl, R)] : 0.0, b2 = tl < T ? st[SS + scan_addr(tl, R)] : 0.0;
    mv2r(M, X1, X2);
    X1 += b1;
    X2 += b2;
  }
  // inclusive lane scan (Kogge-Stone, multipliers (M^R)^(2^d))
  double Y1 = X1, Y2 = X2;
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    const int off = 1 << d;
    double p1 = __shfl_up_sync(0xffffffffu, Y1, off);
    double p2 = __shfl_up_sync(0xffffffffu, Y2, off);
    if (lane >= off) {
      mv2r(MR[d], p1, p2);
      Y1 += p1;
      Y2 += p2;
    }
  }
  // periodic closure: s_{-1} = (I - M^T)^-1 X_{T-1}
  const int last = (T - 1) / R;
  double z1 = __shfl_sync(0xffffffffu, Y1, last), z2 = __shfl_sync(0xffffffffu, Y2, last);
  mv2r(W, z1, z2);
  // my true carry-in: exclusive zero-start prefix + (M^R)^lane s_{-1}
  double s1 = __shfl_up_sync(0xffffffffu, Y1, 1), s2 = __shfl_up_sync(0xffffffffu, Y2, 1);
  if (lane == 0) s1 = s2 = 0.0;
#pragma unroll
  for (int d = 0; d < 5; ++d)
    if ((lane >> d) & 1) mv2r(MR[d], z1, z2);
  s1 += z1;
  s2 += z2;
  // pass 2: propagate true states through my chunks
  for (int i = 0; i < R; ++i) {
    const int tl = base + i;
    if (tl < T) {
      cin[scan_addr(tl, R)] = s1;
      cin[SS + scan_addr(tl, R)] = s2;
      mv2r(M, s1, s2);
      s1 += st[scan_addr(tl, R)];
      s2 += st[SS + scan_addr(tl, R)];
    }
  }
}

// x <- A^{-1} x for the factorised circulant A = K S^s prod_f F_f (in registers)
template <int P>
__device__ void chain_solve(Ctx& c, double (&x)[P]) {
  const StepParams& sp = *c.sp;
  const int T = c.T, t = c.t;
  const int R = scan_R(T), SS = scan_stride(T);
  double* st = c.scan;              // zero-start end states (2 components)
  double* cin = c.scan + 2 * SS;    // carry-in states
  double* sb = c.bc + 4;
  if (sp.shift != 0) {
    __syncthreads();
    if (c.own) chunk_to_row<P>(c.row, t, c.S, x);
    __syncthreads();
    if (c.own) {
#pragma unroll
      for (int q = 0; q < P; ++q) {
        int e = t * P + q - sp.shift;
        e %= c.n;
        e = e < 0 ? e + c.n : e;
        x[q] = c.row[saddr<P>(e, c.S)];
      }
    }
  }
  CL_TR_INIT
  int nwin = 0;  // windowed factors so far (their end-state buffers alternate)
  for (int f = 0; f < sp.nfac; ++f) {
    const Factor& F = sp.fac[f];
    const bool fwd = F.dir > 0;
    const int tl = fwd ? t : T - 1 - t;
    double s1 = 0.0, s2 = 0.0;  // zero-start end state of my chunk
    if (c.own) {
      const double a1 = F.a1, a2 = F.a2;
#pragma unroll
      for (int qq = 0; qq < P; ++qq) {
        const int q = fwd ? qq : P - 1 - qq;
        // the y_{q-2} term first: one FMA latency per point on the carried chain
        const double yv = fma(a1, s1, fma(a2, s2, x[q]));
        x[q] = yv;
        s2 = s1;
        s1 = yv;
      }
      if (!(T % 32 == 0) && F.win == 0) {
        st[scan_addr(tl, R)] = s1;
        st[SS + scan_addr(tl, R)] = s2;
      }
    }
    CL_TR(4)
    const bool hier = (T % 32 == 0);
    double c1 = 0.0, c2 = 0.0;
    if (F.win > 0) {
      // fast-decaying factor: the true carry of chunk tl is exact to rounding
      // from the K previous chunks' zero-start end states (Horner), one barrier
      double* wb = c.scan + 4 * SS + (nwin & 1) * 2 * T;
      ++nwin;
      if (c.own) {
        wb[tl] = s1;
        wb[T + tl] = s2;
      }
      __syncthreads();
      CL_TR(5)
      if (c.own) {
        // Horner over k = K..1: c = M c + s_{tl-k}; compact runtime loop (an
        // unrolled 16-way predicated loop stalls on instruction fetch), next
        // chunk's end state loaded one iteration ahead
        const M2r M = ld_m2(F.M);
        const int K = F.win;
        int u = tl - K;
        u += u < 0 ? T : 0;
        double n1 = wb[u], n2 = wb[T + u];
#pragma unroll 1
        for (int k = K; k >= 1; --k) {
          const double b1 = n1, b2 = n2;
          if (k > 1) {
            u = u + 1 == T ? 0 : u + 1;
            n1 = wb[u];
            n2 = wb[T + u];
          }
          mv2r(M, c1, c2);
          c1 += b1;
          c2 += b2;
        }
      }
      CL_TR(7)
    } else if (hier) {
      // hierarchical parallel scan over logical chunks (warp-level Kogge-Stone,
      // then warp 0 over the warp totals with the periodic closure)
      const int NW = T >> 5, lane = t & 31, w = t >> 5;
      const int ll = fwd ? lane : 31 - lane;
      const int lw = fwd ? w : NW - 1 - w;
      double y1 = s1, y2 = s2;
#pragma unroll
      for (int d = 0; d < 5; ++d) {
        const int off = 1 << d;
        const int src = (fwd ? lane - off : lane + off) & 31;
        double p1 = __shfl_sync(0xffffffffu, y1, src), p2 = __shfl_sync(0xffffffffu, y2, src);
        if (ll >= off) {
          mv2(F.Mpow[d], p1, p2);
          y1 += p1;
          y2 += p2;
        }
      }
      const int s1src = (fwd ? lane - 1 : lane + 1) & 31;
      double e1 = __shfl_sync(0xffffffffu, y1, s1src), e2 = __shfl_sync(0xffffffffu, y2, s1src);
      if (ll == 0) e1 = e2 = 0.0;
      if (ll == 31) {
        st[lw] = y1;
        st[32 + lw] = y2;
      }
      __syncthreads();
      CL_TR(5)
      if (w == 0) {
        double a1w = lane < NW ? st[lane] : 0.0, a2w = lane < NW ? st[32 + lane] : 0.0;
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          const int off = 1 << d;
          double p1 = __shfl_up_sync(0xffffffffu, a1w, off), p2 = __shfl_up_sync(0xffffffffu, a2w, off);
          if (lane >= off) {
            mv2(F.Mpow[5 + d], p1, p2);
            a1w += p1;
            a2w += p2;
          }
        }
        double z1 = __shfl_sync(0xffffffffu, a1w, NW - 1), z2 = __shfl_sync(0xffffffffu, a2w, NW - 1);
        mv2(F.Winv, z1, z2);  // s_{-1}: periodic closure
        double x1 = __shfl_up_sync(0xffffffffu, a1w, 1), x2 = __shfl_up_sync(0xffffffffu, a2w, 1);
        if (lane == 0) x1 = x2 = 0.0;
#pragma unroll
        for (int d = 0; d < 5; ++d)
          if ((lane >> d) & 1) mv2(F.Mpow[5 + d], z1, z2);  // (M^32)^lw s_{-1}
        if (lane < NW) {
          cin[lane] = x1 + z1;
          cin[32 + lane] = x2 + z2;
        }
      }
      __syncthreads();
      CL_TR(6)
      c1 = cin[lw];
      c2 = cin[32 + lw];
#pragma unroll
      for (int d = 0; d < 5; ++d)
        if ((ll >> d) & 1) mv2(F.Mpow[d], c1, c2);  // M^ll C_w
      c1 += e1;
      c2 += e2;
      CL_TR(7)
    } else {
      __syncthreads();
      CL_TR(5)
      if (t < 32) {
        if (T <= 32)
          lane_scan_true(F, st, cin, T, t);
        else
          lane_scan(F, st, cin, sb, T, t);
      }
      CL_TR(6)
      __syncthreads();
      CL_TR(7)
      if (c.own) {
        c1 = cin[scan_addr(tl, R)];
        c2 = cin[SS + scan_addr(tl, R)];
      }
    }
    if (c.own) {
      if (F.win == 0 && !hier && T > 32) {  // add the periodic-closure response M^tl s_{-1}
        double p1 = sb[0], p2 = sb[1];
#pragma unroll
        for (int kb = 0; kb < LOGT; ++kb)
          if ((tl >> kb) & 1) mv2(F.Mpow[kb], p1, p2);
        c1 += p1;
        c2 += p2;
      }
#pragma unroll
      for (int qq = 0; qq < P; ++qq) {
        const int q = fwd ? qq : P - 1 - qq;
        x[q] = fma(F.h1[qq], c1, fma(F.h2[qq], c2, x[q]));
      }
    }
    CL_TR(8)
  }
  if (c.own) {
#pragma unroll
    for (int q = 0; q < P; ++q) x[q] *= sp.gain_inv;
  }
}

// ------------------------------------------------------------------ GMRES

// Krylov basis element (t, q) of vector i: pairs (q, q+1) are stored as one
// 16-byte word at ((q/2) * T + t) * 2 so every warp load is a coalesced LDG.128.
template <int P>
__device__ __forceinline__ void vec_load(const double* __restrict__ Vi, int t, int T, double (&x)[P]) {
  if constexpr (P % 2 == 0) {
    const double2* v2 = reinterpret_cast<const double2*>(Vi);
#pragma unroll
    for (int q = 0; q < P / 2; ++q) {
      const double2 d = v2[q * T + t];
      x[2 * q] = d.x;
      x[2 * q + 1] = d.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < P; ++q) x[q] = Vi[q * T + t];
  }
}
template <int P>
__device__ __forceinline__ void vec_store(double* Vi, int t, int T, const double (&x)[P]) {
  if constexpr (P % 2 == 0) {
    double2* v2 = reinterpret_cast<double2*>(Vi);
#pragma unroll
    for (int q = 0; q < P / 2; ++q) v2[q * T + t] = make_double2(x[2 * q], x[2 * q + 1]);
  } else {
#pragma unroll
    for (int q = 0; q < P; ++q) Vi[q * T + t] = x[q];
  }
}

// Contiguous short stencil (span <= 6, runtime) through a register window of
// P+6 neighbours: one shared load per point instead of one per tap.
template <int P, bool EXACT>
__device__ __forceinline__ void stencil_win_rt(const Ctx& c, int lo, int span, const double* wts,
                                               double (&y)[P]) {
#pragma unroll
  for (int q = 0; q < P; ++q) y[q] = 0.0;
  if (!c.own) return;
  int tb = c.t + lo / P;
  tb = tb >= c.T ? tb - c.T : tb;
  const int r0 = lo & (P - 1);
  double win[P + 6];
#pragma unroll
  for (int w = 0; w < P + 6; ++w) {
    const int cw = r0 + w;
    int tt = tb + cw / P;
    tt = tt >= c.T ? tt - c.T : tt;
    tt = tt >= c.T ? tt - c.T : tt;
    win[w] = c.row[(cw & (P - 1)) * c.S + tt];
  }
#pragma unroll
  for (int k = 0; k <= 6; ++k) {
    if (k <= span) {
      const double wk = wts[k];
#pragma unroll
      for (int q = 0; q < P; ++q) y[q] = madd<EXACT>(y[q], wk, win[q + k]);
    }
  }
}

// (I - phi D) applied to the resident row inside GMRES (DFMA).
template <int P>
__device__ __forceinline__ void apply_op2(const Ctx& c, double (&y)[P]) {
  const StepParams& sp = *c.sp;
  if (!sp.win2_ok) {
    stencil_gen<P, false>(c, sp.ntap2, sp.tap2_off, sp.tap2_w, y);
    return;
  }
  stencil_win_rt<P, false>(c, sp.win2_lo, sp.win2_span, sp.win2_w, y);
}

// (I - phi D) on a basis vector held in registers (P consecutive points per
// thread), symmetric window -R..R: neighbour points come from the adjacent
// lanes by shuffles, across warp boundaries from the per-warp edge slots
// (e[0..2] = lane 0's first three points, e[4..6] = lane 31's last three,
// written before the CTA barrier that precedes this call).  Same taps and
// accumulation order as stencil_win_rt (bitwise the same y), without the
// row round trip through shared memory and its two CTA barriers.
template <int P, int R>
__device__ __forceinline__ void stencil_shfl(const Ctx& c, const double* wts, const double (&v)[P],
                                             const double* edges, double (&y)[P]) {
  const int lane = c.t & 31, wp = c.t >> 5, nw = c.T >> 5;
  double win[P + 2 * R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    win[r] = __shfl_up_sync(0xffffffffu, v[P - R + r], 1);
    win[P + R + r] = __shfl_down_sync(0xffffffffu, v[r], 1);
  }
  if (lane == 0) {
    const double* e = edges + 8 * (wp == 0 ? nw - 1 : wp - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) win[r] = e[4 + 3 - R + r];
  }
  if (lane == 31) {
    const double* e = edges + 8 * (wp == nw - 1 ? 0 : wp + 1);
#pragma unroll
    for (int r = 0; r < R; ++r) win[P + R + r] = e[r];
  }
#pragma unroll
  for (int q = 0; q < P; ++q) win[R + q] = v[q];
#pragma unroll
  for (int q = 0; q < P; ++q) y[q] = 0.0;
#pragma unroll
  for (int k = 0; k <= 2 * R; ++k) {
    const double wk = wts[k];
#pragma unroll
    for (int q = 0; q < P; ++q) y[q] = madd<false>(y[q], wk, win[q + k]);
  }
}

// edge slots of this thread's basis chunk for stencil_shfl (lanes 0 and 31)
template <int P>
__device__ __forceinline__ void put_edges(const Ctx& c, const double (&v)[P], double* edges) {
  const int lane = c.t & 31;
  double* e = edges + 8 * (c.t >> 5);
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < 3; ++r) e[r] = v[r < P ? r : 0];
  }
  if (lane == 31) {
#pragma unroll
    for (int r = 0; r < 3; ++r) e[4 + r] = v[P - 3 + r >= 0 ? P - 3 + r : 0];
  }
}

constexpr int RS_CAP = 24;  // Hessenberg R kept in shared memory for cap <= RS_CAP

// Shared-memory carve-up of the single-CTA GMRES (after the scan area), doubles
struct GmLayout {
  __host__ __device__ static int hcol() { return 0; }
  __host__ __device__ static int ybuf() { return MAX_CAP + 2; }
  __host__ __device__ static int cs() { return ybuf() + MAX_CAP; }
  __host__ __device__ static int sn() { return cs() + MAX_CAP; }
  __host__ __device__ static int gg() { return sn() + MAX_CAP; }
  __host__ __device__ static int Rs() { return gg() + MAX_CAP + 2; }
  __host__ __device__ static int mbar() { return Rs() + RS_CAP * RS_CAP; }
  __host__ __device__ static int edges() { return mbar() + 4; }  // 8 doubles per warp (<= 16 warps)
  __host__ __device__ static int stage() { return edges() + 8 * 16; }  // + 16-byte alignment pad
  __host__ __device__ static int total(int n) { return stage() + 2 + 2 * n; }
};

// Unrestarted GMRES(x0 = 0) on the circulant (taps2) for the CTA's row,
// following circulant.py:262-332: MGS Arnoldi, Givens QR, stop when
// res <= tol or ||h|| <= 1e-14 beta, back substitution, x = V y.
// The basis V lives in this CTA's L2/HBM workspace slot (16-byte coalesced
// layout); the vectors an Arnoldi step needs are streamed into two shared
// memory stages with TMA bulk copies (cp.async.bulk + mbarrier) two ahead of
// use, so MGS reads them at shared-memory latency.  R and the Givens state
// stay in shared memory; the back substitution runs on one warp.  A stage
// keeps the vector it holds across Arnoldi steps (shallow solves -- depth <= 3,
// the common case on many-interval levels -- stream V_0 and V_1 once per
// solve, not once per step), and the async-proxy fence for a new basis vector
// is issued one step after its store (its first TMA read is two steps later),
// so the stores drain off the critical path.
template <int P>
__device__ void gmres_solve(Ctx& c, const double (&b)[P], double (&x)[P], int& depth_out,
                            double& res_out) {
  const StepParams& sp = *c.sp;
  const int n = c.n, T = c.T, t = c.t;
  const int cap = sp.cap;
  double* V = c.ws;
  double* Rg = V + (size_t)(cap + 1) * n;  // global R (cap > RS_CAP only)
  double* hcol = c.gm + GmLayout::hcol();
  double* ybuf = c.gm + GmLayout::ybuf();
  double* cs = c.gm + GmLayout::cs();
  double* sn = c.gm + GmLayout::sn();
  double* gg = c.gm + GmLayout::gg();
  // R in shared memory for cap <= RS_CAP, else in the global slot; accessed
  // through a uniform branch so the shared case compiles to LDS/STS (one
  // pointer selected between the two spaces would be generic)
  double* const Rs = c.gm + GmLayout::Rs();
  const bool rsm = cap <= RS_CAP;
  const int ldr = rsm ? RS_CAP : cap;
  auto rget = [&](int col, int r) -> double {
    const size_t k = (size_t)col * ldr + r;
    return rsm ? Rs[k] : Rg[k];
  };
  auto rset = [&](int col, int r, double v) {
    const size_t k = (size_t)col * ldr + r;
    if (rsm) Rs[k] = v; else Rg[k] = v;
  };
  uint64_t* bar = reinterpret_cast<uint64_t*>(c.gm + GmLayout::mbar());
  // 16-byte aligned stage base by pointer arithmetic on the shared pointer (an
  // integer round trip would lose the address space: generic LD.E instead of LDS)
  double* stage0 = c.gm + GmLayout::stage();
  stage0 += ((uint32_t)__cvta_generic_to_shared(stage0) & 15u) ? 1 : 0;
  const uint32_t vbytes = (uint32_t)n * 8u;
  // held[st]: basis index stage st holds (or will hold once its pending copy
  // lands); pend: stages with a copy in flight.  Uniform across the CTA.
  int held0 = -1, held1 = -1;
  unsigned pend = 0;
#define MGB_ISSUE(i, st)                                                      \
  do {                                                                        \
    if (t == 0) {                                                             \
      mbar_arm(bar + (st), vbytes);                                           \
      bulk_g2s(stage0 + (size_t)(st) * n, V + (size_t)(i) * n, vbytes, bar + (st)); \
    }                                                                         \
    if (st) held1 = (i); else held0 = (i);                                    \
    pend |= 1u << (st);                                                       \
  } while (0)
#define MGB_CONSUME(st, vi)                                                   \
  do {                                                                        \
    if (pend & (1u << (st))) {                                                \
      mbar_wait(bar + (st), (c.phase >> (st)) & 1u);                          \
      c.phase ^= 1u << (st);                                                  \
      pend &= ~(1u << (st));                                                  \
    }                                                                         \
    if (c.own) vec_load<P>(stage0 + (size_t)(st) * n, t, T, vi);              \
  } while (0)
  CL_TR_INIT
  double part = 0.0;
  if (c.own) {
#pragma unroll
    for (int q = 0; q < P; ++q) part = fma(b[q], b[q], part);
  }
  const double beta = sqrt(block_sum(c, part));
  CL_TR(0)
  if (beta == 0.0) {  // zero right-hand side: x = 0, converged (circulant.py:274-278)
#pragma unroll
    for (int q = 0; q < P; ++q) x[q] = 0.0;
    depth_out = 0;
    res_out = 0.0;
    return;
  }
  double v[P];
  const double ib = 1.0 / beta;
#pragma unroll
  for (int q = 0; q < P; ++q) v[q] = b[q] * ib;
  if (c.own) vec_store<P>(V, t, T, v);  // fenced for the TMA after step 0's stencil
  if (t == 0) gg[0] = beta;
  // register/shuffle stencil path: symmetric contiguous operator window of
  // half-width 1..3, every thread owning a chunk, whole warps (uniform)
  double* const edges = c.gm + GmLayout::edges();
  const int rh = sp.win2_span / 2;
  const bool shfl = P >= 4 && sp.win2_ok && (sp.win2_span & 1) == 0 && rh >= 1 && rh <= 3 &&
                    sp.win2_lo == n - rh && T == (int)blockDim.x && (T & 31) == 0 && T <= 512;
  if (shfl) {
    put_edges<P>(c, v, edges);
    __syncthreads();
  }
  double res = 1.0;
  int depth = 0;
  for (int j = 0; j < cap; ++j) {
    if (shfl) {  // own slots only: V_j for the MGS i == j term and x = V y
      chunk_to_row<P>(c.row, t, c.S, v);
    } else {
      __syncthreads();
      if (c.own) chunk_to_row<P>(c.row, t, c.S, v);
      __syncthreads();
    }
    // stream V_0, V_1 while the stencil runs (V_j itself is the row), unless
    // the stages still hold them
    if (j >= 1 && held0 != 0) MGB_ISSUE(0, 0);
    if (j >= 2 && held1 != 1) MGB_ISSUE(1, 1);
    CL_TR(9)
    double w[P];
    if (shfl) {
      if (rh == 2) stencil_shfl<P, 2>(c, sp.win2_w, v, edges, w);
      else if (rh == 3) stencil_shfl<P, 3>(c, sp.win2_w, v, edges, w);
      else stencil_shfl<P, 1>(c, sp.win2_w, v, edges, w);
    } else {
      apply_op2<P>(c, w);
    }
    // generic stores of V_j (previous step / solve start) -> async-proxy reads;
    // the first TMA read of V_j is issued after a later CTA barrier
    asm volatile("fence.proxy.async.global;" ::: "memory");
    CL_TR(1)
    for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
      double vi[P];
      if (i < j) {
        MGB_CONSUME(i & 1, vi);
      } else {  // V_j is the row; idle threads (!c.own) read thread 0's slot,
                // and every use of their values below is guarded by c.own
        const double* rp = c.row + (c.own ? t : 0);
#pragma unroll
        for (int q = 0; q < P; ++q) vi[q] = rp[q * c.S];
      }
      double p0 = 0.0, p1 = 0.0;
      if (c.own) {
#pragma unroll
        for (int q = 0; q < P; q += 2) {
          p0 = fma(w[q], vi[q], p0);
          if (q + 1 < P) p1 = fma(w[q + 1], vi[q + 1], p1);
        }
      }
      CL_TR(2)
      const double h = block_sum(c, p0 + p1);  // every thread has consumed stage i&1
      CL_TR(3)
      if (t == 0) hcol[i] = h;
      if (i + 2 < j) MGB_ISSUE(i + 2, i & 1);
#pragma unroll
      for (int q = 0; q < P; ++q) w[q] = fma(-h, vi[q], w[q]);
    }
    double n0 = 0.0, n1 = 0.0;
    if (c.own) {
#pragma unroll
      for (int q = 0; q < P; q += 2) {
        n0 = fma(w[q], w[q], n0);
        if (q + 1 < P) n1 = fma(w[q + 1], w[q + 1], n1);
      }
    }
    CL_TR(4)
    const double hn = sqrt(block_sum(c, n0 + n1));
    CL_TR(5)
    const bool happy = hn <= 1e-14 * beta;
    const double inv = 1.0 / (hn > 0.0 ? hn : 1.0);
#pragma unroll
    for (int q = 0; q < P; ++q) v[q] = w[q] * inv;
    if (c.own) vec_store<P>(V + (size_t)(j + 1) * n, t, T, v);  // fenced next step
    if (shfl) put_edges<P>(c, v, edges);  // read after the barrier below
    if (t == 0) {  // Givens (circulant.py:308-319), rotated entry carried in a register
      double hi = hcol[0];
#pragma unroll 4
      for (int i = 0; i < j; ++i) {
        const double ci = cs[i], si = sn[i], hi1 = hcol[i + 1];
        rset(j, i, __dadd_rn(__dmul_rn(ci, hi), __dmul_rn(si, hi1)));
        hi = __dadd_rn(__dmul_rn(-si, hi), __dmul_rn(ci, hi1));
      }
      double den = hypot(hi, hn);
      den = den > 0.0 ? den : 1.0;
      const double rd = 1.0 / den;
      const double cj = hi * rd, sj = hn * rd;
      cs[j] = cj;
      sn[j] = sj;
      rset(j, j, __dadd_rn(__dmul_rn(cj, hi), __dmul_rn(sj, hn)));
      const double gj = gg[j];
      gg[j + 1] = __dmul_rn(-sj, gj);
      gg[j] = __dmul_rn(cj, gj);
      const double r = fabs(gg[j + 1]) / beta;
      c.bc[0] = r;
      c.bc[1] = (!(r > sp.tol) || happy) ? 1.0 : 0.0;
    }
    CL_TR(6)
    __syncthreads();
    CL_TR(7)
    CL_TR_STEP
    res = c.bc[0];
    depth = j + 1;
    if (c.bc[1] != 0.0) break;
  }
  const int lane = t & 31;
  if ((t >> 5) == 0) {  // back substitution R y = g, column oriented, lanes own rows
    if (depth <= 32) {
      double y = lane < depth ? gg[lane] : 0.0;
      for (int jj = depth - 1; jj >= 0; --jj) {
        double yj = __shfl_sync(0xffffffffu, y, jj);
        if (yj != 0.0) yj /= rget(jj, jj);
        if (lane == jj) y = yj;
        if (lane < jj) y = __dsub_rn(y, __dmul_rn(yj, rget(jj, lane)));
      }
      if (lane < depth) ybuf[lane] = y;
    } else if (lane == 0) {
      for (int i = 0; i < depth; ++i) ybuf[i] = gg[i];
      for (int jj = depth - 1; jj >= 0; --jj) {
        if (ybuf[jj] != 0.0) {
          ybuf[jj] /= rget(jj, jj);
          const double yj = ybuf[jj];
          for (int i = 0; i < jj; ++i) ybuf[i] = __dsub_rn(ybuf[i], __dmul_rn(yj, rget(jj, i)));
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < P; ++q) x[q] = 0.0;
  if (c.own) {  // x = V y, in basis order.  The last three vectors are on chip:
    // V_{depth-1} is the row, V_{depth-2} / V_{depth-3} are in the stages (every
    // copy has been consumed); the older ones stream from L2 with a two-deep
    // register prefetch.
    const int ng = depth > 3 ? depth - 3 : 0;
    if (ng > 0) {
      double va[P], vb[P];
      vec_load<P>(V, t, T, va);
      if (ng > 1) vec_load<P>(V + n, t, T, vb);
      for (int i = 0; i < ng; ++i) {
        const double yi = ybuf[i];
#pragma unroll
        for (int q = 0; q < P; ++q) {
          x[q] = fma(yi, va[q], x[q]);
          va[q] = vb[q];
        }
        if (i + 2 < ng) vec_load<P>(V + (size_t)(i + 2) * n, t, T, vb);
      }
    }
    for (int i = ng; i < depth; ++i) {
      const double yi = ybuf[i];
      double vi[P];
      if (i == depth - 1) {
#pragma unroll
        for (int q = 0; q < P; ++q) vi[q] = c.row[q * c.S + t];
      } else if (i == held0) {
        vec_load<P>(stage0, t, T, vi);
      } else if (i == held1) {
        vec_load<P>(stage0 + n, t, T, vi);
      } else {
        vec_load<P>(V + (size_t)i * n, t, T, vi);
      }
#pragma unroll
      for (int q = 0; q < P; ++q) x[q] = fma(yi, vi[q], x[q]);
    }
  }
#undef MGB_ISSUE
#undef MGB_CONSUME
  CL_TR(8)
  depth_out = depth;
  res_out = res;
}

// ------------------------------------------------------------- one step

// Precondition: c.row holds the step input x (synchronised).
// Postcondition: y = Phi x (own chunk).  c.row may have been reused; callers
// __syncthreads() before writing it.
template <int P, int KIND, int SPAN, int NST, bool EXACT>
__device__ __forceinline__ void step_once(Ctx& c, const double (&wd)[SPAN + 1], int tb, int r0,
                                          double (&y)[P], int& depth, double& gres) {
  const StepParams& sp = *c.sp;
  if constexpr (KIND == K_WIN) {
    stencil_win<P, SPAN, EXACT>(c, tb, r0, wd, y);
  } else if constexpr (KIND == K_GEN) {
    stencil_gen<P, EXACT>(c, sp.ntap, sp.tap_off, sp.tap_w, y);
  } else if constexpr (KIND == K_SLD) {
    stencil_gen<P, true>(c, sp.ntap, sp.tap_off, sp.tap_w, y);
    chain_solve<P>(c, y);
  } else if constexpr (KIND == K_SLG) {
    double b[P];
    stencil_gen<P, true>(c, sp.ntap, sp.tap_off, sp.tap_w, b);
    gmres_solve<P>(c, b, y, depth, gres);
  } else {  // K_RK: staged Runge-Kutta sweep, stepping.py:363-378
    // NST = stages (+ RK_ZSOLVE: SDIRK stage values from the stage solves)
    constexpr int NS = NST & (RK_ZSOLVE - 1);
    constexpr bool ZS = NST >= RK_ZSOLVE;
    double x[P];
#pragma unroll
    for (int q = 0; q < P; ++q) x[q] = c.own ? c.row[q * c.S + c.t] : 0.0;
    double z[NS][P];
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      double rhs[P];
#pragma unroll
      for (int q = 0; q < P; ++q) rhs[q] = x[q];
#pragma unroll
      for (int j = 0; j < i; ++j) {
        const double aij = sp.A[i * MAX_ST + j];
        if (aij != 0.0) {
#pragma unroll
          for (int q = 0; q < P; ++q) rhs[q] = __dadd_rn(rhs[q], __dmul_rn(aij, z[j][q]));
        }
      }
      if constexpr (ZS) {
        // M y = rhs with M = I - gamma cL  =>  cL y = (y - rhs) / gamma: the
        // stage value without the stencil pass (and its row round trip)
        double r0[P];
#pragma unroll
        for (int q = 0; q < P; ++q) r0[q] = rhs[q];
        if (i > 0) __syncthreads();  // previous solve's carry buffers are free
        chain_solve<P>(c, rhs);
#pragma unroll
        for (int q = 0; q < P; ++q) z[i][q] = __dmul_rn(__dsub_rn(rhs[q], r0[q]), sp.inv_gamma);
        continue;
      }
      if (sp.implicit) chain_solve<P>(c, rhs);
      CL_TR_INIT
      __syncthreads();
      if (c.own) chunk_to_row<P>(c.row, c.t, c.S, rhs);
      __syncthreads();
      CL_TR(1)
      if (sp.win1_ok)
        stencil_win_rt<P, true>(c, sp.win_lo, sp.win_span, sp.win_w, z[i]);
      else
        stencil_gen<P, true>(c, sp.ntap, sp.tap_off, sp.tap_w, z[i]);
      CL_TR(2)
      CL_TR_STEP
    }
#pragma unroll
    for (int q = 0; q < P; ++q) y[q] = x[q];
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      const double bi = sp.b[i];
      if (bi != 0.0) {
#pragma unroll
        for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], __dmul_rn(bi, z[i][q]));
      }
    }
  }
}

// ------------------------------------------------------------ relax kernel

__host__ __device__ constexpr int sp_bytes() { return (int)sizeof(StepParams); }

// MAXT: launch bound (512, or 256 for register-heavy GMRES variants, T <= 256)
// Shared-memory copy of the step parameters: the whole StepParams, or for the
// 2-CTA/SM single-CTA GMRES variant only the prefix before the factor tables
// (which GMRES plans do not use), so two CTAs' slices + TMA stages fit an SM.
template <int KIND, int MINB>
__host__ __device__ constexpr int sp_smem_bytes() {
  return (KIND == K_SLG && MINB > 1) ? (int)((offsetof(StepParams, fac) + 15) / 16 * 16)
                                     : (int)sizeof(StepParams);
}

template <int P, int KIND, int SPAN, int NST, bool EXACT, int MAXT = 512, int MINB = 1>
__global__ void __launch_bounds__(MAXT, MINB) relax_kernel(const StepParams* __restrict__ gp,
                                                           const RelaxLaunch L) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int SPB = sp_smem_bytes<KIND, MINB>();
#ifdef MGB_CL_TRACE
  const long long kt0_ = clock64();
#endif
  {
    const int4* src = reinterpret_cast<const int4*>(gp);
    int4* dst = reinterpret_cast<int4*>(smem_raw);
    for (int i = threadIdx.x; i < SPB / 16; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
#ifdef MGB_CL_TRACE  // slot 10: parameter prologue, slot 11: whole kernel (block 0)
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&g_cl_trace[10], (unsigned long long)(clock64() - kt0_));
#endif
  const StepParams& sp = *reinterpret_cast<const StepParams*>(smem_raw);
  const mgb_relax_args& a = L.a;
  Ctx c;
  c.sp = &sp;
  c.n = sp.n;
  c.T = sp.T;
  c.S = sp.S;
  c.t = threadIdx.x;
  c.own = c.t < c.T;
  c.row = reinterpret_cast<double*>(smem_raw + SPB);
  c.red = c.row + (size_t)P * c.S;
  c.bc = c.red + 64;
  c.scan = c.bc + 8;
  c.gm = c.scan + ((KIND == K_SLD || KIND == K_RK) ? 4 * scan_stride(c.T) + 4 * c.T : 0);
  c.ws = L.ws ? L.ws + (size_t)blockIdx.x * L.ws_slot : nullptr;
  c.parity = 0;
  c.phase = 0;
  if constexpr (KIND == K_SLG) {
    if (threadIdx.x == 0) {
      uint64_t* bar = reinterpret_cast<uint64_t*>(c.gm + GmLayout::mbar());
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  const int n = c.n, t = c.t;

  double wd[SPAN + 1];
  int tb = 0, r0 = 0;
  if constexpr (KIND == K_WIN) {
#pragma unroll
    for (int k = 0; k <= SPAN; ++k) wd[k] = sp.win_w[k];
    tb = t + sp.win_lo / P;
    tb = tb >= c.T ? tb - c.T : tb;
    r0 = sp.win_lo & (P - 1);
  } else {
#pragma unroll
    for (int k = 0; k <= SPAN; ++k) wd[k] = 0.0;
  }
  const int reps = sp.repeat;

  for (long long k = blockIdx.x; k < a.n_intervals; k += gridDim.x) {
    const long long kg = a.k_global0 + k;
    const long long rowbase = k * (long long)a.m;
    double y[P];
    const double* csrc = (kg == 0 && a.c_src0) ? a.c_src0 : (a.c_src ? a.c_src + k * a.c_stride : nullptr);
    if (c.own) {
      if (csrc) {
        load_chunk<P>(csrc, t, y);
      } else {
#pragma unroll
        for (int q = 0; q < P; ++q) y[q] = 0.0;
      }
      if (a.e && kg >= 1) {  // u[m::m] += e[1:] (mgrit.py:246)
        double ev[P];
        load_chunk<P>(a.e + k * a.e_stride, t, ev);
#pragma unroll
        for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], ev[q]);
      }
      if (a.c_out) store_chunk<P>(a.c_out + k * a.c_out_stride, t, y);
    }
    __syncthreads();
    if (c.own) chunk_to_row<P>(c.row, t, c.S, y);
    __syncthreads();
    int depth = 0;
    double gres = 0.0;
    const int nsteps = a.n_fsteps + (a.tail ? 1 : 0);
    for (int j = 1; j <= nsteps; ++j) {
      const bool is_tail = j > a.n_fsteps;
      if (a.g && c.own) {  // this step's rhs chunk into L1 while the step runs (one line per
                           // thread at P = 16): its load after the step no longer waits on L2
        const double* gp1 = a.g + (is_tail ? rowbase + a.m : rowbase + j) * n + (size_t)t * P;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(gp1));
      }
      for (int r = 0; r < reps; ++r) {
        step_once<P, KIND, SPAN, NST, EXACT>(c, wd, tb, r0, y, depth, gres);
        if (r + 1 < reps) {
          __syncthreads();
          if (c.own) chunk_to_row<P>(c.row, t, c.S, y);
          __syncthreads();
        }
      }
      // rhs row of this point; the tail step lands on C-point (k+1)m
      const long long grow = is_tail ? rowbase + a.m : rowbase + j;
      if (!is_tail) {
        if (a.g && c.own) {
          double gv[P];
          load_chunk<P>(a.g + grow * n, t, gv);
#pragma unroll
          for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], gv[q]);  // upd + g (mgrit.py:142)
        }
        __syncthreads();
        if (c.own) chunk_to_row<P>(c.row, t, c.S, y);
        __syncthreads();
        if (a.write_f == 2 || (a.write_f == 1 && j == a.n_fsteps))
          row_to_global<P>(c.row, a.u + grow * n, n, c.S);
      } else if (a.tail == 1) {  // C-relaxation: Phi u_{km+m-1} + g_{(k+1)m} (mgrit.py:148-149)
        if (c.own) {
          if (a.g) {
            double gv[P];
            load_chunk<P>(a.g + grow * n, t, gv);
#pragma unroll
            for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], gv[q]);
          }
          store_chunk<P>(a.tail_out + k * a.tail_stride, t, y);
        }
      } else {  // residual g + Phi u - u_C (mgrit.py:159-161)
        double part = 0.0;
        if (c.own) {
          double r[P];
          if (a.g) {
            double gv[P];
            load_chunk<P>(a.g + grow * n, t, gv);
#pragma unroll
            for (int q = 0; q < P; ++q) r[q] = __dadd_rn(gv[q], y[q]);
          } else {
#pragma unroll
            for (int q = 0; q < P; ++q) r[q] = y[q];
          }
          if (a.z_out) store_chunk<P>(a.z_out + k * a.z_stride, t, r);  // g + Phi u_last
          double cr[P];
          load_chunk<P>(a.cref + k * a.cref_stride, t, cr);
          if (a.cref_e) {
            double ev[P];
            load_chunk<P>(a.cref_e + k * a.cref_e_stride, t, ev);
#pragma unroll
            for (int q = 0; q < P; ++q) cr[q] = __dadd_rn(cr[q], ev[q]);
          }
#pragma unroll
          for (int q = 0; q < P; ++q) {
            r[q] = __dsub_rn(r[q], cr[q]);
            part = fma(r[q], r[q], part);
          }
          if (a.tail_out) store_chunk<P>(a.tail_out + k * a.tail_stride, t, r);
        }
        if (a.partials) {
          const double s = block_sum(c, part);
          if (t == 0) a.partials[k] = s;
        }
      }
    }
    if (a.c_last_out && k == a.n_intervals - 1 && c.own) {  // final C-point (k+1 >= 1)
      double cl[P];
      if (a.c_src) {
        load_chunk<P>(a.c_src + (k + 1) * a.c_stride, t, cl);
      } else {
#pragma unroll
        for (int q = 0; q < P; ++q) cl[q] = 0.0;
      }
      if (a.e) {
        double ev[P];
        load_chunk<P>(a.e + (k + 1) * a.e_stride, t, ev);
#pragma unroll
        for (int q = 0; q < P; ++q) cl[q] = __dadd_rn(cl[q], ev[q]);
      }
      store_chunk<P>(a.c_last_out, t, cl);
    }
    if (t == 0) {
      if (a.stats_depth) a.stats_depth[k] = depth;
      if (a.stats_res) a.stats_res[k] = gres;
    }
  }
#ifdef MGB_CL_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&g_cl_trace[11], (unsigned long long)(clock64() - kt0_));
#endif
}

// x <- A^{-1} x when every factor of A is a windowed (fast-decaying) recurrence
// and the symbol shift is zero: the windowed branch of chain_solve alone (same
// operations in the same order, bitwise the same result), one CTA barrier per
// factor.  Carry states are stored as (s1, s2) pairs at index chunk + RKD_KMAX
// with the last RKD_KMAX chunks replicated in front (the periodic wrap), so the
// look-back reads K consecutive 16-byte words; wb0 = 2 buffers of
// (T + RKD_KMAX) pairs, alternating per factor.
template <int P, bool FWD>
__device__ __forceinline__ void rkd_factor(const RkdFactor& F, double2* wb, int t, int T, bool own,
                                           double (&x)[P]) {
  const int tl = FWD ? t : T - 1 - t;
  if (own) {
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int qq = 0; qq < P; ++qq) {
      constexpr int dummy = 0;
      (void)dummy;
      const int q = FWD ? qq : P - 1 - qq;
      const double yv = fma(F.a1, s1, fma(F.a2, s2, x[q]));
      x[q] = yv;
      s2 = s1;
      s1 = yv;
    }
    wb[tl + RKD_KMAX] = make_double2(s1, s2);
    if (tl >= T - RKD_KMAX) wb[tl + RKD_KMAX - T] = make_double2(s1, s2);
  }
  __syncthreads();
  if (own) {
    double c1 = 0.0, c2 = 0.0;
    const int K = F.win;
    const double2* p = wb + tl + RKD_KMAX - K;  // chunks tl - K .. tl - 1
#pragma unroll 2
    for (int k = 0; k < K; ++k) {
      const double2 bb = p[k];
      const double n1 = fma(F.M[0], c1, F.M[1] * c2);
      const double n2 = fma(F.M[2], c1, F.M[3] * c2);
      c1 = n1 + bb.x;
      c2 = n2 + bb.y;
    }
#pragma unroll
    for (int qq = 0; qq < P; ++qq) {
      const int q = FWD ? qq : P - 1 - qq;
      x[q] = fma(F.h1[qq], c1, fma(F.h2[qq], c2, x[q]));
    }
  }
}

template <int P>
__device__ __forceinline__ void chain_solve_win(const RkdConst& rk, double2* wb0, int t, int T, bool own,
                                                double (&x)[P]) {
#pragma unroll
  for (int f = 0; f < RKD_MAXF; ++f) {
    if (f < rk.nfac) {
      double2* wb = wb0 + (f & 1) * (T + RKD_KMAX);
      if (rk.f[f].dir > 0)
        rkd_factor<P, true>(rk.f[f], wb, t, T, own, x);
      else
        rkd_factor<P, false>(rk.f[f], wb, t, T, own, x);
    }
  }
  if (own) {
#pragma unroll
    for (int q = 0; q < P; ++q) x[q] *= rk.gain_inv;
  }
}

// ------------------------------------------------ staged SDIRK relaxation
// Dedicated kernel for implicit staged Runge-Kutta fine steps (SDIRK,
// stepping.py:355-380) whose stage solves are all fast-decaying factors
// (windowed carries) and whose -cL stencil is contiguous with span <= 6.
// Differences from relax_kernel<K_RK>:
//  * the stage values never round-trip through a resident row: the solved
//    stage y_i stays in registers, only the HL + HR halo points a neighbour's
//    stencil window needs are published to shared memory (3 of 8 for U3), so
//    a stage costs one CTA barrier per factor plus one for the halo;
//  * the Butcher sums are accumulated column-wise in the reference's order:
//    after z_j every later right-hand side rhs_i (i > j) and the step result
//    receive their a_ij z_j / b_j z_j term (rhs_i = x + a_i0 z_0 + a_i1 z_1 ...
//    is formed in exactly that order, stepping.py:366-372, 378), the ones not
//    needed next live in shared memory, so registers hold one stage at a time
//    and the kernel fits two 512-thread CTAs per SM (<= 64 registers);
//  * rows move between registers and HBM directly (16-byte accesses).
constexpr int RKD_MAXH = 6;  // halo points (stencil span)

#ifndef MGB_RKD_MINB
#define MGB_RKD_MINB 2
#endif
template <int P, int NS, bool ZS, int HL, int HR>
__global__ void __launch_bounds__(512, MGB_RKD_MINB) relax_rkd_kernel(const StepParams* __restrict__ gp,
                                                           const RelaxLaunch L) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int SPB = (int)sizeof(StepParams);
  {
    const int4* src = reinterpret_cast<const int4*>(gp);
    int4* dst = reinterpret_cast<int4*>(smem_raw);
    for (int i = threadIdx.x; i < SPB / 16; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const StepParams& sp = *reinterpret_cast<const StepParams*>(smem_raw);
  const mgb_relax_args& a = L.a;
  const int T = sp.T, n = sp.n, t = threadIdx.x;
  const bool own = t < T;
  // shared layout (doubles): red[64] bc[8] | wb[2][T + RKD_KMAX] pairs | edges[span][T] | acc[NS-1][P][T]
  double* base = reinterpret_cast<double*>(smem_raw + SPB);
  Ctx c;
  c.sp = &sp;
  c.n = n;
  c.T = T;
  c.S = sp.S;
  c.t = t;
  c.own = own;
  c.row = nullptr;  // no resident row (shift == 0: checked by the host)
  c.red = base;
  c.bc = base + 64;
  double2* wb = reinterpret_cast<double2*>(base + 72);
  c.scan = nullptr;
  c.gm = nullptr;
  c.ws = nullptr;
  c.parity = 0;
  c.phase = 0;
  double* edges = base + 72 + 4 * (T + RKD_KMAX);
  const RkdConst& rk = L.rk;
  // window of output q: own-chunk points q - HL .. q + HR (HL / HR halo points from
  // chunk t-1 / t+1; the -cL stencil of upwind order p has HL = (p+1)/2, HR = (p-1)/2)
  constexpr int span = HL + HR;
  static_assert(span <= RKD_MAXH && HL <= P && HR <= P, "halo");
  double* acc = edges + (size_t)span * T;
  double wts[span + 1];
#pragma unroll
  for (int k = 0; k <= span; ++k) wts[k] = sp.win_w[k];
  const int tl = t == 0 ? T - 1 : t - 1, tr = t == T - 1 ? 0 : t + 1;

  for (long long k = blockIdx.x; k < a.n_intervals; k += gridDim.x) {
    const long long kg = a.k_global0 + k;
    const long long rowbase = k * (long long)a.m;
    double y[P];
    const double* csrc = (kg == 0 && a.c_src0) ? a.c_src0 : (a.c_src ? a.c_src + k * a.c_stride : nullptr);
    if (own) {
      if (csrc) {
        load_chunk<P>(csrc, t, y);
      } else {
#pragma unroll
        for (int q = 0; q < P; ++q) y[q] = 0.0;
      }
      if (a.e && kg >= 1) {  // u[m::m] += e[1:] (mgrit.py:246)
        double ev[P];
        load_chunk<P>(a.e + k * a.e_stride, t, ev);
#pragma unroll
        for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], ev[q]);
      }
      if (a.c_out) store_chunk<P>(a.c_out + k * a.c_out_stride, t, y);
    }
    const int nsteps = a.n_fsteps + (a.tail ? 1 : 0);
    for (int j = 1; j <= nsteps; ++j) {
      const bool is_tail = j > a.n_fsteps;
      for (int r = 0; r < sp.repeat; ++r) {
        // ---- one SDIRK step y <- Phi y
        double rhs[P];
#pragma unroll
        for (int q = 0; q < P; ++q) rhs[q] = y[q];
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          double r0[ZS ? P : 1];
          if constexpr (ZS) {
#pragma unroll
            for (int q = 0; q < P; ++q) r0[q] = rhs[q];
          }
          if (ZS && i > 0 && rk.nfac < 2) __syncthreads();  // previous solve's carry buffer is free
          chain_solve_win<P>(rk, wb, t, T, own, rhs);  // rhs <- M^-1 rhs (one CTA barrier per factor)
          double hl[HL > 0 ? HL : 1], hr[HR > 0 ? HR : 1];
          if constexpr (!ZS) {
            // publish the halo points: edges[h][t], h < HL: last HL points, then the first HR
            if (own) {
#pragma unroll
              for (int h = 0; h < HL; ++h) edges[h * T + t] = rhs[P - HL + h];
#pragma unroll
              for (int h = 0; h < HR; ++h) edges[(HL + h) * T + t] = rhs[h];
            }
            __syncthreads();
            if (own) {
#pragma unroll
              for (int h = 0; h < HL; ++h) hl[h] = edges[h * T + tl];
#pragma unroll
              for (int h = 0; h < HR; ++h) hr[h] = edges[(HL + h) * T + tr];
            }
          }
          // ---- stage value z_q, then the column-wise Butcher accumulation (reference
          // order, zero entries skipped): acc slot i2 - 2 holds rhs_{i2} for i2 >= i + 2,
          // slot NS - 2 the step result; rhs_{i+1} (or the result after the last stage)
          // goes to registers
          double nxt[P];
          if (own) {
#pragma unroll
            for (int q = 0; q < P; ++q) {
              double zq;
              if constexpr (ZS) {
                // M y = rhs, M = I - gamma cL  =>  cL y = (y - rhs) / gamma (fast mode only)
                zq = __dmul_rn(__dsub_rn(rhs[q], r0[q]), rk.inv_gamma);
              } else {
                // numpy's rolled sum (circulant.py:119-123): out = 0; out += w_k * roll(v)
                zq = 0.0;
#pragma unroll
                for (int kk = 0; kk <= span; ++kk) {
                  const int w = q + kk - HL;  // own-chunk index of the tap
                  const double v = w < 0 ? hl[w + HL < 0 ? 0 : w + HL] : (w >= P ? hr[w - P < HR ? w - P : 0] : rhs[w]);
                  zq = madd<true>(zq, wts[kk], v);
                }
              }
#pragma unroll
              for (int i2 = i + 1; i2 <= NS; ++i2) {
                const double co = i2 < NS ? rk.A[i2 * 3 + i] : rk.b[i];
                double* slot = acc + (size_t)(i2 < NS ? i2 - 2 : NS - 2) * P * T;
                const bool to_regs = (i2 == i + 1 && i2 < NS) || (i2 == NS && i == NS - 1);
                const double b0 = i == 0 ? y[q] : slot[q * T + t];
                const double v = co != 0.0 ? __dadd_rn(b0, __dmul_rn(co, zq)) : b0;
                if (to_regs) nxt[q] = v; else slot[q * T + t] = v;
              }
            }
#pragma unroll
            for (int q = 0; q < P; ++q) rhs[q] = nxt[q];
          }
        }
#pragma unroll
        for (int q = 0; q < P; ++q) y[q] = rhs[q];  // the last column left the step result in rhs
      }
      const long long grow = is_tail ? rowbase + a.m : rowbase + j;
      if (!is_tail) {
        if (own) {
          if (a.g) {
            double gv[P];
            load_chunk<P>(a.g + grow * n, t, gv);
#pragma unroll
            for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], gv[q]);  // upd + g (mgrit.py:142)
          }
          if (a.write_f == 2 || (a.write_f == 1 && j == a.n_fsteps)) store_chunk<P>(a.u + grow * n, t, y);
        }
      } else if (a.tail == 1) {  // C-relaxation (mgrit.py:148-149)
        if (own) {
          if (a.g) {
            double gv[P];
            load_chunk<P>(a.g + grow * n, t, gv);
#pragma unroll
            for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], gv[q]);
          }
          store_chunk<P>(a.tail_out + k * a.tail_stride, t, y);
        }
      } else {  // residual g + Phi u - u_C (mgrit.py:159-161)
        double part = 0.0;
        if (own) {
          double rr[P];
          if (a.g) {
            double gv[P];
            load_chunk<P>(a.g + grow * n, t, gv);
#pragma unroll
            for (int q = 0; q < P; ++q) rr[q] = __dadd_rn(gv[q], y[q]);
          } else {
#pragma unroll
            for (int q = 0; q < P; ++q) rr[q] = y[q];
          }
          if (a.z_out) store_chunk<P>(a.z_out + k * a.z_stride, t, rr);  // g + Phi u_last
          double cr[P];
          load_chunk<P>(a.cref + k * a.cref_stride, t, cr);
          if (a.cref_e) {
            double ev[P];
            load_chunk<P>(a.cref_e + k * a.cref_e_stride, t, ev);
#pragma unroll
            for (int q = 0; q < P; ++q) cr[q] = __dadd_rn(cr[q], ev[q]);
          }
#pragma unroll
          for (int q = 0; q < P; ++q) {
            rr[q] = __dsub_rn(rr[q], cr[q]);
            part = fma(rr[q], rr[q], part);
          }
          if (a.tail_out) store_chunk<P>(a.tail_out + k * a.tail_stride, t, rr);
        }
        if (a.partials) {
          const double sum = block_sum(c, part);
          if (t == 0) a.partials[k] = sum;
        }
      }
    }
    if (a.c_last_out && k == a.n_intervals - 1 && own) {  // final C-point (k+1 >= 1)
      double cl[P];
      if (a.c_src) {
        load_chunk<P>(a.c_src + (k + 1) * a.c_stride, t, cl);
      } else {
#pragma unroll
        for (int q = 0; q < P; ++q) cl[q] = 0.0;
      }
      if (a.e) {
        double ev[P];
        load_chunk<P>(a.e + (k + 1) * a.e_stride, t, ev);
#pragma unroll
        for (int q = 0; q < P; ++q) cl[q] = __dadd_rn(cl[q], ev[q]);
      }
      store_chunk<P>(a.c_last_out, t, cl);
    }
  }
}

// ------------------------------------------- SL + direct correction solve
// Dedicated kernel for the corrected semi-Lagrangian coarse steps with a direct
// solve (stepping.py:546-551: x = (I - phi D)^-1 SL u): the SL interpolation
// stencil is a contiguous window at a far offset (read from the resident row
// through a register window: double-buffered slice with wrap replicas, one CTA
// barrier per step besides the factors'), the factor solves take their
// coefficients and scan tables from the kernel parameters (constant bank) and
// rows move between registers and HBM directly.  Fast-decaying factors use the
// windowed carries of rkd_factor, slow-decaying ones (deep levels) the
// hierarchical scan of chain_solve (warp Kogge-Stone, warp 0 over the warp
// totals with the periodic closure); same operations in the same order as the
// generic kernel.
template <int P, bool FWD>
__device__ __forceinline__ void sld_factor(const SldFactor& F, double2* wb, double* st, int t, int T,
                                           double (&x)[P]) {
  const int tl = FWD ? t : T - 1 - t;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int qq = 0; qq < P; ++qq) {
    const int q = FWD ? qq : P - 1 - qq;
    const double yv = fma(F.a1, s1, fma(F.a2, s2, x[q]));
    x[q] = yv;
    s2 = s1;
    s1 = yv;
  }
  double c1 = 0.0, c2 = 0.0;
  if (F.win > 0) {
    wb[tl + RKD_KMAX] = make_double2(s1, s2);
    if (tl >= T - RKD_KMAX) wb[tl + RKD_KMAX - T] = make_double2(s1, s2);
    __syncthreads();
    const int K = F.win;
    const double2* p = wb + tl + RKD_KMAX - K;  // chunks tl - K .. tl - 1
#pragma unroll 2
    for (int k = 0; k < K; ++k) {
      const double2 bb = p[k];
      const double n1 = fma(F.M[0], c1, F.M[1] * c2);
      const double n2 = fma(F.M[2], c1, F.M[3] * c2);
      c1 = n1 + bb.x;
      c2 = n2 + bb.y;
    }
  } else {
    // hierarchical scan over logical chunks (T a multiple of 32)
    double* cin = st + 64;
    const int NW = T >> 5, lane = t & 31, w = t >> 5;
    const int ll = FWD ? lane : 31 - lane;
    const int lw = FWD ? w : NW - 1 - w;
    double y1 = s1, y2 = s2;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      const int off = 1 << d;
      const int src = (FWD ? lane - off : lane + off) & 31;
      double p1 = __shfl_sync(0xffffffffu, y1, src), p2 = __shfl_sync(0xffffffffu, y2, src);
      if (ll >= off) {
        const double n1 = fma(F.Mpow[d][0], p1, F.Mpow[d][1] * p2);
        const double n2 = fma(F.Mpow[d][2], p1, F.Mpow[d][3] * p2);
        y1 += n1;
        y2 += n2;
      }
    }
    const int s1src = (FWD ? lane - 1 : lane + 1) & 31;
    double e1 = __shfl_sync(0xffffffffu, y1, s1src), e2 = __shfl_sync(0xffffffffu, y2, s1src);
    if (ll == 0) e1 = e2 = 0.0;
    if (ll == 31) {
      st[lw] = y1;
      st[32 + lw] = y2;
    }
    __syncthreads();
    if (w == 0) {
      double a1w = lane < NW ? st[lane] : 0.0, a2w = lane < NW ? st[32 + lane] : 0.0;
#pragma unroll
      for (int d = 0; d < 5; ++d) {
        const int off = 1 << d;
        double p1 = __shfl_up_sync(0xffffffffu, a1w, off), p2 = __shfl_up_sync(0xffffffffu, a2w, off);
        if (lane >= off) {
          const double n1 = fma(F.Mpow[5 + d][0], p1, F.Mpow[5 + d][1] * p2);
          const double n2 = fma(F.Mpow[5 + d][2], p1, F.Mpow[5 + d][3] * p2);
          a1w += n1;
          a2w += n2;
        }
      }
      double z1 = __shfl_sync(0xffffffffu, a1w, NW - 1), z2 = __shfl_sync(0xffffffffu, a2w, NW - 1);
      {  // s_{-1}: periodic closure
        const double n1 = fma(F.Winv[0], z1, F.Winv[1] * z2);
        const double n2 = fma(F.Winv[2], z1, F.Winv[3] * z2);
        z1 = n1;
        z2 = n2;
      }
      double x1 = __shfl_up_sync(0xffffffffu, a1w, 1), x2 = __shfl_up_sync(0xffffffffu, a2w, 1);
      if (lane == 0) x1 = x2 = 0.0;
#pragma unroll
      for (int d = 0; d < 5; ++d)
        if ((lane >> d) & 1) {  // (M^32)^lw s_{-1}
          const double n1 = fma(F.Mpow[5 + d][0], z1, F.Mpow[5 + d][1] * z2);
          const double n2 = fma(F.Mpow[5 + d][2], z1, F.Mpow[5 + d][3] * z2);
          z1 = n1;
          z2 = n2;
        }
      if (lane < NW) {
        cin[lane] = x1 + z1;
        cin[32 + lane] = x2 + z2;
      }
    }
    __syncthreads();
    c1 = cin[lw];
    c2 = cin[32 + lw];
#pragma unroll
    for (int d = 0; d < 5; ++d)
      if ((ll >> d) & 1) {  // M^ll C_w
        const double n1 = fma(F.Mpow[d][0], c1, F.Mpow[d][1] * c2);
        const double n2 = fma(F.Mpow[d][2], c1, F.Mpow[d][3] * c2);
        c1 = n1;
        c2 = n2;
      }
    c1 += e1;
    c2 += e2;
  }
#pragma unroll
  for (int qq = 0; qq < P; ++qq) {
    const int q = FWD ? qq : P - 1 - qq;
    x[q] = fma(F.h1[qq], c1, fma(F.h2[qq], c2, x[q]));
  }
}

template <int P, int SPAN>
__global__ void __launch_bounds__(512, 1) relax_sld_kernel(const StepParams* __restrict__ gp,
                                                           const RelaxLaunch L) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const mgb_relax_args& a = L.a;
  const SldConst& sd = L.sd;
  const int n = gp->n, T = gp->T, t = threadIdx.x;  // T == blockDim.x, a multiple of 32
  const int S = T + WIN_X;                           // chunk row + wrap replica columns
  const int lo = gp->win_lo, reps = gp->repeat;
  int tb = t + lo / P;
  tb = tb >= T ? tb - T : tb;
  const int r0 = lo & (P - 1);
  // shared layout (doubles): red[64] | st/cin[128] | wb[2][T + RKD_KMAX] pairs | row[2][P][S]
  double* base = reinterpret_cast<double*>(smem_raw);
  Ctx c;
  c.red = base;
  c.parity = 0;
  c.T = T;
  c.t = t;
  double* st = base + 64;
  double2* wb = reinterpret_cast<double2*>(base + 192);
  double* row0 = base + 192 + 4 * (T + RKD_KMAX);
  const int PS = P * S;
  double wd[SPAN + 1];
#pragma unroll
  for (int k = 0; k <= SPAN; ++k) wd[k] = L.win_w[k];

  for (long long k = blockIdx.x; k < a.n_intervals; k += gridDim.x) {
    const long long kg = a.k_global0 + k;
    const long long rowbase = k * (long long)a.m;
    double y[P];
    const double* csrc = (kg == 0 && a.c_src0) ? a.c_src0 : (a.c_src ? a.c_src + k * a.c_stride : nullptr);
    if (csrc) {
      load_chunk<P>(csrc, t, y);
    } else {
#pragma unroll
      for (int q = 0; q < P; ++q) y[q] = 0.0;
    }
    if (a.e && kg >= 1) {  // u[m::m] += e[1:] (mgrit.py:246)
      double ev[P];
      load_chunk<P>(a.e + k * a.e_stride, t, ev);
#pragma unroll
      for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], ev[q]);
    }
    if (a.c_out) store_chunk<P>(a.c_out + k * a.c_out_stride, t, y);
    int cur = 0;
    __syncthreads();  // previous interval's readers of both row buffers are done
    {
      double* row = row0;
#pragma unroll
      for (int q = 0; q < P; ++q) {
        row[q * S + t] = y[q];
        if (t < WIN_X) row[q * S + T + t] = y[q];
      }
    }
    __syncthreads();
    const int nsteps = a.n_fsteps + (a.tail ? 1 : 0);
    for (int j = 1; j <= nsteps; ++j) {
      const bool is_tail = j > a.n_fsteps;
      const long long grow = is_tail ? rowbase + a.m : rowbase + j;
      if (a.g) {  // this step's rhs chunk into L1 while the step runs
        const double* gp1 = a.g + grow * n + (size_t)t * P;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(gp1));
      }
      for (int r = 0; r < reps; ++r) {
        // ---- b = SL(row): register window at the departure offset, exact rolled sum
        const double* src = row0 + cur * PS;
        {
          double win[P + SPAN];
#pragma unroll
          for (int w = 0; w < P + SPAN; ++w) {
            const int cw = r0 + w;
            win[w] = src[(cw & (P - 1)) * S + tb + cw / P];
          }
#pragma unroll
          for (int q = 0; q < P; ++q) {
            double acc = 0.0;
#pragma unroll
            for (int kk = 0; kk <= SPAN; ++kk) acc = madd<true>(acc, wd[kk], win[q + kk]);
            y[q] = acc;
          }
        }
        // ---- x = (I - phi D)^-1 b: factorised periodic solve
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          if (f < sd.nfac) {
            double2* wbf = wb + f * (T + RKD_KMAX);
            if (sd.f[f].dir > 0)
              sld_factor<P, true>(sd.f[f], wbf, st, t, T, y);
            else
              sld_factor<P, false>(sd.f[f], wbf, st, t, T, y);
          }
        }
#pragma unroll
        for (int q = 0; q < P; ++q) y[q] *= sd.gain_inv;
        if (r + 1 < reps) {
          double* dst = row0 + (cur ^ 1) * PS;
#pragma unroll
          for (int q = 0; q < P; ++q) {
            dst[q * S + t] = y[q];
            if (t < WIN_X) dst[q * S + T + t] = y[q];
          }
          cur ^= 1;
          __syncthreads();
        }
      }
      if (!is_tail) {
        if (a.g) {
          double gv[P];
          load_chunk<P>(a.g + grow * n, t, gv);
#pragma unroll
          for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], gv[q]);  // upd + g (mgrit.py:142)
        }
        if (a.write_f == 2 || (a.write_f == 1 && j == a.n_fsteps)) store_chunk<P>(a.u + grow * n, t, y);
        if (j < nsteps) {  // republish for the next step
          double* dst = row0 + (cur ^ 1) * PS;
#pragma unroll
          for (int q = 0; q < P; ++q) {
            dst[q * S + t] = y[q];
            if (t < WIN_X) dst[q * S + T + t] = y[q];
          }
          cur ^= 1;
          __syncthreads();
        }
      } else if (a.tail == 1) {  // C-relaxation (mgrit.py:148-149)
        if (a.g) {
          double gv[P];
          load_chunk<P>(a.g + grow * n, t, gv);
#pragma unroll
          for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], gv[q]);
        }
        store_chunk<P>(a.tail_out + k * a.tail_stride, t, y);
      } else {  // residual g + Phi u - u_C (mgrit.py:159-161)
        double part = 0.0;
        double rr[P];
        if (a.g) {
          double gv[P];
          load_chunk<P>(a.g + grow * n, t, gv);
#pragma unroll
          for (int q = 0; q < P; ++q) rr[q] = __dadd_rn(gv[q], y[q]);
        } else {
#pragma unroll
          for (int q = 0; q < P; ++q) rr[q] = y[q];
        }
        {
          double cr[P];
          load_chunk<P>(a.cref + k * a.cref_stride, t, cr);
          if (a.cref_e) {
            double ev[P];
            load_chunk<P>(a.cref_e + k * a.cref_e_stride, t, ev);
#pragma unroll
            for (int q = 0; q < P; ++q) cr[q] = __dadd_rn(cr[q], ev[q]);
          }
#pragma unroll
          for (int q = 0; q < P; ++q) {
            rr[q] = __dsub_rn(rr[q], cr[q]);
            part = fma(rr[q], rr[q], part);
          }
        }
        if (a.tail_out) store_chunk<P>(a.tail_out + k * a.tail_stride, t, rr);
        if (a.partials) {
          const double sum = block_sum(c, part);
          if (t == 0) a.partials[k] = sum;
        }
      }
    }
    if (a.c_last_out && k == a.n_intervals - 1) {  // final C-point (k+1 >= 1)
      double cl[P];
      if (a.c_src) {
        load_chunk<P>(a.c_src + (k + 1) * a.c_stride, t, cl);
      } else {
#pragma unroll
        for (int q = 0; q < P; ++q) cl[q] = 0.0;
      }
      if (a.e) {
        double ev[P];
        load_chunk<P>(a.e + (k + 1) * a.e_stride, t, ev);
#pragma unroll
        for (int q = 0; q < P; ++q) cl[q] = __dadd_rn(cl[q], ev[q]);
      }
      store_chunk<P>(a.c_last_out, t, cl);
    }
  }
}

// ------------------------------------------- explicit-stencil relaxation
// Dedicated kernel for assembled explicit stencils (the fine ERK levels):
// stencil weights are kernel parameters (constant-bank operands, no registers),
// the resident slice is double-buffered (one CTA barrier per step), outputs
// are produced in part-chunks straight into the other buffer (few live
// registers: 2 CTAs/SM at 256 threads, 1 CTA/SM at 512), rows stream to HBM
// with 16-byte stores issued from INSIDE the next step's stencil arithmetic
// (the row just completed is that step's read-only source), so the store
// traffic overlaps the FP64 work instead of following it.  Same argument
// semantics as relax_kernel (mgb_relax_args).
template <int P>
__device__ __forceinline__ void slice_store2(const double* row, double* dst, int i, int S) {
  // elements i, i+1 (i even: same chunk column pair), natural order, streaming
  const int s0 = saddr<P>(i, S);
  __stcs(reinterpret_cast<double2*>(dst + i), make_double2(row[s0], row[s0 + S]));
}

// Fixed-geometry builds (TT = threads = chunks, compile time): the slice row
// stride is the constant WIN_S<TT> and every chunk row is extended by WIN_X
// columns that replicate columns 0..WIN_X-1 (the periodic wrap), so a window
// read is base + immediate: no wrap arithmetic and no address registers.
template <int TT>
struct WinGeo {
  static constexpr int S = TT + 17;  // == 1 (mod 16): conflict-free rows and natural-order copies
};
template <int P, int TT>
__device__ __forceinline__ void slice_put(double* row, int i, double v, int S) {
  const int s = saddr<P>(i, S);
  row[s] = v;
  if (TT > 0 && i < WIN_X * P) row[s + TT] = v;  // wrap replica
}

// One stencil step src -> dst.  ``gdst`` (may be null): natural-order global copy
// of the SOURCE row, issued in pieces between the outputs.
template <int P, int SPAN, bool EXACT, int TT>
__device__ __forceinline__ void win_step(const double* __restrict__ src, double* __restrict__ dst,
                                         int t, int T, int S, int tb, int r0,
                                         const double (&wd)[SPAN + 1], double* __restrict__ gdst, int n, int nthr,
                                         bool own) {
  // outputs per pass (window of H + SPAN in registers)
  // (2 measured fastest on B200 for spans 9 and 30 at 16 points per thread -- cfg4 fine
  // FR / CF 2.16 / 2.34 ms vs 2.26 / 2.44 at 4 and 2.29 / 2.50 at 8: wider parts trade
  // fewer shared loads for registers the FP64 chains need)
#ifndef MGB_WIN_H
#define MGB_WIN_H 2
#endif
  constexpr int H = MGB_WIN_H < P ? MGB_WIN_H : P;
  static_assert(TT == 0 || (P - 1 + P - 1 + SPAN) / P < WIN_X, "wrap replica too narrow");
  int gi = 2 * t;  // next natural-order element pair this thread copies
#pragma unroll
  for (int h = 0; h < P; h += H) {
    double win[H + SPAN];
    if (own) {
#pragma unroll
      for (int w = 0; w < H + SPAN; ++w) {
        const int cw = r0 + h + w;
        if constexpr (TT > 0) {
          win[w] = src[(cw & (P - 1)) * WinGeo<TT>::S + cw / P + tb];
        } else {
          int tt = tb + cw / P;
          tt = tt >= T ? tt - T : tt;
          tt = tt >= T ? tt - T : tt;
          win[w] = src[(cw & (P - 1)) * S + tt];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < H; ++q) {
      if (own) {
        // numpy starts from zeros: 0 + w0*v0 == w0*v0 (up to the sign of an exact zero)
        double acc = EXACT ? __dmul_rn(wd[0], win[q]) : wd[0] * win[q];
#pragma unroll
        for (int k = 1; k <= SPAN; ++k) acc = madd<EXACT>(acc, wd[k], win[q + k]);
        if constexpr (TT > 0) {
          dst[(h + q) * WinGeo<TT>::S + t] = acc;
          if (t < WIN_X) dst[(h + q) * WinGeo<TT>::S + TT + t] = acc;
        } else {
          dst[(h + q) * S + t] = acc;
        }
      }
      if (gdst && ((h + q) & 1) && gi < n) {  // one 16-byte piece of the source row per two outputs
        slice_store2<P>(src, gdst, gi, TT > 0 ? WinGeo<TT>::S : S);
        gi += 2 * nthr;
      }
    }
  }
  if (gdst)
    for (; gi < n; gi += 2 * nthr) slice_store2<P>(src, gdst, gi, TT > 0 ? WinGeo<TT>::S : S);
}

template <int P>
__device__ __forceinline__ void slice_to_global(const double* row, double* dst, int n, int S) {
  // natural-order 16-byte stores (n even), streaming
  for (int i = 2 * threadIdx.x; i < n; i += 2 * blockDim.x) slice_store2<P>(row, dst, i, S);
}

#ifndef MGB_WIN_U
#define MGB_WIN_U 4
#endif
constexpr int WIN_U = MGB_WIN_U;  // row loads in flight per thread at interval head / tail
// one thread issues an L2 prefetch of a contiguous byte range (no registers, no completion)
__device__ __forceinline__ void l2_prefetch(const void* g, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}

template <int P, int SPAN, bool EXACT, int MAXT = 256, int MINB = 2, int TT = 0>
__global__ void __launch_bounds__(MAXT, MINB) relax_win_kernel(const StepParams* __restrict__ gp,
                                                               const RelaxLaunch L) {
  // Natural-order global traffic: thread t touches elements 2t, 2t+1 (+2*blockDim) with
  // 16-byte coalesced accesses and scatters/gathers the slice layout in shared memory.
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = gp->n, T = TT > 0 ? TT : gp->T, S = TT > 0 ? WinGeo<TT>::S : gp->S;
  double wd[SPAN + 1];  // uniform values read from the parameter bank: uniform registers / operands
#pragma unroll
  for (int k = 0; k <= SPAN; ++k) wd[k] = L.win_w[k];
  const int t = threadIdx.x;
  const bool own = TT > 0 ? true : t < T;  // fixed geometry: one chunk per thread
  const int lo = gp->win_lo;
  int tb = t + lo / P;
  tb = tb >= T ? tb - T : tb;
  const int r0 = lo & (P - 1);
  double* const row0 = reinterpret_cast<double*>(smem_raw);
  const int PS = P * S;
  double* red = row0 + 2 * PS;
  const mgb_relax_args& a = L.a;
  const int nthr = TT > 0 ? TT : (int)blockDim.x;
  const uint32_t rowbytes = (uint32_t)n * 8u;
  // Contiguous interval blocks per CTA.  When the residual tail of interval k
  // reads exactly the rows the head of interval k+1 starts from (CF and FR
  // passes: cref = c_src + c_stride, cref_e = e + e_stride), the tail leaves the
  // corrected C-point C_{k+1} (+ e_{k+1}) in the free slice buffer and writes
  // c_out, so the next head needs no global loads (the same __dadd_rn sum).
  const long long nI = a.n_intervals, G = gridDim.x;
  const long long kb0 = (long long)blockIdx.x * nI / G, kb1 = ((long long)blockIdx.x + 1) * nI / G;
  const bool chain = a.tail == 2 && a.c_src && a.cref == a.c_src + a.c_stride &&
                     a.cref_stride == a.c_stride &&
                     ((!a.e && !a.cref_e) ||
                      (a.e && a.cref_e == a.e + a.e_stride && a.cref_e_stride == a.e_stride));
  int have = -1;  // slice buffer already holding this interval's start row
  for (long long k = kb0; k < kb1; ++k) {
    const long long kg = a.k_global0 + k;
    const long long rowbase = k * (long long)a.m;
    const double* csrc = (kg == 0 && a.c_src0) ? a.c_src0 : (a.c_src ? a.c_src + k * a.c_stride : nullptr);
    const double* erow = (a.e && kg >= 1) ? a.e + k * a.e_stride : nullptr;
    __syncthreads();  // previous interval's readers of both buffers are done
    // interval start: C-point (+ correction, mgrit.py:246) -> slice buffer 0 (and c_out)
    // loads batched WIN_U deep (all in flight before the first use)
    const int start_buf = have >= 0 ? have : 0;
    for (int i0 = 2 * t; have < 0 && i0 < n; i0 += 2 * nthr * WIN_U) {
      double2 y[WIN_U], ev[WIN_U];
#pragma unroll
      for (int u = 0; u < WIN_U; ++u) {
        const int i = i0 + 2 * nthr * u;
        y[u] = (csrc && i < n) ? __ldg(reinterpret_cast<const double2*>(csrc + i)) : make_double2(0.0, 0.0);
        ev[u] = (erow && i < n) ? __ldg(reinterpret_cast<const double2*>(erow + i)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < WIN_U; ++u) {
        const int i = i0 + 2 * nthr * u;
        if (i < n) {
          if (erow) {
            y[u].x = __dadd_rn(y[u].x, ev[u].x);
            y[u].y = __dadd_rn(y[u].y, ev[u].y);
          }
          if (a.c_out) *reinterpret_cast<double2*>(a.c_out + k * a.c_out_stride + i) = y[u];
          slice_put<P, TT>(row0, i, y[u].x, S);
          slice_put<P, TT>(row0, i + 1, y[u].y, S);
        }
      }
    }
    have = -1;
    if (t == 0) {  // warm L2 for the next interval this CTA handles
      const long long kn = k + 1;
      if (kn < kb1) {
        if (a.c_src) l2_prefetch(a.c_src + kn * a.c_stride, rowbytes);
        if (a.e) l2_prefetch(a.e + kn * a.e_stride, rowbytes);
        // chained passes: cref[k] == c_src[k+1], already prefetched above
        if (!chain && a.tail == 2 && a.cref) l2_prefetch(a.cref + kn * a.cref_stride, rowbytes);
        if (!chain && a.tail == 2 && a.cref_e) l2_prefetch(a.cref_e + kn * a.cref_e_stride, rowbytes);
      }
      if (a.g) l2_prefetch(a.g + (rowbase + 1) * n, rowbytes * (uint32_t)(a.n_fsteps + (a.tail ? 1 : 0)));
    }
    __syncthreads();
    int cur = start_buf;
    double* pend = nullptr;  // global row of the F-point held by buffer `cur`, not yet stored
    for (int j = 1; j <= a.n_fsteps; ++j) {
      double* src = row0 + cur * PS;
      double* dst = row0 + (cur ^ 1) * PS;
      win_step<P, SPAN, EXACT, TT>(src, dst, t, T, S, tb, r0, wd, pend, n, nthr, own);
      __syncthreads();  // dst complete; src free for step j+1's output
      if (a.g) {  // upd + g (mgrit.py:142), natural order, then republish
        const double* gr = a.g + (rowbase + j) * n;
        for (int i = 2 * t; i < n; i += 2 * nthr) {
          const double2 gv = __ldg(reinterpret_cast<const double2*>(gr + i));
          const int s0 = saddr<P>(i, S), s1 = saddr<P>(i + 1, S);
          slice_put<P, TT>(dst, i, __dadd_rn(dst[s0], gv.x), S);
          slice_put<P, TT>(dst, i + 1, __dadd_rn(dst[s1], gv.y), S);
        }
        __syncthreads();
      }
      cur ^= 1;
      pend = (a.write_f == 2 || (a.write_f == 1 && j == a.n_fsteps)) ? a.u + (rowbase + j) * n : nullptr;
    }
    if (!a.tail && pend) slice_to_global<P>(row0 + cur * PS, pend, n, S);
    if (a.tail) {  // one more step from the last F-point, into the free buffer
      double* const src = row0 + cur * PS;  // free after the step: next start row (chain)
      double* zb = row0 + (cur ^ 1) * PS;
      const bool hand = chain && k + 1 < kb1;
      win_step<P, SPAN, EXACT, TT>(src, zb, t, T, S, tb, r0, wd, pend, n, nthr, own);
      __syncthreads();
      const long long grow = rowbase + a.m;
      double part = 0.0;
      const double* gsrc = a.g ? a.g + grow * n : nullptr;
      const double* crow = a.tail == 2 ? a.cref + k * a.cref_stride : nullptr;
      const double* cerow = (a.tail == 2 && a.cref_e) ? a.cref_e + k * a.cref_e_stride : nullptr;
      for (int i0 = 2 * t; i0 < n; i0 += 2 * nthr * WIN_U) {
        double2 gv[WIN_U], c[WIN_U], ce[WIN_U];
#pragma unroll
        for (int u = 0; u < WIN_U; ++u) {  // loads batched WIN_U deep
          const int i = i0 + 2 * nthr * u;
          const bool in = i < n;
          gv[u] = (gsrc && in) ? __ldg(reinterpret_cast<const double2*>(gsrc + i)) : make_double2(0.0, 0.0);
          c[u] = (crow && in) ? __ldg(reinterpret_cast<const double2*>(crow + i)) : make_double2(0.0, 0.0);
          ce[u] = (cerow && in) ? __ldg(reinterpret_cast<const double2*>(cerow + i)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < WIN_U; ++u) {
          const int i = i0 + 2 * nthr * u;
          if (i >= n) continue;
          double2 z = make_double2(zb[saddr<P>(i, S)], zb[saddr<P>(i + 1, S)]);
          if (gsrc) {
            z.x = __dadd_rn(gv[u].x, z.x);  // g + Phi u (commutative: bitwise either order)
            z.y = __dadd_rn(gv[u].y, z.y);
          }
          if (a.tail == 2 && a.z_out) *reinterpret_cast<double2*>(a.z_out + k * a.z_stride + i) = z;
          if (a.tail == 1) {  // C-relaxation (mgrit.py:148-149)
            *reinterpret_cast<double2*>(a.tail_out + k * a.tail_stride + i) = z;
          } else {  // residual (g + Phi u) - u_C (mgrit.py:159-161)
            double2 cc = c[u];
            if (cerow) {
              cc.x = __dadd_rn(cc.x, ce[u].x);
              cc.y = __dadd_rn(cc.y, ce[u].y);
            }
            if (hand) {  // == the next head's C_{k+1} (+ e_{k+1})
              slice_put<P, TT>(src, i, cc.x, S);
              slice_put<P, TT>(src, i + 1, cc.y, S);
              if (a.c_out) *reinterpret_cast<double2*>(a.c_out + (k + 1) * a.c_out_stride + i) = cc;
            }
            const double2 r = make_double2(__dsub_rn(z.x, cc.x), __dsub_rn(z.y, cc.y));
            part = fma(r.x, r.x, part);
            part = fma(r.y, r.y, part);
            if (a.tail_out) *reinterpret_cast<double2*>(a.tail_out + k * a.tail_stride + i) = r;
          }
        }
      }
      if (hand) have = cur;
      if (a.tail == 2 && a.partials) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        const int w = t >> 5, lane = t & 31;
        if (lane == 0) red[w] = part;
        __syncthreads();
        if (t == 0) {
          double s = 0.0;
          for (int i = 0; i < (nthr >> 5); ++i) s += red[i];
          a.partials[k] = s;
        }
      }
    }
    if (a.c_last_out && k == a.n_intervals - 1) {  // final C-point (k+1 >= 1)
      for (int i = 2 * t; i < n; i += 2 * nthr) {
        double2 v = a.c_src ? __ldg(reinterpret_cast<const double2*>(a.c_src + (k + 1) * a.c_stride + i))
                            : make_double2(0.0, 0.0);
        if (a.e) {
          const double2 ev = __ldg(reinterpret_cast<const double2*>(a.e + (k + 1) * a.e_stride + i));
          v.x = __dadd_rn(v.x, ev.x);
          v.y = __dadd_rn(v.y, ev.y);
        }
        *reinterpret_cast<double2*>(a.c_last_out + i) = v;
      }
    }
  }
}

__global__ void sum_kernel(const double* __restrict__ p, long long n, double* out);

}  // namespace mgb
