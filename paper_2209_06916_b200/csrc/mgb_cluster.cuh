// mgb_cluster.cuh -- semi-Lagrangian + GMRES coarse relaxation on a thread-block
// cluster (sm_100a).
//
// Deep coarse levels have few intervals (cfg2: 32, 4, 1 rows) and each coarse
// step is a capped GMRES solve (circulant.py:262-332) whose cost is a chain of
// dependent reductions.  One CLUSTER of C CTAs (C = 8 or 16) owns one interval:
//   * the periodic row is split into C contiguous slices, one per CTA (SM);
//   * the Krylov basis V (cap+1 vectors) lives in REGISTERS (P <= 2 points per
//     thread), so Arnoldi never touches HBM/L2;
//   * orthogonalisation is CGS2 (two classical Gram-Schmidt passes): each pass
//     is ONE multi-value cluster all-reduce (warp butterflies, then per-CTA
//     partials pushed into every CTA's shared memory over DSMEM, one cluster
//     barrier, fixed rank-order sum -> bitwise identical in every thread), so an
//     Arnoldi step costs 3 cluster reductions instead of j+2 (MGS).  CGS2 and the
//     reference's MGS agree to rounding; the oracle's own reduction-order noise
//     bounds the difference;
//   * the (I - phi D) stencil needs only H <= 4 halo points from the two
//     neighbouring slices, pushed into their halo slots before the norm barrier;
//   * the SL stencil (large departure shift) reads any slice via DSMEM.
// Every CTA evaluates the Givens updates on identical values, so stop decisions
// are uniform across the cluster.
#pragma once
#include <cooperative_groups.h>

#include "mgb_device.cuh"

namespace mgb {
namespace cg = cooperative_groups;

constexpr int CL_H = 4;        // halo reach of the correction stencil
constexpr int CL_MAXW = 8;     // warps per CTA (T <= 256)
constexpr int CL_MAXC = 16;    // CTAs per cluster

template <int CAP>
struct ClLayout {
  // doubles, after the StepParams copy
  static constexpr int N1 = CAP + 1;
  __host__ __device__ static int in_row(int) { return 0; }
  __host__ __device__ static int gm(int nc) { return nc; }
  __host__ __device__ static int wred(int nc) { return gm(nc) + nc + 2 * CL_H; }
  __host__ __device__ static int cred(int nc) { return wred(nc) + (N1 > CL_MAXW ? N1 : CL_MAXW) * N1; }
  __host__ __device__ static int tot(int nc) { return cred(nc) + 2 * CL_MAXC * N1; }
  __host__ __device__ static int hcol(int nc) { return tot(nc) + N1; }
  __host__ __device__ static int Rm(int nc) { return hcol(nc) + N1 + 1; }
  __host__ __device__ static int cs(int nc) { return Rm(nc) + CAP * CAP; }
  __host__ __device__ static int sn(int nc) { return cs(nc) + CAP; }
  __host__ __device__ static int gg(int nc) { return sn(nc) + CAP; }
  __host__ __device__ static int ybuf(int nc) { return gg(nc) + N1; }
  __host__ __device__ static int bc(int nc) { return ybuf(nc) + N1; }
  __host__ __device__ static int mbar(int nc) { return bc(nc) + 8; }
  __host__ __device__ static int Z(int nc) { return mbar(nc) + 2; }
  __host__ __device__ static int V(int nc) { return Z(nc) + N1 * nc; }
  __host__ __device__ static int total(int nc) { return V(nc) + N1 * nc; }
};

struct ClCtx {
  const StepParams* sp;
  double* in_row;
  double* gm;   // gm[0..H) left halo, gm[H..H+nc) own, gm[H+nc..) right halo
  double* wred;
  double* cred;
  double* tot;
  int t, T, nc, C, rank, base, lane, warp, nw, parity;
};

__device__ __forceinline__ uint32_t cl_map(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
// plain store into a peer CTA's shared memory (made visible by the next cluster barrier)
__device__ __forceinline__ void st_cluster_f64(uint32_t rdst, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rdst), "d"(v) : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n"
               ::: "memory");
}

// Warp-level reduce-scatter of up to 32 values: lane l ends up with the warp
// total of value l (31 shuffles instead of 5 per value).
template <int N>
__device__ __forceinline__ double warp_reduce_scatter(const double (&v)[N], int lane) {
  static_assert(N <= 32, "reduce-scatter handles <= 32 values");
  double a[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) a[k] = k < N ? v[k] : 0.0;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      const double send = up ? a[k] : a[k + s];
      const double keep = up ? a[k + s] : a[k];
      a[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return a[0];
}

// Multi-value cluster all-reduce of v[0..cnt), in two phases so that callers
// can test a CTA-uniform flag between them.  Phase A: warp reduction into the
// per-warp slots, CTA barrier.  Phase B: every CTA stores its partials into
// every CTA's receive slots over DSMEM (double-buffered by reduction parity),
// one cluster barrier, then fixed rank-order sums.  (Measured on B200: this is
// ~0.3 us cheaper than st.async + mbarrier completion.)  Sums are taken in
// fixed warp and rank order: bitwise identical in every thread.
template <int N>
__device__ __forceinline__ void cl_sum_a(ClCtx& c, double (&v)[N], int cnt) {
  if (cnt <= 6) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i < cnt) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
      }
    }
    if (c.lane == 0) {
#pragma unroll
      for (int i = 0; i < N; ++i)
        if (i < cnt) c.wred[c.warp * N + i] = v[i];
    }
  } else {
    const double o = warp_reduce_scatter<N>(v, c.lane);
    if (c.lane < cnt) c.wred[c.warp * N + c.lane] = o;
  }
  __syncthreads();
}

template <int N>
__device__ __forceinline__ void cl_sum_b(ClCtx& c, double (&v)[N], int cnt) {
  const int p = c.parity;
  double* cred = c.cred + p * (CL_MAXC * N);
  const uint32_t lcred = smem_u32(cred);
  if (c.t < cnt) {  // cnt <= N <= 32 <= blockDim: thread i owns value i
    double s = 0.0;
    for (int w = 0; w < c.nw; ++w) s += c.wred[w * N + c.t];
    const uint32_t src = lcred + 8u * (c.rank * N + c.t);
    for (int r = 0; r < c.C; ++r) st_cluster_f64(cl_map(src, r), s);
  }
  cluster_barrier();  // peers' partials (and any halo stores) now visible
  if (cnt <= 4) {  // every thread sums the few columns itself (no extra barrier)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i < cnt) {
        double s = 0.0;
        for (int r = 0; r < c.C; ++r) s += cred[r * N + i];
        v[i] = s;
      }
    }
  } else {
    if (c.t < cnt) {
      double s = 0.0;
      for (int r = 0; r < c.C; ++r) s += cred[r * N + c.t];
      c.tot[c.t] = s;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (i < cnt) v[i] = c.tot[i];
  }
  c.parity ^= 1;
}

template <int N>
__device__ __forceinline__ void cl_sum(ClCtx& c, double (&v)[N], int cnt) {
  cl_sum_a<N>(c, v, cnt);
  cl_sum_b<N>(c, v, cnt);
}

// SL stencil on the distributed row (taps anywhere on the periodic mesh)
template <int P>
__device__ __forceinline__ void cl_sl_apply(const ClCtx& c, cg::cluster_group& cl, double (&y)[P]) {
  const StepParams& sp = *c.sp;
  const int n = sp.n;
#pragma unroll
  for (int q = 0; q < P; ++q) y[q] = 0.0;
  for (int k = 0; k < sp.ntap; ++k) {
    const int o = sp.tap_off[k];
    const double wk = sp.tap_w[k];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      int e = c.base + c.t * P + q + o;
      e = e >= n ? e - n : e;
      const int owner = e / c.nc;
      const int loc = e - owner * c.nc;
      const double* src = owner == c.rank ? c.in_row : cl.map_shared_rank(c.in_row, owner);
      y[q] = __dadd_rn(y[q], __dmul_rn(wk, src[loc]));
    }
  }
}

// correction stencil (I - phi D) on the halo'd GMRES row, exact mode
template <int P>
__device__ __forceinline__ void cl_corr_apply(const ClCtx& c, double (&y)[P]) {
  const StepParams& sp = *c.sp;
  const int n = sp.n;
#pragma unroll
  for (int q = 0; q < P; ++q) y[q] = 0.0;
  for (int k = 0; k < sp.ntap2; ++k) {
    int o = sp.tap2_off[k];
    o = o > n / 2 ? o - n : o;
    const double wk = sp.tap2_w[k];
#pragma unroll
    for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], __dmul_rn(wk, c.gm[CL_H + c.t * P + q + o]));
  }
}

// own chunk -> own gm slots + neighbours' halo slots (visible after the next
// reduction's cluster barrier)
template <int P>
__device__ __forceinline__ void cl_publish(const ClCtx& c, const double (&w)[P]) {
  const int l0 = c.t * P;
#pragma unroll
  for (int q = 0; q < P; ++q) c.gm[CL_H + l0 + q] = w[q];
  const int lr = c.rank == 0 ? c.C - 1 : c.rank - 1;
  const int rr = c.rank == c.C - 1 ? 0 : c.rank + 1;
#pragma unroll
  for (int q = 0; q < P; ++q) {
    const int l = l0 + q;
    if (l < CL_H)  // my first points -> left neighbour's right halo
      st_cluster_f64(cl_map(smem_u32(c.gm + CL_H + c.nc + l), lr), w[q]);
    if (l >= c.nc - CL_H)  // my last points -> right neighbour's left halo
      st_cluster_f64(cl_map(smem_u32(c.gm + (l - (c.nc - CL_H))), rr), w[q]);
  }
}

// CTA-partial dot products of the CTA slice `vec` with the basis rows Vs[i]
// (i < nv) and, if `with_norm`, of vec with itself (value index nv).  One warp
// per vector: coalesced lane-strided reads over the whole slice, one butterfly,
// lane 0 stores the CTA partial -- no cross-warp stage.  Ends with a CTA barrier.
__device__ __forceinline__ void cl_dots(ClCtx& c, const double* vec, const double* Vs, int nv,
                                        bool with_norm, int wbeg = 0) {
  const int cnt = nv + (with_norm ? 1 : 0);
  for (int i = c.warp - wbeg; i < cnt && c.warp >= wbeg; i += c.nw - wbeg) {
    const double* vi = i < nv ? Vs + (size_t)i * c.nc : vec;
    double s0 = 0.0, s1 = 0.0;
    int l = c.lane;
    for (; l + 32 < c.nc; l += 64) {
      s0 = fma(vec[l], vi[l], s0);
      s1 = fma(vec[l + 32], vi[l + 32], s1);
    }
    if (l < c.nc) s0 = fma(vec[l], vi[l], s0);
    double sv = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
    if (c.lane == 0) c.wred[i] = sv;
  }
  __syncthreads();
}

// Cluster exchange of the CTA partials c.wred[0..cnt): pushed into every CTA's
// receive slots (double-buffered by parity), one cluster barrier, fixed
// rank-order sums into c.tot[0..cnt) (identical in every CTA), CTA barrier.
__device__ __forceinline__ void cl_exchange(ClCtx& c, int cnt, int N) {
  const int p = c.parity;
  double* cred = c.cred + p * (CL_MAXC * N);
  if (c.t < cnt) {
    const double s = c.wred[c.t];
    const uint32_t src = smem_u32(cred) + 8u * (c.rank * N + c.t);
    for (int r = 0; r < c.C; ++r) st_cluster_f64(cl_map(src, r), s);
  }
  cluster_barrier();  // peers' partials (and halo stores) visible
  if (c.t < cnt) {  // pairwise tree over ranks (C is a power of two): depth log2(C)
    double v[CL_MAXC];
#pragma unroll
    for (int r = 0; r < CL_MAXC; ++r) v[r] = r < c.C ? cred[r * N + c.t] : 0.0;
#pragma unroll
    for (int h = CL_MAXC / 2; h >= 1; h >>= 1)
#pragma unroll
      for (int r = 0; r < h; ++r) v[r] += v[r + h];
    c.tot[c.t] = v[0];
  }
  __syncthreads();
  c.parity ^= 1;
}

// Unrestarted GMRES(x0 = 0) on (I - phi D) for the cluster's distributed row
// (semantics of circulant.py:262-332: stop when res <= tol or ||h|| <= 1e-14 beta,
// Givens QR, back substitution, x = V y).  Arnoldi uses CGS2 with TWO cluster
// reductions per step: pass 1 <w, V>, then pass 2 <w1, V> together with
// ||w1||^2 (||w2||^2 = ||w1||^2 - ||h2||^2, explicit re-reduction if that
// cancels) and w1's halo exchange; A v_{j+1} is updated linearly from A w1 and
// Z = A V, so one stencil application per step.  V and Z live in shared memory
// (each CTA its slice); all loops run to j, not to the cap.  Thread 0 keeps the
// Hessenberg column and applies the Givens rotations; its stop flag is read
// after the next CTA barrier.
template <int P, int CAP>
__device__ void cl_gmres(ClCtx& c, double* sm, const double (&b)[P],
                         double (&x)[P], int& depth_out, double& res_out) {
  const StepParams& sp = *c.sp;
  typedef ClLayout<CAP> LY;
  constexpr int N1 = CAP + 1;
  const int cap = sp.cap, nc = c.nc;
  const int l0 = c.t * P;
  double* hcol = sm + LY::hcol(nc);
  double* Rm = sm + LY::Rm(nc);
  double* cs = sm + LY::cs(nc);
  double* sn = sm + LY::sn(nc);
  double* gg = sm + LY::gg(nc);
  double* ybuf = sm + LY::ybuf(nc);
  double* bc = sm + LY::bc(nc);
  double* Zs = sm + LY::Z(nc);   // Z_i = A v_i
  double* Vs = sm + LY::V(nc);   // v_i
  double* wv = c.gm + CL_H;      // the slice being orthogonalised (halo'd row)
  CL_TR_INIT

  cl_publish<P>(c, b);
  __syncthreads();
  cl_dots(c, wv, Vs, 0, true);
  cl_exchange(c, 1, N1);  // its barrier also publishes b's halos
  const double beta = sqrt(c.tot[0]);
  CL_TR(0)
  if (beta == 0.0) {  // zero right-hand side (circulant.py:274-278)
#pragma unroll
    for (int q = 0; q < P; ++q) x[q] = 0.0;
    depth_out = 0;
    res_out = 0.0;
    return;
  }
  const double ib = 1.0 / beta;
  {
    double z[P];
    cl_corr_apply<P>(c, z);
#pragma unroll
    for (int q = 0; q < P; ++q) {
      Vs[l0 + q] = b[q] * ib;
      Zs[l0 + q] = z[q] * ib;
    }
  }
  if (c.t == 0) {
    gg[0] = beta;
    bc[0] = 1.0;
    bc[1] = 0.0;
  }
  int depth = 0;
  double hn_prev = 0.0;
  bool happy_prev = false;
  for (int j = 0;; ++j) {
    double w[P];
    if (j < cap) {
#pragma unroll
      for (int q = 0; q < P; ++q) {
        w[q] = Zs[(size_t)j * nc + l0 + q];  // A v_j
        wv[l0 + q] = w[q];
      }
    }
    __syncthreads();  // w, V_j, Z_j visible
    if (c.warp == 0) {
      if (c.t == 0 && j > 0) {  // Givens on column j-1 (h = h1 + h2), overlapped with the dots
        const int jc = j - 1;
        const double hn = hn_prev;
        double hi = hcol[0] + c.tot[0];
#pragma unroll 4
        for (int i = 0; i < jc; ++i) {
          const double ci = cs[i], si = sn[i], hi1 = hcol[i + 1] + c.tot[i + 1];
          Rm[jc * CAP + i] = __dadd_rn(__dmul_rn(ci, hi), __dmul_rn(si, hi1));
          hi = __dadd_rn(__dmul_rn(-si, hi), __dmul_rn(ci, hi1));
        }
        double den = hypot(hi, hn);
        den = den > 0.0 ? den : 1.0;
        const double rd = 1.0 / den;
        const double cj = hi * rd, sj = hn * rd;
        cs[jc] = cj;
        sn[jc] = sj;
        Rm[jc * CAP + jc] = __dadd_rn(__dmul_rn(cj, hi), __dmul_rn(sj, hn));
        const double gj = gg[jc];
        gg[jc + 1] = __dmul_rn(-sj, gj);
        gg[jc] = __dmul_rn(cj, gj);
        const double r = fabs(gg[jc + 1]) / beta;
        bc[0] = r;
        bc[1] = (!(r > sp.tol) || happy_prev) ? 1.0 : 0.0;
      }
      if (c.nw == 1 && j < cap) {
        cl_dots(c, wv, Vs, j + 1, false, 0);  // single warp: no spare warps to overlap with
      } else {
        __syncthreads();  // the dot warps' barrier (cl_dots ends with one)
      }
    } else {
      if (j < cap) {
        cl_dots(c, wv, Vs, j + 1, false, 1);
      } else {
        __syncthreads();
      }
    }
    CL_TR(1)
    depth = j;
    if (j == cap || bc[1] != 0.0) break;  // uniform
    cl_exchange(c, j + 1, N1);
    CL_TR(2)
    if (c.t <= j) hcol[c.t] = c.tot[c.t];  // h1 (thread i owns entry i)
    for (int i = 0; i <= j; ++i) {
      const double h = c.tot[i];
#pragma unroll
      for (int q = 0; q < P; ++q) w[q] = fma(-h, Vs[(size_t)i * nc + l0 + q], w[q]);
    }
    cl_publish<P>(c, w);  // w1 into the halo'd row + neighbours' halos
    __syncthreads();
    CL_TR(3)
    cl_dots(c, wv, Vs, j + 1, true);
    cl_exchange(c, j + 2, N1);  // barrier also publishes w1's halos
    CL_TR(4)
    double aw[P];
    cl_corr_apply<P>(c, aw);  // A w1
    double hh0 = 0.0, hh1 = 0.0;
    for (int i = 0; i <= j; ++i) {
      const double h = c.tot[i];
      if (i & 1) hh1 = fma(h, h, hh1); else hh0 = fma(h, h, hh0);
#pragma unroll
      for (int q = 0; q < P; ++q) {
        w[q] = fma(-h, Vs[(size_t)i * nc + l0 + q], w[q]);
        aw[q] = fma(-h, Zs[(size_t)i * nc + l0 + q], aw[q]);
      }
    }
    const double s1 = c.tot[j + 1];
    double hn2 = s1 - (hh0 + hh1);
    if (!(hn2 >= 1e-6 * s1)) {  // cancellation: explicit ||w2||^2 (uniform branch)
      __syncthreads();
#pragma unroll
      for (int q = 0; q < P; ++q) wv[l0 + q] = w[q];
      __syncthreads();
      double hsave = c.t <= j ? c.tot[c.t] : 0.0;  // keep h2 for the Givens
      cl_dots(c, wv, Vs, 0, true);
      cl_exchange(c, 1, N1);
      hn2 = c.tot[0];
      __syncthreads();
      if (c.t <= j) c.tot[c.t] = hsave;
      __syncthreads();
    }
    const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
    CL_TR(5)
    happy_prev = hn <= 1e-14 * beta;
    hn_prev = hn;
    const double inv = 1.0 / (hn > 0.0 ? hn : 1.0);
    if (j + 1 < N1) {
#pragma unroll
      for (int q = 0; q < P; ++q) {
        Vs[(size_t)(j + 1) * nc + l0 + q] = w[q] * inv;
        Zs[(size_t)(j + 1) * nc + l0 + q] = aw[q] * inv;
      }
    }
    CL_TR(6)
#ifdef MGB_CL_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&g_cl_trace[15], 1ull);
#endif
  }
  __syncthreads();
  const double res = depth > 0 ? bc[0] : 1.0;
  if (c.warp == 0) {  // back substitution R y = g, column oriented, lanes own rows
    double y = c.lane < depth ? gg[c.lane] : 0.0;
    for (int jj = depth - 1; jj >= 0; --jj) {
      double yj = __shfl_sync(0xffffffffu, y, jj);
      if (yj != 0.0) yj /= Rm[jj * CAP + jj];
      if (c.lane == jj) y = yj;
      if (c.lane < jj) y = fma(-yj, Rm[jj * CAP + c.lane], y);
    }
    if (c.lane < depth) ybuf[c.lane] = y;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < P; ++q) x[q] = 0.0;
  for (int i = 0; i < depth; ++i) {
    const double yi = ybuf[i];
#pragma unroll
    for (int q = 0; q < P; ++q) x[q] = fma(yi, Vs[(size_t)i * nc + l0 + q], x[q]);
  }
  CL_TR(7)
  depth_out = depth;
  res_out = res;
}

template <int P>
__device__ __forceinline__ void cl_load(const double* __restrict__ src, const ClCtx& c, double (&x)[P]) {
  load_chunk<P>(src + c.base, c.t, x);
}

template <int P>
__device__ __forceinline__ void cl_store(double* dst, const ClCtx& c, const double (&x)[P]) {
  store_chunk<P>(dst + c.base, c.t, x);
}

// Interval relaxation with SL + GMRES steps, one cluster per interval.
// Same argument semantics as relax_kernel (mgb_relax_args).
template <int P, int CAP>
__global__ void __launch_bounds__(256) relax_cluster_kernel(const StepParams* __restrict__ gp,
                                                            const RelaxLaunch L) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  {
    const int4* src = reinterpret_cast<const int4*>(gp);
    int4* dst = reinterpret_cast<int4*>(smem_raw);
    for (int i = threadIdx.x; i < (int)(sizeof(StepParams) / 16); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const StepParams& sp = *reinterpret_cast<const StepParams*>(smem_raw);
  const mgb_relax_args& a = L.a;
  typedef ClLayout<CAP> LY;
  double* sm = reinterpret_cast<double*>(smem_raw + sizeof(StepParams));
  ClCtx c;
  c.sp = &sp;
  c.C = (int)cl.num_blocks();
  c.rank = (int)cl.block_rank();
  c.nc = sp.n / c.C;
  c.T = c.nc / P;
  c.t = threadIdx.x;
  c.lane = c.t & 31;
  c.warp = c.t >> 5;
  c.nw = blockDim.x >> 5;
  c.base = c.rank * c.nc;
  c.in_row = sm + LY::in_row(c.nc);
  c.gm = sm + LY::gm(c.nc);
  c.wred = sm + LY::wred(c.nc);
  c.cred = sm + LY::cred(c.nc);
  c.tot = sm + LY::tot(c.nc);
  c.parity = 0;
  const int n = sp.n, t = c.t;
  const long long cluster_id = blockIdx.x / c.C;
  const long long n_clusters = gridDim.x / c.C;

  for (long long k = cluster_id; k < a.n_intervals; k += n_clusters) {
    const long long kg = a.k_global0 + k;
    const long long rowbase = k * (long long)a.m;
    double y[P];
    const double* csrc = (kg == 0 && a.c_src0) ? a.c_src0 : (a.c_src ? a.c_src + k * a.c_stride : nullptr);
    if (csrc) {
      cl_load<P>(csrc, c, y);
    } else {
#pragma unroll
      for (int q = 0; q < P; ++q) y[q] = 0.0;
    }
    if (a.e && kg >= 1) {
      double ev[P];
      cl_load<P>(a.e + k * a.e_stride, c, ev);
#pragma unroll
      for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], ev[q]);
    }
    if (a.c_out) cl_store<P>(a.c_out + k * a.c_out_stride, c, y);
    cluster_barrier();  // previous interval's remote readers of in_row are done
#pragma unroll
    for (int q = 0; q < P; ++q) c.in_row[t * P + q] = y[q];
    cluster_barrier();
    int depth = 0;
    double gres = 0.0;
    const int nsteps = a.n_fsteps + (a.tail ? 1 : 0);
    for (int j = 1; j <= nsteps; ++j) {
      const bool is_tail = j > a.n_fsteps;
      double b[P];
      CL_TR_INIT
      cl_sl_apply<P>(c, cl, b);
      CL_TR(8)
      cl_gmres<P, CAP>(c, sm, b, y, depth, gres);
      CL_TR(14)
      const long long grow = is_tail ? rowbase + a.m : rowbase + j;
      if (!is_tail) {
        if (a.g) {
          double gv[P];
          cl_load<P>(a.g + grow * n, c, gv);
#pragma unroll
          for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], gv[q]);
        }
        // every CTA passed its SL reads (before the beta barrier): safe to overwrite
#pragma unroll
        for (int q = 0; q < P; ++q) c.in_row[t * P + q] = y[q];
        if (a.write_f == 2 || (a.write_f == 1 && j == a.n_fsteps)) cl_store<P>(a.u + grow * n, c, y);
        cluster_barrier();  // the next SL step reads peers' rows
        CL_TR(9)
      } else if (a.tail == 1) {
        if (a.g) {
          double gv[P];
          cl_load<P>(a.g + grow * n, c, gv);
#pragma unroll
          for (int q = 0; q < P; ++q) y[q] = __dadd_rn(y[q], gv[q]);
        }
        cl_store<P>(a.tail_out + k * a.tail_stride, c, y);
      } else {
        double r[P];
        if (a.g) {
          double gv[P];
          cl_load<P>(a.g + grow * n, c, gv);
#pragma unroll
          for (int q = 0; q < P; ++q) r[q] = __dadd_rn(gv[q], y[q]);
        } else {
#pragma unroll
          for (int q = 0; q < P; ++q) r[q] = y[q];
        }
        double cr[P];
        cl_load<P>(a.cref + k * a.cref_stride, c, cr);
        if (a.cref_e) {
          double ev[P];
          cl_load<P>(a.cref_e + k * a.cref_e_stride, c, ev);
#pragma unroll
          for (int q = 0; q < P; ++q) cr[q] = __dadd_rn(cr[q], ev[q]);
        }
        double part[1] = {0.0};
#pragma unroll
        for (int q = 0; q < P; ++q) {
          r[q] = __dsub_rn(r[q], cr[q]);
          part[0] = fma(r[q], r[q], part[0]);
        }
        if (a.tail_out) cl_store<P>(a.tail_out + k * a.tail_stride, c, r);
        if (a.partials) {
          cl_sum<1>(c, part, 1);
          if (t == 0 && c.rank == 0) a.partials[k] = part[0];
        }
      }
    }
    if (a.c_last_out && k == a.n_intervals - 1) {
      double cvl[P];
      if (a.c_src) {
        cl_load<P>(a.c_src + (k + 1) * a.c_stride, c, cvl);
      } else {
#pragma unroll
        for (int q = 0; q < P; ++q) cvl[q] = 0.0;
      }
      if (a.e) {
        double ev[P];
        cl_load<P>(a.e + (k + 1) * a.e_stride, c, ev);
#pragma unroll
        for (int q = 0; q < P; ++q) cvl[q] = __dadd_rn(cvl[q], ev[q]);
      }
      cl_store<P>(a.c_last_out, c, cvl);
    }
    if (t == 0 && c.rank == 0) {
      if (a.stats_depth) a.stats_depth[k] = depth;
      if (a.stats_res) a.stats_res[k] = gres;
    }
  }
  cluster_barrier();  // no CTA may exit while others still read its shared memory
}

}  // namespace mgb
