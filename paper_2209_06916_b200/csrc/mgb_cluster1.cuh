// mgb_cluster1.cuh -- one-reduction cluster GMRES for the semi-Lagrangian +
// corrected coarse steps (sm_100a).
//
// Same semantics as circulant.py:262-332 (unrestarted GMRES(x0 = 0), stop when
// the Givens residual estimate <= tol or on happy breakdown, back substitution,
// x = V y), restructured so that every Arnoldi step costs ONE cluster
// all-reduce (delayed classical Gram-Schmidt with re-orthogonalisation, DCGS2):
//
//   reduction R_j carries, for the not yet re-orthogonalised candidate u_j,
//     a = V^T u_j, nu = u_j.u_j, b = V^T A u_j, c = u_j.A u_j      (2j+2 values)
//   then, locally and identically in every warp of every CTA:
//     column j-1 of H  = h1 + a,  H[j,j-1] = hn = sqrt(nu - |a|^2)
//     v_j = (u_j - V a) / hn                                  (re-orthogonalised)
//     h1' = V^T A v_j = (b - M a) / hn,  M = V^T A V = H[:j,:j] (Arnoldi relation)
//     h1'_j = v_j.A v_j = (c - 2 a.b + a.M a) / hn^2          (A symmetric)
//     u_{j+1} = A v_j - [V v_j] h1'                            (first CGS pass)
//   and the partial dots of u_{j+1} for R_{j+1}.
// This is CGS2 with the second pass delayed by one step (Swirydowicz et al.,
// "Low synchronization Gram-Schmidt and GMRES algorithms"); it agrees with the
// reference's MGS to rounding, like the two-reduction CGS2 kernel it replaces
// (mgb_cluster.cuh).  A Pythagorean norm that cancels (nu - |a|^2 < nu/2) is
// recomputed explicitly with one extra reduction.
//
// Layout: C CTAs own contiguous slices of nc = n/C points; inside a CTA each of
// NW vector warps owns a contiguous segment of S = 32*SEGK points and an extra
// (scalar) warp runs the Givens QR of column j-1 while the vector warps build
// step j -- the stop decision is read after the step's CTA barrier, so Givens
// is off the critical path.  Basis vectors are stored in shared memory with a
// halo of 3r points (r = reach of the (I - phi D) stencil); a warp recomputes
// v_j on its segment +-3r, A v_j on +-2r, u_{j+1} on +-r and A u_{j+1} on the
// segment from warp-private scratch, so no CTA barrier is needed between the
// stencil applications, and only u_{j+1}'s 3r boundary points travel to the
// neighbouring CTAs (DSMEM stores made visible by the step's cluster barrier).
#pragma once
#include <cooperative_groups.h>

#include "mgb_cluster.cuh"

namespace mgb {

constexpr int C1_MAXR = 3;     // reach of the correction stencil (p <= 5)
constexpr int C1_MAXNW = 16;   // vector warps per CTA
constexpr int C1_SLOTS = 24;   // reduction slots per rank (CAP + 3 <= 24)
constexpr int C1_MAXSL = 16;   // SL taps

struct C1Params {
  int n, nc, C, NW, S, r, HW, LD, ntap, cap, K, pad0_;
  double tol;
  int tap_off[C1_MAXSL];
  double tap_w[C1_MAXSL];
  double w2[2 * C1_MAXR + 1];
};
static_assert(sizeof(C1Params) % 16 == 0, "C1Params must be 16-byte sized");

// row stride = 2 (mod 4) doubles: the transposed dot products (lane i reads row i
// with 16-byte loads) are bank-conflict free
__host__ __device__ inline int c1_ld(int nc, int r) {
  int ld = nc + 6 * r + 1;
  while (ld % 4 != 2) ++ld;
  return ld;
}
// scratch row of a warp: the extended segment + a one-double shift so that the
// own points (offset 3r) start 16-byte aligned
__host__ __device__ inline int c1_xs(int S, int r) { return (S + 6 * r + 4) & ~1; }

// shared-memory layout (doubles, after the C1Params block).  The step input row
// of the SL stencil aliases U[1]'s own points: it is read by peers only before
// the first GMRES reduction, and U[1] is first written after it.
struct C1Layout {
  int V, U, in_row, scr, cred, wred, Hm, R, cs, sn, gg, ybuf, hc, flg, total;
  __host__ __device__ C1Layout(int nc, int NW, int S, int r, int C, int CAP, int K) {
    const int LD = c1_ld(nc, r);
    const int XS = c1_xs(S, r);
    int o = 0;
    V = o;      o += (K < CAP ? K : CAP) * LD + 2;  // + shift: rows' own points 16-byte aligned
    U = o;      o += 2 * LD;
    in_row = U + LD + 3 * r;
    o = (o + 1) & ~1;
    scr = o;    o += NW * 2 * XS + 2;
    o = (o + 1) & ~1;
    cred = o;   o += 2 * C * C1_SLOTS;
    wred = o;   o += NW * C1_SLOTS;
    Hm = o;  // (unused)
    R = o;      o += CAP * CAP;
    cs = o;     o += CAP;
    sn = o;     o += CAP;
    gg = o;     o += CAP + 1;
    ybuf = o;   o += CAP;
    o = (o + 1) & ~1;
    hc = o;     o += CAP + 2 + 2 * CAP + 4 + 2;
    flg = o;    o += 4 + 16 + 2;  // stop, res, -, -, rank partials[16], mbarriers[2]
    total = o;
  }
};

// K = basis vectors resident in shared memory; V_K .. V_{CAP-1} live in the
// CTA's L2-resident workspace slot (same halo'd row layout)
__host__ __device__ inline size_t c1_smem_bytes(int nc, int NW, int S, int r, int C, int CAP, int K) {
  return sizeof(C1Params) + 8 * (size_t)C1Layout(nc, NW, S, r, C, CAP, K).total;
}

// fixed-order warp sums, broadcast from lane 0 (bitwise identical in every lane)
__device__ __forceinline__ double c1_wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}
__device__ __forceinline__ void c1_wsum2(double& a, double& b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  a = __shfl_sync(0xffffffffu, a, 0);
  b = __shfl_sync(0xffffffffu, b, 0);
}

// fixed-order pairwise tree over up to 16 values (zeros beyond cnt)
template <int N>
__device__ __forceinline__ double c1_tree(double (&v)[N]) {
#pragma unroll
  for (int h = N / 2; h >= 1; h >>= 1)
#pragma unroll
    for (int i = 0; i < h; ++i) v[i] += v[i + h];
  return v[0];
}

struct C1Ctx {
  const C1Params* p;
  double *V, *Vg, *U, *in_row, *vx, *zx, *cred, *wred, *Hm, *R, *cs, *sn, *gg, *ybuf, *hc, *flg;
  int K;  // basis rows resident in shared memory
  uint64_t* bar;  // bar[q]: transaction barrier of receive buffer q
  int lane, warp, NW, C, rank, S, seg, r, HW, LD, nc, n, base, q, ph;
  bool vec;
};

// st.async: 8-byte store into a peer CTA's shared memory that completes `bytes`
// on the peer's mbarrier (no release fence on the sender)
__device__ __forceinline__ void c1_st_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               ::"r"(raddr), "l"(__double_as_longlong(v)), "r"(rbar) : "memory");
}
__device__ __forceinline__ void c1_mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(a), "r"(parity) : "memory");
  }
}

// (I - phi D) on warp scratch: out at x from src[x - R .. x + R], exact mode
template <int R>
__device__ __forceinline__ double c1_A(const double (&w)[2 * R + 1], const double* src, int x) {
  double s = 0.0;
#pragma unroll
  for (int d = 0; d <= 2 * R; ++d) s = __dadd_rn(s, __dmul_rn(w[d], src[x - R + d]));
  return s;
}

// halo'd basis row i: shared memory for i < K, else the CTA's workspace slot
// (OVF = false: every row is resident, plain shared-memory addressing)
template <bool OVF>
__device__ __forceinline__ double* c1_row(const C1Ctx& c, int i) {
  if constexpr (!OVF) return c.V + (size_t)i * c.LD + c.HW;
  return (i < c.K ? c.V + (size_t)i * c.LD : c.Vg + (size_t)(i - c.K) * c.LD) + c.HW;
}

// Cluster all-reduce step: the CTA totals of wred slots [0, cnt) go to every
// rank's receive buffer q by st.async, each completing its bytes on that rank's
// bar[q]; every thread then waits for bar[q]'s phase (C ranks' values plus
// `extra` bytes of halo points pushed to this CTA during the step).  No cluster
// barrier: buffer q is rewritten only two reductions later, which needs this
// CTA's next values.
template <int NWMAX>
__device__ __forceinline__ void c1_exchange(C1Ctx& c, int cnt, int extra) {
  const int tid = threadIdx.x;
  if (tid < cnt) {
    double v[NWMAX];
#pragma unroll
    for (int w = 0; w < NWMAX; ++w) v[w] = w < c.NW ? c.wred[w * C1_SLOTS + tid] : 0.0;
    const double s = c1_tree<NWMAX>(v);
    const uint32_t src = smem_u32(c.cred + (size_t)c.q * c.C * C1_SLOTS + c.rank * C1_SLOTS + tid);
    const uint32_t bsrc = smem_u32(c.bar + c.q);
#pragma unroll
    for (int rr = 0; rr < CL_MAXC; ++rr)
      if (rr < c.C) c1_st_async(cl_map(src, rr), s, cl_map(bsrc, rr));
  }
  if (tid == 0) {
    const uint32_t bytes = (uint32_t)(8 * c.C * cnt + extra);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(c.bar + c.q)),
                 "r"(bytes) : "memory");
  }
  c1_mbar_wait(c.bar + c.q, (uint32_t)((c.ph >> c.q) & 1));
  c.ph ^= 1 << c.q;
}

// fixed rank-order (pairwise tree) total of slot s of the reduction in buffer q
__device__ __forceinline__ double c1_total(const C1Ctx& c, int q, int s) {
  const double* b = c.cred + (size_t)q * c.C * C1_SLOTS + s;
  double v[CL_MAXC];
#pragma unroll
  for (int rr = 0; rr < CL_MAXC; ++rr) v[rr] = rr < c.C ? b[rr * C1_SLOTS] : 0.0;
  return c1_tree<CL_MAXC>(v);
}

// SL stencil at local point e (may lie in the halo) from the cluster's rows
__device__ __forceinline__ double c1_sl(const C1Ctx& c, cg::cluster_group& cl, int e) {
  const C1Params& P = *c.p;
  int gi = c.base + e;
  gi = gi < 0 ? gi + c.n : (gi >= c.n ? gi - c.n : gi);
  double s = 0.0;
  for (int k = 0; k < P.ntap; ++k) {
    int src = gi + P.tap_off[k];
    src = src >= c.n ? src - c.n : src;
    const int owner = src / c.nc;
    const int loc = src - owner * c.nc;
    const double* row = owner == c.rank ? c.in_row : cl.map_shared_rank(c.in_row, owner);
    s = __dadd_rn(s, __dmul_rn(P.tap_w[k], row[loc]));
  }
  return s;
}

// Transposed partial dots of this warp's segment for reduction R_{j+1}: lane
// i <= j: V_i.u, lane j+1: u.u, lane j+2: u.Au (u = vx[3r..], Au = zx[3r..]).
// No shuffles; 16-byte loads of rows whose stride is 2 (mod 4) doubles
// (conflict-free), u broadcast.
template <bool OVF>
__device__ __forceinline__ void c1_dots(C1Ctx& c, int j) {
  const int lane = c.lane, S = c.S, off = 3 * c.r;
  if (lane <= j + 2) {
    const double* uu = c.vx + off;
    const double* vr = lane <= j ? c1_row<OVF>(c, lane) + c.seg : (lane == j + 1 ? uu : c.zx + off);
    const double2* v2 = reinterpret_cast<const double2*>(vr);
    const double2* u2 = reinterpret_cast<const double2*>(uu);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int e = 0; e < S / 2; e += 2) {
      const double2 x0 = v2[e], x1 = v2[e + 1], y0 = u2[e], y1 = u2[e + 1];
      a0 = fma(x0.x, y0.x, a0);
      a1 = fma(x0.y, y0.y, a1);
      a2 = fma(x1.x, y1.x, a2);
      a3 = fma(x1.y, y1.y, a3);
    }
    c.wred[c.warp * C1_SLOTS + lane] = (a0 + a1) + (a2 + a3);
  }
}

// Wide segments (SEGK >= 4): lane-parallel products over the lane's own points,
// then fixed-order warp butterflies, four rows interleaved.  Rows as c1_dots.
template <int SEGK, bool OVF>
__device__ __forceinline__ void c1_dots_lanes(C1Ctx& c, int j) {
  const int lane = c.lane, off = 3 * c.r;
  double uo[SEGK], ao[SEGK];
#pragma unroll
  for (int k = 0; k < SEGK; ++k) {
    uo[k] = c.vx[off + lane + 32 * k];
    ao[k] = c.zx[off + lane + 32 * k];
  }
  for (int i0 = 0; i0 <= j + 2; i0 += 4) {
    double p[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int i = i0 + ii;
      double s = 0.0;
      if (i <= j) {
        const double* vr = c1_row<OVF>(c, i) + c.seg + lane;
#pragma unroll
        for (int k = 0; k < SEGK; ++k) s = fma(vr[32 * k], uo[k], s);
      } else if (i == j + 1) {
#pragma unroll
        for (int k = 0; k < SEGK; ++k) s = fma(uo[k], uo[k], s);
      } else if (i == j + 2) {
#pragma unroll
        for (int k = 0; k < SEGK; ++k) s = fma(ao[k], uo[k], s);
      }
      p[ii] = s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) p[ii] += __shfl_xor_sync(0xffffffffu, p[ii], o);
    if (lane == 0) {
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
        if (i0 + ii <= j + 2) c.wred[c.warp * C1_SLOTS + i0 + ii] = p[ii];
    }
  }
}

// One corrected SL coarse step: b = SL(in_row) then x = GMRES(I - phi D, b) on
// this CTA's own points (x[k] = point seg + lane + 32 k of the vector warps).
//
// Arnoldi with one reduction per step.  Reduction R_j carries, for the
// candidate u_j (first Gram-Schmidt pass done, second pending):
//   a = V_{<j}^T u_j,  nu = u_j.u_j,  c = u_j.A u_j                 (j + 2 values)
// Step j then forms (scalar warp, broadcast through shared memory):
//   hn = sqrt(nu - |a|^2) = H[j][j-1];   column j-1 of H = h1 + a  (second pass)
//   v_j = (u_j - V a) / hn                                          (re-orthogonalised)
// and the first pass of the next column.  A = I - phi D is symmetric, so the
// Arnoldi relation A V = V H gives V^T A v_j = hn e_{j-1} (three-term, Lanczos)
// and v_j.A v_j = c / hn^2 - 2 a_{j-1} (up to O(eps^2)):
//   h1' = hn e_{j-1} + hj e_j,   u_{j+1} = A v_j - hn v_{j-1} - hj v_j.
// Whatever the first pass leaves in span(V) is O(eps) and is removed by the
// full second pass one step later, so H and the basis agree with the
// reference's MGS GMRES (circulant.py:262-332) to rounding.
template <int SEGK, int CAP, int R, int NWMAX, bool OVF>
__device__ void c1_step(C1Ctx& c, cg::cluster_group& cl, double (&x)[SEGK], int& depth_out,
                        double& res_out) {
  const C1Params& P = *c.p;
  constexpr int KX = SEGK + 1;  // lane iterations over a segment +- 3r (6r <= 18 < 32)
  constexpr int r = R;
  static_assert(CAP + 3 <= C1_SLOTS, "reduction slots");
  const int LD = c.LD, S = c.S, lane = c.lane;
  double w2[2 * R + 1];
#pragma unroll
  for (int d = 0; d <= 2 * R; ++d) w2[d] = P.w2[d];
  const int XE = S + 6 * r;     // extended segment length
  const int e0 = c.seg - 3 * r; // local index of scratch x = 0
  const bool left_b = c.warp == 0, right_b = c.warp == c.NW - 1;
  auto writes_v = [&](int e) {
    return (e >= c.seg && e < c.seg + S) || (left_b && e < 0) || (right_b && e >= c.nc);
  };
  int pu = 0;  // U buffer holding u_j
  CL_TR_INIT

  // ---- right-hand side b = SL(in_row) on the segment +- 3r, ||b||^2, b.Ab
  if (c.vec) {
    double* Uh = c.U + pu * LD + c.HW;
#pragma unroll
    for (int k = 0; k < KX; ++k) {
      const int xx = lane + 32 * k;
      if (xx < XE) {
        const int e = e0 + xx;
        const double b = c1_sl(c, cl, e);
        c.vx[xx] = b;
        if (writes_v(e)) Uh[e] = b;
      }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < SEGK; ++k) {
      const int xx = 3 * r + lane + 32 * k;
      c.zx[xx] = c1_A<R>(w2, c.vx, xx);
    }
    __syncwarp();
    if constexpr (SEGK >= 4) c1_dots_lanes<SEGK, OVF>(c, -1); else c1_dots<OVF>(c, -1);  // rows: b.b, b.Ab
  }
  CL_TR(8)
  __syncthreads();
  c1_exchange<NWMAX>(c, 2, 0);  // also: every CTA finished its SL reads of in_row
  CL_TR(9)

  // scalar warp state: lane i holds h1_i (first-pass coefficient of the pending column)
  double h1 = 0.0;
  double beta = 0.0, ibeta = 0.0;
  double* coef = c.hc + CAP + 2;  // [i] = a_i (i < j); [CAP..]: inv, hj, hn, flags
  int j = 0;
  for (;; ++j) {
    // ---- step j.  Scalar warp: a_i -> smem, named barrier 1 (arrive only); then
    // |a|^2, hn, 1/hn, hj -> smem, named barrier 2.  Vector warps run the
    // re-orthogonalisation pass u_j - V a between the two barriers.
    double ai = 0.0, hn = 0.0, nu = 0.0;
    const uint32_t nthr = blockDim.x;
    CL_TRS_INIT
    if (!c.vec) {
      const double tot = lane <= j + 1 ? c1_total(c, c.q, lane) : 0.0;
      ai = lane < j ? tot : 0.0;
      if (lane < j) coef[lane] = ai;
      __threadfence_block();
      asm volatile("bar.arrive 1, %0;" ::"r"(nthr) : "memory");
      CL_TRS(10)
      nu = __shfl_sync(0xffffffffu, tot, j);
      const double cc = __shfl_sync(0xffffffffu, tot, (j + 1) & 31);
      const double na2 = c1_wsum(ai * ai);
      const double hn2 = nu - na2;
      hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
      if (j == 0) {
        beta = hn;
        ibeta = beta > 0.0 ? 1.0 / beta : 0.0;
      }
      const double inv = hn > 0.0 ? 1.0 / hn : 1.0;
      const double alast = __shfl_sync(0xffffffffu, ai, (j + 31) & 31);
      if (lane == 0) {
        coef[CAP] = inv;
        coef[CAP + 1] = cc * (inv * inv) - (j > 0 ? 2.0 * alast : 0.0);  // hj = v_j.A v_j
        coef[CAP + 2] = j > 0 ? hn : 0.0;
        coef[CAP + 3] = (j > 0 && !(hn2 >= 0.5 * nu)) ? 1.0 : 0.0;  // cancelling update
        coef[CAP + 4] = beta == 0.0 ? 1.0 : 0.0;                    // zero right-hand side
        coef[CAP + 5] = cc;
      }
      __threadfence_block();
      asm volatile("bar.arrive 2, %0;" ::"r"(nthr) : "memory");
      CL_TRS(11)
    }
    c.q ^= 1;
    const double* Uh = c.U + pu * LD + c.HW;
    double v[KX];  // vector warps: u_j - V a on the segment +- 3r
    if (c.vec) {
      asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
      CL_TR(12)
      if (j < P.cap) {
#pragma unroll
        for (int k = 0; k < KX; ++k) {
          const int xx = lane + 32 * k;
          v[k] = xx < XE ? Uh[e0 + xx] : 0.0;
        }
#pragma unroll
        for (int i0 = 0; i0 < CAP; i0 += 4) {
          if (i0 < j) {
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) {
              const int i = i0 + ii;
              const double a_b = i < j ? coef[i] : 0.0;
              const double* Vi = c1_row<OVF>(c, i < j ? i : 0) + e0;
#pragma unroll
              for (int k = 0; k < KX; ++k) {
                const int xx = lane + 32 * k;
                const double vi = (i < j && xx < XE) ? Vi[xx] : 0.0;
                v[k] = fma(-a_b, vi, v[k]);
              }
            }
          }
        }
      }
      CL_TR(13)
      asm volatile("bar.sync 2, %0;" ::"r"(nthr) : "memory");
    }
    if (coef[CAP + 4] != 0.0) {  // zero right-hand side (circulant.py:274-278), uniform
#pragma unroll
      for (int k = 0; k < SEGK; ++k) x[k] = 0.0;
      depth_out = 0;
      res_out = 0.0;
      return;
    }
    if (coef[CAP + 3] != 0.0) {
      // cancelling Pythagorean update: explicit ||u_j - V a||^2 (uniform branch)
      if (c.vec) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < KX; ++k) {
          const int xx = lane + 32 * k;
          if (xx >= 3 * r && xx < 3 * r + S) s = fma(v[k], v[k], s);
        }
        s = c1_wsum(s);
        if (lane == 0) c.wred[c.warp * C1_SLOTS] = s;
      }
      __syncthreads();
      c1_exchange<NWMAX>(c, 1, 0);
      if (!c.vec) {  // redo the hn-dependent scalars
        const double hn2 = c1_total(c, c.q, 0);
        hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
        const double inv = hn > 0.0 ? 1.0 / hn : 1.0;
        const double alast = __shfl_sync(0xffffffffu, ai, (j + 31) & 31);
        if (lane == 0) {
          coef[CAP] = inv;
          coef[CAP + 1] = coef[CAP + 5] * (inv * inv) - 2.0 * alast;
          coef[CAP + 2] = hn;
        }
      }
      c.q ^= 1;
      __syncthreads();
    }
    CL_TR(0)

    if (!c.vec) {
      // ---- scalar warp: finalise column j-1 (h1 + a, hn) and its Givens rotation
      if (j > 0) {
        const int jc = j - 1;
        if (lane < j) c.hc[lane] = h1 + ai;
        if (lane == 0) c.hc[j] = hn;
        __syncwarp();
        if (lane == 0) {
          double hi = c.hc[0];
          for (int i = 0; i < jc; ++i) {
            const double ci = c.cs[i], si = c.sn[i], hi1 = c.hc[i + 1];
            c.R[jc * CAP + i] = fma(ci, hi, si * hi1);
            hi = fma(-si, hi, ci * hi1);
          }
          double den = sqrt(fma(hi, hi, hn * hn));
          const double rden = den > 0.0 ? 1.0 / den : 1.0;
          const double cj = hi * rden, sj = hn * rden;
          c.cs[jc] = cj;
          c.sn[jc] = sj;
          c.R[jc * CAP + jc] = fma(cj, hi, sj * hn);
          const double gj = c.gg[jc];
          c.gg[jc + 1] = -sj * gj;
          c.gg[jc] = cj * gj;
          const double res = fabs(c.gg[jc + 1]) * ibeta;
          const bool stop = !(res > P.tol) || (hn <= 1e-14 * beta) || j >= P.cap;
          c.flg[0] = stop ? 1.0 : 0.0;
          c.flg[1] = res;
        }
      } else if (lane == 0) {
        c.gg[0] = beta;
        c.flg[0] = 0.0;
        c.flg[1] = 1.0;
      }
      // first-pass coefficients of column j: h1' = hn e_{j-1} + hj e_j
      const double hj = coef[CAP + 1];
      h1 = lane == j ? hj : (lane + 1 == j ? hn : 0.0);
    } else if (j < P.cap) {
      // ---- vector warps: v_j, u_{j+1} = A v_j - hn v_{j-1} - hj v_j, A u_{j+1}, dots
      double* Un = c.U + (pu ^ 1) * LD + c.HW;
      const double inv = coef[CAP];
      double* Vj = c1_row<OVF>(c, j);
#pragma unroll
      for (int k = 0; k < KX; ++k) {
        const int xx = lane + 32 * k;
        if (xx < XE) {
          v[k] *= inv;
          c.vx[xx] = v[k];
          if (writes_v(e0 + xx)) Vj[e0 + xx] = v[k];
        }
      }
      CL_TR(1)
      __syncwarp();
      double u[KX];
      {
        const double hj = coef[CAP + 1], hb = coef[CAP + 2];
        const double* Vp = c1_row<OVF>(c, j > 0 ? j - 1 : 0) + e0;
#pragma unroll
        for (int k = 0; k < KX; ++k) {
          const int xx = lane + 32 * k;
          u[k] = 0.0;
          if (xx >= 2 * r && xx < XE - 2 * r) {
            const double vp = j > 0 ? Vp[xx] : 0.0;
            u[k] = fma(-hj, v[k], fma(-hb, vp, c1_A<R>(w2, c.vx, xx)));
          }
        }
      }
      CL_TR(2)
      __syncwarp();
      {
        const int lr = c.rank == 0 ? c.C - 1 : c.rank - 1;
        const int rr = c.rank == c.C - 1 ? 0 : c.rank + 1;
#pragma unroll
        for (int k = 0; k < KX; ++k) {
          const int xx = lane + 32 * k;
          if (xx >= 2 * r && xx < XE - 2 * r) {
            c.vx[xx] = u[k];
            const int e = e0 + xx;
            if (e >= c.seg && e < c.seg + S) {
              Un[e] = u[k];
              if (left_b && e < 3 * r)  // -> left neighbour's right halo (its bar[q])
                c1_st_async(cl_map(smem_u32(Un + c.nc + e), lr), u[k], cl_map(smem_u32(c.bar + c.q), lr));
              if (right_b && e >= c.nc - 3 * r)  // -> right neighbour's left halo
                c1_st_async(cl_map(smem_u32(Un + (e - c.nc)), rr), u[k], cl_map(smem_u32(c.bar + c.q), rr));
            }
          }
        }
      }
      CL_TR(3)
      __syncwarp();
#pragma unroll
      for (int k = 0; k < SEGK; ++k) {  // A u_{j+1} on the segment
        const int xx = 3 * r + lane + 32 * k;
        c.zx[xx] = c1_A<R>(w2, c.vx, xx);
      }
      __syncwarp();
      if constexpr (SEGK >= 4) c1_dots_lanes<SEGK, OVF>(c, j); else c1_dots<OVF>(c, j);
      CL_TR(4)
    }
    __syncthreads();
    CL_TR(5)
    if (j >= P.cap || c.flg[0] != 0.0) {  // uniform
      if (j < P.cap) {
        // the speculative step pushed u_{j+1}'s halo points to the neighbours' bar[q]:
        // consume that phase so the transaction counts stay aligned
        if (threadIdx.x == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(c.bar + c.q)),
                       "r"((uint32_t)(8 * 6 * r)) : "memory");
        c1_mbar_wait(c.bar + c.q, (uint32_t)((c.ph >> c.q) & 1));
        c.ph ^= 1 << c.q;
        c.q ^= 1;
      }
      break;
    }
    c1_exchange<NWMAX>(c, j + 3, 8 * 6 * r);
    CL_TR(6)
    CL_TR_STEP
    pu ^= 1;
  }
  // ---- back substitution R y = g (scalar warp), x = V y on the own points
  const int depth = j;
  if (!c.vec) {
    double y = lane < depth ? c.gg[lane] : 0.0;
    for (int jj = depth - 1; jj >= 0; --jj) {
      double yj = __shfl_sync(0xffffffffu, y, jj);
      if (yj != 0.0) yj /= c.R[jj * CAP + jj];
      if (lane == jj) y = yj;
      if (lane < jj) y = fma(-yj, c.R[jj * CAP + lane], y);
    }
    if (lane < depth) c.ybuf[lane] = y;
  }
  const double res = c.flg[1];
  __syncthreads();
  if (c.vec) {
#pragma unroll
    for (int k = 0; k < SEGK; ++k) x[k] = 0.0;
    for (int i = 0; i < depth; ++i) {
      const double yi = c.ybuf[i];
#pragma unroll
      for (int k = 0; k < SEGK; ++k) x[k] = fma(yi, c1_row<OVF>(c, i)[c.seg + lane + 32 * k], x[k]);
    }
  }
  CL_TR(7)
  depth_out = depth;
  res_out = res;
}

template <int SEGK>
__device__ __forceinline__ void c1_load(const double* __restrict__ src, const C1Ctx& c, double (&x)[SEGK]) {
#pragma unroll
  for (int k = 0; k < SEGK; ++k) x[k] = __ldg(src + c.base + c.seg + c.lane + 32 * k);
}
template <int SEGK>
__device__ __forceinline__ void c1_store(double* dst, const C1Ctx& c, const double (&x)[SEGK]) {
#pragma unroll
  for (int k = 0; k < SEGK; ++k) dst[c.base + c.seg + c.lane + 32 * k] = x[k];
}

// cluster sum of one per-CTA value into rank 0 (residual partials), fixed order
template <int NWMAX>
__device__ __forceinline__ double c1_sum_to_rank0(C1Ctx& c, double v) {
  if (c.vec) {
    v = c1_wsum(v);
    if (c.lane == 0) c.wred[c.warp * C1_SLOTS] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NWMAX; ++w)
      if (w < c.NW) s += c.wred[w * C1_SLOTS];
    st_cluster_f64(cl_map(smem_u32(c.flg + 4 + c.rank), 0), s);
  }
  cluster_barrier();
  double pr[CL_MAXC];
#pragma unroll
  for (int rr = 0; rr < CL_MAXC; ++rr) pr[rr] = rr < c.C ? c.flg[4 + rr] : 0.0;
  return c1_tree<CL_MAXC>(pr);
}

// Interval relaxation with corrected SL steps, one cluster per interval, same
// argument semantics as relax_kernel / relax_cluster_kernel (mgb_relax_args).
// OVF: basis rows K..CAP-1 may live in the CTA's workspace slot (K < CAP when
// the rows do not all fit the shared-memory budget of the build)
template <int SEGK, int CAP, int R, int NWMAX, int MINB = 1, bool OVF = (SEGK >= 4)>
__global__ void __launch_bounds__(32 * (NWMAX + 1), MINB)
    relax_cl1_kernel(const StepParams* __restrict__ gp, const RelaxLaunch L) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C1Params& P = *reinterpret_cast<C1Params*>(smem_raw);
  const int tid = threadIdx.x;
  const int C = (int)cl.num_blocks();
  const int NW = (int)(blockDim.x >> 5) - 1;
  if (tid == 0) {
    P.n = gp->n;
    P.C = C;
    P.nc = gp->n / C;
    P.NW = NW;
    P.S = P.nc / NW;
    P.r = gp->win2_span / 2;
    P.HW = 3 * P.r;
    P.LD = c1_ld(P.nc, P.r);
    P.ntap = gp->ntap;
    P.cap = gp->cap;
    P.tol = gp->tol;
    P.K = L.ws ? (int)L.ws_slot : CAP;  // ws_slot carries the resident row count
    for (int k = 0; k < gp->ntap && k < C1_MAXSL; ++k) {
      P.tap_off[k] = gp->tap_off[k];
      P.tap_w[k] = gp->tap_w[k];
    }
    for (int d = 0; d <= 2 * P.r; ++d) P.w2[d] = gp->win2_w[d];
  }
  __syncthreads();
  const C1Layout LY(P.nc, NW, P.S, P.r, C, CAP, P.K);
  double* sm = reinterpret_cast<double*>(smem_raw + sizeof(C1Params));
  C1Ctx c;
  c.p = &P;
  c.lane = tid & 31;
  c.warp = tid >> 5;
  c.NW = NW;
  c.C = C;
  c.rank = (int)cl.block_rank();
  c.S = P.S;
  c.seg = c.warp * P.S;
  c.r = P.r;
  c.HW = P.HW;
  c.LD = P.LD;
  c.nc = P.nc;
  c.n = P.n;
  c.base = c.rank * P.nc;
  c.q = 0;
  c.vec = c.warp < NW;
  c.V = sm + LY.V + (P.HW & 1);  // c.V + HW (own point 0 of row 0) is 16-byte aligned
  c.K = P.K;
  // overflow rows share the resident rows' alignment shift (16-byte row loads)
  c.Vg = L.ws ? L.ws + (size_t)blockIdx.x * (size_t)(CAP - P.K) * P.LD + (P.HW & 1) : nullptr;
  c.U = sm + LY.U;
  c.in_row = sm + LY.in_row;
  const int XS = c1_xs(P.S, P.r);
  c.vx = sm + LY.scr + (c.vec ? c.warp : 0) * 2 * XS + ((3 * P.r) & 1);
  c.zx = c.vx + XS;
  c.cred = sm + LY.cred;
  c.wred = sm + LY.wred;
  c.Hm = sm + LY.Hm;
  c.R = sm + LY.R;
  c.cs = sm + LY.cs;
  c.sn = sm + LY.sn;
  c.gg = sm + LY.gg;
  c.ybuf = sm + LY.ybuf;
  c.hc = sm + LY.hc;
  c.flg = sm + LY.flg;
  c.bar = reinterpret_cast<uint64_t*>(c.flg + 20);
  c.ph = 0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(c.bar)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(c.bar + 1)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const mgb_relax_args& a = L.a;
  const int n = P.n;
  const long long cluster_id = blockIdx.x / C;
  const long long n_clusters = gridDim.x / C;
  for (long long k = cluster_id; k < a.n_intervals; k += n_clusters) {
    const long long kg = a.k_global0 + k;
    const long long rowbase = k * (long long)a.m;
    double y[SEGK];
    const double* csrc = (kg == 0 && a.c_src0) ? a.c_src0 : (a.c_src ? a.c_src + k * a.c_stride : nullptr);
    if (c.vec) {
      if (csrc) {
        c1_load<SEGK>(csrc, c, y);
      } else {
#pragma unroll
        for (int q = 0; q < SEGK; ++q) y[q] = 0.0;
      }
      if (a.e && kg >= 1) {
        double ev[SEGK];
        c1_load<SEGK>(a.e + k * a.e_stride, c, ev);
#pragma unroll
        for (int q = 0; q < SEGK; ++q) y[q] = __dadd_rn(y[q], ev[q]);
      }
      if (a.c_out) c1_store<SEGK>(a.c_out + k * a.c_out_stride, c, y);
    }
    cluster_barrier();  // previous interval's remote readers of in_row are done
    if (c.vec) {
#pragma unroll
      for (int q = 0; q < SEGK; ++q) c.in_row[c.seg + c.lane + 32 * q] = y[q];
    }
    cluster_barrier();
    int depth = 0;
    double gres = 0.0;
    const int nsteps = a.n_fsteps + (a.tail ? 1 : 0);
    for (int j = 1; j <= nsteps; ++j) {
      const bool is_tail = j > a.n_fsteps;
      c1_step<SEGK, CAP, R, NWMAX, OVF>(c, cl, y, depth, gres);
      const long long grow = is_tail ? rowbase + a.m : rowbase + j;
      if (!is_tail) {
        if (c.vec) {
          if (a.g) {
            double gv[SEGK];
            c1_load<SEGK>(a.g + grow * n, c, gv);
#pragma unroll
            for (int q = 0; q < SEGK; ++q) y[q] = __dadd_rn(y[q], gv[q]);
          }
          // every CTA finished its SL reads before the first GMRES reduction
#pragma unroll
          for (int q = 0; q < SEGK; ++q) c.in_row[c.seg + c.lane + 32 * q] = y[q];
          if (a.write_f == 2 || (a.write_f == 1 && j == a.n_fsteps)) c1_store<SEGK>(a.u + grow * n, c, y);
        }
        cluster_barrier();  // the next SL step reads peers' rows; GMRES pushes landed
      } else if (a.tail == 1) {
        if (c.vec) {
          if (a.g) {
            double gv[SEGK];
            c1_load<SEGK>(a.g + grow * n, c, gv);
#pragma unroll
            for (int q = 0; q < SEGK; ++q) y[q] = __dadd_rn(y[q], gv[q]);
          }
          c1_store<SEGK>(a.tail_out + k * a.tail_stride, c, y);
        }
      } else {
        double part = 0.0;
        if (c.vec) {
          double rr[SEGK];
          if (a.g) {
            double gv[SEGK];
            c1_load<SEGK>(a.g + grow * n, c, gv);
#pragma unroll
            for (int q = 0; q < SEGK; ++q) rr[q] = __dadd_rn(gv[q], y[q]);
          } else {
#pragma unroll
            for (int q = 0; q < SEGK; ++q) rr[q] = y[q];
          }
          double cr[SEGK];
          c1_load<SEGK>(a.cref + k * a.cref_stride, c, cr);
          if (a.cref_e) {
            double ev[SEGK];
            c1_load<SEGK>(a.cref_e + k * a.cref_e_stride, c, ev);
#pragma unroll
            for (int q = 0; q < SEGK; ++q) cr[q] = __dadd_rn(cr[q], ev[q]);
          }
#pragma unroll
          for (int q = 0; q < SEGK; ++q) {
            rr[q] = __dsub_rn(rr[q], cr[q]);
            part = fma(rr[q], rr[q], part);
          }
          if (a.tail_out) c1_store<SEGK>(a.tail_out + k * a.tail_stride, c, rr);
        }
        if (a.partials) {
          const double tot = c1_sum_to_rank0<NWMAX>(c, part);
          if (tid == 0 && c.rank == 0) a.partials[k] = tot;
        }
      }
    }
    if (a.c_last_out && k == a.n_intervals - 1 && c.vec) {
      double cvl[SEGK];
      if (a.c_src) {
        c1_load<SEGK>(a.c_src + (k + 1) * a.c_stride, c, cvl);
      } else {
#pragma unroll
        for (int q = 0; q < SEGK; ++q) cvl[q] = 0.0;
      }
      if (a.e) {
        double ev[SEGK];
        c1_load<SEGK>(a.e + (k + 1) * a.e_stride, c, ev);
#pragma unroll
        for (int q = 0; q < SEGK; ++q) cvl[q] = __dadd_rn(cvl[q], ev[q]);
      }
      c1_store<SEGK>(a.c_last_out, c, cvl);
    }
    if (tid == 0 && c.rank == 0) {
      if (a.stats_depth) a.stats_depth[k] = depth;
      if (a.stats_res) a.stats_res[k] = gres;
    }
  }
  cluster_barrier();  // no CTA may exit while others still access its shared memory
}

}  // namespace mgb
