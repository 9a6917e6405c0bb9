// mgb_host.cu -- host side of libmgrit_b200.so: device plans for one-step
// operators, spectral factorisation of the implicit circulants, launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "mgb_cluster1.cuh"
#include "mgb_registry.h"

using mgb::Factor;
using mgb::StepParams;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// Launch choices are plan-time parameters with the defaults below.  The MGB_*
// environment variables override them for tooling only (variant sweeps,
// bisection, the chained-interval tests); they are read once per process.
struct Tuning {
  bool debug = false;
  bool no_cluster = false;    // MGB_NO_CLUSTER: single-CTA GMRES on every level
  bool cgs2 = false;          // MGB_CL_CGS2: previous two-reduction cluster kernel
  int c1_c = 0;               // MGB_C1_C: force one cluster size
  bool c1_no_occ2 = false;    // MGB_C1_NO_OCC2: no 2-CTA/SM cluster builds
  bool c1_wide = false;       // MGB_C1_WIDE: allow wide-segment cluster builds
  bool c1_no_split = false;   // MGB_C1_NO_SPLIT: no second launch for a partial last wave
  long long c1_waves = 2;     // MGB_C1_WAVES: cluster waves beyond which the single-CTA kernel runs
  long long cluster_waves = 2;  // MGB_CLUSTER_WAVES: same for the two-reduction kernel
  int c1_segk = 1;            // MGB_C1_SEGK: smallest segment width considered
  bool slg_no_occ2 = false;   // MGB_SLG_NO_OCC2: no 2-CTA/SM single-CTA GMRES build
  bool rk_stencil = false;    // MGB_RK_STENCIL: SDIRK stage values by the stencil in fast mode too
  bool no_rkd = false;        // MGB_NO_RKD: staged SDIRK on the generic kernel
  bool no_sld = false;        // MGB_NO_SLD: SL + direct solve on the generic kernel
  long long max_grid = 0;     // MGB_MAX_GRID: cap the grid (tests: many intervals per CTA)
};
const Tuning& tuning() {
  static const Tuning t = [] {
    Tuning x;
    auto flag = [](const char* k) { return std::getenv(k) != nullptr; };
    auto num = [](const char* k, long long d) { const char* v = std::getenv(k); return v ? std::atoll(v) : d; };
    x.debug = flag("MGB_DEBUG");
    x.no_cluster = flag("MGB_NO_CLUSTER");
    x.cgs2 = flag("MGB_CL_CGS2");
    x.c1_c = (int)num("MGB_C1_C", 0);
    x.c1_no_occ2 = flag("MGB_C1_NO_OCC2");
    x.c1_wide = flag("MGB_C1_WIDE");
    x.c1_no_split = flag("MGB_C1_NO_SPLIT");
    x.c1_waves = num("MGB_C1_WAVES", 2);
    x.cluster_waves = num("MGB_CLUSTER_WAVES", 2);
    x.c1_segk = (int)num("MGB_C1_SEGK", 1);
    x.slg_no_occ2 = flag("MGB_SLG_NO_OCC2");
    x.rk_stencil = flag("MGB_RK_STENCIL");
    x.no_rkd = flag("MGB_NO_RKD");
    x.no_sld = flag("MGB_NO_SLD");
    x.max_grid = num("MGB_MAX_GRID", 0);
    return x;
  }();
  return t;
}

#define CUDA_TRY(expr)                                                           \
  do {                                                                           \
    cudaError_t e_ = (expr);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return fail(MGB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

std::mutex& reg_mutex() {
  static std::mutex m;
  return m;
}
std::map<std::tuple<int, int, int, int, int>, const void*>& registry() {
  static std::map<std::tuple<int, int, int, int, int>, const void*> r;
  return r;
}
// The max-dynamic-shared-memory attribute belongs to the kernel FUNCTION on the
// current device, which several plans (different n_x) share: only ever raise
// it, so a later smaller plan cannot invalidate the launches of an earlier
// larger one.  Tracked per (device, function).
cudaError_t raise_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cur;
  int dev = 0;
  const cudaError_t ed = cudaGetDevice(&dev);
  if (ed != cudaSuccess) return ed;
  std::lock_guard<std::mutex> lk(mu);
  int& have = cur[std::make_pair(dev, fn)];
  if (bytes <= have) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

void ensure_registered() {
  static std::once_flag once;
  std::call_once(once, [] {
    mgb::register_win_exact();
    mgb::register_win_fast();
    mgb::register_gen();
    mgb::register_rk();
    mgb::register_slgc();
    mgb::register_slgc1();
  });
}

// ------------------------------------------------------ long double algebra
using ld = long double;
using cld = std::complex<long double>;

struct M2 {
  ld a, b, c, d;
};
M2 mul(const M2& x, const M2& y) {
  return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c, x.c * y.b + x.d * y.d};
}
M2 mpow(M2 base, long long e) {
  M2 r{1, 0, 0, 1};
  while (e > 0) {
    if (e & 1) r = mul(r, base);
    base = mul(base, base);
    e >>= 1;
  }
  return r;
}
void put(double* dst, const M2& m) {
  dst[0] = (double)m.a;
  dst[1] = (double)m.b;
  dst[2] = (double)m.c;
  dst[3] = (double)m.d;
}

cld peval(const std::vector<cld>& c, cld z) {  // c[k] z^k
  cld acc = 0;
  for (int k = (int)c.size() - 1; k >= 0; --k) acc = acc * z + c[k];
  return acc;
}

// Roots of sum_k c[k] z^k (c.back() != 0): Durand-Kerner + Newton polish.
std::vector<cld> poly_roots(const std::vector<ld>& cr) {
  const int d = (int)cr.size() - 1;
  std::vector<cld> c(d + 1);
  for (int k = 0; k <= d; ++k) c[k] = cld(cr[k] / cr[d], 0);
  ld bound = 0;
  for (int k = 0; k < d; ++k) bound = std::max(bound, std::abs(c[k]));
  bound = 1 + bound;
  std::vector<cld> z(d);
  const cld seed(0.4L, 0.9L);
  cld p = 1;
  for (int i = 0; i < d; ++i) {
    p *= seed;
    z[i] = p * (bound / std::abs(p)) * (ld)(0.5 + 0.5 * (i + 1) / d);
  }
  for (int it = 0; it < 2000; ++it) {
    ld change = 0;
    for (int i = 0; i < d; ++i) {
      cld den = 1;
      for (int j = 0; j < d; ++j)
        if (j != i) den *= (z[i] - z[j]);
      if (std::abs(den) == 0) den = cld(1e-30L, 0);
      cld dz = peval(c, z[i]) / den;
      z[i] -= dz;
      change = std::max(change, std::abs(dz) / std::max((ld)1, std::abs(z[i])));
    }
    if (change < 1e-30L) break;
  }
  // Newton polish
  std::vector<cld> dc(std::max(d, 1));
  for (int k = 1; k <= d; ++k) dc[k - 1] = c[k] * (ld)k;
  for (int i = 0; i < d; ++i) {
    for (int it = 0; it < 8; ++it) {
      cld f = peval(c, z[i]);
      cld fp = peval(dc, z[i]);
      if (std::abs(fp) == 0) break;
      cld dz = f / fp;
      z[i] -= dz;
      if (std::abs(dz) <= 1e-19L * std::max((ld)1, std::abs(z[i]))) break;
    }
  }
  return z;
}

struct FactorDesc {
  ld a1, a2;
  int dir;
  ld rho;  // largest |root| of the factor (decay per point of its recurrence)
};

// Factorise the circulant with stencil (offsets, weights):
//   a(z) = K z^s prod_f F_f(z),  F = (1 - zeta/z)[(1 - conj(zeta)/z)]  (inside roots, forward)
//                              or (1 - z/zeta)[(1 - z/conj(zeta))]  (outside roots, backward)
int factorize(const std::vector<long long>& off, const std::vector<double>& w, int n,
              std::vector<FactorDesc>& facs, ld& K, int& shift) {
  long long lo = off[0], hi = off[0];
  for (auto o : off) {
    lo = std::min(lo, o);
    hi = std::max(hi, o);
  }
  const int d = (int)(hi - lo);
  if (d > 30) return fail(MGB_ERR_UNSUPPORTED, "implicit stencil too wide to factorise");
  std::vector<ld> c(d + 1, 0);
  for (size_t k = 0; k < off.size(); ++k) c[off[k] - lo] += (ld)w[k];
  facs.clear();
  if (d == 0) {
    K = c[0];
    shift = (int)lo;
    if (K == 0) return fail(MGB_ERR_SINGULAR, "zero operator");
    return MGB_OK;
  }
  std::vector<cld> roots = poly_roots(c);
  std::vector<cld> in_r, out_r;
  for (auto& z : roots) {
    const ld m = std::abs(z);
    if (std::fabs(m - 1) < 1e-12L) return fail(MGB_ERR_SINGULAR, "implicit operator singular (root on unit circle)");
    if (std::fabs(z.imag()) <= 1e-14L * m) z = cld(z.real(), 0);
    (m < 1 ? in_r : out_r).push_back(z);
  }
  cld Kc = cld(c[d], 0);
  for (auto& z : out_r) Kc *= -z;
  if (std::fabs(Kc.imag()) > 1e-10L * std::abs(Kc)) return fail(MGB_ERR_INVALID, "non-real gain in factorisation");
  K = Kc.real();
  shift = (int)(lo + (long long)in_r.size());
  auto emit = [&](std::vector<cld>& rs, bool inside) -> int {
    std::vector<bool> used(rs.size(), false);
    ld pending_real = 0;  // real roots of one direction are merged pairwise into
    bool have_pending = false;  // one second-order recurrence (fewer scans)
    for (size_t i = 0; i < rs.size(); ++i) {
      if (used[i]) continue;
      used[i] = true;
      const cld mu = inside ? rs[i] : ((ld)1 / rs[i]);
      if (rs[i].imag() == 0) {
        if (have_pending) {
          const ld r1 = pending_real, r2 = mu.real();
          facs.push_back({r1 + r2, -r1 * r2, inside ? +1 : -1, std::max(std::fabs(r1), std::fabs(r2))});
          have_pending = false;
        } else {
          pending_real = mu.real();
          have_pending = true;
        }
        continue;
      }
      // find conjugate partner
      size_t best = rs.size();
      ld bd = 1e300L;
      for (size_t j = 0; j < rs.size(); ++j) {
        if (used[j]) continue;
        ld dd = std::abs(rs[j] - std::conj(rs[i]));
        if (dd < bd) {
          bd = dd;
          best = j;
        }
      }
      if (best == rs.size() || bd > 1e-8L * std::abs(rs[i]))
        return fail(MGB_ERR_INVALID, "complex root without conjugate partner");
      used[best] = true;
      facs.push_back({2 * mu.real(), -std::norm(mu), inside ? +1 : -1, std::abs(mu)});
    }
    if (have_pending) facs.push_back({pending_real, 0, inside ? +1 : -1, std::fabs(pending_real)});
    return MGB_OK;
  };
  int rc = emit(in_r, true);
  if (rc) return rc;
  rc = emit(out_r, false);
  if (rc) return rc;
  // verify: symbol of the factorisation equals the stencil symbol
  for (int kk = 0; kk < 7; ++kk) {
    const ld om = 2 * 3.14159265358979323846264338327950288L * kk / 7.0L + 0.1L;
    const cld z = std::polar((ld)1, om);
    cld direct = 0;
    for (size_t k = 0; k < off.size(); ++k) direct += (ld)w[k] * std::pow(z, (int)off[k]);
    cld fact = K * std::pow(z, shift);
    for (auto& f : facs) {
      if (f.dir > 0)
        fact *= (ld)1 - f.a1 / z - f.a2 / (z * z);
      else
        fact *= (ld)1 - f.a1 * z - f.a2 * z * z;
    }
    ld scale = 0;
    for (auto ww : w) scale += std::fabs((ld)ww);
    if (std::abs(direct - fact) > 1e-11L * scale)
      return fail(MGB_ERR_INVALID, "factorisation check failed");
  }
  return MGB_OK;
}

void fill_factor_tables(const FactorDesc& fd, int T, int P, Factor& F) {
  std::memset(&F, 0, sizeof(F));
  F.a1 = (double)fd.a1;
  F.a2 = (double)fd.a2;
  F.dir = fd.dir;
  // windowed look-back: the carry of chunk t is exact to rounding from the K
  // previous chunks when (P K + 1) rho^(P K) < 1e-18 (K <= 16, K < T)
  F.win = 0;
  if (fd.rho > 0 && fd.rho < 1) {
    for (int K = 1; K <= 16 && K < T; ++K) {
      const ld pk = (ld)P * K;
      if ((pk + 1) * std::pow(fd.rho, pk) < 1e-18L) {
        F.win = K;
        break;
      }
    }
  } else if (fd.rho == 0) {
    F.win = 1;
  }
  const M2 A{(ld)F.a1, (ld)F.a2, 1, 0};
  M2 Ak = A;
  for (int q = 0; q < P; ++q) {
    F.h1[q] = (double)Ak.a;
    F.h2[q] = (double)Ak.b;
    Ak = mul(A, Ak);
  }
  const M2 M = mpow(A, P);
  put(F.M, M);
  M2 Mp = M;
  for (int k = 0; k < mgb::LOGT; ++k) {
    put(F.Mpow[k], Mp);
    Mp = mul(Mp, Mp);
  }
  const int R = (T + 31) / 32;
  M2 MR = mpow(M, R);
  for (int d = 0; d < 5; ++d) {
    put(F.MR[d], MR);
    MR = mul(MR, MR);
  }
  const M2 MT = mpow(M, T);
  const M2 IM{1 - MT.a, -MT.b, -MT.c, 1 - MT.d};
  const ld det = IM.a * IM.d - IM.b * IM.c;
  const M2 inv{IM.d / det, -IM.b / det, -IM.c / det, IM.a / det};
  put(F.Winv, inv);
}

int choose_layout(int kind, int n, int& P, int& T, int& S) {
  const int pmax = (kind == mgb::K_RK) ? 8 : 16;
  P = 1;
  for (int p = pmax; p >= 1; p >>= 1) {
    if (n % p == 0 && n / p >= 64) {
      P = p;
      break;
    }
  }
  while (n / P > 512 && P < 32 && n % (2 * P) == 0) P *= 2;
  T = n / P;
  if (T > 512 || T * P != n)
    return fail(MGB_ERR_UNSUPPORTED, "n_x=" + std::to_string(n) +
                                         " outside the single-CTA slice envelope (need n_x = T*P, T<=512, P<=32)");
  const int want = (P >= 16) ? 1 : 16 / P;
  S = T;
  while (S % 16 != want % 16) ++S;
  return MGB_OK;
}

long long mod_n(long long o, int n) {
  long long r = o % n;
  return r < 0 ? r + n : r;
}

}  // namespace

namespace mgb {
void register_kernel(const KernelKey& k, const void* fn) {
  std::lock_guard<std::mutex> lk(reg_mutex());
  registry()[std::make_tuple(k.kind, k.P, k.span, k.nst, k.exact)] = fn;
}

__global__ void sum_kernel(const double* __restrict__ p, long long n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += p[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    *out = tot;
  }
}
}  // namespace mgb

struct ClusterVariant {
  int C = 0, P = 0, T = 0, smem = 0, max_clusters = 0;
  bool one_red = false;  // relax_cl1_kernel (one reduction per Arnoldi step)
  int occ = 1;           // CTAs per SM the variant is compiled for
  int K = 0;             // basis rows resident in shared memory (one_red)
  double* ws = nullptr;  // per-CTA overflow rows (K < cap)
  const void* fn = nullptr;
};

struct mgb_step {
  StepParams hp;
  StepParams* dp = nullptr;
  int dkind = 0, P = 1, T = 1, S = 1, span = 0, nst = 1, exact = 1;
  bool vec16 = false;  // relax_win_kernel: 16-byte row accesses
  mgb::RkdConst rk = {};  // relax_rkd_kernel constants
  mgb::SldConst sd = {};  // relax_sld_kernel constants
  int threads = 32, smem = 0, max_grid = 1, sms = 148;
  const void* fn = nullptr;
  // SL_GMRES single-CTA: 2 CTAs/SM variant for levels that need > 1 wave of fn
  const void* fn2 = nullptr;
  int smem2 = 0, max_grid2 = 0;
  double* ws = nullptr;
  long long ws_slot = 0;
  int ws_slots = 0;
  std::vector<ClusterVariant> clusters;  // SL_GMRES: cluster sizes 16, 8, 4, 2
  std::vector<ClusterVariant> clusters1; // SL_GMRES one-reduction variants
};

namespace {
// Arguments of the sub-pass over intervals [k0, k0 + cnt) of pass ``a``.
mgb_relax_args sub_range(const mgb_relax_args& a, long long k0, long long cnt, int n) {
  mgb_relax_args s = a;
  s.n_intervals = cnt;
  s.k_global0 = a.k_global0 + k0;
  const long long rows = k0 * (long long)a.m * n;
  if (s.c_src) s.c_src += k0 * a.c_stride;
  if (s.e) s.e += k0 * a.e_stride;
  if (s.c_out) s.c_out += k0 * a.c_out_stride;
  if (s.u) s.u += rows;
  if (s.g) s.g += rows;
  if (s.tail_out) s.tail_out += k0 * a.tail_stride;
  if (s.cref) s.cref += k0 * a.cref_stride;
  if (s.cref_e) s.cref_e += k0 * a.cref_e_stride;
  if (s.z_out) s.z_out += k0 * a.z_stride;
  if (s.partials) s.partials += k0;
  if (s.stats_depth) s.stats_depth += k0;
  if (s.stats_res) s.stats_res += k0;
  if (k0 + cnt < a.n_intervals) s.c_last_out = nullptr;
  return s;
}

int launch_cluster1(mgb_step* st, const ClusterVariant& v, const mgb_relax_args& a, void* stream) {
  if (a.n_intervals <= 0) return MGB_OK;
  const long long ncl = std::min<long long>(a.n_intervals, v.max_clusters);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncl * v.C));
  cfg.blockDim = dim3(v.T);
  cfg.dynamicSmemBytes = v.smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = v.C;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  const StepParams* dpc = st->dp;
  mgb::RelaxLaunch L1;
  L1.a = a;
  L1.ws = v.ws;         // overflow basis rows (nullptr: all resident)
  L1.ws_slot = v.K;     // resident row count
  void* cargs[] = {(void*)&dpc, (void*)&L1};
  CUDA_TRY(cudaLaunchKernelExC(&cfg, v.fn, cargs));
  g_launches++;
  return MGB_OK;
}

// Cluster launch variants for SL_GMRES: C CTAs per interval, P <= 2 points per
// thread, 32 <= T <= 256 threads per CTA, column cap 10 or 20.
bool try_cluster_variant(ClusterVariant& v) {
  if (raise_smem_attr(v.fn, v.smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (v.C > 8 && cudaFuncSetAttribute(v.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(v.C);
  cfg.blockDim = dim3(v.T);
  cfg.dynamicSmemBytes = v.smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = v.C;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, v.fn, &cfg) != cudaSuccess || ncl < 1) {
    cudaGetLastError();
    return false;
  }
  v.max_clusters = ncl;
  return true;
}

// One-reduction variants (relax_cl1_kernel): the (I - phi D) stencil must be the
// symmetric window -r..r (r <= 3), the SL stencil <= 16 taps; each CTA has
// NW = nc / (32 SEGK) <= 8 vector warps plus the scalar warp.
void prepare_clusters1(mgb_step* st) {
  const StepParams& hp = st->hp;
  const int n = hp.n, cap = hp.cap;
  const int capt = cap <= 10 ? 10 : (cap <= 20 ? 20 : 0);
  if (!capt || !hp.win2_ok || hp.win2_span % 2 || hp.ntap > mgb::C1_MAXSL) return;
  const int r = hp.win2_span / 2;
  if (r > mgb::C1_MAXR || hp.win2_lo != (r == 0 ? 0 : n - r)) return;
  double wmax = 0.0;
  for (int d = 0; d <= 2 * r; ++d) wmax = std::max(wmax, std::fabs(hp.win2_w[d]));
  for (int d = 0; d < r; ++d)  // A symmetric (DCGS2 uses u.A V a = a.V^T A u)
    if (std::fabs(hp.win2_w[d] - hp.win2_w[2 * r - d]) > 1e-12 * wmax) return;
  for (int C : {16, 8, 4, 2, 1}) {
    if (n % C) continue;
    const int nc = n / C;
    int segk = 0, NW = 0, nwmax = 0;
    // (points per lane, vector-warp bound); 16 warps of 32-point segments measured
    // slower than 8 warps of 64 (cfg4 L3: 65.2 vs 63.8 ms)
    const int cand[6][2] = {{1, 8}, {2, 8}, {2, 16}, {4, 16}, {8, 8}, {8, 16}};
    const int min_segk = tuning().c1_segk;
    for (const auto& cd : cand) {
      if (cd[0] < min_segk) continue;
      if (nc % (32 * cd[0])) continue;
      const int nw = nc / (32 * cd[0]);
      if (nw >= 1 && nw <= cd[1] && (cd[1] == 8 || nw > 8)) { segk = cd[0]; NW = nw; nwmax = cd[1]; break; }
    }
    if (!segk || 3 * r > nc) continue;
    for (int occ2 = 0; occ2 < 2; ++occ2) {
      if (occ2 && !(nwmax == 8 && segk == 2 && capt == 20 && r >= 2)) continue;
      const size_t budget = occ2 ? 113 * 1024 : 227 * 1024;
      int K = capt;
      while (K > 1 && mgb::c1_smem_bytes(nc, NW, 32 * segk, r, C, capt, K) > budget) --K;
      // basis rows beyond K live in a workspace slot: only builds compiled for it
      // (wide segments; the 2-CTA/SM overflow build, key 109)
      if (K < capt && segk < 4 && !occ2) continue;
      const int key = occ2 ? (K < capt ? 109 : 108) : nwmax;
      const void* fn = nullptr;
      {
        std::lock_guard<std::mutex> lk(reg_mutex());
        auto it = registry().find(std::make_tuple((int)mgb::K_SLGC1, segk, capt, r, key));
        if (it == registry().end()) continue;
        fn = it->second;
      }
      ClusterVariant v;
      v.C = C;
      v.P = segk;
      v.T = 32 * (NW + 1);
      v.fn = fn;
      v.one_red = true;
      v.occ = occ2 ? 2 : 1;
      v.K = K;
      v.smem = (int)mgb::c1_smem_bytes(nc, NW, 32 * segk, r, C, capt, K);
      if ((size_t)v.smem > budget) continue;
      const bool ok = try_cluster_variant(v);
      if (tuning().debug)
        fprintf(stderr, "[mgb] cl1 variant n=%d C=%d segk=%d T=%d occ2=%d K=%d smem=%d ok=%d max_clusters=%d\n", n,
                C, segk, v.T, occ2, K, v.smem, (int)ok, v.max_clusters);
      if (!ok) continue;
      if (K < capt) {  // overflow rows: one slot of (cap - K) halo'd rows per resident CTA
        const size_t rows = (size_t)(capt - K) * mgb::c1_ld(nc, r);
        // + one double: the slots share the resident rows' 16-byte alignment shift
        if (cudaMalloc(&v.ws, rows * 8 * (size_t)v.max_clusters * C + 16) != cudaSuccess) {
          cudaGetLastError();
          continue;
        }
      }
      st->clusters1.push_back(v);
    }
  }
}

void prepare_clusters(mgb_step* st) {
  if (st->dkind != mgb::K_SLG) return;
  prepare_clusters1(st);
  const int n = st->hp.n, cap = st->hp.cap;
  const int capt = cap <= 10 ? 10 : (cap <= 20 ? 20 : 0);
  if (!capt) return;
  for (int C : {16, 8, 4, 2}) {
    if (n % C) continue;
    const int nc = n / C;
    int P = 0;
    for (int p : {1, 2})  // most warps (up to 8) for the warp-per-vector dot products
      if (nc % p == 0 && nc / p <= 256 && nc / p >= 32 && (nc / p) % 32 == 0) {
        P = p;
        break;
      }
    if (!P) continue;
    // every halo read must come from an adjacent slice
    bool ok = nc >= 2 * mgb::CL_H;
    for (int k = 0; k < st->hp.ntap2; ++k) {
      int o = st->hp.tap2_off[k];
      o = o > n / 2 ? o - n : o;
      ok = ok && std::abs(o) <= mgb::CL_H;
    }
    if (!ok) continue;
    const void* fn = nullptr;
    {
      std::lock_guard<std::mutex> lk(reg_mutex());
      auto it = registry().find(std::make_tuple((int)mgb::K_SLGC, P, capt, 1, 1));
      if (it == registry().end()) continue;
      fn = it->second;
    }
    ClusterVariant v;
    v.C = C;
    v.P = P;
    v.T = nc / P;
    v.fn = fn;
    v.smem = (int)(sizeof(StepParams) + 8 * (size_t)(capt == 10 ? mgb::ClLayout<10>::total(nc)
                                                                  : mgb::ClLayout<20>::total(nc)));
    if (raise_smem_attr(fn, v.smem) != cudaSuccess) continue;
    if (C > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(v.T);
    cfg.dynamicSmemBytes = v.smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = C;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      continue;
    }
    v.max_clusters = ncl;
    st->clusters.push_back(v);
  }
}
}  // namespace

extern "C" {

int mgb_version(void) { return 1; }
const char* mgb_last_error(void) { return g_err.c_str(); }
int64_t mgb_launch_count(void) { return g_launches.load(); }

int mgb_step_create(const mgb_step_desc* d, mgb_step** out) {
  if (!d || !out) return fail(MGB_ERR_INVALID, "null argument");
  *out = nullptr;
  ensure_registered();
  const int n = d->n_x;
  if (n < 1) return fail(MGB_ERR_INVALID, "n_x must be positive");
  if (d->n_taps < 1 || d->n_taps > mgb::MAX_TAPS)
    return fail(MGB_ERR_UNSUPPORTED, "primary stencil must have 1.." + std::to_string(mgb::MAX_TAPS) + " taps");
  auto st = new mgb_step();
  StepParams& hp = st->hp;
  std::memset(&hp, 0, sizeof(hp));
  hp.exact = d->exact ? 1 : 0;
  hp.repeat = std::max(1, (int)d->repeat);
  int dk;
  switch (d->kind) {
    case MGB_STEP_STENCIL: dk = mgb::K_GEN; break;
    case MGB_STEP_RK_STAGED: dk = mgb::K_RK; break;
    case MGB_STEP_SL_DIRECT: dk = mgb::K_SLD; break;
    case MGB_STEP_SL_GMRES: dk = mgb::K_SLG; break;
    default: delete st; return fail(MGB_ERR_INVALID, "unknown step kind");
  }
  int P, T, S;
  long long rk_front = 1;  // first offset of a contiguous -cL stencil (RK kind)
  int rc = choose_layout(dk, n, P, T, S);
  if (rc) { delete st; return rc; }
  hp.n = n; hp.P = P; hp.T = T; hp.S = S;
  hp.ntap = d->n_taps;
  std::vector<long long> off(d->n_taps);
  for (int k = 0; k < d->n_taps; ++k) {
    off[k] = d->offsets[k];
    hp.tap_off[k] = (int)mod_n(off[k], n);
    hp.tap_w[k] = d->weights[k];
  }
  // register-window eligibility (explicit stencils)
  int span = 0;
  if (dk == mgb::K_GEN) {
    bool inc = true;
    for (int k = 1; k < d->n_taps; ++k) inc = inc && off[k] > off[k - 1];
    const long long sp = off.back() - off.front();
    if (inc && sp <= 30 && P >= 4 && T >= 64) {
      for (int s : mgb::kWinSpans)
        if (s >= sp) { span = s; break; }
      dk = mgb::K_WIN;
      hp.win_lo = (int)mod_n(off.front(), n);
      hp.win_span = span;
      for (int k = 0; k < d->n_taps; ++k) hp.win_w[off[k] - off.front()] = d->weights[k];
    }
  }
  if (dk == mgb::K_RK) {
    if (d->stages < 1 || d->stages > mgb::MAX_ST) { delete st; return fail(MGB_ERR_UNSUPPORTED, "1..6 RK stages supported"); }
    hp.stages = d->stages;
    for (int i = 0; i < d->stages; ++i) {
      hp.b[i] = d->rk_b[i];
      for (int j = 0; j < d->stages; ++j) hp.A[i * mgb::MAX_ST + j] = d->rk_a[i * d->stages + j];
    }
    hp.implicit = d->implicit ? 1 : 0;
    if (hp.implicit) {
      // SDIRK with a constant nonzero diagonal, fast (non-exact) mode only: stage
      // values from the solves, z = (y - rhs) / gamma.  Exact mode keeps the
      // reference's z = cL y (stepping.py:374): the subtraction cancels on
      // smooth modes and biases them by ~1e-16 per step (a 3e-12 drift of
      // cfg3's final iterate over 16384 steps).
      const bool stencil_stages = tuning().rk_stencil;
      const double g = hp.A[0];
      bool ok = g != 0.0 && !stencil_stages && !hp.exact;
      for (int i = 1; i < d->stages; ++i) ok = ok && hp.A[i * mgb::MAX_ST + i] == g;
      hp.z_solve = ok ? 1 : 0;
      hp.inv_gamma = ok ? 1.0 / g : 0.0;
    }
    // register-window form of the -cL stencil (contiguous, span <= 6)
    bool inc = true;
    for (int k = 1; k < d->n_taps; ++k) inc = inc && off[k] > off[k - 1];
    const long long sp1 = off.back() - off.front();
    rk_front = inc ? off.front() : 1;
    if (inc && sp1 <= 6 && T >= 8) {
      hp.win1_ok = 1;
      hp.win_lo = (int)mod_n(off.front(), n);
      hp.win_span = (int)sp1;
      for (int k = 0; k < d->n_taps; ++k) hp.win_w[off[k] - off.front()] = d->weights[k];
    }
  }
  hp.gain_inv = 1.0;
  if (((dk == mgb::K_RK && hp.implicit) || dk == mgb::K_SLD) && P > mgb::MAXP) {
    delete st;
    return fail(MGB_ERR_UNSUPPORTED, "implicit banded solves support n_x <= " + std::to_string(512 * mgb::MAXP));
  }
  if ((dk == mgb::K_RK && hp.implicit) || dk == mgb::K_SLD) {
    if (d->n_taps2 < 1) { delete st; return fail(MGB_ERR_INVALID, "implicit operator stencil missing"); }
    std::vector<long long> o2(d->offsets2, d->offsets2 + d->n_taps2);
    std::vector<double> w2(d->weights2, d->weights2 + d->n_taps2);
    std::vector<FactorDesc> facs;
    ld K;
    int shift;
    rc = factorize(o2, w2, n, facs, K, shift);
    if (rc) { delete st; return rc; }
    if ((int)facs.size() > mgb::MAX_FAC) { delete st; return fail(MGB_ERR_UNSUPPORTED, "too many factors"); }
    hp.nfac = (int)facs.size();
    for (int f = 0; f < hp.nfac; ++f) fill_factor_tables(facs[f], T, P, hp.fac[f]);
    if (tuning().debug)
      for (int f = 0; f < hp.nfac; ++f)
        fprintf(stderr, "[mgb] n=%d P=%d T=%d factor %d: a1=%.6g a2=%.6g dir=%d rho=%.4Lf win=%d\n", n, P, T, f,
                hp.fac[f].a1, hp.fac[f].a2, hp.fac[f].dir, facs[f].rho, hp.fac[f].win);
    hp.gain_inv = (double)(1.0L / K);
    hp.shift = (int)mod_n(shift, n);
    if (hp.shift > n / 2) hp.shift -= n;
  }
  if (dk == mgb::K_SLG) {
    if (d->n_taps2 < 1 || d->n_taps2 > mgb::MAX_TAPS2) { delete st; return fail(MGB_ERR_UNSUPPORTED, "GMRES operator stencil size"); }
    hp.ntap2 = d->n_taps2;
    for (int k = 0; k < d->n_taps2; ++k) {
      hp.tap2_off[k] = (int)mod_n(d->offsets2[k], n);
      hp.tap2_w[k] = d->weights2[k];
    }
    {  // register-window form of the (I - phi D) stencil: contiguous, span <= 6
      bool inc = true;
      for (int k = 1; k < d->n_taps2; ++k) inc = inc && d->offsets2[k] > d->offsets2[k - 1];
      const long long sp2 = d->offsets2[d->n_taps2 - 1] - d->offsets2[0];
      if (inc && sp2 <= 6) {
        hp.win2_ok = 1;
        hp.win2_lo = (int)mod_n(d->offsets2[0], n);
        hp.win2_span = (int)sp2;
        for (int k = 0; k < d->n_taps2; ++k) hp.win2_w[d->offsets2[k] - d->offsets2[0]] = d->weights2[k];
      }
    }
    hp.tol = d->gmres_tol;
    hp.cap = std::min((int)d->gmres_cap, n);
    if (hp.cap < 1 || hp.cap > mgb::MAX_CAP) { delete st; return fail(MGB_ERR_UNSUPPORTED, "GMRES cap must be 1..128"); }
  }
  hp.kind = dk;
  st->dkind = dk;
  st->P = P; st->T = T; st->S = S;
  st->span = span;
  // dedicated kernel: even n_x, <= 256 threads at 2 CTAs/SM; fixed-geometry builds
  // (compile-time T, wrap replicas in the slice) for 16 x 256 and 16 x 512
  const bool win_fixed = dk == mgb::K_WIN && P == 16 && (T == 256 || T == 512);
  const bool win_dedicated = dk == mgb::K_WIN && P <= 16 && n % 2 == 0 && (T <= 256 || win_fixed);
  if (win_fixed) st->S = hp.S = S = (T == 256 ? mgb::WinGeo<256>::S : mgb::WinGeo<512>::S);
  st->vec16 = win_dedicated;
  st->nst = dk == mgb::K_RK ? hp.stages + (hp.z_solve ? mgb::RK_ZSOLVE : 0) : 1;
  st->exact = (dk == mgb::K_WIN || dk == mgb::K_GEN) ? hp.exact : 1;
  st->threads = ((T + 31) / 32) * 32;
  size_t dbl = (size_t)P * S + 64 + 8;
  if (dk == mgb::K_RK || dk == mgb::K_SLD) dbl += 4 * (size_t)mgb::scan_stride(T) + 4 * (size_t)T;
  if (dk == mgb::K_SLG) dbl += mgb::GmLayout::total(n);  // Hessenberg state, R, 2 TMA stages
  st->smem = (int)(sizeof(StepParams) + 8 * dbl);
  if (win_dedicated)  // relax_win_kernel: double-buffered slice, weights as kernel parameters
    st->smem = (int)(8 * (2 * (size_t)P * S + 32));  // 2 slices + reduction
  // dedicated SDIRK kernel: 8 (or 4) points per thread, every factor a windowed (fast-decaying)
  // recurrence, no symbol shift, -cL stencil with (HL, HR) halo of upwind order 1 / 3 / 5
  int rkd_key = 0;
  if (dk == mgb::K_RK && hp.implicit && (P == 8 || P == 4) && hp.shift == 0 && hp.win1_ok && hp.stages <= 3 &&
      !tuning().no_rkd) {
    bool allwin = hp.nfac >= 1;
    for (int f = 0; f < hp.nfac; ++f) allwin = allwin && hp.fac[f].win > 0;
    const int HL = (int)-rk_front, HR = hp.win_span - HL;
    allwin = allwin && hp.nfac <= mgb::RKD_MAXF;
    if (allwin && ((HL == 1 && HR == 0) || (HL == 2 && HR == 1) || (HL == 3 && HR == 2)))
      rkd_key = 100 + 10 * HL + HR;
  }
  // dedicated SL + direct-solve kernel: contiguous SL stencil of span 0..5, at most two
  // factors (first / second order), no symbol shift, whole warps
  int sld_key = 0;
  if (dk == mgb::K_SLD && !tuning().no_sld && P >= 4 && P <= 16 && T % 32 == 0 && T <= 512 &&
      hp.shift == 0 && hp.nfac >= 1 && hp.nfac <= 2 && d->n_taps >= 1 && d->n_taps <= 6) {
    bool contig = true;
    for (int k = 1; k < d->n_taps; ++k) contig = contig && off[k] == off[0] + k;
    if (contig) {
      sld_key = 200 + d->n_taps - 1;
      hp.win_lo = (int)mod_n(off[0], n);
      hp.win_span = d->n_taps - 1;
      for (int k = 0; k < d->n_taps; ++k) hp.win_w[k] = d->weights[k];
      st->smem = (int)(8 * (192 + 4 * (size_t)(T + mgb::RKD_KMAX) + 2 * (size_t)P * (T + mgb::WIN_X)));
      mgb::SldConst& sd = st->sd;
      std::memset(&sd, 0, sizeof(sd));
      sd.nfac = hp.nfac;
      sd.gain_inv = hp.gain_inv;
      for (int f = 0; f < hp.nfac; ++f) {
        const Factor& F = hp.fac[f];
        mgb::SldFactor& R = sd.f[f];
        R.a1 = F.a1; R.a2 = F.a2; R.dir = F.dir; R.win = F.win;
        for (int k = 0; k < 4; ++k) { R.M[k] = F.M[k]; R.Winv[k] = F.Winv[k]; }
        for (int q = 0; q < P; ++q) { R.h1[q] = F.h1[q]; R.h2[q] = F.h2[q]; }
        for (int e = 0; e < 10; ++e)
          for (int k = 0; k < 4; ++k) R.Mpow[e][k] = F.Mpow[e][k];
      }
    }
  }
  if (tuning().debug && dk == mgb::K_SLD) {
    fprintf(stderr, "[mgb] sld n=%d P=%d T=%d shift=%d nfac=%d ntaps=%d key=%d offsets:", n, P, T, hp.shift, hp.nfac,
            (int)d->n_taps, sld_key);
    for (int k = 0; k < d->n_taps; ++k) fprintf(stderr, " %lld", off[k]);
    fprintf(stderr, "\n");
  }
  if (rkd_key) {
    st->smem = (int)(sizeof(StepParams) + 8 * (72 + 4 * (size_t)(T + mgb::RKD_KMAX) + (size_t)hp.win_span * T +
                                               (size_t)(hp.stages - 1) * P * T));
    mgb::RkdConst& rk = st->rk;
    std::memset(&rk, 0, sizeof(rk));
    rk.nfac = hp.nfac;
    for (int f = 0; f < hp.nfac; ++f) {
      const Factor& F = hp.fac[f];
      mgb::RkdFactor& R = rk.f[f];
      R.a1 = F.a1; R.a2 = F.a2; R.dir = F.dir; R.win = F.win;
      for (int k = 0; k < 4; ++k) R.M[k] = F.M[k];
      for (int q = 0; q < P; ++q) { R.h1[q] = F.h1[q]; R.h2[q] = F.h2[q]; }
    }
    for (int i = 0; i < hp.stages; ++i) {
      rk.b[i] = hp.b[i];
      for (int j = 0; j < hp.stages; ++j) rk.A[i * 3 + j] = hp.A[i * mgb::MAX_ST + j];
    }
    rk.gain_inv = hp.gain_inv;
    rk.inv_gamma = hp.inv_gamma;
  }
  // SL + GMRES on rows whose single-CTA slice + TMA stages exceed shared memory
  // (n_x > 8192): cluster kernels only
  const bool cluster_only = dk == mgb::K_SLG && st->smem > 227 * 1024;
  if (cluster_only) {
    st->fn = nullptr;
    st->max_grid = 0;
    prepare_clusters(st);
    if (st->clusters1.empty()) {
      delete st;
      return fail(MGB_ERR_UNSUPPORTED, "no cluster GMRES variant for n_x=" + std::to_string(n));
    }
    cudaError_t e0 = cudaMalloc(&st->dp, sizeof(StepParams));
    if (e0 != cudaSuccess) { delete st; return fail(MGB_ERR_CUDA, "cudaMalloc params"); }
    e0 = cudaMemcpy(st->dp, &hp, sizeof(StepParams), cudaMemcpyHostToDevice);
    if (e0 != cudaSuccess) { cudaFree(st->dp); delete st; return fail(MGB_ERR_CUDA, "upload params"); }
    *out = st;
    return MGB_OK;
  }
  {
    std::lock_guard<std::mutex> lk(reg_mutex());
    auto it = registry().end();
    if (dk == mgb::K_SLG && T <= 256)  // register-rich variant (launch bound 256)
      it = registry().find(std::make_tuple(dk, P, span, 2, st->exact));
    if (dk == mgb::K_WIN && !win_dedicated)  // odd n_x / 16384-point rows: generic-kernel variant
      it = registry().find(std::make_tuple(dk, P, span, 2, st->exact));
    if (win_fixed) it = registry().find(std::make_tuple(dk, P, span, T == 512 ? 3 : 4, st->exact));
    if (rkd_key) it = registry().find(std::make_tuple(dk, P, rkd_key, st->nst, st->exact));
    if (sld_key) it = registry().find(std::make_tuple(dk, P, sld_key, 1, 1));
    if (it == registry().end()) it = registry().find(std::make_tuple(dk, P, span, st->nst, st->exact));
    if (it == registry().end()) { delete st; return fail(MGB_ERR_UNSUPPORTED, "no kernel instantiation for this layout"); }
    st->fn = it->second;
  }
  cudaError_t e = raise_smem_attr(st->fn, st->smem);
  if (e != cudaSuccess) { delete st; return fail(MGB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e)); }
  int nb = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, st->fn, st->threads, st->smem);
  if (e != cudaSuccess || nb < 1) {
    delete st;
    return fail(MGB_ERR_UNSUPPORTED, std::string("kernel cannot be resident: ") + cudaGetErrorString(e));
  }
  st->max_grid = nb * sms;
  st->sms = sms;
  if (dk == mgb::K_SLG && T <= 256 && nb == 1) {
    const bool no_occ2 = tuning().slg_no_occ2;
    const void* fn2 = nullptr;
    {
      std::lock_guard<std::mutex> lk(reg_mutex());
      auto it2 = registry().find(std::make_tuple((int)dk, P, span, 3, st->exact));
      if (it2 != registry().end()) fn2 = it2->second;
    }
    const int smem2 = st->smem - (int)sizeof(StepParams) + mgb::sp_smem_bytes<mgb::K_SLG, 2>();
    int nb2 = 0;
    if (fn2 && !no_occ2 && raise_smem_attr(fn2, smem2) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, fn2, st->threads, smem2) == cudaSuccess &&
        nb2 >= 2) {
      st->fn2 = fn2;
      st->smem2 = smem2;
      st->max_grid2 = nb2 * sms;
    }
    cudaGetLastError();
  }
  prepare_clusters(st);
  e = cudaMalloc(&st->dp, sizeof(StepParams));
  if (e != cudaSuccess) { delete st; return fail(MGB_ERR_CUDA, "cudaMalloc params"); }
  e = cudaMemcpy(st->dp, &hp, sizeof(StepParams), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(st->dp); delete st; return fail(MGB_ERR_CUDA, "upload params"); }
  *out = st;
  return MGB_OK;
}

void mgb_step_destroy(mgb_step* st) {
  if (!st) return;
  for (ClusterVariant& v : st->clusters1)
    if (v.ws) cudaFree(v.ws);
  if (st->dp) cudaFree(st->dp);
  if (st->ws) cudaFree(st->ws);
  delete st;
}

int mgb_step_layout(const mgb_step* st, int32_t* threads, int32_t* ppt, int32_t* smem) {
  if (!st) return fail(MGB_ERR_INVALID, "null step");
  if (threads) *threads = st->T;
  if (ppt) *ppt = st->P;
  if (smem) *smem = st->smem;
  return MGB_OK;
}

int mgb_step_reserve_workspace(mgb_step* st, void* stream) {
  (void)stream;
  if (!st) return fail(MGB_ERR_INVALID, "null step");
  if (st->dkind != mgb::K_SLG || st->ws || !st->fn) return MGB_OK;
  const long long cap = st->hp.cap, n = st->hp.n;
  st->ws_slot = (cap + 1) * n + cap * cap + 3 * cap + 1;
  st->ws_slot = (st->ws_slot + 31) / 32 * 32;
  st->ws_slots = std::max(st->max_grid, st->fn2 ? st->max_grid2 : 0);
  CUDA_TRY(cudaMalloc(&st->ws, (size_t)st->ws_slot * st->ws_slots * sizeof(double)));
  return MGB_OK;
}

int mgb_relax(mgb_step* st, const mgb_relax_args* a, void* stream) {
  if (!st || !a) return fail(MGB_ERR_INVALID, "null argument");
  if (a->n_intervals <= 0) return MGB_OK;
  if (a->m < 1 || a->n_fsteps < 0) return fail(MGB_ERR_INVALID, "bad m / n_fsteps");
  if (a->tail == 1 && !a->tail_out) return fail(MGB_ERR_INVALID, "C-relax tail needs tail_out");
  if (a->tail == 2 && !a->cref) return fail(MGB_ERR_INVALID, "residual tail needs cref");
  if (a->write_f && !a->u) return fail(MGB_ERR_INVALID, "write_f needs u");
  if (a->z_out && (a->tail != 2 || !(st->dkind == mgb::K_WIN || st->dkind == mgb::K_GEN ||
                                      (st->dkind == mgb::K_RK))))
    return fail(MGB_ERR_UNSUPPORTED, "z_out needs a residual tail on an explicit or staged-RK plan");
  if (st->vec16) {  // dedicated stencil kernel moves rows with 16-byte accesses
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    const bool ok = al(a->c_src) && al(a->c_src0) && al(a->e) && al(a->c_out) && al(a->c_last_out) &&
                    al(a->u) && al(a->g) && al(a->tail_out) && al(a->cref) && al(a->cref_e) && al(a->z_out) &&
                    a->z_stride % 2 == 0 &&
                    a->c_stride % 2 == 0 && a->e_stride % 2 == 0 && a->c_out_stride % 2 == 0 &&
                    a->tail_stride % 2 == 0 && a->cref_stride % 2 == 0 && a->cref_e_stride % 2 == 0;
    if (!ok) return fail(MGB_ERR_INVALID, "explicit-stencil relax needs 16-byte aligned rows and even strides");
  }
  mgb::RelaxLaunch L;
  L.a = *a;
  L.ws = nullptr;
  L.ws_slot = 0;
  std::memcpy(L.win_w, st->hp.win_w, sizeof(L.win_w));
  L.rk = st->rk;
  L.sd = st->sd;
  long long grid = std::min<long long>(a->n_intervals, st->max_grid);
  // tooling / tests only: cap the grid so that every CTA walks a block of
  // several intervals (the chained head/tail hand-off of relax_win_kernel)
  const long long grid_cap = tuning().max_grid;
  if (grid_cap > 0) grid = std::min(grid, grid_cap);
  const Tuning& tn = tuning();
  const bool no_cluster = tn.no_cluster, cgs2 = tn.cgs2;
  if (st->dkind == mgb::K_SLG && !no_cluster && !cgs2 && !st->clusters1.empty()) {
    // Launch plan over the level's intervals (each a chain of sequential GMRES
    // solves, so a wave costs one chain whatever its width): the variant with
    // the fewest waves of clusters; ties -> larger clusters, except that a 2-CTA/SM build
    // whose basis overflows to the workspace yields to a one-CTA/SM build with every row
    // resident (cfg4 L2: 162 -> 150 ms; cfg2 L2 keeps its resident 2-CTA/SM build).  When the last wave
    // would be partial and a faster variant (one CTA/SM with every basis row
    // resident, at least as large clusters) holds it in one wave of its own,
    // that tail goes to the faster variant as a second launch.
    auto usable = [&](const ClusterVariant& v) {
      if (tn.c1_c && v.C != tn.c1_c) return false;
      if (tn.c1_no_occ2 && v.occ == 2) return false;
      // wide segments (cluster sizes 1-2 on 4096-point rows) measured slower than
      // the single-CTA kernel for many-interval levels: opt-in only -- except on rows
      // too long for the single-CTA kernel (n_x = 16384), where they are the only way
      // to run many intervals at once (cfg5 proxy 16384 x 16384: 970 -> 608 ms)
      if (v.P >= 4 && !tn.c1_wide && !tn.c1_c && st->fn) return false;
      return true;
    };
    const ClusterVariant* best = nullptr;
    long long best_w = 0;
    for (const ClusterVariant& v : st->clusters1) {
      if (!usable(v)) continue;
      const long long w = (a->n_intervals + v.max_clusters - 1) / v.max_clusters;
      if (!best || w < best_w || (w == best_w && best->occ == 2 && best->ws && v.occ == 1 && !v.ws)) { best = &v; best_w = w; }
    }
    // many-interval levels (> max_waves cluster waves) run faster on the single-CTA kernel
    if (best && (best_w <= tn.c1_waves || !st->fn)) {
      long long head = a->n_intervals;
      const ClusterVariant* tailv = nullptr;
      if (best_w >= 2 && !tn.c1_no_split) {
        const long long rem = a->n_intervals - (best_w - 1) * best->max_clusters;
        for (const ClusterVariant& v : st->clusters1) {  // ordered by decreasing cluster size
          if (!usable(v) || v.occ != 1 || v.ws || v.C < best->C || (v.C == best->C && best->occ == 1)) continue;
          if (rem <= v.max_clusters) { tailv = &v; break; }
        }
        if (tailv) head = a->n_intervals - rem;
      }
      int rc = launch_cluster1(st, *best, sub_range(*a, 0, head, st->hp.n), stream);
      if (rc == MGB_OK && tailv)
        rc = launch_cluster1(st, *tailv, sub_range(*a, head, a->n_intervals - head, st->hp.n), stream);
      return rc;
    }
  }
  if (st->dkind == mgb::K_SLG && !no_cluster) {
    const long long max_waves = tn.cluster_waves;
    for (const ClusterVariant& v : st->clusters) {  // largest cluster size within max_waves
      if (a->n_intervals > max_waves * (long long)v.max_clusters) continue;
      const long long ncl = std::min<long long>(a->n_intervals, v.max_clusters);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(ncl * v.C));
      cfg.blockDim = dim3(v.T);
      cfg.dynamicSmemBytes = v.smem;
      cfg.stream = (cudaStream_t)stream;
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = v.C;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      const StepParams* dpc = st->dp;
      void* cargs[] = {(void*)&dpc, (void*)&L};
      CUDA_TRY(cudaLaunchKernelExC(&cfg, v.fn, cargs));
      g_launches++;
      return MGB_OK;
    }
  }
  if (!st->fn) return fail(MGB_ERR_UNSUPPORTED, "this plan runs on cluster kernels only (n_x too long for one CTA)");
  if (st->dkind == mgb::K_SLG) {
    int rc = mgb_step_reserve_workspace(st, stream);
    if (rc) return rc;
    L.ws = st->ws;
    L.ws_slot = st->ws_slot;
    if (st->fn2 && a->n_intervals > st->max_grid) {  // one wave at 2 CTAs/SM instead of two
      const long long grid2 = std::min<long long>(std::min<long long>(a->n_intervals, st->max_grid2),
                                                  st->ws_slots);
      const StepParams* dp2 = st->dp;
      void* args2[] = {(void*)&dp2, (void*)&L};
      CUDA_TRY(cudaLaunchKernel(st->fn2, dim3((unsigned)grid2), dim3(st->threads), args2,
                                (size_t)st->smem2, (cudaStream_t)stream));
      g_launches++;
      return MGB_OK;
    }
    grid = std::min<long long>(grid, st->ws_slots);
    if (grid_cap > 0) grid = std::min(grid, grid_cap);
  }
  const StepParams* dp = st->dp;
  void* args[] = {(void*)&dp, (void*)&L};
  CUDA_TRY(cudaLaunchKernel(st->fn, dim3((unsigned)grid), dim3(st->threads), args, (size_t)st->smem,
                            (cudaStream_t)stream));
  g_launches++;
  return MGB_OK;
}

int mgb_copy_rows(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                  int64_t row_bytes, int64_t rows, void* stream) {
  if (rows <= 0 || row_bytes <= 0) return MGB_OK;
  if (!dst || !src) return fail(MGB_ERR_INVALID, "null pointer");
  if (dst_pitch < row_bytes || src_pitch < row_bytes) return fail(MGB_ERR_INVALID, "pitch < row bytes");
  CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)dst_pitch, src, (size_t)src_pitch, (size_t)row_bytes,
                             (size_t)rows, cudaMemcpyDefault, (cudaStream_t)stream));
  return MGB_OK;
}

int mgb_sum(const double* partials, int64_t n, double* out, void* stream) {
  if (!out) return fail(MGB_ERR_INVALID, "null out");
  if (n <= 0) {
    CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), (cudaStream_t)stream));
    return MGB_OK;
  }
  mgb::sum_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(partials, (long long)n, out);
  CUDA_TRY(cudaGetLastError());
  g_launches++;
  return MGB_OK;
}

}  // extern "C"
