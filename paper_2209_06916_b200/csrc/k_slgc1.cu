// One-reduction cluster GMRES relaxation instantiations (segment = 32*SEGK points
// per vector warp, column cap).
#include "mgb_cluster1.cuh"
#include "mgb_registry.h"

namespace mgb {
#define REG_CL1(SEGK, CAP, R, NWMAX)                                                     \
  register_kernel(KernelKey{K_SLGC1, SEGK, CAP, R, NWMAX},                               \
                  reinterpret_cast<const void*>(&relax_cl1_kernel<SEGK, CAP, R, NWMAX>))
// reach R of (I - phi D^(p+1)): p = 1 -> 1 (cap 10), p = 3 -> 2, p = 5 -> 3 (cap 20);
// NWMAX vector warps per CTA (8: 288 threads, 16: 544 threads with 64-point segments)
// (key 108: every basis row resident; key 109: rows beyond the shared-memory
// budget in the CTA's L2-resident workspace slot)
#define REG_CL1B(SEGK, CAP, R)                                                           \
  register_kernel(KernelKey{K_SLGC1, SEGK, CAP, R, 108},                                 \
                  reinterpret_cast<const void*>(&relax_cl1_kernel<SEGK, CAP, R, 8, 2>)); \
  register_kernel(KernelKey{K_SLGC1, SEGK, CAP, R, 109},                                 \
                  reinterpret_cast<const void*>(&relax_cl1_kernel<SEGK, CAP, R, 8, 2, true>))
void register_slgc1() {
  // two CTAs per SM (<= 112 registers): single-wave launches of mid-sized levels
  REG_CL1B(2, 20, 2);
  REG_CL1B(2, 20, 3);
  // wide segments (cluster sizes 1-4 on long rows): lane-parallel dots, L2 overflow rows
  REG_CL1(4, 20, 2, 16);
  REG_CL1(8, 20, 2, 8);
  REG_CL1(8, 20, 2, 16);
  REG_CL1(4, 20, 3, 16);
  REG_CL1(8, 20, 3, 8);
  REG_CL1(8, 20, 3, 16);
  REG_CL1(4, 10, 1, 16);
  REG_CL1(8, 10, 1, 8);
  REG_CL1(8, 10, 1, 16);
  REG_CL1(1, 10, 1, 8);
  REG_CL1(2, 10, 1, 8);
  REG_CL1(2, 10, 1, 16);
  REG_CL1(1, 20, 2, 8);
  REG_CL1(2, 20, 2, 8);
  REG_CL1(2, 20, 2, 16);
  REG_CL1(1, 20, 3, 8);
  REG_CL1(2, 20, 3, 8);
  REG_CL1(2, 20, 3, 16);
}
}  // namespace mgb

#ifdef MGB_CL_TRACE
extern "C" int mgb_trace_fetch_c1(unsigned long long* out16) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, mgb::g_cl_trace, 16 * sizeof(unsigned long long));
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(mgb::g_cl_trace, z, sizeof(z));
  return (int)cudaGetLastError();
}
#endif
