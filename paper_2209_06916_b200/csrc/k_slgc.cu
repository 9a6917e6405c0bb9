// Cluster GMRES relaxation instantiations (P points per thread, column cap).
#include "mgb_cluster.cuh"
#include "mgb_registry.h"

namespace mgb {
#define REG_CL(P, CAP)                                                                   \
  register_kernel(KernelKey{K_SLGC, P, CAP, 1, 1},                                       \
                  reinterpret_cast<const void*>(&relax_cluster_kernel<P, CAP>))
void register_slgc() {
  REG_CL(1, 10);
  REG_CL(1, 20);
  REG_CL(2, 10);
  REG_CL(2, 20);
}
}  // namespace mgb

#ifdef MGB_CL_TRACE
// trace builds only: fetch and clear the cluster-kernel phase timers
extern "C" int mgb_trace_fetch(unsigned long long* out16) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, mgb::g_cl_trace, 16 * sizeof(unsigned long long));
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(mgb::g_cl_trace, z, sizeof(z));
  return (int)cudaGetLastError();
}
#endif
