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
