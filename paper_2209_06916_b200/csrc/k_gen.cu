// Generic-tap stencil relaxation (exact / fast), semi-Lagrangian + direct
// correction solve, semi-Lagrangian + GMRES correction.
#include "mgb_registry.h"

namespace mgb {
#define GEN_P(P)                    \
  MGB_REG(K_GEN, P, 0, 1, true);  \
  MGB_REG(K_GEN, P, 0, 1, false); \
  MGB_REG(K_SLD, P, 0, 1, true);  \
  MGB_REG(K_SLG, P, 0, 1, true);
void register_gen() {
  // register-rich GMRES variants for T <= 256 (key: nst = 2)
  register_kernel(KernelKey{K_SLG, 16, 0, 2, 1},
                  reinterpret_cast<const void*>(&relax_kernel<16, K_SLG, 0, 1, true, 256>));
  register_kernel(KernelKey{K_SLG, 8, 0, 2, 1},
                  reinterpret_cast<const void*>(&relax_kernel<8, K_SLG, 0, 1, true, 256>));
  GEN_P(1)
  GEN_P(2)
  GEN_P(4)
  GEN_P(8)
  GEN_P(16)
}
}  // namespace mgb

#ifdef MGB_CL_TRACE
extern "C" int mgb_trace_fetch_gen(unsigned long long* out16) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, mgb::g_cl_trace, 16 * sizeof(unsigned long long));
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(mgb::g_cl_trace, z, sizeof(z));
  return (int)cudaGetLastError();
}
#endif
