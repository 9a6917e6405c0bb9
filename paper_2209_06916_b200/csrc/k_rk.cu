// Staged Runge-Kutta relaxation (explicit or SDIRK with factorised stage solves).
#include "mgb_registry.h"

namespace mgb {
#define RK_P(P)                   \
  MGB_REG(K_RK, P, 0, 1, true); \
  MGB_REG(K_RK, P, 0, 2, true); \
  MGB_REG(K_RK, P, 0, 3, true); \
  MGB_REG(K_RK, P, 0, 4, true); \
  MGB_REG(K_RK, P, 0, 5, true); \
  MGB_REG(K_RK, P, 0, 6, true); \
  MGB_REG(K_RK, P, 0, 1 + RK_ZSOLVE, true); \
  MGB_REG(K_RK, P, 0, 2 + RK_ZSOLVE, true); \
  MGB_REG(K_RK, P, 0, 3 + RK_ZSOLVE, true); \
  MGB_REG(K_RK, P, 0, 4 + RK_ZSOLVE, true); \
  MGB_REG(K_RK, P, 0, 5 + RK_ZSOLVE, true); \
  MGB_REG(K_RK, P, 0, 6 + RK_ZSOLVE, true);
void register_rk() {
  RK_P(1)
  RK_P(2)
  RK_P(4)
  RK_P(8)
  RK_P(16)
}
}  // namespace mgb

#ifdef MGB_CL_TRACE
extern "C" int mgb_trace_fetch_rk(unsigned long long* out16) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, mgb::g_cl_trace, 16 * sizeof(unsigned long long));
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(mgb::g_cl_trace, z, sizeof(z));
  return (int)cudaGetLastError();
}
#endif
