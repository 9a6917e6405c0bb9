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
// dedicated SDIRK kernel (8 or 4 points per thread, all factors windowed, shift 0):
// key span = 100 + 10 HL + HR (halo points of the -cL stencil), nst as above
#define RKD_P(P, NS, HL, HR)                                                                   \
  register_kernel(KernelKey{K_RK, P, 100 + 10 * HL + HR, NS, 1},                               \
                  reinterpret_cast<const void*>(&relax_rkd_kernel<P, NS, false, HL, HR>));     \
  register_kernel(KernelKey{K_RK, P, 100 + 10 * HL + HR, NS + RK_ZSOLVE, 1},                   \
                  reinterpret_cast<const void*>(&relax_rkd_kernel<P, NS, true, HL, HR>));
#define RKD(NS, HL, HR) RKD_P(8, NS, HL, HR) RKD_P(4, NS, HL, HR)
void register_rk() {
  RKD(1, 1, 0) RKD(2, 1, 0) RKD(3, 1, 0)
  RKD(1, 2, 1) RKD(2, 2, 1) RKD(3, 2, 1)
  RKD(1, 3, 2) RKD(2, 3, 2) RKD(3, 3, 2)
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
