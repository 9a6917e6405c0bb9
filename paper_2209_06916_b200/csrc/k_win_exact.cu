// Register-window stencil relaxation, exact (mul-then-add, canonical tap
// order: bitwise equal to the reference's rolled sums, circulant.py:119-123).
#include "mgb_registry.h"

#ifndef MGB_WIN_MINB256
#define MGB_WIN_MINB256 2  // CTAs per SM of the 256-thread fixed-geometry build
#endif

namespace mgb {
// key nst = 1: dedicated double-buffered kernel at <= 256 threads, 2 CTAs/SM;
// nst = 2: generic single-buffer slice kernel (fallback: odd n_x, 16384-point rows)
#define WIN_D(P, SPAN)                                                                          \
  register_kernel(KernelKey{K_WIN, P, SPAN, 1, 1},                                              \
                  reinterpret_cast<const void*>(&relax_win_kernel<P, SPAN, true>));             \
  MGB_REG(K_WIN, P, SPAN, 2, true);
// fixed-geometry builds for 16 points per thread: nst = 3: 512 threads (8192-point
// rows), 1 CTA/SM; nst = 4: 256 threads (4096-point rows), 2 CTAs/SM
#define WIN_FIX(SPAN)                                                                           \
  register_kernel(KernelKey{K_WIN, 16, SPAN, 3, 1},                                             \
                  reinterpret_cast<const void*>(&relax_win_kernel<16, SPAN, true, 512, 1, 512>)); \
  register_kernel(KernelKey{K_WIN, 16, SPAN, 4, 1},                                             \
                  reinterpret_cast<const void*>(&relax_win_kernel<16, SPAN, true, 256, MGB_WIN_MINB256, 256>));
#define WIN_P(P) \
  WIN_D(P, 1) WIN_D(P, 2) WIN_D(P, 3) WIN_D(P, 4) WIN_D(P, 5) WIN_D(P, 9) WIN_D(P, 16) WIN_D(P, 30)
void register_win_exact() {
  // n_x = 16384 (cfg5): 32 points per thread, 512 threads, generic single-buffer slice
  MGB_REG(K_WIN, 32, 1, 2, true);
  MGB_REG(K_WIN, 32, 9, 2, true);
  MGB_REG(K_WIN, 32, 30, 2, true);
  WIN_P(4)
  WIN_P(8)
  WIN_P(16)
  WIN_FIX(1) WIN_FIX(2) WIN_FIX(3) WIN_FIX(4) WIN_FIX(5) WIN_FIX(9) WIN_FIX(16) WIN_FIX(30)
}
}  // namespace mgb
