// Register-window stencil relaxation, exact (mul-then-add, canonical tap
// order: bitwise equal to the reference's rolled sums, circulant.py:119-123).
#include "mgb_registry.h"

namespace mgb {
#define WIN_P(P)                    \
  register_kernel(KernelKey{K_WIN, P, 1, 1, 1}, reinterpret_cast<const void*>(&relax_win_kernel<P, 1, true>));  \
  register_kernel(KernelKey{K_WIN, P, 2, 1, 1}, reinterpret_cast<const void*>(&relax_win_kernel<P, 2, true>));  \
  register_kernel(KernelKey{K_WIN, P, 3, 1, 1}, reinterpret_cast<const void*>(&relax_win_kernel<P, 3, true>));  \
  register_kernel(KernelKey{K_WIN, P, 4, 1, 1}, reinterpret_cast<const void*>(&relax_win_kernel<P, 4, true>));  \
  register_kernel(KernelKey{K_WIN, P, 5, 1, 1}, reinterpret_cast<const void*>(&relax_win_kernel<P, 5, true>));  \
  register_kernel(KernelKey{K_WIN, P, 9, 1, 1}, reinterpret_cast<const void*>(&relax_win_kernel<P, 9, true>));  \
  MGB_REG(K_WIN, P, 1, 2, true);  \
  MGB_REG(K_WIN, P, 2, 2, true);  \
  MGB_REG(K_WIN, P, 3, 2, true);  \
  MGB_REG(K_WIN, P, 4, 2, true);  \
  MGB_REG(K_WIN, P, 5, 2, true);  \
  MGB_REG(K_WIN, P, 9, 2, true);  \
  MGB_REG(K_WIN, P, 16, 2, true);  \
  MGB_REG(K_WIN, P, 30, 2, true);
void register_win_exact() {
  // n_x = 16384 (cfg5): 32 points per thread, 512 threads, generic single-buffer slice
  MGB_REG(K_WIN, 32, 1, 2, true);
  MGB_REG(K_WIN, 32, 9, 2, true);
  MGB_REG(K_WIN, 32, 30, 2, true);
  WIN_P(4)
  WIN_P(8)
  WIN_P(16)
}
}  // namespace mgb
