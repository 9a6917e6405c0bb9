// Register-window stencil relaxation, fast mode (DFMA).
#include "mgb_registry.h"

namespace mgb {
#define WIN_P(P)                     \
  register_kernel(KernelKey{K_WIN, P, 1, 1, 0}, reinterpret_cast<const void*>(&relax_win_kernel<P, 1, false>));  \
  register_kernel(KernelKey{K_WIN, P, 2, 1, 0}, reinterpret_cast<const void*>(&relax_win_kernel<P, 2, false>));  \
  register_kernel(KernelKey{K_WIN, P, 3, 1, 0}, reinterpret_cast<const void*>(&relax_win_kernel<P, 3, false>));  \
  register_kernel(KernelKey{K_WIN, P, 4, 1, 0}, reinterpret_cast<const void*>(&relax_win_kernel<P, 4, false>));  \
  register_kernel(KernelKey{K_WIN, P, 5, 1, 0}, reinterpret_cast<const void*>(&relax_win_kernel<P, 5, false>));  \
  register_kernel(KernelKey{K_WIN, P, 9, 1, 0}, reinterpret_cast<const void*>(&relax_win_kernel<P, 9, false>));  \
  MGB_REG(K_WIN, P, 1, 2, false);  \
  MGB_REG(K_WIN, P, 2, 2, false);  \
  MGB_REG(K_WIN, P, 3, 2, false);  \
  MGB_REG(K_WIN, P, 4, 2, false);  \
  MGB_REG(K_WIN, P, 5, 2, false);  \
  MGB_REG(K_WIN, P, 9, 2, false);  \
  MGB_REG(K_WIN, P, 16, 2, false);  \
  MGB_REG(K_WIN, P, 30, 2, false);
void register_win_fast() {
  MGB_REG(K_WIN, 32, 1, 2, false);
  MGB_REG(K_WIN, 32, 9, 2, false);
  MGB_REG(K_WIN, 32, 30, 2, false);
  WIN_P(4)
  WIN_P(8)
  WIN_P(16)
}
}  // namespace mgb
