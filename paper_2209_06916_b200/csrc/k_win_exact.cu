// Register-window stencil relaxation, exact (mul-then-add, canonical tap
// order: bitwise equal to the reference's rolled sums, circulant.py:119-123).
#include "mgb_registry.h"

namespace mgb {
#define WIN_P(P)                    \
  MGB_REG(K_WIN, P, 1, 1, true);  \
  MGB_REG(K_WIN, P, 2, 1, true);  \
  MGB_REG(K_WIN, P, 3, 1, true);  \
  MGB_REG(K_WIN, P, 4, 1, true);  \
  MGB_REG(K_WIN, P, 5, 1, true);  \
  MGB_REG(K_WIN, P, 9, 1, true);  \
  MGB_REG(K_WIN, P, 16, 1, true); \
  MGB_REG(K_WIN, P, 30, 1, true);
void register_win_exact() {
  WIN_P(4)
  WIN_P(8)
  WIN_P(16)
}
}  // namespace mgb
