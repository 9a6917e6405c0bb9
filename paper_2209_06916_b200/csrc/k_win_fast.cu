// Register-window stencil relaxation, fast mode (DFMA).
#include "mgb_registry.h"

namespace mgb {
#define WIN_P(P)                     \
  MGB_REG(K_WIN, P, 1, 1, false);  \
  MGB_REG(K_WIN, P, 2, 1, false);  \
  MGB_REG(K_WIN, P, 3, 1, false);  \
  MGB_REG(K_WIN, P, 4, 1, false);  \
  MGB_REG(K_WIN, P, 5, 1, false);  \
  MGB_REG(K_WIN, P, 9, 1, false);  \
  MGB_REG(K_WIN, P, 16, 1, false); \
  MGB_REG(K_WIN, P, 30, 1, false);
void register_win_fast() {
  WIN_P(4)
  WIN_P(8)
  WIN_P(16)
}
}  // namespace mgb
