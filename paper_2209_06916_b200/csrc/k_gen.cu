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
  GEN_P(1)
  GEN_P(2)
  GEN_P(4)
  GEN_P(8)
  GEN_P(16)
}
}  // namespace mgb
