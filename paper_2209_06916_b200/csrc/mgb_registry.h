// mgb_registry.h -- kernel instantiation registry shared by the kernel TUs.
#pragma once
#include "mgb_device.cuh"

namespace mgb {

using RelaxFn = void (*)(const StepParams*, const RelaxLaunch);

struct KernelKey {
  int kind, P, span, nst, exact;
};

void register_kernel(const KernelKey& key, const void* fn);

void register_win_exact();
void register_win_fast();
void register_gen();
void register_rk();
void register_slgc();
void register_slgc1();

// window spans with a compiled register-window variant
constexpr int kWinSpans[] = {1, 2, 3, 4, 5, 9, 16, 30};

}  // namespace mgb

#define MGB_REG(KIND, P, SPAN, NST, EXACT)                                                     \
  ::mgb::register_kernel(::mgb::KernelKey{KIND, P, SPAN, NST, EXACT},                          \
                         reinterpret_cast<const void*>(&::mgb::relax_kernel<P, KIND, SPAN, NST, EXACT>))
