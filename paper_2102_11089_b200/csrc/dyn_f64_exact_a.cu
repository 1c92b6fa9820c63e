// Dynamic-schedule kernels: double state, KERNEL_EXACT; per (placement mode, kind, lanes per frame).
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* dyn_f64_exact_a_get(int mode, int kind, int g16) {
  if (kind == KIND_RBP) {
    if (g16) return nullptr;  // 16-lane groups measured slower (halves diverge); not built
    switch (mode) {
      case 0: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 0, KIND_RBP, 32>;
      case 1: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 1, KIND_RBP, 32>;
      case 2: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 2, KIND_RBP, 32>;
      case 3: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 3, KIND_RBP, 32>;
    }
  }
  return nullptr;
}
