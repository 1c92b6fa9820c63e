// Dynamic-schedule kernels: double state, KERNEL_EXACT; instantiated per (placement mode, kind).
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* dyn_f64_exact_a_get(int mode, int kind) {
  if (kind == KIND_RBP || KIND_RBP < 0) switch (mode) {
      case 0: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 0, KIND_RBP>;
      case 1: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 1, KIND_RBP>;
      case 2: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 2, KIND_RBP>;
      case 3: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 3, KIND_RBP>;
    }
  if (kind == KIND_CIRBP || KIND_CIRBP < 0) switch (mode) {
      case 0: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 0, KIND_CIRBP>;
      case 1: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 1, KIND_CIRBP>;
      case 2: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 2, KIND_CIRBP>;
      case 3: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 3, KIND_CIRBP>;
    }
  return nullptr;
}
