// Dynamic-schedule kernels: double state, KERNEL_EXACT; instantiated per (placement mode, kind).
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* dyn_f64_exact_b_get(int mode, int kind) {
  if (kind == KIND_LMDRBP || KIND_LMDRBP < 0) switch (mode) {
      case 0: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 0, KIND_LMDRBP>;
      case 1: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 1, KIND_LMDRBP>;
      case 2: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 2, KIND_LMDRBP>;
      case 3: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 3, KIND_LMDRBP>;
    }
  if (kind == KIND_LMD_CIRBP || KIND_LMD_CIRBP < 0) switch (mode) {
      case 0: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 0, KIND_LMD_CIRBP>;
      case 1: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 1, KIND_LMD_CIRBP>;
      case 2: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 2, KIND_LMD_CIRBP>;
      case 3: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 3, KIND_LMD_CIRBP>;
    }
  return nullptr;
}
