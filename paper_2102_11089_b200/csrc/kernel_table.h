// Kernel entry points compiled in separate translation units (parallel build).
#pragma once
#include "ldpc_common.cuh"
void* dyn_f64_exact_a_get(int mode, int kind);
void* dyn_f64_exact_b_get(int mode, int kind);
void* dyn_f64_exact_c_get(int mode, int kind);
void* dyn_f64_exact_d_get(int mode, int kind);
void* dyn_f64_minsum_get(int mode, int kind);
void* dyn_f32_exact_get(int mode, int kind);
void* dyn_f32_minsum_get(int mode, int kind);
// float64 + exact kernels are specialised per schedule kind (sLMDRBP runs the
// LMDRBP kernel); the other variants dispatch on the kind at run time.
inline void* ldpc_dyn_kernel(int f64, int kernel, int mode, int kind) {
  using namespace ldpc;
  if (!f64) return kernel == KERNEL_EXACT ? dyn_f32_exact_get(mode, -1) : dyn_f32_minsum_get(mode, -1);
  if (kernel != KERNEL_EXACT) return dyn_f64_minsum_get(mode, -1);
  switch (kind) {
    case KIND_RBP: case KIND_CIRBP: return dyn_f64_exact_a_get(mode, kind);
    case KIND_LMDRBP: case KIND_SLMDRBP: return dyn_f64_exact_b_get(mode, KIND_LMDRBP);
    case KIND_LMD_CIRBP: return dyn_f64_exact_b_get(mode, kind);
    case KIND_ME_CIRBP: case KIND_ME_LMD_CIRBP: return dyn_f64_exact_c_get(mode, kind);
    default: return dyn_f64_exact_d_get(mode, kind);
  }
}
void* ldpc_fixed_kernel(int f64, int kernel, int layered);
