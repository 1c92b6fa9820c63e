// As dyn_f64_exact_p.cu, for ME-LMD-CIRBP.
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* dyn_f64_exact_q_get(int mode, int kind) {
  if (kind == KIND_ME_LMD_CIRBP) {
    switch (mode) {
      case 0: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 0, KIND_ME_LMD_CIRBP, 32, false, true>;
      case 1: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 1, KIND_ME_LMD_CIRBP, 32, false, true>;
      case 2: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 2, KIND_ME_LMD_CIRBP, 32, false, true>;
      case 3: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 3, KIND_ME_LMD_CIRBP, 32, false, true>;
    }
  }
  return nullptr;
}
