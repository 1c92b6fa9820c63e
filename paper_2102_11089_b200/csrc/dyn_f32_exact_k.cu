// Dynamic-schedule kernels: float state, KERNEL_EXACT, specialised per kind for
// the schedules BASELINE.json runs on the BG-sized codes (RBP, CIRBP, ME-CIRBP)
// in the HBM placements: the run-time-kind build (dyn_f32_exact.cu) is ~1 MB
// of code per kernel, far beyond the instruction caches.
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* dyn_f32_exact_k_get(int mode, int kind) {
  switch (kind) {
    case KIND_RBP:
      if (mode == 2) return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 2, KIND_RBP, 32>;
      if (mode == 3) return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 3, KIND_RBP, 32>;
      break;
    case KIND_CIRBP:
      if (mode == 2) return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 2, KIND_CIRBP, 32>;
      if (mode == 3) return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 3, KIND_CIRBP, 32>;
      break;
    case KIND_ME_CIRBP:
      if (mode == 2) return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 2, KIND_ME_CIRBP, 32>;
      if (mode == 3) return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 3, KIND_ME_CIRBP, 32>;
      break;
  }
  return nullptr;
}
