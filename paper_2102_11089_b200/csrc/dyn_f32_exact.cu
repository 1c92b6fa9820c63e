// Dynamic-schedule kernels: float state, KERNEL_EXACT; instantiated per (placement mode, kind).
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* dyn_f32_exact_get(int mode, int kind) {
  (void)kind;
  switch (mode) {
      case 0: return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 0, -1>;
      case 1: return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 1, -1>;
      case 2: return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 2, -1>;
      case 3: return (void*)dyn_decode_kernel<float, KERNEL_EXACT, 3, -1>;
    }
  return nullptr;
}
