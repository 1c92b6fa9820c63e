// Dynamic-schedule kernels: float state, KERNEL_MINSUM; per (placement mode, kind, lanes per frame).
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* dyn_f32_minsum_get(int mode, int kind, int g16) {
  (void)kind; {
    if (g16) return nullptr;  // 16-lane groups measured slower (halves diverge); not built
    switch (mode) {
      case 0: return (void*)dyn_decode_kernel<float, KERNEL_MINSUM, 0, -1, 32>;
      case 1: return (void*)dyn_decode_kernel<float, KERNEL_MINSUM, 1, -1, 32>;
      case 2: return (void*)dyn_decode_kernel<float, KERNEL_MINSUM, 2, -1, 32>;
      case 3: return (void*)dyn_decode_kernel<float, KERNEL_MINSUM, 3, -1, 32>;
    }
  }
  return nullptr;
}
