// Dynamic-schedule kernels, float32 state (fast mode).
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* ldpc_dyn_kernel_f32(int kernel, int smem) {
  if (kernel == KERNEL_EXACT)
    return smem ? (void*)dyn_decode_kernel<float, KERNEL_EXACT, true> : (void*)dyn_decode_kernel<float, KERNEL_EXACT, false>;
  return smem ? (void*)dyn_decode_kernel<float, KERNEL_MINSUM, true> : (void*)dyn_decode_kernel<float, KERNEL_MINSUM, false>;
}
