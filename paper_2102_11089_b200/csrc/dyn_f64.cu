// Dynamic-schedule kernels, float64 state (reference precision).
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* ldpc_dyn_kernel_f64(int kernel, int smem) {
  if (kernel == KERNEL_EXACT)
    return smem ? (void*)dyn_decode_kernel<double, KERNEL_EXACT, true> : (void*)dyn_decode_kernel<double, KERNEL_EXACT, false>;
  return smem ? (void*)dyn_decode_kernel<double, KERNEL_MINSUM, true> : (void*)dyn_decode_kernel<double, KERNEL_MINSUM, false>;
}
