// Flooding / layered kernels.
#include "fixed_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* ldpc_fixed_kernel(int f64, int kernel) {
  if (f64) return kernel == KERNEL_EXACT ? (void*)fixed_decode_kernel<double, KERNEL_EXACT> : (void*)fixed_decode_kernel<double, KERNEL_MINSUM>;
  return kernel == KERNEL_EXACT ? (void*)fixed_decode_kernel<float, KERNEL_EXACT> : (void*)fixed_decode_kernel<float, KERNEL_MINSUM>;
}
