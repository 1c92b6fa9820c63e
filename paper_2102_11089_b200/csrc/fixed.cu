// Flooding / layered kernels.
#include "fixed_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* ldpc_fixed_pipe_kernel(int f64, int kernel, int layered) {
  if (f64) {
    if (kernel == KERNEL_EXACT)
      return layered ? (void*)fixed_decode_kernel<double, KERNEL_EXACT, true, true> : (void*)fixed_decode_kernel<double, KERNEL_EXACT, false, true>;
    return layered ? (void*)fixed_decode_kernel<double, KERNEL_MINSUM, true, true> : (void*)fixed_decode_kernel<double, KERNEL_MINSUM, false, true>;
  }
  if (kernel == KERNEL_EXACT)
    return layered ? (void*)fixed_decode_kernel<float, KERNEL_EXACT, true, true> : (void*)fixed_decode_kernel<float, KERNEL_EXACT, false, true>;
  return layered ? (void*)fixed_decode_kernel<float, KERNEL_MINSUM, true, true> : (void*)fixed_decode_kernel<float, KERNEL_MINSUM, false, true>;
}
void* ldpc_fixed_kernel(int f64, int kernel, int layered) {
  if (f64) {
    if (kernel == KERNEL_EXACT)
      return layered ? (void*)fixed_decode_kernel<double, KERNEL_EXACT, true> : (void*)fixed_decode_kernel<double, KERNEL_EXACT, false>;
    return layered ? (void*)fixed_decode_kernel<double, KERNEL_MINSUM, true> : (void*)fixed_decode_kernel<double, KERNEL_MINSUM, false>;
  }
  if (kernel == KERNEL_EXACT)
    return layered ? (void*)fixed_decode_kernel<float, KERNEL_EXACT, true> : (void*)fixed_decode_kernel<float, KERNEL_EXACT, false>;
  return layered ? (void*)fixed_decode_kernel<float, KERNEL_MINSUM, true> : (void*)fixed_decode_kernel<float, KERNEL_MINSUM, false>;
}
