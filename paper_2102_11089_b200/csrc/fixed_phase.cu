// Batch-wide phase kernels for flooding / layered (fixed_phase.cuh).
#include "fixed_phase.cuh"
#include "kernel_table.h"
using namespace ldpc;

template <typename T>
static void fill(PhaseKernels& k, int kernel, int layered) {
  k.init = (void*)phase_init_kernel<T>;
  if (kernel == KERNEL_EXACT)
    k.check = layered ? (void*)phase_check_kernel<T, KERNEL_EXACT, true> : (void*)phase_check_kernel<T, KERNEL_EXACT, false>;
  else
    k.check = layered ? (void*)phase_check_kernel<T, KERNEL_MINSUM, true> : (void*)phase_check_kernel<T, KERNEL_MINSUM, false>;
  k.vn = layered ? (void*)phase_vn_kernel<T, true> : (void*)phase_vn_kernel<T, false>;
  k.syndrome = (void*)phase_syndrome_kernel;
  k.finalize = (void*)phase_finalize_kernel;
  k.output = (void*)phase_output_kernel<T>;
}

PhaseKernels ldpc_phase_kernels(int f64, int kernel, int layered) {
  PhaseKernels k{};
  if (f64) fill<double>(k, kernel, layered);
  else fill<float>(k, kernel, layered);
  return k;
}
