// Instantiation of the batch-wide phase kernels for one element type (included
// by fixed_phase_f64.cu / fixed_phase_f32.cu, which differ in FMA contraction:
// float64 must round like the reference, float32 has no bit-order obligation).
#pragma once
#include "fixed_phase.cuh"
#include "kernel_table.h"

template <typename T, int KERNEL, int NC>
static void* tma_check_of(int layered) {
  using namespace ldpc;
  return layered ? (void*)phase_check_tma_kernel<T, KERNEL, true, NC, false>
                 : (void*)phase_check_tma_kernel<T, KERNEL, false, NC, false>;
}

// NC0: consumer-warp count built for this type
template <typename T, int NC0>
static void ldpc_phase_fill(PhaseKernels& k, int kernel, int layered) {
  using namespace ldpc;
  k.init = (void*)phase_init_kernel<T>;
  if (kernel == KERNEL_EXACT) {
    k.check = layered ? (void*)phase_check_kernel<T, KERNEL_EXACT, true> : (void*)phase_check_kernel<T, KERNEL_EXACT, false>;
    k.check_tma = tma_check_of<T, KERNEL_EXACT, NC0>(layered);
  } else {
    k.check = layered ? (void*)phase_check_kernel<T, KERNEL_MINSUM, true> : (void*)phase_check_kernel<T, KERNEL_MINSUM, false>;
    k.check_tma = tma_check_of<T, KERNEL_MINSUM, NC0>(layered);
  }
  k.vn = layered ? (void*)phase_vn_kernel<T, true> : (void*)phase_vn_kernel<T, false>;
  k.syndrome = (void*)phase_syndrome_kernel;
  k.finalize = (void*)phase_finalize_kernel;
  k.output = (void*)phase_output_kernel<T>;
  k.tma_threads = TmaLayout<T, NC0>::kThreads;
  k.tma_smem = TmaLayout<T, NC0>::kBytes;
  k.vn_tma = (void*)phase_vn_tma_kernel<T, 8>;
  // layered: the FUSED build (level map + publication; spill-free), one level per launch
  k.check_tma_fused = kernel == KERNEL_EXACT ? (void*)phase_check_tma_kernel<T, KERNEL_EXACT, true, NC0, true>
                                             : (void*)phase_check_tma_kernel<T, KERNEL_MINSUM, true, NC0, true>;
  k.vn_threads = VnLayout<T, 8>::kThreads;
  k.vn_smem = VnLayout<T, 8>::kBytes;
}
