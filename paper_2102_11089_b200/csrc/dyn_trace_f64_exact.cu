// Dynamic-schedule kernels with want_trace support (double state, KERNEL_EXACT): every
// kind dispatched at run time, pre_total kept for every kind, per-boundary
// trace rows and J(gamma) counts.  Separate from the per-kind production
// kernels so those carry none of this (measured: a runtime flag alone cost
// 5-20% on C1).
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* dyn_trace_f64_exact_get(int mode) {
  switch (mode) {
    case 0: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 0, -1, 32, true>;
    case 1: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 1, -1, 32, true>;
    case 2: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 2, -1, 32, true>;
    case 3: return (void*)dyn_decode_kernel<double, KERNEL_EXACT, 3, -1, 32, true>;
  }
  return nullptr;
}
