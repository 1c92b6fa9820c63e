// Batch-wide phase kernels for flooding / layered (fixed_phase.cuh); the
// instantiations live in fixed_phase_f64.cu / fixed_phase_f32.cu.
#include "kernel_table.h"

PhaseKernels ldpc_phase_kernels(int f64, int kernel, int layered) {
  PhaseKernels k{};
  if (f64) ldpc_phase_fill_f64(k, kernel, layered);
  else ldpc_phase_fill_f32(k, kernel, layered);
  return k;
}
