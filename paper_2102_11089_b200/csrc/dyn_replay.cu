// Replay kernels (debug / audit; dyn_engine.cuh dyn_replay_kernel): float64 and
// float32 state, exact and min-sum check nodes.
#include "dyn_engine.cuh"
#include "kernel_table.h"
using namespace ldpc;
void* ldpc_replay_kernel(int f64, int kernel) {
  if (f64) return kernel == KERNEL_EXACT ? (void*)dyn_replay_kernel<double, KERNEL_EXACT>
                                         : (void*)dyn_replay_kernel<double, KERNEL_MINSUM>;
  return kernel == KERNEL_EXACT ? (void*)dyn_replay_kernel<float, KERNEL_EXACT>
                                : (void*)dyn_replay_kernel<float, KERNEL_MINSUM>;
}
