// float32 phase kernels (built with -fmad=true: no bit-order obligation in fp32).
#include "fixed_phase_impl.cuh"
void ldpc_phase_fill_f32(PhaseKernels& k, int kernel, int layered) { ldpc_phase_fill<float, 8>(k, kernel, layered); }
