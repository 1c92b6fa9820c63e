// float64 phase kernels (built with -fmad=false: the reference's rounding).
#include "fixed_phase_impl.cuh"
void ldpc_phase_fill_f64(PhaseKernels& k, int kernel, int layered) { ldpc_phase_fill<double, 16>(k, kernel, layered); }
