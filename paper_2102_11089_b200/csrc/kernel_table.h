// Kernel entry points compiled in separate translation units (parallel build).
#pragma once
void* ldpc_dyn_kernel_f64(int kernel, int smem);
void* ldpc_dyn_kernel_f32(int kernel, int smem);
void* ldpc_fixed_kernel(int f64, int kernel);
