// Kernel entry points compiled in separate translation units (parallel build).
#pragma once
#include "ldpc_common.cuh"
void* dyn_f64_exact_a_get(int mode, int kind, int g16);
void* dyn_f64_exact_b_get(int mode, int kind, int g16);
void* dyn_f64_exact_c_get(int mode, int kind, int g16);
void* dyn_f64_exact_d_get(int mode, int kind, int g16);
void* dyn_f64_exact_e_get(int mode, int kind, int g16);
void* dyn_f64_exact_p_get(int mode, int kind);  // multi-edge kinds built with round pairing
void* dyn_f64_exact_q_get(int mode, int kind);
void* dyn_f64_minsum_get(int mode, int kind, int g16);
void* dyn_f32_exact_get(int mode, int kind, int g16);
void* dyn_f32_exact_k_get(int mode, int kind);  // per-kind float builds (RBP, CIRBP, ME-CIRBP; modes 2, 3)
void* dyn_f32_minsum_get(int mode, int kind, int g16);
void* dyn_trace_f64_exact_get(int mode);
void* dyn_trace_f64_minsum_get(int mode);
void* dyn_trace_f32_exact_get(int mode);
void* dyn_trace_f32_minsum_get(int mode);
// float64 + exact kernels are specialised per schedule kind (sLMDRBP runs the
// LMDRBP kernel); the other variants dispatch on the kind at run time.
// g16: 16 lanes per frame (two frames per warp; placement modes 1-3 only).
// trace: the want_trace build (dyn_trace_*.cu), 32 lanes, kind at run time.
inline void* ldpc_dyn_kernel(int f64, int kernel, int mode, int kind, int g16, int trace = 0, int pairs = 0) {
  using namespace ldpc;
  if (pairs) {  // round-pairing build: float64 exact multi-edge CI kinds, 32 lanes, untraced
    if (trace || g16 || !f64 || kernel != KERNEL_EXACT) return nullptr;
    return kind == KIND_ME_CIRBP ? dyn_f64_exact_p_get(mode, kind)
                                 : kind == KIND_ME_LMD_CIRBP ? dyn_f64_exact_q_get(mode, kind) : nullptr;
  }
  if (trace) {
    if (g16) return nullptr;
    if (f64) return kernel == KERNEL_EXACT ? dyn_trace_f64_exact_get(mode) : dyn_trace_f64_minsum_get(mode);
    return kernel == KERNEL_EXACT ? dyn_trace_f32_exact_get(mode) : dyn_trace_f32_minsum_get(mode);
  }
  if (g16 && mode == 0) return nullptr;
  if (!f64 && kernel == KERNEL_EXACT && !g16)
    if (void* k = dyn_f32_exact_k_get(mode, kind)) return k;
  if (!f64) return kernel == KERNEL_EXACT ? dyn_f32_exact_get(mode, -1, g16) : dyn_f32_minsum_get(mode, -1, g16);
  if (kernel != KERNEL_EXACT) return dyn_f64_minsum_get(mode, -1, g16);
  switch (kind) {
    case KIND_RBP: return dyn_f64_exact_a_get(mode, kind, g16);
    case KIND_CIRBP: return dyn_f64_exact_b_get(mode, kind, g16);
    case KIND_LMDRBP: case KIND_SLMDRBP: return dyn_f64_exact_c_get(mode, KIND_LMDRBP, g16);
    case KIND_LMD_CIRBP: return dyn_f64_exact_c_get(mode, kind, g16);
    case KIND_ME_CIRBP: case KIND_ME_LMD_CIRBP: return dyn_f64_exact_d_get(mode, kind, g16);
    default: return dyn_f64_exact_e_get(mode, kind, g16);
  }
}
void* ldpc_fixed_kernel(int f64, int kernel, int layered);
void* ldpc_fixed_pipe_kernel(int f64, int kernel, int layered);  // cp.async-pipelined check phase

namespace ldpc {
// traced flooding / layered decode (fixed_trace.cu): one warp per frame
constexpr int kTraceWarps = 8;
struct FixedTraceParams {
  DevGraph g;
  int i_max, k_info;
  const void* llr;
  int llr_f64;
  long long B;
  int8_t* u_hat;
  long long* prop;
  uint8_t* conv;
  long long* counters;
  int* biterr;
  int* biterr_info;
  unsigned long long* next;
  unsigned char* ws;
  long long slot_bytes;
  TraceOut tr;
};
}  // namespace ldpc
void* ldpc_fixed_trace_kernel(int f64, int kernel, int layered);
void* ldpc_replay_kernel(int f64, int kernel);  // dyn_replay.cu

// batch-wide phase kernels for flooding / layered (fixed_phase.cu)
struct PhaseKernels {
  void *init, *check, *vn, *syndrome, *finalize, *output;
  void* check_tma;           // warp-specialised TMA-fed check phase (fixed_tma.cuh)
  void* check_tma_fused;     // same, layered levels in one launch (dependency counters)
  int tma_threads, tma_smem;
  void* vn_tma;              // TMA-fed VN phase over VN strips (flooding)
  int vn_threads, vn_smem;
};
PhaseKernels ldpc_phase_kernels(int f64, int kernel, int layered);
void ldpc_phase_fill_f64(PhaseKernels& k, int kernel, int layered);  // fixed_phase_f64.cu
void ldpc_phase_fill_f32(PhaseKernels& k, int kernel, int layered);  // fixed_phase_f32.cu
