/*
 * ldpc_b200.h -- C ABI of the B200 dynamic-schedule LDPC decoder.
 *
 * Drop-in boundary for the reference's decode path.  The reference binds its
 * engine from Python as
 *   _engine._decode_<kind>(edge_cn, edge_vn, cn_ptr, vn_ptr, vn_edges, chl,
 *                          kernel, i_max, k_info, [gamma | simplified |
 *                          n_p, n_g, seed], c2v, v2c, pre_c2v, residual,
 *                          total, pre_total, ci, counters, biterr,
 *                          biterr_info, trace[, kappa_hits, kappa_trials])
 *   (/root/reference/pkg/src/ldpc_ids/_engine.py:355-765, argument packing at
 *    /root/reference/pkg/src/ldpc_ids/schedules.py:82-108, dispatch at
 *    schedules.py:111-158).
 * Here the graph arrays become an immutable device-resident handle
 * (ldpc_graph_create replaces the per-call CSR/CSC arguments, codes.py:251-275),
 * the per-frame float64 state arrays the caller allocated become a caller-sized
 * workspace, and one call decodes a whole batch of frames on a CUDA stream.
 *
 * All pointers passed to ldpc_decode are DEVICE pointers; ldpc_graph_create
 * takes HOST arrays.  No call synchronises the stream.  Return value 0 = ok,
 * negative = error (ldpc_strerror).
 */
#ifndef LDPC_B200_H
#define LDPC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes */
#define LDPC_OK 0
#define LDPC_ERR_INVALID (-1)     /* bad argument (mirrors the reference's ValueError) */
#define LDPC_ERR_UNSUPPORTED (-2) /* graph exceeds a kernel limit: dynamic schedules d_v <= 32, d_c <= 255 and \
                                     a two-hop set (+ d_v) below 65536; fixed schedules d_c <= one tile */
#define LDPC_ERR_CUDA (-3)        /* CUDA runtime error */
#define LDPC_ERR_WORKSPACE (-4)   /* workspace smaller than ldpc_workspace_size() */

/* schedule kinds: schedules.py:20-21 plus the two fixed/new schedules */
#define LDPC_FLOODING 0
#define LDPC_RBP 1
#define LDPC_CIRBP 2
#define LDPC_LMDRBP 3
#define LDPC_SLMDRBP 4
#define LDPC_LMD_CIRBP 5
#define LDPC_ME_CIRBP 6
#define LDPC_ME_LMD_CIRBP 7
#define LDPC_LAYERED 8
#define LDPC_ME_RBP 9

/* check-node kernels: kernels.py:20 */
#define LDPC_KERNEL_EXACT 0
#define LDPC_KERNEL_MINSUM 1

/* arithmetic of the message state */
#define LDPC_F64 0 /* reference precision (float64), default */
#define LDPC_F32 1 /* fast mode */

typedef struct ldpc_graph ldpc_graph_t;

/* ScheduleConfig (schedules.py:24-44) + launch options */
typedef struct {
  int32_t kind;           /* LDPC_FLOODING .. LDPC_ME_RBP */
  int32_t kernel;         /* LDPC_KERNEL_EXACT / LDPC_KERNEL_MINSUM */
  int32_t i_max;          /* update budget in iterations (i_max * E propagations) */
  int32_t n_p;            /* multi-edge: VNs (edges for ME-RBP) per round */
  int32_t n_g;            /* multi-edge: CI quantiser groups */
  int32_t k_info;         /* info positions for info_bit_errors (n < k_info) */
  double gamma;           /* CIRBP threshold */
  int64_t selection_seed; /* multi-edge RNG seed (int64 bit pattern) */
  int32_t precision;      /* LDPC_F64 / LDPC_F32 */
  int32_t llr_f64;        /* 0: llr is float32[B][N], 1: float64[B][N] */
  int32_t max_resident;   /* 0 = auto; else cap on concurrently decoded frames */
  int32_t placement;      /* dynamic schedules: 0 auto, 1 all state in HBM, 2 per-edge state in HBM,
                             3 all in shared memory, 4 per-edge + per-VN state in HBM (trees in smem) */
  int32_t want_trace;     /* 1: keep pre_total for every kind and allow ldpc_decode_traced outputs
                             (decode(..., want_trace=True), schedules.py:111-158) */
  int32_t variant;        /* 0 = the tuned engine choice; else LDPC_VARIANT_* bits (tests and
                             measurement: pin one engine so the alternatives can be compared) */
} ldpc_sched_t;

/* ldpc_sched_t.variant bits.  Flooding / layered engine (mask LDPC_VARIANT_FIXED_MASK): */
#define LDPC_VARIANT_FIXED_PHASE 0x1   /* batch-wide phase kernels */
#define LDPC_VARIANT_FIXED_TILE 0x2    /* one persistent CTA per 32-frame group */
#define LDPC_VARIANT_FIXED_PIPE 0x3    /* the tile engine with cp.async staging */
#define LDPC_VARIANT_FIXED_MASK 0x3
#define LDPC_VARIANT_CHECK_TMA 0x4     /* phase engine: TMA bulk-copy check kernel */
#define LDPC_VARIANT_CHECK_LEGACY 0x8  /* phase engine: load-wait-compute check kernel */
#define LDPC_VARIANT_NO_LAYERED_SIGN 0x10 /* layered: separate VN pass for sign words */
#define LDPC_VARIANT_LANES32 0x20      /* dynamic: 32 lanes per frame */
#define LDPC_VARIANT_LANES16 0x40      /* dynamic: 16 lanes per frame (2 frames per warp) */
#define LDPC_VARIANT_FULL_TREE 0x80    /* dynamic (debug): recompute every touched tree group */
#define LDPC_VARIANT_ME_PAIRS 0x100    /* multi-edge rounds: disjoint consecutive VN pairs on the two
                                          half-warps (exact; measured slower: the halves diverge) */

/* Build the device-resident Tanner graph (edge ids in (check, vn) order,
 * vn_edges = stable argsort of edge_vn).  Replaces build_tanner's arrays
 * (codes.py:251-275).  Host pointers in; the handle owns device copies. */
int ldpc_graph_create(const int32_t* edge_cn, const int32_t* edge_vn, const int32_t* cn_ptr,
                      const int32_t* vn_ptr, const int32_t* vn_edges, int32_t N, int32_t M,
                      int32_t E, ldpc_graph_t** out);
int ldpc_graph_destroy(ldpc_graph_t* g);

/* graph facts: out[0..6] = N, M, E, max_dv, max_dc, max_two_hop, layered levels */
int ldpc_graph_info(const ldpc_graph_t* g, int64_t* out7);

/* Bytes of device workspace ldpc_decode needs for this batch / schedule. */
int ldpc_workspace_size(const ldpc_graph_t* g, const ldpc_sched_t* s, int64_t B, size_t* bytes);

/* Decode B frames.  Device outputs (row-major, per frame):
 *   u_hat[B][N] int8 (total < 0, schedules.py:147), props[B] int64 (C2V
 *   propagations; iterations_used = props / E), converged[B] uint8,
 *   counters[B][8] int64 (order of _engine.py:17-25), biterr[B][i_max+1] and
 *   biterr_info[B][i_max+1] int32 (E:191-207), kappa_hits/kappa_trials
 *   [B][i_max] int32 (CIRBP only; may be NULL for other kinds). */
int ldpc_decode(const ldpc_graph_t* g, const void* llr, int64_t B, const ldpc_sched_t* s,
                int8_t* u_hat, int64_t* props, uint8_t* converged, int64_t* counters,
                int32_t* biterr, int32_t* biterr_info, int32_t* kappa_hits, int32_t* kappa_trials,
                void* workspace, size_t ws_bytes, void* cuda_stream);

/* ldpc_decode plus the reference's want_trace outputs (s->want_trace must be 1):
 *   trace[B][i_max+1][2N] float64 (may be NULL): per iteration boundary k the
 *   totals, then the pre-totals (E:192-217; flooding/layered: the next
 *   flooding pass's totals, E:768-782), rows after convergence repeated
 *   (E:211-217) -- DecodeResult.trace_llrs (schedules.py:57);
 *   j_counts[i_max+1][n_gamma][2] uint64 (may be NULL), ACCUMULATED (the
 *   caller zeroes it): VNs with D = |p0(total) - p0(pre_total)| >= gammas[gi]
 *   that are correct (total >= 0) / wrong, per boundary -- the counts
 *   sim._sim_block forms from the trace for mc_j_gamma (sim.py:172-183,
 *   339-353), fused so the trace need not be stored.  gammas: device float64. */
int ldpc_decode_traced(const ldpc_graph_t* g, const void* llr, int64_t B, const ldpc_sched_t* s,
                       int8_t* u_hat, int64_t* props, uint8_t* converged, int64_t* counters,
                       int32_t* biterr, int32_t* biterr_info, int32_t* kappa_hits, int32_t* kappa_trials,
                       double* trace, const double* gammas, int32_t n_gamma, uint64_t* j_counts,
                       void* workspace, size_t ws_bytes, void* cuda_stream);

/* Algorithm-4 VN selection (schedules.py:60-79, E:292-352) on the device:
 * ci[N] float64, mask[N] uint8 (NULL = all), out[n_p] int32; *count_dev gets
 * the number selected.  One warp; for API parity and tests. */
int ldpc_select_vns(const double* ci, const uint8_t* mask, int32_t N, int32_t n_g, int32_t n_p,
                    int64_t seed, int32_t* out, int32_t* count_dev, void* cuda_stream);

/* Debug / near-tie tracing: subsequent ldpc_decode calls on this thread write,
 * for each of the first `cap` updates k of frame f, the propagated edge to
 * dev_log[2 * (f * cap + k)] and the committed C2V value (float64 bits) to
 * dev_log[2 * (f * cap + k) + 1] (dynamic schedules only; the caller fills
 * the buffer with -1).  cap = 0 disables. */
int ldpc_set_step_log(int64_t* dev_log, int32_t cap);

/* Debug: subsequent dynamic-schedule decodes on this thread copy frame 0's
 * state right before update `step` into dev_buf (float64): ci[N] and
 * pre_total[N] at [0, 2N) (CI schedules), the RNG state after each Alg.-4
 * selection at [2N, 2N+8192), pre[E] and c2v[E] at [2N+8192, 2N+8192+2E).
 * step < 0 disables. */
int ldpc_set_state_dump(int64_t step, double* dev_buf);

/* On-GPU BPSK/AWGN frames (channel.py:35-86 conventions): out[B][N] (float32,
 * or float64 if out_f64) = clip(2y/sigma^2, +-30) with y = 1 + sigma*z for
 * the transmitted positions n >= n_punct_prefix and 0 for the punctured
 * prefix; frame f uses the counter-based stream keyed by (seed, start + f)
 * (Philox4x32-10 + Box-Muller; statistically equivalent to the host
 * generator, not bit-identical). */
int ldpc_generate_awgn(int32_t N, int32_t n_punct_prefix, int64_t B, double sigma, uint64_t seed,
                       int64_t start, void* out, int32_t out_f64, void* cuda_stream);

/* Number of kernel launches the last ldpc_decode on this thread issued. */
int ldpc_last_launch_count(void);

const char* ldpc_strerror(int code);
int ldpc_version(void);

/* Debug / audit: the GPU side of the reference's stepwise decoder state
 * (kernels.py:98-181, DecoderState.propagate / recompute_all; the survey's
 * ldpc_decode_replay).  Frame f is initialised like every schedule
 * (_init_state, E:106-127) and then propagates the GIVEN edge sequence
 * forced_edges[f][0..steps) (device int32) with pre_total and CI maintained
 * (DecoderState(maintain_ci=True)), instead of selecting edges.  Device outputs:
 *   c2v_trace[B][steps] float64: the C2V value each update commits (E:143);
 *   state_out[B][2E+3N] float64: c2v, pre_c2v, total, pre_total, ci after the
 *     last update (what recompute_all audits);
 *   counters[B][8] int64 (order of _engine.py:17-25).
 * s supplies kernel / precision / llr_f64 (kind and budget are ignored). */
int ldpc_replay_workspace_size(const ldpc_graph_t* g, const ldpc_sched_t* s, int64_t B, size_t* bytes);
int ldpc_decode_replay(const ldpc_graph_t* g, const void* llr, int64_t B, const ldpc_sched_t* s,
                       const int32_t* forced_edges, int32_t steps, double* c2v_trace, double* state_out,
                       int64_t* counters, void* workspace, size_t ws_bytes, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* LDPC_B200_H */
