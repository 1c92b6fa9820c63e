// fixed_phase.cuh -- flooding / row-layered BP as batch-wide phases.
//
// Same arithmetic and layout as fixed_engine.cuh (32-frame groups, rows of
// [item][32 frames], whole-check tiles, ordered products and sums), but the
// work is cut differently: every phase of an iteration is its own grid over
// (frame group, tile) items --
//   check phase  (flooding: one launch; layered: one launch per dependency
//                 level, E:741-745 / oracle decode_layered),
//   VN phase     (totals, sign words, error tallies; E:746-756),
//   syndrome     (parity of the sign words, E:179-188),
//   finalize     (boundary rows, convergence, E:191-217 / E:761-764),
// so all groups of the batch stream through HBM together and a batch that is
// not a multiple of the resident-CTA count has no tail wave (the per-group
// persistent kernel ran 10,000 BG1 frames in two waves of 296 and 17 groups).
// Each item issues all of its row loads before using any, so a CTA keeps a
// whole tile (up to 2 x 128 rows of 128 or 256 bytes) in flight.
#pragma once
#include "fixed_engine.cuh"

namespace ldpc {

constexpr int kPhaseThreads = 256;
constexpr int kPhaseVnChunk = 64;    // VNs per VN-phase item
constexpr int kPhaseChkChunk = 512;  // checks per syndrome item

struct PhaseParams {
  DevGraph g;
  int kernel, i_max, k_info;
  const void* llr;
  int llr_f64;
  long long B;         // frames of this chunk
  long long f_base;    // first frame of this chunk in the caller's arrays
  int groups;          // ceil(B / 32)
  int8_t* u_hat;
  long long* prop;
  uint8_t* conv;
  long long* counters;
  int* biterr;
  int* biterr_info;
  unsigned char* ws;   // per group: chl[N][32], total[N][32], c2v[E][32], sign[N]
  long long slot_bytes;
  long long sign_off;  // byte offset of sign[] in a slot
  unsigned* amask;     // [groups] frames still decoding
  unsigned* unsat;     // [groups] frames with an unsatisfied check at this boundary
  int* errs;           // [groups][32] bit errors at this boundary
  int* errs_info;      // [groups][32]
  int* iters;          // [groups][32] iterations used
  // tiling (fixed_engine.cuh)
  const int* level_tptr;
  const int* tile_eptr;
  const int* te_list;
  const int* te_vn;
  const int2* te_chk;
  const int* tile_cptr;
  const int4* tc_rec;
  // strips (fixed_tma.cuh): s_rec[t] = (first c2v row, k checks, degree d, first run),
  // s_runs = (first VN, staged row | length << 8), s_vn = VN of each staged row
  const int4* s_rec;
  const int2* s_runs;
  const int* s_vn;
  const int* vn_rows;  // [E] c2v row of each vn_edges slot (VN phase)
  // VN strips (flooding VN phase, fixed_tma.cuh): v_rec[t] = (first VN, k, degree, first run),
  // v_runs = (first stored c2v row, staged row | length << 8)
  const int4* v_rec;
  const int2* v_runs;
  int n_vstrips;
  const int* s_lvl;  // [levels + 1] first strip of each level (check strips)
  int layered_sign;  // layered: sign words / error tallies from the check phase (no VN pass)
  int vn_reverse;    // flooding VN phase in reverse group order
  int lwin;          // layered, levels fused: groups per window (0 = all groups)
  int* done;         // [groups] committed check strips per group (layered, levels fused in one launch)
};

#ifndef LDPC_PHASE_DECL_ONLY  // the host launcher only needs PhaseParams

template <typename T>
struct GroupSlot {
  T *chl, *total, *c2v;
  unsigned* sign;
  __device__ GroupSlot(const PhaseParams& p, long long grp) {
    chl = (T*)(p.ws + grp * p.slot_bytes);
    total = chl + (long long)p.g.N * kFixedFrames;
    c2v = total + (long long)p.g.N * kFixedFrames;
    sign = (unsigned*)(p.ws + grp * p.slot_bytes + p.sign_off);
  }
};

// LLRs in (transposed to [N][32]), total = chl, c2v = 0, boundary-0 tallies.
template <typename T>
__global__ void __launch_bounds__(kPhaseThreads) phase_init_kernel(const __grid_constant__ PhaseParams p) {
  constexpr int F = kFixedFrames;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int vchunks = (p.g.N + kPhaseVnChunk - 1) / kPhaseVnChunk;
  const int echunks = (int)(((long long)p.g.E + kPhaseVnChunk * 8 - 1) / (kPhaseVnChunk * 8));
  const long long items = (long long)p.groups * (vchunks + echunks);
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const long long grp = it / (vchunks + echunks);
    const int c = (int)(it - grp * (vchunks + echunks));
    GroupSlot<T> s(p, grp);
    const long long f = grp * F + lane;
    const bool valid = f < p.B;
    if (c == 0 && warp == 0) {
      const unsigned vm = __ballot_sync(kFull, valid);
      if (lane == 0) {
        p.amask[grp] = vm;
        p.unsat[grp] = 0u;
      }
    }
    if (c < vchunks) {
      int errs = 0, ei = 0;
      const int n1 = min(p.g.N, (c + 1) * kPhaseVnChunk);
      for (int n = c * kPhaseVnChunk + warp; n < n1; n += nw) {
        T v = T(0);
        if (valid) {
          const long long x = (p.f_base + f) * p.g.N + n;
          v = p.llr_f64 ? (T)((const double*)p.llr)[x] : (T)((const float*)p.llr)[x];
        }
        s.chl[(long long)n * F + lane] = v;
        s.total[(long long)n * F + lane] = v;
        sign_row<T>(n, v, p.k_info, s.sign, lane, errs, ei);
      }
      if (errs) atomicAdd(&p.errs[grp * F + lane], errs);
      if (ei) atomicAdd(&p.errs_info[grp * F + lane], ei);
    } else {
      const long long e0 = (long long)(c - vchunks) * kPhaseVnChunk * 8 * F;
      const long long e1 = min((long long)p.g.E * F, e0 + (long long)kPhaseVnChunk * 8 * F);
      for (long long x = e0 + threadIdx.x; x < e1; x += blockDim.x) s.c2v[x] = T(0);
    }
  }
}

// Check phase over the tiles [t_lo, t_hi) of one level, every active group.
template <typename T, int KERNEL, bool LAYERED>
__global__ void __launch_bounds__(kPhaseThreads) phase_check_kernel(const __grid_constant__ PhaseParams p, int t_lo,
                                                                     int t_hi) {
  constexpr int F = kFixedFrames;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  extern __shared__ __align__(16) unsigned char phase_smem[];
  T* in_s = (T*)phase_smem;        // [kTileEdges][32]
  T* so = in_s + kTileEdges * F;   // c2v rows
  T* st = so + kTileEdges * F;     // total rows
  const int nti = t_hi - t_lo;
  const long long items = (long long)p.groups * nti;
  constexpr int CH = F * (int)sizeof(T) / 16;  // 16-byte chunks per row
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const long long grp = it / nti;
    const int t = t_lo + (int)(it - grp * nti);
    const unsigned am = p.amask[grp];
    if (!am) continue;  // uniform over the CTA
    GroupSlot<T> s(p, grp);
    const int ea = p.tile_eptr[t], ne = p.tile_eptr[t + 1] - ea;
    // all row loads of the tile in flight at once
    for (int x = tid; x < 2 * ne * CH; x += nt) {
      const int r = x / CH, ch = x - r * CH;
      const int el = r < ne ? r : r - ne;
      const T* src = r < ne ? s.c2v + (long long)(ea + el) * F : s.total + (long long)p.te_vn[ea + el] * F;
      cp_async16((r < ne ? so : st) + el * F + ch * (16 / (int)sizeof(T)), src + ch * (16 / (int)sizeof(T)));
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int x = tid; x < ne * F; x += nt) {  // phase A: check inputs (E:58 / E:73)
      const T v = clampv(st[x] - so[x]);
      in_s[x] = (KERNEL == KERNEL_EXACT) ? cn_in<T>(v) : v;
    }
    __syncthreads();
    const bool act = (am >> lane) & 1u;
    if (sizeof(T) == 4) {  // one warp per check
      for (int ck = p.tile_cptr[t] + warp; ck < p.tile_cptr[t + 1]; ck += nw)
        check_outputs<T, KERNEL, LAYERED>(p.te_vn, in_s, so, p.tc_rec[ck], lane, act, s.c2v, s.total, st);
    } else {  // float64: one warp per edge, the reference's product order
      for (int el = warp; el < ne; el += nw) {
        const T out = tile_out<T, KERNEL>(in_s, p.te_chk[ea + el], el, lane);
        if (act) {
          s.c2v[(long long)(ea + el) * F + lane] = out;  // c2v rows in tile order
          if (LAYERED) s.total[(long long)p.te_vn[ea + el] * F + lane] = st[el * F + lane] + (out - so[el * F + lane]);
        }
      }
    }
    __syncthreads();
  }
}

// VN phase: flooding totals (ordered sums, E:749-750), sign words, error tallies.
template <typename T, bool LAYERED>
__global__ void __launch_bounds__(kPhaseThreads) phase_vn_kernel(const __grid_constant__ PhaseParams p) {
  constexpr int F = kFixedFrames;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const DevGraph& g = p.g;
  const int vchunks = (g.N + kPhaseVnChunk - 1) / kPhaseVnChunk;
  const long long items = (long long)p.groups * vchunks;
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const long long grp = it / vchunks;
    const int c = (int)(it - grp * vchunks);
    const unsigned am = p.amask[grp];
    if (!am) continue;
    GroupSlot<T> s(p, grp);
    const bool act = (am >> lane) & 1u;
    int errs = 0, ei = 0;
    const int n1 = min(g.N, (c + 1) * kPhaseVnChunk);
    for (int n = c * kPhaseVnChunk + warp; n < n1; n += nw) {
      const long long nx = (long long)n * F + lane;
      T v;
      if (!LAYERED && act) {
        v = s.chl[nx];
        const int k0 = g.vn_ptr[n], k1 = g.vn_ptr[n + 1];
        for (int k = k0; k < k1; k += 8) {  // 8 rows in flight, summed in order
          T r[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (k + u < k1) r[u] = s.c2v[(long long)p.vn_rows[k + u] * F + lane];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (k + u < k1) v += r[u];
        }
        s.total[nx] = v;
      } else {
        v = s.total[nx];
      }
      int e_ = 0, i_ = 0;
      sign_row<T>(n, v, p.k_info, s.sign, lane, e_, i_);
      if (act) {
        errs += e_;
        ei += i_;
      }
    }
    if (errs) atomicAdd(&p.errs[grp * F + lane], errs);
    if (ei) atomicAdd(&p.errs_info[grp * F + lane], ei);
  }
}

// Parity of every check from the sign words, 32 frames per word (E:179-188).
static __global__ void __launch_bounds__(kPhaseThreads) phase_syndrome_kernel(const __grid_constant__ PhaseParams p) {
  const DevGraph& g = p.g;
  const int cchunks = (g.M + kPhaseChkChunk - 1) / kPhaseChkChunk;
  const long long items = (long long)p.groups * cchunks;
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const long long grp = it / cchunks;
    const int c = (int)(it - grp * cchunks);
    const unsigned am = p.amask[grp];
    if (!am) continue;
    const unsigned* sg = (const unsigned*)(p.ws + grp * p.slot_bytes + p.sign_off);
    unsigned bad = 0;
    const int m1 = min(g.M, (c + 1) * kPhaseChkChunk);
    for (int m = c * kPhaseChkChunk + threadIdx.x; m < m1; m += blockDim.x) {
      unsigned par = 0;
      for (int e = g.cn_ptr[m]; e < g.cn_ptr[m + 1]; ++e) par ^= sg[g.edge_vn[e]];
      bad |= par;
    }
    bad = __reduce_or_sync(kFull, bad);
    if ((threadIdx.x & 31) == 0 && (bad & am)) atomicOr(&p.unsat[grp], bad & am);
  }
}

// Boundary k: record bit errors, retire converged frames (k > 0), reset tallies.
static __global__ void phase_finalize_kernel(const __grid_constant__ PhaseParams p, int k, int check) {
  constexpr int F = kFixedFrames;
  const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= (long long)p.groups * F) return;
  const long long grp = x / F;
  const int lane = (int)(x - grp * F);
  const long long f = x;
  const unsigned am = p.amask[grp];
  const int I = p.i_max;
  if (f < p.B && ((am >> lane) & 1u)) {
    const long long ff = p.f_base + f;
    const int e = p.errs[x], ei = p.errs_info[x];
    p.biterr[ff * (I + 1) + k] = e;
    p.biterr_info[ff * (I + 1) + k] = ei;
    const bool sat = check && !((p.unsat[grp] >> lane) & 1u);
    if (sat || k == I) {
      p.iters[x] = k;
      p.conv[ff] = sat ? 1 : 0;
      for (int kk = k + 1; kk <= I; ++kk) {  // E:211-217
        p.biterr[ff * (I + 1) + kk] = e;
        p.biterr_info[ff * (I + 1) + kk] = ei;
      }
    }
  }
  p.errs[x] = 0;
  p.errs_info[x] = 0;
  __syncwarp();
  if (lane == 0) {
    unsigned done = 0;
    if (check) done = am & ~p.unsat[grp];
    if (k == I) done = am;
    p.amask[grp] = am & ~done;
    p.unsat[grp] = 0;
  }
}

// Hard decisions and counters (E:192-201, schedules.py:147).
template <typename T>
__global__ void __launch_bounds__(kPhaseThreads) phase_output_kernel(const __grid_constant__ PhaseParams p) {
  constexpr int F = kFixedFrames;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int vchunks = (p.g.N + kPhaseVnChunk - 1) / kPhaseVnChunk;
  const long long items = (long long)p.groups * vchunks;
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const long long grp = it / vchunks;
    const int c = (int)(it - grp * vchunks);
    GroupSlot<T> s(p, grp);
    const long long f = grp * F + lane;
    const int n1 = min(p.g.N, (c + 1) * kPhaseVnChunk);
    for (int n = c * kPhaseVnChunk + warp; n < n1; n += nw)
      if (f < p.B) p.u_hat[(p.f_base + f) * p.g.N + n] = (s.sign[n] >> lane) & 1u;
    if (c == 0 && warp == 0 && f < p.B) {
      const long long ff = p.f_base + f;
      const long long prop = p.i_max == 0 ? 0 : (long long)p.iters[f] * p.g.E;
      p.prop[ff] = prop;
      p.counters[ff * kCounters + C_PROP] = prop;
      p.counters[ff * kCounters + C_V2C] = prop;
      for (int k = 2; k < kCounters; ++k) p.counters[ff * kCounters + k] = 0;
    }
  }
}

#endif  // LDPC_PHASE_DECL_ONLY

}  // namespace ldpc

#include "fixed_tma.cuh"  // TMA-fed check phase (uses PhaseParams / GroupSlot)
