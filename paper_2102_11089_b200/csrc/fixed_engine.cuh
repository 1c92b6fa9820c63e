// fixed_engine.cuh -- flooding and row-layered BP, frame-interleaved, tiled.
//
// Flooding replaces _decode_flooding (E:719-765): per iteration all C2V from
// the previous V2C, then totals and V2C per VN, syndrome at every iteration.
// Layered is the schedule the reference lacks (defined in
// oracle/ldpc_oracle.c): checks m = 0..M-1 in order, each committing
// total += c2v' - c2v.  Checks are grouped into dependency levels on the host
// (a check's level exceeds that of every earlier check sharing a VN), so a
// level runs in parallel and still reproduces the sequential order exactly.
// Flooding is the one-level case (all checks read the previous totals).
//
// Layout: a CTA owns a group of 32 frames; its HBM slot holds chl[N][32],
// total[N][32], c2v[E][32] (frame index fastest, so one warp = 32 frames moves
// one coalesced 256-byte row per access) and sign[N] words.  Only c2v and
// totals are kept: the V2C of an edge is clamp(total - c2v), bit-identical to
// the reference's stored v2c (E:752-754).
//
// Each level is cut (on the host) into tiles of <= kTileEdges edges made of
// whole checks.  Per tile, phase A spreads the tile's edges over all warps:
// gather the c2v row and the total row, form in = tanh(clamp(total - c2v)/2)
// (or v2c for min-sum) into shared memory; phase B gives every (edge, frame)
// a thread: the exact left-to-right product of its check's other inputs from
// shared memory, atanh, store (layered also commits total += new - old).  No
// per-thread arrays, so registers stay low and many warps keep many 256-byte
// rows in flight -- the kernel is HBM-bound on large codes.
//
// Syndrome / bit errors: the VN pass writes each VN's 32 frame sign bits as
// one word (warp ballot) to the L2-resident sign[] array and tallies errors
// per lane; a check's parity for 32 frames is the XOR of its VNs' words.
#pragma once
#include "ldpc_common.cuh"

namespace ldpc {

constexpr int kFixedMaxDc = 32;
constexpr int kFixedFrames = 32;  // frames per CTA (= warp lanes)
constexpr int kTileEdges = 128;   // edges per shared-memory tile

struct FixedParams {
  DevGraph g;
  int kind, kernel, i_max, k_info;
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
  unsigned char* ws;      // per-CTA slot: chl[N][32], total[N][32], c2v[E][32], sign[N]
  long long slot_bytes;
  // tiling of the schedule (flooding: one level in check order; layered: levels)
  int n_levels;
  const int* level_tptr;  // [n_levels+1] tile range of each level
  const int* tile_eptr;   // [n_tiles+1] offsets into te_list
  const int* te_list;     // [E] global edge id, tile order
  const int* te_vn;       // [E] VN of te_list[x] (one load instead of two dependent ones)
  const int2* te_chk;     // [E] tile-local [a, b) of the edge's check
  const int* tile_cptr;   // [n_tiles+1] offsets into tc_rec
  const int4* tc_rec;     // [M] per check in tile order: (local a, degree, first edge id, 0)
};

template <typename T, int KERNEL>
__device__ __forceinline__ T tile_out(const T* in_s, int2 ck, int el, int lane) {
  if (KERNEL == KERNEL_EXACT) {
    T prod = cn_one<T>();
    for (int q = ck.x; q < ck.y; ++q)
      if (q != el) prod = cn_mul(prod, in_s[q * kFixedFrames + lane]);
    return atanh_msg(prod, ck.y - ck.x - 1);
  } else {
    T sign = T(1), mag = Num<T>::kBig;
    for (int q = ck.x; q < ck.y; ++q) {
      if (q == el) continue;
      T v = in_s[q * kFixedFrames + lane];
      if (v < T(0)) { sign = -sign; v = -v; }
      if (v < mag) mag = v;
    }
    return ck.y - ck.x > 1 ? clampv(sign * mag) : T(0);
  }
}

constexpr int kPhaseBRegs = 16;  // checks up to this degree keep their inputs in registers

// Commit of output q of a check (rec = local a, degree, tile position of its
// first edge).  c2v rows are stored in tile order (the position in te_list),
// so a tile's c2v rows are contiguous; layered commits total[vn] = tot + (c2v'
// - c2v) with tot staged from the tile (tot_s) or re-read (+=).
template <typename T, bool LAYERED>
__device__ __forceinline__ void commit_out(const int* te_vn, const T* old_s, const T* tot_s, int la, int ga,
                                           int q, int lane, T out, T* c2v, T* total) {
  constexpr int F = kFixedFrames;
  c2v[(long long)(ga + q) * F + lane] = out;
  if (LAYERED) {
    T* tp = &total[(long long)te_vn[ga + q] * F + lane];
    const T d_ = out - old_s[(la + q) * F + lane];
    if (tot_s) *tp = tot_s[(la + q) * F + lane] + d_;
    else *tp += d_;
  }
}

// All C2V outputs of one check of degree D for one frame (lane), inputs from
// the tile in shared memory, fully unrolled for the degree.  Exact kernel,
// float64: prod_q = prefix(in_0..in_{q-1}) continued by in_{q+1}..in_{d-1} --
// the reference's left-to-right product (E:55-59) with the prefix shared.
// Exact, float32: prefix x suffix (no bit-order obligation in fp32).  Min-sum:
// min1 / min2 / sign parity in one pass -- the same values as the per-output
// loop of E:67-82 (min and sign products do not depend on order).
template <typename T, int KERNEL, bool LAYERED, int D>
__device__ __forceinline__ void check_outputs_d(const int* te_vn, const T* in_s, const T* old_s, int la, int ga,
                                                int lane, bool act, T* c2v, T* total, const T* tot_s) {
  constexpr int F = kFixedFrames;
  T in[D];
#pragma unroll
  for (int q = 0; q < D; ++q) in[q] = in_s[(la + q) * F + lane];
  if (KERNEL == KERNEL_EXACT) {
    constexpr bool kSuffix = sizeof(T) == 4;
    T suf[D];
    if (kSuffix) {
      T acc = cn_one<T>();
#pragma unroll
      for (int q = D - 1; q >= 0; --q) {
        suf[q] = acc;
        acc = cn_mul(acc, in[q]);
      }
    }
    T pre = cn_one<T>();
#pragma unroll
    for (int q = 0; q < D; ++q) {
      T prod = pre;
      if (kSuffix) {
        prod = cn_mul(prod, suf[q]);
      } else {
#pragma unroll
        for (int r = q + 1; r < D; ++r) prod = cn_mul(prod, in[r]);
      }
      const T out = atanh_msg(prod, D - 1);
      pre = cn_mul(pre, in[q]);
      if (act) commit_out<T, LAYERED>(te_vn, old_s, tot_s, la, ga, q, lane, out, c2v, total);
    }
  } else {
    T m1 = Num<T>::kBig, m2 = Num<T>::kBig, sgn = T(1);
    int i1 = -1;
    unsigned negs = 0u;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      T v = clampv(in[q]);
      if (v < T(0)) {
        sgn = -sgn;
        v = -v;
        negs |= 1u << q;
      }
      if (v < m1) {
        m2 = m1;
        m1 = v;
        i1 = q;
      } else if (v < m2) {
        m2 = v;
      }
    }
#pragma unroll
    for (int q = 0; q < D; ++q) {
      const T sign = ((negs >> q) & 1u) ? -sgn : sgn;
      const T out = D > 1 ? clampv(sign * (q == i1 ? m2 : m1)) : T(0);
      if (act) commit_out<T, LAYERED>(te_vn, old_s, tot_s, la, ga, q, lane, out, c2v, total);
    }
  }
}

template <typename T, int KERNEL, bool LAYERED>
__device__ __forceinline__ void check_outputs(const int* te_vn, const T* in_s, const T* old_s, int4 rec, int lane,
                                              bool act, T* c2v, T* total, const T* tot_s = nullptr) {
  const int la = rec.x, d = rec.y, ga = rec.z;
  switch (d) {
#define LDPC_CK(D_) \
  case D_: check_outputs_d<T, KERNEL, LAYERED, D_>(te_vn, in_s, old_s, la, ga, lane, act, c2v, total, tot_s); return;
    LDPC_CK(1) LDPC_CK(2) LDPC_CK(3) LDPC_CK(4) LDPC_CK(5) LDPC_CK(6) LDPC_CK(7) LDPC_CK(8)
    LDPC_CK(9) LDPC_CK(10) LDPC_CK(11) LDPC_CK(12) LDPC_CK(13) LDPC_CK(14) LDPC_CK(15) LDPC_CK(16)
#undef LDPC_CK
    default:
      for (int q = 0; q < d; ++q) {
        const T out = tile_out<T, KERNEL>(in_s, make_int2(la, la + d), la + q, lane);
        if (act) commit_out<T, LAYERED>(te_vn, old_s, tot_s, la, ga, q, lane, out, c2v, total);
      }
  }
}

// Ampere-style asynchronous global->shared copies (LDGSTS), 16 bytes each.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <typename T>
__device__ __forceinline__ void sign_row(int n, T tv, int k_info, unsigned* sign, int lane, int& errs,
                                         int& errs_info) {
  const bool neg = tv < T(0);
  const unsigned w = __ballot_sync(kFull, neg);
  if (lane == 0) sign[n] = w;
  if (neg) {
    ++errs;
    if (n < k_info) ++errs_info;
  }
}

// PIPE: the check phase streams tiles through kFixedStages shared-memory
// stages with cp.async -- tile t+1's c2v and total rows are in flight while
// tile t computes (within a level; layered levels restart the pipeline because
// level L+1 reads the totals level L writes).
constexpr int kFixedStages = 2;

template <typename T, int KERNEL, bool LAYERED, bool PIPE = false>
__global__ void __launch_bounds__(512, 2) fixed_decode_kernel(const __grid_constant__ FixedParams p) {
  const DevGraph& g = p.g;
  constexpr int F = kFixedFrames;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int I = p.i_max;
  T* chl = (T*)(p.ws + (long long)blockIdx.x * p.slot_bytes);
  T* total = chl + (long long)g.N * F;
  T* c2v = total + (long long)g.N * F;
  unsigned* sign = (unsigned*)(c2v + (long long)g.E * F);
  extern __shared__ __align__(16) unsigned char fixed_smem[];
  T* in_s = (T*)fixed_smem;            // [kTileEdges][32]
  T* old_s = in_s + kTileEdges * F;    // [kTileEdges][32], layered only (PIPE: stages follow in_s)
  T* stg = in_s + kTileEdges * F;      // PIPE: [kFixedStages][2][kTileEdges][32] (c2v rows, total rows)
  __shared__ int s_active[F], s_errs[F], s_errs_info[F], s_iter[F];
  __shared__ unsigned s_unsat;
  __shared__ unsigned long long s_grp;
  for (;;) {
    if (tid == 0) s_grp = atomicAdd(p.next, 1ull);
    __syncthreads();
    const long long f0 = (long long)s_grp * F;
    if (f0 >= p.B) break;
    const long long fl_glob = f0 + lane;
    const bool lane_valid = fl_glob < p.B;
    if (tid < F) {
      s_active[tid] = (f0 + tid) < p.B;
      s_iter[tid] = 0;
      s_errs[tid] = s_errs_info[tid] = 0;
    }
    if (tid == 0) s_unsat = 0;
    // load LLRs (transposed into [N][32]), c2v = 0, total = chl; boundary-0 tallies
    int errs = 0, errs_info = 0;
    for (int n = warp; n < g.N; n += nw) {
      T v = T(0);
      if (lane_valid)
        v = p.llr_f64 ? (T)((const double*)p.llr)[fl_glob * g.N + n] : (T)((const float*)p.llr)[fl_glob * g.N + n];
      chl[(long long)n * F + lane] = v;
      total[(long long)n * F + lane] = v;
      sign_row<T>(n, v, p.k_info, sign, lane, errs, errs_info);
    }
    for (long long x = tid; x < (long long)g.E * F; x += nt) c2v[x] = T(0);
    __syncthreads();
    atomicAdd(&s_errs[lane], errs);
    atomicAdd(&s_errs_info[lane], errs_info);
    __syncthreads();
    for (int it = 0;; ++it) {
      if (it > 0) {  // boundary `it`: syndrome from the sign words, 32 frames per check
        unsigned bad = 0;
        for (int m = tid; m < g.M; m += nt) {
          unsigned par = 0;
          for (int e = g.cn_ptr[m]; e < g.cn_ptr[m + 1]; ++e) par ^= sign[g.edge_vn[e]];
          bad |= par;
        }
        bad = __reduce_or_sync(kFull, bad);
        if (lane == 0 && bad) atomicOr(&s_unsat, bad);
      }
      __syncthreads();
      if (tid < F && s_active[tid]) {
        const long long f = f0 + tid;
        p.biterr[f * (I + 1) + it] = s_errs[tid];
        p.biterr_info[f * (I + 1) + it] = s_errs_info[tid];
        bool done = false;
        if (it > 0 && !((s_unsat >> tid) & 1u)) {  // converged at iteration it (E:761-764)
          done = true;
          p.conv[f] = 1;
          for (int kk = it + 1; kk <= I; ++kk) {
            p.biterr[f * (I + 1) + kk] = s_errs[tid];
            p.biterr_info[f * (I + 1) + kk] = s_errs_info[tid];
          }
        } else if (it == I) {
          done = true;
          p.conv[f] = 0;
        }
        if (done) {
          s_active[tid] = 0;
          s_iter[tid] = it;
        }
      }
      __syncthreads();
      unsigned any = 0;
      for (int q = 0; q < F; ++q) any |= s_active[q];
      if (!any) break;
      const bool act = s_active[lane] != 0;
      __syncthreads();
      if (tid < F) s_errs[tid] = s_errs_info[tid] = 0;
      if (tid == 0) s_unsat = 0;
      // ---- check phase, tile by tile, level by level
      if (PIPE) {
        constexpr int S = kFixedStages;
        constexpr int CH = F * (int)sizeof(T) / 16;  // 16-byte chunks per row
        auto stage = [&](int k) { return stg + (long long)k * 2 * kTileEdges * F; };
        auto issue = [&](int t, int k) {
          const int ea = p.tile_eptr[t], ne = p.tile_eptr[t + 1] - ea;
          T* dst = stage(k);
          for (int x = tid; x < 2 * ne * CH; x += nt) {
            const int r = x / CH, ch = x - r * CH;
            const int el = r < ne ? r : r - ne;
            const T* src = r < ne ? c2v + (long long)(ea + el) * F : total + (long long)p.te_vn[ea + el] * F;
            cp_async16(dst + ((r < ne ? 0 : kTileEdges) + el) * F + ch * (16 / (int)sizeof(T)),
                       src + ch * (16 / (int)sizeof(T)));
          }
        };
        for (int L = 0; L < p.n_levels; ++L) {
          const int t0 = p.level_tptr[L], t1 = p.level_tptr[L + 1];
          for (int k = 0; k < S - 1; ++k) {
            if (t0 + k < t1) issue(t0 + k, k);
            cp_async_commit();
          }
          for (int t = t0; t < t1; ++t) {
            if (t + S - 1 < t1) issue(t + S - 1, (t + S - 1 - t0) % S);
            cp_async_commit();
            cp_async_wait<S - 1>();
            __syncthreads();
            const int ea = p.tile_eptr[t], ne = p.tile_eptr[t + 1] - ea;
            const T* so = stage((t - t0) % S);  // c2v rows
            const T* st = so + kTileEdges * F;  // total rows
            for (int x = tid; x < ne * F; x += nt) {  // phase A from shared memory
              const T v = clampv(st[x] - so[x]);
              in_s[x] = (KERNEL == KERNEL_EXACT) ? cn_in<T>(v) : v;  // E:58 / E:73
            }
            __syncthreads();
            if (sizeof(T) == 4) {  // one warp per check (shared prefix products)
              for (int ck = p.tile_cptr[t] + warp; ck < p.tile_cptr[t + 1]; ck += nw)
                check_outputs<T, KERNEL, LAYERED>(p.te_vn, in_s, so, p.tc_rec[ck], lane, act, c2v, total, st);
            } else {  // float64: one warp per edge (register-light)
              for (int el = warp; el < ne; el += nw) {
                const T out = tile_out<T, KERNEL>(in_s, p.te_chk[ea + el], el, lane);
                if (act) {
                  c2v[(long long)(ea + el) * F + lane] = out;
                  if (LAYERED)
                    total[(long long)p.te_vn[ea + el] * F + lane] = st[el * F + lane] + (out - so[el * F + lane]);
                }
              }
            }
            __syncthreads();
          }
        }
        cp_async_wait<0>();
      }
      for (int L = 0; L < (PIPE ? 0 : p.n_levels); ++L) {
        for (int t = p.level_tptr[L]; t < p.level_tptr[L + 1]; ++t) {
          const int ea = p.tile_eptr[t], ne = p.tile_eptr[t + 1] - ea;
          // phase A: 4 edges per warp in flight (loads first, then the math)
          for (int el0 = warp; el0 < ne; el0 += 4 * nw) {
            T o[4], tv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int el = el0 + u * nw;
              if (el < ne) {
                o[u] = c2v[(long long)(ea + el) * F + lane];  // c2v rows in tile order
                tv[u] = total[(long long)p.te_vn[ea + el] * F + lane];
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int el = el0 + u * nw;
              if (el < ne) {
                const T v = clampv(tv[u] - o[u]);
                in_s[el * F + lane] = (KERNEL == KERNEL_EXACT) ? cn_in<T>(v) : v;  // E:58 / E:73
                if (LAYERED) old_s[el * F + lane] = o[u];
              }
            }
          }
          __syncthreads();
          if (sizeof(T) == 4) {
            // phase B (float32): one warp per check, inputs in registers, shared prefix
            for (int ck = p.tile_cptr[t] + warp; ck < p.tile_cptr[t + 1]; ck += nw)
              check_outputs<T, KERNEL, LAYERED>(p.te_vn, in_s, old_s, p.tc_rec[ck], lane, act, c2v, total);
          } else {
            // phase B (float64): one warp per edge -- register-light, so twice the warps
            for (int el = warp; el < ne; el += nw) {
              const T out = tile_out<T, KERNEL>(in_s, p.te_chk[ea + el], el, lane);
              if (act) {
                c2v[(long long)(ea + el) * F + lane] = out;
                if (LAYERED) total[(long long)p.te_vn[ea + el] * F + lane] += out - old_s[el * F + lane];
              }
            }
          }
          __syncthreads();
        }
      }
      // ---- VN pass: totals (flooding), sign words, error tallies
      errs = errs_info = 0;
      for (int n = warp; n < g.N; n += nw) {
        const long long nx = (long long)n * F + lane;
        T s;
        if (!LAYERED && act) {
          s = chl[nx];
          const int k0 = g.vn_ptr[n], k1 = g.vn_ptr[n + 1];
          for (int k = k0; k < k1; k += 8) {  // 8 rows in flight, summed in order (E:749-750)
            T r[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (k + u < k1) r[u] = c2v[(long long)g.vn_edges[k + u] * F + lane];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (k + u < k1) s += r[u];
          }
          total[nx] = s;
        } else {
          s = total[nx];
        }
        sign_row<T>(n, s, p.k_info, sign, lane, errs, errs_info);
      }
      if (act) {
        atomicAdd(&s_errs[lane], errs);
        atomicAdd(&s_errs_info[lane], errs_info);
      }
      __syncthreads();
    }
    // outputs
    for (int n = warp; n < g.N; n += nw)
      if (lane_valid) p.u_hat[fl_glob * g.N + n] = (sign[n] >> lane) & 1u;
    if (tid < F && f0 + tid < p.B) {
      const long long f = f0 + tid;
      const long long prop = I == 0 ? 0 : (long long)s_iter[tid] * g.E;
      p.prop[f] = prop;
      p.counters[f * kCounters + C_PROP] = prop;
      p.counters[f * kCounters + C_V2C] = prop;
      for (int k = 2; k < kCounters; ++k) p.counters[f * kCounters + k] = 0;
    }
    if (I == 0) {  // converged = syndrome of the channel decisions (schedules.py:144-146)
      if (tid == 0) s_unsat = 0;
      __syncthreads();
      unsigned bad = 0;
      for (int m = tid; m < g.M; m += nt) {
        unsigned par = 0;
        for (int e = g.cn_ptr[m]; e < g.cn_ptr[m + 1]; ++e) par ^= sign[g.edge_vn[e]];
        bad |= par;
      }
      bad = __reduce_or_sync(kFull, bad);
      if (lane == 0 && bad) atomicOr(&s_unsat, bad);
      __syncthreads();
      if (tid < F && f0 + tid < p.B) p.conv[f0 + tid] = ((s_unsat >> tid) & 1u) ? 0 : 1;
    }
    __syncthreads();
  }
}

}  // namespace ldpc
