// fixed_tma.cuh -- warp-specialised, TMA-fed check phase for flooding / layered.
//
// Same work as phase_check_kernel (fixed_phase.cuh): every (32-frame group,
// strip) item of one level gets its C2V outputs (E:49-103 arithmetic, the
// reference's operation order in float64) and, for layered, its total commits.
//
// Strips (built on the host, ldpc_capi.cu): k consecutive checks of one level
// with the same degree d (k*d <= kTileEdges), staged SLOT-MAJOR -- row q*k + c
// holds slot q (the q-th edge, ascending VN) of check c.  The c2v rows of the
// flooding / layered schedules are STORED in that order too, so a strip's c2v
// rows are one contiguous block, and for quasi-cyclic codes (a block row's Z
// checks have the same degree; slot q of consecutive checks hits consecutive
// VNs of one circulant) the gathered total rows of a slot are a few contiguous
// VN runs.  The host stores those runs per strip.
//
// Pipeline (kTmaStages shared-memory stages, transaction mbarriers):
//   * one producer warp streams items: one bulk async copy (cp.async.bulk, the
//     TMA engine) for the strip's c2v block and one per total-row run, so a
//     BG1 strip of ~120 edges costs ~8-14 copy instructions instead of 256
//     row gathers.  The next item's strip record and runs are loaded into
//     registers while the current item's copies fly;
//   * consumer warps take whole checks of the staged strip: they form the
//     check inputs tanh(clamp(total - c2v)/2) (or the V2C for min-sum) from
//     the staged rows into registers, compute all outputs, store each output
//     row (one coalesced 32-frame row per warp store) and release the stage
//     through an "empty" mbarrier.  No CTA-wide barrier in the steady state.
#pragma once
#include "fixed_engine.cuh"

namespace ldpc {

constexpr int kTmaStages = 3;

template <typename T, int NC>
struct TmaLayout {
  static constexpr int F = kFixedFrames;
  static constexpr int kRows = kTileEdges * F;              // elements of one row block
  static constexpr int kRowBytes = F * (int)sizeof(T);      // one 32-frame row
  static constexpr int kStageBytes = 2 * kRows * (int)sizeof(T) + kTileEdges * 4;
  static constexpr int kBarOff = kTmaStages * kStageBytes;  // 2 x kTmaStages mbarriers
  static constexpr int kBytes = kBarOff + 2 * kTmaStages * 8;
  static constexpr int kThreads = (NC + 1) * 32;
  static constexpr int kMinBlocks = sizeof(T) == 4 ? 2 : 1;
};

// VN phase (flooding): VN strips of k consecutive VNs with the same degree dv,
// staged rows [s*k + v] = c2v of the v-th VN's s-th edge (vn_edges order),
// then k chl rows.  k*dv <= kTileEdges, k <= kVnStripMax.
constexpr int kVnStripMax = 64;
template <typename T, int NC>
struct VnLayout {
  static constexpr int F = kFixedFrames;
  static constexpr int kRowsMax = kTileEdges + kVnStripMax;
  static constexpr int kRowBytes = F * (int)sizeof(T);
  static constexpr int kStageBytes = kRowsMax * kRowBytes;
  static constexpr int kBarOff = kTmaStages * kStageBytes;
  static constexpr int kBytes = kBarOff + 2 * kTmaStages * 8;
  static constexpr int kThreads = (NC + 1) * 32;
};

// ----------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: the warp sleeps until the phase completes
// (or the hint expires) instead of spinning on issue slots
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
// non-blocking probe of a phase
__device__ __forceinline__ bool mbar_test(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  while (!mbar_try(b, parity)) {
  }
}
// global -> shared bulk copy (TMA engine), completion counted on mbarrier `b`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

// ------------------------------------------------------ fused check math
// Layered: the sign-word / error-tally pass (E:192-201) folded into the check
// phase.  The staged row of a VN's last level in the sweep carries bit 31 in
// s_vn; its new total is final for the iteration, so the warp ballots the 32
// frames' signs there (frames already retired contribute their unchanged
// total) and tallies the bit errors of the active frames.
struct SignSink {
  unsigned* sign;
  int k_info;
  bool on;
  int errs, ei;
};
// Input of staged row x: tanh(clamp(total - c2v)/2) (E:58) or the clamped V2C
// (min-sum, E:73).
template <typename T, int KERNEL>
__device__ __forceinline__ T staged_in(const T* so, const T* st, int x) {
  const T v = clampv(st[x] - so[x]);
  return (KERNEL == KERNEL_EXACT) ? cn_in<T>(v) : v;
}

// Output of staged row r (lane = frame): c2v row e0 + r; layered also commits
// total[vn] = total_old + (c2v_new - c2v_old).
// Commit of staged row r (offset xq; cq = its stored c2v row): the C2V output,
// and for layered total[vn] = total_old + (c2v_new - c2v_old) plus, at the
// VN's last level, its sign word and error tallies.  Stores only for active
// frames (`act`); the whole warp runs this (the ballot needs every lane).
template <typename T, bool LAYERED>
__device__ __forceinline__ void strip_commit_p(const T* so, const T* st, const int* tv, int r, int xq, T* cq, T out,
                                               T* total, int lane, bool act, SignSink& sk) {
  constexpr int F = kFixedFrames;
  if (act) *cq = out;
  if (LAYERED) {
    const T nt = st[xq] + (out - so[xq]);
    const int tvr = tv[r], vn = tvr & 0x7fffffff;
    if (act) total[(long long)vn * F + lane] = nt;
    if (sk.on && tvr < 0) {  // warp-uniform: the same staged row in every lane
      const T fin = act ? nt : st[xq];
      const bool neg = fin < T(0);
      const unsigned wsg = __ballot_sync(kFull, neg);
      if (lane == 0) sk.sign[vn] = wsg;
      if (act && neg) {
        ++sk.errs;
        if (vn < sk.k_info) ++sk.ei;
      }
    }
  }
}

// All outputs of check c of a strip (k checks of degree D, slot-major rows).
// float64 keeps the reference's left-to-right product (shared prefix, then
// the remaining inputs in order); float32 uses prefix x suffix.  Min-sum:
// min1 / min2 / sign parity (order-free, same values as E:67-82).
template <typename T, int KERNEL, bool LAYERED, int D>
__device__ __forceinline__ void strip_check_d(const T* so, const T* st, const int* tv, int c, int k, long long e0,
                                              int lane, T* c2v, T* total, bool act, SignSink& sk) {
  constexpr int F = kFixedFrames;
  const int x0 = c * F + lane, xs = k * F;     // staged offset of slot 0, slot stride
  T* c0 = c2v + ((e0 + c) * F + lane);         // stored c2v row of slot 0
  T in[D];
#pragma unroll
  for (int q = 0; q < D; ++q) in[q] = staged_in<T, KERNEL>(so, st, x0 + q * xs);
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
      pre = cn_mul(pre, in[q]);
      strip_commit_p<T, LAYERED>(so, st, tv, q * k + c, x0 + q * xs, c0 + q * xs, atanh_msg(prod, D - 1), total, lane,
                                 act, sk);
    }
  } else {
    T m1 = Num<T>::kBig, m2 = Num<T>::kBig, sgn = T(1);
    int i1 = -1;
    unsigned negs = 0u;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      T v = in[q];
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
      strip_commit_p<T, LAYERED>(so, st, tv, q * k + c, x0 + q * xs, c0 + q * xs, out, total, lane, act, sk);
    }
  }
}

// Degrees above the unrolled range: each output recomputes its inputs in the
// reference's order (O(d^2) transcendental work; such checks are rare).
template <typename T, int KERNEL, bool LAYERED>
__device__ __noinline__ void strip_check_generic(const T* so, const T* st, const int* tv, int c, int k, int d,
                                                 long long e0, int lane, T* c2v, T* total, bool act, SignSink& sk) {
  constexpr int F = kFixedFrames;
  for (int q = 0; q < d; ++q) {
    T out;
    if (KERNEL == KERNEL_EXACT) {
      T prod = cn_one<T>();
      for (int r = 0; r < d; ++r)
        if (r != q) prod = cn_mul(prod, staged_in<T, KERNEL>(so, st, (r * k + c) * F + lane));
      out = atanh_msg(prod, d - 1);
    } else {
      T sign = T(1), mag = Num<T>::kBig;
      for (int r = 0; r < d; ++r) {
        if (r == q) continue;
        T v = staged_in<T, KERNEL>(so, st, (r * k + c) * F + lane);
        if (v < T(0)) {
          sign = -sign;
          v = -v;
        }
        if (v < mag) mag = v;
      }
      out = d > 1 ? clampv(sign * mag) : T(0);
    }
    strip_commit_p<T, LAYERED>(so, st, tv, q * k + c, (q * k + c) * F + lane, c2v + ((e0 + q * k + c) * F + lane), out,
                               total, lane, act, sk);
  }
}

// The checks c = c0, c0 + step, ... of a staged strip (k checks, degree d).
template <typename T, int KERNEL, bool LAYERED>
__device__ __forceinline__ void strip_checks(const T* so, const T* st, const int* tv, int c0, int step, int k, int d,
                                             long long e0, int lane, T* c2v, T* total, bool act, SignSink& sk) {
  switch (d) {
#define LDPC_SCK(D_)                                                                                     \
  case D_:                                                                                               \
    for (int c = c0; c < k; c += step)                                                                   \
      strip_check_d<T, KERNEL, LAYERED, D_>(so, st, tv, c, k, e0, lane, c2v, total, act, sk);            \
    return;
    LDPC_SCK(1) LDPC_SCK(2) LDPC_SCK(3) LDPC_SCK(4) LDPC_SCK(5) LDPC_SCK(6) LDPC_SCK(7) LDPC_SCK(8)
    LDPC_SCK(9) LDPC_SCK(10) LDPC_SCK(11) LDPC_SCK(12) LDPC_SCK(13) LDPC_SCK(14) LDPC_SCK(15) LDPC_SCK(16)
#undef LDPC_SCK
    default:
      for (int c = c0; c < k; c += step)
        strip_check_generic<T, KERNEL, LAYERED>(so, st, tv, c, k, d, e0, lane, c2v, total, act, sk);
  }
}

#ifndef LDPC_PHASE_DECL_ONLY

// (group, strip) items of the levels [L0, L1): level-major, then group, then
// strip, so a level's items of one group are contiguous and every item's
// dependencies (the group's earlier levels) come earlier in the order.
struct LevelMap {
  const int* lp;  // strip prefix per level (lp[L] = first strip of level L)
  int L0, L1, G, W, Ptot;
  long long wlo, whi;  // item range of the current window of groups [gb, gb + Gw)
  int gb, Gw;
  int L, P, nL;
  long long lo, hi;  // item range of level L within the window
  // Items: windows of W consecutive groups; inside a window level-major, then
  // group, then strip (W = G: the plain level-major order).
  __device__ LevelMap(const int* lp_, int L0_, int L1_, int G_, int W_) : lp(lp_), L0(L0_), L1(L1_), G(G_) {
    W = (W_ <= 0 || W_ > G) ? G : W_;
    Ptot = lp[L1] - lp[L0];
    gb = 0;
    Gw = W < G ? W : G;
    wlo = 0;
    whi = (long long)Gw * Ptot;
    start_level();
  }
  __device__ __forceinline__ void start_level() {
    L = L0;
    lo = wlo;
    P = lp[L];
    nL = lp[L + 1] - P;
    hi = lo + (long long)Gw * nL;
  }
  __device__ __forceinline__ void seek(long long i) {
    while (i >= whi && gb + Gw < G) {
      gb += Gw;
      Gw = G - gb < W ? G - gb : W;
      wlo = whi;
      whi = wlo + (long long)Gw * Ptot;
      start_level();
    }
    while (i >= hi && L + 1 < L1) {
      ++L;
      lo = hi;
      P = lp[L];
      nL = lp[L + 1] - P;
      hi = lo + (long long)Gw * nL;
    }
  }
  __device__ __forceinline__ int group(long long i) const { return gb + (int)((unsigned)(i - lo) / (unsigned)nL); }
  __device__ __forceinline__ int strip(long long i, int g) const {
    return P + (int)(i - lo - (long long)(g - gb) * nL);
  }
};

__device__ __forceinline__ int ld_acquire(const int* a) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// Check phase over the strips of levels [L0, L1), all active groups.
// Block = NC consumer warps + 1 producer warp (the last one).
// dep_base >= 0 (layered, all levels in one launch): an item of level L of
// group g starts loading totals only once p.done[g] >= dep_base + lp[L], i.e.
// once every strip of the group's earlier levels of this iteration has been
// committed (one release-increment per finished item) -- the level order of
// the reference sweep is kept per group while different groups run different
// levels, with no grid-wide barrier or relaunch between levels.
// FUSED: the build with the level map, dependency waits and item publication
// (all layered levels in one launch when dep_base >= 0; with dep_base < 0 it
// runs one level like the plain build -- the layered per-level launches use
// it because ptxas allocates it without spills); the plain build (flooding)
// maps the items of one level range directly.
template <typename T, int KERNEL, bool LAYERED, int NC, bool FUSED>
__global__ void __launch_bounds__(TmaLayout<T, NC>::kThreads, TmaLayout<T, NC>::kMinBlocks)
    phase_check_tma_kernel(const __grid_constant__ PhaseParams p, int L0, int L1, int dep_base, int rev) {
  using L = TmaLayout<T, NC>;
  constexpr int F = kFixedFrames, S = kTmaStages, RPL = kTileEdges / 32;  // runs / rows per lane
  extern __shared__ __align__(128) unsigned char tma_smem[];
  auto so_of = [&](int s) { return (T*)(tma_smem + s * L::kStageBytes); };
  auto st_of = [&](int s) { return (T*)(tma_smem + s * L::kStageBytes) + L::kRows; };
  auto tv_of = [&](int s) { return (int*)(tma_smem + s * L::kStageBytes + 2 * L::kRows * (int)sizeof(T)); };
  unsigned long long* full = (unsigned long long*)(tma_smem + L::kBarOff);
  unsigned long long* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int t0 = p.s_lvl[L0], nti = p.s_lvl[L1] - t0;
  const long long items = (long long)p.groups * nti;  // < 2^31
  LevelMap lm(p.s_lvl, L0, FUSED ? L1 : L0 + 1, p.groups, FUSED && dep_base >= 0 ? p.lwin : 0);
  // item -> (logical group, strip)
  auto item_group = [&](long long i) -> int {
    if (FUSED) {
      lm.seek(i);
      return lm.group(i);
    }
    return (int)((unsigned)i / (unsigned)nti);
  };
  auto item_strip = [&](long long i, int lg) -> int {
    return FUSED ? lm.strip(i, lg) : t0 + (int)(i - (long long)lg * nti);
  };

  if (warp == NC) {  // ---------------- producer
    auto seek = [&](long long i) {
      for (; i < items; i += gridDim.x) {
        const int g = item_group(i);
        if (p.amask[rev ? p.groups - 1 - g : g]) break;
      }
      return i;
    };
    long long it = seek(blockIdx.x);
    int4 rec = make_int4(0, 0, 0, 0);
    int nrun = 0, grp = 0, need = 0;
    int2 run[RPL];
    int vn[RPL];
    auto prefetch = [&](long long i) {
      if (i >= items) return;
      const int lg = item_group(i);
      const int t = item_strip(i, lg);
      grp = rev ? p.groups - 1 - lg : lg;
      if (FUSED) need = dep_base + lm.P;
      rec = p.s_rec[t];
      nrun = p.s_rec[t + 1].w - rec.w;
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        const int r = lane + 32 * j;
        if (r < nrun) run[j] = p.s_runs[rec.w + r];
        if (LAYERED && r < rec.y * rec.z) vn[j] = p.s_vn[rec.x + r];
      }
    };
    prefetch(it);
    // Publication of finished items (levels fused): the consumers' stores are
    // released to this warp by their "empty" arrivals; a gpu-scope fence then
    // makes them visible before the group's counter moves.  Items are
    // published in issue order (pub_k = oldest unpublished), eagerly while
    // this warp waits on a dependency, so a waiting CTA never holds back a
    // finished item another CTA depends on.
    int pub[S];
    int pub_k = 0, kk = 0;
    auto publish_upto = [&](int k_end, bool block) {  // items [pub_k, k_end)
      while (pub_k < k_end) {
        const int s = pub_k % S;
        const unsigned par = (unsigned)(pub_k / S) & 1u;
        if (block) mbar_wait(&empty[s], par);
        else if (!mbar_test(&empty[s], par)) return;
        if (FUSED && dep_base >= 0 && lane == 0) {
          int g = 0;
#pragma unroll
          for (int q = 0; q < S; ++q)
            if (q == s) g = pub[q];
          __threadfence();
          atomicAdd(p.done + g, 1);
        }
        ++pub_k;
      }
    };
    for (; it < items; ++kk) {
      const int s = kk % S;
      if (kk >= S) {  // stage s must be free (fused: and its item published)
        if (FUSED) publish_upto(kk - S + 1, true);
        else mbar_wait(&empty[s], (unsigned)(kk / S - 1) & 1u);
      }
      GroupSlot<T> gs(p, grp);
      const int rows = rec.y * rec.z;
      if (LAYERED) {
        int* tv = tv_of(s);
#pragma unroll
        for (int j = 0; j < RPL; ++j)
          if (lane + 32 * j < rows) tv[lane + 32 * j] = vn[j];
      }
      if (FUSED && dep_base >= 0) {  // the group's earlier levels must be committed
        while (ld_acquire(p.done + grp) < need) {
          publish_upto(kk, false);
          __nanosleep(32);
        }
        asm volatile("fence.proxy.async.global;\n" ::: "memory");  // generic writes -> TMA reads
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_tx(&full[s], 2u * rows * L::kRowBytes);
        bulk_g2s(so_of(s), gs.c2v + (long long)rec.x * F, rows * L::kRowBytes, &full[s]);
      }
      __syncwarp();
      T* st = st_of(s);
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        if (lane + 32 * j < nrun) {
          const int row = run[j].y & 0xff, len = run[j].y >> 8;
          bulk_g2s(st + row * F, gs.total + (long long)run[j].x * F, len * L::kRowBytes, &full[s]);
        }
      }
      if (FUSED) {
#pragma unroll
        for (int q = 0; q < S; ++q)
          if (q == s) pub[q] = grp;
      }
      it = seek(it + gridDim.x);
      prefetch(it);
      if (FUSED) publish_upto(kk, false);  // eagerly
    }
    if (FUSED) publish_upto(kk, true);  // drain: the items still in flight
  } else {  // ---------------- consumers
    long long it = blockIdx.x;
    for (int kk = 0; it < items; it += gridDim.x) {
      const int lg = item_group(it);
      const int grp = rev ? p.groups - 1 - lg : lg;
      const unsigned am = p.amask[grp];
      if (!am) continue;
      const int s = kk % S;
      const unsigned u = (unsigned)(kk / S);
      ++kk;
      const int4 rec = p.s_rec[item_strip(it, lg)];
      GroupSlot<T> gs(p, grp);
      mbar_wait(&full[s], u & 1u);
      SignSink sk{gs.sign, p.k_info, LAYERED && p.layered_sign != 0, 0, 0};
      const bool act = ((am >> lane) & 1u) != 0;
      if (LAYERED) {  // every lane takes part (the sign ballots need the whole warp)
        strip_checks<T, KERNEL, LAYERED>(so_of(s), st_of(s), tv_of(s), warp, NC, rec.y, rec.z, rec.x, lane, gs.c2v,
                                         gs.total, act, sk);
      } else if (act) {
        strip_checks<T, KERNEL, LAYERED>(so_of(s), st_of(s), tv_of(s), warp, NC, rec.y, rec.z, rec.x, lane, gs.c2v,
                                         gs.total, true, sk);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (LAYERED) {
        if (sk.errs) atomicAdd(&p.errs[grp * F + lane], sk.errs);
        if (sk.ei) atomicAdd(&p.errs_info[grp * F + lane], sk.ei);
      }
    }
  }
}

// VN phase of flooding over VN strips (E:746-756): total = chl + the C2V of
// the VN's edges in vn_edges order (the reference's summation order), sign
// words, error tallies.  Producer: one bulk copy of the strip's chl rows and
// one per run of consecutive stored c2v rows.  Consumers: one VN per warp.
template <typename T, int NC>
__global__ void __launch_bounds__(VnLayout<T, NC>::kThreads, sizeof(T) == 4 ? 2 : 1)
    phase_vn_tma_kernel(const __grid_constant__ PhaseParams p) {
  using L = VnLayout<T, NC>;
  constexpr int F = kFixedFrames, S = kTmaStages, RPL = kTileEdges / 32;
  extern __shared__ __align__(128) unsigned char vn_smem[];
  auto stage = [&](int s) { return (T*)(vn_smem + s * L::kStageBytes); };
  unsigned long long* full = (unsigned long long*)(vn_smem + L::kBarOff);
  unsigned long long* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int nvs = p.n_vstrips;
  const long long items = (long long)p.groups * nvs;
  // optional reverse group order (the check phase ends on the last groups)
  auto vgrp = [&](int g) { return p.vn_reverse ? p.groups - 1 - g : g; };
  if (warp == NC) {  // ---------------- producer
    auto seek = [&](long long i) {
      for (; i < items; i += gridDim.x)
        if (p.amask[vgrp((int)((unsigned)i / (unsigned)nvs))]) break;
      return i;
    };
    long long it = seek(blockIdx.x);
    int4 rec = make_int4(0, 0, 0, 0);
    int nrun = 0;
    int2 run[RPL];
    auto prefetch = [&](long long i) {
      if (i >= items) return;
      const int t = (int)((unsigned)i % (unsigned)nvs);
      rec = p.v_rec[t];
      nrun = p.v_rec[t + 1].w - rec.w;
#pragma unroll
      for (int j = 0; j < RPL; ++j)
        if (lane + 32 * j < nrun) run[j] = p.v_runs[rec.w + lane + 32 * j];
    };
    prefetch(it);
    for (int kk = 0; it < items; ++kk) {
      const int s = kk % S;
      const unsigned u = (unsigned)(kk / S);
      if (kk >= S) mbar_wait(&empty[s], (u - 1) & 1u);
      GroupSlot<T> gs(p, vgrp((int)((unsigned)it / (unsigned)nvs)));
      const int k = rec.y, erows = k * rec.z;
      T* sb = stage(s);
      if (lane == 0) {
        mbar_arrive_tx(&full[s], (unsigned)(erows + k) * L::kRowBytes);
        bulk_g2s(sb + erows * F, gs.chl + (long long)rec.x * F, k * L::kRowBytes, &full[s]);
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        if (lane + 32 * j < nrun) {
          const int row = run[j].y & 0xff, len = run[j].y >> 8;
          bulk_g2s(sb + row * F, gs.c2v + (long long)run[j].x * F, len * L::kRowBytes, &full[s]);
        }
      }
      it = seek(it + gridDim.x);
      prefetch(it);
    }
  } else {  // ---------------- consumers
    long long it = blockIdx.x;
    for (int kk = 0; it < items; it += gridDim.x) {
      const int lgv = (int)((unsigned)it / (unsigned)nvs);
      const int grp = vgrp(lgv);
      const unsigned am = p.amask[grp];
      if (!am) continue;
      const int s = kk % S;
      const unsigned u = (unsigned)(kk / S);
      ++kk;
      const int4 rec = p.v_rec[(int)(it - (long long)lgv * nvs)];
      GroupSlot<T> gs(p, grp);
      const bool act = (am >> lane) & 1u;
      const int k = rec.y, dv = rec.z;
      mbar_wait(&full[s], u & 1u);
      const T* sb = stage(s);
      int errs = 0, ei = 0;
      for (int v = warp; v < k; v += NC) {
        const int n = rec.x + v;
        T tv;
        if (act) {
          tv = sb[(k * dv + v) * F + lane];  // chl
          for (int q = 0; q < dv; ++q) tv += sb[(q * k + v) * F + lane];
          gs.total[(long long)n * F + lane] = tv;
        } else {
          tv = gs.total[(long long)n * F + lane];
        }
        int e_ = 0, i_ = 0;
        sign_row<T>(n, tv, p.k_info, gs.sign, lane, e_, i_);
        if (act) {
          errs += e_;
          ei += i_;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (errs) atomicAdd(&p.errs[grp * F + lane], errs);
      if (ei) atomicAdd(&p.errs_info[grp * F + lane], ei);
    }
  }
}


#endif  // LDPC_PHASE_DECL_ONLY

}  // namespace ldpc
