// ldpc_common.cuh -- shared device types and arithmetic for the sm_100a decoder.
//
// Arithmetic follows the reference engine's operation order exactly
// (/root/reference/pkg/src/ldpc_ids/_engine.py, "E:<line>"): ordered tanh
// products, clip to +-(1-1e-12) before atanh, +-30 clamps, the stable logistic.
// Compiled with -fmad=false so no multiply-add is contracted into an FMA that
// the float64 reference would round twice.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ldpc {

constexpr int kCounters = 8;
enum Counter { C_PROP = 0, C_V2C, C_PRE, C_CI, C_CMP, C_MSEL, C_KHITS, C_KTRIALS };  // E:17-25
enum Kernel { KERNEL_EXACT = 0, KERNEL_MINSUM = 1 };                                // E:27-28
enum Kind {
  KIND_FLOODING = 0, KIND_RBP = 1, KIND_CIRBP = 2, KIND_LMDRBP = 3, KIND_SLMDRBP = 4,
  KIND_LMD_CIRBP = 5, KIND_ME_CIRBP = 6, KIND_ME_LMD_CIRBP = 7, KIND_LAYERED = 8, KIND_ME_RBP = 9
};

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxTreeLevels = 6;  // 32-ary: 32^6 > 1e9 leaves

// Immutable device-side Tanner graph (edge ids in (check, vn) order, codes.py:251-275).
struct DevGraph {
  int N, M, E;
  int max_dv, max_dc, max_items;  // max_items = max two-hop set size
  const int* edge_cn;   // [E]
  const int* edge_vn;   // [E]
  const int* cn_ptr;    // [M+1]
  const int* vn_ptr;    // [N+1]
  const int* vn_edges;  // [E]
  // layered schedule: checks grouped in dependency levels (same result as m = 0..M-1 in order)
  int n_levels;
  const int* level_ptr;     // [n_levels+1]
  const int* level_checks;  // [M]
  // packed records for the dynamic engine (one load instead of a dependent chain)
  const int2* ecv;          // [E]  (check, vn) of edge e
  const int4* erec;         // [E]  (check, vn, vn_ptr[vn], degree of vn) of edge e
  const int2* vrec;         // [N]  (vn_ptr[n], degree of n)
  const int4* vadj;         // [E]  per vn_edges slot k: (f, check i of f, cn_ptr[i], cn_ptr[i+1])
  const int* hop_n;         // [E]  two-hop set size of e (pre-C2V refreshes when e propagates)
  const int* hop_distinct;  // [E]  distinct VNs in that set (E:536-549 candidate count)
  const uint8_t* hop_dup;   // [E]  1 if a VN repeats in that set (4-cycle through n*)
  // optional precomputed two-hop tables (null when they would be too large):
  const long long* hop_ptr; // [E]  offset of e's item records in hop_items
  const int2* hop_items;    // item records (g, packed skip | degree | stage base: dyn_engine.cuh Item)
  const int* hop_sbptr;     // [E]  offset of e's per-VN-slot stage bases in hop_sb
  const int* hop_sb;        // stage base of each vn_edges slot of vn(e) (-1 for cn(e))
  // optional per-VN two-hop VN sets (sorted; null when too large): ME round pairing
  const int* vn2_ptr;       // [N+1]
  const int* vn2;           // N2(v) = VNs sharing a check with v, v included
};

// 32-ary max-tree geometry over `n` leaves (levels 1..L; level L has <= 64 nodes,
// scanned two per lane).
struct TreeGeom {
  int levels;                      // number of internal levels (>= 1)
  int size[kMaxTreeLevels + 1];    // size[0] = leaves
  int off[kMaxTreeLevels + 1];     // node offset of level l (l >= 1) inside the key array
  int total;                       // total internal nodes
};

inline TreeGeom make_tree(int n) {
  TreeGeom t{};
  t.size[0] = n;
  int l = 0, tot = 0;
  do {
    int s = (t.size[l] + 31) / 32;
    ++l;
    t.size[l] = s;
    t.off[l] = tot;
    tot += s;
  } while (t.size[l] > 64 && l < kMaxTreeLevels);
  t.levels = l;
  t.total = tot;
  return t;
}

// ------------------------------------------------------------------ math

template <typename T> struct Num;
template <> struct Num<double> {
  using Key = unsigned long long;
  static constexpr double kLlrMax = 30.0;            // E:13
  static constexpr double kAtanhClip = 1.0 - 1e-12;  // E:14
  static constexpr double kBig = 1e300;              // E:68
  __device__ static double tanh_(double x) { return tanh(x); }
  __device__ static double atanh_(double x) { return atanh(x); }
  __device__ static double exp_(double x) { return exp(x); }
  __device__ static double abs_(double x) { return fabs(x); }
  // order-preserving key for values >= +0; 0 is reserved for padding / excluded
  __device__ static Key key(double v) {
    return v >= 0.0 ? (Key)__double_as_longlong(v) + 1ull : 0ull;
  }
};
template <> struct Num<float> {
  using Key = unsigned int;
  static constexpr float kLlrMax = 30.0f;
  static constexpr float kAtanhClip = (float)(1.0 - 1e-12);  // rounds to 1.0f: fp32 saturates earlier
  static constexpr float kBig = 3.0e38f;
  // fp32 fast mode (no bit-parity obligation; tested statistically): SFU
  // forms with flush-to-zero (ex2 / rcp / lg2 approx), and short series where
  // the SFU forms cancel (small |x|), so relative errors stay ~1e-6.
  __device__ static float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
  __device__ static float rcpf(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
  __device__ static float lg2f(float x) { float y; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
  __device__ static float tanh_(float x) {
    const float a = fabsf(x);
    const float t = 1.0f - 2.0f * rcpf(ex2f(2.8853900817779268f * a) + 1.0f);  // 1 - 2/(e^{2a}+1)
    const float s = a * (1.0f - 0.33333333f * a * a);                             // a - a^3/3
    return copysignf(a < 0.03f ? s : t, x);
  }
  __device__ static float atanh_(float x) {
    const float l = 0.34657359027997264f * lg2f((1.0f + x) * rcpf(1.0f - x));  // 0.5 ln((1+x)/(1-x))
    const float s = x * (1.0f + 0.33333333f * x * x);                           // x + x^3/3
    return fabsf(x) < 0.03f ? s : l;
  }
  __device__ static float exp_(float x) { return __expf(x); }
  __device__ static float abs_(float x) { return fabsf(x); }
  __device__ static Key key(float v) { return v >= 0.0f ? __float_as_uint(v) + 1u : 0u; }
};

template <typename T> __device__ __forceinline__ T clampv(T x) {  // E:31-37
  if (x > Num<T>::kLlrMax) return Num<T>::kLlrMax;
  if (x < -Num<T>::kLlrMax) return -Num<T>::kLlrMax;
  return x;
}

// E:40-46: llr >= 0 ? 1 / (1 + exp(-llr)) : exp(llr) / (1 + exp(llr)).  Both
// branches take the same exponential, exp(-|llr|), so one evaluation and one
// division give the reference's value bit for bit -- without the divergent
// double evaluation when a warp holds both signs.
template <typename T> __device__ __forceinline__ T p0(T llr) {
  const T e = Num<T>::exp_(-Num<T>::abs_(llr));
  return (llr >= T(0) ? T(1) : e) / (T(1) + e);
}

template <typename T> __device__ __forceinline__ T ci_of(T tot, T pre_tot) {
  return Num<T>::abs_(p0(tot) - p0(pre_tot));
}

// CI from a per-VN cache of the total (E:127, E:149, E:173).  float64: the
// cache is p0(total) and CI = |p0(total) - p0(pre_total)| as in the reference.
// float32: p0 rounds to 1.0f for LLRs above ~17, so the cache is the total
// itself and CI = p0(t) p0(-pt) |expm1(pt - t)|, the same quantity without the
// cancellation.
template <typename T> __device__ __forceinline__ T p0_cache(T tot) { return p0(tot); }
template <> __device__ __forceinline__ float p0_cache<float>(float tot) { return tot; }
template <typename T> __device__ __forceinline__ T ci_cached(T cache, T pre_tot) {
  return Num<T>::abs_(cache - p0(pre_tot));
}
template <> __device__ __forceinline__ float ci_cached<float>(float tot, float pre_tot) {
  return p0(tot) * p0(-pre_tot) * fabsf(expm1f(pre_tot - tot));
}

// CI evaluation split for the two-hop refresh (dyn_engine.cuh propagate): every
// lane evaluates ONE transcendental chain -- ci_probe(x) -- and the CI is
// ci_join(cache, probe).  float64: probe = p0(x), join = |cache - probe|; the
// updated VN n* itself needs two probes, p0(total) (its new cache) and
// p0(pre_total), taken on two extra lanes of the same pass (kCiSelfLanes) and
// joined across them.  float32: the probe is the whole cancellation-free CI of
// (cache = total, x = pre_total), one extra lane.
template <typename T> struct CiSplit {
  static constexpr int kSelfLanes = 2;
  __device__ static __forceinline__ T probe(T /*cache*/, T x) { return p0(x); }
  __device__ static __forceinline__ T join(T cache, T probe) { return Num<T>::abs_(cache - probe); }
};
template <> struct CiSplit<float> {
  static constexpr int kSelfLanes = 1;
  __device__ static __forceinline__ float probe(float cache, float x) { return ci_cached<float>(cache, x); }
  __device__ static __forceinline__ float join(float /*cache*/, float probe) { return probe; }
};

// ---- exact check-node algebra: input of a V2C, product, product -> C2V.
//
// float64 (the reference's arithmetic, E:55-66 / E:99-103): input tanh(v/2),
// ordinary products, clip to +-(1-1e-12), 2 atanh.
//
// float32 works in the delta (Gallager phi) domain instead, because tanh(v/2)
// rounds to 1.0f once |v| > ~17 and the product would lose the message: the
// input is the SIGNED phi(|v|) = -ln|tanh(v/2)| (sign bit = sign of tanh(v/2)),
// a "product" adds magnitudes and XORs signs, and the C2V is sign * phi(S) with
// phi(x) = log1p(2 / expm1(x)) = 2 atanh(e^-x) (phi is its own inverse).  The
// reference's clip |prod| <= 1-1e-12 is S >= -ln(1-1e-12) (kSclip), so a
// saturated message is phi(kSclip) = 28.32419 like the reference's, not 30.
// Every step is accurate to a few fp32 ulps at any magnitude (checked against
// float64 over random checks: max 6e-6 relative, abs. below 1).
__device__ __forceinline__ float phif(float x) {  // x >= 0; phi(0) = inf, phi(inf) = 0
  return log1pf(2.0f * Num<float>::rcpf(expm1f(x)));
}
constexpr float kSclip = 9.999779e-13f;  // -ln(fl64(1 - 1e-12)): the E:14 clip in the phi domain

template <typename T> __device__ __forceinline__ T cn_in(T v);  // v: clamped V2C (E:58, E:115, E:159)
template <> __device__ __forceinline__ double cn_in<double>(double v) { return tanh(0.5 * v); }
template <> __device__ __forceinline__ float cn_in<float>(float v) { return copysignf(phif(fabsf(v)), v); }

template <typename T> __device__ __forceinline__ T cn_one();  // empty product
template <> __device__ __forceinline__ double cn_one<double>() { return 1.0; }
template <> __device__ __forceinline__ float cn_one<float>() { return 0.0f; }

template <typename T> __device__ __forceinline__ T cn_mul(T a, T b);
template <> __device__ __forceinline__ double cn_mul<double>(double a, double b) { return a * b; }
template <> __device__ __forceinline__ float cn_mul<float>(float a, float b) {
  const unsigned sg = (__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u;
  return __uint_as_float(__float_as_uint(fabsf(a) + fabsf(b)) | sg);
}

// Product -> C2V (E:62-66 / E:99-103).
template <typename T> __device__ __forceinline__ T atanh_msg(T prod, int count) {
  if (count == 0) return T(0);
  if (prod > Num<T>::kAtanhClip) prod = Num<T>::kAtanhClip;
  else if (prod < -Num<T>::kAtanhClip) prod = -Num<T>::kAtanhClip;
  return clampv(T(2) * Num<T>::atanh_(prod));
}
template <> __device__ __forceinline__ float atanh_msg<float>(float x, int count) {
  if (count == 0) return 0.0f;
  const float m = phif(fmaxf(fabsf(x), kSclip));
  return __uint_as_float(__float_as_uint(m) | (__float_as_uint(x) & 0x80000000u));
}

// C2V of check [a, b) excluding edge `skip` from cached inputs `in`:
// exact kernel: in = tanh(v2c/2) (E:85-103); min-sum: in = v2c (E:67-82).
template <typename T, int KERNEL>
__device__ __forceinline__ T cn_msg_cached(const T* in, int a, int b, int skip) {
  if (KERNEL == KERNEL_EXACT) {
    T prod = cn_one<T>();
    for (int e = a; e < b; ++e)
      if (e != skip) prod = cn_mul(prod, in[e]);
    return atanh_msg(prod, b - a - ((skip >= a && skip < b) ? 1 : 0));
  } else {
    T sign = T(1), mag = Num<T>::kBig;
    int count = 0;
    for (int e = a; e < b; ++e) {
      if (e == skip) continue;
      T v = clampv(in[e]);
      if (v < T(0)) { sign = -sign; v = -v; }
      if (v < mag) mag = v;
      ++count;
    }
    if (count == 0) return T(0);
    return clampv(sign * mag);
  }
}

// want_trace outputs (E:192-217, schedules.py:57) and fused J(gamma) counts
// (sim.py:172-183).
struct TraceOut {
  double* trace;           // [B][i_max+1][2N]: totals then pre-totals, or null
  const double* gammas;    // [n_gamma] (device)
  int n_gamma;
  unsigned long long* jc;  // [i_max+1][n_gamma][2]: (correct, wrong) VNs with D >= gamma, or null
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Loads of the immutable graph tables with an L2 evict_last hint (KEEP = the
// HBM placement of a BG-sized code).  There ~1.7 TB/s of per-frame state streams
// through the 126 MB L2, so a line survives ~70 us while a given table line is
// re-read only every few hundred us: without the hint the ~95 MB of tables
// (two-hop items, edge / VN records) are read from HBM on every update, ~20 %
// of its DRAM requests.
__device__ __forceinline__ unsigned long long l2_keep_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <bool KEEP> __device__ __forceinline__ int ldk(const int* p, unsigned long long pol) {
  if (!KEEP) return *p;
  int v;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
template <bool KEEP> __device__ __forceinline__ int ldk(const uint8_t* p, unsigned long long pol) {
  if (!KEEP) return *p;
  int v;
  asm("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
template <bool KEEP> __device__ __forceinline__ long long ldk(const long long* p, unsigned long long pol) {
  if (!KEEP) return *p;
  long long v;
  asm("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
template <bool KEEP> __device__ __forceinline__ int2 ldk(const int2* p, unsigned long long pol) {
  if (!KEEP) return *p;
  int2 v;
  asm("ld.global.nc.L2::cache_hint.v2.b32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}
template <bool KEEP> __device__ __forceinline__ int4 ldk(const int4* p, unsigned long long pol) {
  if (!KEEP) return *p;
  int4 v;
  asm("ld.global.nc.L2::cache_hint.v4.b32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}

// Warp max of keys (REDUX) -> lowest lane holding it.  Returns (key, lane).
__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long k, int* lane_out) {
  unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
  unsigned mh = __reduce_max_sync(kFull, hi);
  unsigned lo_c = (hi == mh) ? lo : 0u;
  unsigned ml = __reduce_max_sync(kFull, lo_c);
  unsigned bal = __ballot_sync(kFull, hi == mh && lo == ml);
  *lane_out = __ffs(bal) - 1;
  return ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ unsigned warp_max_key(unsigned k, int* lane_out) {
  unsigned m = __reduce_max_sync(kFull, k);
  *lane_out = __ffs(__ballot_sync(kFull, k == m)) - 1;
  return m;
}

// Max key with the smallest companion index among ties (index < 2^31).
__device__ __forceinline__ unsigned long long warp_max_key_minidx(unsigned long long k, int idx,
                                                                  int* idx_out) {
  unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
  unsigned mh = __reduce_max_sync(kFull, hi);
  unsigned ml = __reduce_max_sync(kFull, (hi == mh) ? lo : 0u);
  *idx_out = (int)__reduce_min_sync(kFull, (hi == mh && lo == ml) ? (unsigned)idx : 0xffffffffu);
  return ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ unsigned warp_max_key_minidx(unsigned k, int idx, int* idx_out) {
  unsigned m = __reduce_max_sync(kFull, k);
  *idx_out = (int)__reduce_min_sync(kFull, (k == m) ? (unsigned)idx : 0xffffffffu);
  return m;
}

// Same over the lanes of `mask` only (disjoint masks may reduce concurrently).
__device__ __forceinline__ unsigned long long warp_max_key_minidx_masked(unsigned long long k, int idx,
                                                                         unsigned mask, int* idx_out) {
  unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
  unsigned mh = __reduce_max_sync(mask, hi);
  unsigned ml = __reduce_max_sync(mask, (hi == mh) ? lo : 0u);
  *idx_out = (int)__reduce_min_sync(mask, (hi == mh && lo == ml) ? (unsigned)idx : 0xffffffffu);
  return ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ unsigned warp_max_key_minidx_masked(unsigned k, int idx, unsigned mask,
                                                               int* idx_out) {
  unsigned m = __reduce_max_sync(mask, k);
  *idx_out = (int)__reduce_min_sync(mask, (k == m) ? (unsigned)idx : 0xffffffffu);
  return m;
}

__device__ __forceinline__ int warp_sum(int v) { return (int)__reduce_add_sync(kFull, (unsigned)v); }

__device__ __forceinline__ int warp_incl_scan(int v) {
  int lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int t = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

// ------------------------------------------------------------ lane groups
// A frame is decoded by a group of G lanes (G = 32: one warp; G = 16: two
// frames per warp).  All collectives use the group's mask, so the two halves
// of a warp may diverge freely (independent thread scheduling interleaves them).
template <int G>
struct Grp {
  static constexpr int kG = G;
  unsigned mask_;  // warp-level mask of this group's lanes
  int base_;       // first warp lane of the group
  int lane;        // lane within the group
  unsigned lt;     // group-local mask of lower lanes
  // The mask stays a run-time value even for a whole warp (G = 32, loaded through
  // an opaque move in make()): with an immediate full mask nvcc guards every
  // shuffle / vote / reduction with a convergence check and a WARPSYNC.COLLECTIVE
  // slow path (37 of them in the LMDRBP kernel, +25 % executed instructions).
  __device__ __forceinline__ unsigned mask() const { return mask_; }
  __device__ __forceinline__ int base() const { return G == 32 ? 0 : base_; }
  __device__ __forceinline__ static Grp make() {
    Grp g;
    const int wl = threadIdx.x & 31;
    g.base_ = G == 32 ? 0 : (wl / G) * G;
    g.lane = wl - g.base_;
    if (G == 32) asm("mov.b32 %0, 0xffffffff;" : "=r"(g.mask_));
    else g.mask_ = ((1u << G) - 1u) << g.base_;
    g.lt = (1u << g.lane) - 1u;
    return g;
  }
  __device__ __forceinline__ void sync() const { __syncwarp(mask()); }
  template <typename V> __device__ __forceinline__ V shfl(V v, int src) const {
    return __shfl_sync(mask(), v, base() + src);
  }
  template <typename V> __device__ __forceinline__ V shfl_up(V v, int d) const {
    return __shfl_up_sync(mask(), v, d, G);
  }
  template <typename V> __device__ __forceinline__ V shfl_down(V v, int d) const {
    return __shfl_down_sync(mask(), v, d, G);
  }
  __device__ __forceinline__ unsigned ballot(bool p) const { return __ballot_sync(mask(), p) >> base(); }
  __device__ __forceinline__ bool any(bool p) const { return __any_sync(mask(), p); }
  __device__ __forceinline__ unsigned match_any(int v) const { return __match_any_sync(mask(), v) >> base(); }
  __device__ __forceinline__ unsigned rmax(unsigned v) const { return __reduce_max_sync(mask(), v); }
  __device__ __forceinline__ unsigned rmin(unsigned v) const { return __reduce_min_sync(mask(), v); }
  __device__ __forceinline__ int rsum(int v) const { return (int)__reduce_add_sync(mask(), (unsigned)v); }
  __device__ __forceinline__ int incl_scan(int v) const {
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
      int t = __shfl_up_sync(mask(), v, d, G);
      if (lane >= d) v += t;
    }
    return v;
  }
  // max key (lowest lane among ties); returns group lane of the winner
  __device__ __forceinline__ unsigned long long max_key(unsigned long long k, int* ln) const {
    unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
    unsigned mh = rmax(hi);
    unsigned ml = rmax(hi == mh ? lo : 0u);
    *ln = __ffs(ballot(hi == mh && lo == ml)) - 1;
    return ((unsigned long long)mh << 32) | ml;
  }
  __device__ __forceinline__ unsigned max_key(unsigned k, int* ln) const {
    unsigned m = rmax(k);
    *ln = __ffs(ballot(k == m)) - 1;
    return m;
  }
  __device__ __forceinline__ unsigned long long max_key_only(unsigned long long k) const {
    unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
    unsigned mh = rmax(hi);
    unsigned ml = rmax(hi == mh ? lo : 0u);
    return ((unsigned long long)mh << 32) | ml;
  }
  __device__ __forceinline__ unsigned max_key_only(unsigned k) const { return rmax(k); }
  // max key with the smallest companion index among ties
  __device__ __forceinline__ unsigned long long max_key_minidx(unsigned long long k, int idx, int* out) const {
    unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
    unsigned mh = rmax(hi);
    unsigned ml = rmax(hi == mh ? lo : 0u);
    *out = (int)rmin((hi == mh && lo == ml) ? (unsigned)idx : 0xffffffffu);
    return ((unsigned long long)mh << 32) | ml;
  }
  __device__ __forceinline__ unsigned max_key_minidx(unsigned k, int idx, int* out) const {
    unsigned m = rmax(k);
    *out = (int)rmin(k == m ? (unsigned)idx : 0xffffffffu);
    return m;
  }
};

// Rows of boundary k (E:204-207) -- and, once converged, of every later
// boundary (E:215-217) -- plus their J(gamma) counts, D = |p0(total) -
// p0(pre_total)| in float64 like the reference's post-processing of the trace.
template <typename T, int G, int PS = 1>  // PS: word stride of the total and pre_total columns
__device__ void trace_boundary_rows(const TraceOut& to, int N, int I, const T* total, const T* pretot, long long f,
                                    int k, bool conv, const Grp<G>& w) {
  if (!to.trace && !to.jc) return;
  const int last = conv ? I : k;
  if (to.trace)
    for (int kk = k; kk <= last; ++kk) {
      double* row = to.trace + (f * (I + 1) + kk) * 2ll * N;
      for (int n = w.lane; n < N; n += G) {
        row[n] = (double)total[PS * n];
        row[N + n] = (double)pretot[PS * n];
      }
    }
  if (to.jc)
    for (int gi = 0; gi < to.n_gamma; ++gi) {
      const double gm = to.gammas[gi];
      int ok = 0, bad = 0;
      for (int n = w.lane; n < N; n += G) {
        const double t = (double)total[PS * n];
        const double d = fabs(p0(t) - p0((double)pretot[PS * n]));
        if (d >= gm) {
          if (t >= 0.0) ++ok;
          else ++bad;
        }
      }
      ok = w.rsum(ok);
      bad = w.rsum(bad);
      if (w.lane == 0)
        for (int kk = k; kk <= last; ++kk) {
          if (ok) atomicAdd(&to.jc[((long long)kk * to.n_gamma + gi) * 2], (unsigned long long)ok);
          if (bad) atomicAdd(&to.jc[((long long)kk * to.n_gamma + gi) * 2 + 1], (unsigned long long)bad);
        }
    }
  w.sync();
}

}  // namespace ldpc
