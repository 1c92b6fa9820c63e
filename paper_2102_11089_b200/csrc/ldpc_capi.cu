// ldpc_capi.cu -- C ABI (include/ldpc_b200.h): graph handle, workspace sizing,
// launch policy and kernel dispatch for the sm_100a decoder.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/ldpc_b200.h"
#include "dyn_engine.cuh"
#include "fixed_engine.cuh"
#define LDPC_PHASE_DECL_ONLY
#include "fixed_phase.cuh"
#include "kernel_table.h"

using namespace ldpc;

struct Tiling {  // fixed-engine schedule tiling (see fixed_engine.cuh)
  int n_levels;
  std::vector<int> h_level_tptr;  // host copy (phase engine launches one check grid per level)
  int* level_tptr;
  int* tile_eptr;
  int* te_list;
  int* te_vn;
  int2* te_chk;
  int* tile_cptr;
  int4* tc_rec;
};

struct Strips {  // slot-major check strips of the TMA-fed check phase (fixed_tma.cuh)
  std::vector<int> h_level_sptr;  // strip range of each level (host copy)
  int* lvl_sptr;                  // device copy
  int4* rec;                      // [n_strips + 1] (first c2v row, k, d, first run); sentinel .x/.w = totals
  int2* runs;                     // (first VN, staged row | length << 8)
  int* vn;                        // [E] VN of each staged / stored row
  int* vn_rows;                   // [E] stored c2v row of each vn_edges slot
  int rec_count;                  // number of check strips
  int n_vstrips;                  // VN strips (flooding VN phase)
  int4* v_rec;                    // [n_vstrips + 1] (first VN, k, degree, first run)
  int2* v_runs;                   // (first stored c2v row, staged row | length << 8)
};

struct ldpc_graph {
  DevGraph d;
  int* dev_block;  // one allocation for every device array
  int max_dv, max_dc, max_items;
  int min_dv;  // 0 if some VN has no edge
  Tiling flood, layer;
  Strips sflood, slayer;
  int* strip_block;
  int* tile_block;
  unsigned char* hop_block;  // precomputed two-hop tables (may be null)
  int* pair_block;           // per-VN two-hop VN lists (ME round pairing; may be null)
};

namespace {

thread_local int g_last_launches = 0;
thread_local long long* g_step_log = nullptr;
thread_local int g_log_cap = 0;
thread_local long long g_dump_step = -1;
thread_local double* g_dump_buf = nullptr;

inline int cuda_check(cudaError_t e) {
  if (e != cudaSuccess) {
    fprintf(stderr, "ldpc_b200: CUDA error %s\n", cudaGetErrorString(e));
    return LDPC_ERR_CUDA;
  }
  return LDPC_OK;
}

bool is_dynamic(int kind) { return kind != KIND_FLOODING && kind != KIND_LAYERED; }

__host__ __device__ inline long long align16(long long x) { return (x + 15) & ~15ll; }

// Strips of one schedule: per level (checks in level order), runs of
// consecutive checks with the same degree d, k <= kTileEdges / d per strip,
// rows slot-major (row q*k + c = slot q of check c); c2v rows are stored in
// that order.  Total-row runs: maximal spans of consecutive staged rows whose
// VNs are consecutive (one bulk copy each).
struct HostStrips {
  std::vector<int> level_sptr, rec, runs, vn, vn_rows, v_rec, v_runs;
};
void build_strips(HostStrips& h, const std::vector<int>& lvl_ptr, const std::vector<int>& chk,
                  const std::vector<int>& cn_ptr, const int* edge_vn, const std::vector<int>& vn_edges, int E,
                  int N, bool mark_last) {
  std::vector<int> pos(E);
  // mark_last: bit 31 of s_vn flags the row of each VN's last level (layered sign pass)
  std::vector<int> last_level(N, -1);
  if (mark_last)
    for (size_t L = 0; L + 1 < lvl_ptr.size(); ++L)
      for (int i = lvl_ptr[L]; i < lvl_ptr[L + 1]; ++i)
        for (int e = cn_ptr[chk[i]]; e < cn_ptr[chk[i] + 1]; ++e) last_level[edge_vn[e]] = (int)L;
  h.level_sptr.push_back(0);
  int row = 0;
  for (size_t L = 0; L + 1 < lvl_ptr.size(); ++L) {
    int i = lvl_ptr[L];
    while (i < lvl_ptr[L + 1]) {
      const int d = cn_ptr[chk[i] + 1] - cn_ptr[chk[i]];
      const int kmax = std::max(1, kTileEdges / std::max(1, d));
      int j = i + 1;
      while (j < lvl_ptr[L + 1] && j - i < kmax && cn_ptr[chk[j] + 1] - cn_ptr[chk[j]] == d) ++j;
      const int k = j - i;
      h.rec.insert(h.rec.end(), {row, k, d, (int)h.runs.size() / 2});
      int prev = -2, open = -1;
      for (int q = 0; q < d; ++q)
        for (int c = 0; c < k; ++c) {
          const int e = cn_ptr[chk[i + c]] + q, r = q * k + c, v = edge_vn[e];
          pos[e] = row + r;
          h.vn.push_back(mark_last && last_level[v] == (int)L ? (int)(0x80000000u | (unsigned)v) : v);
          if (open >= 0 && v == prev + 1 && (h.runs[open + 1] >> 8) < 255) {
            h.runs[open + 1] += 1 << 8;
          } else {
            open = (int)h.runs.size();
            h.runs.push_back(v);
            h.runs.push_back(r | (1 << 8));
          }
          prev = v;
        }
      row += k * d;
      i = j;
    }
    h.level_sptr.push_back((int)h.rec.size() / 4);
  }
  h.rec.insert(h.rec.end(), {row, 0, 0, (int)h.runs.size() / 2});
  h.vn_rows.resize(E);
  for (int x = 0; x < E; ++x) h.vn_rows[x] = pos[vn_edges[x]];
}

// VN strips over the stored c2v order `vn_rows`: k consecutive VNs of equal
// degree dv (k*dv <= kTileEdges, k <= kVnStripMax), staged rows s*k + v, runs
// of consecutive stored rows.
void build_vn_strips(HostStrips& h, const int* vn_ptr, int N) {
  int n = 0;
  while (n < N) {
    const int dv = vn_ptr[n + 1] - vn_ptr[n];
    const int kmax = std::min(kVnStripMax, std::max(1, kTileEdges / std::max(1, dv)));
    int j = n + 1;
    while (j < N && j - n < kmax && vn_ptr[j + 1] - vn_ptr[j] == dv) ++j;
    const int k = j - n;
    h.v_rec.insert(h.v_rec.end(), {n, k, dv, (int)h.v_runs.size() / 2});
    int prev = -2, open = -1;
    for (int q = 0; q < dv; ++q)
      for (int v = 0; v < k; ++v) {
        const int r = q * k + v, row = h.vn_rows[vn_ptr[n + v] + q];
        if (open >= 0 && row == prev + 1 && (h.v_runs[open + 1] >> 8) < 255) {
          h.v_runs[open + 1] += 1 << 8;
        } else {
          open = (int)h.v_runs.size();
          h.v_runs.push_back(row);
          h.v_runs.push_back(r | (1 << 8));
        }
        prev = row;
      }
    n = j;
  }
  h.v_rec.insert(h.v_rec.end(), {N, 0, 0, (int)h.v_runs.size() / 2});
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int smem_optin() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (n <= 0) n = 227 * 1024;
  }
  return n;
}

// ---------------------------------------------------------- dynamic engine

struct DynPlan {
  DynParams p;
  int mode;  // 0: all smem, 1: E part in HBM, 2: E+N parts in HBM, 3: all HBM
  int g16;   // 16 lanes per frame (2 frames per warp)
  int warps_per_block;
  int blocks;
  long long ws_bytes;  // including the 256-byte header (work counter)
  int smem_bytes;
};

bool ci_kind(int k) {
  return k == KIND_CIRBP || k == KIND_LMD_CIRBP || k == KIND_ME_CIRBP || k == KIND_ME_LMD_CIRBP;
}
bool me_kind(int k) { return k == KIND_ME_CIRBP || k == KIND_ME_LMD_CIRBP || k == KIND_ME_RBP; }

template <typename T>
void dyn_layout(const ldpc_graph* G, const ldpc_sched_t* s, DynParams& p) {
  using Key = typename Num<T>::Key;
  const long long E = G->d.E, N = G->d.N;
  const long long np = std::max(1, s->n_p);
  const bool ci = ci_kind(s->kind), me = me_kind(s->kind);
  long long o = 0;
  auto take = [&](long long bytes) {
    long long r = o;
    o = align16(o + bytes);
    return r;
  };
  // E part
  p.o_c2v = take(E * sizeof(T));
  p.o_pre = take(E * sizeof(T));
  p.o_in = take(E * sizeof(T));
  p.o_res = take(s->kind == KIND_ME_RBP ? E * sizeof(T) : 0);
  p.slotE_bytes = align16(o);
  // N part
  o = 0;
  // per-VN state: 4-word records (pre_total, p0(total), total, ci)
  p.o_total = take(4 * N * sizeof(T));
  p.pt_on = s->want_trace && !ci ? 1 : 0;
  p.o_inpp = take(s->kind == KIND_ME_LMD_CIRBP ? (N + 3) / 4 * 4 : 0);
  p.fast_sel = (me && s->kind != KIND_ME_RBP && s->n_g <= 255) ? 1 : 0;
  p.o_gid = take(p.fast_sel ? (N + 3) / 4 * 4 : 0);
  p.o_gbits = take(p.fast_sel ? (long long)s->n_g * ((N + 31) / 32) * 4 : 0);
  p.o_members = take(me ? std::max(N, np) * 4 : 0);
  p.o_sel = take(me ? np * 4 : 0);
  p.o_chosen = take(s->kind == KIND_ME_LMD_CIRBP ? np * 4 : 0);
  p.o_tmp = take(s->kind == KIND_ME_RBP ? np * sizeof(T) : 0);
  p.slotN_bytes = align16(o);
  // T part
  o = 0;
  p.rgeo = make_tree((int)E);
  p.cgeo = make_tree((int)N);
  const bool rt = s->kind == KIND_RBP || s->kind == KIND_CIRBP || s->kind == KIND_ME_RBP;
  const bool ct = s->kind == KIND_CIRBP;
  p.o_rl1 = take(rt ? p.rgeo.size[1] * (long long)sizeof(L1Node<Key>) : 0);
  p.o_cl1 = take(ct ? p.cgeo.size[1] * (long long)sizeof(L1Node<Key>) : 0);
  p.slotT_bytes = align16(o);
  // U part (always shared memory): tree levels >= 2
  o = 0;
  p.o_rup = take(rt ? (p.rgeo.total - p.rgeo.size[1]) * (long long)sizeof(Key) : 0);
  p.o_cup = take(ct ? (p.cgeo.total - p.cgeo.size[1]) * (long long)sizeof(Key) : 0);
  p.slotU_bytes = align16(o);
  // per-warp shared scratch
  long long so = 0;
  auto stake = [&](long long bytes) {
    long long r = so;
    so = align16(so + bytes);
    return r;
  };
  const long long dl = std::max<long long>(G->max_items + 2, np + 1);
  p.so_items = (int)stake(G->d.hop_items ? 0 : (long long)G->max_items * 8);  // items built on the fly
  stake(kCounters * 8);  // the frame's work counters sit just below the stage area (Ctx::cntp)
  p.so_stage = (int)stake(std::max<long long>(((long long)G->max_items + 32) * sizeof(T), 32 * (4 + sizeof(Key))));
  p.so_nk = (int)stake((long long)G->max_items * std::max(sizeof(Key), sizeof(T)));  // keys; staged C2V values
  p.so_opre = (int)stake(ci || s->want_trace ? (long long)G->max_items * sizeof(T) : 0);
  p.so_cj = (int)stake(ci || s->want_trace ? (long long)G->max_items * 4 : 0);
  p.so_ck = p.so_opre;  // CI keys overwrite each item's old pre once the refresh has read it
  p.dl_cap = (int)dl;
  p.so_dl0 = (int)stake(2 * dl * 4);  // level-2 change list + its ping-pong partner
  p.so_dl1 = (int)stake(dl * 4);
  p.so_sizes = (int)stake(std::max(1, s->n_g) * 4);
  p.so_hist = (int)stake(p.fast_sel ? s->n_g * 4 : 0);
  // multi-edge round pairing (dyn_engine.cuh me_pair_step): a second copy of
  // the per-update scratch [so_items, so_sizes) for the second half-warp
  // (the pairing build exists for float64 exact, untraced; elsewhere the flag is ignored)
  p.me_pairs = (s->kind == KIND_ME_CIRBP || s->kind == KIND_ME_LMD_CIRBP) && G->d.vn2 && sizeof(T) == 8 &&
               s->kernel == KERNEL_EXACT && !s->want_trace && !(s->variant & LDPC_VARIANT_LANES16) &&
               (s->variant & LDPC_VARIANT_ME_PAIRS) ? 1 : 0;
  p.pair_cap = (int)((p.so_nk - p.so_stage) / 4);
  p.so_pair = (int)stake(p.me_pairs ? (long long)(p.so_sizes - p.so_items) : 0);
  p.scratch_bytes = (int)align16(so);
}

template <typename T>
void* pick_dyn_kernel(int kernel, int mode, int kind, int g16, int trace, int pairs) {
  return ldpc_dyn_kernel(sizeof(T) == 8, kernel, mode, kind, g16, trace, pairs);
}

template <typename T>
void* pick_fixed_kernel(int kernel, int layered) {
  return ldpc_fixed_kernel(sizeof(T) == 8, kernel, layered);
}

template <typename T>
int dyn_occupancy(void* fn, int wpb, int smem_bytes) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, wpb * 32, smem_bytes) != cudaSuccess) occ = 0;
  return occ;
}

template <typename T>
int dyn_plan(const ldpc_graph* G, const ldpc_sched_t* s, long long B, DynPlan& pl) {
  memset(&pl, 0, sizeof(pl));
  DynParams& p = pl.p;
  dyn_layout<T>(G, s, p);
  const long long optin = smem_optin() - 1024;
  const long long sE = p.slotE_bytes, sN = p.slotN_bytes, sT = p.slotT_bytes, sc = p.scratch_bytes + p.slotU_bytes;
  const long long sh[4] = {sE + sN + sT + sc, sN + sT + sc, sT + sc, sc};  // shared bytes per frame
  const long long hb[4] = {0, sE, sE + sN, sE + sN + sT};                 // HBM bytes per frame
  struct Cand { int mode, g16, wpb; long long smem; int occ; long long frames; };
  const int lanes_force = (s->variant & LDPC_VARIANT_LANES32) ? 32 : (s->variant & LDPC_VARIANT_LANES16) ? 16 : 0;
  auto make = [&](int mode, int g16) {
    Cand c{mode, g16, 0, 0, 0, 0};
    const int fpw = g16 ? 2 : 1;
    const long long per = sh[mode] * fpw;  // shared bytes per warp
    if (per > optin) return c;
    void* fn = pick_dyn_kernel<T>(s->kernel, mode, s->kind, g16, s->want_trace, p.me_pairs);
    if (!fn) return c;
    // warps per block: the size (<= 8) that leaves the most frames resident
    // (shared memory per SM is allocated in whole blocks)
    const int wmax = per > 32 * 1024 ? 1 : (int)std::min<long long>(8, optin / std::max<long long>(per, 1));
    for (int w = std::max(1, wmax); w >= 1; w = w > 2 ? w / 2 : w - 1) {
      const long long sm = per * w;
      const int occ = dyn_occupancy<T>(fn, w, (int)sm);
      const long long fr = std::min<long long>((long long)occ * w * fpw * sm_count(), B);
      if (fr > c.frames) {
        c.wpb = w;
        c.smem = sm;
        c.occ = occ;
        c.frames = fr;
      }
    }
    return c;
  };
  std::vector<Cand> cands;
  for (int m = 0; m < 4; ++m)
    for (int g16 = 0; g16 < 2; ++g16) {
      if (lanes_force == 16 && !g16) continue;
      if (lanes_force == 32 && g16) continue;
      Cand c = make(m, g16);
      if (c.occ > 0) cands.push_back(c);
    }
  const int want_mode = s->placement == 1 ? 3 : s->placement == 2 ? 1 : s->placement == 3 ? 0
                        : s->placement == 4 ? 2 : -1;
  Cand ch{-1, 0, 0, 0, 0, 0};
  // The update chain is latency-bound, so resident frames decide throughput
  // (measured on C0-C2).  Most resident frames wins; within 10% the more
  // on-chip mode, then 32 lanes per frame, wins.
  long long best = 0;
  for (auto& c : cands)
    if (want_mode < 0 || c.mode == want_mode) best = std::max(best, c.frames);
  for (int m = 0; m < 4 && ch.mode < 0; ++m)
    for (int g16 = 0; g16 < 2 && ch.mode < 0; ++g16)
      for (auto& c : cands)
        if (c.mode == m && c.g16 == g16 && (want_mode < 0 || m == want_mode) && c.frames * 10 >= best * 9) ch = c;
  if (ch.mode < 0 || ch.occ <= 0) return LDPC_ERR_UNSUPPORTED;
  pl.mode = ch.mode;
  pl.g16 = ch.g16;
  pl.warps_per_block = ch.wpb;
  pl.smem_bytes = (int)ch.smem;
  const int fpw = ch.g16 ? 2 : 1;
  long long blocks = (long long)ch.occ * sm_count();
  long long max_frames = B;
  if (s->max_resident > 0) max_frames = std::min<long long>(max_frames, s->max_resident);
  const long long hbm_per_frame = hb[ch.mode];
  if (hbm_per_frame > 0) max_frames = std::min(max_frames, std::max<long long>(1, (24ll << 30) / hbm_per_frame));
  const long long fpb = (long long)pl.warps_per_block * fpw;
  long long need_blocks = (max_frames + fpb - 1) / fpb;
  blocks = std::max<long long>(1, std::min(blocks, need_blocks));
  pl.blocks = (int)blocks;
  pl.ws_bytes = 256 + blocks * fpb * hbm_per_frame;
  return LDPC_OK;
}

// ------------------------------------------------------------ fixed engine

struct FixedPlan {
  FixedParams p;
  void* fn;
  int threads, blocks, smem_bytes;
  long long ws_bytes;
};

int fixed_engine_choice(const ldpc_sched_t* s, long long B);

// traced flooding / layered (fixed_trace.cu): one warp per frame, state in HBM
struct FixedTracePlan {
  FixedTraceParams p;
  int blocks;
  long long ws_bytes;
};

template <typename T>
int fixed_trace_plan(const ldpc_graph* G, const ldpc_sched_t* s, long long B, FixedTracePlan& pl) {
  memset(&pl, 0, sizeof(pl));
  pl.p.slot_bytes = align16((3ll * G->d.E + 3ll * G->d.N) * sizeof(T));
  void* fn = ldpc_fixed_trace_kernel(sizeof(T) == 8, s->kernel, s->kind == KIND_LAYERED);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kTraceWarps * 32, 0) != cudaSuccess || occ < 1) occ = 1;
  long long blocks = std::min<long long>((long long)occ * sm_count(), (B + kTraceWarps - 1) / kTraceWarps);
  if (s->max_resident > 0) blocks = std::min<long long>(blocks, std::max(1, s->max_resident / kTraceWarps));
  const long long cap = std::max<long long>(1, (24ll << 30) / (pl.p.slot_bytes * kTraceWarps));
  pl.blocks = (int)std::max<long long>(1, std::min(blocks, cap));
  pl.ws_bytes = 256 + (long long)pl.blocks * kTraceWarps * pl.p.slot_bytes;
  return LDPC_OK;
}

template <typename T>
int fixed_plan(const ldpc_graph* G, const ldpc_sched_t* s, long long B, FixedPlan& pl) {
  memset(&pl, 0, sizeof(pl));
  const int F = kFixedFrames;
  const bool layered = s->kind == KIND_LAYERED;
  pl.p.slot_bytes = align16((2ll * G->d.N + G->d.E) * F * sizeof(T) + 4ll * G->d.N);
  pl.threads = 512;
  const bool pipe = fixed_engine_choice(s, B) == 2;
  pl.smem_bytes = (pipe ? 1 + 2 * kFixedStages : (layered ? 2 : 1)) * kTileEdges * F * (int)sizeof(T);
  if (pl.smem_bytes > smem_optin() - 1024) return LDPC_ERR_UNSUPPORTED;
  void* fn = pipe ? ldpc_fixed_pipe_kernel(sizeof(T) == 8, s->kernel, layered) : pick_fixed_kernel<T>(s->kernel, layered);
  pl.fn = fn;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem_bytes);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, pl.threads, pl.smem_bytes) != cudaSuccess || occ < 1) occ = 1;
  long long groups = (B + F - 1) / F;
  long long blocks = std::min<long long>((long long)occ * sm_count(), groups);
  if (s->max_resident > 0) blocks = std::min<long long>(blocks, std::max(1, s->max_resident / F));
  long long cap = std::max<long long>(1, (24ll << 30) / pl.p.slot_bytes);
  blocks = std::max<long long>(1, std::min(blocks, cap));
  pl.blocks = (int)blocks;
  pl.ws_bytes = 256 + blocks * pl.p.slot_bytes;
  const Tiling& tl = layered ? G->layer : G->flood;
  pl.p.n_levels = tl.n_levels;
  pl.p.level_tptr = tl.level_tptr;
  pl.p.tile_eptr = tl.tile_eptr;
  pl.p.te_list = tl.te_list;
  pl.p.te_vn = tl.te_vn;
  pl.p.te_chk = tl.te_chk;
  pl.p.tile_cptr = tl.tile_cptr;
  pl.p.tc_rec = tl.tc_rec;
  return LDPC_OK;
}

// ------------------------------------------------- fixed schedules, phase engine

// Engine choice for flooding / layered: "phase" (batch-wide phases, default),
// "tile" (one persistent CTA per 32-frame group), "pipe" (tile + cp.async).
int fixed_engine_choice(const ldpc_sched_t* s, long long B) {
  switch (s->variant & LDPC_VARIANT_FIXED_MASK) {
    case LDPC_VARIANT_FIXED_PHASE: return 0;
    case LDPC_VARIANT_FIXED_TILE: return 1;
    case LDPC_VARIANT_FIXED_PIPE: return 2;
    default: break;
  }
  // float64 with many waves of 32-frame groups: the per-group persistent
  // kernel keeps each group's state L2-hot across iterations and has no tail
  // to speak of (measured on C1: 1.2-1.8x the phase engine); otherwise phases.
  const long long groups = (B + kFixedFrames - 1) / kFixedFrames;
  if (s->precision == LDPC_F64 && groups >= 16ll * sm_count()) return 1;
  return 0;
}

// Phase engine: the TMA-fed strip kernels (fixed_tma.cuh) except float64
// flooding, where the load-wait-compute kernel measured faster (C3: 27 vs 40 ms
// per check launch); LDPC_VARIANT_CHECK_TMA / _LEGACY override.
bool phase_use_tma(const ldpc_sched_t* s) {
  if (s->variant & LDPC_VARIANT_CHECK_TMA) return true;
  if (s->variant & LDPC_VARIANT_CHECK_LEGACY) return false;
  return !(s->precision == LDPC_F64 && s->kind == KIND_FLOODING);
}

struct PhasePlan {
  long long slot, sign_off, groups, chunk, state_off, ws_bytes;
  int smem_check;
};

template <typename T>
int phase_plan(const ldpc_graph* G, long long B, PhasePlan& pl) {
  const long long F = kFixedFrames, N = G->d.N, E = G->d.E;
  pl.sign_off = align16((2 * N + E) * F * (long long)sizeof(T));
  pl.slot = align16(pl.sign_off + 4 * N);
  pl.groups = (B + F - 1) / F;
  const long long per_group_state = 4 + 4 + 3 * 4 * F + 4;  // amask, unsat, errs, errs_info, iters, done
  pl.chunk = std::max<long long>(1, std::min(pl.groups, (24ll << 30) / (pl.slot + per_group_state)));
  // the strip kernels index (group, strip) items in 32 bits
  const long long strips = std::max<long long>({1, (long long)G->sflood.rec_count, (long long)G->slayer.rec_count,
                                                (long long)G->sflood.n_vstrips});
  pl.chunk = std::min(pl.chunk, std::max<long long>(1, 0x7fffffffll / strips));
  pl.state_off = 256 + pl.chunk * pl.slot;
  pl.ws_bytes = pl.state_off + align16(pl.chunk * per_group_state) + 64;
  pl.smem_check = 3 * kTileEdges * (int)F * (int)sizeof(T);
  return LDPC_OK;
}

template <typename T>
int phase_decode(const ldpc_graph* G, const void* llr, long long B, const ldpc_sched_t* s, int8_t* u_hat,
                 int64_t* props, uint8_t* conv, int64_t* counters, int32_t* biterr, int32_t* biterr_info,
                 void* ws, size_t ws_bytes, cudaStream_t st) {
  PhasePlan pl;
  phase_plan<T>(G, B, pl);
  if ((long long)ws_bytes < pl.ws_bytes) return LDPC_ERR_WORKSPACE;
  const bool layered = s->kind == KIND_LAYERED;
  const PhaseKernels K = ldpc_phase_kernels(sizeof(T) == 8, s->kernel, layered);
  const Tiling& tl = layered ? G->layer : G->flood;
  const Strips& sp = layered ? G->slayer : G->sflood;
  cudaFuncSetAttribute(K.check, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem_check);
  // check phase: the TMA-fed warp-specialised kernel unless LDPC_VARIANT_CHECK_LEGACY.
  // Layered runs one check launch per dependency level.  (Round 1 also tried all
  // levels in one launch ordered by per-group dependency counters: within 3 % --
  // the check kernel's DRAM traffic, not the relaunches, bounds the sweep -- and
  // it needs every CTA co-resident, so it was removed; fusing the flooding check
  // and VN phases measured 1.5x slower: VN items stall on the slowest CTA.)
  const bool use_tma = phase_use_tma(s);
  // layered: sign words / error tallies from the check phase (every VN has an
  // edge, so each VN's last-level commit sees its final total);
  // LDPC_VARIANT_NO_LAYERED_SIGN runs the separate VN pass instead
  const bool layered_sign = layered && use_tma && G->min_dv > 0 && !(s->variant & LDPC_VARIANT_NO_LAYERED_SIGN);
  if (use_tma) {
    cudaFuncSetAttribute(K.check_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, K.tma_smem);
    cudaFuncSetAttribute(K.vn_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, K.vn_smem);
    cudaFuncSetAttribute(K.check_tma_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, K.tma_smem);
  }
  auto grid_of = [&](void* fn, int smem, long long items, int threads = kPhaseThreads) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess || occ < 1) occ = 1;
    return (int)std::max<long long>(1, std::min<long long>((long long)occ * sm_count(), items));
  };
  const int I = s->i_max;
  int launches = 0;
  for (long long g0 = 0; g0 < pl.groups; g0 += pl.chunk) {
    PhaseParams p;
    memset(&p, 0, sizeof(p));
    p.g = G->d;
    p.kernel = s->kernel;
    p.i_max = I;
    p.k_info = s->k_info;
    p.llr = llr;
    p.llr_f64 = s->llr_f64;
    p.f_base = g0 * kFixedFrames;
    p.B = std::min<long long>(B - p.f_base, pl.chunk * kFixedFrames);
    p.groups = (int)((p.B + kFixedFrames - 1) / kFixedFrames);
    p.u_hat = u_hat;
    p.prop = (long long*)props;
    p.conv = conv;
    p.counters = (long long*)counters;
    p.biterr = biterr;
    p.biterr_info = biterr_info;
    p.ws = (unsigned char*)ws + 256;
    p.slot_bytes = pl.slot;
    p.sign_off = pl.sign_off;
    unsigned char* sb = (unsigned char*)ws + pl.state_off;
    p.amask = (unsigned*)sb;
    p.unsat = p.amask + pl.chunk;
    p.errs = (int*)(p.unsat + pl.chunk);
    p.errs_info = p.errs + pl.chunk * kFixedFrames;
    p.iters = p.errs_info + pl.chunk * kFixedFrames;
    p.done = p.iters + pl.chunk * kFixedFrames;
    p.s_lvl = sp.lvl_sptr;
    p.layered_sign = layered_sign ? 1 : 0;
    p.vn_reverse = 0;
    p.lwin = 0;
    p.level_tptr = tl.level_tptr;
    p.tile_eptr = tl.tile_eptr;
    p.te_list = tl.te_list;
    p.te_vn = tl.te_vn;
    p.te_chk = tl.te_chk;
    p.tile_cptr = tl.tile_cptr;
    p.tc_rec = tl.tc_rec;
    p.s_rec = sp.rec;
    p.s_runs = sp.runs;
    p.s_vn = sp.vn;
    p.vn_rows = use_tma ? sp.vn_rows : G->d.vn_edges;  // legacy flooding stores c2v in edge order
    p.v_rec = sp.v_rec;
    p.v_runs = sp.v_runs;
    p.n_vstrips = sp.n_vstrips;
    if (int rc = cuda_check(cudaMemsetAsync(p.errs, 0, 2ll * pl.chunk * kFixedFrames * 4, st))) return rc;
    if (int rc = cuda_check(cudaMemsetAsync(p.done, 0, pl.chunk * 4, st))) return rc;
    const long long G_ = p.groups;
    const long long vch = (G->d.N + kPhaseVnChunk - 1) / kPhaseVnChunk;
    const long long ech = ((long long)G->d.E + kPhaseVnChunk * 8 - 1) / (kPhaseVnChunk * 8);
    const long long cch = (G->d.M + kPhaseChkChunk - 1) / kPhaseChkChunk;
    auto launch = [&](void* fn, long long items, int smem, void** args, int threads = kPhaseThreads,
                      bool persistent = true) {
      ++launches;
      const int grid = persistent ? grid_of(fn, smem, items, threads) : (int)items;
      return cuda_check(cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, st));
    };
    void* a1[] = {&p};
    int k = 0, chk = 0;
    void* af[] = {&p, &k, &chk};
    const long long fin_blocks = (G_ * kFixedFrames + 255) / 256;
    if (int rc = launch(K.init, G_ * (vch + ech), 0, a1)) return rc;
    if (I == 0)
      if (int rc = launch(K.syndrome, G_ * cch, 0, a1)) return rc;
    k = 0;
    chk = I == 0 ? 1 : 0;
    if (int rc = launch(K.finalize, fin_blocks, 0, af, 256, false)) return rc;
    for (int it = 1; it <= I; ++it) {
      const std::vector<int>& lvl = use_tma ? sp.h_level_sptr : tl.h_level_tptr;
      const int nlev = (int)lvl.size() - 1;
      {
        for (int L = 0; L < nlev; ++L) {
          int t_lo = lvl[L], t_hi = lvl[L + 1];
          if (t_hi <= t_lo) continue;
          if (use_tma) {
            // alternate the group order level to level: a level starts on the
            // groups the previous one ended with (their totals are L2-hot)
            int L0 = L, L1 = L + 1, dep = -1, rev = (L & 1) ? 1 : 0;
            void* ac[] = {&p, &L0, &L1, &dep, &rev};
            // layered: the FUSED build (spill-free allocation), one level per launch
            void* fn = layered ? K.check_tma_fused : K.check_tma;
            if (int rc = launch(fn, G_ * (t_hi - t_lo), K.tma_smem, ac, K.tma_threads)) return rc;
          } else {
            void* ac[] = {&p, &t_lo, &t_hi};
            if (int rc = launch(K.check, G_ * (t_hi - t_lo), pl.smem_check, ac)) return rc;
          }
        }
      }
      if (use_tma && !layered) {
        if (int rc = launch(K.vn_tma, G_ * sp.n_vstrips, K.vn_smem, a1, K.vn_threads)) return rc;
      } else if (!layered_sign) {
        if (int rc = launch(K.vn, G_ * vch, 0, a1)) return rc;
      }
      if (int rc = launch(K.syndrome, G_ * cch, 0, a1)) return rc;
      k = it;
      chk = 1;
      if (int rc = launch(K.finalize, fin_blocks, 0, af, 256, false)) return rc;
    }
    if (int rc = launch(K.output, G_ * vch, 0, a1)) return rc;
  }
  g_last_launches = launches;
  return LDPC_OK;
}

int validate(const ldpc_graph* G, const ldpc_sched_t* s, long long B) {
  if (!G || !s || B < 0) return LDPC_ERR_INVALID;
  if (s->kind < 0 || s->kind > KIND_ME_RBP) return LDPC_ERR_INVALID;
  if (s->kernel != KERNEL_EXACT && s->kernel != KERNEL_MINSUM) return LDPC_ERR_INVALID;
  if (!(s->gamma >= 0.0 && s->gamma < 1.0)) return LDPC_ERR_INVALID;  // schedules.py:37-38
  if (s->n_p < 1 || s->n_g < 1) return LDPC_ERR_INVALID;              // schedules.py:39-40
  if (s->i_max < 0) return LDPC_ERR_INVALID;                          // schedules.py:41-42
  if (s->precision != LDPC_F64 && s->precision != LDPC_F32) return LDPC_ERR_INVALID;
  if ((s->kind == KIND_ME_CIRBP || s->kind == KIND_ME_LMD_CIRBP) && s->n_p > G->d.N)
    return LDPC_ERR_INVALID;  // schedules.py:136-137
  if (is_dynamic(s->kind) && G->max_dv > 32) return LDPC_ERR_UNSUPPORTED;
  // packed two-hop item records (dyn_engine.cuh Item): degree and stage offsets must fit
  if (is_dynamic(s->kind) && (G->max_dc > kItemMaxDegree || G->max_items + G->max_dv > kItemMaxStage))
    return LDPC_ERR_UNSUPPORTED;
  if (!is_dynamic(s->kind) && G->max_dc > kTileEdges) return LDPC_ERR_UNSUPPORTED;
  if (s->n_g > 4096) return LDPC_ERR_UNSUPPORTED;
  if (s->placement < 0 || s->placement > 4) return LDPC_ERR_INVALID;
  if (s->want_trace != 0 && s->want_trace != 1) return LDPC_ERR_INVALID;
  if (s->variant & ~0x1ff) return LDPC_ERR_INVALID;
  if ((s->variant & LDPC_VARIANT_LANES32) && (s->variant & LDPC_VARIANT_LANES16)) return LDPC_ERR_INVALID;
  if ((s->variant & LDPC_VARIANT_CHECK_TMA) && (s->variant & LDPC_VARIANT_CHECK_LEGACY)) return LDPC_ERR_INVALID;
  return LDPC_OK;
}

template <typename T>
int decode_impl(const ldpc_graph* G, const void* llr, long long B, const ldpc_sched_t* s,
                int8_t* u_hat, int64_t* props, uint8_t* conv, int64_t* counters, int32_t* biterr,
                int32_t* biterr_info, int32_t* kh, int32_t* kt, void* ws, size_t ws_bytes,
                const TraceOut& tr, cudaStream_t st) {
  g_last_launches = 0;
  if (B == 0) return LDPC_OK;
  unsigned long long* next = (unsigned long long*)ws;
  if (!is_dynamic(s->kind) && s->want_trace) {
    FixedTracePlan pl;
    if (int rc = fixed_trace_plan<T>(G, s, B, pl)) return rc;
    if ((long long)ws_bytes < pl.ws_bytes) return LDPC_ERR_WORKSPACE;
    FixedTraceParams& p = pl.p;
    p.g = G->d;
    p.i_max = s->i_max;
    p.k_info = s->k_info;
    p.llr = llr;
    p.llr_f64 = s->llr_f64;
    p.B = B;
    p.u_hat = u_hat;
    p.prop = (long long*)props;
    p.conv = conv;
    p.counters = (long long*)counters;
    p.biterr = biterr;
    p.biterr_info = biterr_info;
    p.next = next;
    p.ws = (unsigned char*)ws + 256;
    p.tr = tr;
    if (int rc = cuda_check(cudaMemsetAsync(next, 0, 16, st))) return rc;
    void* fn = ldpc_fixed_trace_kernel(sizeof(T) == 8, s->kernel, s->kind == KIND_LAYERED);
    void* args[] = {&p};
    if (int rc = cuda_check(cudaLaunchKernel(fn, dim3(pl.blocks), dim3(kTraceWarps * 32), args, 0, st))) return rc;
    g_last_launches = 1;
    return LDPC_OK;
  }
  if (is_dynamic(s->kind)) {
    DynPlan pl;
    if (int rc = dyn_plan<T>(G, s, B, pl)) return rc;
    if ((long long)ws_bytes < pl.ws_bytes) return LDPC_ERR_WORKSPACE;
    if (s->kind == KIND_CIRBP && (!kh || !kt)) return LDPC_ERR_INVALID;
    DynParams& p = pl.p;
    p.g = G->d;
    p.kind = s->kind;
    p.kernel = s->kernel;
    p.i_max = s->i_max;
    p.n_p = s->n_p;
    p.n_g = s->n_g;
    p.k_info = s->k_info;
    p.gamma = s->gamma;
    p.seed = s->selection_seed;
    p.llr = llr;
    p.llr_f64 = s->llr_f64;
    p.B = B;
    p.u_hat = u_hat;
    p.prop = (long long*)props;
    p.conv = conv;
    p.counters = (long long*)counters;
    p.biterr = biterr;
    p.biterr_info = biterr_info;
    p.kh = kh;
    p.kt = kt;
    p.next = next;
    p.step_log = g_step_log;
    p.dbg_full_tree = (s->variant & LDPC_VARIANT_FULL_TREE) ? 1 : 0;
    p.dump_step = g_dump_step;
    p.dump_buf = g_dump_buf;
    p.log_cap = g_log_cap;
    p.ws = (unsigned char*)ws + 256;
    p.tr = tr;
    if (int rc = cuda_check(cudaMemsetAsync(next, 0, 16, st))) return rc;
    void* fn = pick_dyn_kernel<T>(s->kernel, pl.mode, s->kind, pl.g16, s->want_trace, pl.p.me_pairs);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem_bytes);
    void* args[] = {&p};
    if (int rc = cuda_check(cudaLaunchKernel(fn, dim3(pl.blocks), dim3(pl.warps_per_block * 32), args,
                                             pl.smem_bytes, st)))
      return rc;
    g_last_launches = 1;
  } else if (fixed_engine_choice(s, B) == 0) {
    return phase_decode<T>(G, llr, B, s, u_hat, props, conv, counters, biterr, biterr_info, ws, ws_bytes, st);
  } else {
    FixedPlan pl;
    if (int rc = fixed_plan<T>(G, s, B, pl)) return rc;
    if ((long long)ws_bytes < pl.ws_bytes) return LDPC_ERR_WORKSPACE;
    FixedParams& p = pl.p;
    p.g = G->d;
    p.kind = s->kind;
    p.kernel = s->kernel;
    p.i_max = s->i_max;
    p.k_info = s->k_info;
    p.llr = llr;
    p.llr_f64 = s->llr_f64;
    p.B = B;
    p.u_hat = u_hat;
    p.prop = (long long*)props;
    p.conv = conv;
    p.counters = (long long*)counters;
    p.biterr = biterr;
    p.biterr_info = biterr_info;
    p.next = next;
    p.ws = (unsigned char*)ws + 256;
    if (int rc = cuda_check(cudaMemsetAsync(next, 0, 16, st))) return rc;
    if (int rc = cuda_check(cudaMemsetAsync(conv, 0, B, st))) return rc;
    void* args[] = {&p};
    if (int rc = cuda_check(cudaLaunchKernel(pl.fn, dim3(pl.blocks), dim3(pl.threads), args, pl.smem_bytes, st)))
      return rc;
    g_last_launches = 1;
  }
  return LDPC_OK;
}

// ------------------------------------------------------------ select_vns

__global__ void select_vns_kernel(const double* ci, const uint8_t* mask, int N, int n_g, int n_p,
                                  long long seed, int* out, int* count_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  Ctx<double, 32> c;
  memset(&c, 0, sizeof(c));
  c.w = Grp<32>::make();
  c.lane = c.w.lane;
  c.nb = const_cast<double*>(ci) - 3;  // dense CI vector: ci(n) = nb[cs * n + 3]
  c.cs = 1;
  c.sizes = (int*)smem;
  c.members = (int*)(smem + align16((long long)n_g * 4));
  uint8_t* excl = (uint8_t*)(smem + align16((long long)n_g * 4) + align16((long long)(N > n_p ? N : n_p) * 4));
  c.rng = seed;
  for (int n = c.lane; n < N; n += 32) excl[n] = mask ? (mask[n] ? 0 : 1) : 0;
  __syncwarp();
  DynParams p;
  memset(&p, 0, sizeof(p));
  p.g.N = N;
  p.n_g = n_g;
  int cnt = select_vns<double, 32>(p, c, excl, n_p, out);
  if (c.lane == 0) *count_out = cnt;
}

}  // namespace

// ================================================================== C ABI

// replay helpers (ldpc_decode_replay below)
namespace {
template <typename T>
void replay_layout(const ldpc_graph* G, const ldpc_sched_t* s, DynParams& p) {
  ldpc_sched_t r = *s;
  r.kind = KIND_LMD_CIRBP;  // a CI kind without trees: pre_total and CI maintained
  r.want_trace = 0;
  dyn_layout<T>(G, &r, p);
}
int replay_check(const ldpc_graph* G, const ldpc_sched_t* s, long long B) {
  if (!G || !s || B < 0) return LDPC_ERR_INVALID;
  if (s->kernel != KERNEL_EXACT && s->kernel != KERNEL_MINSUM) return LDPC_ERR_INVALID;
  if (s->precision != LDPC_F64 && s->precision != LDPC_F32) return LDPC_ERR_INVALID;
  if (G->max_dv > 32 || G->max_dc > kItemMaxDegree || G->max_items + G->max_dv > kItemMaxStage)
    return LDPC_ERR_UNSUPPORTED;
  return LDPC_OK;
}
}  // namespace

extern "C" {

int ldpc_version(void) { return 10000; }

int ldpc_last_launch_count(void) { return g_last_launches; }

int ldpc_set_state_dump(int64_t step, double* dev_buf) {
  g_dump_step = step;
  g_dump_buf = step >= 0 ? dev_buf : nullptr;
  return LDPC_OK;
}

int ldpc_set_step_log(int64_t* dev_log, int32_t cap) {
  if (cap < 0 || (cap > 0 && !dev_log)) return LDPC_ERR_INVALID;
  g_step_log = cap > 0 ? (long long*)dev_log : nullptr;
  g_log_cap = cap;
  return LDPC_OK;
}

const char* ldpc_strerror(int code) {
  switch (code) {
    case LDPC_OK: return "ok";
    case LDPC_ERR_INVALID: return "invalid argument";
    case LDPC_ERR_UNSUPPORTED: return "graph or configuration exceeds a kernel limit";
    case LDPC_ERR_CUDA: return "CUDA runtime error";
    case LDPC_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown error";
  }
}

int ldpc_graph_create(const int32_t* edge_cn, const int32_t* edge_vn, const int32_t* cn_ptr,
                      const int32_t* vn_ptr, const int32_t* vn_edges, int32_t N, int32_t M,
                      int32_t E, ldpc_graph_t** out) {
  if (!out || N <= 0 || M <= 0 || E <= 0 || !edge_cn || !edge_vn || !cn_ptr || !vn_ptr || !vn_edges)
    return LDPC_ERR_INVALID;
  *out = nullptr;
  // validate the CSR/CSC contract of build_tanner (codes.py:251-275)
  if (cn_ptr[0] != 0 || cn_ptr[M] != E || vn_ptr[0] != 0 || vn_ptr[N] != E) return LDPC_ERR_INVALID;
  for (int e = 0; e < E; ++e) {
    if (edge_cn[e] < 0 || edge_cn[e] >= M || edge_vn[e] < 0 || edge_vn[e] >= N) return LDPC_ERR_INVALID;
    if (e > 0 && (edge_cn[e] < edge_cn[e - 1] || (edge_cn[e] == edge_cn[e - 1] && edge_vn[e] <= edge_vn[e - 1])))
      return LDPC_ERR_INVALID;  // edges must be in strictly increasing (check, vn) order
  }
  for (int m = 0; m < M; ++m)
    for (int e = cn_ptr[m]; e < cn_ptr[m + 1]; ++e)
      if (e < 0 || e >= E || edge_cn[e] != m) return LDPC_ERR_INVALID;
  for (int n = 0; n < N; ++n)
    for (int k = vn_ptr[n]; k < vn_ptr[n + 1]; ++k) {
      int e = vn_edges[k];
      if (e < 0 || e >= E || edge_vn[e] != n) return LDPC_ERR_INVALID;
      if (k > vn_ptr[n] && vn_edges[k] <= vn_edges[k - 1]) return LDPC_ERR_INVALID;
    }
  ldpc_graph* G = new ldpc_graph();
  int max_dv = 0, max_dc = 0;
  for (int n = 0; n < N; ++n) max_dv = std::max(max_dv, vn_ptr[n + 1] - vn_ptr[n]);
  for (int m = 0; m < M; ++m) max_dc = std::max(max_dc, cn_ptr[m + 1] - cn_ptr[m]);
  // largest two-hop set (pre-C2V refresh size) over all edges
  std::vector<long long> hop(N, 0);
  for (int n = 0; n < N; ++n)
    for (int k = vn_ptr[n]; k < vn_ptr[n + 1]; ++k) {
      int i = edge_cn[vn_edges[k]];
      hop[n] += cn_ptr[i + 1] - cn_ptr[i] - 1;
    }
  long long max_items = max_dc;
  for (int e = 0; e < E; ++e) {
    int i = edge_cn[e];
    max_items = std::max(max_items, hop[edge_vn[e]] - (cn_ptr[i + 1] - cn_ptr[i] - 1));
  }
  // layered dependency levels: level(m) = 1 + max level of earlier checks sharing a VN
  std::vector<int> last(N, 0), level(M, 0);
  int n_levels = 0;
  for (int m = 0; m < M; ++m) {
    int lv = 0;
    for (int e = cn_ptr[m]; e < cn_ptr[m + 1]; ++e) lv = std::max(lv, last[edge_vn[e]]);
    level[m] = lv + 1;
    for (int e = cn_ptr[m]; e < cn_ptr[m + 1]; ++e) last[edge_vn[e]] = lv + 1;
    n_levels = std::max(n_levels, lv + 1);
  }
  std::vector<int> level_ptr(n_levels + 1, 0), level_checks(M);
  for (int m = 0; m < M; ++m) level_ptr[level[m]]++;
  for (int l = 0; l < n_levels; ++l) level_ptr[l + 1] += level_ptr[l];
  {
    std::vector<int> fillp(level_ptr.begin(), level_ptr.end() - 1);
    for (int m = 0; m < M; ++m) level_checks[fillp[level[m] - 1]++] = m;
  }
  // fixed-engine tilings: per level, whole checks packed into tiles of <= kTileEdges edges
  struct HostTiling {
    std::vector<int> level_tptr, tile_eptr, te_list, te_chk, tile_cptr, tc_rec;
  } ht[2];
  auto build_tiling = [&](HostTiling& t, const std::vector<int>& lvl_ptr, const std::vector<int>& chk) {
    t.level_tptr.push_back(0);
    t.tile_eptr.push_back(0);
    t.tile_cptr.push_back(0);
    for (size_t L = 0; L + 1 < lvl_ptr.size(); ++L) {
      int cur = 0;
      for (int k = lvl_ptr[L]; k < lvl_ptr[L + 1]; ++k) {
        const int m = chk[k], d = cn_ptr[m + 1] - cn_ptr[m];
        if (cur > 0 && cur + d > kTileEdges) {
          t.tile_eptr.push_back((int)t.te_list.size());
          t.tile_cptr.push_back((int)t.tc_rec.size() / 4);
          cur = 0;
        }
        // (local a, degree, tile-order position of the first edge): c2v rows
        // live in tile order; the flooding tiling is the identity order
        t.tc_rec.insert(t.tc_rec.end(), {cur, d, (int)t.te_list.size(), 0});
        for (int e = cn_ptr[m]; e < cn_ptr[m + 1]; ++e) {
          t.te_list.push_back(e);
          t.te_chk.push_back(cur);
          t.te_chk.push_back(cur + d);
        }
        cur += d;
      }
      if (cur > 0) {
        t.tile_eptr.push_back((int)t.te_list.size());
        t.tile_cptr.push_back((int)t.tc_rec.size() / 4);
      }
      t.level_tptr.push_back((int)t.tile_eptr.size() - 1);
    }
  };
  {
    std::vector<int> all(M), one = {0, M};
    for (int m = 0; m < M; ++m) all[m] = m;
    build_tiling(ht[0], one, all);
    build_tiling(ht[1], level_ptr, level_checks);
  }
  // packed records and per-edge two-hop facts for the dynamic engine
  std::vector<int> ecv(2ull * E), vrec(2ull * N), vadj(4ull * E), erec(4ull * E), hop_n(E), hop_distinct(E);
  std::vector<uint8_t> hop_dup(E, 0);
  for (int e = 0; e < E; ++e) {
    ecv[2 * e] = edge_cn[e];
    ecv[2 * e + 1] = edge_vn[e];
    erec[4 * e] = edge_cn[e];
    erec[4 * e + 1] = edge_vn[e];
    erec[4 * e + 2] = vn_ptr[edge_vn[e]];
    erec[4 * e + 3] = vn_ptr[edge_vn[e] + 1] - vn_ptr[edge_vn[e]];
  }
  for (int n = 0; n < N; ++n) {
    vrec[2 * n] = vn_ptr[n];
    vrec[2 * n + 1] = vn_ptr[n + 1] - vn_ptr[n];
    for (int k = vn_ptr[n]; k < vn_ptr[n + 1]; ++k) {
      int f = vn_edges[k], i = edge_cn[f];
      vadj[4 * k] = f;
      vadj[4 * k + 1] = i;
      vadj[4 * k + 2] = cn_ptr[i];
      vadj[4 * k + 3] = cn_ptr[i + 1];
    }
  }
  {
    std::vector<int> stamp(N, -1);
    for (int e = 0; e < E; ++e) {
      int m_star = edge_cn[e], n_star = edge_vn[e], cnt = 0, distinct = 0;
      for (int k = vn_ptr[n_star]; k < vn_ptr[n_star + 1]; ++k) {
        int i = edge_cn[vn_edges[k]];
        if (i == m_star) continue;
        for (int g2 = cn_ptr[i]; g2 < cn_ptr[i + 1]; ++g2) {
          int j = edge_vn[g2];
          if (j == n_star) continue;
          ++cnt;
          if (stamp[j] != e) {
            stamp[j] = e;
            ++distinct;
          }
        }
      }
      hop_n[e] = cnt;
      hop_distinct[e] = distinct;
      hop_dup[e] = distinct < cnt ? 1 : 0;
    }
  }
  // precomputed two-hop tables (item records + per-slot stage bases), if <= 256 MB
  std::vector<long long> hop_ptr(E + 1, 0);
  std::vector<int> hop_sbptr(E + 1, 0);
  for (int e = 0; e < E; ++e) {
    hop_ptr[e + 1] = hop_ptr[e] + hop_n[e];
    hop_sbptr[e + 1] = hop_sbptr[e] + (vn_ptr[edge_vn[e] + 1] - vn_ptr[edge_vn[e]]);
  }
  const bool want_tab = hop_ptr[E] * 8 + (long long)hop_sbptr[E] * 4 <= (256ll << 20);
  std::vector<int> hop_items, hop_sb;
  if (want_tab) {
    hop_items.reserve(2 * hop_ptr[E]);
    hop_sb.reserve(hop_sbptr[E]);
    for (int e = 0; e < E; ++e) {
      const int m_star = edge_cn[e], n_star = edge_vn[e];
      int sb = 0;
      for (int k = vn_ptr[n_star]; k < vn_ptr[n_star + 1]; ++k) {
        const int f = vn_edges[k], i = edge_cn[f], a = cn_ptr[i], b = cn_ptr[i + 1];
        if (i == m_star) {
          hop_sb.push_back(-1);
          continue;
        }
        hop_sb.push_back(sb);
        for (int g2 = a; g2 < b; ++g2)
          if (g2 != f) hop_items.insert(hop_items.end(), {g2, pack_item(g2 - a, b - a, sb)});
        sb += b - a;
      }
    }
  }
  // one device block (int units): edge_cn, edge_vn, vn_edges [E]; cn_ptr [M+1];
  // vn_ptr [N+1]; level_ptr [L+1]; level_checks [M]; ecv [2E]; vrec [2N];
  // vadj [4E] (16-byte aligned); hop_n [E]; hop_distinct [E]; hop_dup [E bytes]
  size_t base_ints = 3ull * E + (M + 1) + (N + 1) + (n_levels + 1) + M;
  base_ints = (base_ints + 3) & ~size_t(3);
  size_t total = base_ints + 2ull * E + 2ull * N + 8ull * E + 2ull * E + (E + 3) / 4 + 8;
  int* d = nullptr;
  if (cudaMalloc(&d, total * sizeof(int)) != cudaSuccess) {
    delete G;
    return LDPC_ERR_CUDA;
  }
  std::vector<int> h(total);
  size_t o = 0;
  auto put = [&](const int* src, size_t n) {
    size_t r = o;
    memcpy(h.data() + o, src, n * sizeof(int));
    o += n;
    return r;
  };
  size_t oc = put(edge_cn, E), ov = put(edge_vn, E), oe = put(vn_edges, E);
  size_t ocp = put(cn_ptr, M + 1), ovp = put(vn_ptr, N + 1);
  size_t olp = put(level_ptr.data(), n_levels + 1), olc = put(level_checks.data(), M);
  o = base_ints;
  size_t oecv = put(ecv.data(), 2ull * E), ovrec = put(vrec.data(), 2ull * N);
  o = (o + 3) & ~size_t(3);
  size_t ovadj = put(vadj.data(), 4ull * E);
  size_t oerec = put(erec.data(), 4ull * E);
  size_t ohn = put(hop_n.data(), E), ohd = put(hop_distinct.data(), E);
  size_t ohdup = o;
  memcpy(h.data() + o, hop_dup.data(), E);
  if (cudaMemcpy(d, h.data(), total * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    delete G;
    return LDPC_ERR_CUDA;
  }
  // tilings: one more device block
  {
    size_t tot = 0;
    for (auto& t : ht)
      tot += t.level_tptr.size() + t.tile_eptr.size() + 2 * t.te_list.size() + t.te_chk.size() + t.tile_cptr.size() +
             t.tc_rec.size() + 8;
    int* tb = nullptr;
    if (cudaMalloc(&tb, tot * sizeof(int)) != cudaSuccess) {
      cudaFree(d);
      delete G;
      return LDPC_ERR_CUDA;
    }
    std::vector<int> hb;
    hb.reserve(tot);
    Tiling* dst[2] = {&G->flood, &G->layer};
    for (int i = 0; i < 2; ++i) {
      auto& t = ht[i];
      while (hb.size() % 4) hb.push_back(0);  // int4 alignment of tc_rec
      size_t o_rec = hb.size();
      hb.insert(hb.end(), t.tc_rec.begin(), t.tc_rec.end());
      size_t o_chk = hb.size();
      hb.insert(hb.end(), t.te_chk.begin(), t.te_chk.end());
      size_t o_lt = hb.size();
      hb.insert(hb.end(), t.level_tptr.begin(), t.level_tptr.end());
      size_t o_te = hb.size();
      hb.insert(hb.end(), t.tile_eptr.begin(), t.tile_eptr.end());
      size_t o_tl = hb.size();
      hb.insert(hb.end(), t.te_list.begin(), t.te_list.end());
      size_t o_vn = hb.size();
      for (int e : t.te_list) hb.push_back(edge_vn[e]);
      size_t o_cp = hb.size();
      hb.insert(hb.end(), t.tile_cptr.begin(), t.tile_cptr.end());
      dst[i]->tc_rec = (int4*)(tb + o_rec);
      dst[i]->tile_cptr = tb + o_cp;
      dst[i]->n_levels = (int)t.level_tptr.size() - 1;
      dst[i]->te_chk = (int2*)(tb + o_chk);
      dst[i]->level_tptr = tb + o_lt;
      dst[i]->tile_eptr = tb + o_te;
      dst[i]->te_list = tb + o_tl;
      dst[i]->te_vn = tb + o_vn;
      dst[i]->h_level_tptr = t.level_tptr;
    }
    if (cudaMemcpy(tb, hb.data(), hb.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(tb);
      cudaFree(d);
      delete G;
      return LDPC_ERR_CUDA;
    }
    G->tile_block = tb;
  }
  {  // strips of both schedules: one more device block
    HostStrips hs[2];
    std::vector<int> all(M), one = {0, M}, ve(vn_edges, vn_edges + E), cp(cn_ptr, cn_ptr + M + 1);
    for (int m = 0; m < M; ++m) all[m] = m;
    build_strips(hs[0], one, all, cp, edge_vn, ve, E, N, false);
    build_strips(hs[1], level_ptr, level_checks, cp, edge_vn, ve, E, N, true);
    build_vn_strips(hs[0], vn_ptr, N);
    std::vector<int> hb;
    size_t off[2][7];
    for (int i = 0; i < 2; ++i) {
      while (hb.size() % 4) hb.push_back(0);
      off[i][0] = hb.size();
      hb.insert(hb.end(), hs[i].rec.begin(), hs[i].rec.end());
      off[i][1] = hb.size();
      hb.insert(hb.end(), hs[i].runs.begin(), hs[i].runs.end());
      off[i][2] = hb.size();
      hb.insert(hb.end(), hs[i].vn.begin(), hs[i].vn.end());
      off[i][3] = hb.size();
      hb.insert(hb.end(), hs[i].vn_rows.begin(), hs[i].vn_rows.end());
      while (hb.size() % 4) hb.push_back(0);
      off[i][4] = hb.size();
      hb.insert(hb.end(), hs[i].v_rec.begin(), hs[i].v_rec.end());
      off[i][5] = hb.size();
      hb.insert(hb.end(), hs[i].v_runs.begin(), hs[i].v_runs.end());
      off[i][6] = hb.size();
      hb.insert(hb.end(), hs[i].level_sptr.begin(), hs[i].level_sptr.end());
    }
    int* sb = nullptr;
    if (cudaMalloc(&sb, hb.size() * sizeof(int)) != cudaSuccess ||
        cudaMemcpy(sb, hb.data(), hb.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) {
      if (sb) cudaFree(sb);
      cudaFree(G->tile_block);
      cudaFree(d);
      delete G;
      return LDPC_ERR_CUDA;
    }
    Strips* dst[2] = {&G->sflood, &G->slayer};
    for (int i = 0; i < 2; ++i) {
      dst[i]->h_level_sptr = hs[i].level_sptr;
      dst[i]->rec = (int4*)(sb + off[i][0]);
      dst[i]->runs = (int2*)(sb + off[i][1]);
      dst[i]->vn = sb + off[i][2];
      dst[i]->vn_rows = sb + off[i][3];
      dst[i]->n_vstrips = hs[i].v_rec.empty() ? 0 : (int)hs[i].v_rec.size() / 4 - 1;
      dst[i]->rec_count = (int)hs[i].rec.size() / 4 - 1;
      dst[i]->lvl_sptr = sb + off[i][6];
      dst[i]->v_rec = (int4*)(sb + off[i][4]);
      dst[i]->v_runs = (int2*)(sb + off[i][5]);
    }
    G->strip_block = sb;
  }
  if (want_tab) {  // two-hop tables: their own allocation
    const size_t bytes = hop_items.size() * 4 + (size_t)E * 8 + (size_t)E * 4 + hop_sb.size() * 4 + 64;
    unsigned char* hb = nullptr;
    if (cudaMalloc(&hb, bytes) != cudaSuccess) {
      cudaFree(G->strip_block);
      cudaFree(G->tile_block);
      cudaFree(d);
      delete G;
      return LDPC_ERR_CUDA;
    }
    size_t o_items = 0, o_ptr = align16(hop_items.size() * 4), o_sbp = o_ptr + (size_t)E * 8,
           o_sb = o_sbp + (size_t)E * 4;
    bool ok = cudaMemcpy(hb + o_items, hop_items.data(), hop_items.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(hb + o_ptr, hop_ptr.data(), (size_t)E * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(hb + o_sbp, hop_sbptr.data(), (size_t)E * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(hb + o_sb, hop_sb.data(), hop_sb.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) {
      cudaFree(hb);
      cudaFree(G->strip_block);
      cudaFree(G->tile_block);
      cudaFree(d);
      delete G;
      return LDPC_ERR_CUDA;
    }
    G->hop_block = hb;
    G->d.hop_items = (const int2*)(hb + o_items);
    G->d.hop_ptr = (const long long*)(hb + o_ptr);
    G->d.hop_sbptr = (const int*)(hb + o_sbp);
    G->d.hop_sb = (const int*)(hb + o_sb);
  }
  {  // per-VN sorted two-hop VN sets N2(v) = VNs sharing a check with v (v included),
     // the conflict test of multi-edge rounds (dyn_engine.cuh me_pair_disjoint); <= 64 MB
    std::vector<int> v2ptr(N + 1, 0), v2, stamp(N, -1), tmp;
    bool ok = true;
    for (int v = 0; v < N && ok; ++v) {
      tmp.clear();
      for (int k = vn_ptr[v]; k < vn_ptr[v + 1]; ++k) {
        const int i = edge_cn[vn_edges[k]];
        for (int g2 = cn_ptr[i]; g2 < cn_ptr[i + 1]; ++g2) {
          const int j = edge_vn[g2];
          if (stamp[j] != v) {
            stamp[j] = v;
            tmp.push_back(j);
          }
        }
      }
      if (tmp.empty()) tmp.push_back(v);
      std::sort(tmp.begin(), tmp.end());
      v2.insert(v2.end(), tmp.begin(), tmp.end());
      v2ptr[v + 1] = (int)v2.size();
      ok = v2.size() <= (16u << 20);
    }
    G->pair_block = nullptr;
    if (ok) {
      int* pb = nullptr;
      if (cudaMalloc(&pb, (v2ptr.size() + v2.size()) * sizeof(int)) == cudaSuccess &&
          cudaMemcpy(pb, v2ptr.data(), v2ptr.size() * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
          cudaMemcpy(pb + v2ptr.size(), v2.data(), v2.size() * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess) {
        G->pair_block = pb;
        G->d.vn2_ptr = pb;
        G->d.vn2 = pb + v2ptr.size();
      } else if (pb) {
        cudaFree(pb);
      }
    }
  }
  G->dev_block = d;
  G->max_dv = max_dv;
  G->min_dv = N > 0 ? 1 << 30 : 0;
  for (int n = 0; n < N; ++n) G->min_dv = std::min(G->min_dv, vn_ptr[n + 1] - vn_ptr[n]);
  G->max_dc = max_dc;
  G->max_items = (int)max_items;
  DevGraph& dg = G->d;
  dg.N = N;
  dg.M = M;
  dg.E = E;
  dg.max_dv = max_dv;
  dg.max_dc = max_dc;
  dg.max_items = (int)max_items;
  dg.edge_cn = d + oc;
  dg.edge_vn = d + ov;
  dg.vn_edges = d + oe;
  dg.cn_ptr = d + ocp;
  dg.vn_ptr = d + ovp;
  dg.n_levels = n_levels;
  dg.level_ptr = d + olp;
  dg.level_checks = d + olc;
  dg.ecv = (const int2*)(d + oecv);
  dg.vrec = (const int2*)(d + ovrec);
  dg.vadj = (const int4*)(d + ovadj);
  dg.erec = (const int4*)(d + oerec);
  dg.hop_n = d + ohn;
  dg.hop_distinct = d + ohd;
  dg.hop_dup = (const uint8_t*)(d + ohdup);
  *out = G;
  return LDPC_OK;
}

int ldpc_graph_destroy(ldpc_graph_t* G) {
  if (!G) return LDPC_ERR_INVALID;
  cudaFree(G->dev_block);
  cudaFree(G->tile_block);
  cudaFree(G->strip_block);
  if (G->hop_block) cudaFree(G->hop_block);
  if (G->pair_block) cudaFree(G->pair_block);
  delete G;
  return LDPC_OK;
}

int ldpc_graph_info(const ldpc_graph_t* G, int64_t* o) {
  if (!G || !o) return LDPC_ERR_INVALID;
  o[0] = G->d.N;
  o[1] = G->d.M;
  o[2] = G->d.E;
  o[3] = G->max_dv;
  o[4] = G->max_dc;
  o[5] = G->max_items;
  o[6] = G->d.n_levels;
  return LDPC_OK;
}

int ldpc_workspace_size(const ldpc_graph_t* G, const ldpc_sched_t* s, int64_t B, size_t* bytes) {
  if (int rc = validate(G, s, B)) return rc;
  if (!bytes) return LDPC_ERR_INVALID;
  long long ws = 256;
  if (B > 0) {
    if (is_dynamic(s->kind)) {
      DynPlan pl;
      int rc = s->precision == LDPC_F64 ? dyn_plan<double>(G, s, B, pl) : dyn_plan<float>(G, s, B, pl);
      if (rc) return rc;
      ws = pl.ws_bytes;
    } else if (s->want_trace) {
      FixedTracePlan pl;
      int rc = s->precision == LDPC_F64 ? fixed_trace_plan<double>(G, s, B, pl) : fixed_trace_plan<float>(G, s, B, pl);
      if (rc) return rc;
      ws = pl.ws_bytes;
    } else if (fixed_engine_choice(s, B) == 0) {
      PhasePlan pl;
      if (s->precision == LDPC_F64) phase_plan<double>(G, B, pl);
      else phase_plan<float>(G, B, pl);
      ws = pl.ws_bytes;
    } else {
      FixedPlan pl;
      int rc = s->precision == LDPC_F64 ? fixed_plan<double>(G, s, B, pl) : fixed_plan<float>(G, s, B, pl);
      if (rc) return rc;
      ws = pl.ws_bytes;
    }
  }
  *bytes = (size_t)ws;
  return LDPC_OK;
}

int ldpc_decode(const ldpc_graph_t* G, const void* llr, int64_t B, const ldpc_sched_t* s,
                int8_t* u_hat, int64_t* props, uint8_t* converged, int64_t* counters,
                int32_t* biterr, int32_t* biterr_info, int32_t* kappa_hits, int32_t* kappa_trials,
                void* workspace, size_t ws_bytes, void* stream) {
  if (int rc = validate(G, s, B)) return rc;
  if (B > 0 && (!llr || !u_hat || !props || !converged || !counters || !biterr || !biterr_info || !workspace))
    return LDPC_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const TraceOut tr{nullptr, nullptr, 0, nullptr};
  if (s->precision == LDPC_F64)
    return decode_impl<double>(G, llr, B, s, u_hat, props, converged, counters, biterr, biterr_info,
                               kappa_hits, kappa_trials, workspace, ws_bytes, tr, st);
  return decode_impl<float>(G, llr, B, s, u_hat, props, converged, counters, biterr, biterr_info,
                            kappa_hits, kappa_trials, workspace, ws_bytes, tr, st);
}

int ldpc_decode_traced(const ldpc_graph_t* G, const void* llr, int64_t B, const ldpc_sched_t* s,
                       int8_t* u_hat, int64_t* props, uint8_t* converged, int64_t* counters,
                       int32_t* biterr, int32_t* biterr_info, int32_t* kappa_hits, int32_t* kappa_trials,
                       double* trace, const double* gammas, int32_t n_gamma, uint64_t* j_counts,
                       void* workspace, size_t ws_bytes, void* stream) {
  if (int rc = validate(G, s, B)) return rc;
  if (!s->want_trace) return LDPC_ERR_INVALID;
  if (B > 0 && (!llr || !u_hat || !props || !converged || !counters || !biterr || !biterr_info || !workspace))
    return LDPC_ERR_INVALID;
  if (j_counts && (n_gamma < 1 || !gammas)) return LDPC_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const TraceOut tr{trace, gammas, j_counts ? n_gamma : 0, (unsigned long long*)j_counts};
  if (s->precision == LDPC_F64)
    return decode_impl<double>(G, llr, B, s, u_hat, props, converged, counters, biterr, biterr_info,
                               kappa_hits, kappa_trials, workspace, ws_bytes, tr, st);
  return decode_impl<float>(G, llr, B, s, u_hat, props, converged, counters, biterr, biterr_info,
                            kappa_hits, kappa_trials, workspace, ws_bytes, tr, st);
}

int ldpc_select_vns(const double* ci, const uint8_t* mask, int32_t N, int32_t n_g, int32_t n_p,
                    int64_t seed, int32_t* out, int32_t* count_dev, void* stream) {
  if (!ci || !out || !count_dev || N <= 0 || n_g < 1 || n_p < 1 || n_g > 4096) return LDPC_ERR_INVALID;
  long long smem = align16((long long)n_g * 4) + align16((long long)std::max(N, n_p) * 4) + align16(N);
  if (smem > smem_optin()) return LDPC_ERR_UNSUPPORTED;
  cudaFuncSetAttribute((void*)select_vns_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  select_vns_kernel<<<1, 32, smem, (cudaStream_t)stream>>>(ci, mask, N, n_g, n_p, seed, out, count_dev);
  g_last_launches = 1;
  return cuda_check(cudaGetLastError());
}

// ---- replay (debug / audit): DecoderState-style forced edge sequences


int ldpc_replay_workspace_size(const ldpc_graph_t* G, const ldpc_sched_t* s, int64_t B, size_t* bytes) {
  if (int rc = replay_check(G, s, B)) return rc;
  if (!bytes) return LDPC_ERR_INVALID;
  DynParams p;
  memset(&p, 0, sizeof(p));
  if (s->precision == LDPC_F64) replay_layout<double>(G, s, p);
  else replay_layout<float>(G, s, p);
  *bytes = (size_t)(256 + B * (p.slotE_bytes + p.slotN_bytes + p.slotT_bytes));
  return LDPC_OK;
}

int ldpc_decode_replay(const ldpc_graph_t* G, const void* llr, int64_t B, const ldpc_sched_t* s,
                       const int32_t* forced_edges, int32_t steps, double* c2v_trace, double* state_out,
                       int64_t* counters, void* workspace, size_t ws_bytes, void* cuda_stream) {
  g_last_launches = 0;
  if (int rc = replay_check(G, s, B)) return rc;
  if (steps < 0 || (B > 0 && (!llr || !state_out || !counters || (steps > 0 && (!forced_edges || !c2v_trace)))))
    return LDPC_ERR_INVALID;
  if (B == 0) return LDPC_OK;
  size_t need = 0;
  ldpc_replay_workspace_size(G, s, B, &need);
  if (!workspace || ws_bytes < need) return LDPC_ERR_WORKSPACE;
  DynParams p;
  memset(&p, 0, sizeof(p));
  const bool f64 = s->precision == LDPC_F64;
  if (f64) replay_layout<double>(G, s, p);
  else replay_layout<float>(G, s, p);
  p.g = G->d;
  p.kind = KIND_LMD_CIRBP;
  p.kernel = s->kernel;
  p.i_max = s->i_max;
  p.k_info = s->k_info;
  p.seed = s->selection_seed;
  p.llr = llr;
  p.llr_f64 = s->llr_f64;
  p.B = B;
  p.counters = (long long*)counters;
  p.ws = (unsigned char*)workspace + 256;
  const int smem = (int)(p.slotU_bytes + p.scratch_bytes);
  if (smem > smem_optin() - 1024) return LDPC_ERR_UNSUPPORTED;
  void* fn = ldpc_replay_kernel(f64 ? 1 : 0, s->kernel);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  void* args[] = {&p, (void*)&forced_edges, &steps, &c2v_trace, &state_out};
  if (int rc = cuda_check(cudaLaunchKernel(fn, dim3((unsigned)B), dim3(32), args, smem, (cudaStream_t)cuda_stream)))
    return rc;
  g_last_launches = 1;
  return LDPC_OK;
}

}  // extern "C"
