// dyn_engine.cuh -- informed-dynamic-schedule decoders, one warp per frame.
//
// Replaces the reference's numba schedule loops
// (/root/reference/pkg/src/ldpc_ids/_engine.py, "E:<line>"):
//   RBP E:355-385, CIRBP E:388-433, LMDRBP/sLMDRBP E:436-510,
//   LMD-CIRBP E:513-598, ME-CIRBP E:601-643, ME-LMD-CIRBP E:646-716,
//   plus ME-RBP (new; defined in oracle/ldpc_oracle.c).
//
// Design (B200):
//  * persistent grid; each warp pulls frame ids from an atomic work queue, so a
//    frame that converges early frees its warp for the next frame;
//  * a frame's state is split in two parts placed by the host (MODE):
//      per-edge part  c2v, pre, in (= tanh(v2c/2) or v2c) [, res]   E x 3-4 words
//      per-VN part    total [, pre_total, ci], trees, ME scratch    N x 1-3 words
//    MODE 0: both in shared memory; MODE 1: per-edge part in an L2-resident
//    HBM slot, per-VN part in shared memory; MODE 2: both in HBM (huge codes);
//  * the residual is never stored: it is |pre - c2v| exactly (E:144,167), so
//    tree leaves are recomputed from pre and c2v; for RBP-family schedules
//    pre_total / CI are not maintained (the reference keeps them only for its
//    trace output, E:171-176);
//  * the update (_propagate, E:130-176) is a latency-bound serial chain, so it
//    is built to minimise dependent memory round trips: packed graph records,
//    per-edge precomputed two-hop facts, each touched check's inputs staged
//    once into shared memory, then all (d_v-1)(d_c-1) pre-C2V refreshes run
//    lane-parallel with the reference's exact product order;
//  * pre_total accumulations that hit the same VN (4-cycle through n*) are
//    applied in the reference's order (match_any ranks), so float64 results
//    are bit-identical;
//  * global argmax: 32-ary max trees of order-preserving integer keys, one
//    coalesced load + REDUX.MAX per level, lowest index wins ties like the
//    reference's left-preferring segment tree (E:220-257); only the touched
//    32-leaf groups and their ancestors are recomputed.
#pragma once
#include "ldpc_common.cuh"

namespace ldpc {

#ifndef LDPC_DYN_MIN_BLOCKS
#define LDPC_DYN_MIN_BLOCKS 4
#endif
// Resident 256-thread blocks per SM the register budget is cut for: 4 (64
// registers) in general; the float64 RBP and LMDRBP kernels run faster at 6
// (40 registers, more spills, 1.5x the resident frames: C1 -3 % / -16 %),
// while the CI and ME kinds lose (measured with tools/dyn_sweep.py).
#ifndef LDPC_DYN_RBP_BLOCKS
#define LDPC_DYN_RBP_BLOCKS 6
#endif
// BG-sized codes (placement mode 3: the whole state in HBM) are bound by the
// memory system's sector-request rate, where spill traffic competes with the
// state traffic and shared memory already caps the resident warps: RBP runs
// faster at 4 blocks (64 registers; C3 2.39e8 vs 1.76e8 updates/s) and CIRBP at
// 3 (80 registers; C3 6.2e7 vs 5.1e7).
constexpr int dyn_min_blocks(int kind, bool f64, int mode) {
  if (f64 && mode == 3 && (kind == KIND_RBP || kind == KIND_LMDRBP)) return 4;
  if (f64 && mode == 3 && kind == KIND_CIRBP) return 3;
  return (f64 && (kind == KIND_RBP || kind == KIND_LMDRBP)) ? LDPC_DYN_RBP_BLOCKS : LDPC_DYN_MIN_BLOCKS;
}


template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

// Two-hop item record (8 bytes: the table of a BG1-sized code is read from HBM
// on every update, so its size is DRAM traffic): edge g, and packed the
// position of g in its check (skip), the check's degree d and the base of the
// check's inputs in the stage area.
struct Item { int g, skip, d, sb; };
__host__ __device__ __forceinline__ int pack_item(int skip, int d, int sb) { return skip | (d << 8) | (sb << 16); }
__device__ __forceinline__ Item unpack_item(int2 r) {
  Item it;
  it.g = r.x;
  it.skip = r.y & 0xff;
  it.d = (r.y >> 8) & 0xff;
  it.sb = (int)((unsigned)r.y >> 16);
  return it;
}
constexpr int kItemMaxDegree = 255, kItemMaxStage = 65535;

// max-tree storage (see "max trees" below)
template <typename Key>
struct alignas(2 * sizeof(Key)) L1Node {
  Key k;
  int i;
};

template <typename Key>
struct TreeRef {
  L1Node<Key>* l1;  // level 1
  Key* up;          // levels >= 2: level l at up + geo.off[l] - geo.off[2]
};


struct DynParams {
  DevGraph g;
  int kind, kernel, i_max, n_p, n_g, k_info;
  double gamma;
  long long seed;
  const void* llr;
  int llr_f64;
  long long B;
  // outputs
  int8_t* u_hat;          // [B][N]
  long long* prop;        // [B]
  uint8_t* conv;          // [B]
  long long* counters;    // [B][8]
  int* biterr;            // [B][i_max+1]
  int* biterr_info;       // [B][i_max+1]
  int* kh;                // [B][i_max] (CIRBP)
  int* kt;
  unsigned long long* next;
  long long* step_log;    // debug: propagated edge of the first log_cap updates per frame
  int log_cap;
  int dbg_full_tree;      // debug: recompute every touched tree group from its leaves
  long long dump_step;    // debug: copy ci / pre_total of frame 0 before this update
  double* dump_buf;       // [2N]
  // state placement: per-edge (E), per-VN (N) and tree (T) parts
  unsigned char* ws;      // HBM slots
  long long slotE_bytes, slotN_bytes, slotT_bytes;
  long long o_c2v, o_pre, o_in, o_res;                           // E part
  long long o_total /* per-VN records or dense totals */, o_inpp, o_gid, o_gbits, o_members, o_sel, o_chosen, o_tmp;  // N part
  long long o_rl1, o_cl1;                                        // T part: level-1 tree nodes
  long long slotU_bytes, o_rup, o_cup;                           // U part (shared memory): tree levels >= 2
  TreeGeom rgeo, cgeo;
  int scratch_bytes;      // per-warp shared scratch
  int so_items, so_stage, so_nk, so_opre, so_cj, so_ck, so_dl0, so_dl1, so_sizes, so_hist;
  int dl_cap;             // entries of dl0 (twice that allocated: ping-pong for the levels >= 3 fix)
  int me_pairs;           // multi-edge rounds: apply disjoint consecutive VN pairs on the two half-warps
  int pair_cap;           // ints that fit the stage area (conflict-test buffer)
  int so_pair;            // scratch offset of the second half-warp's per-update scratch
  int fast_sel;           // ME kinds with n_g <= 255: maintained groups + histogram
  // want_trace (E:192-217): pre_total upkeep for every kind, per-boundary rows
  // and fused J(gamma) counts (sim.py:172-183)
  int pt_on;              // maintain pre_total (always for CI kinds)
  TraceOut tr;
};

template <typename T, int G>
struct Ctx {
  using Key = typename Num<T>::Key;
  Grp<G> w;            // this frame's lane group
  T *c2v, *pre, *in, *res, *tmp;
  // Per-VN state: one record per VN, (pre_total, p0t = p0_cache(total), total,
  // ci) -- 4 words, one 32-byte sector in float64 -- because a CI-kind update
  // touches these words of ~90 scattered VNs and HBM moves whole sectors: one
  // sector per VN instead of three.  (The RBP family uses only `total`; the
  // record keeps one base pointer and immediate offsets for every kind.)
  T* nb;   // records
  int cs;  // stride of ci in words: 4 (records); 1 when nb = a caller's dense CI vector - 3 (ldpc_select_vns)
  static constexpr int ts = 4;  // stride of total in words
  __device__ __forceinline__ T* tb() const { return nb + 2; }
  __device__ __forceinline__ T& total(int n) const { return nb[4 * n + 2]; }
  __device__ __forceinline__ T& pretot(int n) const { return nb[4 * n]; }
  __device__ __forceinline__ T& p0t(int n) const { return nb[4 * n + 1]; }
  __device__ __forceinline__ T& ci(int n) const { return nb[cs * n + 3]; }
  TreeRef<Key> rt, ct;  // residual tree over E, CI tree over N
  uint8_t* inpp;  // ME-LMD-CIRBP P' membership (E:665)
  uint8_t* gid;   // ME kinds: Alg.-4 group of each VN (maintained)
  int* hist;      // ME kinds: VNs per group (maintained)
  unsigned* gbits;  // ME kinds: membership bitmap of each group (maintained)
  int *members, *sel, *chosen;
  const int2* items;  // two-hop edges of the last update, ascending g: (g, packed skip | d | stage base)
  int2* items_buf;    // per-warp scratch for items built on the fly
  T* stage;       // staged check inputs of the last update
  Key* nk;        // new residual key of each item
  T* cg;          // C2V of each item, staged with its inputs (aliases nk: read before nk is written)
  T* opre;        // old pre of each item (pre_total upkeep)
  int* cj;        // VN of each item (pre_total upkeep; -1: not its last occurrence)
  Key* ck;        // CI key of each item's VN after the refresh (CI tree; aliases opre, read first)
  int *dl0, *dl1; // dirty-node lists for tree maintenance
  int* sizes;     // Alg.4 group histogram
  // work counters (E:17-25): the 8 words just below the stage area of the
  // frame's shared scratch (addressed off `stage`: no register of their own)
  long long* cbase;  // half-warp contexts of a pair step (G = 16): the frame's counters; unused for G = 32
  __device__ __forceinline__ long long* cntp() const {
    if constexpr (G == 32) return (long long*)stage - kCounters;
    else return cbase;
  }
  long long prop;
  long long cur_f;   // frame being decoded
  int nsel;          // Alg.-4 selections made (debug log index)
  long long next_b;  // next single-edge iteration boundary (k * E)
  int it;            // completed iterations
  int lane;          // lane within the group (= w.lane)
  long long rng;
  // Every lane of a whole-warp group performs the same read-add-write (same
  // address, same value: one of the identical stores lands), so there is no
  // divergent lane-0 branch; the half-warps of a pair step add atomically.
  __device__ __forceinline__ void count(int k, long long v) {
    if constexpr (G == 32) {
      cntp()[k] += v;
    } else {
      if (lane == 0) atomicAdd((unsigned long long*)&cntp()[k], (unsigned long long)v);
    }
  }
  // one update's V2C and pre-C2V tallies (adjacent counters 1 and 2).  C_PROP
  // (= prop) and C_CI (= C_PRE for CI kinds) are filled in when the frame ends.
  __device__ __forceinline__ void count_update(int v2c, int pre) {
    static_assert(C_V2C == 1 && C_PRE == 2, "adjacent counters");
    if constexpr (G == 32) {
      long long* q = cntp() + C_V2C;
      q[0] += v2c;
      q[1] += pre;
    } else {
      if (lane == 0) {
        atomicAdd((unsigned long long*)&cntp()[C_V2C], (unsigned long long)v2c);
        atomicAdd((unsigned long long*)&cntp()[C_PRE], (unsigned long long)pre);
      }
    }
  }
  // frame end: counters[f][0..8) with the derived ones (group-converged; syncs first)
  __device__ __forceinline__ void store_counters(long long* out, bool ci_kind) const {
    w.sync();
    if (lane < kCounters) {
      long long v = cntp()[lane];
      if (lane == C_PROP) v = prop;
      if (lane == C_CI) v = ci_kind ? cntp()[C_PRE] : 0;
      out[lane] = v;
    }
  }
};

// residual leaf key: |pre - c2v| (or the stored residual for ME-RBP's exclusion)
template <typename T, bool STORED, int G>
__device__ __forceinline__ typename Num<T>::Key res_key(const Ctx<T, G>& c, int e) {
  if (STORED) return Num<T>::key(c.res[e]);
  return Num<T>::key(Num<T>::abs_(c.pre[e] - c.c2v[e]));
}

// ------------------------------------------------------------- max trees
// Level-1 nodes (one per 32 leaves) hold the group's max key AND its argmax
// leaf (lowest index among equal keys) in one record, so the last step of an
// argmax descent is one load; they live in the frame's tree part (shared
// memory or HBM by placement).  Levels >= 2 (E/1024 keys and fewer: 123 keys
// for a BG1-sized code) always live in shared memory, so a descent or an
// ancestor fix touches HBM at most once.  LeafFn: int -> Key.

__host__ __device__ __forceinline__ int up_off(const TreeGeom& geo, int l) { return geo.off[l] - geo.off[2]; }

template <typename Key, typename LeafFn>
__device__ __forceinline__ Key child_key(const TreeRef<Key>& t, const TreeGeom& geo, int level, int child,
                                         LeafFn leaf) {
  if (child >= geo.size[level]) return Key(0);
  if (level == 0) return leaf(child);
  if (level == 1) return t.l1[child].k;
  return t.up[up_off(geo, level) + child];
}

template <typename Key>
__device__ __forceinline__ void set_node(const TreeRef<Key>& t, const TreeGeom& geo, int level, int q, Key k) {
  if (level == 1) t.l1[q].k = k;
  else t.up[up_off(geo, level) + q] = k;
}

// lane-local scan of node q's 32 children (level l-1), strided by the group
// width; returns the lane's (max key, lowest child index among ties)
template <int G, typename Key, typename LeafFn>
__device__ __forceinline__ Key child_scan(const TreeRef<Key>& t, const TreeGeom& geo, int l, int q, int lane,
                                          LeafFn leaf, int* bi) {
  Key m = 0;
  int b = 0x7fffffff;
#pragma unroll
  for (int c = lane; c < 32; c += G) {
    const Key k = child_key(t, geo, l - 1, q * 32 + c, leaf);
    if (k > m || b == 0x7fffffff) { m = k; b = q * 32 + c; }
  }
  *bi = b;
  return m;
}

template <int G, typename Key, typename LeafFn>
__device__ void tree_build(const TreeRef<Key>& t, const TreeGeom& geo, const Grp<G>& w, LeafFn leaf) {
  for (int q = w.lane; q < geo.size[1]; q += G) {
    Key m = 0;
    int bi = q * 32;
    for (int c = 0; c < 32; ++c) {
      Key k = child_key(t, geo, 0, q * 32 + c, leaf);
      if (k > m) { m = k; bi = q * 32 + c; }
    }
    t.l1[q].k = m;
    t.l1[q].i = bi;
  }
  w.sync();
  for (int l = 2; l <= geo.levels; ++l) {
    for (int q = w.lane; q < geo.size[l]; q += G) {
      Key m = 0;
      for (int c = 0; c < 32; ++c) {
        Key k = child_key(t, geo, l - 1, q * 32 + c, leaf);
        m = k > m ? k : m;
      }
      t.up[up_off(geo, l) + q] = m;
    }
    w.sync();
  }
}

// Full recompute of level-1 group q from its leaves (group-cooperative).
template <int G, typename Key, typename LeafFn>
__device__ __forceinline__ void group_recompute(const TreeRef<Key>& t, const TreeGeom& geo, int q,
                                                const Grp<G>& w, LeafFn leaf) {
  int bi;
  const Key k = child_scan<G>(t, geo, 1, q, w.lane, leaf, &bi);
  int best;
  const Key m = w.max_key_minidx(k, bi, &best);
  if (w.lane == 0) {
    L1Node<Key> nd;
    nd.k = m;
    nd.i = best;
    t.l1[q] = nd;
  }
}

// Recompute the level-1 groups rec[0..n) from their leaves.  With G = 32 the
// leaf loads of up to 4 groups are issued together (one memory round trip for
// them, instead of one per group), then reduced group by group.
template <int G, typename Key, typename LeafFn>
__device__ void group_recompute_list(const TreeRef<Key>& t, const TreeGeom& geo, const int* rec, int n,
                                     const Grp<G>& w, LeafFn leaf) {
  if (G != 32) {
    for (int i = 0; i < n; ++i) group_recompute(t, geo, rec[i] & 0x7fffffff, w, leaf);
    return;
  }
  for (int i0 = 0; i0 < n; i0 += 4) {
    Key k[4];
    int q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      q[j] = i0 + j < n ? (rec[i0 + j] & 0x7fffffff) : -1;
      k[j] = q[j] >= 0 ? child_key(t, geo, 0, q[j] * 32 + w.lane, leaf) : Key(0);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (q[j] < 0) break;
      int best;
      const Key m = w.max_key_minidx(k[j], q[j] * 32 + w.lane, &best);
      if (w.lane == 0) {
        L1Node<Key> nd;
        nd.k = m;
        nd.i = best;
        t.l1[q[j]] = nd;
      }
    }
  }
}

// Recompute the ancestors (levels >= 2, shared memory) of the level-1 groups dl[0..n).
template <int G, typename Key, typename LeafFn>
__device__ void tree_fix_ancestors(const TreeRef<Key>& t, const TreeGeom& geo, int* dl, int* dl2, int n,
                                   const Grp<G>& w, LeafFn leaf, int l0 = 2) {
  for (int l = l0; l <= geo.levels; ++l) {
    int cnt = 0;
    for (int base = 0; base < n; base += G) {
      int idx = base + w.lane;
      int v = idx < n ? (dl[idx] >> 5) : -1;
      int pv = (idx > 0 && idx < n) ? (dl[idx - 1] >> 5) : -2;
      bool keep = idx < n && v != pv;
      unsigned bal = w.ballot(keep);
      if (keep) dl2[cnt + __popc(bal & w.lt)] = v;
      cnt += __popc(bal);
    }
    w.sync();
    int* tmp = dl;
    dl = dl2;
    dl2 = tmp;
    n = cnt;
    for (int i = 0; i < n; ++i) {
      const int q = dl[i];
      int bi;
      const Key m = w.max_key_only(child_scan<G>(t, geo, l, q, w.lane, leaf, &bi));
      if (w.lane == 0) t.up[up_off(geo, l) + q] = m;
    }
    w.sync();
  }
}

// Full recompute of the level-1 groups dl[0..n) and their ancestors.
template <int G, typename Key, typename LeafFn>
__device__ void tree_update_list(const TreeRef<Key>& t, const TreeGeom& geo, int* dl, int* dl2, int n,
                                 const Grp<G>& w, LeafFn leaf) {
  group_recompute_list(t, geo, dl, n, w, leaf);
  w.sync();
  tree_fix_ancestors(t, geo, dl, dl2, n, w, leaf);
}

// Level-2 upkeep for a level-1 group q whose max went Q0 -> Qn (rec: to be
// recomputed from its leaves, new max <= Q0).  A raise is applied at once
// (atomic max into the shared-memory level-2 node; returns true if it raised
// it); a recomputed group that held its parent's max flags the parent for a
// rescan after the recompute (returns hold).  Everything else leaves level 2
// unchanged -- so the common case (a few groups' maxima move below their
// parents') costs no child scan and, with level 1 in HBM, no round trip.
template <typename Key>
__device__ __forceinline__ bool l2_note(const TreeRef<Key>& t, const TreeGeom& geo, int q, Key Q0, Key Qn, bool rec,
                                        bool* hold) {
  *hold = false;
  if (geo.levels < 2) return false;
  Key* K2 = t.up + up_off(geo, 2) + (q >> 5);
  if (rec) {
    *hold = Q0 == *K2;
    return false;
  }
  if (Qn > Q0) return atomicMax(K2, Qn) < Qn;
  return false;
}

// After the level-1 recomputes: rescan the level-2 parents of the flagged
// (holding) recomputed groups rec[i] (bit 31), append every level-2 node that
// changed (raised[0..nr) already listed) and fix levels >= 3 above them.
template <int G, typename Key, typename LeafFn>
__device__ void l2_finish(const TreeRef<Key>& t, const TreeGeom& geo, const int* rec, int nrec, int* ch, int nch,
                          int* ch2, const Grp<G>& w, LeafFn leaf) {
  if (geo.levels < 2) return;
  Key* K2 = t.up + up_off(geo, 2);
  for (int i = 0; i < nrec; ++i) {
    const int r = rec[i];
    if (r >= 0) continue;  // not a holder
    const int p = (r & 0x7fffffff) >> 5;
    int bi;
    const Key m = w.max_key_only(child_scan<G>(t, geo, 2, p, w.lane, leaf, &bi));
    const bool chg = m != K2[p];
    w.sync();
    if (chg) {
      if (w.lane == 0) {
        K2[p] = m;
        ch[nch] = p;
      }
      ++nch;
    }
    w.sync();
  }
  if (geo.levels > 2 && nch > 0) tree_fix_ancestors(t, geo, ch, ch2, nch, w, leaf, 3);
}

// Incremental rule for one leaf e of group q getting key kk, applied to the
// group's (max key Q, argmax I): returns true if the group must be recomputed
// (its argmax leaf decreased).
template <typename Key>
__device__ __forceinline__ bool leaf_rule(Key& Q, int& I, int e, Key kk) {
  if (kk > Q) {
    Q = kk;
    I = e;
  } else if (kk == Q) {
    if (e < I) I = e;
  } else if (e == I) {
    return true;
  }
  return false;
}

// Incremental update of level-1 groups for per-lane leaf changes (leaf e or
// -1, new key kk), lanes of the same group serialised by a match_any leader.
// Appends groups to recompute to rec[] and changed groups to dirty[].
template <int G, typename Key>
__device__ __forceinline__ void apply_leaf_updates(const TreeRef<Key>& t, const TreeGeom& geo, int e, Key kk,
                                                   const Grp<G>& w, int* se, Key* sk, int* rec, int& nrec, int* dirty,
                                                   int& ndirty) {
  L1Node<Key>* L1 = t.l1;
  const int q = e >= 0 ? (e >> 5) : -1;
  se[w.lane] = e;
  sk[w.lane] = kk;
  w.sync();
  const unsigned peers = w.match_any(q);
  const bool leader = e >= 0 && (__ffs(peers) - 1) == w.lane;
  bool r = false, changed = false, hold = false;
  if (leader) {
    // fold the group's changes (each leaf at most once per call): max new key
    // mx (lowest leaf mi) and the new key of the argmax leaf I if it changed;
    // recompute only if I decreased and nothing rose above the old max
    const L1Node<Key> nd = L1[q];
    const Key Q = nd.k;
    const int I = nd.i;
    Key mx = 0, nI = 0;
    int mi = 0x7fffffff;
    bool hasI = false;
    unsigned m = peers;
    while (m) {
      const int s2 = __ffs(m) - 1;
      m &= m - 1;
      const int e2 = se[s2];
      const Key k2 = sk[s2];
      if (k2 > mx || (k2 == mx && e2 < mi)) { mx = k2; mi = e2; }
      if (e2 == I) { hasI = true; nI = k2; }
    }
    Key Qn = Q;
    int In = I;
    if (hasI && nI < Q && !(mx > Q)) {
      r = true;
    } else if (mx > Q) {
      Qn = mx;
      In = mi;
    } else if (mx == Q && mi < I) {
      In = mi;
    }
    if (!r && (Qn != Q || In != I)) {
      L1Node<Key> o;
      o.k = Qn;
      o.i = In;
      L1[q] = o;
    }
    changed = l2_note(t, geo, q, Q, Qn, r, &hold);
  }
  const unsigned rb = w.ballot(r), cb = w.ballot(changed);
  if (r) rec[nrec + __popc(rb & w.lt)] = hold ? (q | (int)0x80000000) : q;
  if (changed) dirty[ndirty + __popc(cb & w.lt)] = q >> 5;
  nrec += __popc(rb);
  ndirty += __popc(cb);
  w.sync();
}

template <int G, typename Key, typename LeafFn>
__device__ int tree_argmax(const TreeRef<Key>& t, const TreeGeom& geo, const Grp<G>& w, LeafFn leaf) {
  const int L = geo.levels, s = geo.size[L];
  Key bk = 0;
  int bq = 0x7fffffff, bi = 0;
  for (int i = w.lane; i < s; i += G) {  // top level (<= 64 nodes)
    Key k;
    int li = 0;
    if (L == 1) {
      const L1Node<Key> nd = t.l1[i];
      k = nd.k;
      li = nd.i;
    } else {
      k = t.up[up_off(geo, L) + i];
    }
    if (k > bk || bq == 0x7fffffff) { bk = k; bq = i; bi = li; }
  }
  int q;
  w.max_key_minidx(bk, bq, &q);
  if (L == 1) return w.shfl(bi, q % G);  // the lane that scanned node q holds its argmax leaf
  for (int l = L - 1; l >= 2; --l) {
    int b;
    const Key k = child_scan<G>(t, geo, l + 1, q, w.lane, leaf, &b);
    int best;
    w.max_key_minidx(k, b, &best);
    q = best;
  }
  // level-1 children of q: key and argmax leaf in one record per lane
  Key ck = 0;
  int cq = 0x7fffffff, ci = 0;
  for (int c = w.lane; c < 32; c += G) {
    const int child = q * 32 + c;
    if (child < geo.size[1]) {
      const L1Node<Key> nd = t.l1[child];
      if (nd.k > ck || cq == 0x7fffffff) { ck = nd.k; cq = child; ci = nd.i; }
    }
  }
  int best;
  w.max_key_minidx(ck, cq, &best);
  // the winning child was scanned by lane (best - 32q) % G; take its argmax leaf
  return w.shfl(ci, (best - q * 32) % G);
}

// ------------------------------------------------------------ argmax scans

// E:260-266 -- first maximum of key(i) over i in [0, n)
template <typename Key, int G, typename KeyFn>
__device__ int argmax_scan(int n, const Grp<G>& w, KeyFn keyf) {
  Key best = 0;
  int bi = 0x7fffffff;
  for (int i = w.lane; i < n; i += G) {
    Key k = keyf(i);
    if (k > best) { best = k; bi = i; }
  }
  int idx;
  w.max_key_minidx(best, bi, &idx);
  return idx;
}

// E:269-276 -- first maximum residual over M(n) in vn_edges order (= edge order)
template <typename T, int G, bool KEEP = false>  // KEEP: L2 evict_last hint on the graph tables (ldk)
__device__ __forceinline__ int argmax_vn_edges(const DevGraph& g, const Ctx<T, G>& c, int n, int* deg = nullptr) {
  using Key = typename Num<T>::Key;
  const unsigned long long pol = KEEP ? l2_keep_policy() : 0ull;
  const int2 vr = ldk<KEEP>(g.vrec + n, pol);
  if (deg) *deg = vr.y;  // the caller's comparison count, without reloading vrec
  Key bk = 0;
  int be = 0x7fffffff;
  for (int k = c.lane; k < vr.y; k += G) {  // vn_edges ascend: first max = lowest edge
    const int e = ldk<KEEP>(g.vn_edges + vr.x + k, pol);
    const Key kk = res_key<T, false, G>(c, e);
    if (kk > bk || be == 0x7fffffff) { bk = kk; be = e; }
  }
  int idx;
  c.w.max_key_minidx(bk, be, &idx);
  return idx;
}

// ------------------------------------------------------- two-hop item table

// Items = {g in N(i)\{f} : f in M(n*), i = cn(f) != m*}, ascending edge id (the
// reference's scan order, E:153-166 / E:450-460).  `adj` is this lane's vadj
// record (lane < d_v), `act` = its check is not m*.  Also lays out the stage
// area: check k's inputs at stage[sbase_k + (e - a_k)].  Returns the count;
// the caller must __syncwarp() before reading the table.
template <typename T, int G>
__device__ __forceinline__ int build_items_from(Ctx<T, G>& c, int4 adj, bool act, int* sbase_out,
                                                int& carry_items, int& carry_stage) {
  const int d = act ? adj.w - adj.z : 0;
  const int packed = act ? ((d - 1) | (d << 16)) : 0;
  const int incl = c.w.incl_scan(packed);
  const int total = c.w.shfl(incl, G - 1);
  const int t0 = carry_items + ((incl - packed) & 0xffff), sbase = carry_stage + ((incl - packed) >> 16);
  if (act) {
    int t = t0;
    for (int e = adj.z; e < adj.w; ++e)
      if (e != adj.x) c.items_buf[t++] = make_int2(e, pack_item(e - adj.z, d, sbase));
  }
  *sbase_out = sbase;
  carry_items += total & 0xffff;
  carry_stage += total >> 16;
  return carry_items;
}

// item table of e (precomputed, or built into the group's scratch)
template <typename T, int G>
__device__ int build_items(const DevGraph& g, Ctx<T, G>& c, int e_star) {
  if (g.hop_items) {
    c.items = g.hop_items + g.hop_ptr[e_star];
    return g.hop_n[e_star];
  }
  c.items = c.items_buf;
  const int2 mn = g.ecv[e_star];
  const int2 vr = g.vrec[mn.y];
  int ci = 0, cs = 0, n = 0, sb;
  for (int k0 = 0; k0 < vr.y; k0 += G) {
    const int k = k0 + c.lane;
    int4 adj = make_int4(-1, -1, 0, 0);
    if (k < vr.y) adj = g.vadj[vr.x + k];
    n = build_items_from<T, G>(c, adj, k < vr.y && adj.y != mn.x, &sb, ci, cs);
  }
  c.w.sync();
  return n;
}

template <typename T>
__device__ __forceinline__ int ci_group(T v, int n_g) {
  int gi = (int)(v * (T)n_g);
  return gi > n_g - 1 ? n_g - 1 : gi;
}

// Alg.-4 group of a VN whose CI was just written (E:304-307), kept with the
// group-size histogram and one membership bitmap per group (n_g x W words,
// W = ceil(N/32)), so a selection round reads k*+1 bitmap rows, not N CIs.
template <typename T, int G>
__device__ __forceinline__ void note_ci_group(Ctx<T, G>& c, int n_g, int W, int j, T v, T v_old) {
  // the old group follows from the old CI (read with the VN's record) -- no load of gid[j]
  const int gn = ci_group(v, n_g), go = ci_group(v_old, n_g);
  if (gn != go) {
    atomicSub(&c.hist[go], 1);
    atomicAdd(&c.hist[gn], 1);
    const unsigned bit = 1u << (j & 31);
    atomicAnd(&c.gbits[go * W + (j >> 5)], ~bit);
    atomicOr(&c.gbits[gn * W + (j >> 5)], bit);
    c.gid[j] = (uint8_t)gn;
  }
}

// CIRBP's CI tree is built over THRESHOLDED keys: a CI below gamma counts as 0.
// CIRBP only asks for the max-CI VN n* and whether ci[n*] < gamma (E:409-417):
// if some CI >= gamma the thresholded maximum is the true one (same lowest-index
// tie-break); if none is, the tree returns VN 0, whose CI is < gamma like the
// true maximum's, and both take the residual-argmax branch -- identical
// decisions and counters.  The gain: a refreshed VN whose CI was and stays below
// gamma (the vast majority of the ~90 per BG1 update, gamma = 0.1) does not
// touch the tree at all.
template <typename T>
__device__ __forceinline__ typename Num<T>::Key ci_tree_key(T ci, T gamma) {
  return Num<T>::key(ci >= gamma ? ci : T(0));
}

// ------------------------------------------------------------- propagate

// E:130-176.  Commit pre_c2v[e*], emit V2C to M(n*)\m*, refresh the two-hop
// pre-C2V (and, for CI schedules, pre_total / CI) state.  Leaves the item
// table of e* for the LMD searches.
// PF (state in HBM, mode 3 -- BG-sized codes): the two-hop inputs are staged
// with the V2C loads and the residual-tree level-1 update runs one lane per
// group run (fewer dependent HBM round trips); with the state in shared memory
// or L2-sized (modes 0-2) the leaner classic order has fewer live registers
// and measured faster (C1).
template <typename T, int KERNEL, bool CI, bool RT, bool CT, bool STORED, int G, bool MG = false, bool TR = false,
          bool PF = true>
__device__ int propagate(const DynParams& p, Ctx<T, G>& c, int e_star) {
  using Key = typename Num<T>::Key;
  const DevGraph& g = p.g;
  const Grp<G>& w = c.w;
  const int lane = c.lane;
  const bool PT = CI || (TR && p.pt_on);  // pre_total upkeep (E:171); TR: traced build
  // Memory round trips are the cost of an update (the chain is serial), so the
  // loads are issued level by level: the edge's records (erec, two-hop table
  // offsets) -> its VN's slots, the committed state, the two-hop items ->
  // the V2C inputs and ALL two-hop inputs / C2V values / pre values together.
  const bool tab = g.hop_items != nullptr;
  const bool pf = PF && tab;
  // graph-table loads keep their lines in L2 where the state streams from HBM (ldk)
  const unsigned long long pol = PF ? l2_keep_policy() : 0ull;
  int n_items = 0, hsp = 0;
  if (tab) {
    c.items = g.hop_items + ldk<PF>(g.hop_ptr + e_star, pol);
    n_items = ldk<PF>(g.hop_n + e_star, pol);
    hsp = ldk<PF>(g.hop_sbptr + e_star, pol);
  } else {
    c.items = c.items_buf;
  }
  const int4 er = ldk<PF>(g.erec + e_star, pol);  // (m*, n*, vn_ptr[n*], d_v(n*))
  const int m_star = er.x, n_star = er.y;
  const int2 vr = make_int2(er.z, er.w);
  int4 adj = make_int4(-1, -1, 0, 0);
  if (lane < vr.y) adj = ldk<PF>(g.vadj + vr.x + lane, pol);
  const bool act = lane < vr.y && adj.y != m_star;
  int sb0 = 0;  // stage base of this lane's check (loaded with the records above, not after the commit)
  if (PF && tab && lane < vr.y) sb0 = ldk<PF>(g.hop_sb + hsp + lane, pol);
  const T old = c.c2v[e_star];
  const T nv = c.pre[e_star];
  const T tot = c.total(n_star) + (nv - old);  // E:147
  T ptn = T(0);  // pre_total of n* (unchanged by this update: the items exclude n*'s edges)
  T cin = T(0);  // CI of n* before this update (its Alg.-4 group)
  if (CI) ptn = c.pretot(n_star);
  if (CI && (MG || CT)) cin = c.ci(n_star);
  const T gam = (T)p.gamma;  // CT: threshold of the CI-tree keys
  const T cf = act ? c.c2v[adj.x] : T(0);
  if (pf) {
    // stage the two-hop inputs now: they do not depend on this update's V2C
    // values (items exclude the V2C edges), and keep each item's C2V (and,
    // with pre_total upkeep, its old pre) for the refresh; two items per pass
    for (int t = lane; t < n_items; t += 2 * G) {
      const int t2 = t + G;
      const Item r = unpack_item(ldk<PF>(c.items + t, pol));
      Item r2 = r;
      if (t2 < n_items) r2 = unpack_item(ldk<PF>(c.items + t2, pol));
      const T x = c.in[r.g], cg = c.c2v[r.g];
      const T x2 = c.in[r2.g], cg2 = c.c2v[r2.g];
      T op = T(0), op2 = T(0);
      int j1 = 0, j2 = 0;
      if (PT) {
        op = c.pre[r.g];
        op2 = c.pre[r2.g];
        j1 = ldk<PF>(g.edge_vn + r.g, pol);
        j2 = ldk<PF>(g.edge_vn + r2.g, pol);
      }
      c.stage[r.sb + r.skip] = x;
      c.cg[t] = cg;
      if (PT) {
        c.opre[t] = op;
        c.cj[t] = j1;
      }
      if (t2 < n_items) {
        c.stage[r2.sb + r2.skip] = x2;
        c.cg[t2] = cg2;
        if (PT) {
          c.opre[t2] = op2;
          c.cj[t2] = j2;
        }
      }
    }
  }
  if (p.dump_buf && c.cur_f == 0 && c.prop == p.dump_step) {
    if (CI)
      for (int n = lane; n < g.N; n += G) {
        p.dump_buf[n] = (double)c.ci(n);
        p.dump_buf[g.N + n] = (double)c.pretot(n);
      }
    for (int e = lane; e < g.E; e += G) {
      p.dump_buf[2 * g.N + 8192 + e] = (double)c.pre[e];
      p.dump_buf[2 * g.N + 8192 + g.E + e] = (double)c.c2v[e];
    }
  }
  w.sync();
  if (lane == 0) {
    if (p.step_log && c.prop < p.log_cap) {  // (edge, committed value bits) pairs
      p.step_log[2 * (c.cur_f * p.log_cap + c.prop)] = e_star;
      p.step_log[2 * (c.cur_f * p.log_cap + c.prop) + 1] = __double_as_longlong((double)nv);
    }
    c.c2v[e_star] = nv;
    if (STORED) c.res[e_star] = T(0);
    c.total(n_star) = tot;  // n*'s own CI (E:148-149) is evaluated on spare lanes of the refresh below
  }
  // V2C to the other checks of n* (E:153-160), also staged; slots in chunks of G
  int ci_ = 0, cs_ = 0;
  for (int k0 = 0; k0 < vr.y; k0 += G) {
    int4 a2 = adj;
    bool act2 = act;
    T cf2 = cf;
    if (k0 > 0) {
      const int k = k0 + lane;
      a2 = make_int4(-1, -1, 0, 0);
      if (k < vr.y) a2 = ldk<PF>(g.vadj + vr.x + k, pol);
      act2 = k < vr.y && a2.y != m_star;
      cf2 = act2 ? c.c2v[a2.x] : T(0);
    }
    int sbase = 0;
    if (tab) {
      if (PF && k0 == 0) sbase = sb0;
      else if (k0 + lane < vr.y) sbase = ldk<PF>(g.hop_sb + hsp + k0 + lane, pol);
    } else {
      n_items = build_items_from<T, G>(c, a2, act2, &sbase, ci_, cs_);
    }
    if (act2) {
      const T v = clampv(tot - cf2);
      const T th = (KERNEL == KERNEL_EXACT) ? cn_in<T>(v) : v;
      c.in[a2.x] = th;
      c.stage[sbase + (a2.x - a2.z)] = th;
    }
  }
  w.sync();
  if (!pf) {
    for (int t = lane; t < n_items; t += G) {  // stage the rest of each check
      const Item r = unpack_item(c.items[t]);
      c.stage[r.sb + r.skip] = c.in[r.g];
    }
    w.sync();
  }
  const bool dup = PT && ldk<PF>(g.hop_dup + e_star, pol) != 0;
  auto item_g = [&](int t) -> int { return ldk<PF>((const int*)(c.items + t), pol); };  // edge id of item t
  // n*'s own CI (E:148-149: its total changed, its pre_total did not) rides on
  // spare lanes of the refresh -- kSelf pseudo-items right after the real ones
  // (kept inside one pass) -- so no lane evaluates an exp/division chain alone.
  constexpr int kSelf = CI ? CiSplit<T>::kSelfLanes : 0;
  int ps0 = n_items;
  if (kSelf == 2 && (ps0 & (G - 1)) == G - 1) ++ps0;
  const int n_loop = CI ? ps0 + kSelf : n_items;
  // two-hop refresh (E:161-176), G edges per pass in reference order
  for (int base = 0; base < n_loop; base += G) {
    const int t = base + lane;
    const bool valid = t < n_items;
    const bool self = CI && t >= ps0 && t < ps0 + kSelf;
    int j = -1;
    T delta = T(0);
    if (valid) {
      const Item r = unpack_item(ldk<PF>(c.items + t, pol));
      const int ge = r.g, skip = r.skip;
      // independent loads first (the pre[] store below would otherwise pin them)
      const T cg = pf ? c.cg[t] : c.c2v[ge];
      T opre = T(0);
      if (PT) {
        j = pf ? c.cj[t] : g.edge_vn[ge];
        opre = pf ? c.opre[t] : c.pre[ge];
      }
      const T* s = c.stage + r.sb;
      T np_;
      if (KERNEL == KERNEL_EXACT) {
        T prod = cn_one<T>();
        for (int q = 0; q < r.d; ++q)
          if (q != skip) prod = cn_mul(prod, s[q]);
        np_ = atanh_msg(prod, r.d - 1);
      } else {
        T sign = T(1), mag = Num<T>::kBig;
        for (int q = 0; q < r.d; ++q) {
          if (q == skip) continue;
          T v = clampv(s[q]);
          if (v < T(0)) { sign = -sign; v = -v; }
          if (v < mag) mag = v;
        }
        np_ = r.d > 1 ? clampv(sign * mag) : T(0);
      }
      if (PT) delta = np_ - opre;
      c.pre[ge] = np_;
      T rv = Num<T>::abs_(np_ - cg);
      if (STORED) c.res[ge] = rv;
      if (RT) c.nk[t] = Num<T>::key(rv);
    }
    if (PT) {
      bool want = false;  // this lane evaluates a CI: (cache, x) -> probe
      T cache = T(0), x = T(0), oci = T(0);
      if (!dup) {
        if (valid) {
          const typename Vec2<T>::type pq = *reinterpret_cast<const typename Vec2<T>::type*>(c.nb + 4 * j);
          if (CI && (MG || CT)) oci = c.ci(j);  // same sector as pq
          x = pq.x + delta;  // E:171
          c.pretot(j) = x;
          if (CI) {
            cache = pq.y;  // E:173 (p0(total[j]) cached)
            want = true;
            if (CT) c.cj[t] = j;
          }
        }
      } else {
        // the same VN reached through two checks (4-cycle): keep the reference's order
        const unsigned peers = w.match_any(j);
        const int rank = __popc(peers & w.lt);
        const int maxrank = (int)w.rmax(valid ? (unsigned)rank : 0u);
        for (int r = 0; r <= maxrank; ++r) {
          if (valid && rank == r) c.pretot(j) += delta;
          w.sync();
        }
        const bool last = valid && ((peers >> lane) >> 1) == 0;
        if (CI && last) {
          x = c.pretot(j);
          cache = c.p0t(j);
          if (MG || CT) oci = c.ci(j);
          want = true;
        }
        if (CT && valid) c.cj[t] = last ? j : -1;  // only the VN's final CI enters the tree
      }
      if (CI) {
        if (self) {  // n*: float64 lanes (p0(total), p0(pre_total)); float32 one lane
          x = (kSelf == 2 && t == ps0) ? tot : ptn;
          cache = tot;
        }
        T pr = T(0);
        if (want || self) pr = CiSplit<T>::probe(cache, x);
        T pr_next = T(0);
        if (kSelf == 2) pr_next = w.shfl_down(pr, 1);
        if (want) {
          const T cv = CiSplit<T>::join(cache, pr);
          c.ci(j) = cv;
          if (CT) {
            const Key kk = ci_tree_key<T>(cv, gam);
            c.ck[t] = kk;
            if (kk == ci_tree_key<T>(oci, gam) && !(cv >= gam)) c.cj[t] = -1;  // below gamma before and after
          }
          if (MG && p.fast_sel) note_ci_group(c, p.n_g, (p.g.N + 31) >> 5, j, cv, oci);
        } else if (self && t == ps0) {
          const T cv = kSelf == 2 ? Num<T>::abs_(pr - pr_next) : pr;
          c.p0t(n_star) = kSelf == 2 ? pr : tot;  // p0_cache(total[n*])
          c.ci(n_star) = cv;
          if (MG && p.fast_sel) note_ci_group(c, p.n_g, (p.g.N + 31) >> 5, n_star, cv, cin);
        }
      }
    }
  }
  w.sync();
  if (RT) {
    // incremental residual-tree update.  The leaf changes (e* -> 0, then the
    // items' new residuals; items ascend, so each 32-leaf group's items form one
    // run) are applied group by group, all groups in parallel: one lane per
    // group loads the level-1 node (one memory round trip for all of them),
    // folds in its changes and writes it back; groups whose argmax leaf
    // decreased below the new maximum are recomputed from their leaves.
    const TreeGeom& geo = p.rgeo;
    L1Node<Key>* L1 = c.rt.l1;
    int nrec = 0, ndirty = 0;
    if (PF) {
    int* segs = (int*)c.stage;  // stage is free again: run starts + sentinel
    const int qs = e_star >> 5;
    int nseg = 0;
    bool covered = false;
    for (int base = 0; base < n_items; base += G) {
      const int t = base + lane;
      const bool valid = t < n_items;
      const int q = valid ? (item_g(t) >> 5) : -1;
      const int qp = (valid && t > 0) ? (item_g(t - 1) >> 5) : -2;
      const bool start = valid && q != qp;
      const unsigned bal = w.ballot(start);
      if (start) segs[nseg + __popc(bal & w.lt)] = t;
      nseg += __popc(bal);
      covered = covered || w.any(start && q == qs);
    }
    if (lane == 0) segs[nseg] = n_items;
    w.sync();
    const int nrun = nseg + (covered ? 0 : 1);  // + e*'s group alone
    const Key k0 = Num<T>::key(T(0));
    for (int s0 = 0; s0 < nrun; s0 += G) {
      const int si = s0 + lane;
      bool rec = false, changed = false, hold = false;
      int q = -1;
      if (si < nrun) {
        int a = 0, b = 0;
        if (si < nseg) {
          a = segs[si];
          b = segs[si + 1];
          q = item_g(a) >> 5;
        } else {
          q = qs;
        }
        const L1Node<Key> nd = L1[q];
        const Key Q = nd.k;
        const int I = nd.i;
        // fold the run's changes: max new key mx (lowest leaf mi), and the
        // new key of the argmax leaf I if it changed
        Key mx = 0, nI = 0;
        int mi = 0x7fffffff;
        bool hasI = false;
        if (q == qs) {
          mx = k0;
          mi = e_star;
          if (e_star == I) { hasI = true; nI = k0; }
        }
        for (int t = a; t < b; ++t) {
          const int e = item_g(t);
          const Key kk = c.nk[t];
          if (kk > mx || (kk == mx && e < mi)) { mx = kk; mi = e; }
          if (e == I) { hasI = true; nI = kk; }
        }
        Key Qn = Q;
        int In = I;
        if (hasI && nI < Q && !(mx > Q)) {
          rec = true;  // the maximum may now sit among unchanged leaves
        } else if (mx > Q) {
          Qn = mx;
          In = mi;
        } else if (mx == Q && mi < I) {
          In = mi;
        }
        if (p.dbg_full_tree) rec = true;
        if (!rec && (Qn != Q || In != I)) {
          L1Node<Key> o;
          o.k = Qn;
          o.i = In;
          L1[q] = o;
        }
        changed = l2_note(c.rt, geo, q, Q, Qn, rec, &hold);
      }
      const unsigned rb = w.ballot(rec), cb = w.ballot(changed);
      if (rec) c.dl1[nrec + __popc(rb & w.lt)] = hold ? (q | (int)0x80000000) : q;
      if (changed) c.dl0[ndirty + __popc(cb & w.lt)] = q >> 5;  // raised level-2 node
      nrec += __popc(rb);
      ndirty += __popc(cb);
    }
    w.sync();
    } else {
      // classic order: e* first, then one pass per G items (the items of one
      // group are consecutive), the group's changes folded by a match_any leader
      const int q = e_star >> 5;
      const L1Node<Key> nd = L1[q];
      Key Q = nd.k;
      int I = nd.i;
      const Key Q0 = Q;
      const bool rec = leaf_rule(Q, I, e_star, Num<T>::key(T(0)));
      bool hold = false;
      const bool raised = l2_note(c.rt, geo, q, Q0, Q, rec, &hold);
      w.sync();
      if (lane == 0) {
        if (rec) c.dl1[nrec] = hold ? (q | (int)0x80000000) : q;
        else {
          L1Node<Key> o;
          o.k = Q;
          o.i = I;
          L1[q] = o;
        }
        if (raised) c.dl0[ndirty] = q >> 5;
      }
      nrec += rec ? 1 : 0;
      ndirty += raised ? 1 : 0;
      w.sync();
      for (int base = 0; base < n_items; base += G) {
        const int t = base + lane;
        const bool valid = t < n_items;
        const int e = valid ? c.items[t].x : -1;
        const int qq = valid ? (e >> 5) : -1;
        const Key kk = valid ? c.nk[t] : Key(0);
        const unsigned peers = w.match_any(qq);
        const bool leader = valid && (__ffs(peers) - 1) == lane;
        Key Qc = 0;
        int Ic = 0;
        if (valid) {
          const L1Node<Key> n2 = L1[qq];
          Qc = n2.k;
          Ic = n2.i;
        }
        // the group's argmax leaf decreased and nothing rose above the old max -> recompute
        const bool dec = valid && ((e == Ic && kk < Qc) || p.dbg_full_tree);
        int bi;
        const Key km = warp_max_key_minidx_masked(kk, e, peers << w.base(), &bi);
        const bool recq = (w.ballot(dec) & peers) != 0 && !(km > Qc);
        bool lrec = false, raisedq = false, holdq = false;
        if (leader) {
          Key Qn = Qc;
          if (recq) {
            lrec = true;
          } else if (km > Qc || (km == Qc && bi < Ic)) {
            Qn = km;
            L1Node<Key> o;
            o.k = km;
            o.i = bi;
            L1[qq] = o;
          }
          raisedq = l2_note(c.rt, geo, qq, Qc, Qn, lrec, &holdq);
        }
        const unsigned rb = w.ballot(lrec), cb = w.ballot(raisedq);
        if (lrec) c.dl1[nrec + __popc(rb & w.lt)] = holdq ? (qq | (int)0x80000000) : qq;
        if (raisedq) c.dl0[ndirty + __popc(cb & w.lt)] = qq >> 5;
        nrec += __popc(rb);
        ndirty += __popc(cb);
        w.sync();
      }
    }
    auto rleaf = [&](int e) -> Key { return res_key<T, STORED, G>(c, e); };
    group_recompute_list(c.rt, geo, c.dl1, nrec, w, rleaf);
    w.sync();
    l2_finish(c.rt, geo, c.dl1, nrec, c.dl0, ndirty, c.dl0 + (geo.levels > 2 ? p.dl_cap : 0), w, rleaf);
  }
  if (CT) {  // incremental CI-tree update: n* first, then the two-hop VNs
    const TreeGeom& geo = p.cgeo;
    L1Node<Key>* L1 = c.ct.l1;
    int* se = (int*)c.stage;  // stage is free again: G (index, key) pairs
    Key* sk = (Key*)(se + 32);
    int nrec = 0, ndirty = 0;
    const T cnew = c.ci(n_star);
    if (cnew >= gam || cin >= gam)
      apply_leaf_updates(c.ct, geo, lane == 0 ? n_star : -1, ci_tree_key<T>(cnew, gam), w, se, sk, c.dl1, nrec,
                         c.dl0, ndirty);
    for (int base = 0; base < n_items; base += G) {  // (VN, key) pairs staged by the refresh
      const int t = base + lane;
      int j = -1;
      Key kk = 0;
      if (t < n_items) {
        j = c.cj[t];
        kk = j >= 0 ? c.ck[t] : Key(0);
      }
      if (!w.any(j >= 0)) continue;  // every VN of this pass stayed below gamma
      apply_leaf_updates(c.ct, geo, j, kk, w, se, sk, c.dl1, nrec, c.dl0, ndirty);
    }
    auto cleaf = [&](int n) -> Key { return ci_tree_key<T>(c.ci(n), gam); };
    group_recompute_list(c.ct, geo, c.dl1, nrec, w, cleaf);
    w.sync();
    l2_finish(c.ct, geo, c.dl1, nrec, c.dl0, ndirty, c.dl0 + (geo.levels > 2 ? p.dl_cap : 0), w, cleaf);
  }
  if (MG && p.fast_sel) w.sync();
  c.count_update(vr.y - 1, n_items);
  return n_items;
}

// ------------------------------------------------------------ boundaries

template <typename T, int G>
__device__ bool syndrome_ok(const DevGraph& g, const T* total, int ts, const Grp<G>& w) {  // E:179-188
  for (int base = 0; base < g.M; base += G) {
    const int m = base + w.lane;
    int par = 0;
    if (m < g.M)
      for (int e = g.cn_ptr[m]; e < g.cn_ptr[m + 1]; ++e) par ^= (total[g.edge_vn[e] * ts] < T(0)) ? 1 : 0;
    if (w.any(par)) return false;
  }
  return true;
}

template <typename T, int G>
__device__ void record_boundary(const DynParams& p, const T* total, int ts, long long f, int k, const Grp<G>& w) {
  int errs = 0, ei = 0;
  for (int n = w.lane; n < p.g.N; n += G)
    if (total[n * ts] < T(0)) {
      ++errs;
      if (n < p.k_info) ++ei;
    }
  errs = w.rsum(errs);
  ei = w.rsum(ei);
  if (w.lane == 0) {
    p.biterr[f * (p.i_max + 1) + k] = errs;
    p.biterr_info[f * (p.i_max + 1) + k] = ei;
  }
}

template <int G>
__device__ __forceinline__ void fill_remaining(const DynParams& p, long long f, int k, const Grp<G>& w) {
  if (w.lane == 0)
    for (int kk = k + 1; kk <= p.i_max; ++kk) {
      p.biterr[f * (p.i_max + 1) + kk] = p.biterr[f * (p.i_max + 1) + k];
      p.biterr_info[f * (p.i_max + 1) + kk] = p.biterr_info[f * (p.i_max + 1) + k];
    }
  w.sync();
}

template <typename T, int G>
__device__ __forceinline__ void trace_rows(const DynParams& p, const T* total, const T* nb, long long f, int k,
                                           bool conv, const Grp<G>& w) {
  trace_boundary_rows<T, G, 4>(p.tr, p.g.N, p.i_max, total, nb, f, k, conv, w);  // records: total = nb[4n+2], pre_total = nb[4n]
}

// single-edge boundary rule (E:377-384): returns true when decoding stops
template <typename T, int G, bool TR>
__device__ __forceinline__ bool single_boundary(const DynParams& p, Ctx<T, G>& c, long long f, bool* conv) {
  if (c.prop != c.next_b) return false;
  c.next_b += p.g.E;
  const int k = ++c.it;
  record_boundary<T, G>(p, c.tb(), c.ts, f, k, c.w);
  if (syndrome_ok<T, G>(p.g, c.tb(), c.ts, c.w)) {
    *conv = true;
    fill_remaining<G>(p, f, k, c.w);
    if (TR) trace_rows<T, G>(p, c.tb(), c.nb, f, k, true, c.w);
    return true;
  }
  if (TR) trace_rows<T, G>(p, c.tb(), c.nb, f, k, false, c.w);
  return false;
}

// multi-edge boundary rule (E:633-642)
template <typename T, int G, bool TR>
__device__ void me_boundaries(const DynParams& p, Ctx<T, G>& c, long long f, int* boundary, bool* conv) {
  const long long E = p.g.E;
  while (*boundary <= p.i_max && c.prop >= (long long)(*boundary) * E) {
    record_boundary<T, G>(p, c.tb(), c.ts, f, *boundary, c.w);
    if (syndrome_ok<T, G>(p.g, c.tb(), c.ts, c.w)) {
      *conv = true;
      fill_remaining<G>(p, f, *boundary, c.w);
    }
    if (TR) trace_rows<T, G>(p, c.tb(), c.nb, f, *boundary, *conv, c.w);
    ++(*boundary);
    if (*conv) break;
  }
}

// ------------------------------------------------- RNG + VN selection (E:279-352)

__device__ __forceinline__ long long rand_next(long long* st) {
  unsigned long long x = (unsigned long long)(*st) * 6364136223846793005ULL + 1442695040888963407ULL;
  *st = (long long)x;
  long long z = (long long)x;
  z ^= z >> 33;
  z = (long long)((unsigned long long)z * 0xFF51AFD7ED558CCDULL);
  z ^= z >> 33;
  if (z < 0) z = -(z + 1);
  return z;
}


// Select up to n_p VNs (excluding n with excl[n] != 0 when excl != nullptr)
// into out[0..count), ascending.  Reproduces _select_vns exactly.
// k* of Alg. 4 from a group-size histogram: the largest k with
// sum_{q >= n_g-k} size[q] <= n_p (E:308-314); *sel_total = that sum.
template <typename T, int G>
__device__ __forceinline__ int kstar_of(Ctx<T, G>& c, const int* hist, int n_g, int n_p, int* sel_total) {
  int k_star = 0, tot = 0;
  if (n_g <= G) {
    const int v = c.lane < n_g ? hist[n_g - 1 - c.lane] : 0;
    const int cum = c.w.incl_scan(v);
    k_star = __popc(c.w.ballot(c.lane < n_g && cum <= n_p));
    tot = c.w.shfl(cum, k_star > 0 ? k_star - 1 : 0);
    if (k_star == 0) tot = 0;
  } else {
    if (c.lane == 0) {
      long long cum = 0;
      for (int k = 1; k <= n_g; ++k) {
        cum += hist[n_g - k];
        if (cum <= n_p) {
          k_star = k;
          tot = (int)cum;
        } else {
          break;
        }
      }
    }
    k_star = c.w.shfl(k_star, 0);
    tot = c.w.shfl(tot, 0);
  }
  *sel_total = tot;
  return k_star;
}

// Alg.-4 tail shared by the selection variants: random fill from the next
// group's members[0..idx) (partial Fisher-Yates, E:316-325), then ascending order.
template <typename T, int G>
__device__ int select_finish(const DynParams& p, Ctx<T, G>& c, int n_p, int* out, int count, int idx,
                             bool want_fill) {
  if (count < n_p && want_fill) {
    int need = n_p - count;
    if (need > idx) need = idx;
    if (c.lane == 0) {
      long long st = c.rng;
      for (int t = 0; t < need; ++t) {
        int r = t + (int)(rand_next(&st) % (long long)(idx - t));
        int tmp = c.members[t];
        c.members[t] = c.members[r];
        c.members[r] = tmp;
        out[count + t] = c.members[t];
      }
      c.rng = st;
    }
    c.rng = c.w.shfl(c.rng, 0);
    count += need;
  }
  c.w.sync();
  if (p.dump_buf && c.cur_f == 0 && c.lane == 0 && c.nsel < 8192)
    p.dump_buf[2 * p.g.N + c.nsel] = __longlong_as_double(c.rng);
  ++c.nsel;
  for (int i = c.lane; i < count; i += G) {
    int v = out[i], r = 0;
    for (int q = 0; q < count; ++q) r += out[q] < v;
    c.members[r] = v;
  }
  c.w.sync();
  for (int i = c.lane; i < count; i += G) out[i] = c.members[i];
  c.w.sync();
  return count;
}

template <typename T, int G>
__device__ int select_vns(const DynParams& p, Ctx<T, G>& c, const uint8_t* excl, int n_p, int* out) {
  if (p.fast_sel && !excl) {  // maintained histogram + group bitmaps
    const int N = p.g.N, n_g = p.n_g, lane = c.lane, W = (N + 31) >> 5;
    int sel_total;
    const int k_star = kstar_of(c, c.hist, n_g, n_p, &sel_total);
    const int thr = n_g - k_star, fill = thr - 1;
    const bool mat = k_star < n_g && sel_total < n_p;  // fill members needed
    const int fill_size = mat ? c.hist[fill] : 0;
    const int need = mat ? min(n_p - sel_total, fill_size) : 0;
    // few picks from a big group: Fisher-Yates on the implicit member list
    // (rank queries on the group bitmap) instead of materialising it
    const bool lazy = mat && 4 * need <= fill_size;
    const unsigned* bits = c.gbits;
    int* wpre = c.members;  // lazy: members before each bitmap word
    int count = 0, idx = 0;
    if (sel_total > 0 || mat) {
      for (int base = 0; base < W; base += G) {
        const int wi = base + lane;
        unsigned sw = 0u, fw = 0u;
        if (wi < W) {
          if (sel_total > 0)
            for (int q = thr; q < n_g; ++q)
              if (c.hist[q]) sw |= bits[q * W + wi];
          if (mat) fw = bits[fill * W + wi];
        }
        const int packed = __popc(sw) | (__popc(fw) << 16);
        const int incl = c.w.incl_scan(packed);
        const int tot = c.w.shfl(incl, G - 1);
        int ps = count + ((incl - packed) & 0xffff);
        int pf = idx + ((incl - packed) >> 16);
        while (sw) {
          out[ps++] = wi * 32 + __ffs(sw) - 1;
          sw &= sw - 1;
        }
        if (lazy) {
          if (wi < W) wpre[wi] = pf;
        } else {
          while (fw) {
            c.members[pf++] = wi * 32 + __ffs(fw) - 1;
            fw &= fw - 1;
          }
        }
        count += tot & 0xffff;
        idx += tot >> 16;
      }
    }
    c.w.sync();
    if (!lazy) return select_finish(p, c, n_p, out, count, idx, mat);
    // lazy partial Fisher-Yates (E:316-325), warp-uniform; overrides (pos, value)
    int* ov = c.members + W;
    const unsigned* fb = bits + (long long)fill * W;
    auto member_at = [&](int pos, int n_ov) -> int {
      int hit = -1;  // latest override of pos
      for (int i0 = 0; i0 < n_ov; i0 += G) {
        const bool h = i0 + lane < n_ov && ov[2 * (i0 + lane)] == pos;
        const unsigned bal = c.w.ballot(h);
        if (bal) hit = c.w.shfl(h ? ov[2 * (i0 + lane) + 1] : 0, 31 - __clz(bal));
      }
      if (hit >= 0) return hit;
      // the bitmap word holding member `pos`: the last word with wpre <= pos
      // (wpre is non-decreasing, wpre[0] = 0).  Two votes -- every S-th word,
      // then the S words of that block -- instead of a linear scan (BG1: 816 words)
      int nle = 0;
      const int S = (W + G - 1) / G;
      if (S <= G && W > G) {
        const unsigned b1 = c.w.ballot(lane * S < W && wpre[lane * S] <= pos);
        const int b0 = (__popc(b1) - 1) * S;
        const unsigned b2 = c.w.ballot(lane < S && b0 + lane < W && wpre[b0 + lane] <= pos);
        nle = b0 + __popc(b2);
      } else {
        for (int base = 0; base < W; base += G) {
          const unsigned bal = c.w.ballot(base + lane < W && wpre[base + lane] <= pos);
          nle += __popc(bal);
          if (bal != (G == 32 ? 0xffffffffu : (1u << G) - 1u)) break;
        }
      }
      const int wsel = nle - 1;
      return wsel * 32 + (int)__fns(fb[wsel], 0, pos - wpre[wsel] + 1);
    };
    long long st = c.rng;
    for (int t = 0; t < need; ++t) {
      const int r = t + (int)(rand_next(&st) % (long long)(idx - t));
      const int vr = member_at(r, t);
      if (t + 1 < need) {
        const int vt = member_at(t, t);
        c.w.sync();
        if (lane == 0) {
          ov[2 * t] = r;
          ov[2 * t + 1] = vt;
        }
      }
      if (lane == 0) out[count + t] = vr;
      c.w.sync();
    }
    c.rng = st;
    return select_finish(p, c, n_p, out, count + need, idx, false);
  }
  if (p.fast_sel) {  // excluded set (ME-LMD-CIRBP top-up): maintained group bytes
    const int N = p.g.N, n_g = p.n_g, lane = c.lane;
    for (int q = lane; q < n_g; q += G) c.sizes[q] = c.hist[q];
    c.w.sync();
    for (int n0 = 4 * lane; n0 < N; n0 += 4 * G) {  // histogram of the non-excluded VNs
      const unsigned xv = *(const unsigned*)(excl + n0);
      if (!xv) continue;
      const unsigned wv = *(const unsigned*)(c.gid + n0);
      for (int b = 0; b < 4 && n0 + b < N; ++b)
        if ((xv >> (8 * b)) & 0xff) atomicSub(&c.sizes[(wv >> (8 * b)) & 0xff], 1);
    }
    c.w.sync();
    int sel_total;
    const int k_star = kstar_of(c, c.sizes, n_g, n_p, &sel_total);
    const int thr = n_g - k_star;
    const int fill = n_g - k_star - 1;
    const bool want_fill = k_star < n_g && sel_total < n_p;
    int count = 0, idx = 0;
    for (int base = 0; base < N; base += 4 * G) {  // 4 VNs per lane, ascending
      const int n0 = base + 4 * lane;
      const unsigned wv = n0 < N ? *(const unsigned*)(c.gid + n0) : 0u;
      const unsigned xv = n0 < N ? *(const unsigned*)(excl + n0) : 0u;
      int sel = 0, fil = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int gb = (wv >> (8 * b)) & 0xff;
        const bool in = n0 + b < N && !((xv >> (8 * b)) & 0xff);
        sel += in && gb >= thr;
        fil += in && want_fill && gb == fill;
      }
      const int packed = sel | (fil << 8);
      const int incl = c.w.incl_scan(packed);
      const int tot = c.w.shfl(incl, G - 1);
      int ps = count + ((incl - packed) & 0xff);
      int pf = idx + ((incl - packed) >> 8);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int gb = (wv >> (8 * b)) & 0xff;
        if (n0 + b >= N) break;
        if ((xv >> (8 * b)) & 0xff) continue;
        if (gb >= thr) out[ps++] = n0 + b;
        else if (want_fill && gb == fill) c.members[pf++] = n0 + b;
      }
      count += tot & 0xff;
      idx += tot >> 8;
    }
    c.w.sync();
    return select_finish(p, c, n_p, out, count, idx, want_fill);
  }
  const int N = p.g.N, n_g = p.n_g, lane = c.lane;
  for (int q = lane; q < n_g; q += G) c.sizes[q] = 0;
  c.w.sync();
  for (int n = lane; n < N; n += G)
    if (!excl || !excl[n]) atomicAdd(&c.sizes[ci_group(c.ci(n), n_g)], 1);
  c.w.sync();
  int sel_total;
  const int k_star = kstar_of(c, c.sizes, n_g, n_p, &sel_total);
  const int thr = n_g - k_star, fill = thr - 1;
  const bool want_fill = k_star < n_g && sel_total < n_p;
  int count = 0, idx = 0;
  for (int base = 0; base < N; base += G) {
    const int n = base + lane;
    int gi = -1;
    if (n < N && (!excl || !excl[n])) gi = ci_group(c.ci(n), n_g);
    const bool s = gi >= thr, f = want_fill && gi == fill;
    const unsigned bs = c.w.ballot(s), bf = c.w.ballot(f);
    if (s) out[count + __popc(bs & c.w.lt)] = n;
    if (f) c.members[idx + __popc(bf & c.w.lt)] = n;
    count += __popc(bs);
    idx += __popc(bf);
  }
  c.w.sync();
  return select_finish(p, c, n_p, out, count, idx, want_fill);
}

// sort ints ascending in place (distinct values), via members[] scratch
template <typename T, int G>
__device__ void sort_small(Ctx<T, G>& c, int* a, int count) {
  for (int i = c.lane; i < count; i += G) {
    int v = a[i], r = 0;
    for (int q = 0; q < count; ++q) r += a[q] < v;
    c.members[r] = v;
  }
  c.w.sync();
  for (int i = c.lane; i < count; i += G) a[i] = c.members[i];
  c.w.sync();
}

// --------------------------------------------------------- local searches

// E:436-469 after propagate(e_prev) left the item table of e_prev.
template <typename T, int G>
__device__ int lmd_next_edge(const DynParams& p, Ctx<T, G>& c, int e_prev, int n_items, bool simplified) {
  using Key = typename Num<T>::Key;
  const DevGraph& g = p.g;
  const int lane = c.lane;
  const int2 mn = g.ecv[e_prev];
  const bool deg1 = g.vrec[mn.y].y == 1;
  Key bk = 0;
  int bi = 0x7fffffff, ncand;
  if (deg1) {
    int a = g.cn_ptr[mn.x], b = g.cn_ptr[mn.x + 1];
    ncand = b - a - 1;
    for (int e = a + lane; e < b; e += G)
      if (e != e_prev) {
        Key k = res_key<T, false, G>(c, e);
        if (k > bk) { bk = k; bi = e; }
      }
  } else {
    ncand = n_items;
    for (int t = lane; t < n_items; t += G) {
      int e = c.items[t].x;
      Key k = res_key<T, false, G>(c, e);
      if (k > bk) { bk = k; bi = e; }
    }
  }
  if (ncand > 1) c.count(C_CMP, ncand - 1);
  if (ncand <= 0) return -1;
  int best;
  c.w.max_key_minidx(bk, bi, &best);
  if (!simplified) {
    int dv_ = 0;
    int np_ = g.edge_vn[best];
    best = argmax_vn_edges<T, G>(g, c, np_, &dv_);
    c.count(C_CMP, dv_ - 1);
  }
  return best;
}

// E:513-552: max-CI VN of the two-hop set of e_prev, ties -> lowest VN; the
// candidate count (deduplicated, E:536-549) is precomputed per edge.
template <typename T, int G>
__device__ int ci_argmax_twohop(const DynParams& p, Ctx<T, G>& c, int e_prev, int n_items, bool have_items) {
  using Key = typename Num<T>::Key;
  const DevGraph& g = p.g;
  const int lane = c.lane;
  const int2 mn = g.ecv[e_prev];
  const bool deg1 = g.vrec[mn.y].y == 1;
  Key bk = 0;
  int bj = 0x7fffffff, ncand;
  if (deg1) {
    int a = g.cn_ptr[mn.x], b = g.cn_ptr[mn.x + 1];
    ncand = b - a - 1;
    for (int e = a + lane; e < b; e += G)
      if (e != e_prev) {
        int j = g.edge_vn[e];
        Key k = Num<T>::key(c.ci(j));
        if (k > bk || (k == bk && j < bj)) { bk = k; bj = j; }
      }
  } else {
    if (!have_items) n_items = build_items<T, G>(g, c, e_prev);
    ncand = g.hop_distinct[e_prev];
    for (int t = lane; t < n_items; t += G) {
      int j = g.edge_vn[c.items[t].x];
      Key k = Num<T>::key(c.ci(j));
      if (k > bk || (k == bk && j < bj)) { bk = k; bj = j; }
    }
  }
  if (ncand > 1) c.count(C_CMP, ncand - 1);
  if (ncand <= 0) return -1;
  int best;
  c.w.max_key_minidx(bk, bj, &best);
  return best;
}

// ---------------------------------------------- multi-edge round pairing
// Within a multi-edge round the reference applies the selected VNs one after
// another in ascending order (E:625-632, SP:407).  Two consecutive VNs a < b
// touch disjoint state -- so their updates commute exactly, bit for bit --
// when no VN lies within one check of both, N2(a) ∩ N2(b) = ∅ (N2(v) = the
// VNs sharing a check with v, v included): then b is not refreshed by a and
// vice versa (b's residuals, total, CI untouched), they share no check (no
// V2C / staged input in common) and no pre_total sum receives updates from
// both (no order-dependent float additions).  Such a pair is applied
// concurrently, one VN per half-warp; otherwise one after the other.
// Opt-in (LDPC_VARIANT_ME_PAIRS): exact, but measured 2x slower on C1
// ME-CIRBP(4) and 1.5x on C3 ME-CIRBP(64) -- the two half-warps run different
// data through data-dependent loops, diverge and serialise, and the conflict
// test costs two extra dependent loads per pair.
template <typename T>
__device__ bool me_pair_disjoint(const DevGraph& g, Ctx<T, 32>& c, int a, int b, int cap) {
  const int a0 = g.vn2_ptr[a], la = g.vn2_ptr[a + 1] - a0;
  const int b0 = g.vn2_ptr[b], lb = g.vn2_ptr[b + 1] - b0;
  if (la > cap) return false;
  int* A = (int*)c.stage;  // free between updates
  for (int t = c.lane; t < la; t += 32) A[t] = g.vn2[a0 + t];
  c.w.sync();
  bool hit = false;
  for (int t = c.lane; t < lb && !hit; t += 32) {
    const int x = g.vn2[b0 + t];
    int lo = 0, hi = la;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (A[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    hit = lo < la && A[lo] == x;
  }
  const bool any = c.w.any(hit);
  c.w.sync();
  return !any;
}

// The half-warp context of half h: the frame's state and selection state are
// shared, the per-update scratch is the half's own.
template <typename T>
__device__ Ctx<T, 16> half_ctx(const DynParams& p, const Ctx<T, 32>& c, int half) {
  Ctx<T, 16> h;
  h.w = Grp<16>::make();
  h.lane = h.w.lane;
  h.c2v = c.c2v; h.pre = c.pre; h.in = c.in; h.res = c.res; h.nb = c.nb; h.cs = c.cs;
  h.tmp = c.tmp;
  h.rt = c.rt; h.ct = c.ct;
  h.inpp = c.inpp; h.gid = c.gid; h.hist = c.hist; h.gbits = c.gbits;
  h.members = c.members; h.sel = c.sel; h.chosen = c.chosen; h.sizes = c.sizes;
  const long long d = half ? (long long)(p.so_pair - p.so_items) : 0;
  auto sh = [&](auto* ptr) { return (decltype(ptr))((unsigned char*)ptr + d); };
  h.items_buf = sh(c.items_buf);
  h.items = h.items_buf;
  h.stage = sh(c.stage);
  h.nk = sh(c.nk);
  h.cg = sh(c.cg);
  h.opre = sh(c.opre);
  h.cj = sh(c.cj);
  h.ck = sh(c.ck);
  h.dl0 = sh(c.dl0);
  h.dl1 = sh(c.dl1);
  h.cbase = c.cntp();  // both halves add (atomically) into the frame's counters
  h.prop = c.prop + half;
  h.cur_f = c.cur_f;
  h.nsel = c.nsel;
  h.next_b = c.next_b;
  h.it = c.it;
  h.rng = c.rng;
  return h;
}

// sel[idx] and sel[idx+1] on the two half-warps (CI kinds: E:625-632 per VN)
template <typename T, int KERNEL, bool TR, bool PF>
__device__ void me_pair_step(const DynParams& p, Ctx<T, 32>& c, int idx, int* chosen) {
  const int half = c.lane >> 4;
  Ctx<T, 16> h = half_ctx<T>(p, c, half);
  const int pv = c.sel[idx + half];
  int dv = 0;
  const int e = argmax_vn_edges<T, 16>(p.g, h, pv, &dv);
  h.count(C_CMP, dv - 1);
  if (chosen && h.lane == 0) chosen[idx + half] = e;
  propagate<T, KERNEL, true, false, false, false, 16, true, TR, PF>(p, h, e);
  __syncwarp();
  c.prop += 2;
}

// --------------------------------------------------------------- decoders

// kind: the decode_frame kind (a compile-time constant in per-kind kernels, so
// the ME-only setup below drops out of the other kernels entirely)
template <typename T, int KERNEL, bool CI, int G, bool TR = false>
__device__ void init_state(const DynParams& p, Ctx<T, G>& c, long long f, int kind) {  // E:106-127
  const DevGraph& g = p.g;
  const int lane = c.lane;
  const float* l32 = (const float*)p.llr + f * g.N;
  const double* l64 = (const double*)p.llr + f * g.N;
  auto chl = [&](int n) -> T { return p.llr_f64 ? (T)l64[n] : (T)l32[n]; };
  for (int e = lane; e < g.E; e += G) {
    T v = clampv(chl(g.edge_vn[e]));
    c.c2v[e] = T(0);
    c.in[e] = (KERNEL == KERNEL_EXACT) ? cn_in<T>(v) : v;
  }
  for (int n = lane; n < g.N; n += G) c.total(n) = chl(n);
  c.w.sync();
  for (int m = lane; m < g.M; m += G) {
    int a = g.cn_ptr[m], b = g.cn_ptr[m + 1];
    for (int e = a; e < b; ++e) c.pre[e] = cn_msg_cached<T, KERNEL>(c.in, a, b, e);
  }
  c.w.sync();
  if (CI || (TR && p.pt_on))
    for (int n = lane; n < g.N; n += G) {
      T acc = chl(n);
      for (int k = g.vn_ptr[n]; k < g.vn_ptr[n + 1]; ++k) acc += c.pre[g.vn_edges[k]];
      c.pretot(n) = acc;  // E:121-125
      if (CI) {
        const T pt = p0_cache(c.total(n));
        c.p0t(n) = pt;
        c.ci(n) = ci_cached(pt, acc);
      }
    }
  if ((kind == KIND_ME_CIRBP || kind == KIND_ME_LMD_CIRBP) && p.fast_sel) {
    const int W = (g.N + 31) >> 5;
    for (int q = lane; q < p.n_g; q += G) c.hist[q] = 0;
    for (int q = lane; q < p.n_g * W; q += G) c.gbits[q] = 0u;
    c.w.sync();
    for (int n = lane; n < g.N; n += G) {
      const int gi = ci_group(c.ci(n), p.n_g);
      c.gid[n] = (uint8_t)gi;
      atomicAdd(&c.hist[gi], 1);
      atomicOr(&c.gbits[gi * W + (n >> 5)], 1u << (n & 31));
    }
  }
  if (kind == KIND_ME_LMD_CIRBP)
    for (int n = lane; n < g.N; n += G) c.inpp[n] = 0;
  c.w.sync();
}

// ME-RBP round selection on a single-level residual tree: the top-m leaves by
// (key desc, index asc) -- the set m repeated argmax-and-exclude passes pick
// (oracle decode_me_rbp).  Any leaf of that set lies in one of the top-m
// level-1 groups ordered by (group max, group index): otherwise m groups rank
// above its own group, and their maxima are m leaves ranking above it.
template <typename T, int G, typename LeafFn>
__device__ void me_topm_registers(const DynParams& p, Ctx<T, G>& c, int m, LeafFn leaf) {
  using Key = typename Num<T>::Key;
  constexpr int kBad = 0x7fffffff;
  const int lane = c.lane, s = p.rgeo.size[1], E = p.g.E;
  const L1Node<Key>* L1 = c.rt.l1;
  Key k0 = lane < s ? L1[lane].k : Key(0), k1 = lane + 32 < s ? L1[lane + 32].k : Key(0);
  bool v0 = lane < s, v1 = lane + 32 < s;
  int gq[4] = {kBad, kBad, kBad, kBad};
  int ng = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (t >= m) break;
    Key bk = 0;
    int bi = kBad;
    if (v0) { bk = k0; bi = lane; }
    if (v1 && (bi == kBad || k1 > bk)) { bk = k1; bi = lane + 32; }
    int q;
    c.w.max_key_minidx(bk, bi, &q);
    if (q == kBad) break;
    gq[t] = q;
    ++ng;
    if (q == lane) v0 = false;
    if (q == lane + 32) v1 = false;
  }
  Key ck[4];
  int ce[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int e = j < ng ? gq[j] * 32 + lane : E;
    ce[j] = e < E ? e : kBad;
    ck[j] = e < E ? leaf(e) : Key(0);
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (t >= m) break;
    Key bk = 0;
    int bi = kBad;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (ce[j] != kBad && (bi == kBad || ck[j] > bk || (ck[j] == bk && ce[j] < bi))) {
        bk = ck[j];
        bi = ce[j];
      }
    int e;
    c.w.max_key_minidx(bk, bi, &e);
    if (lane == 0) c.sel[t] = e;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (ce[j] == e) ce[j] = kBad;
  }
  c.w.sync();
}

template <typename T, int KERNEL, int KF, int G, bool TR, int MODE = 3, bool MP = false>
__device__ void decode_frame(const DynParams& p, Ctx<T, G>& c, long long f) {
  constexpr bool PF = MODE == 3;
  const int kind = KF >= 0 ? KF : p.kind;  // KF: kind fixed at compile time (-1: runtime)
  int dv_ = 0;  // degree of the VN argmax_vn_edges just scanned
  using Key = typename Num<T>::Key;
  const DevGraph& g = p.g;
  const long long E = g.E, budget = (long long)p.i_max * E;
  const int lane = c.lane, I = p.i_max;
  if (lane < kCounters) c.cntp()[lane] = 0;
  c.w.sync();
  c.prop = 0;
  c.cur_f = f;
  c.nsel = 0;
  c.next_b = E;
  c.it = 0;
  c.rng = p.seed;
  bool conv = false;
  if (lane == 0) {
    for (int k = 0; k <= I; ++k) p.biterr[f * (I + 1) + k] = p.biterr_info[f * (I + 1) + k] = 0;
    if (kind == KIND_CIRBP)
      for (int k = 0; k < I; ++k) p.kh[f * I + k] = p.kt[f * I + k] = 0;
  }
  const bool ci_kind = kind == KIND_CIRBP || kind == KIND_LMD_CIRBP || kind == KIND_ME_CIRBP ||
                       kind == KIND_ME_LMD_CIRBP;
  if (ci_kind) init_state<T, KERNEL, true, G, TR>(p, c, f, kind);
  else init_state<T, KERNEL, false, G, TR>(p, c, f, kind);
  record_boundary<T, G>(p, c.tb(), c.ts, f, 0, c.w);
  if (TR) trace_rows<T, G>(p, c.tb(), c.nb, f, 0, false, c.w);
  auto rleaf = [&](int e) -> Key { return res_key<T, false, G>(c, e); };
  auto cleaf = [&](int n) -> Key { return Num<T>::key(c.ci(n)); };

  switch (kind) {
    case KIND_RBP: {  // E:355-385
      tree_build(c.rt, p.rgeo, c.w, rleaf);
      while (c.prop < budget) {
        int e = tree_argmax(c.rt, p.rgeo, c.w, rleaf);
        c.count(C_CMP, E - 1);
        propagate<T, KERNEL, false, true, false, false, G, false, TR, PF>(p, c, e);
        ++c.prop;
        if (single_boundary<T, G, TR>(p, c, f, &conv)) break;
      }
    } break;
    case KIND_CIRBP: {  // E:388-433
      const T gamma = (T)p.gamma;
      auto tleaf = [&](int n) -> Key { return ci_tree_key<T>(c.ci(n), gamma); };  // thresholded CI-tree keys
      tree_build(c.rt, p.rgeo, c.w, rleaf);
      tree_build(c.ct, p.cgeo, c.w, tleaf);
      int kh = 0, kt = 0;  // per-iteration kappa tallies (warp-uniform)
      while (c.prop < budget) {
        const int it = c.it;
        int n_star = tree_argmax(c.ct, p.cgeo, c.w, tleaf);
        c.count(C_CMP, g.N - 1 + 1);
        c.count(C_KTRIALS, 1);
        ++kt;
        bool hit = c.ci(n_star) < gamma;
        int e;
        if (hit) {
          c.count(C_KHITS, 1);
          ++kh;
          e = tree_argmax(c.rt, p.rgeo, c.w, rleaf);
          c.count(C_CMP, E - 1);
        } else {
          e = argmax_vn_edges<T, G, PF>(g, c, n_star, &dv_);
          c.count(C_CMP, dv_ - 1);
        }
        propagate<T, KERNEL, true, true, true, false, G, false, TR, PF>(p, c, e);
        ++c.prop;
        if (c.prop == c.next_b || c.prop >= budget) {
          if (lane == 0) {
            p.kh[f * I + it] = kh;
            p.kt[f * I + it] = kt;
          }
          kh = kt = 0;
        }
        if (single_boundary<T, G, TR>(p, c, f, &conv)) break;
      }
    } break;
    case KIND_LMDRBP:
    case KIND_SLMDRBP: {  // E:472-510
      const bool simplified = p.kind == KIND_SLMDRBP;  // sLMDRBP runs the LMDRBP kernel
      int e = argmax_scan<Key>(g.E, c.w, rleaf);
      c.count(C_CMP, E - 1);
      while (c.prop < budget) {
        int n_items = propagate<T, KERNEL, false, false, false, false, G, false, TR, PF>(p, c, e);
        ++c.prop;
        if (single_boundary<T, G, TR>(p, c, f, &conv)) break;
        if (c.prop >= budget) break;
        int en = lmd_next_edge<T, G>(p, c, e, n_items, simplified);
        if (en < 0) {
          en = argmax_scan<Key>(g.E, c.w, rleaf);
          c.count(C_CMP, E - 1);
        }
        e = en;
      }
    } break;
    case KIND_LMD_CIRBP: {  // E:555-598
      int n_star = argmax_scan<Key>(g.N, c.w, cleaf);
      c.count(C_CMP, g.N - 1);
      int e = argmax_vn_edges<T, G, PF>(g, c, n_star, &dv_);
      c.count(C_CMP, dv_ - 1);
      while (c.prop < budget) {
        int n_items = propagate<T, KERNEL, true, false, false, false, G, false, TR, PF>(p, c, e);
        ++c.prop;
        if (single_boundary<T, G, TR>(p, c, f, &conv)) break;
        if (c.prop >= budget) break;
        int nn = ci_argmax_twohop<T, G>(p, c, e, n_items, true);
        if (nn < 0) {
          nn = argmax_scan<Key>(g.N, c.w, cleaf);
          c.count(C_CMP, g.N - 1);
        }
        e = argmax_vn_edges<T, G>(g, c, nn, &dv_);
        c.count(C_CMP, dv_ - 1);
      }
    } break;
    case KIND_ME_CIRBP: {  // E:601-643
      int boundary = 1;
      while (boundary <= I && !conv) {
        int count = select_vns<T, G>(p, c, nullptr, p.n_p, c.sel);
        c.count(C_MSEL, p.n_g);
        for (int idx = 0; idx < count;) {
          if constexpr (G == 32 && MP) {  // MP: the round-pairing build (opt-in variant)
            if (p.me_pairs && idx + 1 < count && me_pair_disjoint<T>(g, c, c.sel[idx], c.sel[idx + 1], p.pair_cap)) {
              me_pair_step<T, KERNEL, TR, PF>(p, c, idx, nullptr);
              idx += 2;
              continue;
            }
          }
          int pv = c.sel[idx];
          int e = argmax_vn_edges<T, G, PF>(g, c, pv, &dv_);
          c.count(C_CMP, dv_ - 1);
          propagate<T, KERNEL, true, false, false, false, G, true, TR, PF>(p, c, e);
          ++c.prop;
          ++idx;
        }
        me_boundaries<T, G, TR>(p, c, f, &boundary, &conv);
      }
    } break;
    case KIND_ME_LMD_CIRBP: {  // E:646-716
      int boundary = 1;
      int count = select_vns<T, G>(p, c, nullptr, p.n_p, c.sel);
      c.count(C_MSEL, p.n_g);
      while (boundary <= I && !conv) {
        for (int idx = 0; idx < count;) {
          if constexpr (G == 32 && MP) {  // MP: the round-pairing build (opt-in variant)
            if (p.me_pairs && idx + 1 < count && me_pair_disjoint<T>(g, c, c.sel[idx], c.sel[idx + 1], p.pair_cap)) {
              me_pair_step<T, KERNEL, TR, PF>(p, c, idx, c.chosen);
              idx += 2;
              continue;
            }
          }
          int pv = c.sel[idx];
          int e = argmax_vn_edges<T, G, PF>(g, c, pv, &dv_);
          c.count(C_CMP, dv_ - 1);
          if (lane == 0) c.chosen[idx] = e;
          propagate<T, KERNEL, true, false, false, false, G, true, TR, PF>(p, c, e);
          ++c.prop;
          ++idx;
        }
        me_boundaries<T, G, TR>(p, c, f, &boundary, &conv);
        if (conv || boundary > I) break;
        // P' = two-hop max-CI VN of each chosen edge, deduplicated in order
        int npc = 0;
        for (int idx = 0; idx < count; ++idx) {
          int pn = ci_argmax_twohop<T, G>(p, c, c.chosen[idx], 0, false);
          bool add = pn >= 0 && !c.inpp[pn];
          c.w.sync();
          if (add) {
            if (lane == 0) {
              c.inpp[pn] = 1;
              c.sel[npc] = pn;
            }
            ++npc;
          }
          c.w.sync();
        }
        if (npc < p.n_p) {
          int extra = select_vns<T, G>(p, c, c.inpp, p.n_p - npc, c.sel + npc);
          c.count(C_MSEL, p.n_g);
          count = npc + extra;
        } else {
          count = npc;
        }
        for (int idx = lane; idx < npc; idx += G) c.inpp[c.sel[idx]] = 0;
        c.w.sync();
        sort_small<T, G>(c, c.sel, count);
      }
    } break;
    case KIND_ME_RBP: {  // new (oracle/ldpc_oracle.c decode_me_rbp): stored residuals
      for (int e = lane; e < g.E; e += G) c.res[e] = Num<T>::abs_(c.pre[e] - c.c2v[e]);
      c.w.sync();
      auto sleaf = [&](int e) -> Key { return res_key<T, true, G>(c, e); };
      tree_build(c.rt, p.rgeo, c.w, sleaf);
      int boundary = 1;
      const int np_ = p.n_p < g.E ? p.n_p : g.E;
      // single-level residual tree (<= 64 groups of 32 leaves) and M <= 4: the
      // round's top-M set in registers -- top-M groups by (max key, index),
      // which must contain the top-M leaves, then top-M among their leaves --
      // instead of M argmax / exclude / recompute passes over the tree
      const bool reg_topm = G == 32 && p.rgeo.levels == 1 && np_ <= 4;
      while (boundary <= I && !conv && reg_topm) {
        me_topm_registers<T, G>(p, c, np_, sleaf);
        c.count(C_CMP, E - 1);
        sort_small<T, G>(c, c.sel, np_);
        for (int idx = 0; idx < np_; ++idx) {
          propagate<T, KERNEL, false, true, false, true, G, false, TR, PF>(p, c, c.sel[idx]);
          ++c.prop;
        }
        me_boundaries<T, G, TR>(p, c, f, &boundary, &conv);
      }
      while (boundary <= I && !conv) {
        for (int t = 0; t < np_; ++t) {
          int e = tree_argmax(c.rt, p.rgeo, c.w, sleaf);
          if (lane == 0) {
            c.sel[t] = e;
            c.tmp[t] = c.res[e];
            c.res[e] = T(-1);  // excluded: key 0
            c.dl0[0] = e >> 5;
          }
          c.w.sync();
          tree_update_list(c.rt, p.rgeo, c.dl0, c.dl1, 1, c.w, sleaf);
        }
        for (int t = lane; t < np_; t += G) {
          c.res[c.sel[t]] = c.tmp[t];
          c.dl0[t] = c.sel[t] >> 5;
        }
        c.w.sync();
        tree_update_list(c.rt, p.rgeo, c.dl0, c.dl1, np_, c.w, sleaf);
        c.count(C_CMP, E - 1);
        sort_small<T, G>(c, c.sel, np_);
        for (int idx = 0; idx < np_; ++idx) {
          propagate<T, KERNEL, false, true, false, true, G, false, TR, PF>(p, c, c.sel[idx]);
          ++c.prop;
        }
        me_boundaries<T, G, TR>(p, c, f, &boundary, &conv);
      }
    } break;
    default:
      break;
  }
  if (I == 0) conv = syndrome_ok<T, G>(g, c.tb(), c.ts, c.w);  // schedules.py:144-146
  for (int n = lane; n < g.N; n += G) p.u_hat[f * g.N + n] = c.total(n) < T(0) ? 1 : 0;
  c.store_counters(p.counters + f * kCounters, ci_kind);
  if (lane == 0) {
    p.prop[f] = c.prop;
    p.conv[f] = conv ? 1 : 0;
  }
  c.w.sync();
}

// MODE 0: E, N and T parts in shared memory; 1: E in HBM, N and T in shared;
// 2: E and N in HBM, T in shared; 3: everything in HBM.  G lanes per frame
// (32/G frames per warp); slots and scratch are per frame.
template <typename T, int KERNEL, int MODE, int KF, int G, bool TR = false, bool MP = false>
__global__ void __launch_bounds__(256, dyn_min_blocks(KF, sizeof(T) == 8, MODE)) dyn_decode_kernel(const __grid_constant__ DynParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int FPW = 32 / G;  // frames per warp
  const int fpb = (blockDim.x >> 5) * FPW;
  const int fr = (threadIdx.x >> 5) * FPW + (threadIdx.x & 31) / G;  // frame slot in the block
  const long long gf = (long long)blockIdx.x * fpb + fr;
  const long long sE = p.slotE_bytes, sN = p.slotN_bytes, sT = p.slotT_bytes, sU = p.slotU_bytes;
  // shared bytes per frame (the U part always) and HBM bytes per frame for this mode
  const long long sh = (MODE == 0 ? sE + sN + sT : MODE == 1 ? sN + sT : MODE == 2 ? sT : 0) + sU;
  const long long hb = (MODE == 0 ? 0 : MODE == 1 ? sE : MODE == 2 ? sE + sN : sE + sN + sT);
  unsigned char* shw = smem + fr * sh;
  unsigned char* hbw = p.ws + gf * hb;
  unsigned char* bE = MODE == 0 ? shw : hbw;
  unsigned char* bN = MODE == 0 ? shw + sE : MODE == 1 ? shw : hbw + sE;
  unsigned char* bT = MODE == 0 ? shw + sE + sN : MODE == 1 ? shw + sN : MODE == 2 ? shw : hbw + sE + sN;
  unsigned char* bU = shw + (sh - sU);
  unsigned char* scr = smem + (long long)fpb * sh + (long long)fr * p.scratch_bytes;
  using Key = typename Num<T>::Key;
  Ctx<T, G> c;
  c.w = Grp<G>::make();
  c.lane = c.w.lane;
  c.c2v = (T*)(bE + p.o_c2v);
  c.pre = (T*)(bE + p.o_pre);
  c.in = (T*)(bE + p.o_in);
  c.res = (T*)(bE + p.o_res);
  c.nb = (T*)(bN + p.o_total);
  c.cs = 4;
  c.tmp = (T*)(bN + p.o_tmp);
  c.inpp = (uint8_t*)(bN + p.o_inpp);
  c.members = (int*)(bN + p.o_members);
  c.sel = (int*)(bN + p.o_sel);
  c.chosen = (int*)(bN + p.o_chosen);
  c.rt.l1 = (L1Node<Key>*)(bT + p.o_rl1);
  c.rt.up = (Key*)(bU + p.o_rup);
  c.ct.l1 = (L1Node<Key>*)(bT + p.o_cl1);
  c.ct.up = (Key*)(bU + p.o_cup);
  c.items_buf = (int2*)(scr + p.so_items);
  c.items = c.items_buf;
  c.stage = (T*)(scr + p.so_stage);
  c.nk = (Key*)(scr + p.so_nk);
  c.cg = (T*)(scr + p.so_nk);
  c.opre = (T*)(scr + p.so_opre);
  c.cj = (int*)(scr + p.so_cj);
  c.ck = (Key*)(scr + p.so_ck);
  c.dl0 = (int*)(scr + p.so_dl0);
  c.dl1 = (int*)(scr + p.so_dl1);
  c.sizes = (int*)(scr + p.so_sizes);
  c.hist = (int*)(scr + p.so_hist);
  c.gid = (uint8_t*)(bN + p.o_gid);
  c.gbits = (unsigned*)(bN + p.o_gbits);
  for (;;) {
    unsigned long long f = 0;
    if (c.lane == 0) f = atomicAdd(p.next, 1ull);
    f = c.w.shfl(f, 0);
    if ((long long)f >= p.B) break;
    decode_frame<T, KERNEL, KF, G, TR, MODE, MP>(p, c, (long long)f);
  }
}

// ---------------------------------------------------------------- replay
// Debug / audit path, the GPU side of the reference's stepwise DecoderState
// (kernels.py:98-181): after _init_state (E:106-127) frame f propagates the
// GIVEN edges forced[f][0..steps) (E:130-176, pre_total and CI maintained like
// DecoderState(maintain_ci=True)), recording each update's committed C2V value
// in trace[f][k]; then writes counters[f][8] and the state
// out[f] = c2v[E], pre[E], total[N], pre_total[N], ci[N] (float64).  One warp
// per frame (block), every state part in the HBM slot of the frame.  Replaying
// the reference's own edge sequence ties GPU message values to the reference
// update by update, independent of argmax near-ties.
template <typename T, int KERNEL>
__global__ void __launch_bounds__(32) dyn_replay_kernel(const __grid_constant__ DynParams p, const int* forced,
                                                         int steps, double* trace, double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  using Key = typename Num<T>::Key;
  const long long f = blockIdx.x;
  if (f >= p.B) return;
  const long long sE = p.slotE_bytes, sN = p.slotN_bytes, sT = p.slotT_bytes;
  unsigned char* bE = p.ws + f * (sE + sN + sT);
  unsigned char* bN = bE + sE;
  unsigned char* bT = bN + sN;
  unsigned char* bU = smem;
  unsigned char* scr = smem + p.slotU_bytes;
  Ctx<T, 32> c;
  c.w = Grp<32>::make();
  c.lane = c.w.lane;
  c.c2v = (T*)(bE + p.o_c2v);
  c.pre = (T*)(bE + p.o_pre);
  c.in = (T*)(bE + p.o_in);
  c.res = (T*)(bE + p.o_res);
  c.nb = (T*)(bN + p.o_total);
  c.cs = 4;
  c.tmp = (T*)(bN + p.o_tmp);
  c.inpp = (uint8_t*)(bN + p.o_inpp);
  c.members = (int*)(bN + p.o_members);
  c.sel = (int*)(bN + p.o_sel);
  c.chosen = (int*)(bN + p.o_chosen);
  c.gid = (uint8_t*)(bN + p.o_gid);
  c.gbits = (unsigned*)(bN + p.o_gbits);
  c.rt.l1 = (L1Node<Key>*)(bT + p.o_rl1);
  c.rt.up = (Key*)(bU + p.o_rup);
  c.ct.l1 = (L1Node<Key>*)(bT + p.o_cl1);
  c.ct.up = (Key*)(bU + p.o_cup);
  c.items_buf = (int2*)(scr + p.so_items);
  c.items = c.items_buf;
  c.stage = (T*)(scr + p.so_stage);
  c.nk = (Key*)(scr + p.so_nk);
  c.cg = (T*)(scr + p.so_nk);
  c.opre = (T*)(scr + p.so_opre);
  c.cj = (int*)(scr + p.so_cj);
  c.ck = (Key*)(scr + p.so_ck);
  c.dl0 = (int*)(scr + p.so_dl0);
  c.dl1 = (int*)(scr + p.so_dl1);
  c.sizes = (int*)(scr + p.so_sizes);
  c.hist = (int*)(scr + p.so_hist);
  if (c.lane < kCounters) c.cntp()[c.lane] = 0;
  c.w.sync();
  c.prop = 0;
  c.cur_f = f;
  c.nsel = 0;
  c.rng = p.seed;
  init_state<T, KERNEL, true, 32, false>(p, c, f, KIND_LMD_CIRBP);
  for (int k = 0; k < steps; ++k) {
    const int e = forced[f * steps + k];
    if (c.lane == 0) trace[f * steps + k] = (double)c.pre[e];  // the value propagate commits (E:143)
    c.w.sync();
    propagate<T, KERNEL, true, false, false, false, 32, false, false>(p, c, e);
    ++c.prop;
  }
  c.w.sync();
  const DevGraph& g = p.g;
  double* o = out + f * (2ll * g.E + 3ll * g.N);
  for (int e = c.lane; e < g.E; e += 32) {
    o[e] = (double)c.c2v[e];
    o[g.E + e] = (double)c.pre[e];
  }
  for (int n = c.lane; n < g.N; n += 32) {
    o[2 * g.E + n] = (double)c.total(n);
    o[2 * g.E + g.N + n] = (double)c.pretot(n);
    o[2 * g.E + 2 * g.N + n] = (double)c.ci(n);
  }
  c.store_counters(p.counters + f * kCounters, true);
}

}  // namespace ldpc
