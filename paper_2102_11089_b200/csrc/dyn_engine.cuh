// dyn_engine.cuh -- informed-dynamic-schedule decoders, one warp per frame.
//
// Replaces the reference's numba schedule loops
// (/root/reference/pkg/src/ldpc_ids/_engine.py, "E:<line>"):
//   RBP E:355-385, CIRBP E:388-433, LMDRBP/sLMDRBP E:436-510,
//   LMD-CIRBP E:513-598, ME-CIRBP E:601-643, ME-LMD-CIRBP E:646-716,
//   plus ME-RBP (new; defined in oracle/ldpc_oracle.c).
//
// Design (B200):
//  * a persistent grid; each warp pulls frame ids from an atomic work queue,
//    so a frame that converges early frees its warp for the next frame;
//  * a frame's whole message state lives in one "slot": in shared memory when
//    it fits (small codes), else in a per-warp HBM slot that stays hot in L2;
//  * the update (_propagate, E:130-176) is latency-bound and serial per
//    frame, so the kernel minimises its dependent-load chain: packed graph
//    records (edge -> (check, vn); VN slot -> (f, check, check range)) and
//    per-edge precomputed two-hop facts (size, distinct VNs, duplicates);
//  * lanes compute the V2C messages of M(n*)\m*, then the two-hop pre-C2V
//    refresh packs all (d_v-1)(d_c-1) edges across the 32 lanes; pre_total
//    accumulations that hit the same VN (4-cycles through n*) are applied in
//    the reference's order (match_any ranks), so float64 results are
//    bit-identical;
//  * global argmax uses 32-ary max trees of order-preserving integer keys; the
//    argmax descends with one coalesced load + REDUX.MAX per level (lowest
//    index wins ties, like the reference's left-preferring segment tree,
//    E:220-257); after an update only the touched 32-leaf groups and their
//    ancestors are recomputed, one node per lane, level-synchronously.
#pragma once
#include "ldpc_common.cuh"

namespace ldpc {

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
  // per-frame state slots
  unsigned char* ws;
  long long slot_bytes;
  long long o_c2v, o_pre, o_in, o_res, o_total, o_pretot, o_ci, o_rtree, o_ctree, o_mark,
      o_inpp, o_members, o_sel, o_chosen, o_tmp;
  TreeGeom rgeo, cgeo;
  int scratch_bytes;  // per-warp shared scratch
  int so_items, so_itemab, so_dl0, so_dl1, so_sizes;
};

template <typename T>
struct Ctx {
  using Key = typename Num<T>::Key;
  T *c2v, *pre, *in, *res, *total, *pretot, *ci, *tmp;
  Key *rtree, *ctree;
  uint8_t* inpp;  // ME-LMD-CIRBP P' membership (E:665)
  int *members, *sel, *chosen;
  int* items;     // two-hop edge ids of the last update, ascending
  int2* itemab;   // check range [a, b) of each item
  int *dl0, *dl1; // dirty-node lists for tree maintenance
  int* sizes;     // Alg.4 group histogram
  long long cnt[kCounters];
  long long prop;
  long long next_b;  // next single-edge iteration boundary (k * E)
  int it;            // completed iterations (= prop / E, maintained incrementally)
  int lane;
  long long rng;
};

// ------------------------------------------------------------- max trees

template <typename T>
__device__ __forceinline__ typename Num<T>::Key child_key(const typename Num<T>::Key* tree,
                                                          const T* leaves, const TreeGeom& geo,
                                                          int level, int child) {
  if (child >= geo.size[level]) return 0;
  if (level == 0) return Num<T>::key(leaves[child]);
  return tree[geo.off[level] + child];
}

// max over the 32 children of node q at level l (children at l-1), staggered by lane
template <typename T>
__device__ __forceinline__ typename Num<T>::Key node_max(const typename Num<T>::Key* tree,
                                                         const T* leaves, const TreeGeom& geo,
                                                         int l, int q, int lane) {
  using Key = typename Num<T>::Key;
  Key m = 0;
  const int base = q * 32, lim = geo.size[l - 1] - base;
  if (l == 1) {
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      int ch = (c + lane) & 31;
      Key k = ch < lim ? Num<T>::key(leaves[base + ch]) : Key(0);
      m = k > m ? k : m;
    }
  } else {
    const Key* row = tree + geo.off[l - 1] + base;
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      int ch = (c + lane) & 31;
      Key k = ch < lim ? row[ch] : Key(0);
      m = k > m ? k : m;
    }
  }
  return m;
}

template <typename T>
__device__ void tree_build(typename Num<T>::Key* tree, const T* leaves, const TreeGeom& geo, int lane) {
  for (int l = 1; l <= geo.levels; ++l) {
    for (int q = lane; q < geo.size[l]; q += 32) tree[geo.off[l] + q] = node_max<T>(tree, leaves, geo, l, q, lane);
    __syncwarp();
  }
}

// Recompute the level-1 nodes in dl[0..n) and all their ancestors.
// Duplicates in dl are harmless (same value written twice).
template <typename T>
__device__ void tree_update_list(typename Num<T>::Key* tree, const T* leaves, const TreeGeom& geo,
                                 int* dl, int* dl2, int n, int lane) {
  for (int l = 1; l <= geo.levels; ++l) {
    for (int base = 0; base < n; base += 32) {
      int idx = base + lane;
      if (idx < n) {
        int q = dl[idx];
        tree[geo.off[l] + q] = node_max<T>(tree, leaves, geo, l, q, lane);
      }
    }
    __syncwarp();
    if (l == geo.levels) break;
    int cnt = 0;
    for (int base = 0; base < n; base += 32) {
      int idx = base + lane;
      int v = idx < n ? (dl[idx] >> 5) : -1;
      int pv = (idx > 0 && idx < n) ? (dl[idx - 1] >> 5) : -2;
      bool keep = idx < n && v != pv;
      unsigned bal = __ballot_sync(kFull, keep);
      if (keep) dl2[cnt + __popc(bal & lanemask_lt())] = v;
      cnt += __popc(bal);
    }
    __syncwarp();
    int* t = dl;
    dl = dl2;
    dl2 = t;
    n = cnt;
  }
}

template <typename T>
__device__ int tree_argmax(const typename Num<T>::Key* tree, const T* leaves, const TreeGeom& geo,
                           int lane) {
  using Key = typename Num<T>::Key;
  const int L = geo.levels, s = geo.size[L];
  const Key* top = tree + geo.off[L];
  Key k0 = lane < s ? top[lane] : Key(0);
  Key k1 = lane + 32 < s ? top[lane + 32] : Key(0);
  int q;
  warp_max_key_minidx(k1 > k0 ? k1 : k0, k1 > k0 ? lane + 32 : lane, &q);
  for (int l = L - 1; l >= 0; --l) {
    Key k = child_key<T>(tree, leaves, geo, l, q * 32 + lane);
    int ln;
    warp_max_key(k, &ln);
    q = q * 32 + ln;
  }
  return q;
}

// ------------------------------------------------------------ argmax scans

// E:260-266 -- first maximum over values[0..n)
template <typename T>
__device__ int argmax_all(const T* v, int n, int lane) {
  using Key = typename Num<T>::Key;
  Key best = 0;
  int bi = 0x7fffffff;
  for (int i = lane; i < n; i += 32) {
    Key k = Num<T>::key(v[i]);
    if (k > best) { best = k; bi = i; }
  }
  int idx;
  warp_max_key_minidx(best, bi, &idx);
  return idx;
}

// E:269-276 -- first maximum residual over M(n) in vn_edges order (= edge order)
template <typename T>
__device__ __forceinline__ int argmax_vn_edges(const DevGraph& g, const T* res, int n, int lane) {
  using Key = typename Num<T>::Key;
  int2 vr = g.vrec[n];
  int e = lane < vr.y ? g.vn_edges[vr.x + lane] : 0x7fffffff;
  Key k = lane < vr.y ? Num<T>::key(res[e]) : Key(0);
  int idx;
  warp_max_key_minidx(k, e, &idx);
  return idx;
}

// ------------------------------------------------------- two-hop item table

// Items = {g in N(i)\{f} : f in M(n*), i = cn(f) != m*}, in ascending edge id
// (= the reference's scan order, E:153-166 / E:450-460).  `adj` is this lane's
// vadj record (lane < d_v) and `act` says whether its check is != m*.
template <typename T>
__device__ __forceinline__ int build_items_from(Ctx<T>& c, int4 adj, bool act) {
  int cnt = act ? adj.w - adj.z - 1 : 0;
  int incl = warp_incl_scan(cnt);
  int total = __shfl_sync(kFull, incl, 31);
  if (act) {
    int t = incl - cnt;
    const int2 ab = make_int2(adj.z, adj.w);
    for (int e = adj.z; e < adj.w; ++e)
      if (e != adj.x) {
        c.items[t] = e;
        c.itemab[t] = ab;
        ++t;
      }
  }
  __syncwarp();
  return total;
}

template <typename T>
__device__ int build_items(const DevGraph& g, Ctx<T>& c, int e_star) {
  int2 mn = g.ecv[e_star];
  int2 vr = g.vrec[mn.y];
  int4 adj = make_int4(-1, -1, 0, 0);
  if (c.lane < vr.y) adj = g.vadj[vr.x + c.lane];
  return build_items_from<T>(c, adj, c.lane < vr.y && adj.y != mn.x);
}

// ------------------------------------------------------------- propagate

// E:130-176.  Commit pre_c2v[e*], emit V2C to M(n*)\m*, refresh the two-hop
// pre-C2V / residual / pre_total (/ CI) state.  Leaves the item table of e*.
template <typename T, int KERNEL, bool CI, bool RT, bool CT>
__device__ int propagate(const DynParams& p, Ctx<T>& c, int e_star) {
  const DevGraph& g = p.g;
  const int lane = c.lane;
  const int2 mn = g.ecv[e_star];
  const int m_star = mn.x, n_star = mn.y;
  const int2 vr = g.vrec[n_star];
  int4 adj = make_int4(-1, -1, 0, 0);
  if (lane < vr.y) adj = g.vadj[vr.x + lane];
  const bool act = lane < vr.y && adj.y != m_star;
  const T old = c.c2v[e_star];
  const T nv = c.pre[e_star];
  const T tot = c.total[n_star] + (nv - old);  // E:147
  T cf = act ? c.c2v[adj.x] : T(0);
  const bool dup = g.hop_dup[e_star] != 0;
  __syncwarp();
  if (lane == 0) {
    c.c2v[e_star] = nv;
    c.res[e_star] = T(0);
    c.total[n_star] = tot;
    if (CI) c.ci[n_star] = ci_of(tot, c.pretot[n_star]);  // E:148-149
  }
  if (act) {  // V2C to the other checks of n* (E:153-160)
    T v = clampv(tot - cf);
    c.in[adj.x] = (KERNEL == KERNEL_EXACT) ? Num<T>::tanh_(T(0.5) * v) : v;
  }
  const int n_items = build_items_from<T>(c, adj, act);  // ends with __syncwarp
  // two-hop refresh (E:161-176), 32 edges per pass in reference order
  for (int base = 0; base < n_items; base += 32) {
    const int t = base + lane;
    const bool valid = t < n_items;
    int ge = -1, j = -1;
    T delta = T(0);
    if (valid) {
      ge = c.items[t];
      const int2 ab = c.itemab[t];
      j = g.edge_vn[ge];
      T np_ = cn_msg_cached<T, KERNEL>(c.in, ab.x, ab.y, ge);
      T op = c.pre[ge];
      c.pre[ge] = np_;
      c.res[ge] = Num<T>::abs_(np_ - c.c2v[ge]);
      delta = np_ - op;
    }
    if (!dup) {
      if (valid) {
        T pt = c.pretot[j] + delta;  // E:171
        c.pretot[j] = pt;
        if (CI) c.ci[j] = ci_of(c.total[j], pt);  // E:173
      }
    } else {
      // same VN reached through two checks (4-cycle): keep the reference's order
      unsigned peers = __match_any_sync(kFull, j);
      int rank = __popc(peers & lanemask_lt());
      int maxrank = __reduce_max_sync(kFull, valid ? (unsigned)rank : 0u);
      for (int r = 0; r <= maxrank; ++r) {
        if (valid && rank == r) c.pretot[j] += delta;
        __syncwarp();
      }
      bool last = valid && ((peers >> lane) >> 1) == 0;
      if (CI && last) c.ci[j] = ci_of(c.total[j], c.pretot[j]);
    }
    __syncwarp();
  }
  if (RT) {  // dirty res-tree groups: items (ascending) + e*
    int cnt = 0, prev = -1;
    for (int base = 0; base < n_items; base += 32) {
      int t = base + lane;
      int gq = t < n_items ? (c.items[t] >> 5) : 0x7fffffff;
      int up = __shfl_up_sync(kFull, gq, 1);
      if (lane == 0) up = prev;
      bool keep = t < n_items && gq != up;
      unsigned bal = __ballot_sync(kFull, keep);
      if (keep) c.dl0[cnt + __popc(bal & lanemask_lt())] = gq;
      cnt += __popc(bal);
      prev = __shfl_sync(kFull, gq, 31);
    }
    if (lane == 0) c.dl0[cnt] = e_star >> 5;
    __syncwarp();
    tree_update_list<T>(c.rtree, c.res, p.rgeo, c.dl0, c.dl1, cnt + 1, lane);
  }
  if (CT) {  // dirty ci-tree groups: two-hop VNs + n*
    for (int t = lane; t < n_items; t += 32) c.dl0[t] = g.edge_vn[c.items[t]] >> 5;
    if (lane == 0) c.dl0[n_items] = n_star >> 5;
    __syncwarp();
    tree_update_list<T>(c.ctree, c.ci, p.cgeo, c.dl0, c.dl1, n_items + 1, lane);
  }
  c.cnt[C_PROP] += 1;
  c.cnt[C_V2C] += vr.y - 1;
  c.cnt[C_PRE] += n_items;
  if (CI) c.cnt[C_CI] += n_items;
  return n_items;
}

// ------------------------------------------------------------ boundaries

template <typename T>
__device__ bool syndrome_ok(const DevGraph& g, const T* total, int lane) {  // E:179-188
  for (int base = 0; base < g.M; base += 32) {
    int m = base + lane;
    int par = 0;
    if (m < g.M)
      for (int e = g.cn_ptr[m]; e < g.cn_ptr[m + 1]; ++e) par ^= (total[g.edge_vn[e]] < T(0)) ? 1 : 0;
    if (__any_sync(kFull, par)) return false;
  }
  return true;
}

template <typename T>
__device__ void record_boundary(const DynParams& p, const T* total, long long f, int k, int lane) {
  int errs = 0, ei = 0;
  for (int n = lane; n < p.g.N; n += 32)
    if (total[n] < T(0)) {
      ++errs;
      if (n < p.k_info) ++ei;
    }
  errs = warp_sum(errs);
  ei = warp_sum(ei);
  if (lane == 0) {
    p.biterr[f * (p.i_max + 1) + k] = errs;
    p.biterr_info[f * (p.i_max + 1) + k] = ei;
  }
}

__device__ __forceinline__ void fill_remaining(const DynParams& p, long long f, int k, int lane) {
  if (lane == 0)
    for (int kk = k + 1; kk <= p.i_max; ++kk) {
      p.biterr[f * (p.i_max + 1) + kk] = p.biterr[f * (p.i_max + 1) + k];
      p.biterr_info[f * (p.i_max + 1) + kk] = p.biterr_info[f * (p.i_max + 1) + k];
    }
  __syncwarp();
}

// single-edge boundary rule (E:377-384): returns true when decoding stops
template <typename T>
__device__ __forceinline__ bool single_boundary(const DynParams& p, Ctx<T>& c, long long f, bool* conv) {
  if (c.prop != c.next_b) return false;
  c.next_b += p.g.E;
  int k = ++c.it;
  record_boundary<T>(p, c.total, f, k, c.lane);
  if (syndrome_ok<T>(p.g, c.total, c.lane)) {
    *conv = true;
    fill_remaining(p, f, k, c.lane);
    return true;
  }
  return false;
}

// multi-edge boundary rule (E:633-642)
template <typename T>
__device__ void me_boundaries(const DynParams& p, Ctx<T>& c, long long f, int* boundary, bool* conv) {
  long long E = p.g.E;
  while (*boundary <= p.i_max && c.prop >= (long long)(*boundary) * E) {
    record_boundary<T>(p, c.total, f, *boundary, c.lane);
    if (syndrome_ok<T>(p.g, c.total, c.lane)) {
      *conv = true;
      fill_remaining(p, f, *boundary, c.lane);
    }
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

template <typename T>
__device__ __forceinline__ int ci_group(T v, int n_g) {
  int gi = (int)(v * (T)n_g);
  return gi > n_g - 1 ? n_g - 1 : gi;
}

// Select up to n_p VNs (excluding n with excl[n] != 0 when excl != nullptr)
// into out[0..count), ascending.  Reproduces _select_vns exactly.
template <typename T>
__device__ int select_vns(const DynParams& p, Ctx<T>& c, const uint8_t* excl, int n_p, int* out) {
  const int N = p.g.N, n_g = p.n_g, lane = c.lane;
  for (int q = lane; q < n_g; q += 32) c.sizes[q] = 0;
  __syncwarp();
  for (int n = lane; n < N; n += 32)
    if (!excl || !excl[n]) atomicAdd(&c.sizes[ci_group(c.ci[n], n_g)], 1);
  __syncwarp();
  int k_star = 0;
  if (lane == 0) {
    long long cum = 0;
    for (int k = 1; k <= n_g; ++k) {
      cum += c.sizes[n_g - k];
      if (cum <= n_p) k_star = k;
      else break;
    }
  }
  k_star = __shfl_sync(kFull, k_star, 0);
  const int thr = n_g - k_star;
  int count = 0;
  for (int base = 0; base < N; base += 32) {
    int n = base + lane;
    bool s = n < N && (!excl || !excl[n]) && ci_group(c.ci[n], n_g) >= thr;
    unsigned bal = __ballot_sync(kFull, s);
    if (s) out[count + __popc(bal & lanemask_lt())] = n;
    count += __popc(bal);
  }
  __syncwarp();
  if (count < n_p && k_star < n_g) {
    const int fill = n_g - k_star - 1;
    int idx = 0;
    for (int base = 0; base < N; base += 32) {
      int n = base + lane;
      bool s = n < N && (!excl || !excl[n]) && ci_group(c.ci[n], n_g) == fill;
      unsigned bal = __ballot_sync(kFull, s);
      if (s) c.members[idx + __popc(bal & lanemask_lt())] = n;
      idx += __popc(bal);
    }
    __syncwarp();
    int need = n_p - count;
    if (need > idx) need = idx;
    if (lane == 0) {
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
    c.rng = __shfl_sync(kFull, c.rng, 0);
    count += need;
  }
  __syncwarp();
  // ascending sort of out[0..count) (distinct VN ids): rank sort through members[]
  for (int i = lane; i < count; i += 32) {
    int v = out[i], r = 0;
    for (int q = 0; q < count; ++q) r += out[q] < v;
    c.members[r] = v;
  }
  __syncwarp();
  for (int i = lane; i < count; i += 32) out[i] = c.members[i];
  __syncwarp();
  return count;
}

// sort ints ascending in place (distinct values), via members[] scratch
template <typename T>
__device__ void sort_small(Ctx<T>& c, int* a, int count) {
  for (int i = c.lane; i < count; i += 32) {
    int v = a[i], r = 0;
    for (int q = 0; q < count; ++q) r += a[q] < v;
    c.members[r] = v;
  }
  __syncwarp();
  for (int i = c.lane; i < count; i += 32) a[i] = c.members[i];
  __syncwarp();
}

// --------------------------------------------------------- local searches

// E:436-469 after propagate(e_prev) left the item table of e_prev.
template <typename T>
__device__ int lmd_next_edge(const DynParams& p, Ctx<T>& c, int e_prev, int n_items, bool simplified) {
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
    for (int e = a + lane; e < b; e += 32)
      if (e != e_prev) {
        Key k = Num<T>::key(c.res[e]);
        if (k > bk) { bk = k; bi = e; }
      }
  } else {
    ncand = n_items;
    for (int t = lane; t < n_items; t += 32) {
      int e = c.items[t];
      Key k = Num<T>::key(c.res[e]);
      if (k > bk) { bk = k; bi = e; }
    }
  }
  if (ncand > 1) c.cnt[C_CMP] += ncand - 1;
  if (ncand <= 0) return -1;
  int best;
  warp_max_key_minidx(bk, bi, &best);
  if (!simplified) {
    int np_ = g.edge_vn[best];
    best = argmax_vn_edges<T>(g, c.res, np_, lane);
    c.cnt[C_CMP] += g.vrec[np_].y - 1;
  }
  return best;
}

// E:513-552: max-CI VN of the two-hop set of e_prev, ties -> lowest VN; the
// candidate count (deduplicated, E:536-549) is precomputed per edge.
template <typename T>
__device__ int ci_argmax_twohop(const DynParams& p, Ctx<T>& c, int e_prev, int n_items, bool have_items) {
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
    for (int e = a + lane; e < b; e += 32)
      if (e != e_prev) {
        int j = g.edge_vn[e];
        Key k = Num<T>::key(c.ci[j]);
        if (k > bk || (k == bk && j < bj)) { bk = k; bj = j; }
      }
  } else {
    if (!have_items) n_items = build_items<T>(g, c, e_prev);
    ncand = g.hop_distinct[e_prev];
    for (int t = lane; t < n_items; t += 32) {
      int j = g.edge_vn[c.items[t]];
      Key k = Num<T>::key(c.ci[j]);
      if (k > bk || (k == bk && j < bj)) { bk = k; bj = j; }
    }
  }
  if (ncand > 1) c.cnt[C_CMP] += ncand - 1;
  if (ncand <= 0) return -1;
  int best;
  warp_max_key_minidx(bk, bj, &best);
  return best;
}

// --------------------------------------------------------------- decoders

template <typename T, int KERNEL>
__device__ void init_state(const DynParams& p, Ctx<T>& c, long long f) {  // E:106-127
  const DevGraph& g = p.g;
  const int lane = c.lane;
  const float* l32 = (const float*)p.llr + f * g.N;
  const double* l64 = (const double*)p.llr + f * g.N;
  auto chl = [&](int n) -> T { return p.llr_f64 ? (T)l64[n] : (T)l32[n]; };
  for (int e = lane; e < g.E; e += 32) {
    T v = clampv(chl(g.edge_vn[e]));
    c.c2v[e] = T(0);
    c.in[e] = (KERNEL == KERNEL_EXACT) ? Num<T>::tanh_(T(0.5) * v) : v;
  }
  for (int n = lane; n < g.N; n += 32) c.total[n] = chl(n);
  __syncwarp();
  for (int m = lane; m < g.M; m += 32) {
    int a = g.cn_ptr[m], b = g.cn_ptr[m + 1];
    for (int e = a; e < b; ++e) {
      T v = cn_msg_cached<T, KERNEL>(c.in, a, b, e);
      c.pre[e] = v;
      c.res[e] = Num<T>::abs_(v - T(0));
    }
  }
  __syncwarp();
  for (int n = lane; n < g.N; n += 32) {
    T acc = chl(n);
    for (int k = g.vn_ptr[n]; k < g.vn_ptr[n + 1]; ++k) acc += c.pre[g.vn_edges[k]];
    c.pretot[n] = acc;
    c.ci[n] = ci_of(c.total[n], acc);
    c.inpp[n] = 0;
  }
  __syncwarp();
}

template <typename T, int KERNEL>
__device__ void decode_frame(const DynParams& p, Ctx<T>& c, long long f) {
  const DevGraph& g = p.g;
  const long long E = g.E, budget = (long long)p.i_max * E;
  const int lane = c.lane, I = p.i_max;
  for (int k = 0; k < kCounters; ++k) c.cnt[k] = 0;
  c.prop = 0;
  c.next_b = E;
  c.it = 0;
  c.rng = p.seed;
  bool conv = false;
  if (lane == 0) {
    for (int k = 0; k <= I; ++k) p.biterr[f * (I + 1) + k] = p.biterr_info[f * (I + 1) + k] = 0;
    if (p.kind == KIND_CIRBP)
      for (int k = 0; k < I; ++k) p.kh[f * I + k] = p.kt[f * I + k] = 0;
  }
  init_state<T, KERNEL>(p, c, f);
  record_boundary<T>(p, c.total, f, 0, lane);

  switch (p.kind) {
    case KIND_RBP: {  // E:355-385
      tree_build<T>(c.rtree, c.res, p.rgeo, lane);
      while (c.prop < budget) {
        int e = tree_argmax<T>(c.rtree, c.res, p.rgeo, lane);
        c.cnt[C_CMP] += E - 1;
        propagate<T, KERNEL, false, true, false>(p, c, e);
        ++c.prop;
        if (single_boundary<T>(p, c, f, &conv)) break;
      }
    } break;
    case KIND_CIRBP: {  // E:388-433
      tree_build<T>(c.rtree, c.res, p.rgeo, lane);
      tree_build<T>(c.ctree, c.ci, p.cgeo, lane);
      const T gamma = (T)p.gamma;
      int kh = 0, kt = 0;  // per-iteration kappa tallies (lane-uniform)
      while (c.prop < budget) {
        const int it = c.it;
        int n_star = tree_argmax<T>(c.ctree, c.ci, p.cgeo, lane);
        c.cnt[C_CMP] += g.N - 1 + 1;
        c.cnt[C_KTRIALS] += 1;
        ++kt;
        bool hit = c.ci[n_star] < gamma;
        int e;
        if (hit) {
          c.cnt[C_KHITS] += 1;
          ++kh;
          e = tree_argmax<T>(c.rtree, c.res, p.rgeo, lane);
          c.cnt[C_CMP] += E - 1;
        } else {
          e = argmax_vn_edges<T>(g, c.res, n_star, lane);
          c.cnt[C_CMP] += g.vrec[n_star].y - 1;
        }
        propagate<T, KERNEL, true, true, true>(p, c, e);
        ++c.prop;
        const bool at_b = c.prop == c.next_b;
        if (at_b || c.prop >= budget) {
          if (lane == 0) {
            p.kh[f * I + it] = kh;
            p.kt[f * I + it] = kt;
          }
          kh = kt = 0;
        }
        if (single_boundary<T>(p, c, f, &conv)) break;
      }
    } break;
    case KIND_LMDRBP:
    case KIND_SLMDRBP: {  // E:472-510
      const bool simplified = p.kind == KIND_SLMDRBP;
      int e = argmax_all<T>(c.res, g.E, lane);
      c.cnt[C_CMP] += E - 1;
      while (c.prop < budget) {
        int n_items = propagate<T, KERNEL, false, false, false>(p, c, e);
        ++c.prop;
        if (single_boundary<T>(p, c, f, &conv)) break;
        if (c.prop >= budget) break;
        int en = lmd_next_edge<T>(p, c, e, n_items, simplified);
        if (en < 0) {
          en = argmax_all<T>(c.res, g.E, lane);
          c.cnt[C_CMP] += E - 1;
        }
        e = en;
      }
    } break;
    case KIND_LMD_CIRBP: {  // E:555-598
      int n_star = argmax_all<T>(c.ci, g.N, lane);
      c.cnt[C_CMP] += g.N - 1;
      int e = argmax_vn_edges<T>(g, c.res, n_star, lane);
      c.cnt[C_CMP] += g.vrec[n_star].y - 1;
      while (c.prop < budget) {
        int n_items = propagate<T, KERNEL, true, false, false>(p, c, e);
        ++c.prop;
        if (single_boundary<T>(p, c, f, &conv)) break;
        if (c.prop >= budget) break;
        int nn = ci_argmax_twohop<T>(p, c, e, n_items, true);
        if (nn < 0) {
          nn = argmax_all<T>(c.ci, g.N, lane);
          c.cnt[C_CMP] += g.N - 1;
        }
        e = argmax_vn_edges<T>(g, c.res, nn, lane);
        c.cnt[C_CMP] += g.vrec[nn].y - 1;
      }
    } break;
    case KIND_ME_CIRBP: {  // E:601-643
      int boundary = 1;
      while (boundary <= I && !conv) {
        int count = select_vns<T>(p, c, nullptr, p.n_p, c.sel);
        c.cnt[C_MSEL] += p.n_g;
        for (int idx = 0; idx < count; ++idx) {
          int pv = c.sel[idx];
          int e = argmax_vn_edges<T>(g, c.res, pv, lane);
          c.cnt[C_CMP] += g.vrec[pv].y - 1;
          propagate<T, KERNEL, true, false, false>(p, c, e);
          ++c.prop;
        }
        me_boundaries<T>(p, c, f, &boundary, &conv);
      }
    } break;
    case KIND_ME_LMD_CIRBP: {  // E:646-716
      int boundary = 1;
      int count = select_vns<T>(p, c, nullptr, p.n_p, c.sel);
      c.cnt[C_MSEL] += p.n_g;
      while (boundary <= I && !conv) {
        for (int idx = 0; idx < count; ++idx) {
          int pv = c.sel[idx];
          int e = argmax_vn_edges<T>(g, c.res, pv, lane);
          c.cnt[C_CMP] += g.vrec[pv].y - 1;
          if (lane == 0) c.chosen[idx] = e;
          propagate<T, KERNEL, true, false, false>(p, c, e);
          ++c.prop;
        }
        me_boundaries<T>(p, c, f, &boundary, &conv);
        if (conv || boundary > I) break;
        // P' = two-hop max-CI VN of each chosen edge, deduplicated in order
        int npc = 0;
        for (int idx = 0; idx < count; ++idx) {
          int pn = ci_argmax_twohop<T>(p, c, c.chosen[idx], 0, false);
          bool add = pn >= 0 && !c.inpp[pn];
          __syncwarp();
          if (add) {
            if (lane == 0) {
              c.inpp[pn] = 1;
              c.sel[npc] = pn;
            }
            ++npc;
          }
          __syncwarp();
        }
        if (npc < p.n_p) {
          int extra = select_vns<T>(p, c, c.inpp, p.n_p - npc, c.sel + npc);
          c.cnt[C_MSEL] += p.n_g;
          count = npc + extra;
        } else {
          count = npc;
        }
        for (int idx = lane; idx < npc; idx += 32) c.inpp[c.sel[idx]] = 0;
        __syncwarp();
        sort_small<T>(c, c.sel, count);
      }
    } break;
    case KIND_ME_RBP: {  // new (oracle/ldpc_oracle.c decode_me_rbp)
      tree_build<T>(c.rtree, c.res, p.rgeo, lane);
      int boundary = 1;
      const int np_ = p.n_p < g.E ? p.n_p : g.E;
      while (boundary <= I && !conv) {
        for (int t = 0; t < np_; ++t) {
          int e = tree_argmax<T>(c.rtree, c.res, p.rgeo, lane);
          if (lane == 0) {
            c.sel[t] = e;
            c.tmp[t] = c.res[e];
            c.res[e] = T(-1);  // excluded: key 0
            c.dl0[0] = e >> 5;
          }
          __syncwarp();
          tree_update_list<T>(c.rtree, c.res, p.rgeo, c.dl0, c.dl1, 1, lane);
        }
        for (int t = lane; t < np_; t += 32) {
          c.res[c.sel[t]] = c.tmp[t];
          c.dl0[t] = c.sel[t] >> 5;
        }
        __syncwarp();
        tree_update_list<T>(c.rtree, c.res, p.rgeo, c.dl0, c.dl1, np_, lane);
        c.cnt[C_CMP] += E - 1;
        sort_small<T>(c, c.sel, np_);
        for (int idx = 0; idx < np_; ++idx) {
          propagate<T, KERNEL, false, true, false>(p, c, c.sel[idx]);
          ++c.prop;
        }
        me_boundaries<T>(p, c, f, &boundary, &conv);
      }
    } break;
    default:
      break;
  }
  if (I == 0) conv = syndrome_ok<T>(g, c.total, lane);  // schedules.py:144-146
  for (int n = lane; n < g.N; n += 32) p.u_hat[f * g.N + n] = c.total[n] < T(0) ? 1 : 0;
  if (lane < kCounters) {
    long long v = 0;
#pragma unroll
    for (int k = 0; k < kCounters; ++k)
      if (k == lane) v = c.cnt[k];
    p.counters[f * kCounters + lane] = v;
  }
  if (lane == 0) {
    p.prop[f] = c.prop;
    p.conv[f] = conv ? 1 : 0;
  }
  __syncwarp();
}

template <typename T, int KERNEL, bool SMEM>
__global__ void __launch_bounds__(256) dyn_decode_kernel(const __grid_constant__ DynParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  unsigned char* slot = SMEM ? smem + (long long)warp * p.slot_bytes
                             : p.ws + ((long long)blockIdx.x * wpb + warp) * p.slot_bytes;
  unsigned char* scr = smem + (SMEM ? (long long)wpb * p.slot_bytes : 0) + (long long)warp * p.scratch_bytes;
  using Key = typename Num<T>::Key;
  Ctx<T> c;
  c.lane = threadIdx.x & 31;
  c.c2v = (T*)(slot + p.o_c2v);
  c.pre = (T*)(slot + p.o_pre);
  c.in = (T*)(slot + p.o_in);
  c.res = (T*)(slot + p.o_res);
  c.total = (T*)(slot + p.o_total);
  c.pretot = (T*)(slot + p.o_pretot);
  c.ci = (T*)(slot + p.o_ci);
  c.tmp = (T*)(slot + p.o_tmp);
  c.rtree = (Key*)(slot + p.o_rtree);
  c.ctree = (Key*)(slot + p.o_ctree);
  c.inpp = (uint8_t*)(slot + p.o_inpp);
  c.members = (int*)(slot + p.o_members);
  c.sel = (int*)(slot + p.o_sel);
  c.chosen = (int*)(slot + p.o_chosen);
  c.items = (int*)(scr + p.so_items);
  c.itemab = (int2*)(scr + p.so_itemab);
  c.dl0 = (int*)(scr + p.so_dl0);
  c.dl1 = (int*)(scr + p.so_dl1);
  c.sizes = (int*)(scr + p.so_sizes);
  for (;;) {
    unsigned long long f = 0;
    if (c.lane == 0) f = atomicAdd(p.next, 1ull);
    f = __shfl_sync(kFull, f, 0);
    if ((long long)f >= p.B) break;
    decode_frame<T, KERNEL>(p, c, (long long)f);
  }
}

}  // namespace ldpc
