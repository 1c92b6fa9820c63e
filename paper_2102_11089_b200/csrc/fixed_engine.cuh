// fixed_engine.cuh -- flooding and row-layered BP, frame-interleaved.
//
// Flooding replaces _decode_flooding (E:719-765): per iteration all C2V from
// the previous V2C, then totals and V2C per VN, syndrome at every iteration.
// Layered is the schedule the reference lacks (defined in
// oracle/ldpc_oracle.c): checks m = 0..M-1 in order, each committing
// total += c2v' - c2v.  Checks are grouped into dependency levels on the host
// (a check's level exceeds that of every earlier check sharing a VN), so a
// level runs in parallel and still reproduces the sequential order exactly.
//
// Layout: a CTA owns a group of F frames; its state arrays are interleaved
// [item][F] so consecutive lanes are consecutive frames and every message
// access is a coalesced 32 x 8 B row.  Only c2v[E] and total[N] are kept: the
// V2C of an edge is clamp(total - c2v) (bit-identical to the reference's
// stored v2c, E:752-754), so per edge update the traffic is c2v read+write,
// one total gather and the VN-phase re-read -- the 16 + 8N/E B roofline figure
// (in float32 units; double for float64).
#pragma once
#include "ldpc_common.cuh"

namespace ldpc {

constexpr int kFixedMaxDc = 32;

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
  unsigned char* ws;      // per-CTA slot: chl[N][F], total[N][F], c2v[E][F]
  long long slot_bytes;
  int F;                  // frames per CTA (power of two, <= 32)
  int log2F;
};

// C2V of one check for one frame: inputs from total/c2v, outputs written back.
// LAYERED additionally commits total += new - old per edge.
template <typename T, int KERNEL, bool LAYERED>
__device__ __forceinline__ void check_update(const DevGraph& g, int m, int F, int fl, T* c2v, T* total) {
  const int a = g.cn_ptr[m], d = g.cn_ptr[m + 1] - a;
  T in[kFixedMaxDc];
#pragma unroll 4
  for (int q = 0; q < d; ++q) {
    int e = a + q;
    T v = clampv(total[(long long)g.edge_vn[e] * F + fl] - c2v[(long long)e * F + fl]);
    in[q] = (KERNEL == KERNEL_EXACT) ? Num<T>::tanh_(T(0.5) * v) : v;  // E:58 / E:73
  }
  for (int q = 0; q < d; ++q) {
    T out;
    if (KERNEL == KERNEL_EXACT) {
      T prod = T(1);
      for (int r = 0; r < d; ++r)
        if (r != q) prod *= in[r];
      out = atanh_msg(prod, d - 1);
    } else {
      T sign = T(1), mag = Num<T>::kBig;
      for (int r = 0; r < d; ++r) {
        if (r == q) continue;
        T v = in[r];
        if (v < T(0)) { sign = -sign; v = -v; }
        if (v < mag) mag = v;
      }
      out = d > 1 ? clampv(sign * mag) : T(0);
    }
    long long ix = (long long)(a + q) * F + fl;
    if (LAYERED) {
      long long tx = (long long)g.edge_vn[a + q] * F + fl;
      total[tx] += out - c2v[ix];
    }
    c2v[ix] = out;
  }
}

template <typename T, int KERNEL>
__global__ void __launch_bounds__(512) fixed_decode_kernel(const __grid_constant__ FixedParams p) {
  const DevGraph& g = p.g;
  const int F = p.F, lf = p.log2F, tid = threadIdx.x, nt = blockDim.x;
  const int fl = tid & (F - 1), slot_item0 = tid >> lf, items_per_pass = nt >> lf;
  const int I = p.i_max;
  const bool layered = p.kind == KIND_LAYERED;
  T* chl = (T*)(p.ws + (long long)blockIdx.x * p.slot_bytes);
  T* total = chl + (long long)g.N * F;
  T* c2v = total + (long long)g.N * F;
  __shared__ int s_active[32], s_unsat[32], s_errs[32], s_errs_info[32], s_iter[32];
  __shared__ unsigned long long s_grp;
  for (;;) {
    if (tid == 0) s_grp = atomicAdd(p.next, 1ull);
    __syncthreads();
    const long long f0 = (long long)s_grp * F;
    if (f0 >= p.B) break;
    // load channel LLRs, c2v = 0, total = chl
    for (long long x = tid; x < (long long)g.N * F; x += nt) {
      int n = (int)(x >> lf), q = (int)(x & (F - 1));
      long long f = f0 + q;
      T v = T(0);
      if (f < p.B) v = p.llr_f64 ? (T)((const double*)p.llr)[f * g.N + n] : (T)((const float*)p.llr)[f * g.N + n];
      chl[x] = v;
      total[x] = v;
    }
    for (long long x = tid; x < (long long)g.E * F; x += nt) c2v[x] = T(0);
    if (tid < F) {
      s_active[tid] = (f0 + tid) < p.B;
      s_iter[tid] = 0;
    }
    __syncthreads();
    for (int it = 0;; ++it) {
      // record boundary `it` + syndrome for active frames
      if (tid < F) { s_errs[tid] = 0; s_errs_info[tid] = 0; s_unsat[tid] = 0; }
      __syncthreads();
      for (long long x = tid; x < (long long)g.N * F; x += nt) {
        int n = (int)(x >> lf), q = (int)(x & (F - 1));
        if (s_active[q] && total[x] < T(0)) {
          atomicAdd(&s_errs[q], 1);
          if (n < p.k_info) atomicAdd(&s_errs_info[q], 1);
        }
      }
      if (it > 0)
        for (long long x = tid; x < (long long)g.M * F; x += nt) {
          int m = (int)(x >> lf), q = (int)(x & (F - 1));
          if (!s_active[q]) continue;
          int par = 0;
          for (int e = g.cn_ptr[m]; e < g.cn_ptr[m + 1]; ++e)
            par ^= total[(long long)g.edge_vn[e] * F + q] < T(0) ? 1 : 0;
          if (par) s_unsat[q] = 1;
        }
      __syncthreads();
      if (tid < F && s_active[tid]) {
        long long f = f0 + tid;
        p.biterr[f * (I + 1) + it] = s_errs[tid];
        p.biterr_info[f * (I + 1) + it] = s_errs_info[tid];
        bool done = false;
        if (it > 0 && !s_unsat[tid]) {  // converged at iteration it (E:761-764)
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
      int any = 0;
      for (int q = 0; q < F; ++q) any |= s_active[q];
      if (!any) break;
      // one iteration
      if (!layered) {
        for (int m0 = 0; m0 < g.M; m0 += items_per_pass) {
          int m = m0 + slot_item0;
          if (m < g.M && s_active[fl]) check_update<T, KERNEL, false>(g, m, F, fl, c2v, total);
        }
        __syncthreads();
        for (int n0 = 0; n0 < g.N; n0 += items_per_pass) {
          int n = n0 + slot_item0;
          if (n < g.N && s_active[fl]) {
            long long nx = (long long)n * F + fl;
            T s = chl[nx];
            for (int k = g.vn_ptr[n]; k < g.vn_ptr[n + 1]; ++k) s += c2v[(long long)g.vn_edges[k] * F + fl];
            total[nx] = s;
          }
        }
        __syncthreads();
      } else {
        for (int L = 0; L < g.n_levels; ++L) {
          int a = g.level_ptr[L], b = g.level_ptr[L + 1];
          for (int k0 = a; k0 < b; k0 += items_per_pass) {
            int k = k0 + slot_item0;
            if (k < b && s_active[fl]) check_update<T, KERNEL, true>(g, g.level_checks[k], F, fl, c2v, total);
          }
          __syncthreads();
        }
      }
    }
    // outputs
    for (long long x = tid; x < (long long)g.N * F; x += nt) {
      int n = (int)(x >> lf), q = (int)(x & (F - 1));
      long long f = f0 + q;
      if (f < p.B) p.u_hat[f * g.N + n] = total[x] < T(0) ? 1 : 0;
    }
    if (tid < F && f0 + tid < p.B) {
      long long f = f0 + tid;
      long long prop = (long long)s_iter[tid] * g.E;
      if (I == 0) {
        prop = 0;
        // converged = syndrome of the channel decisions (schedules.py:144-146)
        p.conv[f] = 0;
      }
      p.prop[f] = prop;
      p.counters[f * kCounters + C_PROP] = prop;
      p.counters[f * kCounters + C_V2C] = prop;
      for (int k = 2; k < kCounters; ++k) p.counters[f * kCounters + k] = 0;
    }
    if (I == 0) {
      // syndrome of channel decisions
      if (tid < F) s_unsat[tid] = 0;
      __syncthreads();
      for (long long x = tid; x < (long long)g.M * F; x += nt) {
        int m = (int)(x >> lf), q = (int)(x & (F - 1));
        int par = 0;
        for (int e = g.cn_ptr[m]; e < g.cn_ptr[m + 1]; ++e)
          par ^= total[(long long)g.edge_vn[e] * F + q] < T(0) ? 1 : 0;
        if (par) s_unsat[q] = 1;
      }
      __syncthreads();
      if (tid < F && f0 + tid < p.B) p.conv[f0 + tid] = s_unsat[tid] ? 0 : 1;
    }
    __syncthreads();
  }
}

}  // namespace ldpc
