// fixed_trace.cu -- flooding / layered decoding with want_trace outputs.
//
// The reference records, at every iteration boundary, the totals and the
// pre-totals of the next flooding pass (E:192-217 with E:768-782,
// _flood_pre_totals).  The frame-interleaved fixed kernels (fixed_engine.cuh)
// never form those pre-totals, so traced flooding / layered decodes run here:
// one warp per frame, per-frame state in an HBM slot, the same arithmetic as
// the oracle (oracle/ldpc_oracle.c decode_flooding / decode_layered), so the
// decisions, counters and bit-error rows equal the untraced kernels' bit for
// bit.  This is the J(gamma) study path (sim.py:339-353), not the throughput
// path.
#include "kernel_table.h"

namespace ldpc {

template <typename T, int KERNEL>
__device__ __forceinline__ T msg_in(T v) {  // cached check input (E:58 / E:73)
  return KERNEL == KERNEL_EXACT ? cn_in<T>(v) : v;
}

// in[e] = input of edge e from the extrinsic clamp(total - c2v) (E:754), all edges
template <typename T, int KERNEL>
__device__ void inputs_all(const DevGraph& g, const T* total, const T* c2v, T* in, const Grp<32>& w) {
  for (int e = w.lane; e < g.E; e += 32) in[e] = msg_in<T, KERNEL>(clampv(total[g.edge_vn[e]] - c2v[e]));
  w.sync();
}

// out[e] = C2V of every edge from the cached inputs (E:743-745)
template <typename T, int KERNEL>
__device__ void checks_all(const DevGraph& g, const T* in, T* out, const Grp<32>& w) {
  for (int e = w.lane; e < g.E; e += 32) {
    const int m = g.edge_cn[e];
    out[e] = cn_msg_cached<T, KERNEL>(in, g.cn_ptr[m], g.cn_ptr[m + 1], e);
  }
  w.sync();
}

// s[n] = chl[n] + sum of msg over vn_edges, in vn_edges order (E:749-750 / E:777-780)
template <typename T>
__device__ void vn_sums(const DevGraph& g, const T* chl, const T* msg, T* s, const Grp<32>& w) {
  for (int n = w.lane; n < g.N; n += 32) {
    T acc = chl[n];
    for (int k = g.vn_ptr[n]; k < g.vn_ptr[n + 1]; ++k) acc += msg[g.vn_edges[k]];
    s[n] = acc;
  }
  w.sync();
}

template <typename T>
__device__ bool syndrome_ok_w(const DevGraph& g, const T* total, const Grp<32>& w) {  // E:179-188
  for (int m0 = 0; m0 < g.M; m0 += 32) {
    const int m = m0 + w.lane;
    int par = 0;
    if (m < g.M)
      for (int e = g.cn_ptr[m]; e < g.cn_ptr[m + 1]; ++e) par ^= total[g.edge_vn[e]] < T(0) ? 1 : 0;
    if (w.any(par)) return false;
  }
  return true;
}

template <typename T, int KERNEL, bool LAYERED>
__global__ void __launch_bounds__(kTraceWarps * 32) fixed_trace_kernel(FixedTraceParams p) {
  const DevGraph& g = p.g;
  const Grp<32> w = Grp<32>::make();
  const int lane = w.lane, I = p.i_max;
  const long long E = g.E;
  unsigned char* slot = p.ws + ((long long)blockIdx.x * kTraceWarps + (threadIdx.x >> 5)) * p.slot_bytes;
  T* c2v = (T*)slot;
  T* in = c2v + E;
  T* pre = in + E;
  T* total = pre + E;
  T* pretot = total + g.N;
  T* chl = pretot + g.N;
  for (;;) {
    unsigned long long fq = 0;
    if (lane == 0) fq = atomicAdd(p.next, 1ull);
    fq = w.shfl(fq, 0);
    if ((long long)fq >= p.B) break;
    const long long f = (long long)fq;
    for (int n = lane; n < g.N; n += 32) {
      const T v = p.llr_f64 ? (T)((const double*)p.llr)[f * g.N + n] : (T)((const float*)p.llr)[f * g.N + n];
      chl[n] = v;
      total[n] = v;  // E:117 (not clamped)
    }
    for (long long e = lane; e < E; e += 32) c2v[e] = T(0);
    w.sync();
    const bool want = p.tr.trace || p.tr.jc;
    auto boundary = [&](int k, bool conv) {
      int errs = 0, ei = 0;
      for (int n = lane; n < g.N; n += 32)
        if (total[n] < T(0)) {
          ++errs;
          if (n < p.k_info) ++ei;
        }
      errs = w.rsum(errs);
      ei = w.rsum(ei);
      if (lane == 0)
        for (int kk = k; kk <= (conv ? I : k); ++kk) {
          p.biterr[f * (I + 1) + kk] = errs;
          p.biterr_info[f * (I + 1) + kk] = ei;
        }
      if (want) {  // next flooding pass from the current extrinsics (E:768-782)
        inputs_all<T, KERNEL>(g, total, c2v, in, w);
        checks_all<T, KERNEL>(g, in, pre, w);
        vn_sums<T>(g, chl, pre, pretot, w);
        trace_boundary_rows<T, 32>(p.tr, g.N, I, total, pretot, f, k, conv, w);
      }
      w.sync();
    };
    boundary(0, false);
    bool conv = false;
    int it = 0;
    for (it = 1; it <= I; ++it) {
      if (!LAYERED) {  // E:741-756
        inputs_all<T, KERNEL>(g, total, c2v, in, w);
        checks_all<T, KERNEL>(g, in, c2v, w);
        vn_sums<T>(g, chl, c2v, total, w);
      } else {  // rows in order (oracle decode_layered)
        for (int m = 0; m < g.M; ++m) {
          const int a = g.cn_ptr[m], b = g.cn_ptr[m + 1];
          for (int e = a + lane; e < b; e += 32) in[e] = msg_in<T, KERNEL>(clampv(total[g.edge_vn[e]] - c2v[e]));
          w.sync();
          for (int e = a + lane; e < b; e += 32) pre[e] = cn_msg_cached<T, KERNEL>(in, a, b, e);
          w.sync();
          for (int e = a + lane; e < b; e += 32) {
            total[g.edge_vn[e]] += pre[e] - c2v[e];
            c2v[e] = pre[e];
          }
          w.sync();
        }
      }
      const bool ok = syndrome_ok_w<T>(g, total, w);
      boundary(it, ok);
      if (ok) {
        conv = true;
        break;
      }
    }
    if (it > I) it = I;
    if (I == 0) conv = syndrome_ok_w<T>(g, total, w);  // schedules.py:144-146
    for (int n = lane; n < g.N; n += 32) p.u_hat[f * g.N + n] = total[n] < T(0) ? 1 : 0;
    if (lane == 0) {
      const long long prop = I > 0 ? (long long)it * E : 0;
      p.prop[f] = prop;
      p.conv[f] = conv ? 1 : 0;
      p.counters[f * kCounters + C_PROP] = prop;
      p.counters[f * kCounters + C_V2C] = prop;
      for (int k = 2; k < kCounters; ++k) p.counters[f * kCounters + k] = 0;
    }
    w.sync();
  }
}

}  // namespace ldpc

using namespace ldpc;

void* ldpc_fixed_trace_kernel(int f64, int kernel, int layered) {
  if (f64) {
    if (kernel == KERNEL_EXACT)
      return layered ? (void*)fixed_trace_kernel<double, KERNEL_EXACT, true>
                     : (void*)fixed_trace_kernel<double, KERNEL_EXACT, false>;
    return layered ? (void*)fixed_trace_kernel<double, KERNEL_MINSUM, true>
                   : (void*)fixed_trace_kernel<double, KERNEL_MINSUM, false>;
  }
  if (kernel == KERNEL_EXACT)
    return layered ? (void*)fixed_trace_kernel<float, KERNEL_EXACT, true>
                   : (void*)fixed_trace_kernel<float, KERNEL_EXACT, false>;
  return layered ? (void*)fixed_trace_kernel<float, KERNEL_MINSUM, true>
                 : (void*)fixed_trace_kernel<float, KERNEL_MINSUM, false>;
}
