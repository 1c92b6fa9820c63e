// channel_gen.cu -- on-GPU BPSK/AWGN frame generation.
//
// Same channel model and LLR convention as the reference
// (/root/reference/pkg/src/ldpc_ids/channel.py:35-86): all-zero codeword,
// x = +1, y = x + sigma * z, LLR = clip(2 y / sigma^2, +-30) at transmitted
// positions and 0 at punctured ones (a punctured prefix, codes.py:243-248).
// Frames are keyed by (seed, frame index) like channel.frame_rng, so any frame
// can be produced independently; the stream is Philox4x32-10 (counter-based)
// with Box-Muller normals, i.e. statistically -- not bitwise -- equivalent to
// numpy's Philox4x64 + ziggurat stream.  One Philox block yields the two
// 64-bit uniforms of one Box-Muller pair = two channel samples.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/ldpc_b200.h"

namespace {

__device__ __forceinline__ void philox_round(uint32_t (&c)[4], const uint32_t (&k)[2]) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  c[0] = hi1 ^ c[1] ^ k[0];
  c[1] = lo1;
  c[2] = hi0 ^ c[3] ^ k[1];
  c[3] = lo0;
}

// Philox4x32-10 (Salmon et al., SC'11)
__device__ __forceinline__ void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
  uint32_t k[2] = {k0, k1};
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c, k);
    k[0] += 0x9E3779B9u;
    k[1] += 0xBB67AE85u;
  }
}

__device__ __forceinline__ double u01(uint32_t lo, uint32_t hi) {  // (0, 1), 53 bits
  const uint64_t x = ((uint64_t)hi << 32 | lo) >> 11;
  return ((double)x + 0.5) * (1.0 / 9007199254740992.0);
}

template <typename T>
__global__ void awgn_llr_kernel(T* out, int N, int n_punct, long long B, double sigma, unsigned long long seed,
                                long long start) {
  const int n_tx = N - n_punct, pairs = (n_tx + 1) / 2;
  const double scale = 2.0 / (sigma * sigma);
  const long long total = B * (long long)pairs;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < total;
       w += (long long)gridDim.x * blockDim.x) {
    const long long b = w / pairs;
    const int pr = (int)(w - b * pairs);
    const unsigned long long frame = (unsigned long long)(start + b);
    uint32_t c[4] = {(uint32_t)pr, (uint32_t)frame, (uint32_t)(frame >> 32), 0x4C445043u};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double r = sqrt(-2.0 * log(u01(c[0], c[1])));
    double s, co;
    sincospi(2.0 * u01(c[2], c[3]), &s, &co);
    const double z[2] = {r * co, r * s};
    T* row = out + b * (long long)N;
    if (pr == 0)
      for (int n = 0; n < n_punct; ++n) row[n] = T(0);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int t = 2 * pr + q;
      if (t >= n_tx) break;
      const double y = 1.0 + sigma * z[q];
      double l = scale * y;
      l = l > 30.0 ? 30.0 : (l < -30.0 ? -30.0 : l);
      row[n_punct + t] = (T)l;
    }
  }
}

}  // namespace

extern "C" int ldpc_generate_awgn(int32_t N, int32_t n_punct_prefix, int64_t B, double sigma, uint64_t seed,
                                  int64_t start, void* out, int32_t out_f64, void* stream) {
  if (N <= 0 || n_punct_prefix < 0 || n_punct_prefix >= N || B < 0 || !(sigma > 0) || (B > 0 && !out))
    return LDPC_ERR_INVALID;
  if (B == 0) return LDPC_OK;
  const long long pairs = (N - n_punct_prefix + 1) / 2;
  const long long total = B * pairs;
  const int threads = 256;
  const int blocks = (int)((total + threads - 1) / threads < 148 * 16 ? (total + threads - 1) / threads : 148 * 16);
  cudaStream_t st = (cudaStream_t)stream;
  if (out_f64)
    awgn_llr_kernel<double><<<blocks, threads, 0, st>>>((double*)out, N, n_punct_prefix, B, sigma, seed, start);
  else
    awgn_llr_kernel<float><<<blocks, threads, 0, st>>>((float*)out, N, n_punct_prefix, B, sigma, seed, start);
  return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}
