// Random 32-byte-sector access bandwidth of HBM (the access pattern of the
// dynamic-schedule decoder: scattered sector reads / read-modify-writes over a
// multi-GB per-frame state).  Each thread issues independent accesses to
// pseudo-random sectors of a buffer of the given footprint; prints GB/s of
// sector traffic (32 B per read, 64 B per read-modify-write).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o randbw randbw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

template <int RMW, int RUN>  // RUN: consecutive sectors per random position (1 = fully random)
__global__ void __launch_bounds__(256) rand_access(double* buf, unsigned long long n_sectors, int iters,
                                                    double* sink) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (int i = 0; i < iters; i += 4) {
    double v[4];
    unsigned long long s[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned long long pos = mix(tid * 1000003ull + (unsigned long long)(i + k) / RUN) % (n_sectors - RUN);
      s[k] = pos + (unsigned long long)(i + k) % RUN;
      v[k] = buf[s[k] * 4];  // one 8-byte word of the sector
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc += v[k];
      if (RMW) buf[s[k] * 4 + 1] = v[k] + 1.0;
    }
  }
  if (acc == 123.456) *sink = acc;
}

template <int RMW, int RUN>
double run(double* buf, unsigned long long n_sectors, int blocks, int iters, double* sink) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  rand_access<RMW, RUN><<<blocks, 256>>>(buf, n_sectors, 64, sink);  // warm-up
  cudaEventRecord(a);
  rand_access<RMW, RUN><<<blocks, 256>>>(buf, n_sectors, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double acc = (double)blocks * 256 * iters;
  return acc * (RMW ? 64.0 : 32.0) / (ms * 1e-3) / 1e9;
}

int main() {
  double* sink;
  cudaMalloc(&sink, 8);
  const double gbs[] = {0.0625, 1, 4, 16, 32};
  printf("{\"random_sector_bandwidth_GBps\": [\n");
  for (int gi = 0; gi < 5; ++gi) {
    const unsigned long long bytes = (unsigned long long)(gbs[gi] * (1ull << 30));
    double* buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("  {\"footprint_GB\": %g, \"error\": \"alloc\"},\n", gbs[gi]); continue; }
    cudaMemset(buf, 0, bytes);
    const unsigned long long ns = bytes / 32;
    for (int wps = 8; wps <= 64; wps *= 2) {  // resident warps per SM
      const int blocks = 148 * wps / 8;
      const double r1 = run<0, 1>(buf, ns, blocks, 2048, sink);
      const double w1 = run<1, 1>(buf, ns, blocks, 2048, sink);
      const double r4 = run<0, 4>(buf, ns, blocks, 2048, sink);
      printf("  {\"footprint_GB\": %g, \"warps_per_sm\": %d, \"read_GBps\": %.1f, \"rmw_GBps\": %.1f, \"read_runs_of_4_sectors_GBps\": %.1f}%s\n",
             gbs[gi], wps, r1, w1, r4, (gi == 4 && wps == 64) ? "" : ",");
      fflush(stdout);
    }
    cudaFree(buf);
  }
  printf("]}\n");
  return 0;
}
