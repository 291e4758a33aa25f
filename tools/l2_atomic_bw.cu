// l2_atomic_bw.cu -- FP64 reduction (REDG.E.ADD.F64) throughput of this B200, the resource that bounds the
// grouped translations' output accumulation.  Prints one JSON line per pattern / footprint:
// payload bytes (8 per atomic) per second.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/l2_atomic_bw tools/l2_atomic_bw.cu
//
// Patterns: "coalesced": a warp adds to 32 consecutive doubles; "m2l": the translation epilogue's pattern --
// lanes (g, t) add the real and then the imaginary part of row r0 + g of column slot(c0 + 2t + i), i = 0, 1,
// columns s = 136 complex apart (one Y slot each), slots drawn at random within the footprint.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_coalesced(double* y, int64_t n, int iters) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  uint64_t h = 0x9e3779b97f4a7c15ull * (w + 1);
  for (int i = 0; i < iters; ++i) {
    h ^= h >> 31, h *= 0xbf58476d1ce4e5b9ull, h ^= h >> 29;
    const int64_t base = (int64_t)(h % (uint64_t)(n / 32)) * 32;
    atomicAdd(y + base + lane, 1.0);
  }
}

__global__ void k_m2l(double2* y, int64_t nslots, int s, int iters) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  uint64_t h = 0x9e3779b97f4a7c15ull * (w + 7);
  for (int it = 0; it < iters; ++it) {
    h ^= h >> 31, h *= 0xbf58476d1ce4e5b9ull, h ^= h >> 29;
    const int r0 = (int)((h >> 40) % (uint64_t)(s / 8)) * 8;
    for (int i = 0; i < 2; ++i) {
      const int64_t slot = (int64_t)((h + 0x632be59bd9b4e019ull * (2 * t + i)) % (uint64_t)nslots);
      double2* p = y + slot * s + r0 + g;
      atomicAdd(&p->x, 1.0);
      atomicAdd(&p->y, 1.0);
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 2000;
  for (int64_t mb : {32, 96, 1024}) {
    const int64_t n = mb * (1 << 20) / 8;
    double* y;
    cudaMalloc(&y, n * 8);
    cudaMemset(y, 0, n * 8);
    float ms;
    k_coalesced<<<blocks, threads>>>(y, n, 10);
    cudaEventRecord(e0);
    k_coalesced<<<blocks, threads>>>(y, n, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops1 = (double)blocks * threads * iters;
    printf("{\"pattern\": \"coalesced\", \"footprint_mb\": %lld, \"atomics_per_s\": %.4g, \"payload_tb_s\": %.4f}\n",
           (long long)mb, ops1 / (ms * 1e-3), ops1 * 8 / (ms * 1e-3) / 1e12);
    const int s = 136;
    const int64_t nslots = n / 2 / s;
    k_m2l<<<blocks, threads>>>((double2*)y, nslots, s, 10);
    cudaEventRecord(e0);
    k_m2l<<<blocks, threads>>>((double2*)y, nslots, s, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops2 = (double)blocks * threads * iters * 4;
    printf("{\"pattern\": \"m2l\", \"footprint_mb\": %lld, \"atomics_per_s\": %.4g, \"payload_tb_s\": %.4f, \"err\": \"%s\"}\n",
           (long long)mb, ops2 / (ms * 1e-3), ops2 * 8 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(y);
  }
  return 0;
}
