// fp64_peak.cu -- measure the FP64 roofline denominators on this B200 (MEASURED_PEAKS.json has none).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
//
// (1) DFMA: every thread runs 8 independent FMA chains; 148 SMs x many warps.
// (2) DMMA: warp-level mma.sync.aligned.m8n8k4.row.col.f64 (the FP64 tensor path of sm_80+).
// (3) sincos + rsqrt throughput (the P2P kernel's transcendental mix), in evaluations/s.
// Prints one JSON line per repetition (argv[1] repetitions, default 1; tools/fp64_peak.py samples the
// SM clock with nvidia-smi meanwhile): {"dfma_tflops":..., "dmma_tflops":..., "sincos_geval_s":..., "sm_mhz": ...}
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_sincos(double* out, int iters, double k) {
  double acc = 0, r = 1.0 + threadIdx.x * 1e-5;
  for (int i = 0; i < iters; ++i) {
    double s, c;
    sincos(k * r, &s, &c);
    const double ir = rsqrt(r);
    acc += (s + c) * ir;
    r += 1e-7;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256;
  float ms;
  const int reps = argc > 1 ? atoi(argv[1]) : 1;
  for (int rep = 0; rep < reps; ++rep) {
  // DFMA
  const int it1 = 20000;
  k_dfma<<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  k_dfma<<<blocks, threads>>>(d, it1, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma = 2.0 * 8 * (double)it1 * blocks * threads / (ms * 1e-3) / 1e12;
  // DMMA: m8n8k4 = 2*8*8*4 = 512 flop per warp instruction
  const int it2 = 20000;
  k_dmma<<<blocks, threads>>>(d, 100);
  cudaEventRecord(e0);
  k_dmma<<<blocks, threads>>>(d, it2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmma = 512.0 * 4 * (double)it2 * blocks * (threads / 32) / (ms * 1e-3) / 1e12;
  // sincos + rsqrt
  const int it3 = 2000;
  k_sincos<<<blocks, threads>>>(d, 10, 3.0);
  cudaEventRecord(e0);
  k_sincos<<<blocks, threads>>>(d, it3, 3.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double sc = (double)it3 * blocks * threads / (ms * 1e-3) / 1e9;
  cudaError_t err = cudaGetLastError();
  printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"sincos_rsqrt_geval_s\": %.3f, \"sms\": %d, "
         "\"clock_rate_mhz_attr\": %d, \"err\": \"%s\"}\n",
         dfma, dmma, sc, sms, clk / 1000, cudaGetErrorString(err));
  fflush(stdout);
  }
  return 0;
}
