// l2_bw.cu -- L2 read bandwidth on this B200 (for the M2L gather/scatter roofline discussion).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/l2_bw tools/l2_bw.cu && tools/bin/l2_bw
// Reads a buffer of `mb` MiB (16-byte loads, grid-stride) `reps` times after a warm-up pass; for
// buffers well below the 126 MB L2 this is L2 bandwidth, far above it HBM bandwidth.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const double2* __restrict__ a, size_t n, int reps, double* out) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const double2 v = __ldcg(a + i);
      s += v.x + v.y;
    }
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* o;
  cudaMalloc(&o, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int mbs[] = {16, 32, 48, 64, 96, 2048};
  printf("{");
  for (int t = 0; t < 6; ++t) {
    const size_t bytes = (size_t)mbs[t] << 20, n = bytes / 16;
    double2* a;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 0, bytes);
    const int reps = mbs[t] >= 1024 ? 2 : 20;
    k_read<<<sms * 8, 256>>>(a, n, 1, o);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_read<<<sms * 8, 256>>>(a, n, reps, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s\"read_%dMiB_GBs\": %.1f", t ? ", " : "", mbs[t], (double)bytes * reps / (ms * 1e-3) / 1e9);
    cudaFree(a);
  }
  printf("}\n");
  return 0;
}
