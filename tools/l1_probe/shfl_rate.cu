// SHFL throughput and whether it occupies the L1 data pipe (ncu
// l1tex__data_pipe_lsu_wavefronts): a warp issues kIters x 8 independent
// 32-bit shuffles; compared with the same count of LDS.32.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void shfl_kernel(float* out, int sh) {
  float v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = threadIdx.x * (q + 1);
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __shfl_sync(0xffffffffu, v[q], (lane + sh + q) & 31) + 1.0f;
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += v[q];
  if (s == 1.2345f) out[0] = s;
}

__global__ void lds_kernel(float* out, int sh) {
  __shared__ float buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = i;
  __syncthreads();
  float v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = 0.f;
  const int lane = threadIdx.x & 31;
  int idx = lane;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] += buf[(idx + 32 * q) & 1023];
    idx = (idx + sh) & 1023;
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += v[q];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int k = 0; k < 2; ++k) {
      cudaEventRecord(e0);
      if (k == 0) shfl_kernel<<<148 * 4, 512>>>(out, 1);
      else lds_kernel<<<148 * 4, 512>>>(out, 32);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warp_ops = 148.0 * 4 * 16 * kIters * 8;
      printf("%s: %.3f ms, %.2f warp-ops per clock per SM (at 1.965 GHz)\n", k ? "LDS.32" : "SHFL",
             ms, warp_ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
