// Peak DMMA (mma.sync m8n8k4 f64) throughput on sm_100a: register-only loop.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}
int main() {
  double* o; cudaMalloc(&o, 1024 * 8);
  int iters = 20000;
  for (int warps = 1; warps <= 16; warps *= 2) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<148 * 4, 32 * warps>>>(o, 10);
    cudaEventRecord(e0);
    k<<<148 * 4, 32 * warps>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 148.0 * 4 * warps * iters * 8 * 512.0;
    printf("warps/CTA %2d: %.1f TFLOP/s fp64 DMMA\n", warps, flops / ms / 1e9);
  }
  return 0;
}
