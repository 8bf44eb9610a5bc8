// DMMA shapes on sm_100a: m8n8k4 vs m16n8k4 / m16n8k8 / m16n8k16 (sm_90+ PTX).
#include <cstdio>
#include <cuda_runtime.h>
template <int S>
__global__ void k(double* out, int iters) {
  double a[8], b[4], c[4][4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  for (int t = 0; t < 4; ++t) for (int i = 0; i < 4; ++i) c[t][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (S == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a[0]), "d"(b[0]));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a[1]), "d"(b[1]));
      } else if (S == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (S == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) for (int i = 0; i < 4; ++i) s += c[t][i];
  if (s == 12345.0) out[threadIdx.x] = s;
}
template <int S>
void run(const char* name, double flops_per_inst) {
  double* o; cudaMalloc(&o, 1024 * 8);
  int iters = 20000;
  for (int warps = 1; warps <= 8; warps *= 2) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<S><<<148 * 4, 32 * warps>>>(o, 10);
    cudaEventRecord(e0);
    k<S><<<148 * 4, 32 * warps>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 148.0 * 4 * warps * iters * 4 * flops_per_inst;
    printf("%s warps/CTA %d: %.1f TFLOP/s\n", name, warps, flops / ms / 1e9);
  }
}
int main() {
  run<0>("m8n8k4 x2", 1024.0);
  run<1>("m16n8k4", 1024.0);
  run<2>("m16n8k8", 2048.0);
  run<3>("m16n8k16", 4096.0);
  return 0;
}
