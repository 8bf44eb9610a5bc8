// Does a second load to a line whose fill is still pending cost extra L1
// data-pipe wavefronts?  Streaming (L1-missing) forward-like lane pattern:
//   mode 0: one LDG.64 per line visit
//   mode 1: two LDG.64 back to back, words k and k-1 (same lines: the
//           symmetric forward's pair of loads)
//   mode 2: two LDG.64 back to back, the second to another buffer (no shared
//           pending line)
//   mode 3: mode 1 with the k-1 load issued after the first one's data is used
#include <cstdio>
#include <cuda_runtime.h>

constexpr long long kWords = 1LL << 24;   // float2 words = 128 MB

template <int kMode>
__global__ void probe(const float2* __restrict__ buf, const float2* __restrict__ buf2,
                      float* out) {
  const int lane = threadIdx.x & 31;
  const int off = ((lane & 7) * 14) / 10 + 2 * (lane >> 3) + 1;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  long long base = (warp * 1048573LL) & (kWords - 1 - 4096);
  float acc = 0.f;
#pragma unroll 4
  for (int it = 0; it < 2048; ++it) {
    base = (base + 4160) & (kWords - 1 - 4096);   // a new 128-B line every visit
    const float2 a = __ldg(buf + base + off);
    if (kMode == 0) {
      acc += a.x * a.y;
    } else if (kMode == 1) {
      const float2 b = __ldg(buf + base + off - 1);
      acc += a.x * a.y + b.x * b.y;
    } else if (kMode == 2) {
      const float2 b = __ldg(buf2 + base + off - 1);
      acc += a.x * a.y + b.x * b.y;
    } else {
      acc += a.x * a.y;
      const float2 b = __ldg(buf + base + off - 1 + (acc == 1e30f ? 1 : 0));
      acc += b.x * b.y;
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

int main() {
  float2 *buf, *buf2;
  float* out;
  cudaMalloc(&buf, sizeof(float2) * kWords);
  cudaMalloc(&buf2, sizeof(float2) * kWords);
  cudaMemset(buf, 0, sizeof(float2) * kWords);
  cudaMemset(buf2, 0, sizeof(float2) * kWords);
  cudaMalloc(&out, 4);
  probe<0><<<148 * 12, 128>>>(buf, buf2, out);
  probe<1><<<148 * 12, 128>>>(buf, buf2, out);
  probe<2><<<148 * 12, 128>>>(buf, buf2, out);
  probe<3><<<148 * 12, 128>>>(buf, buf2, out);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
