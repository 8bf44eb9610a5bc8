// L1 data-pipe wavefront probe: how many l1tex data-pipe wavefronts does one
// warp-wide LDG.64 cost for the lane address patterns the symmetric forward
// produces?  Each pattern kernel issues kIters loads per warp from an
// L1-resident 32 KB buffer; run under
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts.sum,
//        smsp__inst_executed_op_global_ld.sum,
//        l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum ./l1_wavefronts
// and divide wavefronts by load instructions.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kWords = 4096;   // float2 words = 32 KB

__device__ __forceinline__ int pattern(int p, int lane) {
  const int r = lane & 7, g = lane >> 3;
  switch (p) {
    case 0: return lane;                       // contiguous 256 B
    case 1: return 0;                          // broadcast
    case 2: return r;                          // 4 identical groups of 8 words
    case 3: return r + g;                      // groups shifted by 1 word
    case 4: return (r * 14) / 10 + 2 * g;      // forward-like: du 1.4, 2 px angle drift
    case 5: return r + 16 * g;                 // groups 128 B apart (same banks)
    case 6: return r + 17 * g;                 // groups 136 B apart
    case 7: return 2 * lane;                   // stride 16 B (512 B span)
    case 8: return (lane * 14) / 10;           // 32 rays of one angle, du 1.4
    case 9: return r + 8 * g;                  // 4 disjoint contiguous groups = case 0
    case 10: return (r * 14) / 10 + 5 * g;     // forward-like, wide drift
    case 11: return (r * 10) / 10 + g / 2;     // du 1, small drift
    default: return lane;
  }
}

// kPred: 0 all lanes, 1 upper half-warp off, 2 odd lanes off, 3 random 50 %
template <int P, int kPred>
__global__ void probe(const float2* __restrict__ buf, float* out, int shift) {
  const int lane = threadIdx.x & 31;
  const int off = pattern(P, lane);
  float acc = 0.f;
  unsigned base = (blockIdx.x * 97 + (threadIdx.x >> 5) * 31) & (kWords - 1);
  unsigned h = lane * 2654435761u;
#pragma unroll 8
  for (int it = 0; it < kIters; ++it) {
    base = (base + 61 + shift) & (kWords / 2 - 1);
    bool on = true;
    if (kPred == 1) on = lane < 16;
    if (kPred == 2) on = (lane & 1) == 0;
    if (kPred == 3) { h = h * 1664525u + 1013904223u; on = (h >> 31) != 0; }
    if (on) {
      const float2 v = __ldg(buf + base + off);
      acc += v.x * v.y;
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

template <int P, int kPred>
void run(const float2* buf, float* out, const char* name) {
  probe<P, kPred><<<148, 256>>>(buf, out, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%-28s pattern %2d pred %d: %s\n", name, P, kPred, cudaGetErrorString(e));
}

int main() {
  float2* buf;
  float* out;
  cudaMalloc(&buf, sizeof(float2) * kWords * 2);
  cudaMemset(buf, 0, sizeof(float2) * kWords * 2);
  cudaMalloc(&out, 4);
  run<0, 0>(buf, out, "contiguous");
  run<1, 0>(buf, out, "broadcast");
  run<2, 0>(buf, out, "4 identical groups");
  run<3, 0>(buf, out, "groups +1 word");
  run<4, 0>(buf, out, "forward-like");
  run<5, 0>(buf, out, "groups 128 B apart");
  run<6, 0>(buf, out, "groups 136 B apart");
  run<7, 0>(buf, out, "stride 16 B");
  run<8, 0>(buf, out, "32 rays du 1.4");
  run<9, 0>(buf, out, "disjoint groups");
  run<10, 0>(buf, out, "forward-like wide");
  run<11, 0>(buf, out, "du 1 small drift");
  run<0, 1>(buf, out, "contiguous upper half off");
  run<0, 2>(buf, out, "contiguous odd off");
  run<0, 3>(buf, out, "contiguous random half");
  run<4, 1>(buf, out, "forward-like upper off");
  run<4, 3>(buf, out, "forward-like random half");
  return 0;
}
