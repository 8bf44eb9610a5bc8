// Minimal TMA probe: load one 2-D box with cp.async.bulk.tensor and compare.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int c0, int c1, int variant) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(16 * 64 * 4) : "memory");
    if (variant == 0)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sm)), "l"((unsigned long long)&tmap), "r"(c0), "r"(c1), "r"(smem_u32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sm)), "l"((unsigned long long)&tmap), "r"(c0), "r"(c1), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) out[i] = sm[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int mode = atoi(argv[1]);
  const int W = 200, H = 50;
  std::vector<float> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, W * H * 4); cudaMalloc(&o, 16 * 64 * 4);
  cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  printf("entry %d q %d p %p\n", (int)e, (int)q, p);
  CUtensorMap m;
  cuuint64_t dims[2] = {W, H}; cuuint64_t str[1] = {W * 4}; cuuint32_t box[2] = {64, 16}; cuuint32_t es[2] = {1, 1};
  CUresult r = ((Enc)p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, (mode & 1) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int variant = 0; variant < 2; ++variant) {
    for (int t = 0; t < 3; ++t) {
      int c0 = (mode & 2) ? 0 : (t == 0 ? 10 : (t == 1 ? -5 : 180)), c1 = (mode & 2) ? 0 : (t == 0 ? 3 : (t == 1 ? -2 : 45));
      k<<<1, (mode & 4) ? 32 : 128, 16 * 64 * 4>>>(m, o, c0, c1, variant);
      e = cudaDeviceSynchronize();
      printf("variant %d test %d: %s\n", variant, t, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
      std::vector<float> g(16 * 64);
      cudaMemcpy(g.data(), o, g.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int rr = 0; rr < 16; ++rr) for (int cc = 0; cc < 64; ++cc) {
        int R = c1 + rr, C = c0 + cc;
        float ref = (R >= 0 && R < H && C >= 0 && C < W) ? h[R * W + C] : 0.0f;
        if (g[rr * 64 + cc] != ref) ++bad;
      }
      printf("   mismatches %d\n", bad);
    }
  }
  return 0;
}
