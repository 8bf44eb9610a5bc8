#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int v) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
    if (v >= 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (v <= 1) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
    if (v == 2) {  // expect 0 bytes then plain
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(0) : "memory");
    }
    if (v == 3) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(4096) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(sm)), "l"((unsigned long long)&tmap), "r"(0), "r"(0), "r"(su(&bar)) : "memory");
    }
    if (v == 4) {  // prefetch descriptor only
      asm volatile("prefetch.tensormap [%0];" ::"l"((unsigned long long)&tmap) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
    }
  }
  if (v <= 2 || v == 4) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(&bar)), "r"(0) : "memory");
  } else {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(&bar)), "r"(0) : "memory");
  }
  if (threadIdx.x == 0) out[0] = sm[5];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int v = atoi(argv[1]);
  float *d, *o; cudaMalloc(&d, 64 * 64 * 4); cudaMalloc(&o, 64);
  cudaMemset(d, 0, 64 * 64 * 4);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  alignas(64) CUtensorMap m;
  cuuint64_t dims[2] = {64, 64}; cuuint64_t str[1] = {64 * 4}; cuuint32_t box[2] = {32, 32}; cuuint32_t es[2] = {1, 1};
  CUresult r = ((Enc)p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 32, 8192>>>(m, o, v);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d encode %d -> %s\n", v, (int)r, cudaGetErrorString(e));
  return 0;
}
