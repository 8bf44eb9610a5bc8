// Graph of N dependent tiny kernels: plain launches vs programmatic dependent
// launch (griddepcontrol.wait at kernel start).  Per-node cost on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tiny(float* x, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 0.999f + 1.0f;
}
int main() {
  const int n = 65536, N = 150;
  float* x; cudaMalloc(&x, n * 4); cudaMemset(x, 0, n * 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < N; ++k) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(n / 256); cfg.blockDim = dim3(256); cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = pdl;
      cudaLaunchKernelEx(&cfg, tiny, x, n);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 50; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d: %.2f us per kernel node (%s)\n", pdl, ms * 1e3 / (50.0 * N),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
