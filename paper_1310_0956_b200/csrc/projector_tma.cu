// projector_tma.cu -- TMA-staged symmetric forward projector (fp32 data).
//
// Same arithmetic as fwd_sym_kernel (projector_fast.cu): a thread walks one
// representative ray (angle a in [1, m/2), detector j < ceil(d/2)) slab by slab
// in 32.32 fixed point and accumulates the four symmetric rays (a, j),
// (m-a, j), (a, d-1-j), (m-a, d-1-j).  The difference is where the pixels come
// from: fwd_sym gathers them from L2 (two 4-byte loads per ray-slab, L1 hit rate
// ~50 %, L2-bandwidth bound at n = 4096), this kernel stages them in shared
// memory with the Tensor Memory Accelerator.
//
// Block = 4 consecutive representative angles x 64 rays (256 threads).  The
// slab range of the block is cut into stages of kStage slabs; for each stage
// four 2-D boxes (kStage rows x kWin columns) are fetched with
// cp.async.bulk.tensor from the zero-padded plane (rows s and n-1-s, columns
// around the rays and their x-mirror), double buffered on mbarriers.  The
// window origin of the next stage is a block-wide min over the rays' column
// ranges (one shared-memory reduction per stage).  Consecutive angles differ by
// ~pi/m, so the four angles of a block read almost the same window: every
// staged pixel is used by ~4x more ray-slabs than an L1 line in fwd_sym.
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace wmg {
namespace tma {

constexpr int kStage = 16;     // slabs per stage
constexpr int kWin = 192;      // window columns (floats)
constexpr int kAng = 4;        // angles per block
constexpr int kRays = 64;      // representative rays per angle
constexpr int kBox = kStage * kWin;                 // floats per box
constexpr int kStageFloats = 4 * kBox;              // four boxes per stage
constexpr unsigned kStageBytes = kStageFloats * 4u;
constexpr double kQ32 = 4294967296.0;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float frac1(unsigned lo) {
  return __int_as_float(0x3F800000u | (lo >> 9));
}
__device__ __forceinline__ int hi32(long long v) { return (int)((unsigned long long)v >> 32); }

// k range (window columns needed, k-1 .. k) of one ray over slabs [ra, rb]
__device__ __forceinline__ void ray_cols(long long U0, long long S, int ra, int rb, int& klo,
                                         int& khi) {
  const long long Ua = U0 + (long long)(ra + 1) * S;   // u at the end of slab ra
  const long long Ub = U0 + (long long)(rb + 1) * S;
  klo = hi32(Ua) - 1;
  khi = hi32(Ub);
}

// One launch per major axis (the tensor map must stay in parameter space, so it
// is never selected at run time): group0 = first angle group of this launch.
template <typename TOut>
__global__ void __launch_bounds__(256) fwd_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                      GeomDev G, int group0,
                                                      TOut* __restrict__ sino,
                                                      int* __restrict__ overflow) {
  extern __shared__ __align__(128) float smem[];
  __shared__ unsigned long long bars[2];
  __shared__ int red[4];   // rc0, rc1, kmin, kmax of the next stage
  const int tid = threadIdx.x, lane = tid & 31;
  const int n = G.n, m = G.m, d = G.d;
  const int jh = (d + 1) / 2;
  const int ai = tid / kRays;
  const int a = 1 + (group0 + blockIdx.y) * kAng + ai;
  const int j = blockIdx.x * kRays + (tid % kRays);
  const bool angle_ok = a < m / 2;
  const AngleParams& A = G.ang[angle_ok ? a : 1];
  const CUtensorMap* map = &tmap;
  const int M = kPadMargin;

  // per-ray slab range (as fwd_sym_kernel)
  const double off = (double)j - (double)(d - 1) * 0.5;
  const double u0 = A.u0 + off * A.du;
  const double slope = A.slope;
  int r0 = 0, r1 = n - 1;
  if (!angle_ok || j >= jh) {
    r0 = n; r1 = -1;
  } else if (slope > 0.0) {
    const double ra = floor((-1.0 - u0) / slope) - 1.0;
    const double rb = ceil(((double)n + 1.0 - u0) / slope) + 1.0;
    r0 = (int)fmin(fmax(ra, 0.0), (double)n);
    r1 = (int)fmax(fmin(rb, (double)(n - 1)), -1.0);
  } else if (u0 < -1.0 || u0 > (double)n + 1.0) {
    r0 = n; r1 = -1;
  }
  const long long S = llrint(slope * kQ32);
  const long long U0 = llrint(u0 * kQ32);   // u at the start of slab 0

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    red[0] = n; red[1] = -1;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  {
    const int w0 = __reduce_min_sync(0xffffffffu, r0);
    const int w1 = __reduce_max_sync(0xffffffffu, r1);
    if (lane == 0) {
      atomicMin(&red[0], w0);
      atomicMax(&red[1], w1);
    }
  }
  __syncthreads();
  const int rc0 = red[0], rc1 = red[1];
  float2 accA = make_float2(0.0f, 0.0f), accB = make_float2(0.0f, 0.0f);
  if (rc0 > rc1) {   // nothing to do for this block (uniform)
    goto write_out;
  }
  {
    const int nst = (rc1 - rc0) / kStage + 1;
    // stage window origin: block min of the needed columns
    auto stage_window = [&](int st, int& kb, int& kspan) {
      const int s0 = rc0 + st * kStage;
      const int ra = max(s0, r0), rb = min(s0 + kStage - 1, r1);
      int klo = 1 << 30, khi = -(1 << 30);
      if (ra <= rb) ray_cols(U0, S, ra, rb, klo, khi);
      klo = __reduce_min_sync(0xffffffffu, klo);
      khi = __reduce_max_sync(0xffffffffu, khi);
      __syncthreads();
      if (tid == 0) { red[2] = 1 << 30; red[3] = -(1 << 30); }
      __syncthreads();
      if (lane == 0) { atomicMin(&red[2], klo); atomicMax(&red[3], khi); }
      __syncthreads();
      // TMA box origins must be 16-byte aligned: floor to a multiple of 4 floats
      kb = red[2] & ~3;
      kspan = red[3] - kb + 1;
    };
    auto issue = [&](int st, int kb, int b) {
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int s0 = rc0 + st * kStage;
        float* dst = smem + b * kStageFloats;
        mbar_expect_tx(&bars[b], kStageBytes);
        // rows s0 .. s0+kStage-1: columns [kb, kb+W) and mirrored [n-kb-W, n-kb)
        tma_load_2d(dst + 0 * kBox, map, kb + M, s0, &bars[b]);
        tma_load_2d(dst + 1 * kBox, map, n - kb - kWin + M, s0, &bars[b]);
        // rows n-s0-kStage .. n-s0-1 (the 180-degree images)
        tma_load_2d(dst + 2 * kBox, map, n - kb - kWin + M, n - s0 - kStage, &bars[b]);
        tma_load_2d(dst + 3 * kBox, map, kb + M, n - s0 - kStage, &bars[b]);
      }
    };
    int kb_cur, span;
    stage_window(0, kb_cur, span);
    if (overflow && span > kWin - 2 && tid == 0) atomicAdd(overflow, 1);
    issue(0, kb_cur, 0);
    const float L = A.Lf, Ls = A.Lsf;
    unsigned phase = 0u;
    for (int st = 0; st < nst; ++st) {
      const int b = st & 1;
      int kb_next = 0, span_next = 0;
      if (st + 1 < nst) {
        stage_window(st + 1, kb_next, span_next);
        if (overflow && span_next > kWin - 2 && tid == 0) atomicAdd(overflow, 1);
        issue(st + 1, kb_next, b ^ 1);
      }
      mbar_wait(&bars[b], (phase >> b) & 1u);
      phase ^= 1u << b;
      const float* X0 = smem + b * kStageFloats;   // (s, q)
      const float* X1 = X0 + kBox;                 // (s, n-1-q) mirrored columns
      const float* X2 = X0 + 2 * kBox;             // (n-1-s, n-1-q)
      const float* X3 = X0 + 3 * kBox;             // (n-1-s, q)
      const int s0 = rc0 + st * kStage;
      long long U = U0 + (long long)s0 * S;
#pragma unroll 4
      for (int rr = 0; rr < kStage; ++rr) {
        U += S;
        const int r = s0 + rr;
        const bool valid = (r >= r0) & (r <= r1);
        int c = hi32(U) - kb_cur;                         // window column of k
        c = min(max(c, 1), kWin - 2);
        const float f = frac1((unsigned)U);
        float wh = fminf(fmaf(f, Ls, -Ls), L);
        const float Lv = valid ? L : 0.0f;
        wh = valid ? wh : 0.0f;
        const float2 W = make_float2(wh, wh);
        const float2 LV = make_float2(Lv, Lv);
        const int cm = kWin - 1 - c;                      // mirrored column
        const int rA = rr * kWin, rB = (kStage - 1 - rr) * kWin;
        const float2 v1A = make_float2(X0[rA + c], X1[rA + cm]);
        const float2 v0A = make_float2(X0[rA + c - 1], X1[rA + cm + 1]);
        const float2 v1B = make_float2(X2[rB + cm], X3[rB + c]);
        const float2 v0B = make_float2(X2[rB + cm + 1], X3[rB + c - 1]);
        accA = __ffma2_rn(LV, v0A, accA);
        accA = __ffma2_rn(W, __fadd2_rn(v1A, make_float2(-v0A.x, -v0A.y)), accA);
        accB = __ffma2_rn(LV, v0B, accB);
        accB = __ffma2_rn(W, __fadd2_rn(v1B, make_float2(-v0B.x, -v0B.y)), accB);
      }
      __syncthreads();   // buffer b is refilled by stage st+2
      kb_cur = kb_next;
    }
  }
write_out:
  if (angle_ok && j < jh) {
    const float r_m = A.major ? accB.y : accA.y;    // (m-a, j)
    const float r_mr = A.major ? accA.y : accB.y;   // (m-a, d-1-j)
    sino[(long long)a * d + j] = (TOut)accA.x;
    sino[(long long)(m - a) * d + j] = (TOut)r_m;
    if (d - 1 - j != j) {
      sino[(long long)a * d + (d - 1 - j)] = (TOut)accB.x;
      sino[(long long)(m - a) * d + (d - 1 - j)] = (TOut)r_mr;
    }
  }
}

}  // namespace tma

// ---------------------------------------------------------------------------
// host side: tensor maps over the zero-padded planes (driver entry point via
// the runtime, so the library does not link libcuda directly)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

static bool make_map(CUtensorMap* map, float* plane, int n) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t pitch = (cuuint64_t)(n + 2 * kPadMargin);
  cuuint64_t dims[2] = {pitch, (cuuint64_t)n};
  cuuint64_t strides[1] = {pitch * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)tma::kWin, (cuuint32_t)tma::kStage};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, plane, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// representative angles are grouped by 4; a group must not straddle 45 degrees
bool tma_forward_supported(const GeomDev& G) {
  return G.sym && G.tma_ok && (G.m % 16 == 0) && G.m >= 32 &&
         (G.n + 2 * kPadMargin) % 4 == 0 && encode_fn() != nullptr;
}

// host-side bound on the window a block needs (rays of one angle, stage length,
// spread between the four angles of a group); true if it fits kWin - 2
bool tma_window_fits(const AngleParams* P, int n, int d, int m) {
  const int reps = m / 2 - 1;
  const double half_d = 0.5 * (double)(d - 1);
  for (int g0 = 1; g0 <= reps; g0 += tma::kAng) {
    double du_max = 0.0, slope_max = 0.0, spread = 0.0;
    const int g1 = g0 + tma::kAng - 1 < reps ? g0 + tma::kAng - 1 : reps;
    for (int a = g0; a <= g1; ++a) {
      du_max = fmax(du_max, fabs(P[a].du));
      slope_max = fmax(slope_max, P[a].slope);
      for (int b = g0; b <= g1; ++b) {
        if (P[a].major != P[b].major) return false;
        const double s = fabs(P[a].u0 - P[b].u0) + half_d * fabs(P[a].du - P[b].du) +
                         (double)n * fabs(P[a].slope - P[b].slope);
        spread = fmax(spread, s);
      }
    }
    const double span = tma::kRays * du_max + tma::kStage * slope_max + spread + 4.0 + 3.0;
    if (span > (double)(tma::kWin - 2)) return false;
  }
  return true;
}

template <typename TOut>
cudaError_t tma_forward(const GeomDev& G, float* P, float* PT, TOut* sino, int* overflow,
                        cudaStream_t st) {
  CUtensorMap mP, mPT;
  if (!make_map(&mP, P, G.n) || !make_map(&mPT, PT, G.n)) return cudaErrorNotSupported;
  const size_t smem = 2 * (size_t)tma::kStageBytes;
  cudaError_t e = cudaFuncSetAttribute(tma::fwd_tma_kernel<TOut>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int jh = (G.d + 1) / 2;
  const int reps = G.m / 2 - 1;
  const int groups = (reps + tma::kAng - 1) / tma::kAng;
  const int y_groups = G.m / 16;            // angles 1 .. m/4 are y-major (m % 16 == 0)
  const int gx = (jh + tma::kRays - 1) / tma::kRays;
  if (y_groups > 0) {
    tma::fwd_tma_kernel<TOut><<<dim3(gx, y_groups), 256, smem, st>>>(mP, G, 0, sino, overflow);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (groups > y_groups) {
    tma::fwd_tma_kernel<TOut><<<dim3(gx, groups - y_groups), 256, smem, st>>>(mPT, G, y_groups,
                                                                          sino, overflow);
    e = cudaGetLastError();
  }
  return e;
}

template cudaError_t tma_forward<float>(const GeomDev&, float*, float*, float*, int*,
                                        cudaStream_t);
template cudaError_t tma_forward<double>(const GeomDev&, float*, float*, double*, int*,
                                         cudaStream_t);

}  // namespace wmg
