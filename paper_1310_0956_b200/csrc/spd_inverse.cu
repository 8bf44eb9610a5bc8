// spd_inverse.cu -- batched in-place inverse of SPD leaf Grams on the fp64
// tensor cores (DMMA m8n8k4), for the WMG coarse solves.
//
// Replaces the reference's per-leaf LAPACK potrf (sparse_kernels.py:53-65,
// called from multilevel.py:125-137) followed by cho_solve in every V-cycle
// (sparse_kernels.py:68-75): the V-cycle applies the explicit inverse with
// wmg_batched_gemv, and this file computes that inverse without cuSOLVER.
//
// Algorithm: blocked symmetric sweep (Gauss-Jordan on an SPD matrix, no
// pivoting), block size T = 128.  Sweeping pivot block k of symmetric A:
//     D    = A_kk^-1                          (one CTA per leaf: scalar sweep)
//     A_ij = A_ij - A_ik D A_kj     i, j != k (rank-128 update, DMMA)
//     A_ik = A_ik D,  A_kj = D A_kj            (panel)
//     A_kk = -D
// After all p/T blocks the matrix holds -A^-1.  Only the lower triangle is
// read and maintained (the swept matrix stays symmetric); a last pass writes
// the full, negated, mirrored result row-major for the GEMV.  The pivots are
// the Schur-complement diagonals, i.e. the squared Cholesky pivots, so the
// first non-positive one names the same leading minor as potrf's info.
// Flops: p^3 per leaf (lower-triangle tiles only), all of it in 128x128x128
// DMMA tile products; HBM: the lower triangle read and written once per step.
#include <cuda_runtime.h>

#include <cstdint>

namespace wmg {
namespace spd {

constexpr int T = 128;            // pivot block = output tile
constexpr int KC = 32;            // k chunk per pipeline stage
constexpr int LDSM = KC + 4;      // padded smem row (doubles): conflict-free fragment loads
constexpr int OPND = T * LDSM;    // doubles per staged operand chunk
constexpr int STAGE = 2 * OPND;   // A + B chunk
constexpr int GEMM_SMEM = 2 * STAGE * (int)sizeof(double);   // double-buffered: 147456 B
// update kernel: 128 x 64 tiles, two CTAs per SM (one loads/stores C while the
// other multiplies): 2 x (A 128 + B 64 rows) x LDSM doubles = 110592 B
constexpr int UPD_NC = 64;
constexpr int UPD_SMEM = 2 * (T + UPD_NC) * LDSM * (int)sizeof(double);
constexpr int SQ = T + 1;         // padded row of a full 128x128 tile in smem
constexpr int TILE_SMEM = T * SQ * (int)sizeof(double);      // 132096 B

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp16(double* smem, const double* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// chunk [k0, k0+KC) of 128 rows of A and NC rows of B (row-major, leading dims lda/ldb)
template <int NC>
__device__ __forceinline__ void load_stage(double* sA, double* sB, const double* A, long long lda,
                                           const double* B, long long ldb, int k0) {
#pragma unroll
  for (int i = threadIdx.x; i < T * (KC / 2); i += 256) {
    const int r = i >> 4, v = (i & 15) * 2;
    cp16(sA + r * LDSM + v, A + r * lda + k0 + v);
    if (NC == T || r < NC) cp16(sB + r * LDSM + v, B + r * ldb + k0 + v);
  }
}

// acc (this warp's part of a 128 x NC tile) += A(128 x T) * B(NC x T)^T.
// 8 warps as (8 / CW) rows x CW cols of warp tiles (MI*8) x 32, CW = NC / 32,
// MI = NC / 16; fragment (i, j): rows wr*MI*8 + 8i + g, cols wc*32 + 8j + 2t + {0,1}
// (g = lane / 4, t = lane % 4).  Staged operands: A chunk then B chunk per stage.
template <int NC>
__device__ __forceinline__ void tile_gemm(double (&acc)[NC / 16][4][2], const double* A,
                                          long long lda, const double* B, long long ldb,
                                          double* smem) {
  constexpr int CW = NC / 32, MI = NC / 16;
  constexpr int OPB = NC * LDSM, STG = OPND + OPB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / CW, wc = warp % CW;
  load_stage<NC>(smem, smem + OPND, A, lda, B, ldb, 0);
  cp_commit();
#pragma unroll 1
  for (int kc = 0; kc < T / KC; ++kc) {
    double* cur = smem + (kc & 1) * STG;
    if (kc + 1 < T / KC) {
      double* nxt = smem + ((kc + 1) & 1) * STG;
      load_stage<NC>(nxt, nxt + OPND, A, lda, B, ldb, (kc + 1) * KC);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const double* sA = cur + (wr * MI * 8 + g) * LDSM + t;
    const double* sB = cur + OPND + (wc * 32 + g) * LDSM + t;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double a[MI], b[4];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = sA[i * 8 * LDSM + kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[j * 8 * LDSM + kk];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- kernels
// workspace per leaf: Dneg (T x T) | Uneg (p x T) | P (p x T)

// Sweep the pivot block: S = -A_kk^-1 -> Dneg and tile (k,k).  512 threads;
// thread (q = tid / 128, c = tid % 128) keeps S[q + 4i][c], i < 32, in
// registers.  By symmetry the pivot row is the pivot column, which the four
// threads owning column j publish to shared memory (double-buffered: one
// barrier per step).
__global__ void __launch_bounds__(512, 1) sweep_diag_kernel(int p, double* __restrict__ G,
                                                            long long sG,
                                                            double* __restrict__ work,
                                                            long long sW, int k,
                                                            int* __restrict__ info) {
  __shared__ double col[2][T];
  const int leaf = blockIdx.x;
  const int c = threadIdx.x & (T - 1), q = threadIdx.x >> 7;
  double* Gb = G + leaf * sG + (long long)k * T * p + (long long)k * T;
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int r = q + 4 * i;
    v[i] = c <= r ? Gb[(long long)r * p + c] : Gb[(long long)c * p + r];
  }
  int bad = 0;
#pragma unroll 1
  for (int j = 0; j < T; ++j) {
    double* cj = col[j & 1];
    if (c == j) {
#pragma unroll
      for (int i = 0; i < 32; ++i) cj[q + 4 * i] = v[i];
    }
    __syncthreads();
    double d = cj[j];
    if (!(d > 0.0)) {
      if (!bad) bad = k * T + j + 1;
      d = 1.0;   // keep going (the host raises); no NaN/inf spread
    }
    const double inv = 1.0 / d;
    const double rc = cj[c];
    const int jq = j & 3, ji = j >> 2;
    if (c == j) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = cj[q + 4 * i] * inv;
      if (q == jq) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i == ji) v[i] = -inv;
      }
    } else {
      const double rci = rc * inv;
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fma(-cj[q + 4 * i], rci, v[i]);
      if (q == jq) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i == ji) v[i] = rci;
      }
    }
  }
  if (bad && c == 0 && q == 0 && info[leaf] == 0) info[leaf] = bad;
  double* Dn = work + leaf * sW;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int r = q + 4 * i;
    Dn[r * T + c] = v[i];
    Gb[(long long)r * p + c] = v[i];
  }
}

// Panel: P_I = A_Ik (gathered from tile (I,k) or tile (k,I)^T), Uneg_I = P_I Dneg,
// tile (I,k) <- -Uneg_I (I > k) or tile (k,I) <- -Uneg_I^T (I < k).
__global__ void __launch_bounds__(256, 1) sweep_panel_kernel(int p, double* __restrict__ G,
                                                             long long sG,
                                                             double* __restrict__ work,
                                                             long long sW, int k) {
  extern __shared__ double smem[];
  const int I = blockIdx.x, leaf = blockIdx.y;
  if (I == k) return;
  double* Gb = G + leaf * sG;
  double* Dn = work + leaf * sW;
  double* Un = Dn + (long long)T * T;
  double* P = Un + (long long)p * T;
  double* PI = P + (long long)I * T * T;
  if (I > k) {
    const double* src = Gb + (long long)I * T * p + (long long)k * T;
    for (int idx = threadIdx.x; idx < T * T / 2; idx += 256) {
      const int r = idx >> 6, c = (idx & 63) * 2;
      *reinterpret_cast<double2*>(PI + r * T + c) =
          *reinterpret_cast<const double2*>(src + (long long)r * p + c);
    }
  } else {
    // transpose tile (k, I) through shared memory
    const double* src = Gb + (long long)k * T * p + (long long)I * T;
    for (int idx = threadIdx.x; idx < T * T; idx += 256) {
      const int r = idx >> 7, c = idx & (T - 1);
      smem[r * SQ + c] = src[(long long)r * p + c];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < T * T; idx += 256) {
      const int r = idx >> 7, c = idx & (T - 1);
      PI[idx] = smem[c * SQ + r];
    }
  }
  __syncthreads();
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  tile_gemm<T>(acc, PI, T, Dn, T, smem);   // Dneg is symmetric: rows of Dneg = columns
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp >> 2, wc = warp & 3;
  double* UI = Un + (long long)I * T * T;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = wr * 64 + i * 8 + g, c = wc * 32 + j * 8 + 2 * t;
      *reinterpret_cast<double2*>(UI + r * T + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      if (I > k) {
        *reinterpret_cast<double2*>(Gb + (long long)(I * T + r) * p + k * T + c) =
            make_double2(-acc[i][j][0], -acc[i][j][1]);
      } else {
        Gb[(long long)(k * T + c) * p + I * T + r] = -acc[i][j][0];
        Gb[(long long)(k * T + c + 1) * p + I * T + r] = -acc[i][j][1];
      }
    }
}

__device__ __forceinline__ void lower_tile(int lin, int& I, int& J) {
  int i = (int)((sqrtf(8.0f * (float)lin + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= lin) ++i;
  while (i * (i + 1) / 2 > lin) --i;
  I = i;
  J = lin - i * (i + 1) / 2;
}

// Trailing update of every lower tile (I, J) off the pivot strip, in two
// 128 x 64 halves (blockIdx.x = 2 * tile + half): A_IJ += Uneg_I P_J^T.
__global__ void __launch_bounds__(256, 2) sweep_update_kernel(int p, double* __restrict__ G,
                                                              long long sG,
                                                              const double* __restrict__ work,
                                                              long long sW, int k) {
  extern __shared__ double smem[];
  constexpr int MI = UPD_NC / 16, CW = UPD_NC / 32;
  int I, J;
  lower_tile(blockIdx.x >> 1, I, J);
  if (I == k || J == k) return;
  const int half = blockIdx.x & 1;
  const int leaf = blockIdx.y;
  double* Cb = G + leaf * sG + (long long)I * T * p + (long long)J * T + half * UPD_NC;
  const double* Un = work + leaf * sW + (long long)T * T;
  const double* P = Un + (long long)p * T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / CW, wc = warp % CW;
  double acc[MI][4][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = wr * MI * 8 + i * 8 + g, c = wc * 32 + j * 8 + 2 * t;
      const double2 v = __ldcs(reinterpret_cast<const double2*>(Cb + (long long)r * p + c));
      acc[i][j][0] = v.x;
      acc[i][j][1] = v.y;
    }
  tile_gemm<UPD_NC>(acc, Un + (long long)I * T * T, T,
                    P + (long long)J * T * T + (long long)half * UPD_NC * T, T, smem);
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = wr * MI * 8 + i * 8 + g, c = wc * 32 + j * 8 + 2 * t;
      *reinterpret_cast<double2*>(Cb + (long long)r * p + c) =
          make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// out = -(swept lower triangle), mirrored into the full row-major matrix.
__global__ void __launch_bounds__(256) sweep_finish_kernel(int p, double* __restrict__ G,
                                                          long long sG) {
  extern __shared__ double S[];
  int I, J;
  lower_tile(blockIdx.x, I, J);
  double* Gb = G + blockIdx.y * sG;
  double* src = Gb + (long long)I * T * p + (long long)J * T;
  for (int idx = threadIdx.x; idx < T * T; idx += 256) {
    const int r = idx >> 7, c = idx & (T - 1);
    S[r * SQ + c] = src[(long long)r * p + c];
  }
  __syncthreads();
  if (I == J) {
    for (int idx = threadIdx.x; idx < T * T; idx += 256) {
      const int r = idx >> 7, c = idx & (T - 1);
      src[(long long)r * p + c] = -(c <= r ? S[r * SQ + c] : S[c * SQ + r]);
    }
    return;
  }
  double* dst = Gb + (long long)J * T * p + (long long)I * T;
  for (int idx = threadIdx.x; idx < T * T; idx += 256) {
    const int r = idx >> 7, c = idx & (T - 1);
    src[(long long)r * p + c] = -S[r * SQ + c];
    dst[(long long)r * p + c] = -S[c * SQ + r];
  }
}

}  // namespace spd

size_t spd_inverse_workspace(int batch, int p) {
  return (size_t)batch * ((size_t)spd::T * spd::T + 2ull * (size_t)p * spd::T) * sizeof(double);
}

cudaError_t spd_inverse(int batch, int p, double* G, long long sG, int* info, double* work,
                        cudaStream_t st) {
  using namespace spd;
  if (batch <= 0 || p <= 0) return cudaSuccess;
  cudaError_t e;
  static bool attrs = false;
  if (!attrs) {
    if ((e = cudaFuncSetAttribute(sweep_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  TILE_SMEM)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(sweep_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  GEMM_SMEM)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(sweep_update_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, UPD_SMEM)) !=
        cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(sweep_finish_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_SMEM)) !=
        cudaSuccess)
      return e;
    attrs = true;
  }
  if ((e = cudaMemsetAsync(info, 0, sizeof(int) * (size_t)batch, st)) != cudaSuccess) return e;
  const int nt = p / T;
  const int ntri = nt * (nt + 1) / 2;
  const long long sW = (long long)T * T + 2LL * p * T;
  for (int k = 0; k < nt; ++k) {
    sweep_diag_kernel<<<batch, 512, TILE_SMEM, st>>>(p, G, sG, work, sW, k, info);
    if (nt > 1) {
      sweep_panel_kernel<<<dim3(nt, batch), 256, GEMM_SMEM, st>>>(p, G, sG, work, sW, k);
      sweep_update_kernel<<<dim3(2 * ntri, batch), 256, UPD_SMEM, st>>>(p, G, sG, work, sW, k);
    }
  }
  sweep_finish_kernel<<<dim3(ntri, batch), 256, TILE_SMEM, st>>>(p, G, sG);
  return cudaGetLastError();
}

}  // namespace wmg
