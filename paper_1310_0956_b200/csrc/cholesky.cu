// cholesky.cu -- batched dense Cholesky factorization (potrf) on the fp64
// tensor cores and batched triangular solves (potrs), hand-written.
//
// Replaces the reference's cholesky_factor / cholesky_solve
// (/root/reference/pkg/src/wmgtomo/sparse_kernels.py:53-75: scipy.linalg
// cholesky(lower=True) = LAPACK potrf, cho_solve = potrs) on the device.  The
// WMG V-cycle itself applies explicit leaf inverses (spd_inverse.cu); these
// entry points are the public factor / solve API.
//
// potrf, right-looking, block T = 128, lower factor of row-major G (p x p,
// p % 128 == 0), per pivot block k:
//   diag   one CTA per matrix: unblocked Cholesky of A_kk in registers
//          (thread (q, c) holds rows q + 4i of column c), then the in-place
//          triangular inverse X_k = L_kk^-1 in shared memory;
//   panel  L_Ik = A_Ik X_k^T for I > k           (DMMA 128 x 128 x 128)
//   update A_IJ -= L_Ik L_Jk^T for k < J <= I     (DMMA, 128 x 64 halves)
// p^3 / 3 flops in the tile products.  The diagonal-block inverses X_k are
// kept (p x T doubles per matrix) for the solves.  info = order of the first
// non-positive leading minor (potrf's convention), 0 on success.
//
// potrs: one CTA per (matrix, right-hand side): y = L^-1 b block by block
// (row-block GEMV against the solved prefix, then X_k), z = L^-T y backwards
// (column-block GEMV against the solved suffix, then X_k^T).  Fixed summation
// orders: the results are bit-reproducible.
#include <cuda_runtime.h>

#include <cstdint>

namespace wmg {
namespace spd {
// shared with spd_inverse.cu (same tile GEMM and layout constants)
constexpr int T = 128;
constexpr int KC = 32;
constexpr int LDSM = KC + 4;
constexpr int OPND = T * LDSM;
constexpr int STAGE = 2 * OPND;
constexpr int GEMM_SMEM = 2 * STAGE * (int)sizeof(double);
constexpr int UPD_NC = 64;
constexpr int UPD_SMEM = 2 * (T + UPD_NC) * LDSM * (int)sizeof(double);
constexpr int SQ = T + 1;
constexpr int TILE_SMEM = T * SQ * (int)sizeof(double);
}  // namespace spd

namespace chol {
using spd::T;
using spd::LDSM;
using spd::OPND;
using spd::SQ;

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

template <int NC>
__device__ __forceinline__ void load_stage(double* sA, double* sB, const double* A, long long lda,
                                           const double* B, long long ldb, int k0) {
#pragma unroll
  for (int i = threadIdx.x; i < T * (spd::KC / 2); i += 256) {
    const int r = i >> 4, v = (i & 15) * 2;
    cp16(sA + r * LDSM + v, A + r * lda + k0 + v);
    if (NC == T || r < NC) cp16(sB + r * LDSM + v, B + r * ldb + k0 + v);
  }
}

// acc (this warp's part of a 128 x NC tile) += A(128 x T) B(NC x T)^T, both
// row-major; double-buffered cp.async stages; fragment (i, j) of warp (wr, wc):
// rows wr*MI*8 + 8i + g, cols wc*32 + 8j + 2t + {0,1}.
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
  for (int kc = 0; kc < T / spd::KC; ++kc) {
    double* cur = smem + (kc & 1) * STG;
    if (kc + 1 < T / spd::KC) {
      double* nxt = smem + ((kc + 1) & 1) * STG;
      load_stage<NC>(nxt, nxt + OPND, A, lda, B, ldb, (kc + 1) * spd::KC);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const double* sA = cur + (wr * MI * 8 + g) * LDSM + t;
    const double* sB = cur + OPND + (wc * 32 + g) * LDSM + t;
#pragma unroll
    for (int kk = 0; kk < spd::KC; kk += 4) {
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

__device__ __forceinline__ void lower_tile(int lin, int& I, int& J) {
  int i = (int)((sqrtf(8.0f * (float)lin + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= lin) ++i;
  while (i * (i + 1) / 2 > lin) --i;
  I = i;
  J = lin - i * (i + 1) / 2;
}

// Factor the pivot block and invert its factor.  512 threads; thread
// (q = tid / 128, c = tid % 128) holds A_kk[q + 4i][c], i < 32.
__global__ void __launch_bounds__(512, 1) diag_kernel(int p, double* __restrict__ G, long long sG,
                                                      double* __restrict__ dinv, int k,
                                                      int* __restrict__ info) {
  extern __shared__ double S[];            // T x SQ: L_kk, then X_k in place
  __shared__ double col[2][T];
  const int mtx = blockIdx.x;
  const int c = threadIdx.x & (T - 1), q = threadIdx.x >> 7;
  double* Gb = G + mtx * sG + (long long)k * T * p + (long long)k * T;
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int r = q + 4 * i;
    v[i] = c <= r ? Gb[(long long)r * p + c] : 0.0;
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
    if (!(d > 0.0) || !isfinite(d)) {
      if (!bad) bad = k * T + j + 1;
      d = 1.0;   // keep going (the host raises); no NaN / inf spread
    }
    const double s = sqrt(d);
    const double inv = 1.0 / s;
    if (c == j) {                                // column j of L
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int r = q + 4 * i;
        if (r > j) v[i] = cj[r] * inv;
        else if (r == j) v[i] = s;
      }
    } else if (c > j) {                          // trailing lower part: r >= c > j
      const double lc = cj[c] * inv;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int r = q + 4 * i;
        if (r >= c) v[i] = fma(-(cj[r] * inv), lc, v[i]);
      }
    }
  }
  if (bad && c == 0 && q == 0 && info[mtx] == 0) info[mtx] = bad;
  // L_kk -> G (zeros above the diagonal) and shared memory
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int r = q + 4 * i;
    const double l = c <= r ? v[i] : 0.0;
    Gb[(long long)r * p + c] = l;
    S[r * SQ + c] = l;
  }
  __syncthreads();
  // in-place inverse of the lower triangular L (columns right to left):
  //   X_jj = 1 / L_jj,  X[j+1:, j] = -(X[j+1:, j+1:] L[j+1:, j]) X_jj
  // rows split over the 4 thread quarters (q), the k-sum over a quarter's
  // 128 threads... each row r > j is owned by one thread (tid < T - 1 - j).
  for (int j = T - 1; j >= 0; --j) {
    const double xjj = 1.0 / S[j * SQ + j];
    const int r = j + 1 + threadIdx.x;
    double t = 0.0;
    if (r < T) {
      for (int kk = j + 1; kk <= r; ++kk) t = fma(S[r * SQ + kk], S[kk * SQ + j], t);
    }
    __syncthreads();
    if (r < T) S[r * SQ + j] = -t * xjj;
    if (threadIdx.x == 0) S[j * SQ + j] = xjj;
    __syncthreads();
  }
  double* X = dinv + mtx * (long long)p * T + (long long)k * T * T;
  for (int idx = threadIdx.x; idx < T * T; idx += 512) {
    const int r = idx >> 7, cc = idx & (T - 1);
    X[idx] = cc <= r ? S[r * SQ + cc] : 0.0;
  }
}

// L_Ik = A_Ik X_k^T for I = k + 1 + blockIdx.x (in place in G)
__global__ void __launch_bounds__(256, 1) panel_kernel(int p, double* __restrict__ G, long long sG,
                                                       const double* __restrict__ dinv, int k) {
  extern __shared__ double smem[];
  const int I = k + 1 + blockIdx.x, mtx = blockIdx.y;
  double* A = G + mtx * sG + (long long)I * T * p + (long long)k * T;
  const double* X = dinv + mtx * (long long)p * T + (long long)k * T * T;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  tile_gemm<T>(acc, A, p, X, T, smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp >> 2, wc = warp & 3;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = wr * 64 + i * 8 + g, cc = wc * 32 + j * 8 + 2 * t;
      *reinterpret_cast<double2*>(A + (long long)r * p + cc) =
          make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// A_IJ -= L_Ik L_Jk^T over the trailing lower tiles (k < J <= I), 128 x 64 halves
__global__ void __launch_bounds__(256, 2) update_kernel(int p, double* __restrict__ G, long long sG,
                                                        int k) {
  extern __shared__ double smem[];
  constexpr int NC = spd::UPD_NC, MI = NC / 16, CW = NC / 32;
  int i0, j0;
  lower_tile(blockIdx.x >> 1, i0, j0);
  const int I = k + 1 + i0, J = k + 1 + j0;
  const int half = blockIdx.x & 1;
  double* Gb = G + blockIdx.y * sG;
  double* C = Gb + (long long)I * T * p + (long long)J * T + half * NC;
  const double* LI = Gb + (long long)I * T * p + (long long)k * T;
  const double* LJ = Gb + (long long)(J * T + half * NC) * p + (long long)k * T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / CW, wc = warp % CW;
  double acc[MI][4][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = wr * MI * 8 + i * 8 + g, cc = wc * 32 + j * 8 + 2 * t;
      const double2 v = *reinterpret_cast<const double2*>(C + (long long)r * p + cc);
      acc[i][j][0] = -v.x;                       // -(C) + L_I L_J^T, negated back
      acc[i][j][1] = -v.y;
    }
  tile_gemm<NC>(acc, LI, p, LJ, p, smem);
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = wr * MI * 8 + i * 8 + g, cc = wc * 32 + j * 8 + 2 * t;
      *reinterpret_cast<double2*>(C + (long long)r * p + cc) =
          make_double2(-acc[i][j][0], -acc[i][j][1]);
    }
}

// zero the strictly upper tiles (I < J)
__global__ void __launch_bounds__(256) zero_upper_kernel(int p, double* __restrict__ G,
                                                         long long sG) {
  int I, J;
  lower_tile(blockIdx.x, I, J);                  // (I, J) lower -> tile (J, I) upper
  if (I == J) return;
  double* dst = G + blockIdx.y * sG + (long long)J * T * p + (long long)I * T;
  for (int idx = threadIdx.x; idx < T * T; idx += 256) {
    const int r = idx >> 7, cc = idx & (T - 1);
    dst[(long long)r * p + cc] = 0.0;
  }
}

// One CTA per (right-hand side, matrix): B (p x nrhs row-major per matrix) is
// overwritten with (L L^T)^-1 B.  Dynamic shared memory: 2 p doubles.
__global__ void __launch_bounds__(256) solve_kernel(int p, const double* __restrict__ L,
                                                    long long sL, const double* __restrict__ dinv,
                                                    double* __restrict__ B, long long sB,
                                                    int nrhs) {
  extern __shared__ double sm[];
  double* y = sm;          // p
  double* tb = sm + p;     // T (block right-hand side)
  __shared__ double part[2][T];
  const int col = blockIdx.x, mtx = blockIdx.y;
  const double* Lm = L + mtx * sL;
  const double* Xm = dinv + mtx * (long long)p * T;
  double* Bm = B + mtx * sB;
  const int nt = p / T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < p; i += 256) y[i] = Bm[(long long)i * nrhs + col];
  __syncthreads();
  // forward: y_k = X_k (b_k - L[k rows, :kT] y[:kT])
  for (int kb = 0; kb < nt; ++kb) {
    const int kT = kb * T;
    for (int rr = 0; rr < 16; ++rr) {            // warp w: rows 16 w .. 16 w + 15
      const int r = kT + warp * 16 + rr;
      const double* row = Lm + (long long)r * p;
      double s = 0.0;
      for (int jj = lane; jj < kT; jj += 32) s = fma(row[jj], y[jj], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) tb[warp * 16 + rr] = y[r] - s;
    }
    __syncthreads();
    const double* X = Xm + (long long)kb * T * T;
    for (int rr = 0; rr < 16; ++rr) {
      const int r = warp * 16 + rr;
      double s = 0.0;
      for (int jj = lane; jj <= r; jj += 32) s = fma(X[r * T + jj], tb[jj], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) y[kT + r] = s;
    }
    __syncthreads();
  }
  // backward: z_k = X_k^T (y_k - L[(k+1)T:, k cols]^T z[(k+1)T:])
  const int c = threadIdx.x & (T - 1), hh = threadIdx.x >> 7;
  for (int kb = nt - 1; kb >= 0; --kb) {
    const int kT = kb * T;
    const int r0 = kT + T, nrow = p - r0;
    const int ra = r0 + (nrow * hh) / 2, rb = r0 + (nrow * (hh + 1)) / 2;
    double s = 0.0;
    for (int r = ra; r < rb; ++r) s = fma(Lm[(long long)r * p + kT + c], y[r], s);
    part[hh][c] = s;
    __syncthreads();
    if (hh == 0) tb[c] = y[kT + c] - (part[0][c] + part[1][c]);
    __syncthreads();
    const double* X = Xm + (long long)kb * T * T;
    double z = 0.0;
    if (hh == 0)
      for (int r = c; r < T; ++r) z = fma(X[r * T + c], tb[r], z);
    __syncthreads();
    if (hh == 0) y[kT + c] = z;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < p; i += 256) Bm[(long long)i * nrhs + col] = y[i];
}

}  // namespace chol

size_t cholesky_dinv_elems(int p) { return (size_t)p * chol::T; }

cudaError_t cholesky_factor(int batch, int p, double* G, long long sG, double* dinv, int* info,
                            cudaStream_t st) {
  using namespace chol;
  if (batch <= 0 || p <= 0) return cudaSuccess;
  if (p % T) return cudaErrorInvalidValue;
  cudaError_t e;
  static bool attrs = false;   // idempotent; a racing first call sets the same values
  if (!attrs) {
    if ((e = cudaFuncSetAttribute(diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  spd::TILE_SMEM)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  spd::GEMM_SMEM)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  spd::UPD_SMEM)) != cudaSuccess)
      return e;
    attrs = true;
  }
  if ((e = cudaMemsetAsync(info, 0, sizeof(int) * (size_t)batch, st)) != cudaSuccess) return e;
  const int nt = p / T;
  for (int k = 0; k < nt; ++k) {
    diag_kernel<<<batch, 512, spd::TILE_SMEM, st>>>(p, G, sG, dinv, k, info);
    const int m = nt - 1 - k;
    if (m > 0) {
      panel_kernel<<<dim3(m, batch), 256, spd::GEMM_SMEM, st>>>(p, G, sG, dinv, k);
      update_kernel<<<dim3(m * (m + 1), batch), 256, spd::UPD_SMEM, st>>>(p, G, sG, k);
    }
  }
  if (nt > 1) zero_upper_kernel<<<dim3(nt * (nt + 1) / 2, batch), 256, 0, st>>>(p, G, sG);
  return cudaGetLastError();
}

cudaError_t cholesky_solve(int batch, int p, const double* L, long long sL, const double* dinv,
                           double* B, long long sB, int nrhs, cudaStream_t st) {
  using namespace chol;
  if (batch <= 0 || p <= 0 || nrhs <= 0) return cudaSuccess;
  if (p % T) return cudaErrorInvalidValue;
  const size_t smem = 2 * (size_t)p * sizeof(double);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  solve_kernel<<<dim3(nrhs, batch), 256, smem, st>>>(p, L, sL, dinv, B, sB, nrhs);
  return cudaGetLastError();
}

}  // namespace wmg
