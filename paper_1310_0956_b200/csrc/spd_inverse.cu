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
#include <mutex>
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
// mode 0: every lower tile off the pivot strip k; mode 1 (look-ahead): only the
// strip c = k + 1 (the next pivot's row and column, blockIdx.x over its nt
// tiles); mode 2: every tile off the strips k and c.
__global__ void __launch_bounds__(256, 2) sweep_update_kernel(int p, double* __restrict__ G,
                                                              long long sG,
                                                              const double* __restrict__ work,
                                                              long long sW, int k, int c,
                                                              int mode) {
  extern __shared__ double smem[];
  constexpr int MI = UPD_NC / 16, CW = UPD_NC / 32;
  int I, J;
  if (mode == 1) {
    const int t = blockIdx.x >> 1;
    I = t <= c ? c : t;
    J = t <= c ? t : c;
  } else {
    lower_tile(blockIdx.x >> 1, I, J);
  }
  if (I == k || J == k) return;
  if (mode == 2 && (I == c || J == c)) return;
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


// ------------------------------------------------- packed symmetric storage
// A symmetric p x p matrix (p % 128 == 0) kept as its lower 128 x 128 tiles,
// tile (I, J), I >= J, at index I (I + 1) / 2 + J, each row-major; diagonal
// tiles hold the full (mirrored) tile.  Half the bytes of the dense inverse:
// the V-cycle's coarse solves (one symmetric GEMV per leaf per cycle) stream
// 67 MB instead of 134 MB per 4096^2 leaf.

// pack the lower tiles of a full symmetric matrix (mirrors the diagonal tiles
// from their lower triangles)
__global__ void __launch_bounds__(256) sym_pack_kernel(int p, const double* __restrict__ A,
                                                       long long sA, double* __restrict__ Pk,
                                                       long long sP) {
  int I, J;
  lower_tile(blockIdx.x, I, J);
  const double* src = A + blockIdx.y * sA + (long long)I * T * p + (long long)J * T;
  double* dst = Pk + blockIdx.y * sP + (long long)blockIdx.x * T * T;
  for (int idx = threadIdx.x; idx < T * T / 2; idx += 256) {
    const int r = idx >> 6, c = (idx & 63) * 2;
    double2 v = *reinterpret_cast<const double2*>(src + (long long)r * p + c);
    if (I == J) {
      if (c > r) v.x = src[(long long)c * p + r];
      if (c + 1 > r) v.y = src[(long long)(c + 1) * p + r];
    }
    *reinterpret_cast<double2*>(dst + r * T + c) = v;
  }
}

// One packed tile per CTA, read once: u = A_IJ x_J -> S[K=I][L=J], and for
// I != J also v = A_IJ^T x_I -> S[K=J][L=I].  8 warps x 16 rows; lane = 4
// columns (two 16-byte loads per row, 8 rows in flight); rows reduced with a
// fixed shuffle tree, columns over the warps in warp order (deterministic).
__global__ void __launch_bounds__(256) sym_tile_gemv_kernel(int p, const double* __restrict__ Pk,
                                                            long long sP,
                                                            const double* __restrict__ x,
                                                            long long sx,
                                                            double* __restrict__ S) {
  __shared__ double colp[8][T];
  int I, J;
  lower_tile(blockIdx.x, I, J);
  const int nt = p / T;
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* tile = Pk + b * sP + (long long)blockIdx.x * T * T + (warp * 16) * T + lane * 4;
  const double* xb = x + b * sx;
  const double4 xj = *reinterpret_cast<const double4*>(xb + J * T + lane * 4);
  double* Sb = S + (long long)b * nt * nt * T;
  double cacc[4] = {0.0, 0.0, 0.0, 0.0};
  double rsum = 0.0;   // lane i < 16 ends with row 16 warp + i
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double2 v[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i][0] = __ldcs(reinterpret_cast<const double2*>(tile + (h * 8 + i) * T));
      v[i][1] = __ldcs(reinterpret_cast<const double2*>(tile + (h * 8 + i) * T + 2));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = warp * 16 + h * 8 + i;
      double r = v[i][0].x * xj.x;
      r = fma(v[i][0].y, xj.y, r);
      r = fma(v[i][1].x, xj.z, r);
      r = fma(v[i][1].y, xj.w, r);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
      if (lane == h * 8 + i) rsum = r;
      if (I != J) {
        const double xi = xb[I * T + row];
        cacc[0] = fma(v[i][0].x, xi, cacc[0]);
        cacc[1] = fma(v[i][0].y, xi, cacc[1]);
        cacc[2] = fma(v[i][1].x, xi, cacc[2]);
        cacc[3] = fma(v[i][1].y, xi, cacc[3]);
      }
    }
  }
  if (lane < 16) Sb[((long long)I * nt + J) * T + warp * 16 + lane] = rsum;
  if (I == J) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) colp[warp][lane * 4 + q] = cacc[q];
  __syncthreads();
  if (threadIdx.x < T) {
    double s = colp[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < 8; ++w) s += colp[w][threadIdx.x];
    Sb[((long long)J * nt + I) * T + threadIdx.x] = s;
  }
}

// y_K = sum over L of S[K][L], L ascending
__global__ void __launch_bounds__(T) sym_reduce_kernel(int p, const double* __restrict__ S,
                                                       double* __restrict__ y, long long sy) {
  const int K = blockIdx.x, b = blockIdx.y, nt = p / T;
  const double* src = S + ((long long)b * nt + K) * nt * T + threadIdx.x;
  double s = 0.0;
  for (int L = 0; L < nt; ++L) s += src[(long long)L * T];
  y[b * sy + K * T + threadIdx.x] = s;
}

}  // namespace spd

// two buffer sets (pivot steps alternate): the look-ahead forms step k+1's
// panel while step k's trailing update still reads step k's
size_t spd_inverse_workspace(int batch, int p) {
  return 2ull * (size_t)batch * ((size_t)spd::T * spd::T + 2ull * (size_t)p * spd::T) *
         sizeof(double);
}

namespace {
// Serialises spd_inverse's host-side enqueue: the lazily created per-device
// auxiliary stream, its fork/join events and the kernel attributes are shared
// by every caller, so two threads (or two caller streams) enqueueing at once
// would re-record each other's events between a record and the matching wait.
// Under the lock each call enqueues its whole fork/join chain before the next
// starts; the GPU work of concurrent calls may still overlap (a later call's
// auxiliary items queue behind the earlier call's on the in-order aux stream).
std::mutex g_spd_mutex;
// per-device auxiliary stream + fork/join events of the look-ahead (created once)
struct AuxStreams {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
cudaError_t aux_for_device(AuxStreams*& out) {
  static AuxStreams aux[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  AuxStreams& a = aux[dev];
  if (!a.s) {
    int lo = 0, hi = 0;
    if ((e = cudaDeviceGetStreamPriorityRange(&lo, &hi)) != cudaSuccess) return e;
    // high priority: the pivot sweep and panel (on the critical path) get SMs
    // as soon as trailing-update CTAs retire
    if ((e = cudaStreamCreateWithPriority(&a.s, cudaStreamNonBlocking, hi)) != cudaSuccess)
      return e;
    if ((e = cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  out = &a;
  return cudaSuccess;
}
}  // namespace

cudaError_t spd_inverse(int batch, int p, double* G, long long sG, int* info, double* work,
                        cudaStream_t st) {
  using namespace spd;
  if (batch <= 0 || p <= 0) return cudaSuccess;
  std::lock_guard<std::mutex> lock(g_spd_mutex);
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
  const long long sW1 = (long long)T * T + 2LL * p * T;   // one buffer set per leaf
  const long long sW = 2 * sW1;                          // leaf stride (two sets)
  auto buf = [&](int k) { return work + (k & 1) * sW1; };
  AuxStreams* aux = nullptr;
  if (nt > 2 && (e = aux_for_device(aux)) != cudaSuccess) return e;
  // step 0's pivot sweep and panel
  sweep_diag_kernel<<<batch, 512, TILE_SMEM, st>>>(p, G, sG, buf(0), sW, 0, info);
  if (nt > 1)
    sweep_panel_kernel<<<dim3(nt, batch), 256, GEMM_SMEM, st>>>(p, G, sG, buf(0), sW, 0);
  for (int k = 0; k < nt && nt > 1; ++k) {
    const int c = k + 1;
    if (c < nt && aux) {
      // look-ahead: update strip c first, then form pivot c's sweep and panel on
      // the auxiliary stream while the rest of step k's update runs
      sweep_update_kernel<<<dim3(2 * nt, batch), 256, UPD_SMEM, st>>>(p, G, sG, buf(k), sW, k,
                                                                       c, 1);
      if ((e = cudaEventRecord(aux->fork, st)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(aux->s, aux->fork, 0)) != cudaSuccess) return e;
      sweep_diag_kernel<<<batch, 512, TILE_SMEM, aux->s>>>(p, G, sG, buf(c), sW, c, info);
      sweep_panel_kernel<<<dim3(nt, batch), 256, GEMM_SMEM, aux->s>>>(p, G, sG, buf(c), sW, c);
      if ((e = cudaEventRecord(aux->join, aux->s)) != cudaSuccess) return e;
      sweep_update_kernel<<<dim3(2 * ntri, batch), 256, UPD_SMEM, st>>>(p, G, sG, buf(k), sW, k,
                                                                        c, 2);
      if ((e = cudaStreamWaitEvent(st, aux->join, 0)) != cudaSuccess) return e;
    } else {
      sweep_update_kernel<<<dim3(2 * ntri, batch), 256, UPD_SMEM, st>>>(p, G, sG, buf(k), sW, k,
                                                                        -1, 0);
      if (c < nt) {
        sweep_diag_kernel<<<batch, 512, TILE_SMEM, st>>>(p, G, sG, buf(c), sW, c, info);
        sweep_panel_kernel<<<dim3(nt, batch), 256, GEMM_SMEM, st>>>(p, G, sG, buf(c), sW, c);
      }
    }
  }
  sweep_finish_kernel<<<dim3(ntri, batch), 256, TILE_SMEM, st>>>(p, G, sG);
  return cudaGetLastError();
}

size_t packed_sym_elems(int p) {
  const long long nt = p / spd::T;
  return (size_t)(nt * (nt + 1) / 2) * spd::T * spd::T;
}

size_t packed_symv_scratch(int batch, int p) {
  const long long nt = p / spd::T;
  return (size_t)batch * (size_t)(nt * nt) * spd::T * sizeof(double);
}

cudaError_t sym_pack(int batch, int p, const double* A, long long sA, double* Pk, long long sP,
                     cudaStream_t st) {
  if (batch <= 0 || p <= 0) return cudaSuccess;
  const int nt = p / spd::T;
  spd::sym_pack_kernel<<<dim3(nt * (nt + 1) / 2, batch), 256, 0, st>>>(p, A, sA, Pk, sP);
  return cudaGetLastError();
}

cudaError_t packed_symv(int batch, int p, const double* Pk, long long sP, const double* x,
                        long long sx, double* y, long long sy, double* scratch,
                        cudaStream_t st) {
  if (batch <= 0 || p <= 0) return cudaSuccess;
  const int nt = p / spd::T;
  spd::sym_tile_gemv_kernel<<<dim3(nt * (nt + 1) / 2, batch), 256, 0, st>>>(p, Pk, sP, x, sx,
                                                                           scratch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  spd::sym_reduce_kernel<<<dim3(nt, batch), spd::T, 0, st>>>(p, scratch, y, sy);
  return cudaGetLastError();
}

}  // namespace wmg
