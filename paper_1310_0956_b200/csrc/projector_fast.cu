// projector_fast.cu -- throughput line-intersection projector pair.
//
// Same system matrix as the reference (/root/reference/pkg/src/wmgtomo/
// geometry.py:88-128: exact ray/pixel intersection lengths, axis-aligned rays
// on a grid line belong to the higher-x / higher-y pixel) but evaluated in the
// form that is cheapest on sm_100a, with arbitrary summation order:
//
//  forward  (ray-driven): the ray is walked slab by slab along its major axis
//    (rows for |cos| >= |sin|, columns otherwise; columns are read from a
//    transposed copy of the image so every slab is a contiguous line).  In a
//    slab the ray covers the minor interval [u, u + slope] (slope in [0,1]
//    after an optional mirror), i.e. at most two pixels:
//        w(k_hi) = min(frac(u + slope) * Ls, L),  w(k_hi - 1) = L - w(k_hi)
//    u is carried in 64-bit fixed point (40 fractional bits) so the geometry is
//    exact to ~1e-9 px at every n while the data path is fp32.
//  backward (pixel-driven gather, no atomics): for each angle the pixel's
//    chord function is the trapezoid T(delta) = clamp((hw - |delta|)/(|c||s|),
//    0, 1/max(|c|,|s|)) of the detector offset delta = j - p; at most two
//    detectors are in its support.  p is evaluated in float64.
//
// Tolerance vs the float64 reference: 1e-5 relative (fp32 data), see
// tests/test_gpu_projector.py.
#include <algorithm>
#include <type_traits>

#include <cooperative_groups.h>

#include "common.cuh"

namespace wmg {
namespace fast {

template <typename T>
__device__ __forceinline__ float to_f(T v) { return (float)v; }

// float64 min / max as one DSETP + two selects (fmin / fmax on doubles are a
// NaN-aware ~7-instruction sequence on sm_100a).  A NaN x yields the bound,
// exactly as fmin(x, hi) / fmax(x, 0) do.
__device__ __forceinline__ double dmin_to(double x, double hi) { return x < hi ? x : hi; }
__device__ __forceinline__ double dmax_0(double x) { return x > 0.0 ? x : 0.0; }

template <typename R>
__device__ __forceinline__ R frac_of(long long U);

template <>
__device__ __forceinline__ float frac_of<float>(long long U) {
  // 23 high fractional bits -> [1,2) mantissa -> subtract 1
  const unsigned bits = (unsigned)((unsigned long long)U >> (kFixFrac - 23)) & 0x7FFFFFu;
  return __int_as_float(0x3F800000u | bits) - 1.0f;
}
template <>
__device__ __forceinline__ double frac_of<double>(long long U) {
  const long long m = U & ((1LL << kFixFrac) - 1);
  return (double)m * (1.0 / kFixScale);
}

// per-angle constants in the kernel's arithmetic type
template <typename R> struct Pc;
template <> struct Pc<float> {
  static __device__ __forceinline__ float L(const AngleParams& P) { return P.Lf; }
  static __device__ __forceinline__ float Ls(const AngleParams& P) { return P.Lsf; }
  static __device__ __forceinline__ float hw(const AngleParams& P) { return P.hwf; }
  static __device__ __forceinline__ float ic(const AngleParams& P) { return P.inv_csf; }
};
template <> struct Pc<double> {
  static __device__ __forceinline__ double L(const AngleParams& P) { return P.L; }
  static __device__ __forceinline__ double Ls(const AngleParams& P) { return P.Ls; }
  static __device__ __forceinline__ double hw(const AngleParams& P) { return P.hw; }
  static __device__ __forceinline__ double ic(const AngleParams& P) { return P.inv_cs; }
};

template <typename TIn, typename R>
__device__ __forceinline__ R load_px(const TIn* __restrict__ src, long long rowbase, int k, int n,
                                     int mirror) {
  if (k < 0 || k >= n) return R(0);
  const int kk = mirror ? (n - 1 - k) : k;
  return (R)__ldg(src + rowbase + kk);
}

// One thread per ray, block = consecutive detectors of one angle (blockIdx.y).
template <typename TIn, typename TOut, typename R>
__global__ void __launch_bounds__(128) fwd_kernel(GeomDev G, const TIn* __restrict__ img,
                                                  const TIn* __restrict__ imgT,
                                                  TOut* __restrict__ sino, int pitch) {
  const int a = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= G.d) return;
  const AngleParams& P = G.ang[a];
  const int n = G.n;
  const TIn* __restrict__ src = P.major ? imgT : img;
  const double off = (double)j - (double)(G.d - 1) * 0.5;
  const double u0 = P.u0 + off * P.du;   // minor coordinate at the start of slab 0
  const double slope = P.slope;
  int r0 = 0, r1 = n - 1;
  if (slope > 0.0) {
    const double ra = floor((-1.0 - u0) / slope) - 1.0;
    const double rb = ceil(((double)n + 1.0 - u0) / slope) + 1.0;
    r0 = (int)fmax(ra, 0.0);
    r1 = (int)fmin(rb, (double)(n - 1));
  } else if (u0 < -1.0 || u0 > (double)n + 1.0) {
    r1 = -1;
  }
  const R L = Pc<R>::L(P), Ls = Pc<R>::Ls(P);
  R acc = R(0);
  if constexpr (sizeof(R) == 4) {
    // fp32 data path: 64-bit fixed-point minor coordinate (exact increments)
    const long long S = llrint(slope * kFixScale);
    long long U = llrint(u0 * kFixScale) + (long long)r0 * S;
    for (int r = r0; r <= r1; ++r) {
      const long long Uh = U + S;
      const int k = (int)(Uh >> kFixFrac);
      const R f = frac_of<R>(Uh);
      R wh = f * Ls;
      wh = (wh < L) ? wh : L;              // NaN (0*inf, ray on a grid line) -> L
      const R wl = L - wh;
      const long long rowbase = (long long)r * pitch;
      acc += wh * load_px<TIn, R>(src, rowbase, k, n, P.mirror);
      acc += wl * load_px<TIn, R>(src, rowbase, k - 1, n, P.mirror);
      U = Uh;
    }
  } else {
    // fp64 arithmetic: evaluate u at every slab end directly (no drift)
    for (int r = r0; r <= r1; ++r) {
      const double uh = fma((double)(r + 1), slope, u0);
      const double fk = floor(uh);
      const int k = (int)fk;
      R wh = (uh - fk) * Ls;
      wh = (wh < L) ? wh : L;
      const R wl = L - wh;
      const long long rowbase = (long long)r * pitch;
      acc += wh * load_px<TIn, R>(src, rowbase, k, n, P.mirror);
      acc += wl * load_px<TIn, R>(src, rowbase, k - 1, n, P.mirror);
    }
  }
  sino[(long long)(G.rowmap ? G.rowmap[a] : a) * G.d + j] = (TOut)acc;
}

// One thread per pixel; all threads walk the angles in the same order.
// (row_lo, row_hi: the image rows this launch covers, default all)
template <typename TIn, typename TOut, typename R, bool kAccumulate>
__global__ void __launch_bounds__(256) bwd_kernel(GeomDev G, const TIn* __restrict__ sino,
                                                  TOut* __restrict__ img, int row_lo = 0,
                                                  int row_hi = 0x7fffffff) {
  const int n = G.n;
  const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
  const int row = row_lo + blockIdx.y * 8 + (threadIdx.x >> 5);
  if (ix >= n || row >= n || row >= row_hi) return;
  const double xc = (double)ix - (double)n * 0.5 + 0.5;
  const double yc = (double)n * 0.5 - (double)row - 0.5;
  const double dc = (double)(G.d - 1) * 0.5;
  R acc = R(0);
  for (int a = 0; a < G.m; ++a) {
    const AngleParams& P = G.ang[a];
    const double p = xc * P.c + yc * P.s + dc;   // detector-index coordinate
    const TIn* __restrict__ yrow = sino + (long long)(G.rowmap ? G.rowmap[a] : a) * G.d;
    if (P.axis) {
      const int j = (int)ceil(p - 0.5);
      if (j >= 0 && j < G.d) acc += (R)__ldg(yrow + j);
      continue;
    }
    const double fl = floor(p - (double)P.hw);
    const int j0 = (int)fl + 1;
    const R d0 = (R)(fl + 1.0 - p);
    const R d1 = d0 + R(1);
    const R hw = Pc<R>::hw(P), ic = Pc<R>::ic(P), L = Pc<R>::L(P);
    R w0 = (hw - fabs(d0)) * ic;
    R w1 = (hw - fabs(d1)) * ic;
    w0 = w0 < R(0) ? R(0) : (w0 > L ? L : w0);
    w1 = w1 < R(0) ? R(0) : (w1 > L ? L : w1);
    if (j0 >= 0 && j0 < G.d) acc += w0 * (R)__ldg(yrow + j0);
    if (j0 + 1 >= 0 && j0 + 1 < G.d) acc += w1 * (R)__ldg(yrow + j0 + 1);
  }
  const long long p = (long long)row * n + ix;
  if (kAccumulate)
    img[p] = (TOut)((R)img[p] + acc);
  else
    img[p] = (TOut)acc;
}

// Small grids (n <= 512, e.g. config 1 and the WMG node applies) expose too
// little parallelism for one thread per ray / pixel: 65k rays of 256 serial
// slabs leave the SMs latency-bound.  The split kernels give each ray (pixel)
// kSplit threads -- consecutive slab (angle) segments -- and reduce the
// partial sums in shared memory in segment order (deterministic).
constexpr int kSplit = 8;
constexpr int kSplitAxis = 32;   // slab segments per ray of the two axis-aligned angles
constexpr int kSplitF = 4;   // slab segments per ray of the padded-plane fp64 forward (8: same single-image time, 10 % slower sibling batches)
constexpr int kFwdAG = 4;    // adjacent angles per symmetric-forward block

// block (32 rays, kSplit slab segments); grid (ceil(d/32), m)
template <typename TIn, typename TOut, typename R>
// blockIdx.z selects one image of a batch (images n*n apart, sinograms bs_sino)
__global__ void __launch_bounds__(32 * kSplit) fwd_split_kernel(GeomDev G,
                                                                const TIn* __restrict__ img,
                                                                const TIn* __restrict__ imgT,
                                                                TOut* __restrict__ sino,
                                                                long long bs_sino) {
  __shared__ R part[kSplit][33];
  {
    const long long zi = (long long)blockIdx.z * G.n * G.n;
    img += zi;
    imgT += zi;
    sino += (long long)blockIdx.z * bs_sino;
  }
  const int a = blockIdx.y;
  const int lane = threadIdx.x, seg = threadIdx.y;
  const int j = blockIdx.x * 32 + lane;
  const int n = G.n;
  R acc = R(0);
  if (j < G.d) {
    const AngleParams& P = G.ang[a];
    const TIn* __restrict__ src = P.major ? imgT : img;
    const double off = (double)j - (double)(G.d - 1) * 0.5;
    const double u0 = P.u0 + off * P.du;
    const double slope = P.slope;
    int r0 = 0, r1 = n - 1;
    if (slope > 0.0) {
      const double ra = floor((-1.0 - u0) / slope) - 1.0;
      const double rb = ceil(((double)n + 1.0 - u0) / slope) + 1.0;
      r0 = (int)fmax(ra, 0.0);
      r1 = (int)fmin(rb, (double)(n - 1));
    } else if (u0 < -1.0 || u0 > (double)n + 1.0) {
      r1 = -1;
    }
    const int len = r1 - r0 + 1;
    const int rs = r0 + (len > 0 ? (len * seg) / kSplit : 0);
    const int re = r0 + (len > 0 ? (len * (seg + 1)) / kSplit : 0) - 1;
    const R L = Pc<R>::L(P), Ls = Pc<R>::Ls(P);
    if constexpr (sizeof(R) == 4) {
      const long long S = llrint(slope * kFixScale);
      long long U = llrint(u0 * kFixScale) + (long long)rs * S;
      for (int r = rs; r <= re; ++r) {
        const long long Uh = U + S;
        const int k = (int)(Uh >> kFixFrac);
        R wh = frac_of<R>(Uh) * Ls;
        wh = (wh < L) ? wh : L;
        const long long rowbase = (long long)r * n;
        acc += wh * load_px<TIn, R>(src, rowbase, k, n, P.mirror);
        acc += (L - wh) * load_px<TIn, R>(src, rowbase, k - 1, n, P.mirror);
        U = Uh;
      }
    } else {
      for (int r = rs; r <= re; ++r) {
        const double uh = fma((double)(r + 1), slope, u0);
        const double fk = floor(uh);
        const int k = (int)fk;
        R wh = (uh - fk) * Ls;
        wh = (wh < L) ? wh : L;
        const long long rowbase = (long long)r * n;
        acc += wh * load_px<TIn, R>(src, rowbase, k, n, P.mirror);
        acc += (L - wh) * load_px<TIn, R>(src, rowbase, k - 1, n, P.mirror);
      }
    }
  }
  part[seg][lane] = acc;
  __syncthreads();
  if (seg == 0 && j < G.d) {
    R s = part[0][lane];
#pragma unroll
    for (int q = 1; q < kSplit; ++q) s += part[q][lane];
    sino[(long long)(G.rowmap ? G.rowmap[a] : a) * G.d + j] = (TOut)s;
  }
}

// block (32 pixels of one row, kSplit angle chunks); grid (ceil(n/32), n)
template <typename TIn, typename TOut, typename R, bool kAccumulate>
__global__ void __launch_bounds__(32 * kSplit) bwd_split_kernel(GeomDev G,
                                                                const TIn* __restrict__ sino,
                                                                TOut* __restrict__ img,
                                                                long long bs_sino) {
  __shared__ R part[kSplit][33];
  sino += (long long)blockIdx.z * bs_sino;
  img += (long long)blockIdx.z * G.n * G.n;
  const int n = G.n;
  const int lane = threadIdx.x, seg = threadIdx.y;
  const int ix = blockIdx.x * 32 + lane;
  const int row = blockIdx.y;
  const double xc = (double)ix - (double)n * 0.5 + 0.5;
  const double yc = (double)n * 0.5 - (double)row - 0.5;
  const double dc = (double)(G.d - 1) * 0.5;
  const int a0 = (G.m * seg) / kSplit, a1 = (G.m * (seg + 1)) / kSplit;
  R acc = R(0);
  if (ix < n) {
    for (int a = a0; a < a1; ++a) {
      const AngleParams& P = G.ang[a];
      const double p = xc * P.c + yc * P.s + dc;
      const TIn* __restrict__ yrow = sino + (long long)(G.rowmap ? G.rowmap[a] : a) * G.d;
      if (P.axis) {
        const int j = (int)ceil(p - 0.5);
        if (j >= 0 && j < G.d) acc += (R)__ldg(yrow + j);
        continue;
      }
      const double fl = floor(p - (double)P.hw);
      const int j0 = (int)fl + 1;
      const R d0 = (R)(fl + 1.0 - p);
      const R d1 = d0 + R(1);
      const R hw = Pc<R>::hw(P), ic = Pc<R>::ic(P), L = Pc<R>::L(P);
      R w0 = (hw - fabs(d0)) * ic;
      R w1 = (hw - fabs(d1)) * ic;
      w0 = w0 < R(0) ? R(0) : (w0 > L ? L : w0);
      w1 = w1 < R(0) ? R(0) : (w1 > L ? L : w1);
      if (j0 >= 0 && j0 < G.d) acc += w0 * (R)__ldg(yrow + j0);
      if (j0 + 1 >= 0 && j0 + 1 < G.d) acc += w1 * (R)__ldg(yrow + j0 + 1);
    }
  }
  part[seg][lane] = acc;
  __syncthreads();
  if (seg == 0 && ix < n) {
    R s = part[0][lane];
#pragma unroll
    for (int q = 1; q < kSplit; ++q) s += part[q][lane];
    const long long p = (long long)row * n + ix;
    if (kAccumulate)
      img[p] = (TOut)((R)img[p] + s);
    else
      img[p] = (TOut)s;
  }
}

template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, T* __restrict__ out, int n) {
  __shared__ T tile[32][33];
  in += (long long)blockIdx.z * n * n;     // batch of images
  out += (long long)blockIdx.z * n * n;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = by + i, c = bx + threadIdx.x;
    if (r < n && c < n) tile[i][threadIdx.x] = in[(long long)r * n + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = bx + i, c = by + threadIdx.x;
    if (r < n && c < n) out[(long long)r * n + c] = tile[threadIdx.x][i];
  }
}


// ===========================================================================
// v2 fp32 kernels (the throughput path)
// ===========================================================================

// v2 fixed point: 64-bit with 32 fractional bits, so the integer part is the
// high register and the fraction the low register.  Slope quantisation drift
// over n slabs <= n * 2^-33 px (< 5e-7 px at n = 4096).
constexpr double kQ32 = 4294967296.0;   // 2^32

// low word -> float in [1, 2): 1 + top 23 fraction bits
__device__ __forceinline__ float frac1(unsigned lo) {
  return __int_as_float(0x3F800000u | (lo >> 9));
}
__device__ __forceinline__ int hi32(long long v) { return (int)((unsigned long long)v >> 32); }

// Zero-padded copies for the forward slab walk: P[r][M + k] = img[r][k] and
// PT[c][M + k] = img[k][c], pitch n + 2M, margins zero.
template <typename T>
__global__ void pad_transpose_kernel(const T* __restrict__ in, float* __restrict__ P,
                                     float* __restrict__ PT, int n) {
  __shared__ float tile[32][33];
  const int pitch = n + 2 * kPadMargin;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;   // column / row of the input tile
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = by + i, c = bx + threadIdx.x;
    float v = 0.0f;
    if (r < n && c < n) {
      v = (float)in[(long long)r * n + c];
      P[(long long)r * pitch + kPadMargin + c] = v;
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = bx + i, r = by + threadIdx.x;
    if (r < n && c < n) PT[(long long)c * pitch + kPadMargin + r] = tile[threadIdx.x][i];
  }
  // margins (written by the blocks of the first / last tile column)
  if (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) {
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int r = by + i;
      if (r >= n) continue;
      for (int k = threadIdx.x; k < kPadMargin; k += 32) {
        if (blockIdx.x == 0) {
          P[(long long)r * pitch + k] = 0.0f;
          PT[(long long)r * pitch + k] = 0.0f;
        }
        if (blockIdx.x == gridDim.x - 1) {
          P[(long long)r * pitch + kPadMargin + n + k] = 0.0f;
          PT[(long long)r * pitch + kPadMargin + n + k] = 0.0f;
        }
      }
    }
  }
}

// Mirror-packed padded planes for the symmetric forward: PM[r][M + k] =
// (img[r][k], img[r][n-1-k]) and PMT[c][M + r] = (img[r][c], img[n-1-r][c]),
// float2, margins zero.  A ray's pixel pair in an image and in its x-mirror
// image (k-1, k) / (n-1-k, n-k) then comes from two 64-bit loads of one plane
// (PM[k-1], PM[k]) instead of four 32-bit loads.
template <typename T>
__global__ void pad_mirror_kernel(const T* __restrict__ in, float2* __restrict__ PM,
                                  float2* __restrict__ PMT, int n) {
  __shared__ float tile[32][33];
  __shared__ float tilem[32][33];    // the column-mirrored input tile
  const int pitch = n + 2 * kPadMargin;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = by + i, c = bx + threadIdx.x;
    float v = 0.0f, vm = 0.0f, vr = 0.0f;
    if (r < n && c < n) {
      v = (float)in[(long long)r * n + c];
      vm = (float)in[(long long)r * n + (n - 1 - c)];
      vr = (float)in[(long long)(n - 1 - r) * n + c];
      PM[(long long)r * pitch + kPadMargin + c] = make_float2(v, vm);
    }
    tile[i][threadIdx.x] = v;
    tilem[i][threadIdx.x] = vr;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = bx + i, r = by + threadIdx.x;
    if (r < n && c < n)
      PMT[(long long)c * pitch + kPadMargin + r] =
          make_float2(tile[threadIdx.x][i], tilem[threadIdx.x][i]);
  }
  if (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) {
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int r = by + i;
      if (r >= n) continue;
      for (int k = threadIdx.x; k < kPadMargin; k += 32) {
        const float2 z = make_float2(0.0f, 0.0f);
        if (blockIdx.x == 0) {
          PM[(long long)r * pitch + k] = z;
          PMT[(long long)r * pitch + k] = z;
        }
        if (blockIdx.x == gridDim.x - 1) {
          PM[(long long)r * pitch + kPadMargin + n + k] = z;
          PMT[(long long)r * pitch + kPadMargin + n + k] = z;
        }
      }
    }
  }
}

// Forward: one thread per ray, 128 consecutive detectors of one angle per
// block.  Each warp walks the union of its lanes' slab ranges; the zero margin
// makes out-of-grid reads harmless, so the inner loop has no branches.
// ES = element stride of the planes (1: P / PT; 2: the x-component of the
// mirror-packed float2 planes PM / PMT of the symmetric forward)
template <typename TOut, int ES = 1>
__global__ void __launch_bounds__(128) fwd_v2_kernel(GeomDev G, const float* __restrict__ P,
                                                     const float* __restrict__ PT,
                                                     TOut* __restrict__ sino) {
  const int a = blockIdx.y;
  const int j = blockIdx.x * 128 + threadIdx.x;
  const AngleParams& A = G.ang[a];
  const int n = G.n;
  const int pitch = n + 2 * kPadMargin;
  const double off = (double)j - (double)(G.d - 1) * 0.5;
  const double u0 = A.u0 + off * A.du;
  const double slope = A.slope;
  int r0 = 0, r1 = n - 1;
  if (j >= G.d) {
    r0 = n; r1 = -1;
  } else if (slope > 0.0) {
    const double ra = floor((-1.0 - u0) / slope) - 1.0;
    const double rb = ceil(((double)n + 1.0 - u0) / slope) + 1.0;
    r0 = (int)fmin(fmax(ra, 0.0), (double)n);
    r1 = (int)fmax(fmin(rb, (double)(n - 1)), -1.0);
  } else if (u0 < -1.0 || u0 > (double)n + 1.0) {
    r0 = n; r1 = -1;
  }
  const int rw0 = __reduce_min_sync(0xffffffffu, r0);
  const int rw1 = __reduce_max_sync(0xffffffffu, r1);
  float acc = 0.0f;
  if (rw0 <= rw1) {
    const float* __restrict__ src = (A.major ? PT : P) + ES * kPadMargin;
    const long long S = llrint(slope * kQ32);
    long long U = llrint(u0 * kQ32) + (long long)rw0 * S;
    const float L = A.Lf, Ls = A.Lsf;
    const int mir = A.mirror;
    // mirrored minor axis: pixel k lives at column n-1-k; walk a pointer that
    // moves by -1 per unit of k instead (same instruction count)
    const long long rowstep = pitch;
    long long rowoff = (long long)rw0 * rowstep;
    if (!mir) {
#pragma unroll 4
      for (int r = rw0; r <= rw1; ++r) {
        U += S;
        const int k = hi32(U);
        const float f = frac1((unsigned)U);
        const float wh = fminf(fmaf(f, Ls, -Ls), L);    // NaN (axis: inf-inf) -> L
        const float* p = src + ES * (rowoff + k);
        const float v1 = __ldg(p), v0 = __ldg(p - ES);
        acc = fmaf(L, v0, acc);
        acc = fmaf(wh, v1 - v0, acc);
        rowoff += rowstep;
      }
    } else {
#pragma unroll 4
      for (int r = rw0; r <= rw1; ++r) {
        U += S;
        const int k = hi32(U);
        const float f = frac1((unsigned)U);
        const float wh = fminf(fmaf(f, Ls, -Ls), L);
        const float* p = src + ES * (rowoff + (n - 1 - k));
        const float v1 = __ldg(p), v0 = __ldg(p + ES);
        acc = fmaf(L, v0, acc);
        acc = fmaf(wh, v1 - v0, acc);
        rowoff += rowstep;
      }
    }
  }
  if (j < G.d) sino[(long long)(G.rowmap ? G.rowmap[a] : a) * G.d + j] = (TOut)acc;
}

// fwd_v2_kernel with each ray's slab range split over kSplit segments
// (threadIdx.y), partial sums reduced in shared memory in segment order: for
// the two axis-aligned angles of a symmetric set, which alone launch too few
// rays to fill the GPU (their walk is n slabs long).
template <typename TOut, int ES = 1, int KS = kSplit>
__global__ void __launch_bounds__(32 * KS) fwd_v2_split_kernel(GeomDev G,
                                                                   const float* __restrict__ P,
                                                                   const float* __restrict__ PT,
                                                                   TOut* __restrict__ sino) {
  __shared__ float part[KS][33];
  const int a = blockIdx.y, lane = threadIdx.x, seg = threadIdx.y;
  const int j = blockIdx.x * 32 + lane;
  const AngleParams& A = G.ang[a];
  const int n = G.n;
  const int pitch = n + 2 * kPadMargin;
  const double off = (double)j - (double)(G.d - 1) * 0.5;
  const double u0 = A.u0 + off * A.du;
  const double slope = A.slope;
  int r0 = 0, r1 = n - 1;
  if (j >= G.d) {
    r0 = n; r1 = -1;
  } else if (slope > 0.0) {
    const double ra = floor((-1.0 - u0) / slope) - 1.0;
    const double rb = ceil(((double)n + 1.0 - u0) / slope) + 1.0;
    r0 = (int)fmin(fmax(ra, 0.0), (double)n);
    r1 = (int)fmax(fmin(rb, (double)(n - 1)), -1.0);
  } else if (u0 < -1.0 || u0 > (double)n + 1.0) {
    r0 = n; r1 = -1;
  }
  const int rw0 = __reduce_min_sync(0xffffffffu, r0);
  const int rw1 = __reduce_max_sync(0xffffffffu, r1);
  float acc = 0.0f;
  if (rw0 <= rw1) {
    const int len = rw1 - rw0 + 1;
    const int rs = rw0 + (len * seg) / KS;
    const int re = rw0 + (len * (seg + 1)) / KS - 1;
    const float* __restrict__ src = (A.major ? PT : P) + ES * kPadMargin;
    const long long S = llrint(slope * kQ32);
    long long U = llrint(u0 * kQ32) + (long long)rs * S;
    const float L = A.Lf, Ls = A.Lsf;
    long long rowoff = (long long)rs * pitch;
    if (!A.mirror) {
#pragma unroll 4
      for (int r = rs; r <= re; ++r) {
        U += S;
        const int k = hi32(U);
        const float f = frac1((unsigned)U);
        const float wh = fminf(fmaf(f, Ls, -Ls), L);    // NaN (axis: inf-inf) -> L
        const float* p = src + ES * (rowoff + k);
        const float v1 = __ldg(p), v0 = __ldg(p - ES);
        acc = fmaf(L, v0, acc);
        acc = fmaf(wh, v1 - v0, acc);
        rowoff += pitch;
      }
    } else {
#pragma unroll 4
      for (int r = rs; r <= re; ++r) {
        U += S;
        const int k = hi32(U);
        const float f = frac1((unsigned)U);
        const float wh = fminf(fmaf(f, Ls, -Ls), L);
        const float* p = src + ES * (rowoff + (n - 1 - k));
        const float v1 = __ldg(p), v0 = __ldg(p + ES);
        acc = fmaf(L, v0, acc);
        acc = fmaf(wh, v1 - v0, acc);
        rowoff += pitch;
      }
    }
  }
  part[seg][lane] = acc;
  __syncthreads();
  if (seg == 0 && j < G.d) {
    float sum = part[0][lane];
#pragma unroll
    for (int q = 1; q < KS; ++q) sum += part[q][lane];
    sino[(long long)(G.rowmap ? G.rowmap[a] : a) * G.d + j] = (TOut)sum;
  }
}

// Backward: 32 x 32 pixel tile per block (128 threads; warp w owns rows
// 8w..8w+7, lane = column).  Angles are processed in chunks of 32: the
// detector window of every angle is staged in shared memory as pairs
// (y[j], y[j+1]) and the fixed-point detector coordinate of every lane is
// tabulated, so the per-(pixel, angle) work is integer adds, one LDS.64 and
// the branch-free trapezoid weights.
constexpr int kBwdTile = 32;
constexpr int kBwdChunk = 32;
constexpr int kBwdWin = 64;

template <typename TIn, typename TOut, bool kAccumulate>
__global__ void __launch_bounds__(128) bwd_v2_kernel(GeomDev G, const TIn* __restrict__ sino,
                                                     TOut* __restrict__ img,
                                                     int row_tile0 = 0) {
  __shared__ float2 win[kBwdChunk][kBwdWin];
  __shared__ long long qx[kBwdChunk][kBwdTile];
  __shared__ long long qhead[kBwdChunk];
  __shared__ int jlo_s[kBwdChunk];
  const int n = G.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col0 = blockIdx.x * kBwdTile, row0 = (blockIdx.y + row_tile0) * kBwdTile;
  const double half = (double)n * 0.5, dc = (double)(G.d - 1) * 0.5;
  const double xc0 = (double)col0 - half + 0.5;           // pixel-centre x of the tile origin
  const double yc0 = half - (double)row0 - 0.5;           // pixel-centre y
  const double bias = 1.0 / kQ32;                         // ties of axis angles go up/right
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0f;

  for (int a0 = 0; a0 < G.m; a0 += kBwdChunk) {
    const int na = min(kBwdChunk, G.m - a0);
    __syncthreads();
    if (tid < na) {
      const AngleParams& A = G.ang[a0 + tid];
      const double p0 = xc0 * A.c + yc0 * A.s + dc - A.hw - bias;
      const double t = (double)(kBwdTile - 1);
      const double pmin = p0 + fmin(0.0, t * A.c) + fmin(0.0, -t * A.s);
      const int jlo = (int)floor(pmin) - 1;
      jlo_s[tid] = jlo;
      qhead[tid] = llrint((p0 - (double)jlo) * kQ32);
    }
    __syncthreads();
    // fixed-point coordinate of every lane's column, and the windows
    for (int e = tid; e < na * kBwdTile; e += 128) {
      const int aa = e / kBwdTile, l = e % kBwdTile;
      qx[aa][l] = qhead[aa] + (long long)l * G.ang[a0 + aa].Cfix;
    }
    for (int e = tid; e < na * kBwdWin; e += 128) {
      const int aa = e / kBwdWin, t = e % kBwdWin;
      const int j = jlo_s[aa] + t;
      const int srow = G.rowmap ? G.rowmap[a0 + aa] : a0 + aa;
      const TIn* yrow = sino + (long long)srow * G.d;
      const float v0 = (j >= 0 && j < G.d) ? (float)__ldg(yrow + j) : 0.0f;
      const float v1 = (j + 1 >= 0 && j + 1 < G.d) ? (float)__ldg(yrow + j + 1) : 0.0f;
      win[aa][t] = make_float2(v0, v1);
    }
    __syncthreads();
    for (int aa = 0; aa < na; ++aa) {
      const AngleParams& A = G.ang[a0 + aa];
      const long long S = A.Sfix;
      const float ca0 = A.a0, icb = A.icb, hwic = A.hwic, w1c = A.w1c, L = A.Lf;
      long long Q = qx[aa][lane] - (long long)(8 * warp) * S;
      const float2* wrow = win[aa];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int hi = hi32(Q);
        const float f = frac1((unsigned)Q);
        const float d0 = ca0 - f;                        // delta0 = j0 - p
        const float w0 = fminf(fmaf(-fabsf(d0), icb, hwic), L);
        const float w1 = fmaxf(fmaf(f, icb, w1c), 0.0f);
        const float2 v = wrow[hi + 1];
        acc[i] = fmaf(w0, v.x, acc[i]);
        acc[i] = fmaf(w1, v.y, acc[i]);
        Q -= S;
      }
    }
  }
  const int col = col0 + lane;
  if (col < n) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = row0 + 8 * warp + i;
      if (row < n) {
        const long long p = (long long)row * n + col;
        if (kAccumulate)
          img[p] = (TOut)((float)img[p] + acc[i]);
        else
          img[p] = (TOut)acc[i];
      }
    }
  }
}


// Symmetric backprojector.  For an equiangular angle set (theta_{m-a} = pi -
// theta_a) on a square grid, the trapezoid weights of pixel p at angle a equal
// those of (i) the x-mirrored pixel at angle m-a (same detectors), (ii) the
// 180-degree rotated pixel at angle a (detectors reversed) and (iii) the
// y-mirrored pixel at angle m-a (detectors reversed).  One block owns a 32x32
// tile of the top-left quadrant and its three images; every weight evaluation
// feeds four accumulators (two packed FFMA2 per detector).  Axis-aligned
// angles (0, pi/2) are excluded: the reference's tie rule for rays on grid
// lines is not mirror symmetric, so they run through bwd_v2 afterwards.
constexpr int kSymChunk = 8;

// Warp layout: kWarp2D (default) gives each warp an 8-column x 4-row pixel block
// per step, so its 32 lanes read a detector span of 7|c| + 3|s| < 8 float4 window
// entries (mostly one 128-byte shared wavefront) instead of the 32|c| entries
// (up to four wavefronts) a 32-column row needs; each thread keeps one column
// and 4 rows spaced 8 apart.  !kWarp2D is the row layout (lane = column).
template <typename TIn, typename TOut, bool kAccumulate, bool kWarp2D = true>
__global__ void __launch_bounds__(256, 5) bwd_sym_kernel(GeomDev G, const TIn* __restrict__ sino,
                                                      TOut* __restrict__ img) {
  __shared__ float4 winA[kSymChunk][kBwdWin];   // (y_a[t], y_b[t], y_a[t+1], y_b[t+1])
  __shared__ float4 winB[kSymChunk][kBwdWin];   // same with detectors reversed
  __shared__ long long qx[kSymChunk][kBwdTile];
  __shared__ long long qhead[kSymChunk];
  __shared__ int jlo_s[kSymChunk];
  __shared__ int ang_s[kSymChunk];
  __shared__ int mir_s[kSymChunk];
  const int n = G.n, m = G.m, d = G.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col0 = blockIdx.x * kBwdTile, row0 = blockIdx.y * kBwdTile;
  const double half = (double)n * 0.5, dc = (double)(d - 1) * 0.5;
  const double xc0 = (double)col0 - half + 0.5;
  const double yc0 = half - (double)row0 - 0.5;
  const double bias = 1.0 / kQ32;
  // this thread's tile column and first row; its rows are trow + rstep * i
  const int tcol = kWarp2D ? (warp & 3) * 8 + (lane & 7) : lane;
  const int trow = kWarp2D ? (warp >> 2) * 4 + (lane >> 3) : 4 * warp;
  constexpr int rstep = kWarp2D ? 8 : 1;
  float2 accA[4], accB[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    accA[i] = make_float2(0.0f, 0.0f);
    accB[i] = make_float2(0.0f, 0.0f);
  }
  // primary angles: 1 .. m-1 except m/2 (m - 2 of them)
  for (int c0 = 0; c0 < G.n_prim; c0 += kSymChunk) {
    const int na = min(kSymChunk, G.n_prim - c0);
    __syncthreads();
    if (tid < na) {
      const int q = c0 + tid;                       // 0 .. m-3
      const int a = G.prim[q];
      ang_s[tid] = a;
      mir_s[tid] = G.mir[a] * d;     // sinogram row offset of the mirror angle
      const AngleParams& A = G.ang[a];
      const double p0 = xc0 * A.c + yc0 * A.s + dc - A.hw - bias;
      const double t = (double)(kBwdTile - 1);
      const double pmin = p0 + fmin(0.0, t * A.c) + fmin(0.0, -t * A.s);
      const int jlo = (int)floor(pmin) - 1;
      jlo_s[tid] = jlo;
      qhead[tid] = llrint((p0 - (double)jlo) * kQ32);
    }
    __syncthreads();
    for (int e = tid; e < na * kBwdTile; e += 256) {
      const int aa = e / kBwdTile, l = e % kBwdTile;
      qx[aa][l] = qhead[aa] + (long long)l * G.ang[ang_s[aa]].Cfix;
    }
    for (int e = tid; e < na * kBwdWin; e += 256) {
      const int aa = e / kBwdWin, t = e % kBwdWin;
      const int j = jlo_s[aa] + t;
      const TIn* ya = sino + ang_s[aa] * d;     // m * d < 2^31 (n <= 16384)
      const TIn* yb = sino + mir_s[aa];
      auto ld = [&](const TIn* y, int jj) -> float {
        return (jj >= 0 && jj < d) ? (float)__ldg(y + jj) : 0.0f;
      };
      winA[aa][t] = make_float4(ld(ya, j), ld(yb, j), ld(ya, j + 1), ld(yb, j + 1));
      const int r0 = d - 1 - j, r1 = d - 2 - j;
      winB[aa][t] = make_float4(ld(ya, r0), ld(yb, r0), ld(ya, r1), ld(yb, r1));
    }
    __syncthreads();
    for (int aa = 0; aa < na; ++aa) {
      const AngleParams& A = G.ang[ang_s[aa]];
      const long long S = A.Sfix;
      const float ca0 = A.a0, icb = A.icb, hwic = A.hwic, w1c = A.w1c, L = A.Lf;
      long long Q = qx[aa][tcol] - (long long)trow * S;
      const long long SS = (long long)rstep * S;
      const float4* wa = winA[aa];
      const float4* wb = winB[aa];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int hi = hi32(Q);
        const float f = frac1((unsigned)Q);
        const float d0 = ca0 - f;
        const float w0 = fminf(fmaf(-fabsf(d0), icb, hwic), L);
        const float w1 = fmaxf(fmaf(f, icb, w1c), 0.0f);
        const float2 W0 = make_float2(w0, w0), W1 = make_float2(w1, w1);
        const float4 va = wa[hi + 1];
        const float4 vb = wb[hi + 1];
        accA[i] = __ffma2_rn(W0, make_float2(va.x, va.y), accA[i]);
        accA[i] = __ffma2_rn(W1, make_float2(va.z, va.w), accA[i]);
        accB[i] = __ffma2_rn(W0, make_float2(vb.x, vb.y), accB[i]);
        accB[i] = __ffma2_rn(W1, make_float2(vb.z, vb.w), accB[i]);
        Q -= SS;
      }
    }
  }
  const int col = col0 + tcol;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = row0 + trow + rstep * i;
    const long long p1 = (long long)row * n + col;                       // (p, a)
    const long long p2 = (long long)row * n + (n - 1 - col);             // x-mirror, m-a
    const long long p3 = (long long)(n - 1 - row) * n + (n - 1 - col);   // rotation, a rev
    const long long p4 = (long long)(n - 1 - row) * n + col;             // y-mirror, m-a rev
    if (kAccumulate) {
      img[p1] = (TOut)((float)img[p1] + accA[i].x);
      img[p2] = (TOut)((float)img[p2] + accA[i].y);
      img[p3] = (TOut)((float)img[p3] + accB[i].x);
      img[p4] = (TOut)((float)img[p4] + accB[i].y);
    } else {
      img[p1] = (TOut)accA[i].x;
      img[p2] = (TOut)accA[i].y;
      img[p3] = (TOut)accB[i].x;
      img[p4] = (TOut)accB[i].y;
    }
  }
}


// Symmetric backprojector, run layout (default).  Same four-image weight
// sharing as bwd_sym_kernel, but lane = tile column and every thread owns R
// CONSECUTIVE rows.  Going one row down moves the detector coordinate by
// -sin(theta) in (-1, 0), so the detector pair (j, j+1) of the next row is
// either the same pair or (j-1, j): the thread carries the pair in registers
// and loads only the new lower detector per row -- one float2 (y_a, y_b) and
// one reversed float2 per (pixel, angle) for four images, half the shared
// wavefronts of the float4 windows.  A half-warp is 16 consecutive columns of
// one row: its detector indices span <= 16 consecutive entries, so the LDS.64
// are conflict-free (2 wavefronts each).  Tile: 32 columns x 8R rows.
//
// kCluster (small grids, where the quadrant has too few tiles to fill the
// SMs): the nsplit CTAs of a tile form a thread-block cluster along z, each
// walking a contiguous slice of the primary angles; the partial tiles are then
// summed over the cluster ranks in rank order through DSMEM (each CTA reduces
// and stores a 1/nsplit share of the tile) -- deterministic, no global scratch.
template <typename TIn, typename TOut, bool kAccumulate, int R, bool kCluster = false>
__global__ void __launch_bounds__(256, R == 4 ? 5 : (sizeof(TOut) == 4 ? 4 : 3))
bwd_symrun_kernel(GeomDev G,
                                                            const TIn* __restrict__ sino,
                                                            TOut* __restrict__ img,
                                                            int nsplit = 1) {
  constexpr int TR = 8 * R;                  // tile rows
  constexpr int WIN = R == 4 ? 64 : 96;      // window entries (>= span + 3)
  constexpr int OFF = kSymChunk * WIN;       // winB - winA (float2 entries)
  // win[0][aa][t] = (y_a[jlo+t], y_b[jlo+t]); win[1]: same at detector d-1-(jlo+t)
  __shared__ float2 win[2][kSymChunk][WIN];
  __shared__ long long qx[kSymChunk][kBwdTile];
  __shared__ float4 wc_s[kSymChunk];         // (a0, icb, hwic, w1c)
  __shared__ float2 ls_s[kSymChunk];         // (L, low word of S as bits)
  __shared__ long long qhead[kSymChunk];
  __shared__ int jlo_s[kSymChunk];
  __shared__ int ang_s[kSymChunk];
  __shared__ int mir_s[kSymChunk];
  const int n = G.n, d = G.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col0 = blockIdx.x * kBwdTile, row0 = blockIdx.y * TR;
  const double half = (double)n * 0.5, dc = (double)(d - 1) * 0.5;
  const double xc0 = (double)col0 - half + 0.5;
  const double yc0 = half - (double)row0 - 0.5;
  const double bias = 1.0 / kQ32;
  const int trow = warp * R;
  float2 accA[R], accB[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    accA[i] = make_float2(0.0f, 0.0f);
    accB[i] = make_float2(0.0f, 0.0f);
  }
  const int rank = kCluster ? (int)(blockIdx.z % nsplit) : 0;
  if (kCluster) {
    const long long item = blockIdx.z / nsplit;
    sino += item * G.m * d;
    img += item * n * n;
  }
  const int q_begin = kCluster ? (int)((long long)G.n_prim * rank / nsplit) : 0;
  const int q_end = kCluster ? (int)((long long)G.n_prim * (rank + 1) / nsplit) : G.n_prim;
  for (int c0 = q_begin; c0 < q_end; c0 += kSymChunk) {
    const int na = min(kSymChunk, q_end - c0);
    __syncthreads();
    if (tid < na) {
      const int q = c0 + tid;
      const int a = G.prim[q];
      ang_s[tid] = a;
      mir_s[tid] = G.mir[a] * d;
      const AngleParams& A = G.ang[a];
      const double p0 = xc0 * A.c + yc0 * A.s + dc - A.hw - bias;
      const double pmin = p0 + fmin(0.0, (double)(kBwdTile - 1) * A.c) +
                          fmin(0.0, -(double)(TR - 1) * A.s);
      const int jlo = (int)floor(pmin) - 1;
      jlo_s[tid] = jlo;
      qhead[tid] = llrint((p0 - (double)jlo) * kQ32);
      wc_s[tid] = make_float4(A.a0, A.icb, A.hwic, A.w1c);
      // 0 < sin < 1 for every non-axis angle: S < 2^32, one word
      ls_s[tid] = make_float2(A.Lf, __uint_as_float((unsigned)A.Sfix));
    }
    __syncthreads();
    for (int e = tid; e < na * kBwdTile; e += 256) {
      const int aa = e / kBwdTile, l = e % kBwdTile;
      qx[aa][l] = qhead[aa] + (long long)l * G.ang[ang_s[aa]].Cfix;
    }
    for (int e = tid; e < na * WIN; e += 256) {
      const int aa = e / WIN, t = e % WIN;
      const int j = jlo_s[aa] + t;
      const TIn* ya = sino + ang_s[aa] * d;
      const TIn* yb = sino + mir_s[aa];
      auto ld = [&](const TIn* y, int jj) -> float {
        return (jj >= 0 && jj < d) ? (float)__ldg(y + jj) : 0.0f;
      };
      win[0][aa][t] = make_float2(ld(ya, j), ld(yb, j));
      const int r0 = d - 1 - j;
      win[1][aa][t] = make_float2(ld(ya, r0), ld(yb, r0));
    }
    __syncthreads();
    for (int aa = 0; aa < na; ++aa) {
      const float4 wc = wc_s[aa];
      const float2 ls = ls_s[aa];
      const float ca0 = wc.x, icb = wc.y, hwic = wc.z, w1c = wc.w, L = ls.x;
      const unsigned Slo = __float_as_uint(ls.y);
      const long long Q = qx[aa][lane] - (long long)trow * (long long)Slo;
      unsigned lo = (unsigned)Q;
      const float2* pw = &win[0][aa][hi32(Q) + 1];   // first detector of the pair
      float2 fa = pw[0], sa = pw[1];
      float2 fb = pw[OFF], sb = pw[OFF + 1];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (i > 0) {
          const unsigned lo2 = lo - Slo;
          const bool moved = lo2 > lo;   // borrow: the pair slid down one detector
          lo = lo2;
          pw -= moved ? 1 : 0;
          sa = moved ? fa : sa;
          sb = moved ? fb : sb;
          fa = pw[0];
          fb = pw[OFF];
        }
        const float f = frac1(lo);
        const float d0 = ca0 - f;
        const float w0 = fminf(fmaf(-fabsf(d0), icb, hwic), L);
        const float w1 = fmaxf(fmaf(f, icb, w1c), 0.0f);
        const float2 W0 = make_float2(w0, w0), W1 = make_float2(w1, w1);
        accA[i] = __ffma2_rn(W0, fa, accA[i]);
        accA[i] = __ffma2_rn(W1, sa, accA[i]);
        accB[i] = __ffma2_rn(W0, fb, accB[i]);
        accB[i] = __ffma2_rn(W1, sb, accB[i]);
      }
    }
  }
  if constexpr (kCluster) {
    // partial tile -> shared memory as [slot = 2 i + (A|B)][thread]; rank r
    // sums elements [E r / nsplit, E (r + 1) / nsplit) over the ranks in order
    namespace cg = cooperative_groups;
    constexpr int E = 2 * R * 256;
    __shared__ float2 part[E];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      part[(2 * i) * 256 + tid] = accA[i];
      part[(2 * i + 1) * 256 + tid] = accB[i];
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int e0 = E * rank / nsplit, e1 = E * (rank + 1) / nsplit;
    for (int e = e0 + tid; e < e1; e += 256) {
      float2 v = cl.map_shared_rank(part, 0)[e];
      for (int z = 1; z < nsplit; ++z) {
        const float2 u = cl.map_shared_rank(part, z)[e];
        v.x += u.x;
        v.y += u.y;
      }
      const int slot = e >> 8, src = e & 255;
      const int row = row0 + (src >> 5) * R + (slot >> 1), col = col0 + (src & 31);
      long long pa, pb;
      if ((slot & 1) == 0) {
        pa = (long long)row * n + col;                          // (p, a)
        pb = (long long)row * n + (n - 1 - col);                // x-mirror, m-a
      } else {
        pa = (long long)(n - 1 - row) * n + (n - 1 - col);      // rotation, a rev
        pb = (long long)(n - 1 - row) * n + col;                // y-mirror, m-a rev
      }
      if (kAccumulate) {
        img[pa] = (TOut)((float)img[pa] + v.x);
        img[pb] = (TOut)((float)img[pb] + v.y);
      } else {
        img[pa] = (TOut)v.x;
        img[pb] = (TOut)v.y;
      }
    }
    cl.sync();   // peers' shared memory must outlive the remote reads
  } else {
    const int col = col0 + lane;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int row = row0 + trow + i;
      const long long p1 = (long long)row * n + col;                       // (p, a)
      const long long p2 = (long long)row * n + (n - 1 - col);             // x-mirror, m-a
      const long long p3 = (long long)(n - 1 - row) * n + (n - 1 - col);   // rotation, a rev
      const long long p4 = (long long)(n - 1 - row) * n + col;             // y-mirror, m-a rev
      if (kAccumulate) {
        img[p1] = (TOut)((float)img[p1] + accA[i].x);
        img[p2] = (TOut)((float)img[p2] + accA[i].y);
        img[p3] = (TOut)((float)img[p3] + accB[i].x);
        img[p4] = (TOut)((float)img[p4] + accB[i].y);
      } else {
        img[p1] = (TOut)accA[i].x;
        img[p2] = (TOut)accA[i].y;
        img[p3] = (TOut)accB[i].x;
        img[p4] = (TOut)accB[i].y;
      }
    }
  }
}

// Eight-image backprojector (transposition-closed symmetric sets: with every
// theta in (0, pi/4) also pi/2 - theta).  Pixel (x, y) at theta and the
// transposed pixel (y, x) at pi/2 - theta share the detector coordinate and the
// trapezoid (|cos|, |sin| swap), so one weight evaluation serves the four
// mirror/rotation images of bwd_symrun and their four transposes.  The
// primaries are the angles with |cos| > sin (q8; their transposed rows u1, u2
// read through windows C, D); pi/4 and 3 pi/4 run with four images (l4).
// A block owns the tile pair (tau, tau^T) of the top-left quadrant (32 x 32
// tiles, lane = column, 4 consecutive rows per thread, the run-layout window
// slide): phase 1 walks base tile tau, phase 2 base tau^T.  Each base adds its
// mirror images to its own orbit and its transposed images to the other
// tile's orbit; the two orbits are combined in shared memory (every element
// has one writer per step) and each output pixel is written once -- no
// atomics, deterministic.  Diagonal tiles (tau = tau^T) take phase 1 only.
constexpr int kS8Win = 64;
// Banded launches (pair0 >= 0): tile pairs enumerated by their smaller
// quadrant index s = min(i, j) (s = 0: qt pairs, s = 1: qt - 1, ...) and
// blockIdx.x offset by pair0.  After the pairs of s < S have run, quadrant
// row-blocks 0..S-1 -- image rows [0, 32 S) and [n - 32 S, n) -- are final,
// so a sharded backprojection can allreduce them while the rest runs.
__device__ __forceinline__ void minmajor_unrank(int lin, int qt, int& I, int& J) {
  int s = 0;
  while (lin >= qt - s) {
    lin -= qt - s;
    ++s;
  }
  I = s + lin;
  J = s;
}

template <typename TIn, typename TOut, bool kAccumulate>
__global__ void __launch_bounds__(256, 4) bwd_sym8_kernel(GeomDev G,
                                                          const TIn* __restrict__ sino,
                                                          TOut* __restrict__ img,
                                                          int pair0 = -1) {
  constexpr int R = 4;
  constexpr int OFF = kSymChunk * kS8Win;      // window stride (float2 entries)
  __shared__ float2 win[4][kSymChunk][kS8Win]; // A (a, mir a), B reversed, C, D (u1, u2)
  __shared__ long long qx[kSymChunk][kBwdTile];
  __shared__ float4 wc_s[kSymChunk];
  __shared__ float2 ls_s[kSymChunk];
  __shared__ long long qhead[kSymChunk];
  __shared__ int jlo_s[kSymChunk];
  __shared__ int rows_s[kSymChunk][4];         // a, mir a, u1, u2 (sinogram rows)
  __shared__ int rev_s[kSymChunk];
  // orbit(tau), orbit(tau^T): [2][4][32][33] floats of dynamic shared memory
  extern __shared__ float orb_dyn[];
  float(*orb)[4][kBwdTile][kBwdTile + 1] =
      reinterpret_cast<float(*)[4][kBwdTile][kBwdTile + 1]>(orb_dyn);
  const int n = G.n, d = G.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int ti, tj;
  if (pair0 < 0)
    tri_unrank(blockIdx.x, ti, tj);
  else
    minmajor_unrank(pair0 + (int)blockIdx.x, n / 64, ti, tj);
  const bool diag = ti == tj;
  const int trow = warp * R;
  const double half = (double)n * 0.5, dc = (double)(d - 1) * 0.5;
  const double bias = 1.0 / kQ32;
  float2 accA[R], accB[R], accC[R], accD[R];

  for (int phase = 0; phase < (diag ? 1 : 2); ++phase) {
    __syncthreads();   // phase 0's orbit writes before phase 1 accumulates onto them
    // base tile: rows R0.., cols C0..
    const int R0 = (phase == 0 ? ti : tj) * kBwdTile, C0 = (phase == 0 ? tj : ti) * kBwdTile;
    const double xc0 = (double)C0 - half + 0.5;
    const double yc0 = half - (double)R0 - 0.5;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      accA[i] = accB[i] = accC[i] = accD[i] = make_float2(0.0f, 0.0f);
    }
    // list 0: q8 (eight images), list 1: l4 (four images)
    for (int list = 0; list < 2; ++list) {
      const int cnt = list == 0 ? G.n_q8 : G.n_l4;
      for (int c0 = 0; c0 < cnt; c0 += kSymChunk) {
        const int na = min(kSymChunk, cnt - c0);
        __syncthreads();
        if (tid < na) {
          int a, u1 = 0, u2 = 0, rv = 0;
          if (list == 0) {
            const int* e = G.q8 + 4 * (c0 + tid);
            a = e[0]; u1 = e[1]; u2 = e[2]; rv = e[3];
          } else {
            a = G.l4[c0 + tid];
          }
          rows_s[tid][0] = a;
          rows_s[tid][1] = G.mir[a];
          rows_s[tid][2] = u1;
          rows_s[tid][3] = u2;
          rev_s[tid] = rv;
          const AngleParams& A = G.ang[a];
          const double p0 = xc0 * A.c + yc0 * A.s + dc - A.hw - bias;
          const double pmin = p0 + fmin(0.0, (double)(kBwdTile - 1) * A.c) +
                              fmin(0.0, -(double)(kBwdTile - 1) * A.s);
          const int jlo = (int)floor(pmin) - 1;
          jlo_s[tid] = jlo;
          qhead[tid] = llrint((p0 - (double)jlo) * kQ32);
          wc_s[tid] = make_float4(A.a0, A.icb, A.hwic, A.w1c);
          ls_s[tid] = make_float2(A.Lf, __uint_as_float((unsigned)A.Sfix));
        }
        __syncthreads();
        for (int e = tid; e < na * kBwdTile; e += 256) {
          const int aa = e / kBwdTile, l = e % kBwdTile;
          qx[aa][l] = qhead[aa] + (long long)l * G.ang[rows_s[aa][0]].Cfix;
        }
        const int nwin = list == 0 ? 4 : 2;
        for (int e = tid; e < na * kS8Win; e += 256) {
          const int aa = e / kS8Win, t = e % kS8Win;
          const int j = jlo_s[aa] + t, jr = d - 1 - j;
          auto ld = [&](int row, int jj) -> float {
            return (jj >= 0 && jj < d) ? (float)__ldg(sino + (long long)row * d + jj) : 0.0f;
          };
          const int ra = rows_s[aa][0], rb = rows_s[aa][1];
          win[0][aa][t] = make_float2(ld(ra, j), ld(rb, j));
          win[1][aa][t] = make_float2(ld(ra, jr), ld(rb, jr));
          if (nwin == 4) {
            const int r1 = rows_s[aa][2], r2 = rows_s[aa][3];
            const bool rv = rev_s[aa] != 0;
            const float2 dir = make_float2(ld(r1, j), ld(r2, j));
            const float2 rvs = make_float2(ld(r1, jr), ld(r2, jr));
            win[2][aa][t] = rv ? rvs : dir;
            win[3][aa][t] = rv ? dir : rvs;
          }
        }
        __syncthreads();
        for (int aa = 0; aa < na; ++aa) {
          const float4 wc = wc_s[aa];
          const float2 ls = ls_s[aa];
          const float ca0 = wc.x, icb = wc.y, hwic = wc.z, w1c = wc.w, L = ls.x;
          const unsigned Slo = __float_as_uint(ls.y);
          const long long Q = qx[aa][lane] - (long long)trow * (long long)Slo;
          unsigned lo = (unsigned)Q;
          const float2* pw = &win[0][aa][hi32(Q) + 1];
          float2 fa = pw[0], sa = pw[1], fb = pw[OFF], sb = pw[OFF + 1];
          if (list == 0) {
            float2 fc = pw[2 * OFF], sc = pw[2 * OFF + 1], fd = pw[3 * OFF], sd = pw[3 * OFF + 1];
#pragma unroll
            for (int i = 0; i < R; ++i) {
              if (i > 0) {
                const unsigned lo2 = lo - Slo;
                const bool moved = lo2 > lo;
                lo = lo2;
                pw -= moved ? 1 : 0;
                sa = moved ? fa : sa;
                sb = moved ? fb : sb;
                sc = moved ? fc : sc;
                sd = moved ? fd : sd;
                fa = pw[0];
                fb = pw[OFF];
                fc = pw[2 * OFF];
                fd = pw[3 * OFF];
              }
              const float f = frac1(lo);
              const float d0 = ca0 - f;
              const float w0 = fminf(fmaf(-fabsf(d0), icb, hwic), L);
              const float w1 = fmaxf(fmaf(f, icb, w1c), 0.0f);
              const float2 W0 = make_float2(w0, w0), W1 = make_float2(w1, w1);
              accA[i] = __ffma2_rn(W1, sa, __ffma2_rn(W0, fa, accA[i]));
              accB[i] = __ffma2_rn(W1, sb, __ffma2_rn(W0, fb, accB[i]));
              accC[i] = __ffma2_rn(W1, sc, __ffma2_rn(W0, fc, accC[i]));
              accD[i] = __ffma2_rn(W1, sd, __ffma2_rn(W0, fd, accD[i]));
            }
          } else {
#pragma unroll
            for (int i = 0; i < R; ++i) {
              if (i > 0) {
                const unsigned lo2 = lo - Slo;
                const bool moved = lo2 > lo;
                lo = lo2;
                pw -= moved ? 1 : 0;
                sa = moved ? fa : sa;
                sb = moved ? fb : sb;
                fa = pw[0];
                fb = pw[OFF];
              }
              const float f = frac1(lo);
              const float d0 = ca0 - f;
              const float w0 = fminf(fmaf(-fabsf(d0), icb, hwic), L);
              const float w1 = fmaxf(fmaf(f, icb, w1c), 0.0f);
              const float2 W0 = make_float2(w0, w0), W1 = make_float2(w1, w1);
              accA[i] = __ffma2_rn(W1, sa, __ffma2_rn(W0, fa, accA[i]));
              accB[i] = __ffma2_rn(W1, sb, __ffma2_rn(W0, fb, accB[i]));
            }
          }
        }
      }
    }
    // orbit images, local (row, col) in the base tile: 0 (r, c), 1 (r, n-1-c),
    // 2 (n-1-r, n-1-c), 3 (n-1-r, c).  The transposed images of base pixel
    // (lr, lc) are the images {0: D.x, 1: D.y, 2: C.x, 3: C.y} of pixel (lc, lr)
    // of the other tile.
    float(*own)[kBwdTile][kBwdTile + 1] = orb[phase];
    float(*oth)[kBwdTile][kBwdTile + 1] = orb[diag ? 0 : 1 - phase];
    if (phase == 0) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        own[0][trow + i][lane] = accA[i].x;
        own[1][trow + i][lane] = accA[i].y;
        own[2][trow + i][lane] = accB[i].x;
        own[3][trow + i][lane] = accB[i].y;
      }
      if (!diag) {
#pragma unroll
        for (int i = 0; i < R; ++i) {
          oth[0][lane][trow + i] = accD[i].x;
          oth[1][lane][trow + i] = accD[i].y;
          oth[2][lane][trow + i] = accC[i].x;
          oth[3][lane][trow + i] = accC[i].y;
        }
      } else {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < R; ++i) {
          oth[0][lane][trow + i] += accD[i].x;
          oth[1][lane][trow + i] += accD[i].y;
          oth[2][lane][trow + i] += accC[i].x;
          oth[3][lane][trow + i] += accC[i].y;
        }
      }
    } else {
      // own = orbit(tau^T) already holds phase 1's transposed images
#pragma unroll
      for (int i = 0; i < R; ++i) {
        own[0][trow + i][lane] += accA[i].x;
        own[1][trow + i][lane] += accA[i].y;
        own[2][trow + i][lane] += accB[i].x;
        own[3][trow + i][lane] += accB[i].y;
        oth[0][lane][trow + i] += accD[i].x;
        oth[1][lane][trow + i] += accD[i].y;
        oth[2][lane][trow + i] += accC[i].x;
        oth[3][lane][trow + i] += accC[i].y;
      }
    }
  }
  __syncthreads();
  for (int t = 0; t < (diag ? 1 : 2); ++t) {
    const int R0 = (t == 0 ? ti : tj) * kBwdTile, C0 = (t == 0 ? tj : ti) * kBwdTile;
    const float(*o)[kBwdTile][kBwdTile + 1] = orb[t];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int lr = trow + i;
      const int row = R0 + lr, col = C0 + lane;
      const long long p1 = (long long)row * n + col;
      const long long p2 = (long long)row * n + (n - 1 - col);
      const long long p3 = (long long)(n - 1 - row) * n + (n - 1 - col);
      const long long p4 = (long long)(n - 1 - row) * n + col;
      if (kAccumulate) {
        img[p1] = (TOut)((float)img[p1] + o[0][lr][lane]);
        img[p2] = (TOut)((float)img[p2] + o[1][lr][lane]);
        img[p3] = (TOut)((float)img[p3] + o[2][lr][lane]);
        img[p4] = (TOut)((float)img[p4] + o[3][lr][lane]);
      } else {
        img[p1] = (TOut)o[0][lr][lane];
        img[p2] = (TOut)o[1][lr][lane];
        img[p3] = (TOut)o[2][lr][lane];
        img[p4] = (TOut)o[3][lr][lane];
      }
    }
  }
}

// Symmetric forward.  Rays (a, j), (m-a, j), (a, d-1-j), (m-a, d-1-j) see the
// same weights on the slab-coordinate images (s, q), (s, n-1-q), (n-1-s, n-1-q),
// (n-1-s, q) of one walk (x-mirror / 180-degree rotation of the grid), so one
// thread walks a representative ray a in [1, m/2), j < ceil(d/2) and
// accumulates all four.  Representative angles are never mirrored (slope > 0).
// Block layout: kAG == 1 -> 128 consecutive rays of one angle; kAG == 4 -> the
// same 32 rays of 4 adjacent angles.  Adjacent angles walk nearly the same
// pixels slab after slab (rays of neighbouring angles through the same
// detector cross at the centre and drift apart by < 2 px per angle step at
// the image edge).  kMix (default) packs 8 rays x 4 angles into each warp, so
// one warp load touches ~2-3 sectors instead of 6-7 (32 rays span ~45 px): the
// forward is bound by L1 sector throughput, and this cuts the sector requests
// 2.3x (profiles/r1b_fwd_variants_ncu.txt).  Without kMix the 4 angles are 4
// warps that share L1 lines (2.4x less L2 traffic, little time gained).
// kSeg > 1 (small grids, where the ray groups alone do not fill the SMs):
// blockDim.y = kSeg warps-groups split the warp's slab range into kSeg
// contiguous row segments; partial sums are combined in segment order through
// shared memory (deterministic).
template <typename TOut, int kAG, bool kLock = false, bool kMix = false, bool kPM = false,
          int kSeg = 1, int kStride = 1>
__global__ void __launch_bounds__((kAG == 1 && !kMix) ? 128 : 32 * kAG * kSeg) fwd_sym_kernel(GeomDev G, const float* __restrict__ P,
                                                      const float* __restrict__ PT,
                                                      TOut* __restrict__ sino, int band_lo = 0,
                                                      int band_hi = 1 << 30, int band_acc = 0) {
  // Banded passes are chained with programmatic dependent launches: every block
  // releases the next pass at once, so that pass's blocks fill the SMs this
  // pass's last wave leaves idle; the next pass walks its own slab band (it
  // reads only the planes) and waits for this pass to be complete just before
  // it adds its partial sums to the sinogram (griddepcontrol.wait below).  Both
  // instructions are no-ops for launches without the attribute.
  asm volatile("griddepcontrol.launch_dependents;");
  int hidx, j;
  if (kAG == 1 && !kMix) {
    hidx = blockIdx.y;
    j = blockIdx.x * 128 + threadIdx.x;
  } else if (kMix) {
    // lanes = 8 rays x 4 adjacent angles: the warp's addresses span ~8 rays
    // (2-3 sectors per load instead of 6-7 for 32 rays of one angle); the warp
    // walks the union of its lanes' slab ranges (see clampk below).
    // kStride > 1: the block's kAG ray octets are kStride octets apart (kStride
    // consecutive blocks interleave over kAG * kStride octets), so no two warps
    // of a block load the same L1 lines: warps of one block that shared lines
    // at octet boundaries cost extra L1 data-pipe wavefronts (2.34 instead of
    // 2.09 per LDG.64; n = 4096 forward 16.8 -> 15.5 ms, profiles/r2s_*)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    hidx = blockIdx.y * 4 + (lane >> 3);
    j = ((blockIdx.x / kStride) * kAG * kStride + (blockIdx.x % kStride) + warp * kStride) * 8 +
        (lane & 7);
  } else {
    hidx = blockIdx.y * kAG + (threadIdx.x >> 5);
    j = blockIdx.x * 32 + (threadIdx.x & 31);
    if (!kLock && hidx >= G.n_half) return;          // whole warp
  }
  const bool hvalid = hidx < G.n_half;
  if ((kLock || kMix) && !hvalid) hidx = G.n_half - 1;   // keep barriers / warp votes whole
  const int a = G.half[hidx];
  const int b = G.mir[a];
  const int d = G.d, m = G.m, n = G.n;
  const int jh = (d + 1) / 2;
  const AngleParams& A = G.ang[a];
  const int pitch = n + 2 * kPadMargin;
  const double off = (double)j - (double)(d - 1) * 0.5;
  const double u0 = A.u0 + off * A.du;
  const double slope = A.slope;
  int r0 = 0, r1 = n - 1;
  if (j >= jh) {
    r0 = n; r1 = -1;
  } else if (slope > 0.0) {
    const double ra = floor((-1.0 - u0) / slope) - 1.0;
    const double rb = ceil(((double)n + 1.0 - u0) / slope) + 1.0;
    r0 = (int)fmin(fmax(ra, 0.0), (double)n);
    r1 = (int)fmax(fmin(rb, (double)(n - 1)), -1.0);
  } else if (u0 < -1.0 || u0 > (double)n + 1.0) {
    r0 = n; r1 = -1;
  }
  int rw0 = __reduce_min_sync(0xffffffffu, r0);
  int rw1 = __reduce_max_sync(0xffffffffu, r1);
  // slab band [band_lo, band_hi) of a banded pass (the planes' working set of
  // one pass stays L2-resident); band_acc: add to the partial sums in sino
  rw0 = max(rw0, band_lo);
  rw1 = min(rw1, band_hi - 1);
  if (kSeg > 1 && rw0 <= rw1) {   // this segment's share of the warp's slab range
    const int len = rw1 - rw0 + 1, sg = threadIdx.y;
    const int rs = rw0 + (len * sg) / kSeg;
    rw1 = rw0 + (len * (sg + 1)) / kSeg - 1;
    rw0 = rs;
  }
  if (kLock) {
    // lockstep: the block's warps (adjacent angles) walk the union slab range
    // together, so each image line is fetched into L1 once for all of them;
    // slabs outside a ray's own range read the zero margins (k clamped)
    __shared__ int s_lo, s_hi;
    if (threadIdx.x == 0) { s_lo = 0x7fffffff; s_hi = -1; }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { atomicMin(&s_lo, rw0); atomicMax(&s_hi, rw1); }
    __syncthreads();
    rw0 = s_lo;
    rw1 = s_hi;
  }
  // A warp walks the union of its lanes' slab ranges; when its lanes belong to
  // different angles (kMix) a lane's u can leave the image by more than the
  // padding (angles far apart in a shard, or of different major axis near 45
  // degrees): then k is clamped into the zero margins.  The host marks the
  // 4-angle groups where the margins suffice (GeomDev::gsafe).
  const bool clampk = kLock || (kMix && !G.gsafe[blockIdx.y]);   // block-uniform
  float2 accA = make_float2(0.0f, 0.0f);   // (s, q), (s, n-1-q)
  float2 accB = make_float2(0.0f, 0.0f);   // (n-1-s, n-1-q), (n-1-s, q)
  if (rw0 <= rw1) {
    const float* __restrict__ src = (A.major ? PT : P) + kPadMargin;
    const long long S = llrint(slope * kQ32);
    long long U = llrint(u0 * kQ32) + (long long)rw0 * S;
    const float L = A.Lf, Ls = A.Lsf;
    const float2 LL = make_float2(L, L);
    // 32-bit unsigned element offsets from one base (margin keeps them >= 0)
    unsigned rowA = (unsigned)(rw0 * pitch + kPadMargin);
    unsigned rowB = (unsigned)((n - 1 - rw0) * pitch + kPadMargin);
    const float* __restrict__ base = src - kPadMargin;
    const unsigned up = (unsigned)pitch;
    // the walk, versioned on the clamp (the flag is block-uniform)
    auto walk = [&](auto clampTag) {
      int r = rw0;
      // batches of 4 slabs: all 32 loads are issued before any is consumed
      for (; r + 3 <= rw1; r += 4) {
        if (kLock) __syncthreads();
        float2 v1A[4], v0A[4], v1B[4], v0B[4];
        float wh[4];
  #pragma unroll
        for (int q = 0; q < 4; ++q) {
          U += S;
          int k = hi32(U);
          if constexpr (decltype(clampTag)::value) k = min(max(k, 2 - kPadMargin), n + kPadMargin - 3);
          const float f = frac1((unsigned)U);
          wh[q] = fminf(fmaf(f, Ls, -Ls), L);
          const int km = n - 1 - k;
          if constexpr (kPM) {
            // mirror-packed planes: (pixel, x-mirror pixel) per 64-bit load
            const float2* b2 = reinterpret_cast<const float2*>(base);
            const float2* pA = b2 + (rowA + (unsigned)k);   // k - 1 is pA[-1]: one
            const float2* pB = b2 + (rowB + (unsigned)k);   // address per row
            const float2 a1 = __ldg(pA), a0 = __ldg(pA - 1);
            const float2 c1 = __ldg(pB), c0 = __ldg(pB - 1);
            v1A[q] = a1;
            v0A[q] = a0;
            v1B[q] = make_float2(c1.y, c1.x);
            v0B[q] = make_float2(c0.y, c0.x);
          } else {
            const float* pa1 = base + (rowA + (unsigned)k);
            const float* pa2 = base + (rowA + (unsigned)km);
            const float* pb1 = base + (rowB + (unsigned)km);
            const float* pb2 = base + (rowB + (unsigned)k);
            v1A[q] = make_float2(__ldg(pa1), __ldg(pa2));
            v0A[q] = make_float2(__ldg(pa1 - 1), __ldg(pa2 + 1));
            v1B[q] = make_float2(__ldg(pb1), __ldg(pb2));
            v0B[q] = make_float2(__ldg(pb1 + 1), __ldg(pb2 - 1));
          }
          rowA += up;
          rowB -= up;
        }
  #pragma unroll
        for (int q = 0; q < 4; ++q) {
          // (L - wh) v0 + wh v1: two packed FMAs per image pair, no subtraction
          const float2 W = make_float2(wh[q], wh[q]);
          const float wl = L - wh[q];
          const float2 WL = make_float2(wl, wl);
          accA = __ffma2_rn(WL, v0A[q], accA);
          accA = __ffma2_rn(W, v1A[q], accA);
          accB = __ffma2_rn(WL, v0B[q], accB);
          accB = __ffma2_rn(W, v1B[q], accB);
        }
      }
      for (; r <= rw1; ++r) {
        U += S;
        int k = hi32(U);
        if constexpr (decltype(clampTag)::value) k = min(max(k, 2 - kPadMargin), n + kPadMargin - 3);
        const float f = frac1((unsigned)U);
        const float wh = fminf(fmaf(f, Ls, -Ls), L);
        const float2 W = make_float2(wh, wh);
        const int km = n - 1 - k;
        float2 v1A, v0A, v1B, v0B;
        if constexpr (kPM) {
          const float2* b2 = reinterpret_cast<const float2*>(base);
          const float2* pA = b2 + (rowA + (unsigned)k);
          const float2* pB = b2 + (rowB + (unsigned)k);
          v1A = __ldg(pA);
          v0A = __ldg(pA - 1);
          const float2 c1 = __ldg(pB), c0 = __ldg(pB - 1);
          v1B = make_float2(c1.y, c1.x);
          v0B = make_float2(c0.y, c0.x);
        } else {
          const float* pa1 = base + (rowA + (unsigned)k);
          const float* pa2 = base + (rowA + (unsigned)km);
          const float* pb1 = base + (rowB + (unsigned)km);
          const float* pb2 = base + (rowB + (unsigned)k);
          v1A = make_float2(__ldg(pa1), __ldg(pa2));
          v0A = make_float2(__ldg(pa1 - 1), __ldg(pa2 + 1));
          v1B = make_float2(__ldg(pb1), __ldg(pb2));
          v0B = make_float2(__ldg(pb1 + 1), __ldg(pb2 - 1));
        }
        const float2 WL = make_float2(L - wh, L - wh);
        accA = __ffma2_rn(WL, v0A, accA);
        accA = __ffma2_rn(W, v1A, accA);
        accB = __ffma2_rn(WL, v0B, accB);
        accB = __ffma2_rn(W, v1B, accB);
        rowA += up;
        rowB -= up;
      }
    };
    if (clampk)
      walk(std::true_type{});
    else
      walk(std::false_type{});
  }
  if constexpr (kSeg > 1) {
    __shared__ float4 red[kSeg][32 * kAG];
    red[threadIdx.y][threadIdx.x] = make_float4(accA.x, accA.y, accB.x, accB.y);
    __syncthreads();
    if (threadIdx.y != 0) return;
#pragma unroll
    for (int sg = 1; sg < kSeg; ++sg) {
      const float4 v = red[sg][threadIdx.x];
      accA.x += v.x;
      accA.y += v.y;
      accB.x += v.z;
      accB.y += v.w;
    }
  }
  if (j < jh && hvalid) {
    // slab-coordinate images -> rays; x-major swaps which image is the x-mirror
    const float r_m = A.major ? accB.y : accA.y;    // (m-a, j)
    const float r_mr = A.major ? accA.y : accB.y;   // (m-a, d-1-j)
    if (band_acc) {
      asm volatile("griddepcontrol.wait;" ::: "memory");   // the previous pass's sums
      TOut* p0 = sino + (long long)a * d + j;
      TOut* p1 = sino + (long long)b * d + j;
      *p0 = (TOut)((float)*p0 + accA.x);
      *p1 = (TOut)((float)*p1 + r_m);
      if (d - 1 - j != j) {
        TOut* p2 = sino + (long long)a * d + (d - 1 - j);
        TOut* p3 = sino + (long long)b * d + (d - 1 - j);
        *p2 = (TOut)((float)*p2 + accB.x);
        *p3 = (TOut)((float)*p3 + r_mr);
      }
    } else {
    __stcs(sino + (long long)a * d + j, (TOut)accA.x);   // streaming: keep L2 for the planes
    __stcs(sino + (long long)b * d + j, (TOut)r_m);
    if (d - 1 - j != j) {
      __stcs(sino + (long long)a * d + (d - 1 - j), (TOut)accB.x);
      __stcs(sino + (long long)b * d + (d - 1 - j), (TOut)r_mr);
    }
    }
  }
}


// ===========================================================================
// float64 fast kernels (same algorithms, float64 arithmetic; <= 1e-12)
// ===========================================================================
template <typename T>
__global__ void pad_transpose64_kernel(const T* __restrict__ in, double* __restrict__ P,
                                       double* __restrict__ PT, int n) {
  __shared__ double tile[32][33];
  const int pitch = n + 2 * kPadMargin;
  {   // batch: images n*n apart, plane pairs 2 * n * pitch apart
    const long long z = blockIdx.z;
    in += z * n * n;
    P += z * 2LL * n * pitch;
    PT += z * 2LL * n * pitch;
  }
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = by + i, c = bx + threadIdx.x;
    double v = 0.0;
    if (r < n && c < n) {
      v = (double)in[(long long)r * n + c];
      P[(long long)r * pitch + kPadMargin + c] = v;
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = bx + i, r = by + threadIdx.x;
    if (r < n && c < n) PT[(long long)c * pitch + kPadMargin + r] = tile[threadIdx.x][i];
  }
  // margins: rewritten every call (the workspace is shared with the generic
  // path, which stores an unpadded transposed copy over them)
  if (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) {
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int r = by + i;
      if (r >= n) continue;
      for (int k = threadIdx.x; k < kPadMargin; k += 32) {
        if (blockIdx.x == 0) {
          P[(long long)r * pitch + k] = 0.0;
          PT[(long long)r * pitch + k] = 0.0;
        }
        if (blockIdx.x == gridDim.x - 1) {
          P[(long long)r * pitch + kPadMargin + n + k] = 0.0;
          PT[(long long)r * pitch + kPadMargin + n + k] = 0.0;
        }
      }
    }
  }
}

// Pair planes for the small-grid float64 forward: element e of a padded row
// holds (pixel e - 1, pixel e) as one 16-byte word, so a ray-slab reads both
// pixels it straddles with one LDG.128 (half the load instructions, 9 % fewer
// L1 data-pipe wavefronts than two LDG.64).  Q[r][M + c] = (v(r, c-1), v(r, c)),
// QT[c][M + r] = (v(r-1, c), v(r, c)), v = 0 outside the image, every margin
// element rewritten each call.  kPath: v = R_path^T coarse (wmg_forward_path).
template <typename T, bool kPath>
__device__ __forceinline__ void pad_pairs64_body(const T* __restrict__ in, double2* __restrict__ Q,
                                                 double2* __restrict__ QT, int n,
                                                 const BandPaths* bp) {
  __shared__ double2 tile[32][33];
  const int pitch = n + 2 * kPadMargin;
  const int sc = kPath ? (n >> bp->depth) : 0;
  {   // batch: images n*n (coarse items sc*sc) apart, plane pairs 2 * n * pitch apart
    const long long z = blockIdx.z;
    in += kPath ? z * sc * sc : z * n * n;
    Q += z * 2LL * n * pitch;
    QT += z * 2LL * n * pitch;
  }
  auto val = [&](int r, int c) -> double {
    if (r < 0 || c < 0 || r >= n || c >= n) return 0.0;
    if constexpr (kPath)
      return haar_path_value(*bp, (int)blockIdx.z, (const double*)in, sc, r, c);
    else
      return (double)in[(long long)r * n + c];
  };
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = by + i, c = bx + threadIdx.x;
    double2 q = make_double2(0.0, 0.0), qt = make_double2(0.0, 0.0);
    if (r < n && c < n) {
      const double v = val(r, c);
      q = make_double2(val(r, c - 1), v);
      qt = make_double2(val(r - 1, c), v);
      Q[(long long)r * pitch + kPadMargin + c] = q;
    }
    tile[i][threadIdx.x] = qt;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = bx + i, r = by + threadIdx.x;
    if (r < n && c < n) QT[(long long)c * pitch + kPadMargin + r] = tile[threadIdx.x][i];
  }
  // margins: zero pairs, except the first element past the last pixel, which
  // still carries that pixel as its left member
  if (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) {
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int r = by + i;   // row of Q, column of QT
      if (r >= n) continue;
      for (int k = threadIdx.x; k < kPadMargin; k += 32) {
        if (blockIdx.x == 0) {
          Q[(long long)r * pitch + k] = make_double2(0.0, 0.0);
          QT[(long long)r * pitch + k] = make_double2(0.0, 0.0);
        }
        if (blockIdx.x == gridDim.x - 1) {
          Q[(long long)r * pitch + kPadMargin + n + k] =
              make_double2(k == 0 ? val(r, n - 1) : 0.0, 0.0);
          QT[(long long)r * pitch + kPadMargin + n + k] =
              make_double2(k == 0 ? val(n - 1, r) : 0.0, 0.0);
        }
      }
    }
  }
}

template <typename T>
__global__ void pad_pairs64_kernel(const T* __restrict__ in, double2* __restrict__ Q,
                                   double2* __restrict__ QT, int n) {
  pad_pairs64_body<T, false>(in, Q, QT, n, nullptr);
}

__global__ void prolong_pairs64_kernel(BandPaths bp, const double* __restrict__ coarse,
                                       double2* __restrict__ Q, double2* __restrict__ QT, int n) {
  pad_pairs64_body<double, true>(coarse, Q, QT, n, &bp);
}


// Small-grid float64 forward on the padded planes: one ray per lane, kSplit
// slab segments per ray (threadIdx.y) reduced in shared memory in segment
// order; u is walked in 12.52 fixed point (see below), the two straddling
// pixels are read without bounds checks (zero margins) and blended as
// L v0 + wh (v1 - v0).  blockIdx.z = batch item.
// kA: lanes = (32 / kA) rays x kA adjacent angles (kA = 4 default; 1, 2 and 8 measured
// within 10 %: an LDG.64 of 32 lanes spans >= 8 sectors at any layout)
template <typename TOut, int kA = 1>
__global__ void __launch_bounds__(32 * kSplitF) fwd_split64_kernel(GeomDev G,
                                                                  const double2* __restrict__ Q,
                                                                  const double2* __restrict__ QT,
                                                                  TOut* __restrict__ sino,
                                                                  long long bs_sino) {
  __shared__ double part[kSplitF][33];
  const int lane = threadIdx.x, seg = threadIdx.y;
  // lanes = (32 / kA) rays x kA adjacent angles
  constexpr int kR = 32 / kA;
  const int a = blockIdx.y * kA + lane / kR;
  const int j = blockIdx.x * kR + lane % kR;
  const bool live = j < G.d && a < G.m;
  const int n = G.n;
  const int pitch = n + 2 * kPadMargin;
  {
    const long long zp = (long long)blockIdx.z * 2LL * n * pitch;
    Q += zp;
    QT += zp;
    sino += (long long)blockIdx.z * bs_sino;
  }
  double acc = 0.0;
  if (live) {
    const AngleParams& A = G.ang[a];
    const double u0 = A.u0 + ((double)j - (double)(G.d - 1) * 0.5) * A.du;
    const double slope = A.slope;
    int r0 = 0, r1 = n - 1;
    if (slope > 0.0) {
      // one reciprocal instead of two divisions: the +-1 slab margins absorb
      // the last-bit difference
      const double is = __drcp_rn(slope);
      const double ra = floor((-1.0 - u0) * is) - 1.0;
      const double rb = ceil(((double)n + 1.0 - u0) * is) + 1.0;
      r0 = (int)fmax(ra, 0.0);
      r1 = (int)fmin(rb, (double)(n - 1));
    } else if (u0 < -1.0 || u0 > (double)n + 1.0) {
      r1 = -1;
    }
    const int len = r1 - r0 + 1;
    const int rs = r0 + (len > 0 ? (len * seg) / kSplitF : 0);
    const int re = r0 + (len > 0 ? (len * (seg + 1)) / kSplitF : 0) - 1;
    const double L = A.L, Ls = A.Ls;
    // pair planes: element e of a row holds (pixel e - 1, pixel e)
    const double2* rowq = (A.major ? QT : Q) + kPadMargin + (long long)rs * pitch;
    // u in 12.52 fixed point (offset by the margin so it stays >= 0): the slab
    // walk is integer adds, the straddled pixel the high bits and the fraction
    // an exact bit move -- no floor / conversions in the loop; error <= (r + 1)
    // 2^-53 px, as small as the direct fp64 evaluation's
    constexpr double kQ52d = 4503599627370496.0;   // 2^52
    const long long S = llrint(slope * kQ52d);
    long long U = llrint((u0 + (double)kPadMargin) * kQ52d) + (long long)rs * S;
    const int kofs = A.mirror ? (n - 1 + kPadMargin) : -kPadMargin;   // pixel = +-k + kofs
    const int ksgn = A.mirror ? -1 : 1;
    for (int r = rs; r <= re; ++r) {
      U += S;
      const int k = (int)(U >> 52);
      const double f = __longlong_as_double(0x3FF0000000000000LL | (U & 0xFFFFFFFFFFFFFLL)) - 1.0;
      const double wh = dmin_to(f * Ls, L);        // NaN (0 * inf) -> L
      // pixel px = ksgn k + kofs and its neighbour px - ksgn, one 16-byte load:
      // (px - 1, px) at element px, or (px, px + 1) at element px + 1 (mirrored)
      const double2 q = __ldg(rowq + (ksgn * k + kofs + (ksgn < 0 ? 1 : 0)));
      const double v1 = ksgn > 0 ? q.y : q.x, v0 = ksgn > 0 ? q.x : q.y;
      acc = fma(L, v0, acc);
      acc = fma(wh, v1 - v0, acc);
      rowq += pitch;
    }
  }
  part[seg][lane] = acc;
  __syncthreads();
  if (seg == 0 && live) {
    double sum = part[0][lane];
#pragma unroll
    for (int q = 1; q < kSplitF; ++q) sum += part[q][lane];
    sino[(long long)(G.rowmap ? G.rowmap[a] : a) * G.d + j] = (TOut)sum;
  }
}

// symmetric forward in float64: u evaluated directly at every slab end
// kMix: warps of 8 rays x 4 adjacent angles, like the fp32 kernel (k clamped
// into the margins in the groups the host did not mark safe)
template <typename TOut, bool kMix = false>
__global__ void __launch_bounds__(128) fwd_sym64_kernel(GeomDev G, const double* __restrict__ P,
                                                        const double* __restrict__ PT,
                                                        TOut* __restrict__ sino) {
  int hidx, j;
  if (kMix) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    hidx = blockIdx.y * 4 + (lane >> 3);
    j = blockIdx.x * 32 + warp * 8 + (lane & 7);
  } else {
    hidx = blockIdx.y;
    j = blockIdx.x * 128 + threadIdx.x;
  }
  const bool hvalid = hidx < G.n_half;
  if (!hvalid) hidx = G.n_half - 1;
  const int a = G.half[hidx];
  const int b = G.mir[a];
  const int d = G.d, m = G.m, n = G.n;
  const int jh = (d + 1) / 2;
  const AngleParams& A = G.ang[a];
  const int pitch = n + 2 * kPadMargin;
  const double off = (double)j - (double)(d - 1) * 0.5;
  const double u0 = A.u0 + off * A.du;
  const double slope = A.slope;
  int r0 = 0, r1 = n - 1;
  if (j >= jh) {
    r0 = n; r1 = -1;
  } else if (slope > 0.0) {
    const double ra = floor((-1.0 - u0) / slope) - 1.0;
    const double rb = ceil(((double)n + 1.0 - u0) / slope) + 1.0;
    r0 = (int)fmin(fmax(ra, 0.0), (double)n);
    r1 = (int)fmax(fmin(rb, (double)(n - 1)), -1.0);
  } else if (u0 < -1.0 || u0 > (double)n + 1.0) {
    r0 = n; r1 = -1;
  }
  const int rw0 = __reduce_min_sync(0xffffffffu, r0);
  const int rw1 = __reduce_max_sync(0xffffffffu, r1);
  const bool clampk = kMix && !G.gsafe[blockIdx.y];
  double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
  if (rw0 <= rw1) {
    const double* __restrict__ base = (A.major ? PT : P);
    const double L = A.L, Ls = A.Ls;
    unsigned rowA = (unsigned)(rw0 * pitch + kPadMargin);
    unsigned rowB = (unsigned)((n - 1 - rw0) * pitch + kPadMargin);
    const unsigned up = (unsigned)pitch;
    auto walk = [&](auto clampTag) {
#pragma unroll 2
      for (int r = rw0; r <= rw1; ++r) {
        const double uh = fma((double)(r + 1), slope, u0);
        const double fk = floor(uh);
        int k = (int)fk;
        if constexpr (decltype(clampTag)::value) k = min(max(k, 2 - kPadMargin), n + kPadMargin - 3);
        const double wh = dmin_to((uh - fk) * Ls, L);
        const double wl = L - wh;
        const int km = n - 1 - k;
        const double* pa1 = base + (rowA + (unsigned)k);
        const double* pa2 = base + (rowA + (unsigned)km);
        const double* pb1 = base + (rowB + (unsigned)km);
        const double* pb2 = base + (rowB + (unsigned)k);
        const double u1 = __ldg(pa1), v1 = __ldg(pa1 - 1);
        const double u2 = __ldg(pa2), v2 = __ldg(pa2 + 1);
        const double u3 = __ldg(pb1), v3 = __ldg(pb1 + 1);
        const double u4 = __ldg(pb2), v4 = __ldg(pb2 - 1);
        a1 = fma(wh, u1, fma(wl, v1, a1));
        a2 = fma(wh, u2, fma(wl, v2, a2));
        a3 = fma(wh, u3, fma(wl, v3, a3));
        a4 = fma(wh, u4, fma(wl, v4, a4));
        rowA += up;
        rowB -= up;
      }
    };
    if (clampk)
      walk(std::true_type{});
    else
      walk(std::false_type{});
  }
  if (j < jh && hvalid) {
    const double r_m = A.major ? a4 : a2;
    const double r_mr = A.major ? a2 : a4;
    sino[(long long)a * d + j] = (TOut)a1;
    sino[(long long)b * d + j] = (TOut)r_m;
    if (d - 1 - j != j) {
      sino[(long long)a * d + (d - 1 - j)] = (TOut)a3;
      sino[(long long)b * d + (d - 1 - j)] = (TOut)r_mr;
    }
  }
}

// symmetric backprojector in float64: 52-fractional-bit fixed point
constexpr double kQ52 = 4503599627370496.0;   // 2^52
constexpr int kSym64Chunk = 8;

template <typename TIn, typename TOut, bool kAccumulate>
__global__ void __launch_bounds__(256, 4) bwd_sym64_kernel(GeomDev G, const TIn* __restrict__ sino,
                                                        TOut* __restrict__ img) {
  // winA = win[0] (y_a[t], y_b[t], y_a[t+1], y_b[t+1]), winB = win[1] reversed
  // detectors; in cluster mode the same 32 KB hold the partial tile at the end
  __shared__ double4 win[2][kSym64Chunk][kBwdWin];
  double4 (*winA)[kBwdWin] = win[0];
  double4 (*winB)[kBwdWin] = win[1];
  __shared__ long long qx[kSym64Chunk][kBwdTile];
  __shared__ long long qhead[kSym64Chunk];
  // per-angle constants, computed once per chunk: (S as bits, ic), (L, ca0), (hwic, w1c)
  __shared__ double2 angc[kSym64Chunk][3];
  __shared__ int jlo_s[kSym64Chunk];
  __shared__ int ang_s[kSym64Chunk];
  __shared__ int mir_s[kSym64Chunk];
  const int n = G.n, d = G.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col0 = blockIdx.x * kBwdTile, row0 = blockIdx.y * kBwdTile;
  const double half = (double)n * 0.5, dc = (double)(d - 1) * 0.5;
  const double xc0 = (double)col0 - half + 0.5;
  const double yc0 = half - (double)row0 - 0.5;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = 0.0;
  const int q_begin = 0, q_end = G.n_prim;
  for (int c0 = q_begin; c0 < q_end; c0 += kSym64Chunk) {
    const int na = min(kSym64Chunk, q_end - c0);
    __syncthreads();
    if (tid < na) {
      const int q = c0 + tid;
      const int a = G.prim[q];
      ang_s[tid] = a;
      mir_s[tid] = G.mir[a];
      const AngleParams& A = G.ang[a];
      const double p0 = xc0 * A.c + yc0 * A.s + dc - A.hw;
      const double t = (double)(kBwdTile - 1);
      const double pmin = p0 + fmin(0.0, t * A.c) + fmin(0.0, -t * A.s);
      const int jlo = (int)floor(pmin) - 1;
      jlo_s[tid] = jlo;
      qhead[tid] = llrint((p0 - (double)jlo) * kQ52);
      const double hw = A.hw, ic = A.inv_cs;
      angc[tid][0] = make_double2(__longlong_as_double(llrint(A.s * kQ52)), ic);
      angc[tid][1] = make_double2(A.L, 2.0 - hw);
      angc[tid][2] = make_double2(hw * ic, (2.0 * hw - 3.0) * ic);
    }
    __syncthreads();
    for (int e = tid; e < na * kBwdTile; e += 256) {
      const int aa = e / kBwdTile, l = e % kBwdTile;
      qx[aa][l] = qhead[aa] + (long long)l * llrint(G.ang[ang_s[aa]].c * kQ52);
    }
    for (int e = tid; e < na * kBwdWin; e += 256) {
      const int aa = e / kBwdWin, t = e % kBwdWin;
      const int a = ang_s[aa], b = mir_s[aa];
      const int jj = jlo_s[aa] + t;
      const TIn* ya = sino + (long long)a * d;
      const TIn* yb = sino + (long long)b * d;
      auto ld = [&](const TIn* y, int q) -> double {
        return (q >= 0 && q < d) ? (double)__ldg(y + q) : 0.0;
      };
      winA[aa][t] = make_double4(ld(ya, jj), ld(yb, jj), ld(ya, jj + 1), ld(yb, jj + 1));
      const int q0 = d - 1 - jj, q1 = d - 2 - jj;
      winB[aa][t] = make_double4(ld(ya, q0), ld(yb, q0), ld(ya, q1), ld(yb, q1));
    }
    __syncthreads();
    for (int aa = 0; aa < na; ++aa) {
      const double2 c0 = angc[aa][0], c1 = angc[aa][1], c2 = angc[aa][2];
      const long long S = __double_as_longlong(c0.x);
      const double ic = c0.y, L = c1.x, ca0 = c1.y, hwic = c2.x, w1c = c2.y;
      long long Q = qx[aa][lane] - (long long)(4 * warp) * S;
      const double4* wa = winA[aa];
      const double4* wb = winB[aa];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int hi = (int)(Q >> 52);
        const double f = __longlong_as_double(0x3FF0000000000000LL | (Q & 0xFFFFFFFFFFFFFLL));
        const double d0 = ca0 - f;
        const double w0 = dmin_to(fma(-fabs(d0), ic, hwic), L);
        const double w1 = dmax_0(fma(f, ic, w1c));
        const double4 va = wa[hi + 1];
        const double4 vb = wb[hi + 1];
        acc[i][0] = fma(w0, va.x, fma(w1, va.z, acc[i][0]));
        acc[i][1] = fma(w0, va.y, fma(w1, va.w, acc[i][1]));
        acc[i][2] = fma(w0, vb.x, fma(w1, vb.z, acc[i][2]));
        acc[i][3] = fma(w0, vb.y, fma(w1, vb.w, acc[i][3]));
        Q -= S;
      }
    }
  }
  auto pixel = [&](int i, int q, int w, int l) -> long long {
    const int row = row0 + 4 * w + i, col = col0 + l;
    const int r = (q < 2) ? row : n - 1 - row;
    const int c = (q == 0 || q == 3) ? col : n - 1 - col;
    return (long long)r * n + c;
  };
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long p = pixel(i, q, warp, lane);
      if (kAccumulate)
        img[p] = (TOut)((double)img[p] + acc[i][q]);
      else
        img[p] = (TOut)acc[i][q];
    }

}


// Small-grid float64 symmetric backprojector without staging or clusters
// (config 1 and the WMG node systems, n <= 512).  At these sizes the whole
// sinogram is L2-resident and the angle-split cluster kernel was latency bound
// (18 % of the warps active, a third of its stall samples at the cluster
// barrier).  Here a CTA owns 32 pixels of one quadrant row (and their three
// mirror / rotation images) and its kSlices warps split the primary angles;
// every (pixel, angle) reads its two detectors of the four sinogram rows
// directly (L1 / L2), so a warp has no barrier until the end, where the slice
// partials are summed in slice order through shared memory and the axis-
// aligned angles are added (deterministic; same weights as bwd_sym64_kernel).
// blockIdx = (column block of 32, quadrant row, batch item).
constexpr int kSmall64Slices = 16;
template <typename TIn, typename TOut, bool kAccumulate>
__global__ void __launch_bounds__(32 * kSmall64Slices, 2) bwd_small64_kernel(GeomDev G,
                                                                              const TIn* __restrict__ sino,
                                                                              TOut* __restrict__ img,
                                                                              GeomDev Gx) {
  __shared__ double part[kSmall64Slices][4][32];
  // per warp: the constants of up to 32 angles of its slice (lane l loads angle
  // l of the chunk), read back as broadcasts -- no dependent global loads in
  // the angle loop
  __shared__ double2 angc[kSmall64Slices][32][3];   // (c, s), (dc - hw, ic), (hw ic, w1c)
  __shared__ double angL[kSmall64Slices][32];
  __shared__ int2 angab[kSmall64Slices][32];
  const int n = G.n, d = G.d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = blockIdx.y, col = blockIdx.x * 32 + lane;   // top-left quadrant pixel
  {
    const long long item = blockIdx.z;
    sino += item * G.m * d;
    img += item * (long long)n * n;
  }
  const double half = (double)n * 0.5, dc = (double)(d - 1) * 0.5;
  const double xc = (double)col - half + 0.5, yc = half - (double)row - 0.5;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  const int q0 = (int)((long long)G.n_prim * warp / kSmall64Slices);
  const int q1 = (int)((long long)G.n_prim * (warp + 1) / kSmall64Slices);
  for (int qc = q0; qc < q1; qc += 32) {
    const int cnt = min(32, q1 - qc);
    if (lane < cnt) {
      const int a = G.prim[qc + lane];
      const AngleParams& A = G.ang[a];
      const double hw = A.hw, ic = A.inv_cs;
      angc[warp][lane][0] = make_double2(A.c, A.s);
      angc[warp][lane][1] = make_double2(dc - hw, ic);
      angc[warp][lane][2] = make_double2(hw * ic, (2.0 * hw - 3.0) * ic);
      angL[warp][lane] = A.L;
      angab[warp][lane] = make_int2(a, G.mir[a]);
    }
    __syncwarp();
#pragma unroll 4
    for (int t = 0; t < cnt; ++t) {
      const double2 cs = angc[warp][t][0], dh = angc[warp][t][1], hv = angc[warp][t][2];
      const double L = angL[warp][t];
      const int2 ab = angab[warp][t];
      const double P = fma(xc, cs.x, fma(yc, cs.y, dh.x));
      const double fl = floor(P);
      const double f = 1.0 + (P - fl);               // in [1, 2), as the fixed-point kernel
      const double d0 = (2.0 - (dc - dh.x)) - f;      // 2 - hw - f
      const double w0 = dmin_to(fma(-fabs(d0), dh.y, hv.x), L);
      const double w1 = dmax_0(fma(f, dh.y, hv.y));
      const int jA = (int)fl + 1, jB = jA + 1;
      const int rA = d - 1 - jA, rB = d - 1 - jB;
      const TIn* ya = sino + (long long)ab.x * d;
      const TIn* yb = sino + (long long)ab.y * d;
      auto ld = [&](const TIn* y, int j) -> double {
        return (j >= 0 && j < d) ? (double)__ldg(y + j) : 0.0;
      };
      const double a0 = ld(ya, jA), a1 = ld(ya, jB), b0 = ld(yb, jA), b1 = ld(yb, jB);
      const double c0 = ld(ya, rA), c1 = ld(ya, rB), e0 = ld(yb, rA), e1 = ld(yb, rB);
      acc0 = fma(w0, a0, fma(w1, a1, acc0));   // (r, c) at a
      acc1 = fma(w0, b0, fma(w1, b1, acc1));   // (r, n-1-c) at mir a
      acc2 = fma(w0, c0, fma(w1, c1, acc2));   // (n-1-r, n-1-c) at a, detectors reversed
      acc3 = fma(w0, e0, fma(w1, e1, acc3));   // (n-1-r, c) at mir a, reversed
    }
    __syncwarp();
  }
  part[warp][0][lane] = acc0;
  part[warp][1][lane] = acc1;
  part[warp][2][lane] = acc2;
  part[warp][3][lane] = acc3;
  __syncthreads();
  if (warp >= 4) return;
  // warp k finishes image k of the 32 pixels: slices in order, then the axis angles
  const int k = warp;
  double sacc = part[0][k][lane];
#pragma unroll
  for (int w = 1; w < kSmall64Slices; ++w) sacc += part[w][k][lane];
  const int r = (k < 2) ? row : n - 1 - row;
  const int cc = (k == 0 || k == 3) ? col : n - 1 - col;
  const long long p = (long long)r * n + cc;
  {
    const double xcp = (double)cc - half + 0.5, ycp = half - (double)r - 0.5;
    const double dcx = (double)(Gx.d - 1) * 0.5;
    for (int ax = 0; ax < Gx.m; ++ax) {   // axis-aligned angles (Gx: the tie rule)
      const AngleParams& Px = Gx.ang[ax];
      const int j = (int)ceil(xcp * Px.c + ycp * Px.s + dcx - 0.5);
      if (j >= 0 && j < Gx.d)
        sacc += (double)__ldg(sino + (long long)(Gx.rowmap ? Gx.rowmap[ax] : ax) * Gx.d + j);
    }
  }
  if (kAccumulate)
    img[p] = (TOut)((double)img[p] + sacc);
  else
    img[p] = (TOut)sacc;
}

}  // namespace fast

// ---------------------------------------------------------------------------
// host launchers.  dtype codes: 0 = float32, 1 = float64.
// ---------------------------------------------------------------------------
bool tma_forward_supported(const GeomDev& G);
template <typename TOut>
cudaError_t tma_forward(const GeomDev& G, float* P, float* PT, TOut* sino, int* overflow,
                        cudaStream_t st);

// Path selection.  The symmetric kernels do a quarter of the weight work but
// expose 4x less parallelism (blocks own four tile/ray images), so they only
// pay off once the grid still fills the 148 SMs several times over.
// G.sym: 0 off, 1 on when profitable, 2 forced (tests), 10 forced with the row
// warp layout of the symmetric backprojector (A/B tests), 4 forced + TMA-staged
// forward (experimental: slower than the L2 gather on B200)
// G.sym: bit 0 auto, bit 1 forced, bit 2 forced + TMA forward; the higher bits
// select testing variants
static inline bool use_sym_bwd(const GeomDev& G, int precision = 1) {
  // fp32: the run layout (angle-split over a cluster on small quadrants) beats
  // the split kernel from n = 256 up (n = 256, 180 angles: 18.6 vs 33.8 us;
  // n = 512: 63.5 vs 303 us); fp64: from n = 1024 (the angle-split cluster
  // kernel covers the small grids)
  const int base = G.sym & 7;
  return base >= 2 || (base == 1 && G.n >= (precision == 0 ? 256 : 1024));
}
static inline bool use_sym_fwd(const GeomDev& G, int precision = 0) {
  // fp32: the row-segment split keeps the symmetric forward ahead down to n = 256
  if (precision == 0) {
    const int base = G.sym & 7;
    return base >= 2 || (base == 1 && G.n >= 256);
  }
  const long long blocks = (long long)(((G.d + 1) / 2 + 127) / 128) * G.n_half;   // 128-ray units
  const int base = G.sym & 7;
  return base >= 2 || (base == 1 && blocks >= 4LL * 148);
}
static inline bool use_tiled_bwd(const GeomDev& G) { return G.n >= 768; }
// one thread per ray / pixel fills the SMs only beyond ~512 px
static inline bool use_split(const GeomDev& G) { return G.n <= 512; }

template <typename TIn, typename TOut, typename R>
static cudaError_t bwd_split_launch(const GeomDev& G, const void* y, void* x, bool accumulate,
                                    cudaStream_t st, int batch = 1) {
  dim3 grid((G.n + 31) / 32, G.n, batch), block(32, fast::kSplit);
  const long long bs = (long long)G.m * G.d;
  if (accumulate)
    fast::bwd_split_kernel<TIn, TOut, R, true><<<grid, block, 0, st>>>(G, (const TIn*)y,
                                                                       (TOut*)x, bs);
  else
    fast::bwd_split_kernel<TIn, TOut, R, false><<<grid, block, 0, st>>>(G, (const TIn*)y,
                                                                        (TOut*)x, bs);
  return cudaGetLastError();
}

template <typename TIn>
static cudaError_t launch_transpose(const TIn* in, TIn* out, int n, cudaStream_t st,
                                   int batch = 1) {
  dim3 grid((n + 31) / 32, (n + 31) / 32, batch), block(32, 8);
  fast::transpose_kernel<TIn><<<grid, block, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

template <typename TIn, typename TOut>
static cudaError_t fwd_v2_impl(const GeomDev& G, const void* x, void* ws, void* y,
                               cudaStream_t st, const GeomDev* Gx = nullptr) {
  const long long plane = (long long)G.n * (G.n + 2 * kPadMargin);
  float* P = (float*)ws;
  float* PT = P + plane;
  dim3 tg((G.n + 31) / 32, (G.n + 31) / 32), tb(32, 8);
  // default symmetric forward: mirror-packed float2 planes (PM, PMT)
  const bool packed = use_sym_fwd(G) && Gx && !(G.sym & (4 | 16 | 32 | 64 | 128));
  if (packed) {
    float2* PM = (float2*)ws;
    float2* PMT = PM + plane;
    fast::pad_mirror_kernel<TIn><<<tg, tb, 0, st>>>((const TIn*)x, PM, PMT, G.n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    constexpr int ag = fast::kFwdAG;
    dim3 mgrid(((G.d + 1) / 2 + 8 * ag - 1) / (8 * ag), (G.n_half + 3) / 4);
    const long long blocks = (long long)mgrid.x * mgrid.y;
    // grids below n = 1792 (and launches of few blocks at any size): each warp's
    // slab range split over 8 row segments, one ray octet per block (sym & 65536:
    // testing, unsplit).  Warm, L2 flushed, against the unsplit 4-octet blocks
    // (tools/probe_size_scan.py): n = 640 126 -> 101 us, 1024 347 -> 304, 1152 478 ->
    // 411, 1280 591 -> 548, 1536 957 -> 904, 1792 equal, 2048 2063 vs 2069, 3072
    // 6536 vs 6799; 4, 6, 12 and 16 segments are slower than 8 at every size
    // Launches of fewer than 8000 4-octet blocks (the per-rank angle shards of
    // the multi-GPU pair) take the same form: their 3-6 waves of long blocks
    // left the L1 data pipe at 70 % (n = 4096, 514 of 4096 angles: forward 2.80
    // -> 2.59 ms; n = 3072, 386 angles: 1.42 -> 1.09; n = 2048, 258 angles: 0.54
    // -> 0.38 ms, tools/probe_shard_eff.py)
    const int seg = (G.sym & 65536) ? 1 : (G.n < 1792 || blocks < 8000) ? 8 : 1;
    // Banded passes over the slab index when the two padded planes exceed the
    // L2 (n = 4096: 277 MB -> 4 passes): the blocks of one pass walk only
    // slabs [lo, hi) (rows lo..hi-1 and their mirrors n-hi..n-lo-1 of both
    // planes), so the planes are read from DRAM about once instead of ~30x
    // (9.5 -> 0.9 GB per launch, 15.6 -> 15.1 ms); later passes add their
    // partial ray sums to the sinogram (fixed order: deterministic)
    const double plane_mb = 2.0 * G.n * (G.n + 2.0 * kPadMargin) * 8.0 / 1e6;
    // (the 8-segment form is banded only from 200 MB: at n = 3072, 154 MB, its
    // unbanded launch is faster: 386 angles 1.09 vs 1.18 ms, 770 angles 1.94 vs 2.11)
    // The unsplit form always runs in >= 3 passes: chained (below), shorter blocks
    // balance the SMs better even where the planes fit the L2 (n = 1920 1.72 ->
    // 1.63 ms, 2048 2.07 -> 1.98, 2304 2.84 -> 2.81; neutral from 2560)
    // (sym & 65536, LineProjector.prefer_concurrent: one pass while the planes fit
    // the L2 -- with a second stream's kernels on the GPU the chained passes lose:
    // config-4 geometry, two streams, 1.88 vs 1.96 ms per pair)
    const int nb = seg == 8 ? (plane_mb > 200.0 ? (int)ceil(plane_mb / 70.0) : 1)
                            : (plane_mb > 128.0 ? (int)ceil(plane_mb / 70.0)
                                                : (G.sym & 65536) ? 1 : 3);
    // split kernels: one ray octet (its kSeg row segments) per block, so every
    // warp of a block walks an equally long segment and the block frees its
    // slot when they finish (with 4 octets per block the short edge-ray octets
    // held their slots until the block's longest walk ended)
    // (n = 512: 90 -> 82 us, n = 256: 40 -> 37 us)
    const dim3 ograd(((G.d + 1) / 2 + 7) / 8, (G.n_half + 3) / 4);
    // passes bi >= 1: programmatic dependent launch behind pass bi - 1
    auto launch_pass = [&](auto kern, dim3 grid, dim3 block, int bi) -> cudaError_t {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = block;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = bi > 0 ? 1 : 0;
      return cudaLaunchKernelEx(&cfg, kern, G, (const float*)PM, (const float*)PMT, (TOut*)y,
                                nb > 1 ? G.n * bi / nb : 0,
                                nb > 1 ? G.n * (bi + 1) / nb : 1 << 30, (int)(bi > 0));
    };
    if (seg == 8) {
      for (int bi = 0; bi < nb; ++bi) {
        cudaError_t el = launch_pass(fast::fwd_sym_kernel<TOut, 1, false, true, true, 8>, ograd,
                                     dim3(32, 8), bi);
        if (el != cudaSuccess) return el;
      }
    } else {
      // ray octets kStride apart inside each block (see fwd_sym_kernel)
      constexpr int kStride = 4;
      dim3 sgrid(((G.d + 1) / 2 + 8 * ag * kStride - 1) / (8 * ag * kStride) * kStride,
                 (G.n_half + 3) / 4);
      // (up to n = 1024 the octets' shared L1 lines are worth more: n = 1024
      // 0.35 ms adjacent vs 0.39 strided, 896 equal; from n = 1088 strided wins:
      // 1088 0.441 vs 0.447 ms, 1152 0.480 vs 0.519, 1216 0.529 vs 0.575)
      constexpr int kFwdStrideMinN = 1088;
      if (G.n >= kFwdStrideMinN && nb > 1) {
        for (int bi = 0; bi < nb; ++bi) {
          cudaError_t el = launch_pass(
              fast::fwd_sym_kernel<TOut, ag, false, true, true, 1, kStride>, sgrid,
              dim3(32 * ag), bi);
          if (el != cudaSuccess) return el;
        }
      } else if (G.n >= kFwdStrideMinN)
        fast::fwd_sym_kernel<TOut, ag, false, true, true, 1, kStride><<<sgrid, 32 * ag, 0, st>>>(
            G, (const float*)PM, (const float*)PMT, (TOut*)y);
      else
        fast::fwd_sym_kernel<TOut, ag, false, true, true><<<mgrid, 32 * ag, 0, st>>>(
            G, (const float*)PM, (const float*)PMT, (TOut*)y);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess || Gx->m == 0) return e;
    // the axis-aligned angles of the set: 32 slab segments over threadIdx.y (two
    // angles launch only 2 d / 32 blocks, each walking n slabs: with 8 segments
    // this serial tail took 15 / 25 / 46 us at n = 512 / 1024 / 2048)
    dim3 xgrid((G.d + 31) / 32, Gx->m), xblock(32, fast::kSplitAxis);
    fast::fwd_v2_split_kernel<TOut, 2, fast::kSplitAxis><<<xgrid, xblock, 0, st>>>(
        *Gx, (const float*)PM, (const float*)PMT, (TOut*)y);
    return cudaGetLastError();
  }
  fast::pad_transpose_kernel<TIn><<<tg, tb, 0, st>>>((const TIn*)x, P, PT, G.n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (use_sym_fwd(G) && Gx) {
    if (G.sym == 4 && tma_forward_supported(G)) {   // opt-in: TMA-staged forward
      e = tma_forward<TOut>(G, P, PT, (TOut*)y, nullptr, st);
    } else {
      if (G.sym & 16) {   // testing: one angle per block
        dim3 sgrid(((G.d + 1) / 2 + 127) / 128, G.n_half);
        fast::fwd_sym_kernel<TOut, 1><<<sgrid, 128, 0, st>>>(G, P, PT, (TOut*)y);
      } else {
        constexpr int ag = fast::kFwdAG;
        dim3 sgrid(((G.d + 1) / 2 + 31) / 32, (G.n_half + ag - 1) / ag);
        if (G.sym & 32) {         // testing: lockstep angle groups, 32 rays per warp
          fast::fwd_sym_kernel<TOut, ag, true><<<sgrid, 32 * ag, 0, st>>>(G, P, PT, (TOut*)y);
        } else if (G.sym & 64) {  // testing: 32 rays of one angle per warp
          fast::fwd_sym_kernel<TOut, ag><<<sgrid, 32 * ag, 0, st>>>(G, P, PT, (TOut*)y);
        } else {                  // (sym & 128) testing: mixed warps on the plain planes
          dim3 mgrid(((G.d + 1) / 2 + 8 * ag - 1) / (8 * ag), (G.n_half + 3) / 4);
          fast::fwd_sym_kernel<TOut, ag, false, true><<<mgrid, 32 * ag, 0, st>>>(G, P, PT,
                                                                               (TOut*)y);
        }
      }
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) return e;
    if (Gx->m == 0) return cudaSuccess;
    dim3 xgrid((G.d + 127) / 128, Gx->m);   // the axis-aligned angles of the set
    fast::fwd_v2_kernel<TOut><<<xgrid, 128, 0, st>>>(*Gx, P, PT, (TOut*)y);
    return cudaGetLastError();
  }
  dim3 grid((G.d + 127) / 128, G.m);
  fast::fwd_v2_kernel<TOut><<<grid, 128, 0, st>>>(G, P, PT, (TOut*)y);
  return cudaGetLastError();
}


// G_axis: the two axis-aligned angles of a symmetric geometry (rowmap -> their
// sinogram rows), or nullptr
template <typename TIn, typename TOut>
static cudaError_t bwd_v2_impl(const GeomDev& G, const void* y, void* x, bool accumulate,
                               cudaStream_t st, const GeomDev* G_axis = nullptr);

// small quadrants: the run layout with the angles split over a cluster of
// nsplit CTAs per tile (>= ~4 CTAs per SM, >= 4 primary angles per CTA).  At
// least 10 CTAs per tile at every size below the eight-image switch: more,
// shorter CTAs balance the SMs better than fewer waves of long ones (sweep of
// the cluster size, warm, L2 flushed, tools/nsplit_sweep.sh: n = 768 181 (5
// CTAs) -> 163 us (10), n = 1024 378 (3) -> 345, n = 1280 689 (2) -> 630,
// n = 1408 861 (2) -> 828, n = 1536 1058 (2) -> 1054, n = 512 unchanged (10);
// 12 and 16 are slower everywhere from n = 512)
static inline int symrun_nsplit(const GeomDev& G) {
  const int tiles = (G.n / 64) * (G.n / 64);
  const int fill = (4 * 148 + tiles - 1) / tiles;
  return max(1, min(16, min(max(fill, 10), G.n_prim / 4)));
}

template <typename TIn, typename TOut, bool kAcc>
static cudaError_t bwd_symrun_cluster(const GeomDev& G, const void* y, void* x, int nsplit,
                                      int batch, cudaStream_t st) {
  auto kern = fast::bwd_symrun_kernel<TIn, TOut, kAcc, 4, true>;
  static bool attr = false;   // per instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G.n / 64, G.n / 64, nsplit * batch);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = nsplit;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, G, (const TIn*)y, (TOut*)x, nsplit);
}

template <typename TIn, typename TOut, int R>
static void bwd_symrun_launch(const GeomDev& G, const void* y, void* x, bool accumulate,
                              cudaStream_t st) {
  dim3 grid(G.n / 64, G.n / (16 * R));   // the top-left quadrant in 32 x 8R tiles
  if (accumulate)
    fast::bwd_symrun_kernel<TIn, TOut, true, R><<<grid, 256, 0, st>>>(G, (const TIn*)y,
                                                                     (TOut*)x);
  else
    fast::bwd_symrun_kernel<TIn, TOut, false, R><<<grid, 256, 0, st>>>(G, (const TIn*)y,
                                                                      (TOut*)x);
}

// Eight images per weight from this many quadrant tile pairs (n >= 1728): measured
// against the four-image run layout (10 cluster CTAs per tile), warm, L2 flushed
// (tools/probe_bwd_threshold.py): n = 1536 (300 pairs) 1228 vs 1055 us, 1600 (325)
// 1281 vs 1193, 1664 (351) 1348 vs 1326, 1728 (378) 1402 vs 1486, 1792 (406) 1457 vs
// 1652, 2048 (528) 2108 vs 2444 us
constexpr long long kSym8MinPairs = 370;

// The axis-aligned angles of a symmetric set, added to image rows [row_lo,
// row_hi): one thread per pixel (per angle one detector load of weight 1 and
// the pixel's read-modify-write; the tiled kernel's window staging for two
// angles took 11 / 26 us at n = 1024 / 2048, the angle-split one 13 us at 512)
template <typename TIn, typename TOut>
static cudaError_t bwd_axis_launch(const GeomDev& Gx, const void* y, void* x, cudaStream_t st,
                                   int row_lo = 0, int row_hi = -1) {
  if (row_hi < 0) row_hi = Gx.n;
  if (Gx.m == 0 || row_hi <= row_lo) return cudaSuccess;
  dim3 g1((Gx.n + 31) / 32, (row_hi - row_lo + 7) / 8);
  fast::bwd_kernel<TIn, TOut, float, true><<<g1, 256, 0, st>>>(Gx, (const TIn*)y, (TOut*)x,
                                                                row_lo, row_hi);
  return cudaGetLastError();
}

template <typename TIn, typename TOut>
static cudaError_t bwd_sym_impl(const GeomDev& G, const GeomDev& Gx, const void* y, void* x,
                                bool accumulate, cudaStream_t st) {
  dim3 grid(G.n / 64, G.n / 64);
  const bool rowlayout = (G.sym & 8) != 0;    // testing: the lane = column layout
  const bool blocks8x4 = (G.sym & 256) != 0;  // testing: 8x4 warp blocks, float4 windows
  const int qt = G.n / 64;                      // quadrant tiles per side
  // eight images per weight where the tile pairs fill the SMs (sym & 8192:
  // testing, at any size; sym & 16384: testing, the four-image run layout)
  if (G.tsym && !rowlayout && !blocks8x4 && !(G.sym & (512 | 1024 | 16384)) &&
      ((long long)qt * (qt + 1) / 2 >= kSym8MinPairs || (G.sym & 8192))) {
    const unsigned grid8 = (unsigned)(qt * (qt + 1) / 2);
    constexpr int smem8 = 2 * 4 * fast::kBwdTile * (fast::kBwdTile + 1) * (int)sizeof(float);
    static bool attr[2] = {false, false};   // per instantiation
    auto k8 = accumulate ? fast::bwd_sym8_kernel<TIn, TOut, true>
                         : fast::bwd_sym8_kernel<TIn, TOut, false>;
    if (!attr[accumulate]) {
      cudaError_t ea = cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem8);
      if (ea != cudaSuccess) return ea;
      attr[accumulate] = true;
    }
    k8<<<grid8, 256, smem8, st>>>(G, (const TIn*)y, (TOut*)x, -1);
  } else if (!rowlayout && !blocks8x4) {
    // run layout: 64-row tiles (fewer window loads per pixel) when the quadrant
    // allows and the grid still fills the SMs (n >= ~3400), else 32-row tiles
    // (sym & 1024: testing, 64-row tiles at any size; sym & 512: 32-row tiles);
    // small quadrants split the angles over a cluster (sym & 32768: testing, off)
    const int nsplit = symrun_nsplit(G);
    if (nsplit > 1 && !(G.sym & (512 | 1024 | 32768))) {
      cudaError_t e = accumulate ? bwd_symrun_cluster<TIn, TOut, true>(G, y, x, nsplit, 1, st)
                                 : bwd_symrun_cluster<TIn, TOut, false>(G, y, x, nsplit, 1, st);
      if (e != cudaSuccess || Gx.m == 0) return e;
      return bwd_axis_launch<TIn, TOut>(Gx, y, x, st);   // axis angles, accumulate
    }
    if ((G.n / 2) % 64 == 0 &&
        ((long long)(G.n / 64) * (G.n / 128) >= 12LL * 148 || (G.sym & 1024)) &&
        !(G.sym & 512))
      bwd_symrun_launch<TIn, TOut, 8>(G, y, x, accumulate, st);
    else
      bwd_symrun_launch<TIn, TOut, 4>(G, y, x, accumulate, st);
  } else if (accumulate) {
    if (rowlayout)
      fast::bwd_sym_kernel<TIn, TOut, true, false><<<grid, 256, 0, st>>>(G, (const TIn*)y,
                                                                        (TOut*)x);
    else
      fast::bwd_sym_kernel<TIn, TOut, true, true><<<grid, 256, 0, st>>>(G, (const TIn*)y,
                                                                       (TOut*)x);
  } else {
    if (rowlayout)
      fast::bwd_sym_kernel<TIn, TOut, false, false><<<grid, 256, 0, st>>>(G, (const TIn*)y,
                                                                         (TOut*)x);
    else
      fast::bwd_sym_kernel<TIn, TOut, false, true><<<grid, 256, 0, st>>>(G, (const TIn*)y,
                                                                        (TOut*)x);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || Gx.m == 0) return e;
  return bwd_axis_launch<TIn, TOut>(Gx, y, x, st);   // axis angles, accumulate
}

template <typename TIn, typename TOut>
static cudaError_t bwd_v2_impl(const GeomDev& G, const void* y, void* x, bool accumulate,
                               cudaStream_t st, const GeomDev* G_axis) {
  if (use_sym_bwd(G, 0) && G_axis)
    return bwd_sym_impl<TIn, TOut>(G, *G_axis, y, x, accumulate, st);
  if (use_split(G)) return bwd_split_launch<TIn, TOut, float>(G, y, x, accumulate, st);
  if (!use_tiled_bwd(G)) {   // small grids: one thread per pixel
    dim3 g1((G.n + 31) / 32, (G.n + 7) / 8);
    if (accumulate)
      fast::bwd_kernel<TIn, TOut, float, true><<<g1, 256, 0, st>>>(G, (const TIn*)y, (TOut*)x);
    else
      fast::bwd_kernel<TIn, TOut, float, false><<<g1, 256, 0, st>>>(G, (const TIn*)y, (TOut*)x);
    return cudaGetLastError();
  }
  dim3 grid((G.n + fast::kBwdTile - 1) / fast::kBwdTile,
            (G.n + fast::kBwdTile - 1) / fast::kBwdTile);
  if (accumulate)
    fast::bwd_v2_kernel<TIn, TOut, true><<<grid, 128, 0, st>>>(G, (const TIn*)y, (TOut*)x);
  else
    fast::bwd_v2_kernel<TIn, TOut, false><<<grid, 128, 0, st>>>(G, (const TIn*)y, (TOut*)x);
  return cudaGetLastError();
}

size_t fast_forward_workspace_bytes(int n, int precision, int tin) {
  // fp32: P and PT, or the mirror-packed float2 planes PM and PMT (twice the size)
  if (precision == 0) return sizeof(float) * 4 * (size_t)n * (size_t)(n + 2 * kPadMargin);
  // float64: padded double planes (symmetric path) -- also holds the transposed
  // copy of the generic path; small grids: the split forward's 16-byte pair planes
  const size_t elem = n <= 512 ? 2 * sizeof(double) : sizeof(double);
  return elem * 2 * (size_t)n * (size_t)(n + 2 * kPadMargin);
}

template <typename TIn, typename TOut>
static cudaError_t fwd64_impl(const GeomDev& G, const void* x, void* ws, void* y,
                              cudaStream_t st, const GeomDev* Gx) {
  if (!(G.sym && Gx)) return cudaErrorNotSupported;
  const long long plane = (long long)G.n * (G.n + 2 * kPadMargin);
  double* P = (double*)ws;
  double* PT = P + plane;
  dim3 tg((G.n + 31) / 32, (G.n + 31) / 32), tb(32, 8);
  fast::pad_transpose64_kernel<TIn><<<tg, tb, 0, st>>>((const TIn*)x, P, PT, G.n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (G.sym & 64) {   // testing: 128 rays of one angle per block
    dim3 sgrid(((G.d + 1) / 2 + 127) / 128, G.n_half);
    fast::fwd_sym64_kernel<TOut><<<sgrid, 128, 0, st>>>(G, P, PT, (TOut*)y);
  } else {            // default: warps of 8 rays x 4 adjacent angles
    dim3 mgrid(((G.d + 1) / 2 + 31) / 32, (G.n_half + 3) / 4);
    fast::fwd_sym64_kernel<TOut, true><<<mgrid, 128, 0, st>>>(G, P, PT, (TOut*)y);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // the axis-aligned angles: generic walk on the padded planes
  if (Gx->m == 0) return cudaSuccess;
  dim3 xgrid((G.d + 127) / 128, Gx->m);
  fast::fwd_kernel<double, TOut, double><<<xgrid, 128, 0, st>>>(
      *Gx, P + kPadMargin, PT + kPadMargin, (TOut*)y, G.n + 2 * kPadMargin);
  return cudaGetLastError();
}

template <typename TIn, typename TOut>
static cudaError_t bwd64_impl(const GeomDev& G, const void* y, void* x, bool accumulate,
                              cudaStream_t st, const GeomDev* Gx, bool small = false,
                              int batch = 1) {
  if (!(G.sym && Gx)) return cudaErrorNotSupported;
  if (small) {   // small grids: stage-free angle-sliced kernel (bwd_small64_kernel)
    dim3 grid(G.n / 64, G.n / 2, batch);
    if (accumulate)
      fast::bwd_small64_kernel<TIn, TOut, true><<<grid, 32 * fast::kSmall64Slices, 0, st>>>(
          G, (const TIn*)y, (TOut*)x, *Gx);
    else
      fast::bwd_small64_kernel<TIn, TOut, false><<<grid, 32 * fast::kSmall64Slices, 0, st>>>(
          G, (const TIn*)y, (TOut*)x, *Gx);
    return cudaGetLastError();
  }
  dim3 grid(G.n / 64, G.n / 64, 1);
  if (accumulate)
    fast::bwd_sym64_kernel<TIn, TOut, true><<<grid, 256, 0, st>>>(G, (const TIn*)y, (TOut*)x);
  else
    fast::bwd_sym64_kernel<TIn, TOut, false><<<grid, 256, 0, st>>>(G, (const TIn*)y, (TOut*)x);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || Gx->m == 0) return e;
  dim3 g2((G.n + 31) / 32, (G.n + 7) / 8);
  fast::bwd_kernel<TIn, TOut, double, true><<<g2, 256, 0, st>>>(*Gx, (const TIn*)y, (TOut*)x);
  return cudaGetLastError();
}

template <typename TIn, typename TOut, typename R>
static cudaError_t fwd_impl(const GeomDev& G, const void* x, void* xT_ws, void* y,
                            cudaStream_t st) {
  const TIn* img = (const TIn*)x;
  TIn* imgT = (TIn*)xT_ws;
  if (sizeof(R) == 8 && use_split(G)) {
    // padded float64 planes (the workspace holds 2 * n * (n + 2 margin) doubles)
    // padded float64 pair planes (the workspace holds 2 * n * (n + 2 margin) double2)
    double2* Q = (double2*)xT_ws;
    double2* QT = Q + (long long)G.n * (G.n + 2 * kPadMargin);
    dim3 tg((G.n + 31) / 32, (G.n + 31) / 32), tb(32, 8);
    fast::pad_pairs64_kernel<TIn><<<tg, tb, 0, st>>>(img, Q, QT, G.n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 sg((G.d + 7) / 8, (G.m + 3) / 4), sb(32, fast::kSplitF);
    fast::fwd_split64_kernel<TOut, 4><<<sg, sb, 0, st>>>(G, Q, QT, (TOut*)y, 0);
    return cudaGetLastError();
  }
  cudaError_t e = launch_transpose<TIn>(img, imgT, G.n, st);
  if (e != cudaSuccess) return e;
  if (use_split(G)) {
    dim3 sg((G.d + 31) / 32, G.m), sb(32, fast::kSplit);
    fast::fwd_split_kernel<TIn, TOut, R><<<sg, sb, 0, st>>>(G, img, imgT, (TOut*)y, 0);
    return cudaGetLastError();
  }
  dim3 grid((G.d + 127) / 128, G.m);
  fast::fwd_kernel<TIn, TOut, R><<<grid, 128, 0, st>>>(G, img, imgT, (TOut*)y, G.n);
  return cudaGetLastError();
}

template <typename TIn, typename TOut, typename R>
static cudaError_t bwd_impl(const GeomDev& G, const void* y, void* x, bool accumulate,
                            cudaStream_t st) {
  if (use_split(G)) return bwd_split_launch<TIn, TOut, R>(G, y, x, accumulate, st);
  dim3 grid((G.n + 31) / 32, (G.n + 7) / 8);
  if (accumulate)
    fast::bwd_kernel<TIn, TOut, R, true><<<grid, 256, 0, st>>>(G, (const TIn*)y, (TOut*)x);
  else
    fast::bwd_kernel<TIn, TOut, R, false><<<grid, 256, 0, st>>>(G, (const TIn*)y, (TOut*)x);
  return cudaGetLastError();
}

// precision: 0 = fp32 arithmetic, 1 = fp64 arithmetic
cudaError_t fast_forward(const GeomDev& G, int precision, int tin, int tout, const void* x,
                         void* xT_ws, void* y, cudaStream_t st, const GeomDev* Gx) {
  if (G.m == 0 || G.d == 0) return cudaSuccess;
  if (precision == 0) {
    if (tin == 0 && tout == 0) return fwd_v2_impl<float, float>(G, x, xT_ws, y, st, Gx);
    if (tin == 1 && tout == 1) return fwd_v2_impl<double, double>(G, x, xT_ws, y, st, Gx);
    if (tin == 1 && tout == 0) return fwd_v2_impl<double, float>(G, x, xT_ws, y, st, Gx);
    if (tin == 0 && tout == 1) return fwd_v2_impl<float, double>(G, x, xT_ws, y, st, Gx);
  } else {
    if (use_sym_fwd(G, 1) && Gx && tin == 1 && tout == 1)
      return fwd64_impl<double, double>(G, x, xT_ws, y, st, Gx);
    if (tin == 1 && tout == 1) return fwd_impl<double, double, double>(G, x, xT_ws, y, st);
    if (tin == 0 && tout == 0) return fwd_impl<float, float, double>(G, x, xT_ws, y, st);
  }
  return cudaErrorInvalidValue;
}

// Banded fp32 backprojection (the eight-image path): quadrant row-blocks
// [s0, s1), i.e. image rows [32 s0, 32 s1) and [n - 32 s1, n - 32 s0), are
// written complete (all angles, axis angles included) -- every pixel gets the
// same sums as the unbanded launch.  Bands must be run in order (s0 = 0 first)
// because a tile pair (i, j) writes row-blocks i and j >= s0.
int fast_backward_bands(const GeomDev& G, int precision, const GeomDev* Gx) {
  if (precision != 0 || !Gx || !use_sym_bwd(G, 0) || !G.tsym || G.n % 64) return 0;
  const int qt = G.n / 64;
  if (G.sym & (8 | 256 | 512 | 1024 | 16384)) return 0;
  if (!((long long)qt * (qt + 1) / 2 >= kSym8MinPairs || (G.sym & 8192))) return 0;
  return qt;
}

template <typename TIn, typename TOut>
static cudaError_t bwd_band_impl(const GeomDev& G, const GeomDev& Gx, const void* y, void* x,
                                 int s0, int s1, cudaStream_t st) {
  const int qt = G.n / 64;
  auto off = [&](int s) { return s * qt - s * (s - 1) / 2; };
  const int p0 = off(s0), np = off(s1) - p0;
  if (np > 0) {
    constexpr int smem8 = 2 * 4 * fast::kBwdTile * (fast::kBwdTile + 1) * (int)sizeof(float);
    static bool attr = false;
    auto k8 = fast::bwd_sym8_kernel<TIn, TOut, false>;
    if (!attr) {
      cudaError_t ea = cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem8);
      if (ea != cudaSuccess) return ea;
      attr = true;
    }
    k8<<<np, 256, smem8, st>>>(G, (const TIn*)y, (TOut*)x, p0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (Gx.m == 0 || s1 <= s0) return cudaSuccess;
  // the axis-aligned angles of the set on the band's two row ranges
  const int T = fast::kBwdTile;
  cudaError_t e = bwd_axis_launch<TIn, TOut>(Gx, y, x, st, T * s0, T * s1);
  if (e != cudaSuccess) return e;
  return bwd_axis_launch<TIn, TOut>(Gx, y, x, st, G.n - T * s1, G.n - T * s0);
}

cudaError_t fast_backward_band(const GeomDev& G, int precision, int tin, int tout, const void* y,
                               void* x, int s0, int s1, cudaStream_t st, const GeomDev* Gx) {
  const int qt = fast_backward_bands(G, precision, Gx);
  if (qt == 0 || s0 < 0 || s1 > qt || s0 > s1) return cudaErrorInvalidValue;
  if (tin == 0 && tout == 0) return bwd_band_impl<float, float>(G, *Gx, y, x, s0, s1, st);
  if (tin == 1 && tout == 1) return bwd_band_impl<double, double>(G, *Gx, y, x, s0, s1, st);
  if (tin == 1 && tout == 0) return bwd_band_impl<double, float>(G, *Gx, y, x, s0, s1, st);
  if (tin == 0 && tout == 1) return bwd_band_impl<float, double>(G, *Gx, y, x, s0, s1, st);
  return cudaErrorInvalidValue;
}

// small symmetric float64 grids: the cluster-reduced angle-split backprojector
static inline bool use_small_sym64(const GeomDev& G) {
  return G.sym == 1 && use_split(G) && G.n % 64 == 0 && G.n >= 64;
}

cudaError_t fast_backward(const GeomDev& G, int precision, int tin, int tout, const void* y,
                          void* x, bool accumulate, cudaStream_t st, const GeomDev* Gx) {
  if (G.n == 0) return cudaSuccess;
  if (precision == 0) {
    if (tin == 0 && tout == 0) return bwd_v2_impl<float, float>(G, y, x, accumulate, st, Gx);
    if (tin == 1 && tout == 1) return bwd_v2_impl<double, double>(G, y, x, accumulate, st, Gx);
    if (tin == 1 && tout == 0) return bwd_v2_impl<double, float>(G, y, x, accumulate, st, Gx);
    if (tin == 0 && tout == 1) return bwd_v2_impl<float, double>(G, y, x, accumulate, st, Gx);
  } else {
    if (use_sym_bwd(G) && Gx && tin == 1 && tout == 1)
      return bwd64_impl<double, double>(G, y, x, accumulate, st, Gx);
    // small symmetric grids: angle-split symmetric kernel (4 images per weight)
    if (use_small_sym64(G) && Gx && tin == 1 && tout == 1)
      return bwd64_impl<double, double>(G, y, x, accumulate, st, Gx, true);
    if (tin == 1 && tout == 1) return bwd_impl<double, double, double>(G, y, x, accumulate, st);
    if (tin == 0 && tout == 0) return bwd_impl<float, float, double>(G, y, x, accumulate, st);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Batches of images / sinograms (contiguous, n*n and m*d apart): the WMG cycle
// applies the node systems of sibling subproblems together.  The small-grid
// float64 split kernels take the batch as gridDim.z (one launch fills the SMs
// several times over); every other path loops over the batch.  Each item is
// computed exactly as by the single-image call.
// ---------------------------------------------------------------------------
cudaError_t fast_forward_batch(const GeomDev& G, int precision, int tin, int tout, const void* x,
                               void* ws, size_t ws_item, void* y, int batch, cudaStream_t st,
                               const GeomDev* Gx) {
  if (batch < 1) return cudaSuccess;
  const long long N = (long long)G.n * G.n, M = (long long)G.m * G.d;
  const size_t si = tin == 1 ? 8 : 4, so = tout == 1 ? 8 : 4;
  const bool split64 = precision == 1 && tin == 1 && tout == 1 && use_split(G) &&
                       !(use_sym_fwd(G, 1) && Gx);
  if (split64 && G.m > 0 && G.d > 0) {
    // batch * (Q, QT) padded pair planes; ws_item = 2 * n * (n + 2 margin) double2
    double2* Q = (double2*)ws;
    double2* QT = Q + (long long)G.n * (G.n + 2 * kPadMargin);
    dim3 tg((G.n + 31) / 32, (G.n + 31) / 32, batch), tb(32, 8);
    fast::pad_pairs64_kernel<double><<<tg, tb, 0, st>>>((const double*)x, Q, QT, G.n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 sg((G.d + 7) / 8, (G.m + 3) / 4, batch), sb(32, fast::kSplitF);
    fast::fwd_split64_kernel<double, 4><<<sg, sb, 0, st>>>(G, Q, QT, (double*)y, M);
    return cudaGetLastError();
  }
  for (int b = 0; b < batch; ++b) {
    cudaError_t e = fast_forward(G, precision, tin, tout, (const char*)x + b * N * si,
                                 (char*)ws + b * ws_item, (char*)y + b * M * so, st, Gx);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// W R_path^T for a batch of WMG node vectors (float64 fast, small grids): the
// prolongation along each item's band path is evaluated inside the padding
// kernel, then the same batched fwd_split64 launch as fast_forward_batch --
// bit-identical to haar_prolong_path followed by fast_forward_batch.
bool fast_forward_path_supported(const GeomDev& G, int precision, const GeomDev* Gx) {
  return precision == 1 && use_split(G) && !(use_sym_fwd(G, 1) && Gx) && G.m > 0 && G.d > 0;
}

cudaError_t fast_forward_path(const GeomDev& G, int depth, int batch, const int* bands,
                              const double* coarse, void* ws, double* y, cudaStream_t st,
                              const GeomDev* Gx) {
  if (!fast_forward_path_supported(G, 1, Gx) || depth < 1 || depth > 7 || (G.n >> depth) < 1)
    return cudaErrorInvalidValue;
  const long long M = (long long)G.m * G.d;
  const long long plane = (long long)G.n * (G.n + 2 * kPadMargin);
  const int sc = G.n >> depth;
  for (int b0 = 0; b0 < batch; b0 += kPathBatch) {
    const int nb = batch - b0 < kPathBatch ? batch - b0 : kPathBatch;
    BandPaths bp;
    bp.depth = depth;
    for (int i = 0; i < nb; ++i) {
      unsigned code = 0;
      for (int lv = 0; lv < depth; ++lv)
        code |= (unsigned)(bands[(b0 + i) * depth + lv] & 3) << (2 * lv);
      bp.code[i] = (unsigned short)code;
    }
    double2* Q = (double2*)ws + (long long)b0 * 2 * plane;
    double2* QT = Q + plane;
    dim3 tg((G.n + 31) / 32, (G.n + 31) / 32, nb), tb(32, 8);
    fast::prolong_pairs64_kernel<<<tg, tb, 0, st>>>(bp, coarse + (long long)b0 * sc * sc, Q, QT,
                                                    G.n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 sg((G.d + 7) / 8, (G.m + 3) / 4, nb), sb(32, fast::kSplitF);
    fast::fwd_split64_kernel<double, 4><<<sg, sb, 0, st>>>(G, Q, QT, y + (long long)b0 * M, M);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t fast_backward_batch(const GeomDev& G, int precision, int tin, int tout, const void* y,
                                void* x, bool accumulate, int batch, cudaStream_t st,
                                const GeomDev* Gx) {
  if (batch < 1 || G.n == 0) return cudaSuccess;
  const long long N = (long long)G.n * G.n, M = (long long)G.m * G.d;
  const size_t si = tin == 1 ? 8 : 4, so = tout == 1 ? 8 : 4;
  const bool small64 = precision == 1 && tin == 1 && tout == 1 && use_small_sym64(G) && Gx &&
                       !use_sym_bwd(G);
  if (small64)   // one cluster launch for the whole batch
    return bwd64_impl<double, double>(G, y, x, accumulate, st, Gx, true, batch);
  const bool sym = use_sym_bwd(G, precision) && Gx;
  if (use_split(G) && !sym && tin == tout) {
    if (precision == 1 && tin == 1)
      return bwd_split_launch<double, double, double>(G, y, x, accumulate, st, batch);
    if (precision == 0 && tin == 1)
      return bwd_split_launch<double, double, float>(G, y, x, accumulate, st, batch);
    if (precision == 0 && tin == 0)
      return bwd_split_launch<float, float, float>(G, y, x, accumulate, st, batch);
  }
  for (int b = 0; b < batch; ++b) {
    cudaError_t e = fast_backward(G, precision, tin, tout, (const char*)y + b * M * si,
                                  (char*)x + b * N * so, accumulate, st, Gx);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace wmg
