// vecops.cu -- Krylov vector kernels (float64) and Haar intergrid kernels.
//
// Deterministic reduction ("DET_SUM"), shared bit for bit with the CPU
// restatement in oracle/solvers.py (det_sum):
//   * element values v_i are formed with individually rounded ops (no FMA),
//   * the vector is cut into 1024-element chunks (zero padded); in chunk c,
//     lane l of a warp sums v[c*1024 + k*32 + l] for k = 0..31 sequentially,
//     then the 32 lane sums are combined by the fixed tree
//     s[l] += s[l + off], off = 16, 8, 4, 2, 1 (lane 0 holds the chunk sum),
//   * the chunk sums are reduced by the same procedure until one value is left.
// Every Krylov dot/norm in the GPU solvers uses it, so GPU and oracle residual
// histories agree to the last bit (SURVEY.md s8(c) "parity protocol").
//
// Haar kernels follow /root/reference/pkg/src/wmgtomo/multilevel.py:36-79
// (coefficients +-fl(fl(1/sqrt 2)^2) = +-0.4999999999999999, 2x2 block in the
// order (2i,2k), (2i,2k+1), (2i+1,2k), (2i+1,2k+1); csr_matvec summation from
// 0.0) and the band accumulation of wtg_apply (multilevel.py:175-198).
#include "common.cuh"

namespace wmg {
namespace vec {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

enum RedOp : int { kDot = 0, kSqDiff = 1, kSum = 2, kDotDiff = 3, kSq = 4 };

struct RedArgs {
  const double* a[8];
  const double* b[8];
  const double* c[8];
  int op[8];
};

__device__ __forceinline__ double combine(int op, double a, double b, double c) {
  if (op == kSum) return a;
  if (op == kSq) return dmul(a, a);
  if (op == kDot) return dmul(a, b);
  if (op == kSqDiff) {
    const double t = dsub(a, b);
    return dmul(t, t);
  }
  return dmul(a, dsub(b, c));   // kDotDiff
}

// level 1: 8 warps per block, one chunk of 1024 elements per warp.  The
// operands of a lane's 32 elements are loaded in two batches of 16 before any
// is summed (a dependent load per element left the small vectors of config 1
// at 19 us per reduction, latency bound); the summation order is unchanged.
__global__ void __launch_bounds__(256) det_level1(long long n, RedArgs A, double* partials,
                                                  long long C) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long chunk = (long long)blockIdx.x * 8 + warp;
  const int k = blockIdx.y;
  if (chunk >= C) return;
  const long long base = chunk * 1024;
  const int op = A.op[k];
  const double* __restrict__ pa = A.a[k];
  const double* __restrict__ pb = A.b[k];
  const double* __restrict__ pc = A.c[k];
  const bool use_b = op != kSum && op != kSq, use_c = op == kDotDiff;
  double s = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double va[16], vb[16], vc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const long long i = base + (h * 16 + q) * 32 + lane;
      const bool ok = i < n;
      va[q] = ok ? pa[i] : 0.0;
      vb[q] = (ok && use_b) ? pb[i] : 0.0;
      vc[q] = (ok && use_c) ? pc[i] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const long long i = base + (h * 16 + q) * 32 + lane;
      const double v = (i < n) ? combine(op, va[q], vb[q], vc[q]) : 0.0;
      s = (h == 0 && q == 0) ? v : dadd(s, v);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s = dadd(s, __shfl_down_sync(0xffffffffu, s, off));
  if (lane == 0) partials[(long long)k * C + chunk] = s;
}

// chunk reduce of one warp over buf[0..len) (zero padded), chunk index c;
// all 32 loads issued before the (unchanged) sequential sum
__device__ __forceinline__ double warp_chunk(const double* buf, long long len, long long c,
                                             int lane) {
  const long long base = c * 1024;
  double v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const long long i = base + r * 32 + lane;
    v[r] = (i < len) ? buf[i] : 0.0;
  }
  double s = v[0];
#pragma unroll
  for (int r = 1; r < 32; ++r) s = dadd(s, v[r]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s = dadd(s, __shfl_down_sync(0xffffffffu, s, off));
  return s;
}

// finish: one block (32 warps) per reduction; level 2 (C <= 2^20 chunk sums,
// i.e. n <= 2^30) into shared memory, level 3 by warp 0.
__global__ void __launch_bounds__(1024) det_finish(const double* partials, long long C,
                                                   double* out) {
  __shared__ double lvl[1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x;
  const double* buf = partials + (long long)k * C;
  if (C == 1) {
    if (threadIdx.x == 0) out[k] = buf[0];
    return;
  }
  const long long C2 = (C + 1023) / 1024;
  for (long long c = warp; c < C2; c += 32) {
    const double s = warp_chunk(buf, C, c, lane);
    if (lane == 0) lvl[c] = s;
  }
  __syncthreads();
  if (C2 == 1) {
    if (threadIdx.x == 0) out[k] = lvl[0];
    return;
  }
  if (warp == 0) {
    const double s = warp_chunk(lvl, C2, 0, lane);
    if (lane == 0) out[k] = s;
  }
}

// max |a - b| (or max |a| when b == nullptr); order independent
__global__ void maxabs_kernel(long long n, const double* a, const double* b,
                              unsigned long long* out) {
  double m = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = b ? fabs(dsub(a[i], b[i])) : fabs(a[i]);
    m = fmax(m, v);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// ---------------------------------------------------------------------------
// elementwise kernels; every op individually rounded, same as numpy
// ---------------------------------------------------------------------------
#define GRID_LOOP(i, n)                                                            \
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (n); \
       i += (long long)gridDim.x * blockDim.x)

// out = y + s * (alpha * x), s = +1 / -1   (numpy: y + alpha*x, y - alpha*x)
__global__ void axpy_kernel(long long n, double* out, const double* y, double alpha, int sgn,
                            const double* x) {
  GRID_LOOP(i, n) {
    const double t = dmul(alpha, x[i]);
    out[i] = sgn > 0 ? dadd(y[i], t) : dsub(y[i], t);
  }
}

// out = a*x + b*y (+ c*z)  evaluated as ((a*x + b*y) + c*z)
__global__ void lincomb_kernel(long long n, double* out, double a, const double* x, double b,
                               const double* y, double c, const double* z) {
  GRID_LOOP(i, n) {
    double t = dadd(dmul(a, x[i]), dmul(b, y[i]));
    if (z) t = dadd(t, dmul(c, z[i]));
    out[i] = t;
  }
}

// BiCGStab direction: p = r + beta * (p - omega * v)   (solvers.py:207)
__global__ void bicg_p_kernel(long long n, double* p, const double* r, double beta, double omega,
                              const double* v) {
  GRID_LOOP(i, n) { p[i] = dadd(r[i], dmul(beta, dsub(p[i], dmul(omega, v[i])))); }
}

// x = x + alpha*ph + omega*sh   (solvers.py:229)
__global__ void bicg_x_kernel(long long n, double* x, double alpha, const double* ph,
                              double omega, const double* sh) {
  GRID_LOOP(i, n) { x[i] = dadd(dadd(x[i], dmul(alpha, ph[i])), dmul(omega, sh[i])); }
}

// out = a * x (scale), or out = x * y elementwise when y != nullptr
__global__ void scale_kernel(long long n, double* out, double a, const double* x,
                             const double* y) {
  GRID_LOOP(i, n) { out[i] = y ? dmul(x[i], y[i]) : dmul(a, x[i]); }
}

// WMG node smoother sweep, fused: z += omega * (c .* (r - az))  (az == nullptr: az = 0);
// the same rounded operations as the unfused axpy / hadamard / axpy sequence
__global__ void smooth_update_kernel(long long n, double* z, double omega, const double* c,
                                     const double* r, const double* az) {
  GRID_LOOP(i, n) {
    const double res = az ? dsub(r[i], az[i]) : r[i];
    z[i] = dadd(z[i], dmul(omega, dmul(c[i], res)));
  }
}

// inverse with the SIRT zero convention: out = s > 0 ? 1/s : 0 (solvers.py:84-85)
__global__ void recip_kernel(long long n, double* out, const double* s) {
  GRID_LOOP(i, n) { out[i] = s[i] > 0.0 ? __drcp_rn(s[i]) : 0.0; }
}

// SIRT update (solvers.py:125-128): upd = c*g; if lam>0: upd -= lam*(c*x); x += upd
__global__ void sirt_update_kernel(long long n, double* x, const double* c, const double* g,
                                   double lam) {
  GRID_LOOP(i, n) {
    double upd = dmul(c[i], g[i]);
    if (lam > 0.0) upd = dsub(upd, dmul(lam, dmul(c[i], x[i])));
    x[i] = dadd(x[i], upd);
  }
}

// out = g + lam*v  (normal_operator, solvers.py:151-153; only when lam != 0)
// out = g - lam*v  (sgn < 0, CGLS gradient W^T r - lam x)
__global__ void add_scaled_kernel(long long n, double* out, const double* g, double lam, int sgn,
                                  const double* v) {
  GRID_LOOP(i, n) {
    const double t = dmul(lam, v[i]);
    out[i] = sgn > 0 ? dadd(g[i], t) : dsub(g[i], t);
  }
}

// w = w - sum_i h_i v_i, i ascending (classical Gram-Schmidt update, GMRES)
__global__ void cgs_update_kernel(long long n, int k, double* w, const double* V, long long ldv,
                                  const double* h) {
  GRID_LOOP(i, n) {
    double t = w[i];
    for (int q = 0; q < k; ++q) t = dsub(t, dmul(h[q], V[(long long)q * ldv + i]));
    w[i] = t;
  }
}

// out = sum_i c_i v_i, i ascending starting from c_0 v_0 (GMRES solution update)
__global__ void combo_kernel(long long n, int k, double* out, const double* V, long long ldv,
                             const double* cf, int accumulate) {
  GRID_LOOP(i, n) {
    double t = accumulate ? out[i] : 0.0;
    for (int q = 0; q < k; ++q) {
      const double pr = dmul(cf[q], V[(long long)q * ldv + i]);
      t = (q == 0 && !accumulate) ? pr : dadd(t, pr);
    }
    out[i] = t;
  }
}

// dtype casts for the fp32-projector / fp64-Krylov configurations
__global__ void cast_f64_f32(long long n, float* out, const double* in) {
  GRID_LOOP(i, n) { out[i] = (float)in[i]; }
}
__global__ void cast_f32_f64(long long n, double* out, const float* in) {
  GRID_LOOP(i, n) { out[i] = (double)in[i]; }
}

// ---------------------------------------------------------------------------
// Haar intergrid operators on a side x side row-major grid
// band: 0 LL, 1 LH, 2 HL, 3 HH.  kron(row factor, col factor) with the row
// factor acting along y (multilevel.py:61-79): LH = kron(J, S), HL = kron(S, J).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void band_signs(int band, double& s00, double& s01, double& s10,
                                           double& s11) {
  haar_band_signs(band, s00, s01, s10, s11);
}

// coarse[b][(i,k)] = R_b fine, for the bands in mask (bit b); out laid out as
// out + b_slot * side^2/4 where b_slot counts the selected bands in order
__global__ void haar_restrict_kernel(int side, const double* __restrict__ fine, int band_mask,
                                     double* __restrict__ out) {
  const int hs = side / 2;
  const long long nc = (long long)hs * hs;
  GRID_LOOP(q, nc) {
    const int i = (int)(q / hs), k = (int)(q % hs);
    const long long f0 = (long long)(2 * i) * side + 2 * k;
    const double x00 = fine[f0], x01 = fine[f0 + 1];
    const double x10 = fine[f0 + side], x11 = fine[f0 + side + 1];
    int slot = 0;
    for (int b = 0; b < 4; ++b) {
      if (!((band_mask >> b) & 1)) continue;
      double s00, s01, s10, s11;
      band_signs(b, s00, s01, s10, s11);
      double acc = 0.0;
      acc = dadd(acc, dmul(s00, x00));
      acc = dadd(acc, dmul(s01, x01));
      acc = dadd(acc, dmul(s10, x10));
      acc = dadd(acc, dmul(s11, x11));
      out[(long long)slot * nc + q] = acc;
      ++slot;
    }
  }
}

// Band paths of a batch of WMG nodes: wmg::BandPaths (common.cuh).
// fine_i (n x n) = R_{b0}^T ... R_{b(k-1)}^T coarse_i, coarsest level first:
// the level-by-level prolongations (haar_prolong_kernel) fused into one pass,
// the same sequence of sign * h products per fine pixel (bit-identical).
// blockIdx.y = batch item; coarse items nc apart, fine items n^2 apart.
__global__ void haar_prolong_path_kernel(int n, BandPaths bp, const double* __restrict__ coarse,
                                         double* __restrict__ fine) {
  const int k = bp.depth, item = blockIdx.y;
  const int sc = n >> k;
  const long long nf = (long long)n * n;
  const double* cin = coarse + (long long)item * sc * sc;
  double* fout = fine + (long long)item * nf;
  GRID_LOOP(f, nf) {
    const int r = (int)(f / n), c = (int)(f % n);
    fout[f] = haar_path_value(bp, item, cin, sc, r, c);
  }
}

// coarse_i = R_{b(k-1)} ... R_{b0} fine_i: the level-by-level restrictions
// (haar_restrict_kernel, one band each) fused: each output sums its 4^k fine
// pixels in nested 2 x 2 groups, children in CSR order, every partial sum
// formed exactly as the per-level kernel forms it (bit-identical).
__global__ void haar_restrict_path_kernel(int n, BandPaths bp, const double* __restrict__ fine,
                                          double* __restrict__ coarse) {
  const int k = bp.depth, item = blockIdx.y;
  const unsigned code = bp.code[item];
  const int sc = n >> k;
  const long long nc = (long long)sc * sc;
  const double* fin = fine + (long long)item * n * n;
  double* cout = coarse + (long long)item * nc;
  GRID_LOOP(q, nc) {
    const int qi = (int)(q / sc), qk = (int)(q % sc);
    double acc[12];
    for (int lv = 0; lv < k; ++lv) acc[lv] = 0.0;
    double v = 0.0;
    const int leaves = 1 << (2 * k);
    for (int t = 0; t < leaves; ++t) {
      int r = qi << k, c = qk << k;
      // digit of level lv is bits [2 lv, 2 lv + 1] of t (level 0 = finest)
      for (int lv = 0; lv < k; ++lv) {
        const int dg = (t >> (2 * lv)) & 3;
        r += (dg >> 1) << lv;
        c += (dg & 1) << lv;
      }
      v = fin[(long long)r * n + c];
      for (int lv = 0; lv < k; ++lv) {
        const int dg = (t >> (2 * lv)) & 3;
        double s[4];
        band_signs((code >> (2 * lv)) & 3, s[0], s[1], s[2], s[3]);
        acc[lv] = dadd(acc[lv], dmul(s[dg], v));
        if (dg != 3) break;
        v = acc[lv];
        acc[lv] = 0.0;
      }
    }
    cout[q] = v;
  }
}

// fine = (accumulate ? fine : 0) + R_b^T coarse  (one product per fine pixel)
__global__ void haar_prolong_kernel(int side, const double* __restrict__ coarse, int band,
                                    double* __restrict__ fine, int accumulate) {
  const long long nf = (long long)side * side;
  const int hs = side / 2;
  double s[4];
  band_signs(band, s[0], s[1], s[2], s[3]);
  GRID_LOOP(f, nf) {
    const int r = (int)(f / side), col = (int)(f % side);
    const int q = (r >> 1) * hs + (col >> 1);
    const double v = dmul(s[((r & 1) << 1) | (col & 1)], coarse[q]);
    fine[f] = accumulate ? dadd(fine[f], v) : v;
  }
}


// Batched forms for the sibling batches of the hybrid cycle (one launch per
// batch instead of one per node; every element computed exactly as by the
// single-item kernels above).  blockIdx.y = batch item.
__global__ void haar_restrict_batch_kernel(int side, const double* __restrict__ fine,
                                           int band_mask, double* __restrict__ out) {
  const int item = blockIdx.y;
  const int hs = side / 2;
  const long long nc = (long long)hs * hs;
  const int nb = __popc(band_mask & 15);
  fine += (long long)item * side * side;
  out += (long long)item * nb * nc;
  GRID_LOOP(q, nc) {
    const int i = (int)(q / hs), k = (int)(q % hs);
    const long long f0 = (long long)(2 * i) * side + 2 * k;
    const double x00 = fine[f0], x01 = fine[f0 + 1];
    const double x10 = fine[f0 + side], x11 = fine[f0 + side + 1];
    int slot = 0;
    for (int b = 0; b < 4; ++b) {
      if (!((band_mask >> b) & 1)) continue;
      double s00, s01, s10, s11;
      band_signs(b, s00, s01, s10, s11);
      double acc = 0.0;
      acc = dadd(acc, dmul(s00, x00));
      acc = dadd(acc, dmul(s01, x01));
      acc = dadd(acc, dmul(s10, x10));
      acc = dadd(acc, dmul(s11, x11));
      out[(long long)slot * nc + q] = acc;
      ++slot;
    }
  }
}

// fine_b = (accumulate ? fine_b : first product) + R_{band 1}^T c_b1 + ... in band
// order, one dadd per band exactly as successive haar_prolong_kernel calls
struct BandList {
  int n;
  int code[4];
};
__global__ void haar_prolong_batch_kernel(int side, BandList bl, const double* __restrict__ coarse,
                                          double* __restrict__ fine, int accumulate) {
  const int item = blockIdx.y;
  const long long nf = (long long)side * side;
  const int hs = side / 2;
  const long long nc = (long long)hs * hs;
  coarse += (long long)item * bl.n * nc;
  fine += (long long)item * nf;
  GRID_LOOP(f, nf) {
    const int r = (int)(f / side), col = (int)(f % side);
    const long long q = (long long)(r >> 1) * hs + (col >> 1);
    const int sl = ((r & 1) << 1) | (col & 1);
    double x = 0.0;
    for (int i = 0; i < bl.n; ++i) {
      double s[4];
      band_signs(bl.code[i], s[0], s[1], s[2], s[3]);
      const double v = dmul(s[sl], coarse[(long long)i * nc + q]);
      x = (i == 0 && !accumulate) ? v : dadd(i == 0 ? fine[f] : x, v);
    }
    fine[f] = x;
  }
}

// z_b += omega_b * (c_b .* (r_b - az_b)) for a batch of node smoothers
constexpr int kSmoothBatch = 64;
struct SmoothArgs {
  double omega[kSmoothBatch];
  const double* c[kSmoothBatch];
};
__global__ void smooth_update_batch_kernel(long long n, double* z, SmoothArgs A, const double* r,
                                           const double* az) {
  const int item = blockIdx.y;
  const double omega = A.omega[item];
  const double* __restrict__ c = A.c[item];
  z += item * n;
  r += item * n;
  if (az) az += item * n;
  GRID_LOOP(i, n) {
    const double res = az ? dsub(r[i], az[i]) : r[i];
    z[i] = dadd(z[i], dmul(omega, dmul(c[i], res)));
  }
}

// ---------------------------------------------------------------------------
// Batched dense float64 GEMV for the WMG coarse solves: y_b = A_b x_b with the
// stored SPD inverse A_b (p x p, row-major).  HBM-bound: every element of A is
// read once, coalesced; x_b is staged in shared memory; each warp reduces its
// rows with a fixed shuffle tree (deterministic).
// ---------------------------------------------------------------------------

// rpw rows per warp (8 warps per block): chosen by the launcher so that even a
// single 4096^2 matrix spreads over enough blocks to stream at HBM rate
__global__ void __launch_bounds__(256) batched_gemv_kernel(int p, const double* __restrict__ A,
                                                           long long sA,
                                                           const double* __restrict__ x,
                                                           long long sx, double* __restrict__ y,
                                                           long long sy, int rpw) {
  extern __shared__ double xs[];
  const int b = blockIdx.y;
  const double* Ab = A + (long long)b * sA;
  const double* xb = x + (long long)b * sx;
  for (int i = threadIdx.x; i < p; i += blockDim.x) xs[i] = xb[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * 8 * rpw + warp * rpw;
  for (int rr = 0; rr < rpw; ++rr) {
    const int row = row0 + rr;
    if (row >= p) break;
    const double* Ar = Ab + (long long)row * p;
    double acc = 0.0;
    if ((p & 1) == 0) {
      // 16-byte loads, two accumulators, 4 loads in flight per lane: the
      // stored inverses are streamed at HBM rate
      const double2* Ar2 = reinterpret_cast<const double2*>(Ar);
      const double2* xs2 = reinterpret_cast<const double2*>(xs);
      double acc1 = 0.0;
      const int p2 = p >> 1;
#pragma unroll 4
      for (int c = lane; c < p2; c += 32) {
        const double2 a = __ldg(Ar2 + c);
        const double2 xv = xs2[c];
        acc = fma(a.x, xv.x, acc);
        acc1 = fma(a.y, xv.y, acc1);
      }
      acc += acc1;
    } else {
      for (int c = lane; c < p; c += 32) acc = fma(__ldg(Ar + c), xs[c], acc);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
    if (lane == 0) y[(long long)b * sy + row] = acc;
  }
}


// ---------------------------------------------------------------------------
// device-resident Krylov scalars (graph-capturable solver iterations)
// ---------------------------------------------------------------------------
// out = y + sgn * (coef[0] * x)
__global__ void axpy_dev_kernel(long long n, double* out, const double* y,
                                const double* __restrict__ coef, int sgn, const double* x) {
  const double alpha = coef[0];
  GRID_LOOP(i, n) {
    const double t = dmul(alpha, x[i]);
    out[i] = sgn > 0 ? dadd(y[i], t) : dsub(y[i], t);
  }
}
// out = a * x + coef[0] * y
__global__ void lincomb_dev_kernel(long long n, double* out, double a, const double* x,
                                   const double* __restrict__ coef, const double* y) {
  const double b = coef[0];
  GRID_LOOP(i, n) { out[i] = dadd(dmul(a, x[i]), dmul(b, y[i])); }
}

// CGLS / flexible PCG-NE scalar recurrences on the slot vector S:
//  S[0] gamma, S[1] <q,q>, S[2] <p,p>, S[3] alpha, S[4] beta, S[5] <s,s>,
//  S[6] <z,s>, S[7] <z,s-s_old>, S[8] breakdown flag
// op 0: delta = qq (+ lam pp); alpha = gamma / delta (0 and flag on breakdown)
// op 1: beta = ss / gamma; gamma = ss           (CGLS)
// op 2: beta = pr / gamma; gamma = zs           (flexible PCG-NE)
__global__ void cgls_scalars_kernel(double* S, double lam, int op) {
  if (threadIdx.x || blockIdx.x) return;
  if (op == 0) {
    const double delta = lam != 0.0 ? dadd(S[1], dmul(lam, S[2])) : S[1];
    const bool ok = delta > 0.0 && isfinite(delta);
    S[3] = ok ? S[0] / delta : 0.0;
    if (!ok) S[8] = 1.0;
  } else if (op == 1) {
    S[4] = S[5] / S[0];
    S[0] = S[5];
  } else {
    S[4] = S[7] / S[0];
    S[0] = S[6];
  }
}

// --- fused forms (unsharded, vectors of at most 2^20 elements) ---
// The reduction's last level, the scalar recurrence and the vector update in
// one kernel: every block finishes the <= 1024 level-1 chunk sums itself (one
// warp, the order det_finish uses, so every block holds the bit-identical
// value), forms the coefficient and updates its share of the vectors; block 0
// publishes the scalars.  Same arithmetic as det_finish + cgls_scalars +
// axpy_dev / lincomb_dev, five launches fewer per iteration.  gamma lives in
// two slots so that no block reads a slot another block writes in the same
// launch: the update kernel reads S[11] and commits it to S[0], the direction
// kernel reads S[0] and writes the new gamma to S[11].
__device__ __forceinline__ double finish_small(const double* partials, long long C, int lane) {
  if (C == 1) return partials[0];
  return __shfl_sync(0xffffffffu, warp_chunk(partials, C, 0, lane), 0);
}

// x += alpha p, r -= alpha q with alpha = gamma / (<q,q> + lam <p,p>); partials:
// level 1 of <q,q>; partials_pp (lam != 0 only): level 1 of <p,p>
__global__ void __launch_bounds__(256) cgls_update_kernel(long long n_img, long long n_sino,
                                                          double* x, const double* p, double* r,
                                                          const double* q,
                                                          const double* partials, long long C,
                                                          const double* partials_pp,
                                                          long long Cpp, double lam, double* S) {
  __shared__ double sh_alpha;
  if (threadIdx.x < 32) {
    const double qq = finish_small(partials, C, threadIdx.x);
    const double pp = lam != 0.0 ? finish_small(partials_pp, Cpp, threadIdx.x) : 0.0;
    if (threadIdx.x == 0) {
      const double gamma = S[11];
      const double delta = lam != 0.0 ? dadd(qq, dmul(lam, pp)) : qq;
      const bool ok = delta > 0.0 && isfinite(delta);
      const double alpha = ok ? gamma / delta : 0.0;
      sh_alpha = alpha;
      if (blockIdx.x == 0) {
        S[1] = qq;
        S[2] = pp;
        S[3] = alpha;
        S[0] = gamma;
        if (!ok) S[8] = 1.0;
      }
    }
  }
  __syncthreads();
  const double alpha = sh_alpha;
  GRID_LOOP(i, n_img) { x[i] = dadd(x[i], dmul(alpha, p[i])); }
  GRID_LOOP(j, n_sino) { r[j] = dsub(r[j], dmul(alpha, q[j])); }
}

// p = z + beta p.  mode 1 (CGLS): partials of <s,s>; beta = ss / gamma, gamma' = ss.
// mode 2 (flexible PCG-NE): partials of <s,s>, <z,s>, <z,s-s_old>; beta = pr / gamma,
// gamma' = zs.
__global__ void __launch_bounds__(256) cgls_direction_kernel(long long n, double* p,
                                                             const double* z,
                                                             const double* partials, long long C,
                                                             int mode, double* S) {
  __shared__ double sh_beta;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const double ss = finish_small(partials, C, lane);
    double zs = 0.0, pr = 0.0;
    if (mode == 2) {
      zs = finish_small(partials + C, C, lane);
      pr = finish_small(partials + 2 * C, C, lane);
    }
    if (lane == 0) {
      const double gamma = S[0];
      const double beta = (mode == 1 ? ss : pr) / gamma;
      sh_beta = beta;
      if (blockIdx.x == 0) {
        S[5] = ss;
        if (mode == 2) {
          S[6] = zs;
          S[7] = pr;
        }
        S[4] = beta;
        S[11] = mode == 1 ? ss : zs;
      }
    }
  }
  __syncthreads();
  const double beta = sh_beta;
  GRID_LOOP(i, n) { p[i] = dadd(dmul(1.0, z[i]), dmul(beta, p[i])); }
}

}  // namespace vec

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static inline unsigned grid_for(long long n, int tpb) {
  long long g = (n + tpb - 1) / tpb;
  if (g > 148LL * 32) g = 148LL * 32;
  if (g < 1) g = 1;
  return (unsigned)g;
}

cudaError_t det_reduce(long long n, int K, const int* ops, const double* const* a,
                       const double* const* b, const double* const* c, double* scratch,
                       double* out, cudaStream_t st) {
  if (K < 1 || K > 8) return cudaErrorInvalidValue;
  vec::RedArgs A;
  for (int k = 0; k < 8; ++k) {
    A.a[k] = k < K ? a[k] : nullptr;
    A.b[k] = (k < K && b) ? b[k] : nullptr;
    A.c[k] = (k < K && c) ? c[k] : nullptr;
    A.op[k] = k < K ? ops[k] : 0;
  }
  if (n <= 0) {
    return out ? cudaMemsetAsync(out, 0, sizeof(double) * K, st) : cudaErrorInvalidValue;
  }
  const long long C = (n + 1023) / 1024;
  if (C > 1024LL * 1024LL) return cudaErrorInvalidValue;
  dim3 grid((unsigned)((C + 7) / 8), K);
  vec::det_level1<<<grid, 256, 0, st>>>(n, A, scratch, C);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !out) return e;   // out == nullptr: level-1 chunk sums only
  vec::det_finish<<<K, 1024, 0, st>>>(scratch, C, out);
  return cudaGetLastError();
}

// fused CGLS steps on the level-1 chunk sums a det_reduce(..., out = nullptr) left
// in ``partials`` (reduction k at partials + k * C, C = ceil(n / 1024) <= 1024)
cudaError_t cgls_update(long long n_img, long long n_sino, double* x, const double* p, double* r,
                        const double* q, const double* partials, const double* partials_pp,
                        double lam, double* S, cudaStream_t st) {
  const long long C = (n_sino + 1023) / 1024, Cpp = (n_img + 1023) / 1024;
  if (n_img <= 0 || n_sino <= 0 || C > 1024 || Cpp > 1024) return cudaErrorInvalidValue;
  if (lam != 0.0 && !partials_pp) return cudaErrorInvalidValue;
  const long long nmax = n_img > n_sino ? n_img : n_sino;
  vec::cgls_update_kernel<<<grid_for(nmax, 256), 256, 0, st>>>(n_img, n_sino, x, p, r, q,
                                                               partials, C, partials_pp, Cpp,
                                                               lam, S);
  return cudaGetLastError();
}

cudaError_t cgls_direction(long long n, double* p, const double* z, const double* partials,
                           int mode, double* S, cudaStream_t st) {
  const long long C = (n + 1023) / 1024;
  if (n <= 0 || C > 1024 || (mode != 1 && mode != 2)) return cudaErrorInvalidValue;
  vec::cgls_direction_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, p, z, partials, C, mode, S);
  return cudaGetLastError();
}

long long det_scratch_len(long long n, int K) { return ((n + 1023) / 1024 + 1) * (long long)K; }

cudaError_t maxabs(long long n, const double* a, const double* b, double* out_bits,
                   cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out_bits, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  if (n <= 0) return cudaSuccess;
  vec::maxabs_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, a, b, (unsigned long long*)out_bits);
  return cudaGetLastError();
}

#define LAUNCH_EW(kernel, n, ...)                                        \
  do {                                                                   \
    if ((n) <= 0) return cudaSuccess;                                    \
    kernel<<<grid_for((n), 256), 256, 0, st>>>((n), __VA_ARGS__);        \
    return cudaGetLastError();                                           \
  } while (0)

cudaError_t ew_axpy(long long n, double* out, const double* y, double alpha, int sgn,
                    const double* x, cudaStream_t st) {
  LAUNCH_EW(vec::axpy_kernel, n, out, y, alpha, sgn, x);
}
cudaError_t ew_lincomb(long long n, double* out, double a, const double* x, double b,
                       const double* y, double c, const double* z, cudaStream_t st) {
  LAUNCH_EW(vec::lincomb_kernel, n, out, a, x, b, y, c, z);
}
cudaError_t ew_bicg_p(long long n, double* p, const double* r, double beta, double omega,
                      const double* v, cudaStream_t st) {
  LAUNCH_EW(vec::bicg_p_kernel, n, p, r, beta, omega, v);
}
cudaError_t ew_bicg_x(long long n, double* x, double alpha, const double* ph, double omega,
                      const double* sh, cudaStream_t st) {
  LAUNCH_EW(vec::bicg_x_kernel, n, x, alpha, ph, omega, sh);
}
cudaError_t ew_scale(long long n, double* out, double a, const double* x, const double* y,
                     cudaStream_t st) {
  LAUNCH_EW(vec::scale_kernel, n, out, a, x, y);
}
cudaError_t ew_recip(long long n, double* out, const double* s, cudaStream_t st) {
  LAUNCH_EW(vec::recip_kernel, n, out, s);
}
cudaError_t ew_smooth_update(long long n, double* z, double omega, const double* c,
                            const double* r, const double* az, cudaStream_t st) {
  LAUNCH_EW(vec::smooth_update_kernel, n, z, omega, c, r, az);
}
cudaError_t ew_sirt_update(long long n, double* x, const double* c, const double* g, double lam,
                           cudaStream_t st) {
  LAUNCH_EW(vec::sirt_update_kernel, n, x, c, g, lam);
}
cudaError_t ew_add_scaled(long long n, double* out, const double* g, double lam, int sgn,
                          const double* v, cudaStream_t st) {
  LAUNCH_EW(vec::add_scaled_kernel, n, out, g, lam, sgn, v);
}
cudaError_t ew_cgs_update(long long n, int k, double* w, const double* V, long long ldv,
                          const double* h, cudaStream_t st) {
  LAUNCH_EW(vec::cgs_update_kernel, n, k, w, V, ldv, h);
}
cudaError_t ew_combo(long long n, int k, double* out, const double* V, long long ldv,
                     const double* cf, int accumulate, cudaStream_t st) {
  LAUNCH_EW(vec::combo_kernel, n, k, out, V, ldv, cf, accumulate);
}
cudaError_t ew_cast(long long n, int to_f32, void* out, const void* in, cudaStream_t st) {
  if (to_f32) {
    LAUNCH_EW(vec::cast_f64_f32, n, (float*)out, (const double*)in);
  } else {
    LAUNCH_EW(vec::cast_f32_f64, n, (double*)out, (const float*)in);
  }
}

cudaError_t batched_gemv(int batch, int p, const double* A, long long sA, const double* x,
                         long long sx, double* y, long long sy, cudaStream_t st) {
  if (batch <= 0 || p <= 0) return cudaSuccess;
  const size_t smem = sizeof(double) * (size_t)p;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(vec::batched_gemv_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  // rows per warp: 4 when the batch alone fills the GPU, down to 1 otherwise
  int rpw = 4;
  while (rpw > 1 && (long long)((p + 8 * rpw - 1) / (8 * rpw)) * batch < 4LL * 148) rpw >>= 1;
  dim3 grid((p + 8 * rpw - 1) / (8 * rpw), batch);
  vec::batched_gemv_kernel<<<grid, 256, smem, st>>>(p, A, sA, x, sx, y, sy, rpw);
  return cudaGetLastError();
}

cudaError_t ew_axpy_dev(long long n, double* out, const double* y, const double* coef, int sgn,
                        const double* x, cudaStream_t st) {
  LAUNCH_EW(vec::axpy_dev_kernel, n, out, y, coef, sgn, x);
}
cudaError_t ew_lincomb_dev(long long n, double* out, double a, const double* x,
                           const double* coef, const double* y, cudaStream_t st) {
  LAUNCH_EW(vec::lincomb_dev_kernel, n, out, a, x, coef, y);
}
cudaError_t cgls_scalars(double* S, double lam, int op, cudaStream_t st) {
  vec::cgls_scalars_kernel<<<1, 32, 0, st>>>(S, lam, op);
  return cudaGetLastError();
}

cudaError_t haar_restrict(int side, const double* fine, int band_mask, double* out,
                          cudaStream_t st) {
  const long long nc = (long long)(side / 2) * (side / 2);
  if (nc <= 0) return cudaSuccess;
  vec::haar_restrict_kernel<<<grid_for(nc, 256), 256, 0, st>>>(side, fine, band_mask, out);
  return cudaGetLastError();
}

cudaError_t haar_prolong_path(int n, int depth, int batch, const int* bands,
                              const double* coarse, double* fine, cudaStream_t st) {
  const int sc = n >> depth;
  for (int b0 = 0; b0 < batch; b0 += kPathBatch) {
    const int nb = batch - b0 < kPathBatch ? batch - b0 : kPathBatch;
    BandPaths bp;
    bp.depth = depth;
    for (int i = 0; i < nb; ++i) {
      unsigned code = 0;
      for (int lv = 0; lv < depth; ++lv) code |= (unsigned)(bands[(b0 + i) * depth + lv] & 3) << (2 * lv);
      bp.code[i] = (unsigned short)code;
    }
    const long long nf = (long long)n * n;
    dim3 grid(grid_for(nf, 256), nb);
    vec::haar_prolong_path_kernel<<<grid, 256, 0, st>>>(n, bp, coarse + (long long)b0 * sc * sc,
                                                        fine + (long long)b0 * nf);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t haar_restrict_path(int n, int depth, int batch, const int* bands, const double* fine,
                               double* coarse, cudaStream_t st) {
  const int sc = n >> depth;
  for (int b0 = 0; b0 < batch; b0 += kPathBatch) {
    const int nb = batch - b0 < kPathBatch ? batch - b0 : kPathBatch;
    BandPaths bp;
    bp.depth = depth;
    for (int i = 0; i < nb; ++i) {
      unsigned code = 0;
      for (int lv = 0; lv < depth; ++lv) code |= (unsigned)(bands[(b0 + i) * depth + lv] & 3) << (2 * lv);
      bp.code[i] = (unsigned short)code;
    }
    const long long nc = (long long)sc * sc;
    dim3 grid(grid_for(nc, 128), nb);
    vec::haar_restrict_path_kernel<<<grid, 128, 0, st>>>(n, bp, fine + (long long)b0 * n * n,
                                                         coarse + (long long)b0 * nc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t haar_prolong(int side, const double* coarse, int band, double* fine, int accumulate,
                         cudaStream_t st) {
  const long long nf = (long long)side * side;
  if (nf <= 0) return cudaSuccess;
  vec::haar_prolong_kernel<<<grid_for(nf, 256), 256, 0, st>>>(side, coarse, band, fine,
                                                              accumulate);
  return cudaGetLastError();
}

cudaError_t haar_restrict_batch(int side, int batch, const double* fine, int band_mask,
                                double* out, cudaStream_t st) {
  const long long nc = (long long)(side / 2) * (side / 2);
  if (nc <= 0 || batch <= 0) return cudaSuccess;
  dim3 grid(grid_for(nc, 256), batch);
  vec::haar_restrict_batch_kernel<<<grid, 256, 0, st>>>(side, fine, band_mask, out);
  return cudaGetLastError();
}

cudaError_t haar_prolong_batch(int side, int batch, int nbands, const int* bands,
                               const double* coarse, double* fine, int accumulate,
                               cudaStream_t st) {
  const long long nf = (long long)side * side;
  if (nf <= 0 || batch <= 0 || nbands <= 0) return cudaSuccess;
  vec::BandList bl;
  bl.n = nbands;
  for (int i = 0; i < 4; ++i) bl.code[i] = i < nbands ? (bands[i] & 3) : 0;
  dim3 grid(grid_for(nf, 256), batch);
  vec::haar_prolong_batch_kernel<<<grid, 256, 0, st>>>(side, bl, coarse, fine, accumulate);
  return cudaGetLastError();
}

cudaError_t ew_smooth_update_batch(long long n, int batch, double* z, const double* omegas,
                                   const double* const* cs, const double* r, const double* az,
                                   cudaStream_t st) {
  if (n <= 0 || batch <= 0) return cudaSuccess;
  for (int b0 = 0; b0 < batch; b0 += vec::kSmoothBatch) {
    const int nb = batch - b0 < vec::kSmoothBatch ? batch - b0 : vec::kSmoothBatch;
    vec::SmoothArgs A;
    for (int i = 0; i < nb; ++i) {
      A.omega[i] = omegas[b0 + i];
      A.c[i] = cs[b0 + i];
    }
    dim3 grid(grid_for(n, 256), nb);
    vec::smooth_update_batch_kernel<<<grid, 256, 0, st>>>(n, z + (long long)b0 * n, A,
                                                          r + (long long)b0 * n,
                                                          az ? az + (long long)b0 * n : nullptr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace wmg
