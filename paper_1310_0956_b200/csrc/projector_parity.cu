// projector_parity.cu -- bit-exact float64 line-intersection projector pair.
//
// These kernels reproduce, entry for entry and sum for sum, the reference's
// stored system matrix and scipy's SpMV summation orders:
//
//  * weights   : /root/reference/pkg/src/wmgtomo/geometry.py:88-128
//                (crossings t = (line - o.c)/(-s), (line - o.s)/c; sorted;
//                 seg = t[q+1]-t[q] > 1e-12; midpoint floor -> pixel)
//  * W x       : geometry.py:200-206 -> csr_matvec: per ray, 0.0 + w1 x1 + ...
//                in ascending flat pixel index, every product rounded (no FMA)
//  * W^T y     : geometry.py:209-215 / solvers.py:111 -> per pixel, ascending
//                ray index (angle-major, detector ascending)
//  * row sums  : solvers.py:81 -> np.add.reduceat = first + numpy pairwise(rest)
//  * col sums  : solvers.py:82 -> ones @ W (same order as W^T y)
//
// All float64 arithmetic goes through __dadd_rn/__dmul_rn/__ddiv_rn so the
// compiler can neither contract into FMA nor reassociate.  The forward kernel
// is ray-driven (one thread per ray, slab walk rows top->bottom, columns
// ascending inside a row = ascending flat index).  The backprojector is an
// atomics-free pixel-driven gather (one thread per pixel, angles ascending,
// detectors ascending).  A segment whose midpoint falls outside the slab the
// walk expects (possible only for segments of length ~1e-12 near a grid corner)
// is counted in a device "anomaly" counter; the parity tests require zero.
#include "joseph_walker.cuh"

namespace wmg {
namespace parity {

template <typename Walker>
__global__ void fwd_kernel(GeomDev G, const double* __restrict__ x, double* __restrict__ y,
                           int* __restrict__ anomaly) {
  const long long ray = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (ray >= (long long)G.m * G.d) return;
  const int a = (int)(ray / G.d), j = (int)(ray % G.d);
  const AngleParams P = G.ang[a];
  Walker wk;
  wk.init(G.n, G.d, P.c, P.s, j);
  double acc = 0.0;
  long long flat;
  double w;
  while (wk.next(flat, w)) acc = dadd(acc, dmul(w, __ldg(x + flat)));
  y[ray] = acc;
  if (wk.anomalies && anomaly) atomicAdd(anomaly, wk.anomalies);
}

// CSR export: counts (pass 0) then fill at indptr (pass 1)
template <typename Walker>
__global__ void csr_kernel(GeomDev G, int pass, long long* __restrict__ counts,
                           const long long* __restrict__ indptr, long long* __restrict__ cols,
                           double* __restrict__ vals, int* __restrict__ anomaly) {
  const long long ray = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (ray >= (long long)G.m * G.d) return;
  const int a = (int)(ray / G.d), j = (int)(ray % G.d);
  const AngleParams P = G.ang[a];
  Walker wk;
  wk.init(G.n, G.d, P.c, P.s, j);
  long long flat, cnt = 0;
  double w;
  if (pass == 0) {
    while (wk.next(flat, w)) ++cnt;
    counts[ray] = cnt;
    if (wk.anomalies && anomaly) atomicAdd(anomaly, wk.anomalies);
  } else {
    long long base = indptr[ray];
    while (wk.next(flat, w)) {
      cols[base + cnt] = flat;
      vals[base + cnt] = w;
      ++cnt;
    }
  }
}

// numpy pairwise sum pulled from the walker (loops_utils.h.src, block 128)
template <typename Walker>
__device__ __forceinline__ double pull(Walker& wk) {
  long long f;
  double w = 0.0;
  wk.next(f, w);
  return w;
}

// one leaf block of numpy's pairwise sum (n <= 128)
template <typename Walker>
__device__ double pairwise_leaf(Walker& wk, long long n) {
  if (n < 8) {
    double r = -0.0;
    for (long long i = 0; i < n; ++i) r = dadd(r, pull(wk));
    return r;
  }
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = pull(wk);
  long long i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = dadd(acc[q], pull(wk));
  }
  double r = dadd(dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3])),
                  dadd(dadd(acc[4], acc[5]), dadd(acc[6], acc[7])));
  for (; i < n; ++i) r = dadd(r, pull(wk));
  return r;
}

// numpy pairwise sum of the next n walker entries, evaluated with an explicit
// post-order task stack (no device recursion): split n -> (h, n - h) with
// h = n/2 - (n/2) % 8 until n <= 128, then lhs + rhs.
template <typename Walker>
__device__ double pairwise_pull(Walker& wk, long long n) {
  long long task[48];      // >= 0: evaluate a node of that size; -1: combine
  double val[24];
  int nt = 0, nv = 0;
  task[nt++] = n;
  while (nt > 0) {
    const long long m = task[--nt];
    if (m < 0) {
      const double b = val[--nv];
      const double a = val[--nv];
      val[nv++] = dadd(a, b);
    } else if (m <= 128) {
      val[nv++] = pairwise_leaf(wk, m);
    } else {
      long long h = m / 2;
      h -= h % 8;
      task[nt++] = -1;        // combine after both halves
      task[nt++] = m - h;     // right half (evaluated second)
      task[nt++] = h;         // left half (evaluated first)
    }
  }
  return val[0];
}

template <typename Walker>
__global__ void rowsum_kernel(GeomDev G, double* __restrict__ out) {
  const long long ray = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (ray >= (long long)G.m * G.d) return;
  const int a = (int)(ray / G.d), j = (int)(ray % G.d);
  const AngleParams P = G.ang[a];
  Walker wk;
  wk.init(G.n, G.d, P.c, P.s, j);
  long long flat, cnt = 0;
  double w;
  while (wk.next(flat, w)) ++cnt;
  if (cnt == 0) { out[ray] = 0.0; return; }
  wk.init(G.n, G.d, P.c, P.s, j);
  const double first = pull(wk);
  out[ray] = dadd(first, pairwise_pull(wk, cnt - 1));
}

// Pixel-driven exact backprojection.  y == nullptr means y = 1 (column sums).
template <bool kAccumulate>
__global__ void bwd_kernel(GeomDev G, const double* __restrict__ y, double* __restrict__ x,
                           int* __restrict__ anomaly) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = G.n;
  if (p >= (long long)n * n) return;
  const int row = (int)(p / n), ix = (int)(p % n);
  const int iy = n - 1 - row;
  const double half = (double)n * 0.5;
  const double xl = dsub((double)ix, half), xr = dsub((double)(ix + 1), half);
  const double yb = dsub((double)iy, half), yt = dsub((double)(iy + 1), half);
  const double dc = (double)(G.d - 1) * 0.5;
  double acc = kAccumulate ? x[p] : 0.0;
  int anomalies = 0;
  for (int a = 0; a < G.m; ++a) {
    const double c = G.ang[a].c, s = G.ang[a].s;
    // candidate detectors from the projected pixel corners (margin 1)
    const double u1 = xl * c + yb * s, u2 = xr * c + yb * s;
    const double u3 = xl * c + yt * s, u4 = xr * c + yt * s;
    const double umin = fmin(fmin(u1, u2), fmin(u3, u4));
    const double umax = fmax(fmax(u1, u2), fmax(u3, u4));
    int j0 = (int)floor(umin + dc) - 1;
    int j1 = (int)ceil(umax + dc) + 1;
    j0 = max(j0, 0);
    j1 = min(j1, G.d - 1);
    const long long rowbase = (long long)a * G.d;
    for (int j = j0; j <= j1; ++j) {
      RayGeom g;
      g.init(n, G.d, c, s, j);
      double tq, tq1;
      if (g.hasx && g.hasy) {
        const double ta = ddiv(dsub(xl, g.ox), g.dx), tb = ddiv(dsub(xr, g.ox), g.dx);
        const double tc = ddiv(dsub(yb, g.oy), g.dy), td = ddiv(dsub(yt, g.oy), g.dy);
        tq = fmax(fmin(ta, tb), fmin(tc, td));
        tq1 = fmin(fmax(ta, tb), fmax(tc, td));
        if (!(tq1 > tq)) continue;
      } else if (g.hasy) {
        const double tc = ddiv(dsub(yb, g.oy), g.dy), td = ddiv(dsub(yt, g.oy), g.dy);
        tq = fmin(tc, td);
        tq1 = fmax(tc, td);
      } else {
        const double ta = ddiv(dsub(xl, g.ox), g.dx), tb = ddiv(dsub(xr, g.ox), g.dx);
        tq = fmin(ta, tb);
        tq1 = fmax(ta, tb);
      }
      int jx, jy;
      double seg;
      if (!g.segment(tq, tq1, jx, jy, seg)) continue;
      if (jx != ix || jy != iy) {
        // the midpoint rule assigns this segment elsewhere; only an issue
        // when the ray genuinely crosses this pixel (mode 0 did check t order)
        if (g.hasx && g.hasy) ++anomalies;
        continue;
      }
      acc = dadd(acc, y ? dmul(seg, __ldg(y + rowbase + j)) : seg);
    }
  }
  x[p] = acc;
  if (anomalies && anomaly) atomicAdd(anomaly, anomalies);
}

// Joseph backprojection, pixel-driven: per angle the (at most ~3) rays whose
// interpolation pair covers the pixel, ascending ray index (csc order); each
// weight is re-derived exactly as JosephWalker emits it.
template <bool kAccumulate>
__global__ void jbwd_kernel(GeomDev G, const double* __restrict__ y, double* __restrict__ x) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = G.n;
  if (p >= (long long)n * n) return;
  const int row = (int)(p / n), col = (int)(p % n);
  double acc = kAccumulate ? x[p] : 0.0;
  for (int a = 0; a < G.m; ++a) {
    JosephAngle ja;
    ja.init(n, G.d, G.ang[a].c, G.ang[a].s);
    const int kk = ja.ydom ? n - 1 - row : col;
    const int idx = ja.ydom ? col : n - 1 - row;
    // cont(j) ~ idx + 1/2 at the centre of the pixel's support
    const double ctr = (double)kk - ja.hc;
    const double oest = ((double)idx + 0.5 - ja.hc + ctr * ja.r) * ja.q;
    const int jc = (int)floor(oest + ja.dc + 0.5);
    const int j0 = max(jc - 3, 0), j1 = min(jc + 3, G.d - 1);
    const long long rowbase = (long long)a * G.d;
    for (int j = j0; j <= j1; ++j) {
      const double w = ja.weight(j, kk, idx);
      if (w > 0.0) acc = dadd(acc, y ? dmul(w, __ldg(y + rowbase + j)) : w);
    }
  }
  x[p] = acc;
}

}  // namespace parity

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
cudaError_t parity_forward(const GeomDev& G, const double* x, double* y, int* anomaly,
                           cudaStream_t st) {
  const long long rays = (long long)G.m * G.d;
  if (rays == 0) return cudaSuccess;
  const int tpb = 128;
  const unsigned grid = (unsigned)((rays + tpb - 1) / tpb);
  if (G.joseph)
    parity::fwd_kernel<parity::JosephWalker><<<grid, tpb, 0, st>>>(G, x, y, anomaly);
  else
    parity::fwd_kernel<parity::RayWalker><<<grid, tpb, 0, st>>>(G, x, y, anomaly);
  return cudaGetLastError();
}

cudaError_t parity_backward(const GeomDev& G, const double* y, double* x, bool accumulate,
                            int* anomaly, cudaStream_t st) {
  const long long pix = (long long)G.n * G.n;
  if (pix == 0) return cudaSuccess;
  const int tpb = 128;
  const unsigned grid = (unsigned)((pix + tpb - 1) / tpb);
  if (G.joseph) {
    if (accumulate)
      parity::jbwd_kernel<true><<<grid, tpb, 0, st>>>(G, y, x);
    else
      parity::jbwd_kernel<false><<<grid, tpb, 0, st>>>(G, y, x);
    return cudaGetLastError();
  }
  if (accumulate)
    parity::bwd_kernel<true><<<grid, tpb, 0, st>>>(G, y, x, anomaly);
  else
    parity::bwd_kernel<false><<<grid, tpb, 0, st>>>(G, y, x, anomaly);
  return cudaGetLastError();
}

cudaError_t parity_row_sums(const GeomDev& G, double* out, cudaStream_t st) {
  const long long rays = (long long)G.m * G.d;
  if (rays == 0) return cudaSuccess;
  const int tpb = 64;
  const unsigned grid = (unsigned)((rays + tpb - 1) / tpb);
  if (G.joseph)
    parity::rowsum_kernel<parity::JosephWalker><<<grid, tpb, 0, st>>>(G, out);
  else
    parity::rowsum_kernel<parity::RayWalker><<<grid, tpb, 0, st>>>(G, out);
  return cudaGetLastError();
}

cudaError_t parity_csr(const GeomDev& G, int pass, long long* counts, const long long* indptr,
                       long long* cols, double* vals, int* anomaly, cudaStream_t st) {
  const long long rays = (long long)G.m * G.d;
  if (rays == 0) return cudaSuccess;
  const int tpb = 128;
  const unsigned grid = (unsigned)((rays + tpb - 1) / tpb);
  if (G.joseph)
    parity::csr_kernel<parity::JosephWalker><<<grid, tpb, 0, st>>>(G, pass, counts, indptr, cols,
                                                                   vals, anomaly);
  else
    parity::csr_kernel<parity::RayWalker><<<grid, tpb, 0, st>>>(G, pass, counts, indptr, cols,
                                                                vals, anomaly);
  return cudaGetLastError();
}

}  // namespace wmg
