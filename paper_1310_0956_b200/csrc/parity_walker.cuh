// parity_walker.cuh -- exact float64 ray walker shared by the parity kernels.
// See projector_parity.cu for the parity contract and reference citations.
#pragma once
#include "common.cuh"

namespace wmg {
namespace parity {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Per-ray constants, evaluated exactly as the reference does.
struct RayGeom {
  int n;
  double half, ox, oy, dx, dy;
  bool hasx, hasy;

  __device__ __forceinline__ void init(int n_, int d, double c, double s, int j) {
    n = n_;
    half = (double)n_ * 0.5;                              // n / 2.0
    const double off = dsub((double)j, (double)(d - 1) * 0.5);  // arange - (d-1)/2.0
    ox = dmul(off, c);
    oy = dmul(off, s);
    dx = -s;
    dy = c;
    hasx = fabs(dx) > 1e-12;
    hasy = fabs(dy) > 1e-12;
  }
  __device__ __forceinline__ double line(int k) const { return dsub((double)k, half); }
  __device__ __forceinline__ double tx(int k) const { return ddiv(dsub(line(k), ox), dx); }
  __device__ __forceinline__ double ty(int k) const { return ddiv(dsub(line(k), oy), dy); }

  // The reference's per-segment evaluation (geometry.py:110-119).
  __device__ __forceinline__ bool segment(double tq, double tq1, int& ix, int& iy,
                                          double& seg) const {
    seg = dsub(tq1, tq);
    if (!(isfinite(seg) && seg > 1e-12)) return false;
    const double tm = dmul(0.5, dadd(tq1, tq));
    const double xm = dadd(ox, dmul(tm, dx));
    const double ym = dadd(oy, dmul(tm, dy));
    const double fx = floor(dadd(xm, half));
    const double fy = floor(dadd(ym, half));
    if (!(fx >= 0.0 && fx < (double)n && fy >= 0.0 && fy < (double)n)) return false;
    ix = (int)fx;
    iy = (int)fy;
    return true;
  }
};

// Generator over one ray's CSR row in ascending flat index.
struct RayWalker {
  RayGeom g;
  int mode;       // 0: slab walk (rows), 2: horizontal ray (single row)
  int state;      // 0 setup slab, 1 crossings, 2 closing segment, 3 done
  int iy;         // geometric slab (row from the bottom), walks n-1 .. 0
  int k, kend;
  double t_lo, t_hi, upper, ty_cache;
  long long last_flat;
  int anomalies;

  __device__ __forceinline__ void init(int n, int d, double c, double s, int j) {
    g.init(n, d, c, s, j);
    anomalies = 0;
    last_flat = -1;
    if (g.hasy) {
      mode = 0;
      state = 0;
      iy = n - 1;
      ty_cache = g.ty(n);
    } else if (g.hasx) {
      mode = 2;
      state = 1;
      k = 0;
      ty_cache = g.tx(0);   // cache tx(k)
    } else {
      state = 3;
    }
  }

  __device__ __forceinline__ bool produce(int ix, int iy_mid, int iy_expect, double seg,
                                          long long& flat, double& w) {
    flat = (long long)(g.n - 1 - iy_mid) * g.n + ix;
    if (iy_mid != iy_expect || flat <= last_flat) ++anomalies;
    last_flat = flat;
    w = seg;
    return true;
  }

  __device__ bool next(long long& flat, double& w) {
    int ix, iym;
    double seg;
    if (mode == 2) {
      // horizontal: tx decreasing in k; columns ascending = k ascending,
      // segment (tx[k+1], tx[k]); the row is fixed by ym = oy.
      while (state == 1) {
        if (k >= g.n) { state = 3; return false; }
        const double a = ty_cache;         // tx(k)
        const double b = g.tx(k + 1);
        ty_cache = b;
        ++k;
        if (g.segment(b, a, ix, iym, seg)) {
          const int expect = (int)floor(dadd(g.oy, g.half));
          return produce(ix, iym, expect, seg, flat, w);
        }
      }
      return false;
    }
    for (;;) {
      if (state == 3) return false;
      if (state == 0) {
        if (iy < 0) { state = 3; return false; }
        const double tA = g.ty(iy);
        const double tB = ty_cache;
        ty_cache = tA;
        t_lo = fmin(tA, tB);
        t_hi = fmax(tA, tB);
        upper = t_hi;
        if (g.hasx) {
          // x is decreasing in t (dx = -s < 0): x(t_hi) <= x(t_lo)
          const double xa = dadd(dadd(g.ox, dmul(t_hi, g.dx)), g.half);
          const double xb = dadd(dadd(g.ox, dmul(t_lo, g.dx)), g.half);
          if (xb < -2.0 || xa > (double)g.n + 2.0) { --iy; continue; }
          double fa = floor(xa) - 1.0, fb = ceil(xb) + 1.0;
          fa = fmax(fa, 0.0);
          fb = fmin(fb, (double)g.n);
          k = (int)fa;
          kend = (int)fb;
        } else {
          const double xa = dadd(g.ox, g.half);
          if (xa < -2.0 || xa > (double)g.n + 2.0) { --iy; continue; }
          k = 1;
          kend = 0;   // no x crossings
        }
        state = 1;
      }
      if (state == 1) {
        while (k <= kend) {
          const double txk = g.tx(k);
          ++k;
          if (t_lo < txk && txk < t_hi) {
            const double tq1 = upper;
            upper = txk;
            if (g.segment(txk, tq1, ix, iym, seg)) return produce(ix, iym, iy, seg, flat, w);
          }
        }
        state = 2;
      }
      if (state == 2) {
        state = 0;
        const int expect = iy;
        --iy;
        if (g.segment(t_lo, upper, ix, iym, seg)) return produce(ix, iym, expect, seg, flat, w);
      }
    }
  }
};

}  // namespace parity
}  // namespace wmg
