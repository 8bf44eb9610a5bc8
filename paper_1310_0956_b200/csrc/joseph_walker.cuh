// joseph_walker.cuh -- exact float64 generator over one ray's row of the
// reference's Joseph (interpolating) system matrix, in ascending flat pixel
// index (the CSR order), so the parity forward / CSR / row-sum kernels can be
// instantiated on it exactly as on the line-intersection RayWalker.
//
// Reference: /root/reference/pkg/src/wmgtomo/geometry.py:131-175.  Per angle,
// the dominant axis is y when |c| >= |s| (slabs = pixel rows, interpolation
// along x), else x.  For ray j (offset o_j) and slab k (pixel-centre coordinate
// ctr_k = k - (n-1)/2 along the dominant axis):
//     cont = (o_j / q - ctr_k * (p / q)) + (n - 1) / 2       (q, p) = (c, s) or (s, c)
//     i0 = floor(cont),  w1 = cont - i0
//     entries (i0, 1 - w1) and (i0 + 1, w1), each kept if the index is inside
//     the grid and the weight is > 0, value = weight * (1 / |q|);
// flat index = (n-1-k) * n + idx (y-dominant) or (n-1-idx) * n + k (x-dominant).
// Every operation is one IEEE op in the reference's order (numpy evaluates the
// same expression element-wise), hence bit-identical weights.
//
// CSR order.  y-dominant: rows ascend as k descends, columns i0 < i0 + 1 -- a
// plain walk.  x-dominant: row r = n-1-idx collects the slabs k whose i0 is idx
// (weight 1 - w1) or idx - 1 (weight w1); i0 is monotone in k (every operation
// above is monotone), so both sets are contiguous k ranges found by binary
// search, visited rows ascending and k ascending inside a row.
#pragma once
#include "parity_walker.cuh"

namespace wmg {
namespace parity {

struct JosephWalker {
  int n;
  bool ydom;
  double t1, r, scale, hc;
  // y-dominant walk
  int kc, e;
  bool have;
  double w1c;
  int i0c;
  // x-dominant walk
  bool dec;
  int v, vstop, phase, k, kend;
  bool typeA;
  int anomalies;   // interface parity with RayWalker (always 0)

  __device__ __forceinline__ double cont(int kk) const {
    const double ctr = dsub((double)kk, hc);
    return dadd(dsub(t1, dmul(ctr, r)), hc);
  }
  __device__ __forceinline__ int i0_of(int kk, double& w1) const {
    const double ct = cont(kk);
    const double f = floor(ct);
    w1 = dsub(ct, f);
    return (int)f;
  }
  __device__ __forceinline__ int i0_only(int kk) const {
    double w1;
    return i0_of(kk, w1);
  }
  // first k in [0, n] with pred(i0(k)); pred monotone false -> true
  __device__ int first_le(int u) const {      // i0 non-increasing: i0(k) <= u
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (i0_only(mid) <= u) hi = mid; else lo = mid + 1;
    }
    return lo;
  }
  __device__ int first_ge(int u) const {      // i0 non-decreasing: i0(k) >= u
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (i0_only(mid) >= u) hi = mid; else lo = mid + 1;
    }
    return lo;
  }
  // k range of slabs with i0 == u
  __device__ __forceinline__ void range_of(int u, int& a, int& b) const {
    if (dec) { a = first_le(u); b = first_le(u - 1); }
    else { a = first_ge(u); b = first_ge(u + 1); }
  }
  __device__ __forceinline__ void setup_phase() {
    // dec: [K_v (A), K_{v-1} (B)];  inc: [K_{v-1} (B), K_v (A)]
    const bool first = (phase == 0);
    typeA = dec ? first : !first;
    range_of(typeA ? v : v - 1, k, kend);
  }

  __device__ __forceinline__ void init(int n_, int d, double c, double s, int j) {
    n = n_;
    anomalies = 0;
    hc = (double)(n_ - 1) * 0.5;
    const double off = dsub((double)j, (double)(d - 1) * 0.5);
    ydom = fabs(c) >= fabs(s);
    const double q = ydom ? c : s, p = ydom ? s : c;
    t1 = ddiv(off, q);
    r = ddiv(p, q);
    scale = ddiv(1.0, fabs(q));
    if (ydom) {
      kc = n_ - 1;
      e = 0;
      have = false;
      return;
    }
    const int ia = i0_only(0), ib = i0_only(n_ - 1);
    dec = ib < ia;
    const int vmax = max(ia, ib) + 1, vmin = min(ia, ib);
    v = min(vmax, n_ - 1);
    vstop = max(vmin, 0);
    phase = 0;
    if (v >= vstop) setup_phase();
    else { k = 0; kend = 0; }
  }

  __device__ bool next(long long& flat, double& val) {
    if (ydom) {
      while (kc >= 0) {
        if (!have) {
          i0c = i0_of(kc, w1c);
          have = true;
          e = 0;
        }
        const int idx = i0c + e;
        const double w = e ? w1c : dsub(1.0, w1c);
        const int slab = kc;
        if (++e == 2) { have = false; --kc; }
        if (idx >= 0 && idx < n && w > 0.0) {
          flat = (long long)(n - 1 - slab) * n + idx;
          val = dmul(w, scale);
          return true;
        }
      }
      return false;
    }
    while (v >= vstop) {
      while (k < kend) {
        const int kk = k++;
        double w1;
        i0_of(kk, w1);
        const double w = typeA ? dsub(1.0, w1) : w1;
        if (w > 0.0) {
          flat = (long long)(n - 1 - v) * n + kk;
          val = dmul(w, scale);
          return true;
        }
      }
      if (phase == 0) {
        phase = 1;
      } else {
        phase = 0;
        --v;
        if (v < vstop) break;
      }
      setup_phase();
    }
    return false;
  }
};

// Joseph weight of ray j at pixel (slab kk, interpolation index idx) for one
// angle, as stored in the reference CSR (0 when the ray does not touch it).
struct JosephAngle {
  bool ydom;
  double r, scale, q, hc, dc;
  __device__ __forceinline__ void init(int n, int d, double c, double s) {
    ydom = fabs(c) >= fabs(s);
    q = ydom ? c : s;
    const double p = ydom ? s : c;
    r = ddiv(p, q);
    scale = ddiv(1.0, fabs(q));
    hc = (double)(n - 1) * 0.5;
    dc = (double)(d - 1) * 0.5;
  }
  __device__ __forceinline__ double weight(int j, int kk, int idx) const {
    const double off = dsub((double)j, dc);
    const double ctr = dsub((double)kk, hc);
    const double ct = dadd(dsub(ddiv(off, q), dmul(ctr, r)), hc);
    const double f = floor(ct);
    const int i0 = (int)f;
    const double w1 = dsub(ct, f);
    double w;
    if (i0 == idx) w = dsub(1.0, w1);
    else if (i0 == idx - 1) w = w1;
    else return 0.0;
    return w > 0.0 ? dmul(w, scale) : 0.0;
  }
};

}  // namespace parity
}  // namespace wmg
