// common.cuh -- shared types for the sm_100a projector / solver kernels.
//
// Conventions follow the reference geometry (/root/reference/pkg/src/wmgtomo/
// geometry.py:1-21): n x n unit pixels centred at the origin, image vectors
// row-major with row 0 at the top (largest y), sinograms angle-major m x d,
// ray point = o*(c, s) + t*(-s, c), detector offsets o_j = j - (d-1)/2.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace wmg {

// Per-angle parameters.  (c, s) are the reference's snapped trig values
// (geometry.py:77-85), computed on the host with numpy so the device never
// evaluates cos/sin itself.  The remaining fields drive the fast kernels'
// slab walk and are derived on the host in float64.
struct AngleParams {
  double c, s;        // snapped cos / sin
  // ---- fast slab-walk parameters -------------------------------------
  // The ray is walked slab by slab along its major axis (image rows when
  // |c| >= |s|, columns otherwise).  u is the minor-axis grid coordinate in
  // [0, n]; after the optional mirror u -> n - u the slope per slab is >= 0.
  double u0;          // u at slab 0 for detector offset o = 0 (after mirror)
  double du;          // du / do (per unit detector offset, after mirror)
  double slope;       // du per slab, >= 0
  double L;           // ray length per full slab = 1 / |major component|
  double Ls;          // ray length per unit u = 1 / |minor component| (inf if 0)
  // ---- pixel-driven (backprojection) trapezoid -------------------------
  double hw;          // (|c| + |s|) / 2 : half support in detector units
  double inv_cs;      // 1 / (|c| |s|) (unused when axis aligned)
  float Lf, Lsf, hwf, inv_csf;   // float copies for the fp32 kernels
  // ---- tiled fp32 backprojector (fixed-point detector coordinate) -------
  long long Cfix, Sfix;  // c * 2^32, s * 2^32: detector-index step per +1 column / +1 row
  float a0;              // 2 - hw
  float icb;             // 1/(|c||s|), or 2^60 for axis-aligned angles (finite: no inf-inf)
  float hwic;            // hw * icb
  float w1c;             // (2 hw - 3) * icb
  int major;          // 0: slabs are rows (y-major), 1: slabs are columns
  int mirror;         // 1 when the minor axis is mirrored
  int axis;           // 1 when s == 0 or c == 0 (exact axis-aligned angle)
  int pad_;
};

struct GeomDev {
  int n;              // pixels per side
  int d;              // detectors per angle
  int m;              // angles
  const AngleParams* ang;   // device table, length m
  const int* rowmap;  // optional: sinogram row of local angle a (nullptr = a)
  int sym;            // 1: angle set symmetric under theta -> pi - theta (fast kernels
                      //    may share weights across mirror images), n % 64 == 0
  int tma_ok;         // 1: the TMA-staged forward's window bound holds for every group
  int joseph;         // 1: Joseph interpolation weights (parity kernels only)
  // mirror pairs of a symmetric angle set (sym != 0): mir[a] = local index of
  // the angle pi - theta_a (-1 for the axis angles 0, pi/2); prim = every
  // non-axis angle (n_prim); half = the ones with 0 < theta < pi/2 (n_half)
  const int* mir;
  const int* prim;
  const int* half;
  const int* gsafe;   // per 4-angle group of half: 1 = forward needs no k clamp
  int n_prim, n_half;
  // transposition symmetry (theta -> pi/2 - theta, sym != 0 and tsym != 0): the
  // 8-image backprojector walks q8 (n_q8 entries of 4 ints: primary angle
  // alpha with |cos| > sin, rows u1, u2 of the transposed images and a flag:
  // 1 = their direct / reversed windows swap) and l4 (n_l4 self-transposed
  // primaries, pi/4 and 3pi/4, taken with four images)
  const int* q8;
  const int* l4;
  int n_q8, n_l4;
  int tsym;
};

// Fixed-point minor coordinate used by the fast kernels: 64-bit signed with
// 40 fractional bits (|u| < 2^22 is ample for n <= 8192).
constexpr int kFixFrac = 40;
constexpr double kFixScale = 1099511627776.0;  // 2^40
// zero margin (pixels) around the padded image copies read by the fast
// forward kernel: >= 31 * sqrt(2) + 2 so a warp can walk its union slab range
constexpr int kPadMargin = 64;

// linear index -> (I, J), I >= J, of the lower triangle in row order
__device__ __forceinline__ void tri_unrank(int lin, int& I, int& J) {
  int i = (int)((sqrtf(8.0f * (float)lin + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= lin) ++i;
  while (i * (i + 1) / 2 > lin) --i;
  I = i;
  J = lin - i * (i + 1) / 2;
}

// Haar band coefficient signs of the 2 x 2 block (2i,2k), (2i,2k+1), (2i+1,2k),
// (2i+1,2k+1) times h = fl(fl(1/sqrt 2)^2) (multilevel.py:36-53): band 0 LL,
// 1 LH (wavelet along rows), 2 HL (along columns), 3 HH
__device__ __forceinline__ void haar_band_signs(int band, double& s00, double& s01, double& s10,
                                                double& s11) {
  const double h = 0.4999999999999999;
  const bool wy = (band == 1 || band == 3);
  const bool wx = (band == 2 || band == 3);
  s00 = h;
  s01 = wx ? -h : h;
  s10 = wy ? -h : h;
  s11 = (wx != wy) ? -h : h;
}

// band paths of a batch of WMG nodes: depth and, per item, the bands of levels
// 0..depth-1 in 2-bit fields (level 0 = the finest), passed by value so the
// launches stay graph-capturable
constexpr int kPathBatch = 128;
struct BandPaths {
  int depth;
  unsigned short code[kPathBatch];
};

// fine pixel (r, c) of R_path^T coarse, coarsest level first: the same chain
// of sign * h products as the level-by-level prolongations (bit-identical)
__device__ __forceinline__ double haar_path_value(const BandPaths& bp, int item,
                                                  const double* __restrict__ coarse, int sc,
                                                  int r, int c) {
  const int k = bp.depth;
  const unsigned code = bp.code[item];
  double v = coarse[(long long)(r >> k) * sc + (c >> k)];
  for (int lv = k - 1; lv >= 0; --lv) {
    double s[4];
    haar_band_signs((code >> (2 * lv)) & 3, s[0], s[1], s[2], s[3]);
    v = __dmul_rn(s[(((r >> lv) & 1) << 1) | ((c >> lv) & 1)], v);
  }
  return v;
}

}  // namespace wmg
