// capi.cu -- extern "C" boundary (include/wmgb200.h).  Argument validation and
// error mapping live here; the kernels live in projector_*.cu, vecops.cu and
// multilevel.cu.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <new>
#include <algorithm>
#include <vector>

#include "../../include/wmgb200.h"
#include "common.cuh"

namespace wmg {
cudaError_t parity_forward(const GeomDev&, const double*, double*, int*, cudaStream_t);
cudaError_t parity_backward(const GeomDev&, const double*, double*, bool, int*, cudaStream_t);
cudaError_t parity_row_sums(const GeomDev&, double*, cudaStream_t);
cudaError_t parity_csr(const GeomDev&, int, long long*, const long long*, long long*, double*,
                       int*, cudaStream_t);
cudaError_t fast_forward(const GeomDev&, int, int, int, const void*, void*, void*, cudaStream_t,
                         const GeomDev*);
cudaError_t fast_backward(const GeomDev&, int, int, int, const void*, void*, bool, cudaStream_t,
                          const GeomDev*);
cudaError_t fast_forward_batch(const GeomDev&, int, int, int, const void*, void*, size_t, void*,
                               int, cudaStream_t, const GeomDev*);
int fast_backward_bands(const GeomDev&, int, const GeomDev*);
cudaError_t fast_backward_band(const GeomDev&, int, int, int, const void*, void*, int, int,
                               cudaStream_t, const GeomDev*);
cudaError_t fast_backward_batch(const GeomDev&, int, int, int, const void*, void*, bool, int,
                                cudaStream_t, const GeomDev*);
size_t fast_forward_workspace_bytes(int, int, int);
cudaError_t det_reduce(long long, int, const int*, const double* const*, const double* const*,
                       const double* const*, double*, double*, cudaStream_t);
long long det_scratch_len(long long, int);
cudaError_t maxabs(long long, const double*, const double*, double*, cudaStream_t);
cudaError_t ew_axpy(long long, double*, const double*, double, int, const double*, cudaStream_t);
cudaError_t ew_lincomb(long long, double*, double, const double*, double, const double*, double,
                       const double*, cudaStream_t);
cudaError_t ew_bicg_p(long long, double*, const double*, double, double, const double*,
                      cudaStream_t);
cudaError_t ew_bicg_x(long long, double*, double, const double*, double, const double*,
                      cudaStream_t);
cudaError_t ew_scale(long long, double*, double, const double*, const double*, cudaStream_t);
cudaError_t ew_recip(long long, double*, const double*, cudaStream_t);
cudaError_t ew_smooth_update(long long, double*, double, const double*, const double*,
                            const double*, cudaStream_t);
cudaError_t ew_sirt_update(long long, double*, const double*, const double*, double,
                           cudaStream_t);
cudaError_t ew_add_scaled(long long, double*, const double*, double, int, const double*,
                          cudaStream_t);
cudaError_t ew_cgs_update(long long, int, double*, const double*, long long, const double*,
                          cudaStream_t);
cudaError_t ew_combo(long long, int, double*, const double*, long long, const double*, int,
                     cudaStream_t);
cudaError_t ew_cast(long long, int, void*, const void*, cudaStream_t);
cudaError_t haar_restrict(int, const double*, int, double*, cudaStream_t);
cudaError_t haar_prolong_path(int, int, int, const int*, const double*, double*, cudaStream_t);
cudaError_t haar_restrict_path(int, int, int, const int*, const double*, double*, cudaStream_t);
cudaError_t ew_axpy_dev(long long, double*, const double*, const double*, int, const double*,
                        cudaStream_t);
cudaError_t ew_lincomb_dev(long long, double*, double, const double*, const double*,
                           const double*, cudaStream_t);
cudaError_t cgls_scalars(double*, double, int, cudaStream_t);
cudaError_t cgls_update(long long, long long, double*, const double*, double*, const double*,
                        const double*, const double*, double, double*, cudaStream_t);
cudaError_t cgls_direction(long long, double*, const double*, const double*, int, double*,
                           cudaStream_t);
cudaError_t batched_gemv(int, int, const double*, long long, const double*, long long, double*,
                         long long, cudaStream_t);
cudaError_t haar_prolong(int, const double*, int, double*, int, cudaStream_t);
cudaError_t leaf_factor(const GeomDev&, int, const int*, long long, long long, double*,
                        cudaStream_t);
cudaError_t leaf_gram(const GeomDev&, int, const int*, double*, int*, cudaStream_t);
size_t spd_inverse_workspace(int, int);
cudaError_t spd_inverse(int, int, double*, long long, int*, double*, cudaStream_t);
size_t cholesky_dinv_elems(int);
cudaError_t cholesky_factor(int, int, double*, long long, double*, int*, cudaStream_t);
cudaError_t cholesky_solve(int, int, const double*, long long, const double*, double*, long long,
                           int, cudaStream_t);
size_t packed_sym_elems(int);
size_t packed_symv_scratch(int, int);
cudaError_t sym_pack(int, int, const double*, long long, double*, long long, cudaStream_t);
cudaError_t packed_symv(int, int, const double*, long long, const double*, long long, double*,
                        long long, double*, cudaStream_t);
bool tma_window_fits(const AngleParams*, int, int, int);
cudaError_t h2d_staged(void*, const void*, size_t, void*, int, cudaStream_t);
bool fast_forward_path_supported(const GeomDev&, int, const GeomDev*);
cudaError_t fast_forward_path(const GeomDev&, int, int, const int*, const double*, void*, double*,
                              cudaStream_t, const GeomDev*);
cudaError_t haar_restrict_batch(int, int, const double*, int, double*, cudaStream_t);
cudaError_t haar_prolong_batch(int, int, int, const int*, const double*, double*, int,
                               cudaStream_t);
cudaError_t ew_smooth_update_batch(long long, int, double*, const double*, const double* const*,
                                   const double*, const double*, cudaStream_t);
}  // namespace wmg

struct wmg_geometry {
  wmg::GeomDev dev;
  wmg::AngleParams* d_ang;
  // symmetric angle sets: the two axis-aligned angles as their own geometry
  wmg::GeomDev axis;
  wmg::AngleParams* d_axis;
  int* d_mir;      // mirror / primary / half / axis-row tables (symmetric sets)
  int sym_capable;
};

static thread_local char g_err[512] = "";

static int fail(int code, const char* fmt, const char* detail = "") {
  snprintf(g_err, sizeof(g_err), fmt, detail);
  return code;
}

static int cuda_rc(cudaError_t e) {
  if (e == cudaSuccess) return WMG_OK;
  return fail(WMG_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
}

#define STREAM(s) (reinterpret_cast<cudaStream_t>(s))

extern "C" {

int wmg_version(void) { return 1; }
const char* wmg_last_error(void) { return g_err; }

int wmg_geometry_create(int n, int n_detectors, int n_angles, const double* cos_h,
                        const double* sin_h, wmg_geometry** out) {
  if (!out) return fail(WMG_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1 || n_detectors < 1 || n_angles < 1)
    return fail(WMG_EINVAL, "geometry dimensions must be positive");
  if (n > 16384) return fail(WMG_EINVAL, "n > 16384 is not supported");
  if (!cos_h || !sin_h) return fail(WMG_EINVAL, "cos/sin tables are NULL");
  std::vector<wmg::AngleParams> P((size_t)n_angles);
  const double half = 0.5 * n;
  for (int a = 0; a < n_angles; ++a) {
    const double c = cos_h[a], s = sin_h[a];
    if (!std::isfinite(c) || !std::isfinite(s) || s < 0.0)
      return fail(WMG_EINVAL, "angles must lie in [0, pi) (sin >= 0)");
    wmg::AngleParams& q = P[(size_t)a];
    memset(&q, 0, sizeof(q));
    q.c = c;
    q.s = s;
    const double ac = std::fabs(c), as = std::fabs(s);
    const double inf = std::numeric_limits<double>::infinity();
    if (ac >= as) {   // y-major: slabs are rows (top -> bottom), minor = column
      const double t = s / c;
      q.major = 0;
      q.u0 = half * (1.0 - t);
      q.du = 1.0 / c;
      q.slope = t;
      q.mirror = t < 0.0;
      q.L = 1.0 / ac;
      q.Ls = as == 0.0 ? inf : 1.0 / as;
    } else {          // x-major: slabs are columns (left -> right), minor = row
      const double ct = c / s;
      q.major = 1;
      q.u0 = half * (1.0 - ct);
      q.du = -1.0 / s;
      q.slope = ct;
      q.mirror = ct <= 0.0;   // theta = pi/2: ties go to the upper row
      q.L = 1.0 / as;
      q.Ls = ac == 0.0 ? inf : 1.0 / ac;
    }
    if (q.mirror) {
      q.u0 = (double)n - q.u0;
      q.du = -q.du;
      q.slope = -q.slope;
    }
    q.axis = (c == 0.0 || s == 0.0) ? 1 : 0;
    q.hw = 0.5 * (ac + as);
    q.inv_cs = q.axis ? 0.0 : 1.0 / (ac * as);
    q.Lf = (float)q.L;
    q.Lsf = (float)q.Ls;
    q.hwf = (float)q.hw;
    q.inv_csf = (float)q.inv_cs;
    q.Cfix = llrint(c * 4294967296.0);   // 2^32: v2 backprojector fixed point
    q.Sfix = llrint(s * 4294967296.0);
    q.a0 = (float)(2.0 - q.hw);
    const double icb = q.axis ? 1152921504606846976.0 : q.inv_cs;   // 2^60
    q.icb = (float)icb;
    q.hwic = (float)(q.hw * icb);
    q.w1c = (float)((2.0 * q.hw - 3.0) * icb);
  }
  // Mirror symmetry: every non-axis angle theta has its mirror pi - theta in
  // the set (to 1e-12); the axis angles (0, pi/2; any subset of them) run
  // through the plain kernels as their own sub-geometry.  Any angle subset
  // closed under the mirror qualifies (e.g. the per-rank shards of
  // sharding.shard_angles), n % 64 == 0 for the quadrant tiling.
  std::vector<int> mir((size_t)n_angles, -1), prim, halfv, axis_idx;
  bool sym = (n % 64 == 0);
  {
    std::vector<int> lo, hi;   // 0 < theta < pi/2 ascending; pi/2 < theta < pi ascending
    for (int a = 0; a < n_angles; ++a) {
      const double c = cos_h[a], s = sin_h[a];
      if (c == 0.0 || s == 0.0) axis_idx.push_back(a);
      else if (c > 0.0) lo.push_back(a);
      else hi.push_back(a);
    }
    auto by_angle = [&](int x, int y) { return cos_h[x] > cos_h[y]; };   // cos decreasing
    std::sort(lo.begin(), lo.end(), by_angle);
    std::sort(hi.begin(), hi.end(), by_angle);
    if (lo.size() != hi.size() || lo.empty()) sym = false;
    for (size_t i = 0; sym && i < lo.size(); ++i) {
      const int a = lo[i], b = hi[hi.size() - 1 - i];
      if (std::fabs(cos_h[b] + cos_h[a]) > 1e-12 || std::fabs(sin_h[b] - sin_h[a]) > 1e-12)
        sym = false;
      mir[(size_t)a] = b;
      mir[(size_t)b] = a;
    }
    if (sym) {
      for (int a = 0; a < n_angles; ++a)
        if (mir[(size_t)a] >= 0) prim.push_back(a);
      halfv = lo;
      // The symmetric forward puts 4 consecutive entries of this list into one
      // warp (8 rays x 4 angles), which pays off when the 4 angles are adjacent
      // (their rays read the same words slab after slab).  Runs of adjacent
      // angles (gap <= 1.5 x the smallest gap of the set) are cut into groups of
      // 4; what is left of each run goes to the end of the list.  An equiangular
      // set is one run (order unchanged); a per-rank shard dealt in chunks of 4
      // adjacent angles (sharding.shard_angles "quad") keeps every chunk in one warp.
      if (halfv.size() > 4) {
        std::vector<double> th(halfv.size());
        for (size_t i = 0; i < halfv.size(); ++i)
          th[i] = std::atan2(sin_h[halfv[i]], cos_h[halfv[i]]);
        double gmin = 1e300;
        for (size_t i = 1; i < th.size(); ++i) gmin = std::min(gmin, th[i] - th[i - 1]);
        std::vector<int> grouped, rest;
        for (size_t i = 0; i < halfv.size();) {
          size_t j = i + 1;
          while (j < halfv.size() && th[j] - th[j - 1] <= 1.5 * gmin) ++j;
          const size_t full = (j - i) / 4 * 4;
          grouped.insert(grouped.end(), halfv.begin() + i, halfv.begin() + i + full);
          rest.insert(rest.end(), halfv.begin() + i + full, halfv.begin() + j);
          i = j;
        }
        grouped.insert(grouped.end(), rest.begin(), rest.end());
        halfv.swap(grouped);
      }
    }
  }
  // Transposition symmetry (theta -> pi/2 - theta, to 1e-12): every primary with
  // |cos| > sin has its partners pi/2 -+ theta in the set, and each primary with
  // |cos| < sin is the partner of exactly one mirror pair; pi/4 and 3pi/4 (their
  // own transposes) stay four-image primaries.  Then the backprojector shares one
  // weight evaluation among eight (pixel, angle) pairs.
  std::vector<int> q8, l4;
  bool tsym = sym;
  if (tsym) {
    std::vector<int> byc(prim);
    std::sort(byc.begin(), byc.end(), [&](int x, int y) { return cos_h[x] < cos_h[y]; });
    std::vector<int> cover((size_t)n_angles, 0);
    for (int a : prim) {
      const double c = cos_h[a], s = sin_h[a];
      if (std::fabs(std::fabs(c) - s) <= 1e-12) { l4.push_back(a); continue; }
      if (std::fabs(c) < s) continue;   // a partner of some |cos| > sin primary
      auto it = std::lower_bound(byc.begin(), byc.end(), s - 1e-12,
                                 [&](int x, double v) { return cos_h[x] < v; });
      int ta = -1;
      for (; it != byc.end() && cos_h[*it] <= s + 1e-12; ++it)
        if (std::fabs(sin_h[*it] - std::fabs(c)) <= 1e-12) { ta = *it; break; }
      if (ta < 0 || mir[(size_t)ta] < 0) { tsym = false; break; }
      const int tb = mir[(size_t)ta];
      ++cover[(size_t)ta];
      ++cover[(size_t)tb];
      if (c > 0.0) q8.insert(q8.end(), {a, ta, tb, 0});
      else q8.insert(q8.end(), {a, tb, ta, 1});
    }
    for (size_t i = 0; tsym && i < prim.size(); ++i) {
      const int a = prim[i];
      const double c = std::fabs(cos_h[a]), s = sin_h[a];
      if (c < s && std::fabs(c - s) > 1e-12 && cover[(size_t)a] != 2) tsym = false;
    }
    if (!tsym) { q8.clear(); l4.clear(); }
  }
  // the TMA-staged forward (opt-in experiment) assumes the full equiangular layout
  bool std_layout = sym && n_angles % 2 == 0 && axis_idx.size() == 2 && axis_idx[0] == 0 &&
                    axis_idx[1] == n_angles / 2;
  for (int a = 1; std_layout && a < n_angles; ++a)
    if (a != n_angles / 2 && mir[(size_t)a] != n_angles - a) std_layout = false;
  wmg_geometry* g = new (std::nothrow) wmg_geometry;
  if (!g) return fail(WMG_EINVAL, "out of host memory");
  g->d_ang = nullptr;
  g->d_axis = nullptr;
  g->d_mir = nullptr;
  const int n_axis = (int)axis_idx.size();
  cudaError_t e = cudaMalloc(&g->d_ang, sizeof(wmg::AngleParams) * (size_t)n_angles);
  if (e == cudaSuccess)
    e = cudaMemcpy(g->d_ang, P.data(), sizeof(wmg::AngleParams) * (size_t)n_angles,
                   cudaMemcpyHostToDevice);
  // Per 4-angle group of the symmetric forward (warps of 8 rays x 4 angles walk
  // the union of their lanes' slab ranges): 1 when every lane's minor
  // coordinate stays within kPadMargin - 4 pixels of the image over that
  // union, so the zero margins absorb it and k needs no clamp.  u is linear in
  // the detector offset and the slab, so the spread between two lanes is
  // largest at a corner (j in {0, d/2}, slab in {0, n}); same major axis only.
  std::vector<int> gsafe;
  if (sym) {
    const int ng = ((int)halfv.size() + 3) / 4;
    const double jh = (double)((n_detectors + 1) / 2), dcen = (n_detectors - 1) * 0.5;
    for (int gi = 0; gi < ng; ++gi) {
      bool safe = true;
      double dmax = 0.0;
      const int g0 = gi * 4, g1 = std::min((int)halfv.size(), g0 + 4);
      for (int x = g0; x < g1 && safe; ++x) {
        const wmg::AngleParams& A = P[(size_t)halfv[(size_t)x]];
        dmax = std::max(dmax, 8.0 * std::fabs(A.du));        // rays of one lane group
        for (int y = g0; y < g1; ++y) {
          const wmg::AngleParams& Bq = P[(size_t)halfv[(size_t)y]];
          if (A.major != Bq.major) { safe = false; break; }
          for (double jj : {0.0, jh})
            for (double rr : {0.0, (double)n}) {
              const double ua = A.u0 + (jj - dcen) * A.du + rr * A.slope;
              const double ub = Bq.u0 + (jj - dcen) * Bq.du + rr * Bq.slope;
              dmax = std::max(dmax, std::fabs(ua - ub) + 8.0 * std::fabs(A.du));
            }
        }
      }
      gsafe.push_back(safe && dmax + 4.0 < (double)wmg::kPadMargin ? 1 : 0);
    }
  }
  if (e == cudaSuccess && sym) {
    // one int table: mir (m) | prim (n_prim) | half (n_half) | axis rowmap (n_axis)
    //                | group-safe flags (ceil(n_half / 4))
    std::vector<int> tab(mir);
    tab.insert(tab.end(), prim.begin(), prim.end());
    tab.insert(tab.end(), halfv.begin(), halfv.end());
    tab.insert(tab.end(), axis_idx.begin(), axis_idx.end());
    tab.insert(tab.end(), gsafe.begin(), gsafe.end());
    tab.insert(tab.end(), q8.begin(), q8.end());   // | q8 (4 n_q8) | l4 (n_l4)
    tab.insert(tab.end(), l4.begin(), l4.end());
    e = cudaMalloc(&g->d_mir, sizeof(int) * tab.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(g->d_mir, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && n_axis > 0) {
      std::vector<wmg::AngleParams> ax;
      for (int a : axis_idx) ax.push_back(P[(size_t)a]);
      e = cudaMalloc(&g->d_axis, sizeof(wmg::AngleParams) * ax.size());
      if (e == cudaSuccess)
        e = cudaMemcpy(g->d_axis, ax.data(), sizeof(wmg::AngleParams) * ax.size(),
                       cudaMemcpyHostToDevice);
    }
  }
  if (e != cudaSuccess) {
    if (g->d_ang) cudaFree(g->d_ang);
    if (g->d_axis) cudaFree(g->d_axis);
    if (g->d_mir) cudaFree(g->d_mir);
    delete g;
    return cuda_rc(e);
  }
  g->dev.n = n;
  g->dev.d = n_detectors;
  g->dev.m = n_angles;
  g->dev.ang = g->d_ang;
  g->dev.rowmap = nullptr;
  g->dev.sym = sym ? 1 : 0;
  g->dev.tma_ok =
      (std_layout && wmg::tma_window_fits(P.data(), n, n_detectors, n_angles)) ? 1 : 0;
  g->dev.joseph = 0;
  g->dev.mir = sym ? g->d_mir : nullptr;
  g->dev.prim = sym ? g->d_mir + n_angles : nullptr;
  g->dev.half = sym ? g->d_mir + n_angles + prim.size() : nullptr;
  g->dev.n_prim = (int)prim.size();
  g->dev.n_half = (int)halfv.size();
  g->dev.gsafe = sym ? g->d_mir + n_angles + prim.size() + halfv.size() + axis_idx.size()
                     : nullptr;
  {
    const size_t off_q8 = (size_t)n_angles + prim.size() + halfv.size() + axis_idx.size() +
                          gsafe.size();
    g->dev.tsym = (sym && tsym) ? 1 : 0;
    g->dev.q8 = g->dev.tsym ? g->d_mir + off_q8 : nullptr;
    g->dev.l4 = g->dev.tsym ? g->d_mir + off_q8 + q8.size() : nullptr;
    g->dev.n_q8 = g->dev.tsym ? (int)(q8.size() / 4) : 0;
    g->dev.n_l4 = g->dev.tsym ? (int)l4.size() : 0;
  }
  g->sym_capable = sym ? 1 : 0;
  g->axis = g->dev;
  g->axis.m = n_axis;
  g->axis.ang = g->d_axis;
  g->axis.rowmap = sym ? g->d_mir + n_angles + prim.size() + halfv.size() : nullptr;
  g->axis.sym = 0;
  g->axis.tsym = 0;
  g->axis.tma_ok = 0;
  g->axis.joseph = 0;
  *out = g;
  return WMG_OK;
}

int wmg_geometry_destroy(wmg_geometry* g) {
  if (!g) return WMG_OK;
  cudaError_t e = cudaFree(g->d_ang);
  if (g->d_axis) cudaFree(g->d_axis);
  if (g->d_mir) cudaFree(g->d_mir);
  delete g;
  return cuda_rc(e);
}

int wmg_geometry_symmetry(wmg_geometry* g, int set, int* enabled) {
  if (!g) return fail(WMG_EINVAL, "geometry is NULL");
  // 0 off, 1 auto, 2 forced, 4 forced + TMA forward; testing variants of the
  // forced mode: +8 row-layout backprojector, +16 one-angle forward blocks,
  // +256 the 8x4-block float4-window backprojector, +512 / +1024 run layout with
  // R = 4 / R = 8 rows per thread at any size, +8192 / +16384 the eight-image
  // backprojector forced at any size / disabled, +32768 (with +16384) the run
  // layout without the small-grid angle-split cluster, +65536 the symmetric
  // forward without the small-grid row-segment split
  if (set == 0 || set == 1 || set == 2 || set == 4 || set == 10 || set == 18 || set == 26 || set == 34 || set == 66 || set == 130 ||
      set == 258 || set == 514 || set == 1026 || set == 8194 ||
      set == 16386 || set == 49154 || set == 65538)
    g->dev.sym = (set && g->sym_capable) ? set : 0;
  if (enabled) *enabled = g->dev.sym;
  return WMG_OK;
}

int wmg_geometry_transposition(const wmg_geometry* g, int* closed) {
  if (!g || !closed) return fail(WMG_EINVAL, "NULL argument");
  *closed = g->dev.tsym;
  return WMG_OK;
}

int wmg_geometry_kernel(wmg_geometry* g, int set, int* kernel) {
  if (!g) return fail(WMG_EINVAL, "geometry is NULL");
  if (set == WMG_KERNEL_LINE || set == WMG_KERNEL_JOSEPH) {
    g->dev.joseph = (set == WMG_KERNEL_JOSEPH);
    g->axis.joseph = g->dev.joseph;
  } else if (set >= 0) {
    return fail(WMG_EINVAL, "unknown ray kernel");
  }
  if (kernel) *kernel = g->dev.joseph ? WMG_KERNEL_JOSEPH : WMG_KERNEL_LINE;
  return WMG_OK;
}

int wmg_geometry_shape(const wmg_geometry* g, long long* n_rows, long long* n_cols) {
  if (!g) return fail(WMG_EINVAL, "geometry is NULL");
  if (n_rows) *n_rows = (long long)g->dev.m * g->dev.d;
  if (n_cols) *n_cols = (long long)g->dev.n * g->dev.n;
  return WMG_OK;
}

int wmg_forward_workspace(const wmg_geometry* g, int precision, int dtype_in, size_t* bytes) {
  if (!g || !bytes) return fail(WMG_EINVAL, "NULL argument");
  *bytes = wmg::fast_forward_workspace_bytes(g->dev.n, precision, dtype_in);
  return WMG_OK;
}

static int check_types(int mode, int precision, int tin, int tout) {
  if (mode == WMG_MODE_PARITY) {
    if (tin != WMG_F64 || tout != WMG_F64)
      return fail(WMG_EINVAL, "parity mode is float64 only");
    return WMG_OK;
  }
  if (mode != WMG_MODE_FAST) return fail(WMG_EINVAL, "unknown projector mode");
  if ((tin != WMG_F32 && tin != WMG_F64) || (tout != WMG_F32 && tout != WMG_F64))
    return fail(WMG_EINVAL, "unknown dtype");
  if (precision != WMG_F32 && precision != WMG_F64) return fail(WMG_EINVAL, "unknown precision");
  if (precision == WMG_F64 && tin != tout)
    return fail(WMG_EINVAL, "fast float64 arithmetic needs equal in/out dtypes");
  return WMG_OK;
}

int wmg_forward(const wmg_geometry* g, int mode, int precision, int dtype_in, int dtype_out,
                const void* x, void* y, void* workspace, int* anomaly, void* stream) {
  if (!g || !x || !y) return fail(WMG_EINVAL, "NULL argument");
  int rc = check_types(mode, precision, dtype_in, dtype_out);
  if (rc) return rc;
  if (mode == WMG_MODE_PARITY)
    return cuda_rc(wmg::parity_forward(g->dev, (const double*)x, (double*)y, anomaly,
                                       STREAM(stream)));
  if (g->dev.joseph) return fail(WMG_EINVAL, "the Joseph kernel has parity (float64) mode only");
  if (!workspace) return fail(WMG_EINVAL, "fast forward needs a workspace");
  return cuda_rc(wmg::fast_forward(g->dev, precision, dtype_in, dtype_out, x, workspace, y,
                                   STREAM(stream), g->dev.sym ? &g->axis : nullptr));
}

int wmg_backward(const wmg_geometry* g, int mode, int precision, int dtype_in, int dtype_out,
                 const void* y, void* x, int accumulate, int* anomaly, void* stream) {
  if (!g || !x) return fail(WMG_EINVAL, "NULL argument");
  int rc = check_types(mode, precision, dtype_in, dtype_out);
  if (rc) return rc;
  if (mode == WMG_MODE_PARITY)
    return cuda_rc(wmg::parity_backward(g->dev, (const double*)y, (double*)x, accumulate != 0,
                                        anomaly, STREAM(stream)));
  if (!y) return fail(WMG_EINVAL, "y is NULL");
  if (g->dev.joseph) return fail(WMG_EINVAL, "the Joseph kernel has parity (float64) mode only");
  return cuda_rc(wmg::fast_backward(g->dev, precision, dtype_in, dtype_out, y, x,
                                    accumulate != 0, STREAM(stream),
                                    g->dev.sym ? &g->axis : nullptr));
}

int wmg_backward_bands(const wmg_geometry* g, int precision, int* bands) {
  if (!g || !bands) return fail(WMG_EINVAL, "NULL argument");
  *bands = g->dev.sym ? wmg::fast_backward_bands(g->dev, precision, &g->axis) : 0;
  return WMG_OK;
}

int wmg_backward_band(const wmg_geometry* g, int precision, int dtype_in, int dtype_out,
                      const void* y, void* x, int band0, int band1, void* stream) {
  if (!g || !x || !y) return fail(WMG_EINVAL, "NULL argument");
  int rc = check_types(WMG_MODE_FAST, precision, dtype_in, dtype_out);
  if (rc) return rc;
  const int nb = g->dev.sym ? wmg::fast_backward_bands(g->dev, precision, &g->axis) : 0;
  if (nb == 0) return fail(WMG_EINVAL, "no banded backprojection for this geometry / mode");
  if (band0 < 0 || band1 > nb || band0 > band1) return fail(WMG_EINVAL, "band range");
  return cuda_rc(wmg::fast_backward_band(g->dev, precision, dtype_in, dtype_out, y, x, band0,
                                         band1, STREAM(stream), &g->axis));
}

int wmg_forward_path_supported(const wmg_geometry* g, int precision, int* ok) {
  if (!g || !ok) return fail(WMG_EINVAL, "NULL argument");
  *ok = (!g->dev.joseph &&
         wmg::fast_forward_path_supported(g->dev, precision, g->dev.sym ? &g->axis : nullptr))
            ? 1
            : 0;
  return WMG_OK;
}

int wmg_forward_path(const wmg_geometry* g, const double* coarse, int depth, int batch,
                     const int* bands, double* y, void* workspace, void* stream) {
  if (batch == 0 && g) return WMG_OK;
  if (!g || !coarse || !bands || !y || !workspace) return fail(WMG_EINVAL, "NULL argument");
  if (batch < 0) return fail(WMG_EINVAL, "negative batch");
  if (depth < 1 || depth > 7) return fail(WMG_EINVAL, "depth must be in [1, 7]");
  for (long long i = 0; i < (long long)batch * depth; ++i)
    if (bands[i] < 0 || bands[i] > 3) return fail(WMG_EINVAL, "bad band");
  if ((g->dev.n >> depth) << depth != g->dev.n)
    return fail(WMG_EINVAL, "2^depth must divide n");
  int ok = 0;
  wmg_forward_path_supported(g, 1, &ok);
  if (!ok) return fail(WMG_EINVAL, "no fused path forward for this geometry");
  return cuda_rc(wmg::fast_forward_path(g->dev, depth, batch, bands, coarse, workspace, y,
                                        STREAM(stream), g->dev.sym ? &g->axis : nullptr));
}

int wmg_forward_batch(const wmg_geometry* g, int mode, int precision, int dtype_in,
                      int dtype_out, const void* x, void* y, int batch, void* workspace,
                      void* stream) {
  if (batch == 0 && g) return WMG_OK;
  if (!g || !x || !y) return fail(WMG_EINVAL, "NULL argument");
  if (batch < 0) return fail(WMG_EINVAL, "negative batch");
  int rc = check_types(mode, precision, dtype_in, dtype_out);
  if (rc) return rc;
  const long long N = (long long)g->dev.n * g->dev.n, M = (long long)g->dev.m * g->dev.d;
  if (mode == WMG_MODE_PARITY) {
    for (int b = 0; b < batch; ++b) {
      cudaError_t e = wmg::parity_forward(g->dev, (const double*)x + b * N, (double*)y + b * M,
                                          nullptr, STREAM(stream));
      if (e != cudaSuccess) return cuda_rc(e);
    }
    return WMG_OK;
  }
  if (g->dev.joseph) return fail(WMG_EINVAL, "the Joseph kernel has parity (float64) mode only");
  if (!workspace) return fail(WMG_EINVAL, "fast forward needs a workspace");
  const size_t ws_item = wmg::fast_forward_workspace_bytes(g->dev.n, precision, dtype_in);
  return cuda_rc(wmg::fast_forward_batch(g->dev, precision, dtype_in, dtype_out, x, workspace,
                                         ws_item, y, batch, STREAM(stream),
                                         g->dev.sym ? &g->axis : nullptr));
}

int wmg_backward_batch(const wmg_geometry* g, int mode, int precision, int dtype_in,
                       int dtype_out, const void* y, void* x, int batch, int accumulate,
                       void* stream) {
  if (batch == 0 && g) return WMG_OK;
  if (!g || !x || !y) return fail(WMG_EINVAL, "NULL argument");
  if (batch < 0) return fail(WMG_EINVAL, "negative batch");
  int rc = check_types(mode, precision, dtype_in, dtype_out);
  if (rc) return rc;
  const long long N = (long long)g->dev.n * g->dev.n, M = (long long)g->dev.m * g->dev.d;
  if (mode == WMG_MODE_PARITY) {
    for (int b = 0; b < batch; ++b) {
      cudaError_t e = wmg::parity_backward(g->dev, (const double*)y + b * M, (double*)x + b * N,
                                           accumulate != 0, nullptr, STREAM(stream));
      if (e != cudaSuccess) return cuda_rc(e);
    }
    return WMG_OK;
  }
  if (g->dev.joseph) return fail(WMG_EINVAL, "the Joseph kernel has parity (float64) mode only");
  return cuda_rc(wmg::fast_backward_batch(g->dev, precision, dtype_in, dtype_out, y, x,
                                          accumulate != 0, batch, STREAM(stream),
                                          g->dev.sym ? &g->axis : nullptr));
}

int wmg_row_sums(const wmg_geometry* g, double* out, void* stream) {
  if (!g || !out) return fail(WMG_EINVAL, "NULL argument");
  return cuda_rc(wmg::parity_row_sums(g->dev, out, STREAM(stream)));
}

int wmg_col_sums(const wmg_geometry* g, double* out, void* stream) {
  if (!g || !out) return fail(WMG_EINVAL, "NULL argument");
  return cuda_rc(wmg::parity_backward(g->dev, nullptr, out, false, nullptr, STREAM(stream)));
}

int wmg_csr_counts(const wmg_geometry* g, long long* counts, int* anomaly, void* stream) {
  if (!g || !counts) return fail(WMG_EINVAL, "NULL argument");
  return cuda_rc(wmg::parity_csr(g->dev, 0, counts, nullptr, nullptr, nullptr, anomaly,
                                 STREAM(stream)));
}

int wmg_csr_fill(const wmg_geometry* g, const long long* indptr, long long* cols, double* vals,
                 void* stream) {
  if (!g || !indptr || !cols || !vals) return fail(WMG_EINVAL, "NULL argument");
  return cuda_rc(wmg::parity_csr(g->dev, 1, nullptr, indptr, cols, vals, nullptr,
                                 STREAM(stream)));
}

long long wmg_det_scratch_len(long long n, int K) { return wmg::det_scratch_len(n, K); }

static int det_args_check(long long n, int K, const int* ops, const double* const* a,
                          const double* const* b, const double* const* c, const double* scratch) {
  if (K < 1 || K > 8 || !ops || !a || !scratch)
    return fail(WMG_EINVAL, "bad det_reduce arguments");
  if (n > 1024LL * 1024LL * 1024LL) return fail(WMG_EINVAL, "vector longer than 2^30");
  for (int k = 0; k < K; ++k) {
    if (ops[k] < 0 || ops[k] > 4) return fail(WMG_EINVAL, "unknown reduction op");
    if (!a[k]) return fail(WMG_EINVAL, "NULL operand");
    if ((ops[k] == WMG_RED_DOT || ops[k] == WMG_RED_SQDIFF || ops[k] == WMG_RED_DOTDIFF) &&
        (!b || !b[k]))
      return fail(WMG_EINVAL, "NULL operand");
    if (ops[k] == WMG_RED_DOTDIFF && (!c || !c[k])) return fail(WMG_EINVAL, "NULL operand");
  }
  return WMG_OK;
}

int wmg_det_reduce(long long n, int K, const int* ops, const double* const* a,
                   const double* const* b, const double* const* c, double* scratch, double* out,
                   void* stream) {
  if (!out) return fail(WMG_EINVAL, "bad det_reduce arguments");
  const int rc = det_args_check(n, K, ops, a, b, c, scratch);
  if (rc) return rc;
  return cuda_rc(wmg::det_reduce(n, K, ops, a, b, c, scratch, out, STREAM(stream)));
}

int wmg_det_partials(long long n, int K, const int* ops, const double* const* a,
                     const double* const* b, const double* const* c, double* partials,
                     void* stream) {
  const int rc = det_args_check(n, K, ops, a, b, c, partials);
  if (rc) return rc;
  if (n < 1) return fail(WMG_EINVAL, "det_partials: empty vector");
  return cuda_rc(wmg::det_reduce(n, K, ops, a, b, c, partials, nullptr, STREAM(stream)));
}

int wmg_maxabs(long long n, const double* a, const double* b, double* out, void* stream) {
  if (!a || !out) return fail(WMG_EINVAL, "NULL argument");
  return cuda_rc(wmg::maxabs(n, a, b, out, STREAM(stream)));
}

#define REQ(p) \
  if (!(p)) return fail(WMG_EINVAL, "NULL argument")

int wmg_axpy(long long n, double* out, const double* y, double alpha, int sgn, const double* x,
             void* stream) {
  REQ(out && y && x);
  return cuda_rc(wmg::ew_axpy(n, out, y, alpha, sgn, x, STREAM(stream)));
}
int wmg_lincomb(long long n, double* out, double a, const double* x, double b, const double* y,
                double c, const double* z, void* stream) {
  REQ(out && x && y);
  return cuda_rc(wmg::ew_lincomb(n, out, a, x, b, y, c, z, STREAM(stream)));
}
int wmg_bicg_p(long long n, double* p, const double* r, double beta, double omega,
               const double* v, void* stream) {
  REQ(p && r && v);
  return cuda_rc(wmg::ew_bicg_p(n, p, r, beta, omega, v, STREAM(stream)));
}
int wmg_bicg_x(long long n, double* x, double alpha, const double* ph, double omega,
               const double* sh, void* stream) {
  REQ(x && ph && sh);
  return cuda_rc(wmg::ew_bicg_x(n, x, alpha, ph, omega, sh, STREAM(stream)));
}
int wmg_scale(long long n, double* out, double a, const double* x, const double* y,
              void* stream) {
  REQ(out && x);
  return cuda_rc(wmg::ew_scale(n, out, a, x, y, STREAM(stream)));
}
int wmg_recip(long long n, double* out, const double* s, void* stream) {
  REQ(out && s);
  return cuda_rc(wmg::ew_recip(n, out, s, STREAM(stream)));
}
int wmg_smooth_update(long long n, double* z, double omega, const double* c, const double* r,
                      const double* az, void* stream) {
  REQ(z && c && r);
  return cuda_rc(wmg::ew_smooth_update(n, z, omega, c, r, az, STREAM(stream)));
}
int wmg_sirt_update(long long n, double* x, const double* c, const double* g, double lam,
                    void* stream) {
  REQ(x && c && g);
  return cuda_rc(wmg::ew_sirt_update(n, x, c, g, lam, STREAM(stream)));
}
int wmg_add_scaled(long long n, double* out, const double* g, double lam, int sgn,
                   const double* v, void* stream) {
  REQ(out && g && v);
  return cuda_rc(wmg::ew_add_scaled(n, out, g, lam, sgn, v, STREAM(stream)));
}
int wmg_cgs_update(long long n, int k, double* w, const double* V, long long ldv,
                   const double* h, void* stream) {
  REQ(w && V && h);
  if (k < 0) return fail(WMG_EINVAL, "k < 0");
  return cuda_rc(wmg::ew_cgs_update(n, k, w, V, ldv, h, STREAM(stream)));
}
int wmg_combo(long long n, int k, double* out, const double* V, long long ldv, const double* cf,
              int accumulate, void* stream) {
  REQ(out && V && cf);
  if (k < 0) return fail(WMG_EINVAL, "k < 0");
  return cuda_rc(wmg::ew_combo(n, k, out, V, ldv, cf, accumulate, STREAM(stream)));
}
int wmg_axpy_dev(long long n, double* out, const double* y, const double* coef, int sgn,
                 const double* x, void* stream) {
  REQ(out && y && coef && x);
  return cuda_rc(wmg::ew_axpy_dev(n, out, y, coef, sgn, x, STREAM(stream)));
}
int wmg_lincomb_dev(long long n, double* out, double a, const double* x, const double* coef,
                    const double* y, void* stream) {
  REQ(out && x && coef && y);
  return cuda_rc(wmg::ew_lincomb_dev(n, out, a, x, coef, y, STREAM(stream)));
}
int wmg_cgls_scalars(double* S, double lam, int op, void* stream) {
  REQ(S);
  if (op < 0 || op > 2) return fail(WMG_EINVAL, "bad scalar op");
  return cuda_rc(wmg::cgls_scalars(S, lam, op, STREAM(stream)));
}
int wmg_cgls_update(long long n_img, long long n_sino, double* x, const double* p, double* r,
                    const double* q, const double* partials, const double* partials_pp,
                    double lam, double* S, void* stream) {
  REQ(x && p && r && q && partials && S);
  if (n_img <= 0 || n_sino <= 0 || n_sino > (1LL << 20) || n_img > (1LL << 20))
    return fail(WMG_EINVAL, "cgls_update: lengths must be in [1, 2^20]");
  if (lam != 0.0 && !partials_pp)
    return fail(WMG_EINVAL, "cgls_update: lam != 0 needs the <p,p> chunk sums");
  return cuda_rc(wmg::cgls_update(n_img, n_sino, x, p, r, q, partials, partials_pp, lam, S,
                                  STREAM(stream)));
}
int wmg_cgls_direction(long long n, double* p, const double* z, const double* partials, int mode,
                       double* S, void* stream) {
  REQ(p && z && partials && S);
  if (n <= 0 || n > (1LL << 20)) return fail(WMG_EINVAL, "cgls_direction: n not in [1, 2^20]");
  if (mode != 1 && mode != 2) return fail(WMG_EINVAL, "cgls_direction: mode must be 1 or 2");
  return cuda_rc(wmg::cgls_direction(n, p, z, partials, mode, S, STREAM(stream)));
}
int wmg_h2d_staged(void* dst, const void* src, size_t bytes, void* pinned, int threads,
                   void* stream) {
  if (bytes == 0) return WMG_OK;
  if (!dst || !src || !pinned) return fail(WMG_EINVAL, "h2d_staged: NULL buffer");
  if (threads < 1 || threads > 64) return fail(WMG_EINVAL, "h2d_staged: threads not in [1, 64]");
  return cuda_rc(wmg::h2d_staged(dst, src, bytes, pinned, threads, STREAM(stream)));
}

int wmg_cast(long long n, int to_f32, void* out, const void* in, void* stream) {
  REQ(out && in);
  return cuda_rc(wmg::ew_cast(n, to_f32, out, in, STREAM(stream)));
}

int wmg_batched_gemv(int batch, int p, const double* A, long long strideA, const double* x,
                     long long stridex, double* y, long long stridey, void* stream) {
  REQ(A && x && y);
  if (batch < 0 || p < 0) return fail(WMG_EINVAL, "negative size");
  if (p > 24576) return fail(WMG_EINVAL, "p > 24576 (shared-memory staging of x)");
  return cuda_rc(wmg::batched_gemv(batch, p, A, strideA, x, stridex, y, stridey, STREAM(stream)));
}

int wmg_haar_restrict(int side, const double* fine, int band_mask, double* out, void* stream) {
  REQ(fine && out);
  if (side < 2 || side % 2) return fail(WMG_EINVAL, "grid side must be even and >= 2");
  if (band_mask < 1 || band_mask > 15) return fail(WMG_EINVAL, "bad band mask");
  return cuda_rc(wmg::haar_restrict(side, fine, band_mask, out, STREAM(stream)));
}

int wmg_haar_prolong(int side, const double* coarse, int band, double* fine, int accumulate,
                     void* stream) {
  REQ(coarse && fine);
  if (side < 2 || side % 2) return fail(WMG_EINVAL, "grid side must be even and >= 2");
  if (band < 0 || band > 3) return fail(WMG_EINVAL, "bad band");
  return cuda_rc(wmg::haar_prolong(side, coarse, band, fine, accumulate, STREAM(stream)));
}

int wmg_haar_restrict_batch(int side, int batch, const double* fine, int band_mask, double* out,
                            void* stream) {
  if (batch == 0) return WMG_OK;
  REQ(fine && out);
  if (batch < 0) return fail(WMG_EINVAL, "negative batch");
  if (side < 2 || side % 2) return fail(WMG_EINVAL, "grid side must be even and >= 2");
  if (band_mask < 1 || band_mask > 15) return fail(WMG_EINVAL, "bad band mask");
  return cuda_rc(wmg::haar_restrict_batch(side, batch, fine, band_mask, out, STREAM(stream)));
}

int wmg_haar_prolong_batch(int side, int batch, int nbands, const int* bands,
                           const double* coarse, double* fine, int accumulate, void* stream) {
  if (batch == 0) return WMG_OK;
  REQ(bands && coarse && fine);
  if (batch < 0) return fail(WMG_EINVAL, "negative batch");
  if (side < 2 || side % 2) return fail(WMG_EINVAL, "grid side must be even and >= 2");
  if (nbands < 1 || nbands > 4) return fail(WMG_EINVAL, "nbands must be in [1, 4]");
  for (int i = 0; i < nbands; ++i)
    if (bands[i] < 0 || bands[i] > 3) return fail(WMG_EINVAL, "bad band");
  return cuda_rc(wmg::haar_prolong_batch(side, batch, nbands, bands, coarse, fine, accumulate,
                                         STREAM(stream)));
}

int wmg_smooth_update_batch(long long n, int batch, double* z, const double* omegas,
                            const double* const* c, const double* r, const double* az,
                            void* stream) {
  if (batch == 0) return WMG_OK;
  REQ(z && omegas && c && r);
  if (batch < 0) return fail(WMG_EINVAL, "negative batch");
  for (int i = 0; i < batch; ++i)
    if (!c[i]) return fail(WMG_EINVAL, "NULL smoother scaling");
  return cuda_rc(wmg::ew_smooth_update_batch(n, batch, z, omegas, c, r, az, STREAM(stream)));
}

static int check_path(int n, int depth, int batch, const int* bands) {
  if (!bands && batch > 0 && depth > 0) return fail(WMG_EINVAL, "bands is NULL");
  if (depth < 0 || depth > 7) return fail(WMG_EINVAL, "depth must be in [0, 7]");
  if (batch < 0) return fail(WMG_EINVAL, "negative batch");
  if (n < 1 || (n >> depth) << depth != n) return fail(WMG_EINVAL, "n is not divisible by 2^depth");
  for (long long i = 0; i < (long long)batch * depth; ++i)
    if (bands[i] < 0 || bands[i] > 3) return fail(WMG_EINVAL, "bad band");
  return WMG_OK;
}

int wmg_haar_prolong_path(int n, int depth, int batch, const int* bands, const double* coarse,
                          double* fine, void* stream) {
  REQ(coarse && fine);
  int rc = check_path(n, depth, batch, bands);
  if (rc) return rc;
  if (batch == 0) return WMG_OK;
  return cuda_rc(wmg::haar_prolong_path(n, depth, batch, bands, coarse, fine, STREAM(stream)));
}

int wmg_haar_restrict_path(int n, int depth, int batch, const int* bands, const double* fine,
                           double* coarse, void* stream) {
  REQ(coarse && fine);
  int rc = check_path(n, depth, batch, bands);
  if (rc) return rc;
  if (batch == 0) return WMG_OK;
  return cuda_rc(wmg::haar_restrict_path(n, depth, batch, bands, fine, coarse, STREAM(stream)));
}

int wmg_leaf_factor(const wmg_geometry* g, int depth, const int* bands, long long ray0,
                    long long nrays, double* P, void* stream) {
  REQ(g && bands && P);
  if (depth < 1 || depth > 12) return fail(WMG_EINVAL, "bad depth");
  if ((g->dev.n >> depth) << depth != g->dev.n)
    return fail(WMG_EINVAL, "n is not divisible by 2^depth");
  const long long rays = (long long)g->dev.m * g->dev.d;
  if (ray0 < 0 || nrays < 0 || ray0 + nrays > rays) return fail(WMG_EDIM, "ray range");
  for (int i = 0; i < depth; ++i)
    if (bands[i] < 0 || bands[i] > 3) return fail(WMG_EINVAL, "bad band");
  if (nrays == 0) return WMG_OK;
  return cuda_rc(wmg::leaf_factor(g->dev, depth, bands, ray0, nrays, P, STREAM(stream)));
}

int wmg_leaf_gram(const wmg_geometry* g, int depth, const int* bands, double* gram,
                  int* overflow, void* stream) {
  REQ(g && bands && gram && overflow);
  if (depth < 1 || depth > 12) return fail(WMG_EINVAL, "bad depth");
  if ((g->dev.n >> depth) << depth != g->dev.n)
    return fail(WMG_EINVAL, "n is not divisible by 2^depth");
  for (int i = 0; i < depth; ++i)
    if (bands[i] < 0 || bands[i] > 3) return fail(WMG_EINVAL, "bad band");
  if (g->dev.joseph) return fail(WMG_EINVAL, "the sparse leaf Gram implements line weights only");
  if (g->dev.m == 0 || g->dev.d == 0) return WMG_OK;
  return cuda_rc(wmg::leaf_gram(g->dev, depth, bands, gram, overflow, STREAM(stream)));
}

int wmg_spd_inverse_workspace(int batch, int p, size_t* bytes) {
  REQ(bytes);
  if (batch < 0 || p < 0) return fail(WMG_EINVAL, "negative size");
  *bytes = wmg::spd_inverse_workspace(batch, p);
  return WMG_OK;
}

int wmg_spd_inverse(int batch, int p, double* G, long long strideG, int* info, void* work,
                    void* stream) {
  REQ(G && info && work);
  if (batch < 0 || p < 0) return fail(WMG_EINVAL, "negative size");
  if (p % 128) return fail(WMG_EINVAL, "p must be a multiple of 128 (pad with identity)");
  if (batch > 1 && strideG < (long long)p * p) return fail(WMG_EDIM, "batch stride < p*p");
  if (batch > 65535) return fail(WMG_EINVAL, "batch > 65535");
  return cuda_rc(wmg::spd_inverse(batch, p, G, strideG, info, static_cast<double*>(work),
                                  STREAM(stream)));
}

int wmg_cholesky_dinv_elems(int p, long long* elems) {
  REQ(elems);
  if (p < 0) return fail(WMG_EINVAL, "negative size");
  if (p % 128) return fail(WMG_EINVAL, "p must be a multiple of 128 (pad with identity)");
  *elems = (long long)wmg::cholesky_dinv_elems(p);
  return WMG_OK;
}

int wmg_cholesky_factor(int batch, int p, double* G, long long strideG, double* dinv, int* info,
                        void* stream) {
  REQ(G && dinv && info);
  if (batch < 0 || p < 0) return fail(WMG_EINVAL, "negative size");
  if (p % 128) return fail(WMG_EINVAL, "p must be a multiple of 128 (pad with identity)");
  if (batch > 1 && strideG < (long long)p * p) return fail(WMG_EDIM, "batch stride < p*p");
  if (batch > 65535) return fail(WMG_EINVAL, "batch > 65535");
  return cuda_rc(wmg::cholesky_factor(batch, p, G, strideG, dinv, info, STREAM(stream)));
}

int wmg_cholesky_solve(int batch, int p, const double* L, long long strideL, const double* dinv,
                       double* B, long long strideB, int nrhs, void* stream) {
  REQ(L && dinv && B);
  if (batch < 0 || p < 0 || nrhs < 0) return fail(WMG_EINVAL, "negative size");
  if (p % 128) return fail(WMG_EINVAL, "p must be a multiple of 128 (pad with identity)");
  if (p > 12800) return fail(WMG_EINVAL, "p > 12800 (solve keeps two p-vectors in shared memory)");
  if (batch > 1 && (strideL < (long long)p * p || strideB < (long long)p * nrhs))
    return fail(WMG_EDIM, "batch stride too small");
  if (batch > 65535 || nrhs > 65535) return fail(WMG_EINVAL, "batch or nrhs > 65535");
  return cuda_rc(wmg::cholesky_solve(batch, p, L, strideL, dinv, B, strideB, nrhs,
                                     STREAM(stream)));
}

int wmg_packed_sym_sizes(int batch, int p, long long* elems_per_matrix, size_t* scratch_bytes) {
  if (batch < 0 || p < 0) return fail(WMG_EINVAL, "negative size");
  if (p % 128) return fail(WMG_EINVAL, "p must be a multiple of 128");
  if (elems_per_matrix) *elems_per_matrix = (long long)wmg::packed_sym_elems(p);
  if (scratch_bytes) *scratch_bytes = wmg::packed_symv_scratch(batch, p);
  return WMG_OK;
}

int wmg_sym_pack(int batch, int p, const double* A, long long strideA, double* packed,
                 long long strideP, void* stream) {
  REQ(A && packed);
  if (batch < 0 || p < 0) return fail(WMG_EINVAL, "negative size");
  if (p % 128) return fail(WMG_EINVAL, "p must be a multiple of 128");
  if (batch > 1 && (strideA < (long long)p * p || strideP < (long long)wmg::packed_sym_elems(p)))
    return fail(WMG_EDIM, "batch stride too small");
  if (batch > 65535) return fail(WMG_EINVAL, "batch > 65535");
  return cuda_rc(wmg::sym_pack(batch, p, A, strideA, packed, strideP, STREAM(stream)));
}

int wmg_packed_symv(int batch, int p, const double* packed, long long strideP, const double* x,
                    long long stridex, double* y, long long stridey, double* scratch,
                    void* stream) {
  REQ(packed && x && y && scratch);
  if (batch < 0 || p < 0) return fail(WMG_EINVAL, "negative size");
  if (p % 128) return fail(WMG_EINVAL, "p must be a multiple of 128");
  if (batch > 65535) return fail(WMG_EINVAL, "batch > 65535");
  return cuda_rc(wmg::packed_symv(batch, p, packed, strideP, x, stridex, y, stridey, scratch,
                                  STREAM(stream)));
}

}  // extern "C"
