// multilevel.cu -- WMG hierarchy setup kernel.
//
// The reference stores, per hierarchy node, the tall-and-skinny factor
// P = W R_path^T built by repeated sparse products (multilevel.py:123-148,
// sparse_kernels.py:30-39) and, at the coarsest level, the dense Gram
// P^T P + lambda I (multilevel.py:125-130).  Here P is never formed for the
// internal nodes (their node systems are applied matrix-free: prolong -> pair
// -> restrict).  For a leaf L the factor is generated directly from the exact
// ray walk: every entry (ray i, pixel f, w_if) is scattered with the leaf's
// Haar-packet coefficient H_L(f) into P_L[i, block(f)], where H_L(f) is the
// value the path prolongation R_path^T e_q takes at f (one +-0.4999999999999999
// factor per level, rounded in prolongation order, as haar_prolong computes).
// The Gram is then one float64 GEMM P_L^T P_L on the GPU.
#include "parity_walker.cuh"

namespace wmg {
namespace ml {

__device__ __forceinline__ double band_sign(int band, int ry, int cx) {
  const double h = 0.4999999999999999;
  const bool wy = (band == 1 || band == 3) && ry;
  const bool wx = (band == 2 || band == 3) && cx;
  return (wy != wx) ? -h : h;
}

// bands[t] is the band taken at depth t+1 (t = 0 is the root's child)
struct LeafPath {
  int depth;
  int bands[12];
};

// P (rays x p, row-major, zero-initialised by the caller) for ray range
// [ray0, ray0 + nrays)
__global__ void leaf_factor_kernel(GeomDev G, LeafPath path, long long ray0, long long nrays,
                                   double* __restrict__ P) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrays) return;
  const long long ray = ray0 + t;
  const int a = (int)(ray / G.d), j = (int)(ray % G.d);
  const int n = G.n;
  const int k = path.depth;
  const int side_c = n >> k;
  const long long pdim = (long long)side_c * side_c;
  parity::RayWalker wk;
  wk.init(n, G.d, G.ang[a].c, G.ang[a].s, j);
  long long flat;
  double w;
  double* row = P + t * pdim;
  while (wk.next(flat, w)) {
    const int r = (int)(flat / n), c = (int)(flat % n);
    // prolongation from the leaf up: coarsest factor first
    double h = 1.0;
    for (int lv = k - 1; lv >= 0; --lv) {
      const double sg = band_sign(path.bands[lv], (r >> lv) & 1, (c >> lv) & 1);
      h = parity::dmul(sg, h);
    }
    const long long q = (long long)(r >> k) * side_c + (c >> k);
    row[q] = parity::dadd(row[q], parity::dmul(w, h));
  }
}

}  // namespace ml

cudaError_t leaf_factor(const GeomDev& G, int depth, const int* bands, long long ray0,
                        long long nrays, double* P, cudaStream_t st) {
  if (depth < 1 || depth > 12 || nrays <= 0) return cudaErrorInvalidValue;
  ml::LeafPath path;
  path.depth = depth;
  for (int i = 0; i < 12; ++i) path.bands[i] = i < depth ? bands[i] : 0;
  const int tpb = 128;
  ml::leaf_factor_kernel<<<(unsigned)((nrays + tpb - 1) / tpb), tpb, 0, st>>>(G, path, ray0,
                                                                              nrays, P);
  return cudaGetLastError();
}

}  // namespace wmg
