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
#include "joseph_walker.cuh"

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
template <typename Walker>
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
  Walker wk;
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

// ---------------------------------------------------------------------------
// Sparse leaf Gram  G_L += P_L^T P_L  (lower triangle), without forming P_L.
//
// A row of P_L (one ray) has only ~n/B * (|c|+|s|) nonzeros, the coarse blocks
// the ray crosses, so the dense GEMM wastes a factor p / nnz_row (~50 at
// config 2).  One CTA takes a bundle of NB consecutive rays of one angle.  In
// slab coordinates (the fast walk: slabs along the major axis, minor
// coordinate u, slope >= 0) the bundle crosses, in each coarse slab-row R, at
// most kWc consecutive coarse minor indices [clo[R], clo[R] + kWc), so its
// rows of P_L live in a (NB x side_c*kWc) local matrix V in shared memory:
//   pass 1  per (ray, R): the minor extent -> clo[R] (shared atomicMin)
//   pass 2  per (ray, R): walk the B fine slabs of R, weights from the fp64
//           slab formula (<= 1e-12 of the exact weights, as the fast fp64
//           projector), times H_L(pixel); V and a ray-occupancy bitmask per
//           local block
//   pass 3  every local pair (i >= j) whose masks intersect: the dot over the
//           shared rays, one fp64 atomicAdd into the lower triangle of G_L.
// The Gram of one leaf (p^2 fp64; the lower half is written) stays resident in
// the 126 MB L2 at config 2 (p = 4096: 67 MB), so the atomics resolve in L2.
// ---------------------------------------------------------------------------
constexpr int kWc = 4;

__global__ void __launch_bounds__(256) leaf_gram_kernel(GeomDev G, LeafPath path, int NB,
                                                        unsigned long long* __restrict__ gram,
                                                        double scale,
                                                        int* __restrict__ overflow) {
  extern __shared__ double smem[];
  const int a = blockIdx.y;
  const int j0 = blockIdx.x * NB;
  const int n = G.n, k = path.depth, B = 1 << k, sc = n >> k;
  const int Q = sc * kWc;
  const long long p = (long long)sc * sc;
  const AngleParams& A = G.ang[a];
  double* V = smem;                                   // [Q][NB]
  unsigned* mask = (unsigned*)(V + (size_t)Q * NB);   // [Q]
  int* clo = (int*)(mask + Q);                        // [sc]
  int* chi = clo + sc;                                // [sc]
  const int tid = threadIdx.x;
  for (int i = tid; i < Q * NB; i += blockDim.x) V[i] = 0.0;
  for (int i = tid; i < Q; i += blockDim.x) mask[i] = 0u;
  for (int i = tid; i < sc; i += blockDim.x) { clo[i] = 0x7fffffff; chi[i] = -1; }
  __syncthreads();

  const double slope = A.slope;
  const int items = NB * sc;
  // pass 1: coarse minor extent of the bundle per coarse slab-row
  for (int it = tid; it < items; it += blockDim.x) {
    const int r = it % NB, R = it / NB, j = j0 + r;
    if (j >= G.d) continue;
    const double u0 = A.u0 + ((double)j - (double)(G.d - 1) * 0.5) * A.du;
    const int s0 = R * B;
    int kmin = (int)floor(fma((double)s0, slope, u0)) - 1;
    int kmax = (int)floor(fma((double)(s0 + B), slope, u0));
    kmin = max(kmin, 0);
    kmax = min(kmax, n - 1);
    if (kmin > kmax) continue;
    const int lo = A.mirror ? n - 1 - kmax : kmin;
    const int hi = A.mirror ? n - 1 - kmin : kmax;
    atomicMin(&clo[R], lo >> k);
    atomicMax(&chi[R], hi >> k);
  }
  __syncthreads();
  for (int R = tid; R < sc; R += blockDim.x)
    if (chi[R] >= 0 && chi[R] - clo[R] >= kWc) atomicOr(overflow, 1);
  // |H_L| (same rounding sequence as the prolongation: one factor per level)
  double mag = 1.0;
  for (int lv = k - 1; lv >= 0; --lv) mag = parity::dmul(0.4999999999999999, mag);
  const double L = A.L, Ls = A.Ls;
  // sign of H_L(row, col) = parity of the wavelet bits the path selects
  unsigned ymask = 0u, xmask = 0u;
  for (int lv = 0; lv < k; ++lv) {
    const int band = path.bands[lv];
    if (band == 1 || band == 3) ymask |= 1u << lv;
    if (band == 2 || band == 3) xmask |= 1u << lv;
  }
  // pass 2: local rows of P_L
  for (int it = tid; it < items; it += blockDim.x) {
    const int r = it % NB, R = it / NB, j = j0 + r;
    if (j >= G.d || chi[R] < 0) continue;
    const double u0 = A.u0 + ((double)j - (double)(G.d - 1) * 0.5) * A.du;
    const int base = clo[R];
    double acc[kWc];
#pragma unroll
    for (int l = 0; l < kWc; ++l) acc[l] = 0.0;
    for (int s = R * B; s < R * B + B; ++s) {
      const double uh = fma((double)(s + 1), slope, u0);
      const double fk = floor(uh);
      const int kh = (int)fk;
      double wh = (uh - fk) * Ls;
      wh = (wh < L) ? wh : L;            // NaN (ray on a grid line) -> L
      const double wl = L - wh;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int kp = kh - e;
        const double w = e ? wl : wh;
        if (kp < 0 || kp >= n || w == 0.0) continue;
        const int kk = A.mirror ? n - 1 - kp : kp;
        const int row = A.major ? kk : s, col = A.major ? s : kk;
        const bool neg = (__popc((unsigned)row & ymask) + __popc((unsigned)col & xmask)) & 1;
        const double v = w * (neg ? -mag : mag);
        const int l = (kk >> k) - base;
#pragma unroll
        for (int q = 0; q < kWc; ++q)
          if (q == l) acc[q] += v;
      }
    }
#pragma unroll
    for (int l = 0; l < kWc; ++l) {
      if (acc[l] != 0.0) {
        V[(size_t)(R * kWc + l) * NB + r] = acc[l];
        atomicOr(&mask[R * kWc + l], 1u << r);
      }
    }
  }
  __syncthreads();
  // pass 3: pairs of crossed local blocks that share a ray.  The crossed blocks
  // are compacted first (their order does not matter: the fixed-point atomics
  // are associative), so the pair loop skips the empty ones.
  int* act = chi + sc;                                // [Q]
  __shared__ int nact_s;
  if (tid == 0) nact_s = 0;
  __syncthreads();
  for (int i = tid; i < Q; i += blockDim.x)
    if (mask[i]) act[atomicAdd(&nact_s, 1)] = i;
  __syncthreads();
  const int nact = nact_s;
  const long long npairs = (long long)nact * (nact + 1) / 2;
  for (long long t = tid; t < npairs; t += blockDim.x) {
    int u, v;
    tri_unrank((int)t, u, v);
    const int i = act[u], jj = act[v];
    unsigned mm = mask[i] & mask[jj];
    if (!mm) continue;
    double sum = 0.0;
    while (mm) {
      const int r = __ffs(mm) - 1;
      mm &= mm - 1;
      sum = fma(V[(size_t)i * NB + r], V[(size_t)jj * NB + r], sum);
    }
    const int Ri = i / kWc, Rj = jj / kWc;
    const int ci = clo[Ri] + i % kWc, cj = clo[Rj] + jj % kWc;
    long long gi = A.major ? (long long)ci * sc + Ri : (long long)Ri * sc + ci;
    long long gj = A.major ? (long long)cj * sc + Rj : (long long)Rj * sc + cj;
    if (gi < gj) { const long long tmp = gi; gi = gj; gj = tmp; }
    // fixed-point accumulation: integer adds are associative, so the Gram is
    // bit-reproducible whatever order the bundles' atomics land in
    atomicAdd(&gram[gi * p + gj], (unsigned long long)llrint(sum * scale));
  }
}

// fixed point (int64 bits stored in the Gram buffer) -> float64, in place
__global__ void fixed_to_double_kernel(double* __restrict__ g, long long count, double inv) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) g[i] = (double)__double_as_longlong(g[i]) * inv;
}

}  // namespace ml

size_t leaf_gram_smem(int n, int depth, int nb) {
  const int sc = n >> depth;
  const int Q = sc * ml::kWc;
  return (size_t)Q * nb * sizeof(double) + (size_t)Q * sizeof(unsigned) + 2 * sc * sizeof(int) +
         (size_t)Q * sizeof(int);
}

cudaError_t leaf_gram(const GeomDev& G, int depth, const int* bands, double* gram, int* overflow,
                      cudaStream_t st) {
  if (depth < 1 || depth > 12) return cudaErrorInvalidValue;
  ml::LeafPath path;
  path.depth = depth;
  for (int i = 0; i < 12; ++i) path.bands[i] = i < depth ? bands[i] : 0;
  const int nb = min(16, 1 << depth);
  const size_t smem = leaf_gram_smem(G.n, depth, nb);
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(ml::leaf_gram_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((G.d + nb - 1) / nb, G.m);
  // Fixed-point scale: every |entry| <= m (sqrt2 B + 2) * 2 (a block's P entry
  // is at most sqrt2 in magnitude, at most sqrt2 B + 2 rays of an angle cross
  // a block), so 2^e with e = 61 - ceil(log2(bound)) leaves headroom for the
  // sum and a resolution ~1e-13 of the bound (cf. the 1e-16 relative rounding
  // of a float64 sum over ~1e3 terms).
  const double B = (double)(1 << depth);
  const double bound = 2.0 * (double)G.m * (1.4142135623730951 * B + 2.0);
  const int ex = 61 - (int)ceil(log2(bound));
  const double scale = ldexp(1.0, ex);
  ml::leaf_gram_kernel<<<grid, 256, smem, st>>>(G, path, nb, (unsigned long long*)gram, scale,
                                                overflow);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  const long long count = (long long)(G.n >> depth) * (G.n >> depth);
  const long long total = count * count;
  ml::fixed_to_double_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(gram, total,
                                                                            1.0 / scale);
  return cudaGetLastError();
}

cudaError_t leaf_factor(const GeomDev& G, int depth, const int* bands, long long ray0,
                        long long nrays, double* P, cudaStream_t st) {
  if (depth < 1 || depth > 12 || nrays <= 0) return cudaErrorInvalidValue;
  ml::LeafPath path;
  path.depth = depth;
  for (int i = 0; i < 12; ++i) path.bands[i] = i < depth ? bands[i] : 0;
  const int tpb = 128;
  const unsigned grid = (unsigned)((nrays + tpb - 1) / tpb);
  if (G.joseph)
    ml::leaf_factor_kernel<parity::JosephWalker><<<grid, tpb, 0, st>>>(G, path, ray0, nrays, P);
  else
    ml::leaf_factor_kernel<parity::RayWalker><<<grid, tpb, 0, st>>>(G, path, ray0, nrays, P);
  return cudaGetLastError();
}

}  // namespace wmg
