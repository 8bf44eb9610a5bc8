/*
 * wmgb200.h -- C ABI of the B200-native WMG tomography hot path.
 *
 * Library: paper_1310_0956_b200/lib/libwmgb200.so (sm_100a).  Every entry point
 * takes plain pointers and sizes; device buffers are CALLER-OWNED.  The only
 * internal allocations belong to a geometry handle: its per-angle and
 * mirror-pair tables (wmg_geometry_create, freed by wmg_geometry_destroy).  All
 * work is asynchronous on the caller's CUDA stream (cudaStream_t passed as
 * void*, NULL = legacy default stream).  Functions are reentrant; a geometry may
 * be shared across threads and streams, except that the setters
 * (wmg_geometry_symmetry / wmg_geometry_kernel) must not race launches.
 *
 * Return codes (mapped by the Python host layer the way the reference raises):
 *   WMG_OK        0
 *   WMG_EINVAL    1  invalid argument                -> ValueError
 *   WMG_EDIM      2  dimension mismatch              -> DimensionMismatchError
 *   WMG_ENOTSPD   3  not symmetric positive definite -> NotPositiveDefiniteError
 *   WMG_ECUDA     4  CUDA launch / runtime error     -> RuntimeError
 * wmg_last_error() returns a thread-local message for the last failure.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/wmgtomo):
 *   geometry.py:68-74   build_geometry / Geometry   -> wmg_geometry_create
 *   geometry.py:178-197 build_projector (CSR W)     -> (matrix-free) wmg_forward /
 *                                                      wmg_backward; exact CSR export
 *                                                      via wmg_csr_counts / wmg_csr_fill
 *   geometry.py:200-206 apply        (W x)          -> wmg_forward
 *   geometry.py:209-215 apply_transpose (W^T y)     -> wmg_backward
 *   solvers.py:79-86    sirt_scaling (row/col sums) -> wmg_row_sums / wmg_col_sums
 *   solvers.py:116-135  sirt_solve vector ops       -> wmg_sirt_update, wmg_det_reduce
 *   solvers.py:140-156  normal_operator (+lambda v) -> wmg_add_scaled
 *   solvers.py:195-241  bicgstab_solve vector ops   -> wmg_bicg_p, wmg_bicg_x, wmg_axpy,
 *                                                      wmg_det_reduce
 *   phantom.py:64-75    error_metrics               -> wmg_det_reduce(SQDIFF), wmg_maxabs
 *   multilevel.py:36-79 haar_* / build_intergrid_set-> wmg_haar_restrict / wmg_haar_prolong
 *   multilevel.py:123-130 leaf Gram assembly        -> wmg_leaf_gram (sparse) or
 *                                                      wmg_leaf_factor (+ DGEMM)
 *   sparse_kernels.py:53-65 potrf of the leaf Grams  -> wmg_spd_inverse (batched fp64 DMMA sweep)
 *   sparse_kernels.py:68-75 cho_solve in the V-cycle -> wmg_packed_symv (packed symmetric
 *                                                      inverse) / wmg_batched_gemv (dense)
 *   multilevel.py:109-113 node systems, siblings     -> wmg_forward_batch / wmg_backward_batch
 *   geometry.py:131-175 _joseph_entries             -> wmg_geometry_kernel (JOSEPH)
 *   (CGLS / PCG-NE, not in the reference)           -> wmg_cgls_scalars, wmg_axpy_dev,
 *                                                      wmg_lincomb_dev (device scalars)
 */
#ifndef WMGB200_H
#define WMGB200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WMG_OK 0
#define WMG_EINVAL 1
#define WMG_EDIM 2
#define WMG_ENOTSPD 3
#define WMG_ECUDA 4

/* projector modes */
#define WMG_MODE_PARITY 0 /* float64, bit-exact reference weights and sum order */
#define WMG_MODE_FAST 1   /* fixed-point geometry, any summation order */
/* ray kernels (geometry.py:178-185) */
#define WMG_KERNEL_LINE 0   /* exact intersection lengths (default) */
#define WMG_KERNEL_JOSEPH 1 /* two-pixel interpolation per slab; PARITY mode only */
/* dtypes / precisions */
#define WMG_F32 0
#define WMG_F64 1

/* deterministic reduction ops (wmg_det_reduce) */
#define WMG_RED_DOT 0     /* sum a_i * b_i            */
#define WMG_RED_SQDIFF 1  /* sum (a_i - b_i)^2        */
#define WMG_RED_SUM 2     /* sum a_i                  */
#define WMG_RED_DOTDIFF 3 /* sum a_i * (b_i - c_i)    */
#define WMG_RED_SQ 4      /* sum a_i^2                */

typedef struct wmg_geometry wmg_geometry;

int wmg_version(void);
const char *wmg_last_error(void);

/* Geometry: n x n unit pixels, n_detectors rays per angle (spacing 1), and
 * n_angles angles given by their SNAPPED cos/sin (host arrays, float64),
 * i.e. geometry.py:77-85 evaluated on the host.  Angles must lie in [0, pi). */
int wmg_geometry_create(int n, int n_detectors, int n_angles, const double *cos_h,
                        const double *sin_h, wmg_geometry **out);
int wmg_geometry_destroy(wmg_geometry *g);
int wmg_geometry_shape(const wmg_geometry *g, long long *n_rows, long long *n_cols);
/* Mirror-symmetry acceleration of the FAST kernels.  Available when the angle set
 * satisfies theta_{m-a} = pi - theta_a (to 1e-12) with exact axis angles at a = 0
 * and m/2 and n % 64 == 0 (e.g. build_geometry grids); then one weight evaluation
 * serves four (pixel, angle) pairs.  set = 0 disables it, 1 enables it where
 * profitable (large grids; the default when available), 2 forces it at every
 * size (testing), 4 forces it with the experimental TMA-staged forward, -1 only
 * queries; *enabled receives the state. */
int wmg_geometry_symmetry(wmg_geometry *g, int set, int *enabled);

/* *closed = 1 when the angle set is also closed under theta -> pi/2 - theta
 * (the eight-image backprojector applies), else 0 */
int wmg_geometry_transposition(const wmg_geometry *g, int *closed);
/* Ray kernel of the geometry's system matrix: set = WMG_KERNEL_LINE or
 * WMG_KERNEL_JOSEPH (build_projector(g, kernel=...), geometry.py:178-185), -1
 * only queries.  Joseph geometries support the PARITY projector pair, CSR
 * export, row/column sums and wmg_leaf_factor; the FAST kernels and
 * wmg_leaf_gram return WMG_EINVAL for them. */
int wmg_geometry_kernel(wmg_geometry *g, int set, int *kernel);

/* bytes of caller workspace wmg_forward (mode FAST) needs: zero-padded image
 * copies in both orientations for fp32 arithmetic, a transposed copy otherwise */
int wmg_forward_workspace(const wmg_geometry *g, int precision, int dtype_in, size_t *bytes);

/* y = W x (length m*d).  mode PARITY requires dtype_in = dtype_out = F64 and
 * ignores precision/workspace; anomaly (device int*, may be NULL) counts
 * segments whose midpoint pixel contradicts the walk (0 on all pinned sizes). */
int wmg_forward(const wmg_geometry *g, int mode, int precision, int dtype_in, int dtype_out,
                const void *x, void *y, void *workspace, int *anomaly, void *stream);

/* x = W^T y (accumulate = 1: x += W^T y).  PARITY: y == NULL means y = 1. */
int wmg_backward(const wmg_geometry *g, int mode, int precision, int dtype_in, int dtype_out,
                 const void *y, void *x, int accumulate, int *anomaly, void *stream);

/* Banded fast backprojection (fp32 arithmetic, eight-image kernels; for
 * angle-sharded solves that overlap the allreduce of W^T y with the rest of
 * the backprojection).  *bands = number of quadrant row-blocks qt = n / 64 when
 * the geometry takes the banded path in this precision, else 0.
 * wmg_backward_band writes bands [band0, band1): image rows [32 band0,
 * 32 band1) and [n - 32 band1, n - 32 band0) receive their complete W^T y
 * (bit-identical to wmg_backward); calls must cover 0..qt in increasing
 * order on one stream.  Same reference function as wmg_backward
 * (geometry.py:209-215). */
int wmg_backward_bands(const wmg_geometry *g, int precision, int *bands);
/* W R_path^T for a batch of WMG node vectors (the prolongation of the node
 * systems, multilevel.py:109-113, fused into the float64 fast forward): item b
 * = coarse + b (n >> depth)^2, bands[b depth + lv] = its band at level lv (lv 0
 * the finest; 0 LL, 1 LH, 2 HL, 3 HH), sinograms n_angles * n_detectors apart;
 * workspace = batch * wmg_forward_workspace(FLOAT64, FLOAT64) bytes.  Bit-
 * identical to wmg_haar_prolong_path + wmg_forward_batch (FAST, float64);
 * available when wmg_forward_path_supported (small grids) reports 1. */
int wmg_forward_path_supported(const wmg_geometry *g, int precision, int *ok);
int wmg_forward_path(const wmg_geometry *g, const double *coarse, int depth, int batch,
                     const int *bands, double *y, void *workspace, void *stream);
int wmg_backward_band(const wmg_geometry *g, int precision, int dtype_in, int dtype_out,
                      const void *y, void *x, int band0, int band1, void *stream);

/* Batched W x / W^T y over `batch` contiguous images (n*n apart) and sinograms
 * (n_angles*n_detectors apart), each item computed exactly as by wmg_forward /
 * wmg_backward (the WMG cycle applies sibling node systems together; on small
 * grids the float64 fast kernels take the batch in one launch).  workspace:
 * batch * wmg_forward_workspace bytes (FAST mode). */
int wmg_forward_batch(const wmg_geometry *g, int mode, int precision, int dtype_in,
                      int dtype_out, const void *x, void *y, int batch, void *workspace,
                      void *stream);
int wmg_backward_batch(const wmg_geometry *g, int mode, int precision, int dtype_in,
                       int dtype_out, const void *y, void *x, int batch, int accumulate,
                       void *stream);

/* exact reference row sums (np.add.reduceat) and column sums (ones @ W) */
int wmg_row_sums(const wmg_geometry *g, double *out, void *stream);
int wmg_col_sums(const wmg_geometry *g, double *out, void *stream);

/* exact CSR export (entry for entry equal to build_projector): counts per ray,
 * then fill at a caller-built indptr (int64) */
int wmg_csr_counts(const wmg_geometry *g, long long *counts, int *anomaly, void *stream);
int wmg_csr_fill(const wmg_geometry *g, const long long *indptr, long long *cols, double *vals,
                 void *stream);

/* deterministic float64 reductions: out[k] = DET_SUM over i of op_k(a_k, b_k, c_k)
 * for k < K <= 8.  scratch: wmg_det_scratch_len(n, K) doubles of device memory. */
long long wmg_det_scratch_len(long long n, int K);
int wmg_det_reduce(long long n, int K, const int *ops, const double *const *a,
                   const double *const *b, const double *const *c, double *scratch,
                   double *out, void *stream);
/* out[0] = max |a - b| (b may be NULL: max |a|) */
int wmg_maxabs(long long n, const double *a, const double *b, double *out, void *stream);

/* elementwise float64 ops (individually rounded, no FMA) */
int wmg_axpy(long long n, double *out, const double *y, double alpha, int sgn, const double *x,
             void *stream);
int wmg_lincomb(long long n, double *out, double a, const double *x, double b, const double *y,
                double c, const double *z, void *stream);
int wmg_bicg_p(long long n, double *p, const double *r, double beta, double omega,
               const double *v, void *stream);
int wmg_bicg_x(long long n, double *x, double alpha, const double *ph, double omega,
               const double *sh, void *stream);
int wmg_scale(long long n, double *out, double a, const double *x, const double *y,
              void *stream);
int wmg_recip(long long n, double *out, const double *s, void *stream);
/* WMG node smoother sweep: z += omega * (c .* (r - az)),
 * az may be NULL (z = 0 before the first sweep). */
int wmg_smooth_update(long long n, double *z, double omega, const double *c, const double *r,
                      const double *az, void *stream);
int wmg_sirt_update(long long n, double *x, const double *c, const double *g, double lam,
                    void *stream);
int wmg_add_scaled(long long n, double *out, const double *g, double lam, int sgn,
                   const double *v, void *stream);
int wmg_cgs_update(long long n, int k, double *w, const double *V, long long ldv,
                   const double *h, void *stream);
int wmg_combo(long long n, int k, double *out, const double *V, long long ldv, const double *cf,
              int accumulate, void *stream);
int wmg_cast(long long n, int to_f32, void *out, const void *in, void *stream);
/* Host -> device copy of a caller's pageable vector (the numpy `w @ x` calls,
 * geometry.py:200-215) staged through `pinned` (>= bytes of page-locked host
 * memory): host threads copy 4 MB chunks, each chunk's DMA is issued on the
 * stream as soon as it has landed.  Returns once every DMA is issued; `pinned`
 * may be reused after the stream passes them. */
int wmg_h2d_staged(void *dst, const void *src, size_t bytes, void *pinned, int threads,
                   void *stream);
/* device-coefficient variants (coefficient read from device memory, so solver
 * iterations can be captured in a CUDA graph): out = y + sgn*(coef[0]*x);
 * out = a*x + coef[0]*y */
int wmg_axpy_dev(long long n, double *out, const double *y, const double *coef, int sgn,
                 const double *x, void *stream);
int wmg_lincomb_dev(long long n, double *out, double a, const double *x, const double *coef,
                    const double *y, void *stream);
/* CGLS / flexible PCG-NE scalar recurrences on device slots (see vecops.cu):
 * op 0 alpha = gamma/(qq + lam pp); op 1 beta = ss/gamma; op 2 beta = pr/gamma */
int wmg_cgls_scalars(double *S, double lam, int op, void *stream);
/* Fused forms for vectors of at most 2^20 elements (the last
 * reduction level, the scalar recurrence and the vector update in one launch;
 * bit-identical to wmg_det_reduce + wmg_cgls_scalars + wmg_axpy_dev /
 * wmg_lincomb_dev).  wmg_det_partials runs level 1 of wmg_det_reduce only:
 * reduction k's ceil(n/1024) chunk sums at partials + k * ceil(n/1024)
 * (wmg_det_scratch_len doubles).  gamma is read from S[11] by wmg_cgls_update
 * (which commits it to S[0]) and written to S[11] by wmg_cgls_direction.
 *   wmg_cgls_update:    partials of <q,q> (and, when lam != 0, partials_pp of <p,p>; else
 *                       NULL);  alpha = gamma / (qq + lam pp);  x += alpha p;  r -= alpha q
 *   wmg_cgls_direction: mode 1: partials of <s,s>; beta = ss / gamma; gamma' = ss
 *                       mode 2: partials of <s,s>, <z,s>, <z,s - s_old>; beta = pr / gamma;
 *                       gamma' = zs;   then p = z + beta p */
int wmg_det_partials(long long n, int K, const int *ops, const double *const *a,
                     const double *const *b, const double *const *c, double *partials,
                     void *stream);
int wmg_cgls_update(long long n_img, long long n_sino, double *x, const double *p, double *r,
                    const double *q, const double *partials, const double *partials_pp,
                    double lam, double *S, void *stream);
int wmg_cgls_direction(long long n, double *p, const double *z, const double *partials, int mode,
                       double *S, void *stream);

/* Haar intergrid operators (side even).  band: 0 LL, 1 LH, 2 HL, 3 HH.
 * restrict: out holds one (side/2)^2 block per band set in band_mask, in band
 * order.  prolong: fine = (accumulate ? fine : 0) + R_band^T coarse. */
int wmg_haar_restrict(int side, const double *fine, int band_mask, double *out, void *stream);
/* Batched forms for the sibling batches of the hybrid cycle (wtg_apply,
 * multilevel.py:175-198), bit-identical to one wmg_haar_restrict /
 * wmg_haar_prolong / wmg_smooth_update call per item: items contiguous (fine
 * side^2 apart, coarse nbands * (side/2)^2 apart, smoother vectors n apart).
 * wmg_haar_prolong_batch applies the nbands bands in the order given, each
 * added to the running fine value (the first one overwrites when !accumulate);
 * wmg_smooth_update_batch takes host arrays of per-item omegas and scaling
 * pointers (device memory). */
int wmg_haar_restrict_batch(int side, int batch, const double *fine, int band_mask, double *out,
                            void *stream);
int wmg_haar_prolong_batch(int side, int batch, int nbands, const int *bands,
                           const double *coarse, double *fine, int accumulate, void *stream);
int wmg_smooth_update_batch(long long n, int batch, double *z, const double *omegas,
                            const double *const *c, const double *r, const double *az,
                            void *stream);
int wmg_haar_prolong(int side, const double *coarse, int band, double *fine, int accumulate,
                     void *stream);

/* WMG coarse solves: y_b = A_b x_b for b < batch, A_b p x p row-major float64
 * (the stored SPD inverse of leaf b's Gram), p <= 24576.  Replaces the
 * reference's cho_solve (sparse_kernels.py:68-75) inside the V-cycle. */
int wmg_batched_gemv(int batch, int p, const double *A, long long strideA, const double *x,
                     long long stridex, double *y, long long stridey, void *stream);

/* Band-path Haar operators of a batch of WMG nodes (bands: host int[batch *
 * depth], item i's bands of levels 0..depth-1, level 0 = the finest, codes
 * LL 0, LH 1, HL 2, HH 3): fine_i (n x n) = R_path_i^T coarse_i and coarse_i =
 * R_path_i fine_i ((n >> depth)^2 each; items contiguous).  The per-level
 * wmg_haar_prolong / wmg_haar_restrict fused into one launch, bit-identical to
 * applying them level by level (the reference's Kronecker products,
 * multilevel.py:36-79, along the node's path). */
int wmg_haar_prolong_path(int n, int depth, int batch, const int *bands, const double *coarse,
                          double *fine, void *stream);
int wmg_haar_restrict_path(int n, int depth, int batch, const int *bands, const double *fine,
                           double *coarse, void *stream);

/* WMG leaf factor rows P_L[ray0 : ray0 + nrays, :] (row-major, caller zeroes P)
 * for the leaf reached by bands[0..depth) from the root. */
int wmg_leaf_factor(const wmg_geometry *g, int depth, const int *bands, long long ray0,
                    long long nrays, double *P, void *stream);

/* WMG leaf Gram, sparse: gram (p x p row-major float64, p = (n >> depth)^2,
 * zeroed by the caller) receives the lower triangle of P_L^T P_L, accumulated
 * per ray bundle without forming P_L (weights from the fp64 slab formula,
 * <= 1e-12 of the exact ones) in 64-bit fixed point, so the result is
 * bit-reproducible; *overflow (device int, caller-zeroed) is set if a bundle's
 * footprint exceeded the kernel's window (then the result is incomplete).
 * Replaces the reference's P^T P of multilevel.py:125-130. */
int wmg_leaf_gram(const wmg_geometry *g, int depth, const int *bands, double *gram,
                  int *overflow, void *stream);

/* bytes of caller workspace wmg_spd_inverse needs for `batch` matrices of order p */
int wmg_spd_inverse_workspace(int batch, int p, size_t *bytes);

/* In-place inverse of `batch` SPD matrices G_b (p x p row-major float64 at
 * G + b * strideG; only the lower triangle is read; p % 128 == 0 -- pad with an
 * identity block otherwise): on return G_b holds the full symmetric G_b^-1.
 * Blocked symmetric sweep on the fp64 tensor cores (DMMA), p^3 flops per
 * matrix.  info (device int[batch], written) = 0, or the order of the first
 * leading minor that is not positive definite (potrf's convention; G_b is then
 * garbage).  Replaces the reference's per-leaf potrf (sparse_kernels.py:53-65,
 * called at multilevel.py:125-137) plus the inverse the V-cycle's GEMV needs.
 * Thread safety: calls are serialised by an internal lock (they share one
 * per-device look-ahead stream and its events); callers on different streams
 * are safe, their device work may overlap. */
int wmg_spd_inverse(int batch, int p, double *G, long long strideG, int *info, void *work,
                    void *stream);

/* Dense Cholesky factorization (LAPACK potrf, lower) of `batch` SPD matrices
 * G_b (p x p row-major float64 at G + b * strideG; p % 128 == 0 -- pad with an
 * identity block otherwise; only the lower triangle is read), in place: on
 * return G_b = L_b with zeros above the diagonal.  Right-looking, 128-blocks,
 * panel and trailing update on the fp64 tensor cores (DMMA).  dinv (device,
 * batch * wmg_cholesky_dinv_elems(p) doubles, written) receives the inverses
 * of the 128 x 128 diagonal blocks of L_b for wmg_cholesky_solve.  info
 * (device int[batch], written) = 0 or the order of the first leading minor
 * that is not positive definite (potrf's info).  Replaces scipy.linalg.
 * cholesky(lower=True) in cholesky_factor (sparse_kernels.py:53-65). */
int wmg_cholesky_dinv_elems(int p, long long *elems);
int wmg_cholesky_factor(int batch, int p, double *G, long long strideG, double *dinv, int *info,
                        void *stream);

/* Solve L_b L_b^T Z = B_b in place (LAPACK potrs): B_b is p x nrhs row-major
 * at B + b * strideB; L, dinv from wmg_cholesky_factor; p <= 12800.  One CTA
 * per (right-hand side, matrix), blocked forward / backward substitution in a
 * fixed summation order (bit-reproducible).  Replaces cho_solve in
 * cholesky_solve (sparse_kernels.py:68-75). */
int wmg_cholesky_solve(int batch, int p, const double *L, long long strideL, const double *dinv,
                       double *B, long long strideB, int nrhs, void *stream);

/* Packed symmetric storage (p % 128 == 0): the lower 128 x 128 tiles of a
 * symmetric matrix, tile (I, J), I >= J, at index I (I + 1) / 2 + J, each
 * row-major, diagonal tiles full.  *elems_per_matrix = doubles per packed
 * matrix; *scratch_bytes = device scratch wmg_packed_symv needs for `batch`
 * matrices (either pointer may be NULL). */
int wmg_packed_sym_sizes(int batch, int p, long long *elems_per_matrix, size_t *scratch_bytes);

/* packed_b <- lower tiles of the full symmetric A_b (row-major p x p) */
int wmg_sym_pack(int batch, int p, const double *A, long long strideA, double *packed,
                 long long strideP, void *stream);

/* y_b = A_b x_b for packed symmetric A_b: every tile is read once (its
 * transpose product serves the mirrored block), partial products summed in a
 * fixed order (deterministic).  The WMG coarse solves (reference cho_solve,
 * sparse_kernels.py:68-75) with half the bytes of wmg_batched_gemv. */
int wmg_packed_symv(int batch, int p, const double *packed, long long strideP, const double *x,
                    long long stridex, double *y, long long stridey, double *scratch,
                    void *stream);

#ifdef __cplusplus
}
#endif
#endif /* WMGB200_H */
