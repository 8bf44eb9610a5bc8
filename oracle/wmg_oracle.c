/*
 * wmg_oracle.c -- CPU ORACLE for the line-intersection projector pair.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it, and there only as the
 * checker (or the timed CPU baseline), never as the product path.
 *
 * It is a plain-C restatement of the reference algorithm, compiled with
 * -ffp-contract=off so every product and sum is individually rounded exactly
 * as numpy/scipy do on x86-64:
 *
 *   ray crossings, sort, segment/midpoint filter, flat index
 *       <- /root/reference/pkg/src/wmgtomo/geometry.py:88-128 (_line_entries)
 *   COO -> sum_duplicates -> CSR -> sort_indices
 *       <- geometry.py:186-197 (build_projector); scipy _coo._sum_duplicates
 *          (lexsort, stable, then np.add.reduceat)
 *   W x  (sequential per row, ascending column, starts at 0.0)
 *       <- geometry.py:200-206 (apply) -> scipy sparsetools csr_matvec
 *   W^T y (per pixel, ascending ray index)
 *       <- geometry.py:209-215 (apply_transpose) -> csc_matvec; solvers.py:111
 *   row sums = first + numpy pairwise sum of the rest (np.add.reduceat)
 *       <- solvers.py:79-86 (sirt_scaling) -> scipy _minor_reduce
 *   column sums = W^T 1 (same order as W^T y)
 *       <- solvers.py:82 -> scipy _spbase.sum(axis=0) = ones @ W
 *
 * Parity of this restatement is pinned against the reference itself by
 * tests/golden/make_golden.py (sha256 of the reference CSR arrays and of
 * W x / W^T y on seeded vectors), checked in tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

/* ------------------------------------------------------------------------ */
/* minimal dynamic parallel-for over [0, total) with pthreads                 */
/* ------------------------------------------------------------------------ */
typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi, void *scratch);
typedef struct {
    range_fn fn;
    void *ctx;
    int64_t total, grain;
    int64_t next; /* guarded by mu */
    pthread_mutex_t mu;
    int n;        /* grid side for scratch */
    int fail;
} pool_t;

static int g_threads = 0;

int orc_set_threads(int t) { g_threads = t; return 0; }

int orc_num_threads(void)
{
    if (g_threads > 0) return g_threads;
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

/* ------------------------------------------------------------------------ */
/* numpy pairwise summation (loops_utils.h.src, PW_BLOCKSIZE = 128)          */
/* ------------------------------------------------------------------------ */
static double np_pairwise(const double *a, int64_t n)
{
    if (n < 8) {
        double r = -0.0;
        for (int64_t i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double acc[8];
        for (int k = 0; k < 8; ++k) acc[k] = a[k];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) acc[k] += a[i + k];
        double r = ((acc[0] + acc[1]) + (acc[2] + acc[3])) +
                   ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        for (; i < n; ++i) r += a[i];
        return r;
    }
    int64_t h = n / 2;
    h -= h % 8;
    return np_pairwise(a, h) + np_pairwise(a + h, n - h);
}

/* np.add.reduceat over one non-empty segment: first element + pairwise(rest) */
static double np_reduceat_segment(const double *a, int64_t n)
{
    return a[0] + np_pairwise(a + 1, n - 1);
}

double orc_reduceat_segment(const double *a, int64_t n)
{
    return n > 0 ? np_reduceat_segment(a, n) : 0.0;
}

/* ------------------------------------------------------------------------ */
/* one ray of the line kernel                                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t col;
    double val;
    int64_t order; /* position in the ray's t-sorted segment list */
} entry_t;

static int cmp_double(const void *pa, const void *pb)
{
    double a = *(const double *)pa, b = *(const double *)pb;
    return (a > b) - (a < b);
}

static int cmp_entry(const void *pa, const void *pb)
{
    const entry_t *a = (const entry_t *)pa, *b = (const entry_t *)pb;
    if (a->col != b->col) return (a->col > b->col) - (a->col < b->col);
    return (a->order > b->order) - (a->order < b->order); /* stable */
}

/*
 * Entries of ray j for an angle with snapped trig (c, s); the caller supplies
 * scratch of 2(n+1) doubles (t) and 2n+1 entries (e).  Returns the number of
 * CSR entries written to cols/vals (sorted by column, duplicates merged the way
 * COO.sum_duplicates does).  *n_dup receives the number of merged duplicates.
 */
static int64_t ray_entries(int n, int d, double c, double s, int j,
                           double *t, entry_t *e, int64_t *cols, double *vals,
                           int64_t *n_dup)
{
    const double half = n / 2.0;
    const double off = ((double)j - (d - 1) / 2.0) * 1.0;
    const double ox = off * c, oy = off * s;
    const double dx = -s, dy = c;
    const int use_x = fabs(dx) > 1e-12, use_y = fabs(dy) > 1e-12;
    for (int k = 0; k <= n; ++k) {
        const double line = ((double)k - n / 2.0) * 1.0;
        t[k] = use_x ? (line - ox) / dx : INFINITY;
        t[n + 1 + k] = use_y ? (line - oy) / dy : INFINITY;
    }
    qsort(t, (size_t)(2 * (n + 1)), sizeof(double), cmp_double);
    int64_t ne = 0;
    for (int q = 0; q < 2 * n + 1; ++q) {
        const double seg = t[q + 1] - t[q];
        double tm = 0.5 * (t[q + 1] + t[q]);
        const int good = isfinite(seg) && seg > 1e-12;
        if (!good) tm = 0.0;
        const double xm = ox + tm * dx;
        const double ym = oy + tm * dy;
        const double fx = floor(xm + half), fy = floor(ym + half);
        if (!good) continue;
        if (!(fx >= 0.0 && fx < (double)n && fy >= 0.0 && fy < (double)n)) continue;
        const int64_t ix = (int64_t)fx, iy = (int64_t)fy;
        e[ne].col = (int64_t)(n - 1 - iy) * n + ix;
        e[ne].val = seg;
        e[ne].order = ne;
        ++ne;
    }
    qsort(e, (size_t)ne, sizeof(entry_t), cmp_entry);
    /* sum_duplicates: np.add.reduceat over runs of equal column */
    int64_t out = 0, dups = 0;
    double run[64];
    for (int64_t i = 0; i < ne;) {
        int64_t k = i + 1;
        while (k < ne && e[k].col == e[i].col) ++k;
        double v;
        if (k - i == 1) {
            v = e[i].val;
        } else {
            int64_t len = k - i;
            if (len > 64) len = 64; /* never happens for a line kernel */
            for (int64_t r = 0; r < len; ++r) run[r] = e[i + r].val;
            v = np_reduceat_segment(run, len);
            dups += (k - i) - 1;
        }
        cols[out] = e[i].col;
        vals[out] = v;
        ++out;
        i = k;
    }
    if (n_dup) *n_dup += dups;
    return out;
}

/*
 * Entries of ray j under the Joseph kernel (geometry.py:131-175): per slab k of
 * the dominant axis, cont = (o/q - ctr_k * (p/q)) + (n-1)/2, i0 = floor(cont),
 * w1 = cont - i0; pixels (i0, 1 - w1) and (i0 + 1, w1) inside the grid with a
 * positive weight, value = weight * (1/|q|).  Sorted by column (no duplicates
 * can occur within a ray).
 */
static int64_t joseph_entries(int n, int d, double c, double s, int j, entry_t *e,
                              int64_t *cols, double *vals)
{
    const double off = ((double)j - (d - 1) / 2.0) * 1.0;
    const double hc = (n - 1) / 2.0;
    const int ydom = fabs(c) >= fabs(s);
    const double q = ydom ? c : s, p = ydom ? s : c;
    const double t1 = off / q, r = p / q, scale = 1.0 / fabs(q);
    int64_t ne = 0;
    for (int k = 0; k < n; ++k) {
        const double ctr = ((double)k - hc) * 1.0;
        const double cont = (t1 - ctr * r) + hc;
        const double f = floor(cont);
        const int64_t i0 = (int64_t)f;
        const double w1 = cont - f;
        for (int t = 0; t < 2; ++t) {
            const int64_t idx = i0 + t;
            const double w = t ? w1 : 1.0 - w1;
            if (idx < 0 || idx >= n || !(w > 0.0)) continue;
            e[ne].col = ydom ? (int64_t)(n - 1 - k) * n + idx : (int64_t)(n - 1 - idx) * n + k;
            e[ne].val = w * scale;
            e[ne].order = ne;
            ++ne;
        }
    }
    qsort(e, (size_t)ne, sizeof(entry_t), cmp_entry);
    for (int64_t i = 0; i < ne; ++i) {
        cols[i] = e[i].col;
        vals[i] = e[i].val;
    }
    return ne;
}

/* ray kernel of the oracle's entry points: 0 line (default), 1 Joseph */
static int g_kernel = 0;
int orc_set_kernel(int k) { g_kernel = k; return 0; }

static int64_t entries(int n, int d, double c, double s, int j, double *t, entry_t *e,
                       int64_t *cols, double *vals, int64_t *n_dup)
{
    if (g_kernel == 1) return joseph_entries(n, d, c, s, j, e, cols, vals);
    return ray_entries(n, d, c, s, j, t, e, cols, vals, n_dup);
}

/* scratch for one thread */
typedef struct {
    double *t;
    entry_t *e;
    int64_t *cols;
    double *vals;
} scratch_t;

static int scratch_alloc(scratch_t *sc, int n)
{
    sc->t = (double *)malloc(sizeof(double) * (size_t)(2 * (n + 1)));
    sc->e = (entry_t *)malloc(sizeof(entry_t) * (size_t)(2 * n + 2));
    sc->cols = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * n + 2));
    sc->vals = (double *)malloc(sizeof(double) * (size_t)(2 * n + 2));
    return sc->t && sc->e && sc->cols && sc->vals;
}

static void scratch_free(scratch_t *sc)
{
    free(sc->t); free(sc->e); free(sc->cols); free(sc->vals);
}

/* ------------------------------------------------------------------------ */
/* thread pool driver                                                         */
/* ------------------------------------------------------------------------ */
static void *pool_worker(void *arg)
{
    pool_t *p = (pool_t *)arg;
    scratch_t sc;
    if (!scratch_alloc(&sc, p->n)) {
        pthread_mutex_lock(&p->mu);
        p->fail = 1;
        pthread_mutex_unlock(&p->mu);
        scratch_free(&sc);
        return NULL;
    }
    for (;;) {
        pthread_mutex_lock(&p->mu);
        const int64_t lo = p->next;
        p->next += p->grain;
        pthread_mutex_unlock(&p->mu);
        if (lo >= p->total) break;
        const int64_t hi = lo + p->grain < p->total ? lo + p->grain : p->total;
        p->fn(p->ctx, lo, hi, &sc);
    }
    scratch_free(&sc);
    return NULL;
}

static int par_for(int n, int64_t total, int64_t grain, range_fn fn, void *ctx)
{
    pool_t p;
    p.fn = fn; p.ctx = ctx; p.total = total; p.grain = grain > 0 ? grain : 1;
    p.next = 0; p.n = n; p.fail = 0;
    pthread_mutex_init(&p.mu, NULL);
    int nt = orc_num_threads();
    if (nt > 256) nt = 256;
    pthread_t th[256];
    int started = 0;
    for (int t = 1; t < nt; ++t)
        if (pthread_create(&th[started], NULL, pool_worker, &p) == 0) ++started;
    pool_worker(&p);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&p.mu);
    return p.fail ? -1 : 0;
}

typedef struct {
    int n, d;
    const double *cs, *sn;
    int64_t *counts;
    const int64_t *indptr;
    int64_t *indices;
    double *data;
    const double *x;
    double *y;
    int64_t dups;
    pthread_mutex_t mu;
} job_t;

static void job_counts(void *ctx, int64_t lo, int64_t hi, void *scr)
{
    job_t *J = (job_t *)ctx;
    scratch_t *sc = (scratch_t *)scr;
    int64_t dd = 0;
    for (int64_t ray = lo; ray < hi; ++ray) {
        const int a = (int)(ray / J->d), j = (int)(ray % J->d);
        J->counts[ray] = entries(J->n, J->d, J->cs[a], J->sn[a], j, sc->t, sc->e,
                                     sc->cols, sc->vals, &dd);
    }
    pthread_mutex_lock(&J->mu);
    J->dups += dd;
    pthread_mutex_unlock(&J->mu);
}

static void job_fill(void *ctx, int64_t lo, int64_t hi, void *scr)
{
    job_t *J = (job_t *)ctx;
    scratch_t *sc = (scratch_t *)scr;
    for (int64_t ray = lo; ray < hi; ++ray) {
        const int a = (int)(ray / J->d), j = (int)(ray % J->d);
        const int64_t k = entries(J->n, J->d, J->cs[a], J->sn[a], j, sc->t, sc->e,
                                      sc->cols, sc->vals, NULL);
        memcpy(J->indices + J->indptr[ray], sc->cols, sizeof(int64_t) * (size_t)k);
        memcpy(J->data + J->indptr[ray], sc->vals, sizeof(double) * (size_t)k);
    }
}

static void job_forward(void *ctx, int64_t lo, int64_t hi, void *scr)
{
    job_t *J = (job_t *)ctx;
    scratch_t *sc = (scratch_t *)scr;
    for (int64_t ray = lo; ray < hi; ++ray) {
        const int a = (int)(ray / J->d), j = (int)(ray % J->d);
        const int64_t k = entries(J->n, J->d, J->cs[a], J->sn[a], j, sc->t, sc->e,
                                      sc->cols, sc->vals, NULL);
        double acc = 0.0;
        for (int64_t i = 0; i < k; ++i) acc += sc->vals[i] * J->x[sc->cols[i]];
        J->y[ray] = acc;
    }
}

/* ------------------------------------------------------------------------ */
/* public oracle entry points (ctypes)                                        */
/* ------------------------------------------------------------------------ */

/* per-ray entry counts (length m*d); returns total duplicates merged, or -1 */
int64_t orc_row_counts(int n, int d, int m, const double *cs, const double *sn,
                       int64_t *counts)
{
    job_t J;
    memset(&J, 0, sizeof(J));
    J.n = n; J.d = d; J.cs = cs; J.sn = sn; J.counts = counts;
    pthread_mutex_init(&J.mu, NULL);
    const int rc = par_for(n, (int64_t)m * d, 64, job_counts, &J);
    pthread_mutex_destroy(&J.mu);
    return rc ? -1 : J.dups;
}

/* fill a CSR whose indptr (length m*d+1) the caller built from row counts */
int orc_fill_csr(int n, int d, int m, const double *cs, const double *sn,
                 const int64_t *indptr, int64_t *indices, double *data)
{
    job_t J;
    memset(&J, 0, sizeof(J));
    J.n = n; J.d = d; J.cs = cs; J.sn = sn; J.indptr = indptr;
    J.indices = indices; J.data = data;
    return par_for(n, (int64_t)m * d, 64, job_fill, &J);
}

/* matrix-free forward projection (bitwise = CSR W x); rays in parallel */
int orc_forward(int n, int d, int m, const double *cs, const double *sn,
                const double *x, double *y)
{
    job_t J;
    memset(&J, 0, sizeof(J));
    J.n = n; J.d = d; J.cs = cs; J.sn = sn; J.x = x; J.y = y;
    return par_for(n, (int64_t)m * d, 64, job_forward, &J);
}

/* matrix-free backprojection; sequential over rays (bitwise = csc_matvec) */
int orc_backward(int n, int d, int m, const double *cs, const double *sn,
                 const double *y, double *x)
{
    scratch_t sc;
    if (!scratch_alloc(&sc, n)) { scratch_free(&sc); return -1; }
    for (int64_t p = 0; p < (int64_t)n * n; ++p) x[p] = 0.0;
    for (int64_t ray = 0; ray < (int64_t)m * d; ++ray) {
        const int a = (int)(ray / d), j = (int)(ray % d);
        const int64_t k = entries(n, d, cs[a], sn[a], j, sc.t, sc.e, sc.cols,
                                      sc.vals, NULL);
        for (int64_t i = 0; i < k; ++i) x[sc.cols[i]] += sc.vals[i] * y[ray];
    }
    scratch_free(&sc);
    return 0;
}

/* ---- stored-CSR SpMV (the reference's per-pair work), rows in parallel ---- */
typedef struct {
    const int64_t *indptr, *indices;
    const double *data, *x;
    double *y;
} spmv_t;

static void job_spmv(void *ctx, int64_t lo, int64_t hi, void *scr)
{
    (void)scr;
    spmv_t *J = (spmv_t *)ctx;
    for (int64_t i = lo; i < hi; ++i) {
        double acc = 0.0;
        for (int64_t k = J->indptr[i]; k < J->indptr[i + 1]; ++k)
            acc += J->data[k] * J->x[J->indices[k]];
        J->y[i] = acc;
    }
}

/* y = A x for a CSR A (csr_matvec order, bitwise); rows in parallel.  Used for
 * W x with W's CSR and for W^T y with the CSR of W^T (solvers.py:111). */
int orc_csr_matvec(int64_t n_rows, const int64_t *indptr, const int64_t *indices,
                   const double *data, const double *x, double *y)
{
    spmv_t J = {indptr, indices, data, x, y};
    return par_for(1, n_rows, 256, job_spmv, &J);
}

/* row sums with np.add.reduceat semantics; empty rows give 0.0 */
void orc_csr_row_sums(int64_t n_rows, const int64_t *indptr, const double *data,
                      double *out)
{
    for (int64_t i = 0; i < n_rows; ++i) {
        const int64_t len = indptr[i + 1] - indptr[i];
        out[i] = len > 0 ? np_reduceat_segment(data + indptr[i], len) : 0.0;
    }
}
