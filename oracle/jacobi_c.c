/* TEST INFRASTRUCTURE ONLY — threaded C restatement of the reference
 * Jacobi3D stencil, face pack/unpack and sequential oracle.
 *
 * Reference: /root/reference/pkg/src/charmlet/jacobi3d.py (cl/jacobi3d.py)
 *   stencil   cl/jacobi3d.py:165-172 (and 192-196): (((((x-+x+)+y-)+y+)+z-)+z+)/6.0
 *   residual  cl/jacobi3d.py:197-198: max |nxt - cur| over the interior
 *   pack      cl/jacobi3d.py:157-158 with _face_slices(d, True)  102-112
 *   unpack    cl/jacobi3d.py:160-163 with _face_slices(d, False) 102-112
 *   oracle    cl/jacobi3d.py:181-200
 * Layout: padded C-order (bx+2, by+2, bz+2), z contiguous, x slowest.
 * Built with -ffp-contract=off -fno-fast-math so every add and the divide
 * are single IEEE operations in the reference's order (bit-exact with numpy).
 * Only tests/, smoke() and bench.py's CPU-baseline legs load this library. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define IDX(i, j, k) (((size_t)(i) * (size_t)(py) + (size_t)(j)) * (size_t)(pz) + (size_t)(k))

int orc_max_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/* One relaxation sweep over planes [i0, i1) of the interior; optional
 * residual (max |new - old|) returned through *res. */
static double sweep(const double *cur, double *nxt, long bx, long by, long bz,
                    long i0, long i1, int want_res) {
    const long py = by + 2, pz = bz + 2;
    double worst = 0.0;
    (void)bx;
    for (long i = i0; i < i1; ++i)
        for (long j = 1; j <= by; ++j) {
            const double *xm = cur + IDX(i - 1, j, 0), *xp = cur + IDX(i + 1, j, 0);
            const double *ym = cur + IDX(i, j - 1, 0), *yp = cur + IDX(i, j + 1, 0);
            const double *c = cur + IDX(i, j, 0);
            double *o = nxt + IDX(i, j, 0);
            for (long k = 1; k <= bz; ++k) {
                double t = xm[k] + xp[k];
                t = t + ym[k];
                t = t + yp[k];
                t = t + c[k - 1];
                t = t + c[k + 1];
                t = t / 6.0;
                o[k] = t;
                if (want_res) {
                    /* NaN propagates, as in numpy's max (cl/jacobi3d.py:198) */
                    double dlt = fabs(t - c[k]);
                    if (dlt > worst || dlt != dlt) worst = dlt;
                }
            }
        }
    return worst;
}

typedef struct {
    const double *cur;
    double *nxt;
    long bx, by, bz, i0, i1;
    int want_res;
    double res;
} slab_t;

static void *slab_main(void *arg) {
    slab_t *s = (slab_t *)arg;
    s->res = sweep(s->cur, s->nxt, s->bx, s->by, s->bz, s->i0, s->i1, s->want_res);
    return NULL;
}

/* Static split of the x planes over nthreads pthreads (<=0: all cores).
 * max is order-independent, so the residual does not depend on the split. */
static double fan_out(const double *cur, double *nxt, long bx, long by, long bz,
                      int nthreads, int want_res) {
    if (nthreads <= 0) nthreads = orc_max_threads();
    if (nthreads > bx) nthreads = (int)bx;
    if (nthreads < 1) nthreads = 1;
    slab_t *s = (slab_t *)calloc((size_t)nthreads, sizeof(slab_t));
    pthread_t *t = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    double worst = 0.0;
    for (int q = 0; q < nthreads; ++q) {
        s[q] = (slab_t){cur, nxt, bx, by, bz, 1 + bx * q / nthreads,
                        1 + bx * (q + 1) / nthreads, want_res, 0.0};
        if (q > 0) pthread_create(&t[q], NULL, slab_main, &s[q]);
    }
    slab_main(&s[0]);
    for (int q = 0; q < nthreads; ++q) {
        if (q > 0) pthread_join(t[q], NULL);
        if (s[q].res > worst || s[q].res != s[q].res) worst = s[q].res;
    }
    free(s);
    free(t);
    return worst;
}

void orc_stencil(const double *cur, double *nxt, long bx, long by, long bz, int nthreads) {
    fan_out(cur, nxt, bx, by, bz, nthreads, 0);
}

double orc_stencil_residual(const double *cur, double *nxt, long bx, long by, long bz,
                            int nthreads) {
    return fan_out(cur, nxt, bx, by, bz, nthreads, 1);
}

/* Face plane geometry: axis a = d/2, plane = interior ? (d odd ? n : 1)
 * : (d odd ? n+1 : 0). The face is C-order over the two remaining axes. */
static long face_plane(int d, long n, int interior) {
    if (d & 1) return interior ? n : n + 1;
    return interior ? 1 : 0;
}

static void face_copy(double *f, long bx, long by, long bz, int d, double *buf, int pack) {
    const long py = by + 2, pz = bz + 2;
    const int a = d / 2;
    if (a == 0) {
        long i = face_plane(d, bx, pack);
        for (long j = 1; j <= by; ++j)
            for (long k = 1; k <= bz; ++k) {
                double *p = f + IDX(i, j, k), *q = buf + (j - 1) * bz + (k - 1);
                if (pack) *q = *p; else *p = *q;
            }
    } else if (a == 1) {
        long j = face_plane(d, by, pack);
        for (long i = 1; i <= bx; ++i)
            for (long k = 1; k <= bz; ++k) {
                double *p = f + IDX(i, j, k), *q = buf + (i - 1) * bz + (k - 1);
                if (pack) *q = *p; else *p = *q;
            }
    } else {
        long k = face_plane(d, bz, pack);
        for (long i = 1; i <= bx; ++i)
            for (long j = 1; j <= by; ++j) {
                double *p = f + IDX(i, j, k), *q = buf + (i - 1) * by + (j - 1);
                if (pack) *q = *p; else *p = *q;
            }
    }
}

void orc_pack(const double *field, long bx, long by, long bz, int d, double *out) {
    face_copy((double *)field, bx, by, bz, d, out, 1);
}

void orc_unpack(double *field, long bx, long by, long bz, int d, const double *in) {
    face_copy(field, bx, by, bz, d, (double *)in, 0);
}

/* Sequential oracle: returns 0 on success, -1 on allocation failure.
 * out_interior: nx*ny*nz doubles (C order); residuals: iters doubles. */
int orc_sequential(long nx, long ny, long nz, int iters, double hot, double background,
                   double fill, double *out_interior, double *residuals, int nthreads) {
    const long py = ny + 2, pz = nz + 2;
    const size_t n = (size_t)(nx + 2) * py * pz;
    double *g = (double *)malloc(n * sizeof(double));
    double *h = (double *)malloc(n * sizeof(double));
    if (!g || !h) {
        free(g);
        free(h);
        return -1;
    }
    for (size_t q = 0; q < n; ++q) g[q] = background;
    for (long i = 1; i <= nx; ++i)
        for (long j = 1; j <= ny; ++j)
            for (long k = 1; k <= nz; ++k) g[IDX(i, j, k)] = fill;
    for (size_t q = 0; q < (size_t)py * pz; ++q) g[q] = hot;
    memcpy(h, g, n * sizeof(double));
    for (int it = 0; it < iters; ++it) {
        double r = orc_stencil_residual(g, h, nx, ny, nz, nthreads);
        if (residuals) residuals[it] = r;
        double *t = g;
        g = h;
        h = t;
    }
    for (long i = 1; i <= nx; ++i)
        for (long j = 1; j <= ny; ++j)
            memcpy(out_interior + ((size_t)(i - 1) * ny + (j - 1)) * nz, g + IDX(i, j, 1),
                   (size_t)nz * sizeof(double));
    free(g);
    free(h);
    return 0;
}
