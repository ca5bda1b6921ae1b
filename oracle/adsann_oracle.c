/* oracle/adsann_oracle.c — TEST INFRASTRUCTURE ONLY.  See adsann_oracle.h.
 *
 * Each function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).  Written from the reference's documented
 * behaviour; compiled with -ffp-contract=off so every multiply and add
 * rounds separately, exactly as the reference's -O3 x86-64 build does.
 */
#include "adsann_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char *orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ rng
 * rng.hpp:36-97.  Output i depends only on (seed, i). */
static uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

orc_rng orc_rng_make(uint64_t seed) {
    orc_rng r = {seed, 0, 0.0, 0};
    return r;
}

orc_rng orc_rng_for_stream(uint64_t seed, uint64_t tag) { return orc_rng_make(mix64(seed ^ tag)); }

uint64_t orc_rng_next_u64(orc_rng *r) {
    r->counter += 1;
    return mix64(r->seed + r->counter * 0x9E3779B97F4A7C15ULL);
}

double orc_rng_uniform(orc_rng *r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

double orc_rng_uniform_open0(orc_rng *r) {
    return (double)((orc_rng_next_u64(r) >> 11) + 1) * 0x1.0p-53;
}

uint64_t orc_rng_below(orc_rng *r, uint64_t n) { return orc_rng_next_u64(r) % n; }

/* rng.hpp:76-88: Box-Muller, cos variate returned first, sin variate cached. */
double orc_rng_normal(orc_rng *r) {
    if (r->has_cached) {
        r->has_cached = 0;
        return r->cached;
    }
    const double u1 = orc_rng_uniform_open0(r);
    const double u2 = orc_rng_uniform(r);
    const double mag = sqrt(-2.0 * log(u1));
    const double ang = 6.283185307179586476925286766559 * u2;
    r->cached = mag * sin(ang);
    r->has_cached = 1;
    return mag * cos(ang);
}

int orc_rng_draw(uint64_t seed, uint64_t tag, int use_stream, int kind, uint64_t arg,
                 int64_t count, void *out) {
    orc_rng r = use_stream ? orc_rng_for_stream(seed, tag) : orc_rng_make(seed);
    for (int64_t i = 0; i < count; ++i) {
        switch (kind) {
            case 0: ((uint64_t *)out)[i] = orc_rng_next_u64(&r); break;
            case 1: ((double *)out)[i] = orc_rng_uniform(&r); break;
            case 2: ((double *)out)[i] = orc_rng_normal(&r); break;
            default:
                if (arg == 0) return fail(1, "below: n must be > 0");
                ((uint64_t *)out)[i] = orc_rng_below(&r, arg);
                break;
        }
    }
    return 0;
}

/* ------------------------------------------------------------ transform */
#define TAG_TRANSFORM 0x9d5c41cf0f5e6a31ULL /* rng.hpp:27 */
#define TAG_KMEANS 0x6b1febc8d1a07445ULL    /* rng.hpp:29 */

static double dotd(const double *a, const double *b, int32_t n) {
    double s = 0.0;
    for (int32_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* transform.cpp:35-44: subtract projections on the already-orthonormal rows. */
static void project_out(double *m, int32_t dim, int32_t i) {
    double *v = m + (size_t)i * dim;
    for (int32_t j = 0; j < i; ++j) {
        const double *qj = m + (size_t)j * dim;
        const double proj = dotd(v, qj, dim);
        for (int32_t c = 0; c < dim; ++c) v[c] -= proj * qj[c];
    }
}

/* transform.cpp:47-97 */
int orc_generate_orthogonal(int32_t dim, uint64_t seed, double *out) {
    if (dim < 1) return fail(1, "generate_orthogonal: dim must be >= 1");
    orc_rng rng = orc_rng_for_stream(seed, TAG_TRANSFORM);
    const size_t nn = (size_t)dim * dim;
    for (size_t e = 0; e < nn; ++e) out[e] = orc_rng_normal(&rng);
    for (int32_t i = 0; i < dim; ++i) {
        double *v = out + (size_t)i * dim;
        for (int attempt = 0;; ++attempt) {
            project_out(out, dim, i);
            project_out(out, dim, i);
            const double norm = sqrt(dotd(v, v, dim));
            if (norm > 1e-8) {
                for (int32_t c = 0; c < dim; ++c) v[c] /= norm;
                break;
            }
            if (attempt > 8) return fail(2, "generate_orthogonal: could not orthonormalize");
            for (int32_t c = 0; c < dim; ++c) v[c] = orc_rng_normal(&rng);
        }
    }
    double worst = 0.0;
    for (int32_t i = 0; i < dim; ++i)
        for (int32_t j = i; j < dim; ++j) {
            const double g = dotd(out + (size_t)i * dim, out + (size_t)j * dim, dim);
            const double dev = fabs(g - (i == j ? 1.0 : 0.0));
            if (dev > worst) worst = dev;
        }
    if (worst > 1e-10) return fail(2, "generate_orthogonal: deviation %g exceeds 1e-10", worst);
    return 0;
}

/* transform.cpp:103-117: y_i = sum_j P[i][j] * x_j, fp64, stored fp32. */
int orc_apply_prefix(const double *P, int32_t dim, const float *x, int32_t d, float *y) {
    if (d < 0 || d > dim) return fail(1, "apply_prefix: d out of range");
    for (int32_t i = 0; i < d; ++i) {
        const double *row = P + (size_t)i * dim;
        double s = 0.0;
        for (int32_t j = 0; j < dim; ++j) s += row[j] * (double)x[j];
        y[i] = (float)s;
    }
    return 0;
}

/* transform.cpp:131-149 */
int orc_apply_dataset(const double *P, int32_t dim, const float *X, int32_t n, float *Y) {
    for (int64_t i = 0; i < n; ++i) orc_apply_prefix(P, dim, X + i * dim, dim, Y + i * dim);
    return 0;
}

/* transform.cpp:119-129: acc[j] += P[i][j] * x_i, rows outer. */
int orc_apply_transpose(const double *P, int32_t dim, const float *x, float *y) {
    double *acc = calloc((size_t)dim, sizeof(double));
    if (!acc) return fail(2, "oom");
    for (int32_t i = 0; i < dim; ++i) {
        const double *row = P + (size_t)i * dim;
        const double xi = x[i];
        for (int32_t j = 0; j < dim; ++j) acc[j] += row[j] * xi;
    }
    for (int32_t j = 0; j < dim; ++j) y[j] = (float)acc[j];
    free(acc);
    return 0;
}

/* ------------------------------------------------------------------ dco */

/* dco.cpp:63-68 */
int orc_threshold_multiplier(int32_t d, double eps0, double *out) {
    if (d < 1) return fail(1, "threshold_multiplier: d must be >= 1");
    if (!(eps0 > 0.0)) return fail(1, "threshold_multiplier: epsilon0 must be > 0");
    *out = 1.0 + eps0 / sqrt((double)d);
    return 0;
}

/* dco.cpp:32-37 + 54-61: factor[k] = (1 + eps0/sqrt(k))^2 * k / D, factor[0] = 0. */
int orc_ad_context(double eps0, int32_t delta_d, int32_t dim, double *factor) {
    if (!(eps0 > 0.0)) return fail(1, "dco: epsilon0 must be > 0");
    if (delta_d < 1 || delta_d > dim) return fail(1, "dco: delta_d must be in [1, D]");
    factor[0] = 0.0;
    for (int32_t k = 1; k < dim; ++k) {
        const double mult = 1.0 + eps0 / sqrt((double)k);
        factor[k] = mult * mult * (double)k / (double)dim;
    }
    return 0;
}

/* dco.hpp:86-93 */
double orc_l2_sq(const float *a, const float *b, int32_t d) {
    double s = 0.0;
    for (int32_t i = 0; i < d; ++i) {
        const double diff = (double)a[i] - (double)b[i];
        s += diff * diff;
    }
    return s;
}

typedef struct {
    int positive;
    double dist_sq, observed;
    int32_t dims;
} scan_out;

/* dco.hpp:122-148 (factor != NULL) and dco.hpp:152-177 (factor == NULL:
 * the exact partial scan, i.e. the test against r^2 itself). */
static scan_out scan(const float *data, const float *query, int32_t dim, int32_t d_start,
                     double s_start, double r, const double *factor, int32_t delta_d,
                     int test_at_start) {
    const double r_sq = r * r;
    double s = s_start;
    int32_t d = d_start;
    scan_out o;
    if (test_at_start && d > 0 && d < dim && s > (factor ? factor[d] * r_sq : r_sq)) {
        o.positive = 0;
        o.dist_sq = 0.0;
        o.observed = factor ? sqrt(s * dim / d) : sqrt(s);
        o.dims = d;
        return o;
    }
    while (d < dim) {
        const int32_t stop = d + delta_d < dim ? d + delta_d : dim;
        const float *a = data + (d - d_start);
        const float *b = query + (d - d_start);
        for (int32_t i = 0; i < stop - d; ++i) {
            const double diff = (double)a[i] - (double)b[i];
            s += diff * diff;
        }
        d = stop;
        if (d < dim && s > (factor ? factor[d] * r_sq : r_sq)) {
            o.positive = 0;
            o.dist_sq = 0.0;
            o.observed = factor ? sqrt(s * dim / d) : sqrt(s);
            o.dims = d;
            return o;
        }
    }
    o.positive = s <= r_sq;
    o.dist_sq = s;
    o.observed = sqrt(s);
    o.dims = dim;
    return o;
}

int orc_scan_kernel(int kind, const float *data, const float *query, int32_t dim,
                    int32_t d_start, double s_start, double r, double eps0, int32_t delta_d,
                    int test_at_start, int *positive, double *dist_sq, double *observed,
                    int *dims) {
    double *factor = NULL;
    if (kind == 0) {
        factor = malloc(sizeof(double) * (size_t)(dim > 0 ? dim : 1));
        const int rc = orc_ad_context(eps0, delta_d, dim, factor);
        if (rc) {
            free(factor);
            return rc;
        }
    }
    const scan_out o = scan(data, query, dim, d_start, s_start, r, factor, delta_d, test_at_start);
    free(factor);
    *positive = o.positive;
    *dist_sq = o.dist_sq;
    *observed = o.observed;
    *dims = o.dims;
    return 0;
}

/* dco.cpp:70-110 with validate_query dco.cpp:23-30 */
int orc_dco(int kind, const float *o, int32_t n_o, const float *q, int32_t n_q, double r,
            double eps0, int32_t delta_d, int *positive, double *distance, double *observed,
            int *dims) {
    if (n_o != n_q) return fail(1, "dco: vector lengths differ");
    if (n_o == 0) return fail(1, "dco: empty vectors");
    if (!(r >= 0.0) || !isfinite(r)) return fail(1, "dco: threshold must be finite and >= 0");
    const int32_t dim = n_o;
    if (kind == 0) { /* fd_scan */
        const double s = orc_l2_sq(o, q, dim);
        const double dist = sqrt(s);
        *positive = dist <= r;
        *observed = dist;
        *dims = dim;
        *distance = *positive ? dist : NAN;
        return 0;
    }
    scan_out res;
    if (kind == 1) { /* pd_scan */
        if (delta_d < 1 || delta_d > dim) return fail(1, "pd_scan: delta_d must be in [1, D]");
        res = scan(o, q, dim, 0, 0.0, r, NULL, delta_d, 0);
    } else { /* ad_sampling */
        double *factor = malloc(sizeof(double) * (size_t)dim);
        const int rc = orc_ad_context(eps0, delta_d, dim, factor);
        if (rc) {
            free(factor);
            return rc;
        }
        res = scan(o, q, dim, 0, 0.0, r, factor, delta_d, 0);
        free(factor);
    }
    *positive = res.positive;
    *observed = res.observed;
    *dims = res.dims;
    *distance = res.positive ? res.observed : NAN;
    return 0;
}

int orc_ad_scan_pairs(const float *X, const float *Q, int32_t dim, int64_t npairs,
                      const int64_t *rows, const int32_t *qidx, const double *r, double eps0,
                      int32_t delta_d, int pd_mode, uint8_t *positive, int32_t *dims,
                      double *dist_sq, double *observed) {
    double *factor = NULL;
    if (!pd_mode) {
        factor = malloc(sizeof(double) * (size_t)dim);
        const int rc = orc_ad_context(eps0, delta_d, dim, factor);
        if (rc) {
            free(factor);
            return rc;
        }
    }
    for (int64_t i = 0; i < npairs; ++i) {
        const scan_out o = scan(X + rows[i] * dim, Q + (int64_t)qidx[i] * dim, dim, 0, 0.0, r[i],
                                factor, delta_d, 0);
        positive[i] = (uint8_t)o.positive;
        dims[i] = o.dims;
        dist_sq[i] = o.positive ? o.dist_sq : NAN;
        observed[i] = o.observed;
    }
    free(factor);
    return 0;
}

/* --------------------------------------------------------------- kmeans */

/* ivf.cpp:36-60: nearest centroid, ties to the lowest index; objective is
 * the sequential fp64 sum of the per-point minima. */
static double assign_points(const float *X, int32_t n, int32_t d, const float *C, int32_t k,
                            int32_t *assignment, double *best_d2) {
    for (int64_t i = 0; i < n; ++i) {
        const float *x = X + i * d;
        double best = INFINITY;
        int32_t arg = 0;
        for (int32_t c = 0; c < k; ++c) {
            const double d2 = orc_l2_sq(x, C + (int64_t)c * d, d);
            if (d2 < best) {
                best = d2;
                arg = c;
            }
        }
        assignment[i] = arg;
        best_d2[i] = best;
    }
    double obj = 0.0;
    for (int64_t i = 0; i < n; ++i) obj += best_d2[i];
    return obj;
}

/* The assignment step on its own (ivf.cpp:36-60): nearest centroid by exact fp64
 * l2_sq, lowest id on ties; what build_ivf's buckets come from. */
int orc_assign(const float *X, int32_t n, int32_t d, const float *C, int32_t k, int32_t *assignment) {
    if (k < 1 || n < 0) return fail(1, "assign: bad shape");
    double *best = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    (void)assign_points(X, n, d, C, k, assignment, best);
    free(best);
    return 0;
}

/* ivf.cpp:62-117: k-means++ seeding with a sequential fp64 CDF walk. */
static void kmeanspp(const float *X, int32_t n, int32_t d, int32_t k, orc_rng *rng, float *C) {
    double *min_d2 = malloc(sizeof(double) * (size_t)n);
    char *chosen = calloc((size_t)n, 1);
    for (int32_t i = 0; i < n; ++i) min_d2[i] = INFINITY;
    int32_t pick = (int32_t)orc_rng_below(rng, (uint64_t)n);
    for (int32_t c = 0;; ++c) {
        chosen[pick] = 1;
        memcpy(C + (int64_t)c * d, X + (int64_t)pick * d, sizeof(float) * (size_t)d);
        if (c + 1 == k) break;
        const float *cent = C + (int64_t)c * d;
        for (int64_t i = 0; i < n; ++i) {
            const double d2 = orc_l2_sq(X + i * d, cent, d);
            if (d2 < min_d2[i]) min_d2[i] = d2;
        }
        double total = 0.0;
        for (int32_t i = 0; i < n; ++i) total += min_d2[i];
        pick = -1;
        if (total > 0.0) {
            const double u = orc_rng_uniform(rng) * total;
            double cum = 0.0;
            for (int32_t i = 0; i < n; ++i) {
                cum += min_d2[i];
                if (cum > u) {
                    pick = i;
                    break;
                }
            }
            if (pick < 0)
                for (int32_t i = n - 1; i >= 0; --i)
                    if (min_d2[i] > 0.0) {
                        pick = i;
                        break;
                    }
        }
        if (pick < 0) {
            for (int32_t i = 0; i < n; ++i)
                if (!chosen[i]) {
                    pick = i;
                    break;
                }
            if (pick < 0) pick = 0;
        }
    }
    free(min_d2);
    free(chosen);
}

/* ivf.cpp:121-190 */
/* The engine's "seeded sample" initialisation (ads_kmeans init 1, used for the
 * configs whose k-means++ would take too long; not a reference algorithm): a
 * partial Fisher-Yates shuffle of the row ids drawn from the same
 * Rng::for_stream(seed, kKmeans) stream, centroid c = row perm[c]. */
static void sample_init(const float *X, int32_t n, int32_t d, int32_t k, orc_rng *rng, float *C) {
    int32_t *perm = malloc(sizeof(int32_t) * (size_t)n);
    for (int32_t i = 0; i < n; ++i) perm[i] = i;
    for (int32_t c = 0; c < k; ++c) {
        const int64_t j = c + (int64_t)(orc_rng_next_u64(rng) % (uint64_t)(n - c));
        const int32_t tmp = perm[c];
        perm[c] = perm[j];
        perm[j] = tmp;
        memcpy(C + (int64_t)c * d, X + (int64_t)perm[c] * d, sizeof(float) * (size_t)d);
    }
    free(perm);
}

int orc_kmeans(const float *X, int32_t n, int32_t d, int32_t k, int max_iters, uint64_t seed,
               float *centroids, int32_t *assignment, double *objective, int *iterations) {
    return orc_kmeans_init(X, n, d, k, max_iters, seed, 0, centroids, assignment, objective,
                           iterations);
}

int orc_kmeans_init(const float *X, int32_t n, int32_t d, int32_t k, int max_iters, uint64_t seed,
                    int init, float *centroids, int32_t *assignment, double *objective,
                    int *iterations) {
    if (k < 1) return fail(1, "kmeans: k must be >= 1");
    if (k > n) return fail(1, "kmeans: k exceeds the number of points");
    orc_rng rng = orc_rng_for_stream(seed, TAG_KMEANS);
    if (init == 1) sample_init(X, n, d, k, &rng, centroids);
    else kmeanspp(X, n, d, k, &rng, centroids);
    double *best_d2 = malloc(sizeof(double) * (size_t)n);
    double *sums = malloc(sizeof(double) * (size_t)k * d);
    int64_t *counts = malloc(sizeof(int64_t) * (size_t)k);
    char *stolen = malloc((size_t)n);
    double prev_obj = INFINITY;
    *iterations = 0;
    for (int iter = 0; iter < max_iters; ++iter) {
        const double obj = assign_points(X, n, d, centroids, k, assignment, best_d2);
        *iterations = iter + 1;
        memset(sums, 0, sizeof(double) * (size_t)k * d);
        memset(counts, 0, sizeof(int64_t) * (size_t)k);
        for (int64_t i = 0; i < n; ++i) {
            const int32_t c = assignment[i];
            double *s = sums + (int64_t)c * d;
            for (int32_t j = 0; j < d; ++j) s[j] += X[i * d + j];
            ++counts[c];
        }
        for (int32_t c = 0; c < k; ++c) {
            if (counts[c] == 0) continue;
            for (int32_t j = 0; j < d; ++j)
                centroids[(int64_t)c * d + j] =
                    (float)(sums[(int64_t)c * d + j] / (double)counts[c]);
        }
        memset(stolen, 0, (size_t)n);
        for (int32_t c = 0; c < k; ++c) {
            if (counts[c] != 0) continue;
            double far_d2 = -1.0;
            int32_t far_i = -1;
            for (int32_t i = 0; i < n; ++i) {
                if (stolen[i]) continue;
                if (best_d2[i] > far_d2) {
                    far_d2 = best_d2[i];
                    far_i = i;
                }
            }
            if (far_i < 0) continue;
            stolen[far_i] = 1;
            memcpy(centroids + (int64_t)c * d, X + (int64_t)far_i * d, sizeof(float) * (size_t)d);
        }
        if (prev_obj < INFINITY) {
            const double denom = obj > 1e-30 ? obj : 1e-30;
            if (fabs(prev_obj - obj) / denom < 1e-4) break;
        }
        prev_obj = obj;
    }
    *objective = assign_points(X, n, d, centroids, k, assignment, best_d2);
    free(best_d2);
    free(sums);
    free(counts);
    free(stolen);
    return 0;
}

/* ----------------------------------------------------------- brute force */

/* bench.cpp:31-61: the K smallest (d2, id) pairs, lexicographic, ascending. */
int orc_brute_force_knn(const float *base, int32_t n, int32_t d, const float *queries,
                        int32_t nq, int32_t K, int32_t *ids) {
    if (K < 1) return fail(1, "brute_force_knn: K must be >= 1");
    if (K > n) return fail(1, "brute_force_knn: K exceeds dataset size");
    double *kd = malloc(sizeof(double) * (size_t)K);
    int32_t *ki = malloc(sizeof(int32_t) * (size_t)K);
    for (int64_t qi = 0; qi < nq; ++qi) {
        const float *q = queries + qi * d;
        int32_t cnt = 0;
        for (int32_t i = 0; i < n; ++i) {
            const double d2 = orc_l2_sq(base + (int64_t)i * d, q, d);
            if (cnt == K && !(d2 < kd[K - 1] || (d2 == kd[K - 1] && i < ki[K - 1]))) continue;
            int32_t pos = cnt < K ? cnt : K - 1;
            while (pos > 0 && (kd[pos - 1] > d2 || (kd[pos - 1] == d2 && ki[pos - 1] > i))) {
                kd[pos] = kd[pos - 1];
                ki[pos] = ki[pos - 1];
                --pos;
            }
            kd[pos] = d2;
            ki[pos] = i;
            if (cnt < K) ++cnt;
        }
        memcpy(ids + qi * K, ki, sizeof(int32_t) * (size_t)K);
    }
    free(kd);
    free(ki);
    return 0;
}

/* ------------------------------------------------------------------ ivf */

/* ivf.cpp:211-256 (layout only; clustering supplied by the caller). */
int orc_ivf_layout(int32_t n, int32_t d, int32_t k, int32_t d1, int split, const double *P,
                   const float *centroids_t, const int32_t *assignment, const float *raw,
                   const float *t, int64_t *list_off, int32_t *ids_flat, float *vec_t,
                   float *vec_raw, float *a1_t, float *a2_t, float *a1_raw, float *a2_raw,
                   float *centroids_raw) {
    if (split && (d1 < 1 || d1 >= d)) return fail(1, "build_ivf: split layout needs 1 <= d1 < D");
    if (k < 1) return fail(1, "layout: k must be >= 1");
    for (int32_t c = 0; c <= k; ++c) list_off[c] = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (assignment[i] < 0 || assignment[i] >= k) return fail(1, "layout: bad assignment");
        list_off[assignment[i] + 1]++;
    }
    for (int32_t c = 0; c < k; ++c) list_off[c + 1] += list_off[c];
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)k);
    memcpy(fill, list_off, sizeof(int64_t) * (size_t)k);
    for (int32_t i = 0; i < n; ++i) ids_flat[fill[assignment[i]]++] = i; /* ascending ids */
    free(fill);
    const int32_t d2 = d - d1;
    for (int64_t p = 0; p < n; ++p) {
        const float *xt = t + (int64_t)ids_flat[p] * d;
        const float *xr = raw + (int64_t)ids_flat[p] * d;
        if (vec_t) memcpy(vec_t + p * d, xt, sizeof(float) * (size_t)d);
        if (vec_raw) memcpy(vec_raw + p * d, xr, sizeof(float) * (size_t)d);
        if (split) {
            if (a1_t) memcpy(a1_t + p * d1, xt, sizeof(float) * (size_t)d1);
            if (a2_t) memcpy(a2_t + p * d2, xt + d1, sizeof(float) * (size_t)d2);
            if (a1_raw) memcpy(a1_raw + p * d1, xr, sizeof(float) * (size_t)d1);
            if (a2_raw) memcpy(a2_raw + p * d2, xr + d1, sizeof(float) * (size_t)d2);
        }
    }
    if (centroids_raw)
        for (int32_t c = 0; c < k; ++c)
            orc_apply_transpose(P, d, centroids_t + (int64_t)c * d, centroids_raw + (int64_t)c * d);
    return 0;
}

typedef struct {
    double dist;
    int32_t id;
} pair_t;

static int pair_lt(pair_t a, pair_t b) { return a.dist < b.dist || (a.dist == b.dist && a.id < b.id); }

/* ivf.cpp:283-292: (l2_sq(centroid, q), id) pairs, partial sort, first nprobe. */
int orc_probe_order(const float *centroids, int32_t L, int32_t d, const float *q,
                    int32_t nprobe, int32_t *order) {
    pair_t *best = malloc(sizeof(pair_t) * (size_t)nprobe);
    int32_t cnt = 0;
    for (int32_t c = 0; c < L; ++c) {
        pair_t p = {orc_l2_sq(centroids + (int64_t)c * d, q, d), c};
        if (cnt == nprobe && !pair_lt(p, best[nprobe - 1])) continue;
        int32_t pos = cnt < nprobe ? cnt : nprobe - 1;
        while (pos > 0 && pair_lt(p, best[pos - 1])) {
            best[pos] = best[pos - 1];
            --pos;
        }
        best[pos] = p;
        if (cnt < nprobe) ++cnt;
    }
    for (int32_t i = 0; i < nprobe; ++i) order[i] = best[i].id;
    free(best);
    return 0;
}

/* ivf.cpp:262-281: bounded max-heap keyed on (dist, id) pairs; kept here as
 * an ascending array so that the back is priority_queue::top(). */
typedef struct {
    pair_t *a;
    int32_t cnt, cap;
} heap_t;

static double heap_threshold(const heap_t *h) { return h->cnt < h->cap ? INFINITY : h->a[h->cnt - 1].dist; }

static void heap_offer(heap_t *h, double dist, int32_t id) {
    if (h->cnt == h->cap) {
        if (!(dist < h->a[h->cnt - 1].dist)) return; /* strict: ties not inserted */
        h->cnt--;                                    /* pop the max pair */
    }
    pair_t p = {dist, id};
    int32_t pos = h->cnt;
    while (pos > 0 && pair_lt(p, h->a[pos - 1])) {
        h->a[pos] = h->a[pos - 1];
        --pos;
    }
    h->a[pos] = p;
    h->cnt++;
}

/* Shared body.  Refresh before candidate i when i == 0, or (waves == NULL)
 * i >= first && (i - first) % step == 0, or (waves != NULL) i is the stream
 * position of the first candidate of probe rank waves[j] (j < nwaves). */
static int ivf_query_impl(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                          int32_t nprobe, int mode, double eps0, int32_t delta_d, int64_t first,
                          int64_t step, int32_t probe_lo, double r0, const int32_t *waves,
                          int32_t nwaves, int32_t lag, int32_t *ids, double *dists, int32_t *count,
                          uint64_t *stats);

int orc_ivf_query(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                  int32_t nprobe, int mode, double eps0, int32_t delta_d, int64_t first,
                  int64_t step, int32_t *ids, double *dists, int32_t *count, uint64_t *stats) {
    return ivf_query_impl(idx, q_t, q_raw, K, nprobe, mode, eps0, delta_d, first, step, 0, INFINITY,
                          NULL, 0, 0, ids, dists, count, stats);
}

int orc_ivf_query_waves(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                        int32_t nprobe, int mode, double eps0, int32_t delta_d,
                        const int32_t *wave_ranks, int32_t nwaves, int32_t *ids, double *dists,
                        int32_t *count, uint64_t *stats) {
    return ivf_query_impl(idx, q_t, q_raw, K, nprobe, mode, eps0, delta_d, 1, 1, 0, INFINITY,
                          wave_ranks, nwaves, 0, ids, dists, count, stats);
}

int orc_ivf_query_ext(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                      int32_t nprobe, int mode, double eps0, int32_t delta_d, int64_t first,
                      int64_t step, int32_t probe_lo, double r0, int32_t *ids, double *dists,
                      int32_t *count, uint64_t *stats) {
    if (probe_lo < 0 || probe_lo > nprobe) return fail(1, "ivf_query: probe_lo must be in [0, n_probe]");
    if (!(r0 >= 0.0)) return fail(1, "ivf_query: the initial radius must be >= 0");
    return ivf_query_impl(idx, q_t, q_raw, K, nprobe, mode, eps0, delta_d, first, step, probe_lo, r0,
                          NULL, 0, 0, ids, dists, count, stats);
}

/* lag = 1: the positives of a chunk are offered one refresh later, so the
 * candidates of chunk j see the heap after chunks 0 .. j-2 (the GPU's mixed
 * scan re-walks a chunk's undecided candidates during the next chunk).
 * lag = 2: the same from chunk 2 on; chunk 1 still sees chunk 0's positives
 * (the GPU's overlapped chunks, opts.lag = 1: chunk c >= 2 is tested against
 * the thresholds after chunk c - 2, chunk 1 against chunk 0's). */
int orc_ivf_query_lag(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                      int32_t nprobe, int mode, double eps0, int32_t delta_d, int64_t first,
                      int64_t step, int32_t lag, int32_t *ids, double *dists, int32_t *count,
                      uint64_t *stats) {
    if (lag < 0 || lag > 2) return fail(1, "ivf_query: lag must be 0, 1 or 2");
    return ivf_query_impl(idx, q_t, q_raw, K, nprobe, mode, eps0, delta_d, first, step, 0, INFINITY,
                          NULL, 0, lag, ids, dists, count, stats);
}

/* probe_lo / r0 (the sharded search's second wave): only the lists at probe
 * ranks probe_lo .. n_probe-1 are scanned, and r starts at the bound r0 and
 * is min(r0, heap threshold) at every refresh (the heap's max never exceeds
 * r0 once full, since every positive satisfied dist <= r). */
static int ivf_query_impl(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                          int32_t nprobe, int mode, double eps0, int32_t delta_d, int64_t first,
                          int64_t step, int32_t probe_lo, double r0, const int32_t *waves,
                          int32_t nwaves, int32_t lag, int32_t *ids, double *dists, int32_t *count,
                          uint64_t *stats) {
    /* ivf.cpp:299-307 */
    if (K < 1) return fail(1, "ivf_query: K must be >= 1");
    if (nprobe < 1 || nprobe > idx->k_clusters)
        return fail(1, "ivf_query: n_probe must be in [1, k_clusters]");
    const int split_mode = mode == 3 || mode == 4;
    if (split_mode && !idx->split) return fail(1, "ivf_query: split mode needs a split-layout index");
    const int transformed = mode == 2 || mode == 3;
    const float *q = transformed ? q_t : q_raw;
    if (!q) return fail(1, "ivf_query: missing query vector");
    if (first < 1 || step < 1) return fail(1, "ivf_query: bad threshold schedule");
    if (split_mode ? !(transformed ? idx->a1_t : idx->a1_raw) : !(transformed ? idx->vec_t : idx->vec_raw))
        return fail(1, "ivf_query: the layout lacks the arrays this mode reads");
    const int32_t d = idx->d, d1 = idx->d1;

    double *factor = NULL;
    if (transformed) { /* ivf.cpp:313 */
        factor = malloc(sizeof(double) * (size_t)d);
        const int rc = orc_ad_context(eps0, delta_d, d, factor);
        if (rc) {
            free(factor);
            return rc;
        }
    }
    int32_t *probes = malloc(sizeof(int32_t) * (size_t)nprobe);
    orc_probe_order(transformed ? idx->centroids_t : idx->centroids_raw, idx->k_clusters, d, q,
                    nprobe, probes);

    heap_t heap = {malloc(sizeof(pair_t) * (size_t)K), 0, K};
    int64_t total = 0;
    for (int32_t i = probe_lo; i < nprobe; ++i) total += idx->list_off[probes[i] + 1] - idx->list_off[probes[i]];
    pair_t *pending = malloc(sizeof(pair_t) * (size_t)(total > 0 ? total : 1));
    int64_t npend = 0;
    /* lag 1: the previous chunk's positives, offered at the next refresh */
    pair_t *held = malloc(sizeof(pair_t) * (size_t)(total > 0 ? total : 1));
    int64_t nheld = 0;
    uint64_t dims = 0;
    double r = r0;

    /* Split modes precompute the A1 prefix of every candidate first
     * (ivf.cpp:366-386); contiguous modes scan in one pass. */
    double *prefix = NULL;
    if (split_mode) {
        prefix = malloc(sizeof(double) * (size_t)(total > 0 ? total : 1));
        const float *a1 = mode == 3 ? idx->a1_t : idx->a1_raw;
        int64_t i = 0;
        for (int32_t pi = probe_lo; pi < nprobe; ++pi)
            for (int64_t p = idx->list_off[probes[pi]]; p < idx->list_off[probes[pi] + 1]; ++p, ++i) {
                double s = 0.0;
                for (int32_t j = 0; j < d1; ++j) {
                    const double diff = (double)a1[p * d1 + j] - (double)q[j];
                    s += diff * diff;
                }
                prefix[i] = s;
            }
        dims += (uint64_t)total * (uint64_t)d1;
    }

    /* refresh marks (stream positions) for the wave schedule */
    char *mark = NULL;
    if (waves) {
        mark = calloc((size_t)(total + 1), 1);
        int64_t pos = 0;
        int32_t wj = 0;
        for (int32_t pi = probe_lo; pi < nprobe; ++pi) {
            while (wj < nwaves && waves[wj] < pi) ++wj;
            if (wj < nwaves && waves[wj] == pi) mark[pos] = 1;
            pos += idx->list_off[probes[pi] + 1] - idx->list_off[probes[pi]];
        }
    }
    int64_t i = 0, nref = 0;
    for (int32_t pi = probe_lo; pi < nprobe; ++pi) {
        const int32_t c = probes[pi];
        for (int64_t p = idx->list_off[c]; p < idx->list_off[c + 1]; ++p, ++i) {
            if (i == 0 || (waves ? mark[i] : (i >= first && (i - first) % step == 0))) {
                const int64_t ref = nref++; /* 0 at the stream start, c at the start of chunk c */
                if (lag == 1 || (lag == 2 && ref >= 2)) {
                    for (int64_t j = 0; j < nheld; ++j) heap_offer(&heap, held[j].dist, held[j].id);
                    pair_t *t = held;
                    held = pending;
                    pending = t;
                    nheld = npend;
                } else {
                    for (int64_t j = 0; j < npend; ++j) heap_offer(&heap, pending[j].dist, pending[j].id);
                }
                npend = 0;
                const double ht = heap_threshold(&heap); /* ivf.cpp:331, 391 */
                r = ht < r0 ? ht : r0;
            }
            const int32_t id = idx->ids_flat[p];
            if (!split_mode) {
                const float *vec = (transformed ? idx->vec_t : idx->vec_raw) + p * d;
                if (mode == 0) { /* ivf.cpp:334-339 */
                    const double s = orc_l2_sq(vec, q, d);
                    dims += (uint64_t)d;
                    const double dist = sqrt(s);
                    if (dist <= r) pending[npend++] = (pair_t){dist, id};
                } else {
                    const scan_out o = scan(vec, q, d, 0, 0.0, r, mode == 2 ? factor : NULL,
                                            delta_d, 0);
                    dims += (uint64_t)o.dims;
                    if (o.positive) pending[npend++] = (pair_t){o.observed, id};
                }
            } else { /* ivf.cpp:389-400 */
                const float *a2 = mode == 3 ? idx->a2_t : idx->a2_raw;
                const scan_out o = scan(a2 + p * (d - d1), q + d1, d, d1, prefix[i], r,
                                        mode == 3 ? factor : NULL, delta_d, 1);
                dims += (uint64_t)(o.dims - d1);
                if (o.positive) pending[npend++] = (pair_t){o.observed, id};
            }
        }
    }
    for (int64_t j = 0; j < nheld; ++j) heap_offer(&heap, held[j].dist, held[j].id);
    for (int64_t j = 0; j < npend; ++j) heap_offer(&heap, pending[j].dist, pending[j].id);

    *count = heap.cnt;
    for (int32_t j = 0; j < heap.cnt; ++j) {
        ids[j] = heap.a[j].id;
        dists[j] = heap.a[j].dist;
    }
    stats[0] = dims;
    stats[1] = (uint64_t)total;
    stats[2] = (uint64_t)total;
    free(factor);
    free(probes);
    free(heap.a);
    free(pending);
    free(held);
    free(prefix);
    free(mark);
    return 0;
}

/* bench.cpp:303-392 verify_theory: every (query, object) pair gets one
 * adaptive comparison with delta_d = 1 against the exact K-th nearest
 * squared distance r_sq of that query; reject_at[g] = the first d in [1, D)
 * with s_d > factor_g[d] * r_sq (the grid sorted ascending; a larger
 * epsilon0 never rejects earlier).  dims adds reject_at or D; a failure is
 * a positive (d2 <= r_sq) object that some epsilon0 rejects.  Outputs per
 * sorted grid entry: eps_sorted, dims (sum), failures; plus positives. */
static int cmp_double(const void *a, const void *b) {
    const double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

int orc_verify_theory(const float *X, int32_t n, int32_t d, const float *Q, int32_t nq, int32_t K,
                      const double *grid, int32_t G, double *eps_sorted, uint64_t *dims,
                      uint64_t *failures, uint64_t *positives) {
    if (K < 1 || K > n) return fail(1, "verify_theory: bad K");
    for (int32_t g = 0; g < G; ++g) eps_sorted[g] = grid[g];
    qsort(eps_sorted, (size_t)G, sizeof(double), cmp_double);
    double *factor = malloc(sizeof(double) * (size_t)G * (size_t)(d > 0 ? d : 1));
    for (int32_t g = 0; g < G; ++g) {
        const int rc = orc_ad_context(eps_sorted[g], 1, d, factor + (size_t)g * d);
        if (rc) {
            free(factor);
            return rc;
        }
        dims[g] = 0;
        failures[g] = 0;
    }
    *positives = 0;
    double *dist_sq = malloc(sizeof(double) * (size_t)n);
    double *kth = malloc(sizeof(double) * (size_t)n);
    int32_t *reject_at = malloc(sizeof(int32_t) * (size_t)(G > 0 ? G : 1));
    for (int32_t qi = 0; qi < nq; ++qi) {
        const float *q = Q + (size_t)qi * d;
        for (int32_t i = 0; i < n; ++i) dist_sq[i] = orc_l2_sq(X + (size_t)i * d, q, d);
        memcpy(kth, dist_sq, sizeof(double) * (size_t)n);
        qsort(kth, (size_t)n, sizeof(double), cmp_double);
        const double r_sq = kth[K - 1];
        for (int32_t i = 0; i < n; ++i) {
            const int positive = dist_sq[i] <= r_sq;
            if (positive) ++*positives;
            const float *o = X + (size_t)i * d;
            double s = 0.0;
            int32_t first_active = 0;
            for (int32_t g = 0; g < G; ++g) reject_at[g] = 0;
            for (int32_t dd = 1; dd < d && first_active < G; ++dd) {
                const double a = (double)o[dd - 1] - (double)q[dd - 1];
                s += a * a;
                while (first_active < G && s > factor[(size_t)first_active * d + dd] * r_sq) {
                    reject_at[first_active] = dd;
                    ++first_active;
                }
            }
            for (int32_t g = 0; g < G; ++g) {
                if (reject_at[g] > 0) {
                    dims[g] += (uint64_t)reject_at[g];
                    if (positive) ++failures[g];
                } else {
                    dims[g] += (uint64_t)d;
                }
            }
        }
    }
    free(factor);
    free(dist_sq);
    free(kth);
    free(reject_at);
    return 0;
}

/* ------------------------------------------------------------ mixture generator
 * Restatement of the engine's seeded Gaussian-mixture generator (the
 * benchmark configs' synthetic stand-in for the paper's datasets, DESIGN.md
 * §6), built on the reference's Rng (rng.hpp:36-97).  The bench's reference
 * arm generates config data with it, so that arm never loads the product
 * library; tests pin it bit-for-bit against ads_synth_rows.  Row r depends
 * only on (desc, r): component draw = counter r of the component stream,
 * noise = normals r*d .. r*d+d-1 of the noise stream.  Multi-threaded over
 * output rows (results do not depend on the thread count). */
#include <pthread.h>

#define TAG_CENTERS 0x43454e5445525331ULL /* "CENTERS1" */
#define TAG_COMP 0x434f4d504f4e5431ULL    /* "COMPONT1" */
#define TAG_NOISE 0x4e4f495345303031ULL   /* "NOISE001" */

typedef struct {
    const orc_synth_desc *s;
    const double *centers, *sig;
    uint64_t role_seed;
    int64_t row_lo, stride, lo, hi;
    float *out;
} synth_job;

static void *synth_work(void *arg) {
    const synth_job *j = (const synth_job *)arg;
    const orc_synth_desc *s = j->s;
    const int32_t d = s->d, C = s->components;
    double *row = (double *)malloc(sizeof(double) * (size_t)d);
    orc_rng comp = orc_rng_make(mix64(j->role_seed ^ TAG_COMP));
    orc_rng noise = orc_rng_for_stream(j->role_seed, TAG_NOISE);
    for (int64_t i = j->lo; i < j->hi; ++i) {
        const int64_t r = j->row_lo + i * j->stride;
        comp.counter = (uint64_t)r;
        /* normal m = r*d: pair p = m/2 consumes counters 2p+1, 2p+2 */
        const uint64_t m = (uint64_t)r * (uint64_t)d;
        noise.counter = 2 * (m / 2);
        noise.has_cached = 0;
        if (m % 2) (void)orc_rng_normal(&noise);
        int32_t c;
        if (s->assign_mode == 1) c = (int32_t)((r * C) / (s->n > 0 ? s->n : 1));
        else c = (int32_t)orc_rng_below(&comp, (uint64_t)C);
        const double *cc = j->centers + (size_t)c * d;
        double nrm = 0.0;
        for (int32_t k = 0; k < d; ++k) {
            double x = cc[k] + j->sig[k] * orc_rng_normal(&noise);
            if (s->kind == 1) x = fmin(255.0, fmax(0.0, round(x)));
            else if (s->kind == 2) x = fmin(1.0, fmax(0.0, x));
            row[k] = x;
            nrm += x * x;
        }
        float *o = j->out + (size_t)i * d;
        if (s->kind == 3) {
            const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
            for (int32_t k = 0; k < d; ++k) o[k] = (float)(row[k] * inv);
        } else {
            for (int32_t k = 0; k < d; ++k) o[k] = (float)row[k];
        }
    }
    free(row);
    return NULL;
}

int orc_synth_rows(const orc_synth_desc *s, int64_t row_lo, int64_t count, int64_t stride,
                   int32_t threads, float *out) {
    if (s->n < 0 || s->d < 1 || s->components < 1) return fail(1, "synth: bad shape");
    if (!(s->sigma >= 0.0)) return fail(1, "synth: sigma must be >= 0");
    if (count < 0 || stride < 1 || row_lo < 0 || (count > 0 && row_lo + (count - 1) * stride >= s->n))
        return fail(1, "synth: row range outside [0, n)");
    const int32_t d = s->d, C = s->components;
    double *centers = (double *)malloc(sizeof(double) * (size_t)C * d);
    double *sig = (double *)malloc(sizeof(double) * (size_t)d);
    orc_rng rng = orc_rng_for_stream(s->seed, TAG_CENTERS);
    for (size_t e = 0; e < (size_t)C * d; ++e) {
        if (s->kind == 1 || s->kind == 2)
            centers[e] = s->center_lo + (s->center_hi - s->center_lo) * orc_rng_uniform(&rng);
        else
            centers[e] = s->center_scale * orc_rng_normal(&rng);
    }
    for (int32_t k = 0; k < d; ++k)
        sig[k] = s->decay ? s->sigma / sqrt(1.0 + (double)k / 32.0) : s->sigma;
    const uint64_t role_seed = mix64(s->seed ^ (s->role * 0x9E3779B97F4A7C15ULL + 1));
    int32_t nt = threads < 1 ? 1 : (threads > 256 ? 256 : threads);
    if (count < 4096) nt = 1;
    synth_job jobs[256];
    pthread_t th[256];
    for (int32_t t = 0; t < nt; ++t) {
        synth_job j = {s, centers, sig, role_seed, row_lo, stride, count * t / nt,
                       count * (t + 1) / nt, out};
        jobs[t] = j;
    }
    for (int32_t t = 1; t < nt; ++t) pthread_create(&th[t], NULL, synth_work, &jobs[t]);
    synth_work(&jobs[0]);
    for (int32_t t = 1; t < nt; ++t) pthread_join(th[t], NULL);
    free(centers);
    free(sig);
    return 0;
}
