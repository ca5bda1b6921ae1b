/* oracle/adsann_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference's IVF/IVF++
 * ADSampling path (arXiv 2303.09855, /root/reference/proj).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker.  The product (paper_2303_09855_b200) never links or
 * calls it.
 *
 * Pinning: every function is checked bit-for-bit against the reference
 * itself (oracle/_ref/libadsann_ref.so, built from the reference sources
 * by oracle/Makefile) and against the committed golden vectors in
 * tests/golden/ (generated from that library by tests/golden/make_golden.py).
 *
 * Arithmetic contract (as in the reference, compiled without FMA):
 * fp64 accumulation over fp32 inputs in index order, one rounding per
 * operation: diff = (double)a - (double)b; s = s + diff*diff.
 *
 * Status codes: 0 ok, 1 invalid argument (std::invalid_argument in the
 * reference), 2 runtime error (std::runtime_error).
 */
#ifndef ADSANN_ORACLE_H
#define ADSANN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char *orc_last_error(void);

/* rng.hpp:36-97 — counter-based SplitMix64 + Box-Muller. */
typedef struct {
    uint64_t seed, counter;
    double cached;
    int has_cached;
} orc_rng;

orc_rng orc_rng_make(uint64_t seed);
orc_rng orc_rng_for_stream(uint64_t seed, uint64_t tag);
uint64_t orc_rng_next_u64(orc_rng *r);
double orc_rng_uniform(orc_rng *r);
double orc_rng_uniform_open0(orc_rng *r);
uint64_t orc_rng_below(orc_rng *r, uint64_t n);
double orc_rng_normal(orc_rng *r);
/* same contract as ref_rng_draw */
int orc_rng_draw(uint64_t seed, uint64_t tag, int use_stream, int kind, uint64_t arg,
                 int64_t count, void *out);

/* transform.cpp:47-169 */
int orc_generate_orthogonal(int32_t dim, uint64_t seed, double *out);
int orc_apply_dataset(const double *P, int32_t dim, const float *X, int32_t n, float *Y);
int orc_apply_prefix(const double *P, int32_t dim, const float *x, int32_t d, float *y);
int orc_apply_transpose(const double *P, int32_t dim, const float *x, float *y);

/* dco.cpp:54-110, dco.hpp:86-177 */
int orc_threshold_multiplier(int32_t d, double eps0, double *out);
int orc_ad_context(double eps0, int32_t delta_d, int32_t dim, double *factor);
double orc_l2_sq(const float *a, const float *b, int32_t d);
int orc_scan_kernel(int kind, const float *data, const float *query, int32_t dim,
                    int32_t d_start, double s_start, double r, double eps0, int32_t delta_d,
                    int test_at_start, int *positive, double *dist_sq, double *observed,
                    int *dims);
int orc_dco(int kind, const float *o, int32_t n_o, const float *q, int32_t n_q, double r,
            double eps0, int32_t delta_d, int *positive, double *distance, double *observed,
            int *dims);
int orc_ad_scan_pairs(const float *X, const float *Q, int32_t dim, int64_t npairs,
                      const int64_t *rows, const int32_t *qidx, const double *r, double eps0,
                      int32_t delta_d, int pd_mode, uint8_t *positive, int32_t *dims,
                      double *dist_sq, double *observed);

/* ivf.cpp:36-190 */
int orc_kmeans(const float *X, int32_t n, int32_t d, int32_t k, int max_iters, uint64_t seed,
               float *centroids, int32_t *assignment, double *objective, int *iterations);
/* nearest centroid per row (ivf.cpp:36-60 assignment; lowest id on ties) */
int orc_assign(const float *X, int32_t n, int32_t d, const float *C, int32_t k, int32_t *assignment);
/* init 0: k-means++ (the reference, ivf.cpp:62-117); 1: the engine's seeded-sample
 * init (ads_kmeans init 1; config 3/5 builds), followed by the same Lloyd loop. */
int orc_kmeans_init(const float *X, int32_t n, int32_t d, int32_t k, int max_iters, uint64_t seed,
                    int init, float *centroids, int32_t *assignment, double *objective,
                    int *iterations);

/* bench.cpp:31-61 */
int orc_brute_force_knn(const float *base, int32_t n, int32_t d, const float *queries,
                        int32_t nq, int32_t K, int32_t *ids);

/* ivf.cpp:192-258 layout part: buckets in ascending id order, bucket-major
 * copies and the A1/A2 split.  Outputs: list_off[k+1], ids_flat[n],
 * vec_t/vec_raw[n*d], a1_*[n*d1], a2_*[n*(d-d1)] (split only; may be NULL),
 * centroids_raw[k*d] = P^T centroids_t. */
int orc_ivf_layout(int32_t n, int32_t d, int32_t k, int32_t d1, int split, const double *P,
                   const float *centroids_t, const int32_t *assignment, const float *raw,
                   const float *t, int64_t *list_off, int32_t *ids_flat, float *vec_t,
                   float *vec_raw, float *a1_t, float *a2_t, float *a1_raw, float *a2_raw,
                   float *centroids_raw);

typedef struct {
    int32_t n, d, k_clusters, d1, split;
    const float *centroids_t, *centroids_raw;
    const int64_t *list_off; /* k+1 */
    const int32_t *ids_flat;
    const float *vec_t, *vec_raw;           /* contiguous modes */
    const float *a1_t, *a2_t, *a1_raw, *a2_raw; /* split modes */
} orc_ivf;

/* ivf.cpp:296-419.  mode: 0 kFd, 1 kPd, 2 kAd, 3 kAdSplit, 4 kPdSplit.
 * Threshold schedule: the running K-th distance r is re-read before
 * candidate i when i is a refresh point; i = 0 always is, then i = first,
 * first+step, ...  Positives found between refresh points are offered to
 * the bounded heap (in candidate order) at the next refresh point.
 * first = step = 1 is exactly the reference (r re-read before every
 * candidate); larger values model the GPU's batched threshold refresh.
 * stats[0..2] = dims_evaluated, dco_count, candidates. */
int orc_ivf_query(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                  int32_t nprobe, int mode, double eps0, int32_t delta_d, int64_t first,
                  int64_t step, int32_t *ids, double *dists, int32_t *count, uint64_t *stats);

/* Same, with the threshold refreshed at probe-rank wave boundaries: before the
 * first candidate of probe rank wave_ranks[j] (ascending, wave_ranks[0] = 0)
 * — the GPU's list-major wave schedule. */
int orc_ivf_query_waves(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                        int32_t nprobe, int mode, double eps0, int32_t delta_d,
                        const int32_t *wave_ranks, int32_t nwaves, int32_t *ids, double *dists,
                        int32_t *count, uint64_t *stats);

/* probe_order, ivf.cpp:283-292 */
/* ivf_query restricted to probe ranks [probe_lo, n_probe) with the radius
 * starting at r0 (+inf: the plain query); the sharded search's second wave. */
int orc_ivf_query_ext(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                      int32_t nprobe, int mode, double eps0, int32_t delta_d, int64_t first,
                      int64_t step, int32_t probe_lo, double r0, int32_t *ids, double *dists,
                      int32_t *count, uint64_t *stats);
/* lag 1: a chunk's positives are offered one refresh later (chunk j sees the
 * heap after chunks 0 .. j-2); lag 0 = orc_ivf_query. */
int orc_ivf_query_lag(const orc_ivf *idx, const float *q_t, const float *q_raw, int32_t K,
                      int32_t nprobe, int mode, double eps0, int32_t delta_d, int64_t first,
                      int64_t step, int32_t lag, int32_t *ids, double *dists, int32_t *count,
                      uint64_t *stats);
int orc_probe_order(const float *centroids, int32_t L, int32_t d, const float *q,
                    int32_t nprobe, int32_t *order);


/* bench.cpp:303-392 fixed-threshold study (delta_d = 1, r_sq = exact K-th
 * nearest squared distance); per ascending grid entry: summed dims and
 * failures; positives counts objects with d2 <= r_sq over all queries. */
int orc_verify_theory(const float *X, int32_t n, int32_t d, const float *Q, int32_t nq, int32_t K,
                      const double *grid, int32_t G, double *eps_sorted, uint64_t *dims,
                      uint64_t *failures, uint64_t *positives);

/* The benchmark configs' seeded Gaussian-mixture generator (restated from the
 * engine's ads_synth_rows; same field meaning as ads_synth_desc): rows
 * row_lo + i*stride, i < count, on `threads` host threads. */
typedef struct {
    int64_t n;
    int32_t d, components;
    uint64_t seed, role;
    int32_t kind;
    double center_scale, center_lo, center_hi, sigma;
    int32_t decay, assign_mode, threads;
} orc_synth_desc;
int orc_synth_rows(const orc_synth_desc *s, int64_t row_lo, int64_t count, int64_t stride,
                   int32_t threads, float *out);

#ifdef __cplusplus
}
#endif
#endif
