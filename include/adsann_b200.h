/* include/adsann_b200.h — the C-ABI drop-in boundary of the B200 IVF++ ADSampling engine.
 *
 * The reference (arXiv 2303.09855, /root/reference/proj) exposes a C++ header
 * API in namespace adsann and no FFI.  Each entry point below replaces one
 * reference function or type for the IVF/IVF++ ADSampling path; the
 * replaced interface is cited as file:line (relative to
 * /root/reference/proj).  Plain pointers and sizes only: no torch, no C++
 * types.  Every call returns an ads_status; ads_last_error() gives the
 * message of the last failure on the calling thread.
 *
 * Arithmetic contract: every distance, partial sum and threshold is computed
 * on the GPU in IEEE fp64 with the reference's operation order (diff =
 * (double)a - (double)b; s = s + diff*diff, index order, no FMA), so DCO
 * decisions, dims, distances and probe orders are bit-identical to the
 * reference on the same fp32 inputs.
 *
 * Host pointers vs device pointers: functions ending in _device take device
 * pointers and enqueue on the context's stream without synchronising; all
 * others take host pointers and return when the results are on the host.
 */
#ifndef ADSANN_B200_H
#define ADSANN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ADS_OK = 0,
    ADS_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    ADS_RUNTIME_ERROR = 2,    /* std::runtime_error in the reference */
    ADS_CUDA_ERROR = 3        /* CUDA failure (mapped to std::runtime_error by facades) */
} ads_status;

/* IvfMode, ivf.hpp:43-49 (same numbering). */
typedef enum {
    ADS_MODE_FD = 0,       /* IVF   : full scan of raw vectors */
    ADS_MODE_PD = 1,       /* IVF*  : partial scan of raw vectors */
    ADS_MODE_AD = 2,       /* IVF+  : ADSampling on transformed vectors */
    ADS_MODE_AD_SPLIT = 3, /* IVF++ : ADSampling, A1/A2 two-array layout */
    ADS_MODE_PD_SPLIT = 4  /* IVF** : partial scan, two-array layout */
} ads_mode;

/* DCO kinds for the batched fixed-threshold entry points (dco.hpp:69-71). */
typedef enum { ADS_DCO_FD = 0, ADS_DCO_PD = 1, ADS_DCO_AD = 2 } ads_dco_kind;

const char *ads_last_error(void);
int ads_version(void);
/* Number of visible CUDA devices (0 when none). */
int ads_device_count(int32_t *count);

/* ------------------------------------------------------------------ host-side pieces
 * Rng (rng.hpp:36-97): counter-based SplitMix64 + Box-Muller.  kind 0 next_u64,
 * 1 uniform(), 2 normal(), 3 below(arg).  out holds count uint64 or double. */
int ads_rng_draw(uint64_t seed, uint64_t tag, int32_t use_stream, int32_t kind, uint64_t arg,
                 int64_t count, void *out);
/* generate_orthogonal, transform.hpp:45 / transform.cpp:47-97 (host, fp64). */
int ads_generate_orthogonal(int32_t dim, uint64_t seed, double *P_out);
/* threshold_multiplier, dco.hpp:67 / dco.cpp:63-68. */
int ads_threshold_multiplier(int32_t d, double epsilon0, double *out);
/* AdContext::factor, dco.hpp:101-108 / dco.cpp:54-61 (dim entries, [0] = 0). */
int ads_ad_context(double epsilon0, int32_t delta_d, int32_t dim, double *factor_out);
/* Seeded Gaussian-mixture generator used by the benchmark configs (host, multi-threaded,
 * deterministic in (seed) regardless of thread count).  See DESIGN.md §Data. */
typedef struct {
    int64_t n;          /* rows to generate */
    int32_t d;          /* dimension */
    int32_t components; /* mixture size */
    uint64_t seed;
    uint64_t role;      /* distinct per role (base / queries) */
    int32_t kind;       /* 0 gmm-normal, 1 gmm-uint8 (round+clip 0..255), 2 gmm-unit-box (clip 0..1),
                           3 gmm-unit-sphere (normalised) */
    double center_scale, center_lo, center_hi; /* kind 0/3: N(0,scale^2); 1/2: U(lo,hi) */
    double sigma;       /* within-component sigma (dimension 0 for decaying kinds) */
    int32_t decay;      /* 1: sigma_j = sigma / sqrt(1 + j/32) */
    int32_t assign_mode;/* 0: component = below(components) per row; 1: component-major blocks */
    int32_t threads;    /* 0 = hardware concurrency */
} ads_synth_desc;
int ads_synth(const ads_synth_desc *desc, float *out, int32_t *component_out /* nullable */);
/* Rows row_lo + i*stride (i < count) of the same n-row mixture, bit-identical to
 * those rows of ads_synth's output (row r depends only on (desc, r)): chunked
 * generation of config 5 and its strided k-means sample. */
int ads_synth_rows(const ads_synth_desc *desc, int64_t row_lo, int64_t count, int64_t stride, float *out,
                   int32_t *component_out /* nullable */);

/* ------------------------------------------------------------------ device context */
typedef struct ads_ctx ads_ctx;
int ads_ctx_create(int32_t device, ads_ctx **out);
int ads_ctx_destroy(ads_ctx *ctx);
int ads_ctx_sync(ads_ctx *ctx);
/* The context's cudaStream_t (as void*), so a host can enqueue collectives on it. */
int ads_ctx_stream(ads_ctx *ctx, void **stream);
/* Device memory helpers (so hosts without torch can stage resident inputs). */
int ads_dev_alloc(ads_ctx *ctx, int64_t bytes, void **dptr);
int ads_dev_free(ads_ctx *ctx, void *dptr);
int ads_memcpy_h2d(ads_ctx *ctx, void *dst, const void *src, int64_t bytes);
int ads_memcpy_d2h(ads_ctx *ctx, void *dst, const void *src, int64_t bytes);
int ads_memset_device(ads_ctx *ctx, void *dst, int32_t value, int64_t bytes);
/* Pinned host memory (for the end-to-end path). */
int ads_host_alloc_pinned(int64_t bytes, void **hptr);
int ads_host_free_pinned(void *hptr);
/* Stream-ordered timing with CUDA events on the context's stream. */
int ads_timer_start(ads_ctx *ctx);
int ads_timer_stop(ads_ctx *ctx, float *ms);
/* Device-side L2 flush (writes a buffer larger than L2 on the context stream). */
int ads_flush_l2(ads_ctx *ctx);

/* ------------------------------------------------------------------ transform
 * y = P x in fp64, stored fp32: apply / apply_prefix / apply_dataset,
 * transform.hpp:48-58 / transform.cpp:99-149; apply_transpose transform.cpp:119-129. */
typedef struct ads_transform ads_transform;
int ads_transform_create(ads_ctx *ctx, const double *P_host, int32_t dim, ads_transform **out);
int ads_transform_destroy(ads_transform *t);
int ads_apply_dataset(ads_transform *t, const float *X, int64_t n, float *Y);
int ads_apply_dataset_device(ads_transform *t, const float *dX, int64_t n, float *dY);
int ads_apply_transpose(ads_transform *t, const float *X, int64_t n, float *Y);
/* The same rotation on the tensor cores (tcgen05 kind::tf32, 3xTF32 split:
 * X P^T ~= Xh Ph^T + Xh Pl^T + Xl Ph^T, fp32 accumulation): not bit-identical
 * to apply_dataset's fp64 result (|error| ~1e-7 |x| typical, measured by the
 * parity tests); dim must be a multiple of 4 and >= 32.  The engine's own search and
 * build paths keep the exact fp64 transform. */
int ads_apply_dataset_tc(ads_transform *t, const float *X, int64_t n, float *Y);
int ads_apply_dataset_tc_device(ads_transform *t, const float *dX, int64_t n, float *dY);
int ads_apply_transpose_device(ads_transform *t, const float *dX, int64_t n, float *dY);

/* ------------------------------------------------------------------ fixed-threshold DCOs
 * One ad_scan / pd_scan_kernel / l2_sq comparison per (query, candidate row),
 * dco.hpp:86-177, with a caller-supplied threshold r per query (the
 * fixed-threshold study, bench.cpp:303-392, and the config-4 microbench).
 * Candidates of query q: rows cand_rows[cand_off[q] .. cand_off[q+1]) when
 * cand_rows != NULL, else the window win_start[q] .. + win_len (mod n_rows).
 * Outputs are indexed by the DCO's global index (cand_off[q] + j, or q*win_len + j);
 * any output pointer may be NULL.  dist_sq holds S_D for positives (NaN else),
 * observed is the reference's estimate at termination. */
typedef struct {
    const float *X;       /* n_rows x dim rows (device for _device, host otherwise) */
    int64_t n_rows;
    int32_t dim;
    const float *Q;       /* nq x dim */
    int32_t nq;
    const int64_t *cand_off;  /* nq+1 */
    const int64_t *cand_rows;
    const int64_t *win_start; /* nq */
    int64_t win_len;
    const double *r;      /* nq thresholds (distances, not squared); may be +inf */
    int32_t kind;         /* ads_dco_kind */
    double epsilon0;
    int32_t delta_d;
    uint8_t *positive;
    int32_t *dims;
    double *dist_sq;
    double *observed;
    uint64_t *dims_per_query; /* nq sums of dims (the roofline byte counter) */
} ads_dco_batch;
int ads_dco_fixed(ads_ctx *ctx, const ads_dco_batch *b);
/* Device pointers; enqueued on the context's stream (window mode returns before the
 * kernel ends: ads_ctx_sync or a stream-ordered read follows). */
int ads_dco_fixed_device(ads_ctx *ctx, const ads_dco_batch *b);
/* The partial squared distances every DCO kind tests, for a batch of rows against one
 * query: dout[c * nb + t] = S_{min((t+1) delta_d, dim)} of row dcand[c] (nb =
 * ceil(dim / delta_d)), fp64 in the reference's order (dco.hpp:122-177).  A caller whose
 * threshold changes between comparisons (the HNSW beam search, hnsw.cpp:214-243, where
 * r moves after every neighbour) replays ad_scan / pd_scan_kernel / l2_sq decisions
 * from them exactly.  Device pointers, enqueued on the context's stream. */
int ads_dco_prefix_sums_device(ads_ctx *ctx, const float *dX, int64_t n_rows, int32_t dim, const float *dq,
                               const int64_t *dcand, int32_t nc, int32_t delta_d, double *dout);
/* Validated single DCO: fd_scan / pd_scan / ad_sampling, dco.hpp:69-71, dco.cpp:70-110.
 * distance is NaN when the outcome is negative (std::optional empty). */
int ads_dco(ads_ctx *ctx, int32_t kind, const float *o, int32_t n_o, const float *q, int32_t n_q,
            double r, double epsilon0, int32_t delta_d, int32_t *positive, double *distance,
            double *observed, int32_t *dims_used);

/* ------------------------------------------------------------------ verify_theory
 * The fixed-threshold study of bench.cpp:303-392 (bench.hpp:90-99): for every
 * query, r_sq = the exact K-th smallest squared distance over all n rows;
 * every (query, row) pair gets a delta_d = 1 adaptive comparison per grid
 * epsilon0.  Rows come back sorted by epsilon0 (ascending):
 * failure_rate = failures / positives, avg_dims = dims / (nq * n).  Any
 * output pointer may be NULL.  Xt / Qt are transformed host arrays. */
int ads_verify_theory(ads_ctx *ctx, const float *Xt, int64_t n, int32_t d, const float *Qt,
                      int32_t nq, int32_t K, const double *grid, int32_t G, double *eps_sorted,
                      double *failure_rate, double *avg_dims, uint64_t *failures,
                      uint64_t *positives);

/* ------------------------------------------------------------------ exact k-NN
 * brute_force_knn, bench.hpp:34 / bench.cpp:31-61: the K smallest (d2, id) pairs. */
int ads_brute_force_knn(ads_ctx *ctx, const float *base, int64_t n, int32_t d,
                        const float *queries, int32_t nq, int32_t K, int32_t *ids);
int ads_brute_force_knn_device(ads_ctx *ctx, const float *dbase, int64_t n, int32_t d,
                               const float *dqueries, int32_t nq, int32_t K, int32_t *dids);

/* ------------------------------------------------------------------ k-means (ivf.hpp:39, ivf.cpp:36-190)
 * init 0 = k-means++ exactly as the reference (sequential fp64 CDF walk),
 * 1 = k distinct seeded samples (for configs whose k-means++ is too long). */
int ads_kmeans(ads_ctx *ctx, const float *X, int64_t n, int32_t d, int32_t k, int32_t max_iters,
               uint64_t seed, int32_t init, float *centroids, int32_t *assignment,
               double *objective, int32_t *iterations);

/* ------------------------------------------------------------------ IVF index (ivf.hpp:55-74)
 * The device index always stores the A1/A2 split arrays (bucket-major) for the
 * transformed space and, when raw vectors are supplied, for the raw space; the
 * reference's contiguous arrays are the same bytes re-blocked, so every IvfMode
 * is served from them with the reference's arithmetic order. */
typedef struct {
    int32_t n, d, k_clusters, d1;
    int32_t layout;               /* 0 kContiguous, 1 kSplit (ivf.hpp:41) */
    uint64_t seed;
    const float *centroids_t;     /* k x d */
    const float *centroids_raw;   /* k x d, nullable (raw modes unavailable) */
    const int64_t *list_off;      /* k+1 bucket offsets into the flat arrays */
    const int32_t *ids_flat;      /* n, ascending ids per bucket */
    const float *vec_t;           /* n x d bucket-major (used when a1_t is NULL) */
    const float *vec_raw;         /* n x d, nullable */
    const float *a1_t, *a2_t;     /* split arrays, nullable */
    const float *a1_raw, *a2_raw;
    const double *P;              /* d x d transform, nullable (enables on-device query rotation) */
} ads_ivf_desc;
typedef struct ads_ivf ads_ivf;
int ads_ivf_create(ads_ctx *ctx, const ads_ivf_desc *desc, ads_ivf **out);
/* build_ivf, ivf.hpp:76-78 / ivf.cpp:192-258, on the GPU: k-means over the
 * transformed vectors, buckets, centroids_raw = P^T centroids_t, split arrays.
 * raw/t are host arrays (n x d).  max_iters 25 and init 0 reproduce the reference. */
int ads_ivf_build(ads_ctx *ctx, const float *raw, const float *t, int32_t n, int32_t d,
                  const double *P, int32_t k, uint64_t seed, int32_t layout, int32_t d1,
                  int32_t max_iters, int32_t init, ads_ivf **out);
/* build_ivf for data that does not fit the reference's flow (config 5,
 * 1e8 rows): dT is the transformed dataset on the device (n x d); k-means
 * (seeded sample init, max_iters Lloyd iterations) runs on every
 * (n / sample)-th row, then every row goes to its nearest centroid through the
 * certified coarse prefilter at nprobe = 1 (the exact fp64 argmin, lowest id
 * on ties); split layout at d1, transformed space only (AD / AD-split modes). */
int ads_ivf_build_sampled_device(ads_ctx *ctx, const float *dT, int64_t n, int32_t d, const double *P,
                                 int32_t k, uint64_t seed, int32_t d1, int32_t max_iters, int64_t sample,
                                 ads_ivf **out);
/* The same build fed in row chunks, for datasets generated or loaded piecewise and
 * for list-sharded indexes: create; train (k-means with seeded sample
 * init on the given transformed sample rows, device pointer) or set_centroids (host
 * k x d); add_device every transformed row in order (row ids = row_lo ..); then
 * finish, which lays out only the lists with keep[c] != 0 (keep NULL = all; ids stay
 * global, like ads_ivf_subset) and may be called once per shard.  list_sizes gives the
 * k list sizes of the whole dataset (for partitioning lists across GPUs).  Fed with
 * the strided sample and every row, it is ads_ivf_build_sampled_device. */
typedef struct ads_ivf_builder ads_ivf_builder;
int ads_ivf_builder_create(ads_ctx *ctx, int64_t n, int32_t d, const double *P, int32_t k, uint64_t seed,
                           int32_t d1, ads_ivf_builder **out);
int ads_ivf_builder_train_device(ads_ivf_builder *b, const float *dS, int64_t sample, int32_t max_iters);
int ads_ivf_builder_set_centroids(ads_ivf_builder *b, const float *centroids);
int ads_ivf_builder_centroids(ads_ivf_builder *b, float *centroids);
int ads_ivf_builder_add_device(ads_ivf_builder *b, const float *dT, int64_t row_lo, int64_t rows);
int ads_ivf_builder_list_sizes(ads_ivf_builder *b, int64_t *sizes);
/* The staged transformed rows (n x d, by row id; device memory owned by the builder,
 * valid until destroy): e.g. for an exact ground truth before they are released. */
int ads_ivf_builder_rows_device(ads_ivf_builder *b, const float **rows);
int ads_ivf_builder_finish(ads_ivf_builder *b, const uint8_t *keep, ads_ivf **out);
int ads_ivf_builder_destroy(ads_ivf_builder *b);
int ads_ivf_destroy(ads_ivf *idx);
/* save_ivf / load_ivf, ivf.hpp:91-92 / ivf.cpp:423-501: the reference's on-disk
 * format (meta.txt + centroids_*.fvecs, buckets.ivecs (ragged), vec_*.fvecs and, for
 * the split layout, a1_* / a2_*.fvecs), so a directory written by adsann::save_ivf
 * loads here and the reverse.  An index without raw vectors (config 5) is written
 * without the raw files, which the reference's format cannot express (its read_fvecs
 * rejects empty files): such a directory loads into the engine only.  P (nullable) is
 * not part of the format (the reference keeps TransformMatrix apart, save_matrix);
 * pass it to enable on-device query rotation. */
int ads_ivf_save(ads_ivf *idx, const char *dir);
int ads_ivf_load(ads_ctx *ctx, const char *dir, const double *P, ads_ivf **out);
/* meta[0..6] = n, d, k_clusters, d1, layout, seed, has_raw */
int ads_ivf_meta(ads_ivf *idx, int64_t *meta);
/* Copy the index back to the host (any pointer nullable). */
int ads_ivf_export(ads_ivf *idx, float *centroids_t, float *centroids_raw, int64_t *list_off,
                   int32_t *ids_flat, float *a1_t, float *a2_t, float *a1_raw, float *a2_raw);

/* Threshold refresh schedule and launch knobs.  The running K-th distance r is
 * re-read before candidate i of a query's probe-ordered stream when i = 0,
 * first, first+step, ...; first = step = 1 is the reference's per-candidate
 * refresh (ivf.cpp:331, 391), larger values batch it. */
typedef struct {
    int64_t first;         /* default K */
    int64_t step;          /* 0 (default): 64 (D <= 256) or 128 candidates per warp; see ads_ivf_search_plan */
    int32_t warps_per_cta; /* 0 (default): 4 for D <= 256, else 8 */
    int32_t queries_per_cta; /* reserved: the query-major kernel serves one query per CTA */
    int32_t ctas_per_sm;   /* 0 = occupancy maximum */
    int32_t time_stages;   /* 1: record per-stage CUDA-event times (ads_ivf_last_timings) */
    int32_t scheduler;     /* must be 0 (query-major, one CTA per query) */
    int32_t tile;          /* -1: no dense prefix phase (lane walk only); >= 0 (default 64): the
                              IVF++ scan's dense A1 prefix phase where the index holds the
                              interleaved A1 copy (long lists, d1 = 32).  Results do not depend
                              on it. */
    int32_t query_order;   /* order in which the batch's queries are served; results do not
                              depend on it.  2 (default): longest first (descending candidate
                              count), which shortens the tail of the persistent scan grid;
                              1: L2-friendly (by the nearest list's position in a
                              nearest-neighbour chain of centroids); 0: input order */
    int32_t coarse_mode;   /* 0 (default): certified prefilter — approximate distances from a
                              tcgen05 TF32 GEMM (fp32 FMA when D % 4 != 0) with a rigorous error
                              bound — plus exact fp64 rescoring of every centroid that can reach the
                              top-nprobe; 2: the same with the fp32-FMA GEMM; 1: exact fp64
                              distance to every centroid.  All give probe_order's exact (d2, id)
                              order. */
    int32_t rotate_mode;   /* when the queries come untransformed (Q_t == NULL): 2 (default) the
                              3xTF32 tensor-core rotation of ads_apply_dataset_tc for batches of >= 64
                              queries with D % 4 == 0 and D >= 32 (~1e-7 relative of the exact
                              rotation; results then follow those queries), else the exact one;
                              0 the exact fp64 rotation, bit-identical to apply(); 1 always the
                              tensor cores (D % 4 == 0, D >= 32) */
    int32_t probe_lo;      /* scan only the lists at probe ranks probe_lo .. n_probe-1
                              (default 0) */
    const double *r0;      /* nullable: per-query initial radius (a distance); r starts
                              at r0[q] and is min(r0[q], heap threshold) at every refresh.  Host
                              memory for ads_ivf_search, device memory for ads_ivf_search_device.
                              With probe_lo this is the second wave of the sharded search: probe
                              ranks [0, w) first, all-reduce (min) of the K-th distances, then
                              [w, n_probe) from the global bound. */
    int32_t walk;          /* lane walk of the IVF++ scan: 1 exact fp64; 2 certified fp32 walk with an exact
                              fp64 re-walk of every undecided or possibly positive candidate (results
                              identical to the exact walk; 32-float segments); 0 (default)
                              picks 2 when a query streams >= 32 000 candidates on average, else 1 */
    int32_t lag;           /* overlapped chunks (exact walk on 16-byte lines, no dense phase, no untested
                              prefix): lanes that find a chunk's stream exhausted start on the next
                              chunk, and every chunk c >= 2 is tested against the thresholds after
                              chunk c - 2 (chunk 1 against chunk 0's), a deterministic schedule the
                              oracle replays.  1: wherever the plan takes it; -1: never (every chunk
                              sees the thresholds after the one before it); 0 (default): when the engine
                              also picks the schedule (step 0, no probe_lo / r0) and walks are >= 8
                              segments.  ads_ivf_search_plan reports the choice. */
} ads_search_opts;
void ads_search_opts_default(ads_search_opts *o);

/* ivf_query, ivf.hpp:87-89 / ivf.cpp:296-419, batched over nq queries.
 * Q_t: transformed queries (AD modes); when NULL and the index holds P, the
 * queries are rotated on the device from Q_raw (apply, transform.cpp:99).
 * Q_raw: raw queries (FD/PD modes, and rotation input).  Outputs per query:
 * ids/dists (K slots, sorted ascending by (dist, id), padded with -1 / NaN),
 * counts, dims_evaluated (result.hpp:25), candidates (result.hpp:27). */
int ads_ivf_search(ads_ivf *idx, const float *Q_t, const float *Q_raw, int32_t nq, int32_t K,
                   int32_t nprobe, int32_t mode, double epsilon0, int32_t delta_d,
                   const ads_search_opts *opts, int32_t *ids, double *dists, int32_t *counts,
                   uint64_t *dims, uint64_t *candidates);
int ads_ivf_search_device(ads_ivf *idx, const float *dQ_t, const float *dQ_raw, int32_t nq,
                          int32_t K, int32_t nprobe, int32_t mode, double epsilon0,
                          int32_t delta_d, const ads_search_opts *opts, int32_t *dids,
                          double *ddists, int32_t *dcounts, uint64_t *ddims,
                          uint64_t *dcandidates);
/* The scan schedule ads_ivf_search would use for these arguments (no search runs):
 * the threshold refresh schedule (first, step: the oracle replays it), the CTA width,
 * the lane walk (1 exact fp64, 2 certified fp32 + exact re-walk) and whether the dense
 * A1 prefix phase runs, and lag: 1 when the chunks overlap (opts.lag = 1 on a plan that
 * takes it).  Results depend on (first, step, lag) only.  Outputs may be NULL. */
int ads_ivf_search_plan(ads_ivf *idx, int32_t K, int32_t nprobe, int32_t mode, double epsilon0,
                        int32_t delta_d, const ads_search_opts *opts, int64_t *first, int64_t *step,
                        int32_t *warps_per_cta, int32_t *walk, int32_t *dense, int32_t *lag);
/* probe_order, ivf.cpp:283-292, batched: nprobe list ids per query. */
int ads_ivf_probe_order(ads_ivf *idx, const float *Q, int32_t nq, int32_t nprobe,
                        int32_t transformed, int32_t *probes);
/* Stage times (ms) of the last search with opts.time_stages: [rotate, coarse, select, scan]. */
int ads_ivf_last_timings(ads_ivf *idx, float *ms4);

/* Coarse prefilter counters of the index's last search / probe_order call:
 * out[0] queries, out[1] centroids rescored exactly (>= queries * nprobe),
 * out[2] queries that fell back to scoring every centroid exactly. */
int ads_ivf_coarse_stats(ads_ivf *idx, uint64_t *out);

/* ------------------------------------------------------------------ list sharding (multi-GPU)
 * Shard of an index for one GPU: same k_clusters, centroids and P (probe order is
 * global), but only lists with keep[c] != 0 keep their rows; the others become
 * empty.  Searching the shard scans the global probe-ordered candidate stream
 * restricted to the owned lists.  No reference counterpart (the reference is
 * single-process); the merged result is the K smallest (dist, id) pairs. */
int ads_ivf_subset(ads_ivf *src, const uint8_t *keep, ads_ivf **out);
/* Per query, the K smallest (dist, id) pairs (ties by id; NaN / id<0 entries
 * ignored) among G result lists of K: dists/ids are [G][nq][K] (the layout of
 * an all-gather of per-shard outputs). */
int ads_merge_topk(ads_ctx *ctx, const double *dists, const int32_t *ids, int32_t G, int32_t nq,
                   int32_t K, int32_t *out_ids, double *out_dists, int32_t *out_counts);
int ads_merge_topk_device(ads_ctx *ctx, const double *ddists, const int32_t *dids, int32_t G,
                          int32_t nq, int32_t K, int32_t *dout_ids, double *dout_dists,
                          int32_t *dout_counts);

#ifdef __cplusplus
}
#endif
#endif
