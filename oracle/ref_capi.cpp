// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libadsann_ref.so).  It lets the Python tests and the
// bench's `--impl reference` arm drive the reference's own code path
// with plain pointers.  Nothing here re-implements the reference: every
// entry point forwards to the adsann:: function it names.
//
// Status codes: 0 ok, 1 std::invalid_argument, 2 std::runtime_error / other.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "adsann/bench.hpp"
#include "adsann/dco.hpp"
#include "adsann/hnsw.hpp"
#include "adsann/ivf.hpp"
#include "adsann/rng.hpp"
#include "adsann/transform.hpp"
#include "adsann/vecio.hpp"

using namespace adsann;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Dataset make_ds(const float* x, std::int32_t n, std::int32_t d) {
    Dataset ds;
    ds.n = n;
    ds.d = d;
    ds.data.assign(x, x + static_cast<std::size_t>(n) * d);
    return ds;
}

TransformMatrix make_m(const double* P, std::int32_t dim) {
    TransformMatrix m;
    m.dim = dim;
    m.entries.assign(P, P + static_cast<std::size_t>(dim) * dim);
    return m;
}

void fill_outcome(const DcoOutcome& o, int* positive, double* distance, double* observed,
                  int* dims) {
    *positive = o.positive ? 1 : 0;
    *distance = o.distance ? *o.distance : std::nan("");
    *observed = o.observed;
    *dims = o.dims_used;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// kind 0: next_u64 (written as uint64 bits), 1: uniform(), 2: normal(), 3: below(arg)
int ref_rng_draw(std::uint64_t seed, std::uint64_t tag, int use_stream, int kind,
                 std::uint64_t arg, std::int64_t count, void* out) {
    return guard([&] {
        Rng rng = use_stream ? Rng::for_stream(seed, tag) : Rng(seed);
        for (std::int64_t i = 0; i < count; ++i) {
            switch (kind) {
                case 0: static_cast<std::uint64_t*>(out)[i] = rng.next_u64(); break;
                case 1: static_cast<double*>(out)[i] = rng.uniform(); break;
                case 2: static_cast<double*>(out)[i] = rng.normal(); break;
                default: static_cast<std::uint64_t*>(out)[i] = rng.below(arg); break;
            }
        }
    });
}

int ref_generate_orthogonal(std::int32_t dim, std::uint64_t seed, double* out) {
    return guard([&] {
        const TransformMatrix m = generate_orthogonal(dim, seed);
        std::memcpy(out, m.entries.data(), m.entries.size() * sizeof(double));
    });
}

int ref_apply_dataset(const double* P, std::int32_t dim, const float* X, std::int32_t n,
                      float* Y) {
    return guard([&] {
        const Dataset out = apply_dataset(make_m(P, dim), make_ds(X, n, dim));
        std::memcpy(Y, out.data.data(), out.data.size() * sizeof(float));
    });
}

int ref_apply_prefix(const double* P, std::int32_t dim, const float* x, std::int32_t d,
                     float* y) {
    return guard([&] {
        const std::vector<float> v =
            apply_prefix(make_m(P, dim), std::span<const float>(x, dim), d);
        std::memcpy(y, v.data(), v.size() * sizeof(float));
    });
}

int ref_apply_transpose(const double* P, std::int32_t dim, const float* x, float* y) {
    return guard([&] {
        const std::vector<float> v = apply_transpose(make_m(P, dim), std::span<const float>(x, dim));
        std::memcpy(y, v.data(), v.size() * sizeof(float));
    });
}

int ref_threshold_multiplier(std::int32_t d, double eps0, double* out) {
    return guard([&] { *out = threshold_multiplier(d, DcoConfig{eps0, 32}); });
}

int ref_ad_context(double eps0, std::int32_t delta_d, std::int32_t dim, double* factor) {
    return guard([&] {
        const AdContext ctx(DcoConfig{eps0, delta_d}, dim);
        std::memcpy(factor, ctx.factor.data(), ctx.factor.size() * sizeof(double));
    });
}

// Raw inline kernels (dco.hpp:122-177).  kind 0 = ad_scan, 1 = pd_scan_kernel.
int ref_scan_kernel(int kind, const float* data, const float* query, std::int32_t dim,
                    std::int32_t d_start, double s_start, double r, double eps0,
                    std::int32_t delta_d, int test_at_start, int* positive, double* dist_sq,
                    double* observed, int* dims) {
    return guard([&] {
        AdResult res;
        if (kind == 0) {
            const AdContext ctx(DcoConfig{eps0, delta_d}, dim);
            res = ad_scan(data, query, dim, d_start, s_start, r, ctx, test_at_start != 0);
        } else {
            res = pd_scan_kernel(data, query, dim, d_start, s_start, r, delta_d,
                                 test_at_start != 0);
        }
        *positive = res.positive;
        *dist_sq = res.dist_sq;
        *observed = res.observed;
        *dims = res.dims;
    });
}

// Validated single-DCO API (dco.cpp:70-110).  kind 0 fd_scan, 1 pd_scan, 2 ad_sampling.
// n_o / n_q are the two vector lengths (they may differ: validation test).
int ref_dco(int kind, const float* o, std::int32_t n_o, const float* q, std::int32_t n_q,
            double r, double eps0, std::int32_t delta_d, int* positive, double* distance,
            double* observed, int* dims) {
    return guard([&] {
        const DcoQuery dq{std::span<const float>(o, n_o), std::span<const float>(q, n_q), r};
        DcoOutcome out;
        if (kind == 0) out = fd_scan(dq);
        else if (kind == 1) out = pd_scan(dq, delta_d);
        else out = ad_sampling(dq, DcoConfig{eps0, delta_d});
        fill_outcome(out, positive, distance, observed, dims);
    });
}

// Batched ad_scan over explicit (query, row) pairs with one threshold per pair,
// from d_start = 0 without a start test — one DCO as ivf_query's kAd loop runs
// it (ivf.cpp:349).  Used to pin fixed-threshold decisions.
int ref_ad_scan_pairs(const float* X, const float* Q, std::int32_t dim, std::int64_t npairs,
                      const std::int64_t* rows, const std::int32_t* qidx, const double* r,
                      double eps0, std::int32_t delta_d, int pd_mode, std::uint8_t* positive,
                      std::int32_t* dims, double* dist_sq, double* observed) {
    return guard([&] {
        const AdContext ctx(DcoConfig{eps0, delta_d}, dim);
        for (std::int64_t i = 0; i < npairs; ++i) {
            const float* x = X + rows[i] * dim;
            const float* q = Q + static_cast<std::int64_t>(qidx[i]) * dim;
            const AdResult res = pd_mode ? pd_scan_kernel(x, q, dim, 0, 0.0, r[i], delta_d, false)
                                         : ad_scan(x, q, dim, 0, 0.0, r[i], ctx, false);
            positive[i] = res.positive;
            dims[i] = res.dims;
            dist_sq[i] = res.positive ? res.dist_sq : std::nan("");
            observed[i] = res.observed;
        }
    });
}

int ref_kmeans(const float* X, std::int32_t n, std::int32_t d, std::int32_t k, int max_iters,
               std::uint64_t seed, float* centroids, std::int32_t* assignment,
               double* objective, int* iterations) {
    return guard([&] {
        const KmeansResult km = kmeans(make_ds(X, n, d), k, max_iters, seed);
        std::memcpy(centroids, km.centroids.data.data(), km.centroids.data.size() * sizeof(float));
        std::memcpy(assignment, km.assignment.data(), km.assignment.size() * sizeof(std::int32_t));
        *objective = km.objective;
        *iterations = km.iterations;
    });
}

int ref_synth_dataset(std::int32_t n, std::int32_t d, std::int32_t blobs, double spread,
                      std::uint64_t seed, float* out, float* centers_out) {
    return guard([&] {
        Dataset centers;
        const Dataset ds = synth_dataset(n, d, blobs, spread, seed, &centers);
        std::memcpy(out, ds.data.data(), ds.data.size() * sizeof(float));
        if (centers_out)
            std::memcpy(centers_out, centers.data.data(), centers.data.size() * sizeof(float));
    });
}

int ref_brute_force_knn(const float* base, std::int32_t n, std::int32_t d, const float* queries,
                        std::int32_t nq, std::int32_t K, std::int32_t* ids) {
    return guard([&] {
        const GroundTruth gt = brute_force_knn(make_ds(base, n, d), make_ds(queries, nq, d), K);
        std::memcpy(ids, gt.ids.data(), gt.ids.size() * sizeof(std::int32_t));
    });
}

// ---------------------------------------------------------------- IVF index handles

void* ref_ivf_build(const float* raw, const float* t, std::int32_t n, std::int32_t d,
                    const double* P, std::int32_t k, std::uint64_t seed, int layout,
                    std::int32_t d1) {
    IvfIndex* out = nullptr;
    const int rc = guard([&] {
        out = new IvfIndex(build_ivf(make_ds(raw, n, d), make_ds(t, n, d), make_m(P, d), k, seed,
                                     layout ? IvfLayout::kSplit : IvfLayout::kContiguous, d1));
    });
    return rc == 0 ? out : nullptr;
}

// Assemble an IvfIndex from a precomputed clustering (centroids + per-point
// assignment) exactly as build_ivf lays it out after its kmeans call
// (ivf.cpp:211-256): ascending ids per bucket, bucket-major copies, split
// arrays.  This lets the reference search an index built elsewhere (e.g. on
// the GPU for configs whose reference k-means would take hours).
void* ref_ivf_assemble(std::int32_t n, std::int32_t d, std::int32_t k, std::int32_t d1,
                       int layout, std::uint64_t seed, const double* P, const float* centroids_t,
                       const std::int32_t* assignment, const float* raw, const float* t) {
    IvfIndex* idx = nullptr;
    const int rc = guard([&] {
        if (layout && (d1 < 1 || d1 >= d)) throw std::invalid_argument("assemble: bad d1");
        auto* x = new IvfIndex();
        x->n = n;
        x->d = d;
        x->k_clusters = k;
        x->d1 = d1;
        x->layout = layout ? IvfLayout::kSplit : IvfLayout::kContiguous;
        x->seed = seed;
        x->centroids_t = make_ds(centroids_t, k, d);
        x->buckets.assign(k, {});
        for (std::int32_t i = 0; i < n; ++i) x->buckets.at(assignment[i]).push_back(i);
        const TransformMatrix m = make_m(P, d);
        x->centroids_raw.n = k;
        x->centroids_raw.d = d;
        x->centroids_raw.data.resize(static_cast<std::size_t>(k) * d);
        for (std::int32_t c = 0; c < k; ++c) {
            const std::vector<float> back =
                apply_transpose(m, std::span<const float>(x->centroids_t.row(c), d));
            std::copy(back.begin(), back.end(), x->centroids_raw.row(c));
        }
        x->vec_t.resize(static_cast<std::size_t>(n) * d);
        x->vec_raw.resize(static_cast<std::size_t>(n) * d);
        std::size_t pos = 0;
        for (std::int32_t c = 0; c < k; ++c)
            for (const std::int32_t id : x->buckets[c]) {
                x->ids_flat.push_back(id);
                std::memcpy(&x->vec_t[pos * d], t + static_cast<std::size_t>(id) * d, d * 4);
                std::memcpy(&x->vec_raw[pos * d], raw + static_cast<std::size_t>(id) * d, d * 4);
                ++pos;
            }
        if (layout) {
            const std::int32_t d2 = d - d1;
            x->a1_t.resize(static_cast<std::size_t>(n) * d1);
            x->a2_t.resize(static_cast<std::size_t>(n) * d2);
            x->a1_raw.resize(static_cast<std::size_t>(n) * d1);
            x->a2_raw.resize(static_cast<std::size_t>(n) * d2);
            for (std::size_t p = 0; p < static_cast<std::size_t>(n); ++p) {
                std::memcpy(&x->a1_t[p * d1], &x->vec_t[p * d], d1 * 4);
                std::memcpy(&x->a2_t[p * d2], &x->vec_t[p * d + d1], d2 * 4);
                std::memcpy(&x->a1_raw[p * d1], &x->vec_raw[p * d], d1 * 4);
                std::memcpy(&x->a2_raw[p * d2], &x->vec_raw[p * d + d1], d2 * 4);
            }
        }
        idx = x;
    });
    return rc == 0 ? idx : nullptr;
}

// The IVF++ (kAdSplit) subset of that index: ivf_query in kAdSplit reads only
// centroids_t, buckets, ids_flat, a1_t and a2_t (ivf.cpp:296-419), so for
// config 5 (1e8 x 96) only those are built (~39 GB instead of six full copies).
// Other modes must not be run on it.  t holds the transformed rows by id.
void* ref_ivf_assemble_split(std::int32_t n, std::int32_t d, std::int32_t k, std::int32_t d1,
                             std::uint64_t seed, const float* centroids_t,
                             const std::int32_t* assignment, const float* t) {
    IvfIndex* idx = nullptr;
    const int rc = guard([&] {
        if (d1 < 1 || d1 >= d) throw std::invalid_argument("assemble: bad d1");
        auto* x = new IvfIndex();
        x->n = n;
        x->d = d;
        x->k_clusters = k;
        x->d1 = d1;
        x->layout = IvfLayout::kSplit;
        x->seed = seed;
        x->centroids_t = make_ds(centroids_t, k, d);
        x->buckets.assign(k, {});
        for (std::int32_t i = 0; i < n; ++i) x->buckets.at(assignment[i]).push_back(i);
        const std::int32_t d2 = d - d1;
        x->ids_flat.reserve(n);
        x->a1_t.resize(static_cast<std::size_t>(n) * d1);
        x->a2_t.resize(static_cast<std::size_t>(n) * d2);
        std::size_t p = 0;
        for (std::int32_t c = 0; c < k; ++c)
            for (const std::int32_t id : x->buckets[c]) {
                x->ids_flat.push_back(id);
                const float* row = t + static_cast<std::size_t>(id) * d;
                std::memcpy(&x->a1_t[p * d1], row, d1 * 4);
                std::memcpy(&x->a2_t[p * d2], row + d1, d2 * 4);
                ++p;
            }
        idx = x;
    });
    return rc == 0 ? idx : nullptr;
}

// The same from an existing bucket-major split layout (e.g. one exported from the
// GPU engine): list_off (k+1), ids_flat, a1_t (n x d1), a2_t (n x (d-d1)).
void* ref_ivf_from_split_layout(std::int32_t n, std::int32_t d, std::int32_t k, std::int32_t d1,
                                std::uint64_t seed, const float* centroids_t,
                                const std::int64_t* list_off, const std::int32_t* ids_flat,
                                const float* a1_t, const float* a2_t) {
    IvfIndex* idx = nullptr;
    const int rc = guard([&] {
        if (d1 < 1 || d1 >= d) throw std::invalid_argument("assemble: bad d1");
        if (list_off[0] != 0 || list_off[k] != n) throw std::invalid_argument("assemble: bad list_off");
        auto* x = new IvfIndex();
        x->n = n;
        x->d = d;
        x->k_clusters = k;
        x->d1 = d1;
        x->layout = IvfLayout::kSplit;
        x->seed = seed;
        x->centroids_t = make_ds(centroids_t, k, d);
        x->buckets.assign(k, {});
        for (std::int32_t c = 0; c < k; ++c)
            x->buckets[c].assign(ids_flat + list_off[c], ids_flat + list_off[c + 1]);
        x->ids_flat.assign(ids_flat, ids_flat + n);
        x->a1_t.assign(a1_t, a1_t + static_cast<std::size_t>(n) * d1);
        x->a2_t.assign(a2_t, a2_t + static_cast<std::size_t>(n) * (d - d1));
        idx = x;
    });
    return rc == 0 ? idx : nullptr;
}

void ref_ivf_free(void* h) { delete static_cast<IvfIndex*>(h); }

// meta[0..5] = n, d, k_clusters, d1, layout, seed
int ref_ivf_meta(void* h, std::int64_t* meta) {
    return guard([&] {
        const auto* x = static_cast<const IvfIndex*>(h);
        meta[0] = x->n;
        meta[1] = x->d;
        meta[2] = x->k_clusters;
        meta[3] = x->d1;
        meta[4] = x->layout == IvfLayout::kSplit;
        meta[5] = static_cast<std::int64_t>(x->seed);
    });
}

// Any output pointer may be null.  list_sizes has k entries.
int ref_ivf_export(void* h, float* centroids_t, float* centroids_raw, std::int32_t* list_sizes,
                   std::int32_t* ids_flat, float* vec_t, float* vec_raw, float* a1_t, float* a2_t,
                   float* a1_raw, float* a2_raw) {
    return guard([&] {
        const auto* x = static_cast<const IvfIndex*>(h);
        auto cp = [](void* dst, const void* src, std::size_t bytes) {
            if (dst && bytes) std::memcpy(dst, src, bytes);
        };
        cp(centroids_t, x->centroids_t.data.data(), x->centroids_t.data.size() * 4);
        cp(centroids_raw, x->centroids_raw.data.data(), x->centroids_raw.data.size() * 4);
        if (list_sizes)
            for (std::int32_t c = 0; c < x->k_clusters; ++c)
                list_sizes[c] = static_cast<std::int32_t>(x->buckets[c].size());
        cp(ids_flat, x->ids_flat.data(), x->ids_flat.size() * 4);
        cp(vec_t, x->vec_t.data(), x->vec_t.size() * 4);
        cp(vec_raw, x->vec_raw.data(), x->vec_raw.size() * 4);
        cp(a1_t, x->a1_t.data(), x->a1_t.size() * 4);
        cp(a2_t, x->a2_t.data(), x->a2_t.size() * 4);
        cp(a1_raw, x->a1_raw.data(), x->a1_raw.size() * 4);
        cp(a2_raw, x->a2_raw.data(), x->a2_raw.size() * 4);
    });
}

int ref_save_ivf(void* h, const char* dir) {
    return guard([&] { save_ivf(*static_cast<const IvfIndex*>(h), dir); });
}

void* ref_load_ivf(const char* dir) {
    IvfIndex* out = nullptr;
    const int rc = guard([&] { out = new IvfIndex(load_ivf(dir)); });
    return rc == 0 ? out : nullptr;
}

// One ivf_query call (ivf.cpp:296).  stats[0..2] = dims_evaluated, dco_count, candidates.
// ids/dists must hold K entries; *count receives the number of results.
int ref_ivf_query(void* h, const float* q_t, const float* q_raw, std::int32_t K,
                  std::int32_t nprobe, int mode, double eps0, std::int32_t delta_d,
                  std::int32_t* ids, double* dists, std::int32_t* count, std::uint64_t* stats) {
    return guard([&] {
        const KnnResult res = ivf_query(*static_cast<const IvfIndex*>(h), q_t, q_raw, K, nprobe,
                                        static_cast<IvfMode>(mode), DcoConfig{eps0, delta_d});
        *count = static_cast<std::int32_t>(res.ids.size());
        for (std::size_t j = 0; j < res.ids.size(); ++j) {
            ids[j] = res.ids[j];
            dists[j] = res.dists[j];
        }
        stats[0] = res.stats.dims_evaluated;
        stats[1] = res.stats.dco_count;
        stats[2] = res.stats.candidates;
    });
}

// Many queries, optionally on several host threads (disjoint query ranges; the
// index is immutable).  When rotate != 0 the transformed query is
// produced inside the loop with adsann::apply (the run_timed protocol,
// bench.cpp:143-146) from P; otherwise Qt is used as given.  ids/dists are
// nq*K (padded with -1 / NaN), dims per query; *seconds = wall time of the loop.
int ref_ivf_query_batch(void* h, const double* P, int rotate, const float* Qt, const float* Qr,
                        std::int32_t nq, std::int32_t K, std::int32_t nprobe, int mode,
                        double eps0, std::int32_t delta_d, int nthreads, std::int32_t* ids,
                        double* dists, std::uint64_t* dims, double* seconds) {
    return guard([&] {
        const auto* idx = static_cast<const IvfIndex*>(h);
        const std::int32_t d = idx->d;
        TransformMatrix m;
        if (rotate) m = make_m(P, d);
        const IvfMode md = static_cast<IvfMode>(mode);
        const bool transformed = md == IvfMode::kAd || md == IvfMode::kAdSplit;
        std::vector<std::string> errs(std::max(1, nthreads));
        auto work = [&](int t, std::int32_t lo, std::int32_t hi) {
            try {
                for (std::int32_t qi = lo; qi < hi; ++qi) {
                    const float* qr = Qr ? Qr + static_cast<std::size_t>(qi) * d : nullptr;
                    std::vector<float> qt_buf;
                    const float* qt = Qt ? Qt + static_cast<std::size_t>(qi) * d : nullptr;
                    if (rotate && transformed) {
                        qt_buf = adsann::apply(m, std::span<const float>(qr, d));
                        qt = qt_buf.data();
                    }
                    const KnnResult res =
                        ivf_query(*idx, qt, qr, K, nprobe, md, DcoConfig{eps0, delta_d});
                    for (std::int32_t j = 0; j < K; ++j) {
                        const bool ok = j < static_cast<std::int32_t>(res.ids.size());
                        ids[static_cast<std::size_t>(qi) * K + j] = ok ? res.ids[j] : -1;
                        dists[static_cast<std::size_t>(qi) * K + j] = ok ? res.dists[j] : std::nan("");
                    }
                    dims[qi] = res.stats.dims_evaluated;
                }
            } catch (const std::exception& e) {
                errs[t] = e.what();
            }
        };
        const auto t0 = std::chrono::steady_clock::now();
        if (nthreads <= 1) {
            work(0, 0, nq);
        } else {
            // dynamic scheduling: threads take queries from a shared counter in
            // blocks of 4, so uneven per-query costs do not idle the other threads
            std::atomic<std::int32_t> next{0};
            std::vector<std::thread> th;
            for (int t = 0; t < nthreads; ++t)
                th.emplace_back([&, t] {
                    for (;;) {
                        const std::int32_t lo = next.fetch_add(4);
                        if (lo >= nq) break;
                        work(t, lo, std::min<std::int32_t>(nq, lo + 4));
                    }
                });
            for (auto& x : th) x.join();
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (const auto& e : errs)
            if (!e.empty()) throw std::invalid_argument(e);
    });
}

// ---- HNSW (hnsw.hpp:44-105): build / save / load / query, for the facade parity test.
void* ref_hnsw_build(const float* raw, const float* t, std::int32_t n, std::int32_t d, std::int32_t M,
                     std::int32_t ef, std::uint64_t seed) {
    HnswGraph* g = nullptr;
    const int rc = guard([&] { g = new HnswGraph(build_hnsw(make_ds(raw, n, d), make_ds(t, n, d), M, ef, seed)); });
    return rc == 0 ? g : nullptr;
}

void* ref_hnsw_load(const char* dir, const float* raw, const float* t, std::int32_t n, std::int32_t d) {
    HnswGraph* g = nullptr;
    const int rc = guard([&] { g = new HnswGraph(load_hnsw(dir, make_ds(raw, n, d), make_ds(t, n, d))); });
    return rc == 0 ? g : nullptr;
}

int ref_hnsw_save(void* g, const char* dir) {
    return guard([&] { save_hnsw(*static_cast<const HnswGraph*>(g), dir); });
}

void ref_hnsw_free(void* g) { delete static_cast<HnswGraph*>(g); }

// stats[0..3] = dims_evaluated, dco_count, hops, candidates
int ref_hnsw_query(void* g, const float* q_t, const float* q_raw, std::int32_t K, std::int32_t nef, int mode,
                   double eps0, std::int32_t delta_d, std::int32_t* ids, double* dists, std::int32_t* count,
                   std::uint64_t* stats) {
    return guard([&] {
        const KnnResult r = hnsw_query(*static_cast<const HnswGraph*>(g), q_t, q_raw, K, nef,
                                       static_cast<HnswMode>(mode), DcoConfig{eps0, delta_d});
        *count = static_cast<std::int32_t>(r.ids.size());
        for (std::size_t j = 0; j < r.ids.size(); ++j) {
            ids[j] = r.ids[j];
            dists[j] = r.dists[j];
        }
        stats[0] = r.stats.dims_evaluated;
        stats[1] = r.stats.dco_count;
        stats[2] = r.stats.hops;
        stats[3] = r.stats.candidates;
    });
}

int ref_verify_theory(const float* X, std::int32_t n, std::int32_t d, const float* Q,
                      std::int32_t nq, std::int32_t K, const double* grid, std::int32_t G,
                      double* failure_rate, double* avg_dims, std::uint64_t* failures,
                      std::uint64_t* positives) {
    return guard([&] {
        const auto rows = verify_theory(make_ds(X, n, d), make_ds(Q, nq, d), K,
                                        std::vector<double>(grid, grid + G));
        for (std::int32_t g = 0; g < G; ++g) {
            failure_rate[g] = rows[g].failure_rate;
            avg_dims[g] = rows[g].avg_dims;
            failures[g] = rows[g].failures;
            positives[g] = rows[g].positives;
        }
    });
}

}  // extern "C"
