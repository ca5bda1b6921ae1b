// adsann facade — the benchmark sweeps (reference: bench.hpp:50-83, bench.cpp:97-301).
//
// sweep_ivf keeps the reference's protocol (per nprobe, the full-scan run pins
// the 100 % dimension count; accuracy columns from the first repetition; QPS
// the median over `reps`; query rotation inside the timed region) but runs
// each repetition as ONE batched search of the whole query set on the B200
// (ads_apply_dataset + ads_ivf_search, the reference's per-candidate threshold
// refresh, so the accuracy columns equal the reference's).  sweep_hnsw runs
// hnsw_query per query (DCOs on the B200, facade_hnsw.cpp).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <vector>

#include "adsann/bench.hpp"
#include "adsann/transform.hpp"
#include "adsann_b200.h"
#include "detail.hpp"

namespace adsann {

namespace {

// Exact distances of the ground-truth ids in the raw space (bench.cpp:97-107).
std::vector<double> truth_distances(const Dataset& base, const Dataset& queries, const GroundTruth& gt,
                                    std::int32_t K) {
    std::vector<double> out(static_cast<std::size_t>(gt.n_queries) * K);
    for (std::int32_t q = 0; q < gt.n_queries; ++q)
        for (std::int32_t j = 0; j < K; ++j) {
            const float* a = base.row(gt.row(q)[j]);
            const float* b = queries.row(q);
            double s = 0.0;
            for (std::int32_t c = 0; c < base.d; ++c) {
                const double t = static_cast<double>(a[c]) - static_cast<double>(b[c]);
                s += t * t;
            }
            out[static_cast<std::size_t>(q) * K + j] = std::sqrt(s);
        }
    return out;
}

struct Observed {
    double recall = 0.0, avg_ratio = 0.0, avg_dims = 0.0, qps = 0.0;
    std::int32_t flagged = 0;
};

double median_of(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const std::size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

// Accuracy columns of one pass (bench.cpp:150-171) from per-query results.
void score(Observed& o, const std::vector<KnnResult>& res, const GroundTruth& gt, const std::vector<double>& gtd,
           std::int32_t K) {
    double rs = 0.0, ratio = 0.0;
    std::int32_t ratio_n = 0, flagged = 0;
    std::uint64_t dims = 0;
    for (std::size_t q = 0; q < res.size(); ++q) {
        const KnnResult& r = res[q];
        dims += r.stats.dims_evaluated;
        rs += recall(r.ids, std::span<const std::int32_t>(gt.row(static_cast<std::int32_t>(q)), gt.k_max), K);
        if (static_cast<std::int32_t>(r.dists.size()) >= K) {
            const auto a = avg_distance_ratio(r.dists, std::span<const double>(gtd.data() + q * K, K), K);
            if (a) {
                ratio += *a;
                ++ratio_n;
            } else {
                ++flagged;
            }
        } else {
            ++flagged;
        }
    }
    const double nq = static_cast<double>(res.size());
    o.recall = rs / nq;
    o.avg_ratio = ratio_n > 0 ? ratio / ratio_n : 0.0;
    o.avg_dims = static_cast<double>(dims) / nq;
    o.flagged = flagged;
}

template <typename Pass>
Observed timed(int reps, const GroundTruth& gt, const std::vector<double>& gtd, std::int32_t K, const Pass& pass) {
    Observed o;
    std::vector<double> qps;
    for (int rep = 0; rep < std::max(reps, 1); ++rep) {
        std::vector<KnnResult> res;
        const auto t0 = std::chrono::steady_clock::now();
        pass(res);
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        qps.push_back(static_cast<double>(res.size()) / secs);
        if (rep == 0) score(o, res, gt, gtd, K);
    }
    o.qps = median_of(std::move(qps));
    return o;
}

BenchRecord record(const char* algo, std::int32_t param, const Observed& o, const Observed& full) {
    BenchRecord r;
    r.algo = algo;
    r.param = param;
    r.qps = o.qps;
    r.recall = o.recall;
    r.avg_ratio = o.avg_ratio;
    r.avg_dims = o.avg_dims;
    r.dims_pct = full.avg_dims > 0 ? 100.0 * o.avg_dims / full.avg_dims : 0.0;
    r.flagged_queries = o.flagged;
    return r;
}

}  // namespace

const char* ivf_algo_label(IvfMode mode) {
    switch (mode) {
        case IvfMode::kFd: return "IVF";
        case IvfMode::kPd: return "IVF*";
        case IvfMode::kPdSplit: return "IVF**";
        case IvfMode::kAd: return "IVF+";
        case IvfMode::kAdSplit: return "IVF++";
    }
    return "?";
}

const char* hnsw_algo_label(HnswMode mode) {
    switch (mode) {
        case HnswMode::kPlain: return "HNSW";
        case HnswMode::kPd: return "HNSW*";
        case HnswMode::kPlus: return "HNSW+";
        case HnswMode::kPlusPlus: return "HNSW++";
    }
    return "?";
}

std::vector<BenchRecord> sweep_ivf(const IvfIndex& idx, const TransformMatrix& m, const Dataset& base_raw,
                                   const Dataset& queries_raw, const GroundTruth& gt,
                                   const std::vector<IvfMode>& modes, const std::vector<std::int32_t>& nprobe_grid,
                                   const SweepOptions& opt) {
    if (gt.k_max < opt.K) throw std::invalid_argument("sweep_ivf: ground truth too short");
    const std::vector<double> gtd = truth_distances(base_raw, queries_raw, gt, opt.K);
    ads_ivf* h = detail::ivf_handle(idx);
    ads_transform* tr = detail::transform_handle(m);
    const std::int32_t nq = queries_raw.n, K = opt.K, Kc = std::max(K, 1);
    std::vector<float> qt(queries_raw.data.size());
    std::vector<std::int32_t> ids(static_cast<std::size_t>(nq) * Kc), cnt(nq);
    std::vector<double> dists(ids.size());
    std::vector<std::uint64_t> dims(nq), cand(nq);
    ads_search_opts so;
    ads_search_opts_default(&so);
    so.first = 1;  // the reference's per-candidate threshold refresh (ivf.cpp:331, 391)
    so.step = 1;

    std::vector<BenchRecord> out;
    for (const std::int32_t np : nprobe_grid) {
        auto run = [&](IvfMode mode, int reps) {
            const bool transformed = mode == IvfMode::kAd || mode == IvfMode::kAdSplit;
            return timed(reps, gt, gtd, K, [&](std::vector<KnnResult>& res) {
                if (transformed)  // run_timed rotates every query inside the timed loop
                    detail::check_rc(ads_apply_dataset(tr, queries_raw.data.data(), nq, qt.data()));
                detail::check_rc(ads_ivf_search(h, transformed ? qt.data() : nullptr, queries_raw.data.data(), nq, K,
                                                np, static_cast<std::int32_t>(mode), opt.cfg.epsilon0,
                                                opt.cfg.delta_d, &so, ids.data(), dists.data(), cnt.data(),
                                                dims.data(), cand.data()));
                res.resize(static_cast<std::size_t>(nq));
                for (std::int32_t q = 0; q < nq; ++q) {
                    KnnResult& r = res[q];
                    r.ids.assign(ids.begin() + static_cast<std::ptrdiff_t>(q) * Kc,
                                 ids.begin() + static_cast<std::ptrdiff_t>(q) * Kc + cnt[q]);
                    r.dists.assign(dists.begin() + static_cast<std::ptrdiff_t>(q) * Kc,
                                   dists.begin() + static_cast<std::ptrdiff_t>(q) * Kc + cnt[q]);
                    r.stats.dims_evaluated = dims[q];
                    r.stats.dco_count = r.stats.candidates = cand[q];
                }
            });
        };
        const bool fd_requested = std::find(modes.begin(), modes.end(), IvfMode::kFd) != modes.end();
        const Observed full = run(IvfMode::kFd, fd_requested ? opt.reps : 1);
        for (const IvfMode mode : modes)
            out.push_back(record(ivf_algo_label(mode), np, mode == IvfMode::kFd ? full : run(mode, opt.reps), full));
    }
    return out;
}

std::vector<BenchRecord> sweep_hnsw(const HnswGraph& g, const TransformMatrix& m, const Dataset& base_raw,
                                    const Dataset& queries_raw, const GroundTruth& gt,
                                    const std::vector<HnswMode>& modes, const std::vector<std::int32_t>& nef_grid,
                                    const SweepOptions& opt) {
    if (gt.k_max < opt.K) throw std::invalid_argument("sweep_hnsw: ground truth too short");
    const std::vector<double> gtd = truth_distances(base_raw, queries_raw, gt, opt.K);
    std::vector<BenchRecord> out;
    for (const std::int32_t nef : nef_grid) {
        auto run = [&](HnswMode mode, int reps) {
            const bool transformed = mode == HnswMode::kPlus || mode == HnswMode::kPlusPlus;
            return timed(reps, gt, gtd, opt.K, [&](std::vector<KnnResult>& res) {
                res.clear();
                for (std::int32_t q = 0; q < queries_raw.n; ++q) {
                    const float* qr = queries_raw.row(q);
                    if (transformed) {
                        const std::vector<float> qt = apply(m, std::span<const float>(qr, queries_raw.d));
                        res.push_back(hnsw_query(g, qt.data(), qr, opt.K, nef, mode, opt.cfg));
                    } else {
                        res.push_back(hnsw_query(g, nullptr, qr, opt.K, nef, mode, opt.cfg));
                    }
                }
            });
        };
        const bool plain_requested = std::find(modes.begin(), modes.end(), HnswMode::kPlain) != modes.end();
        const Observed full = run(HnswMode::kPlain, plain_requested ? opt.reps : 1);
        for (const HnswMode mode : modes)
            out.push_back(
                record(hnsw_algo_label(mode), nef, mode == HnswMode::kPlain ? full : run(mode, opt.reps), full));
    }
    return out;
}

void write_bench_csv(const std::vector<BenchRecord>& records, const std::filesystem::path& path) {
    std::ofstream f(path, std::ios::trunc);
    if (!f) throw std::runtime_error("cannot open " + path.string() + " for writing");
    f << "algo,param,qps,recall,avg_ratio,avg_dims,dims_pct\n";
    for (const BenchRecord& r : records) {
        char line[256];
        std::snprintf(line, sizeof(line), "%s,%d,%.2f,%.6f,%.6f,%.2f,%.2f\n", r.algo.c_str(), r.param, r.qps,
                      r.recall, r.avg_ratio, r.avg_dims, r.dims_pct);
        f << line;
    }
}

}  // namespace adsann
