// adsann facade — HNSW+ / HNSW++ with the distance comparisons on the B200.
//
// Graph construction and traversal stay on the host, as in the reference
// (hnsw.cpp:120-212 build, 258-379 query); SURVEY §8(f) row 4 puts the graph
// walk itself out of the GPU's scope.  What moves to the GPU is the DCO: the
// reference's DcoRunner (hnsw.cpp:214-243) evaluates one neighbour at a time
// against a threshold r that can change after every comparison (a positive
// enters the routing / top-K set and shrinks it).  Here every hop sends its
// whole neighbour batch to the GPU in one launch (ads_dco_prefix_sums_device:
// the fp64 partial sums at every Δd boundary and at D, in the reference's
// arithmetic order) and the host replays ad_scan / pd_scan_kernel / l2_sq
// (dco.hpp:86-177) from those sums, neighbour by neighbour, with the
// threshold in force at that moment.  The replay reads the same partial sums
// the reference compares, so decisions, dims, observed distances and results
// are identical to adsann::hnsw_query (tests/test_gpu_hnsw.py).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <fstream>
#include <limits>
#include <mutex>
#include <queue>
#include <stdexcept>
#include <string>
#include <vector>

#include "adsann/hnsw.hpp"
#include "adsann/rng.hpp"
#include "adsann_b200.h"
#include "detail.hpp"

namespace adsann {

namespace {

constexpr double kInfD = std::numeric_limits<double>::infinity();
using Pair = std::pair<double, std::int32_t>;
using PairMax = std::priority_queue<Pair>;
using PairMin = std::priority_queue<Pair, std::vector<Pair>, std::greater<Pair>>;

// fp64 distance in the reference's order (dco.hpp:86-97); construction only.
double exact_dist(const float* a, const float* b, std::int32_t d) {
    double s = 0.0;
    for (std::int32_t j = 0; j < d; ++j) {
        const double t = static_cast<double>(a[j]) - static_cast<double>(b[j]);
        s += t * t;
    }
    return std::sqrt(s);
}

// ------------------------------------------------------------------ construction
class GraphBuilder {
public:
    explicit GraphBuilder(HnswGraph& g) : g_(g), mark_(static_cast<std::size_t>(g.n), 0u) {}

    void add(std::int32_t v) {
        const std::int32_t top = g_.levels[v];
        g_.links[v].assign(static_cast<std::size_t>(top) + 1, {});
        if (g_.entry_point < 0) {  // first vertex
            g_.entry_point = v;
            g_.max_layer = top;
            return;
        }
        const float* x = row(v);
        // greedy descent through the layers above v's own
        std::int32_t at = g_.entry_point;
        double at_d = exact_dist(x, row(at), g_.d);
        for (std::int32_t layer = g_.max_layer; layer > top; --layer) {
            for (bool moved = true; moved;) {
                moved = false;
                const std::vector<std::int32_t>& nbrs = g_.links[at][layer];
                for (std::size_t k = 0; k < nbrs.size(); ++k) {
                    const double dn = exact_dist(x, row(nbrs[k]), g_.d);
                    if (dn < at_d) {
                        at_d = dn;
                        at = nbrs[k];
                        moved = true;
                    }
                }
            }
        }
        // connect on every layer from min(top, max_layer) down to 0
        for (std::int32_t layer = std::min(top, g_.max_layer); layer >= 0; --layer) {
            const std::vector<Pair> near = beam(x, at, g_.ef_construction, layer);
            std::vector<std::int32_t> chosen = diverse(near, g_.M);
            const std::int32_t cap = layer == 0 ? 2 * g_.M : g_.M;
            for (const std::int32_t u : chosen) {
                std::vector<std::int32_t>& back = g_.links[u][layer];
                back.push_back(v);
                if (static_cast<std::int32_t>(back.size()) > cap) shrink(u, layer, cap);
            }
            g_.links[v][layer] = std::move(chosen);
            at = near.front().second;
        }
        if (top > g_.max_layer) {
            g_.max_layer = top;
            g_.entry_point = v;
        }
    }

private:
    const float* row(std::int32_t i) const { return g_.data_t.row(i); }

    // Best-first search of one layer with a result set of size ef; (dist, id) ascending.
    std::vector<Pair> beam(const float* x, std::int32_t start, std::int32_t ef, std::int32_t layer) {
        ++stamp_;
        PairMax best;
        PairMin open;
        const double d0 = exact_dist(x, row(start), g_.d);
        best.emplace(d0, start);
        open.emplace(d0, start);
        mark_[start] = stamp_;
        double worst = d0;
        const std::size_t cap = static_cast<std::size_t>(ef);
        while (!open.empty()) {
            const Pair c = open.top();
            if (c.first > worst && best.size() == cap) break;
            open.pop();
            for (const std::int32_t u : g_.links[c.second][layer]) {
                if (mark_[u] == stamp_) continue;
                mark_[u] = stamp_;
                const double du = exact_dist(x, row(u), g_.d);
                if (best.size() < cap || du < best.top().first) {
                    open.emplace(du, u);
                    best.emplace(du, u);
                    if (best.size() > cap) best.pop();
                    worst = best.top().first;
                }
            }
        }
        std::vector<Pair> out;
        out.reserve(best.size());
        for (; !best.empty(); best.pop()) out.push_back(best.top());
        std::sort(out.begin(), out.end());
        return out;
    }

    // Heuristic neighbour choice: keep a candidate (ascending distance) unless some
    // already-kept neighbour is strictly closer to it than the anchor is.
    std::vector<std::int32_t> diverse(const std::vector<Pair>& cand, std::int32_t limit) const {
        std::vector<std::int32_t> keep;
        for (const Pair& c : cand) {
            if (static_cast<std::int32_t>(keep.size()) >= limit) break;
            const bool dominated = std::any_of(keep.begin(), keep.end(), [&](std::int32_t k) {
                return exact_dist(row(c.second), row(k), g_.d) < c.first;
            });
            if (!dominated) keep.push_back(c.second);
        }
        return keep;
    }

    void shrink(std::int32_t u, std::int32_t layer, std::int32_t cap) {
        std::vector<std::int32_t>& nb = g_.links[u][layer];
        std::vector<Pair> cand(nb.size());
        for (std::size_t k = 0; k < nb.size(); ++k) cand[k] = {exact_dist(row(u), row(nb[k]), g_.d), nb[k]};
        std::sort(cand.begin(), cand.end());
        nb = diverse(cand, cap);
    }

    HnswGraph& g_;
    std::vector<std::uint32_t> mark_;
    std::uint32_t stamp_ = 0;
};

// ------------------------------------------------------------------ query-time DCOs
struct Outcome {
    bool positive;
    double observed;
    std::int32_t dims;
};

}  // namespace

// Device state of a graph: both vector sets uploaded once, plus per-hop staging.
struct DeviceHnsw {
    std::mutex mu;
    float* xt = nullptr;
    float* xr = nullptr;
    float* q = nullptr;
    std::int64_t* cand = nullptr;
    double* sums = nullptr;
    std::int64_t* h_cand = nullptr;  // pinned
    double* h_sums = nullptr;        // pinned
    std::int32_t cap = 0, nb_cap = 0;
    ~DeviceHnsw() {
        ads_ctx* ctx = detail::engine_ctx();
        for (void* p : {static_cast<void*>(xt), static_cast<void*>(xr), static_cast<void*>(q),
                        static_cast<void*>(cand), static_cast<void*>(sums)})
            if (p) ads_dev_free(ctx, p);
        if (h_cand) ads_host_free_pinned(h_cand);
        if (h_sums) ads_host_free_pinned(h_sums);
    }
};

namespace {

// One hop's worth of comparisons for one query.
class HopEvaluator {
public:
    HopEvaluator(const HnswGraph& g, const float* q, HnswMode mode, const DcoConfig& cfg, QueryStats& st)
        : g_(g), mode_(mode), st_(st),
          dd_(mode == HnswMode::kPlain ? g.d : (mode == HnswMode::kPd ? std::min(cfg.delta_d, g.d) : cfg.delta_d)),
          nb_((g.d + dd_ - 1) / dd_) {
        using detail::check_rc;
        ads_ctx* ctx = detail::engine_ctx();
        if (!g.device) g.device = std::make_shared<DeviceHnsw>();
        dev_ = g.device.get();
        lock_ = std::unique_lock<std::mutex>(dev_->mu);
        const bool transformed = mode == HnswMode::kPlus || mode == HnswMode::kPlusPlus;
        float*& X = transformed ? dev_->xt : dev_->xr;
        const Dataset& src = transformed ? g.data_t : g.data_raw;
        if (!X) {
            check_rc(ads_dev_alloc(ctx, static_cast<std::int64_t>(src.data.size() * 4) + 4,
                                   reinterpret_cast<void**>(&X)));
            check_rc(ads_memcpy_h2d(ctx, X, src.data.data(), static_cast<std::int64_t>(src.data.size() * 4)));
        }
        X_ = X;
        if (!dev_->q) check_rc(ads_dev_alloc(ctx, 4 * static_cast<std::int64_t>(g.d), reinterpret_cast<void**>(&dev_->q)));
        check_rc(ads_memcpy_h2d(ctx, dev_->q, q, 4 * static_cast<std::int64_t>(g.d)));
        if (transformed) {  // AdContext(cfg, d) (dco.cpp:54-61), which also validates cfg
            factor_.resize(static_cast<std::size_t>(g.d));
            check_rc(ads_ad_context(cfg.epsilon0, cfg.delta_d, g.d, factor_.data()));
        }
    }

    // GPU partial sums of a batch, then replay decision k with threshold r_of(k).
    void load(const std::vector<std::int32_t>& ids) {
        using detail::check_rc;
        ads_ctx* ctx = detail::engine_ctx();
        const std::int32_t nc = static_cast<std::int32_t>(ids.size());
        if (nc == 0) return;
        grow(nc);
        for (std::int32_t k = 0; k < nc; ++k) dev_->h_cand[k] = ids[k];
        check_rc(ads_memcpy_h2d(ctx, dev_->cand, dev_->h_cand, 8 * static_cast<std::int64_t>(nc)));
        check_rc(ads_dco_prefix_sums_device(ctx, X_, g_.n, g_.d, dev_->q, dev_->cand, nc, dd_, dev_->sums));
        check_rc(ads_memcpy_d2h(ctx, dev_->h_sums, dev_->sums, 8 * static_cast<std::int64_t>(nc) * nb_));
    }

    // dco.hpp:122-177 replayed on the sums of batch entry k.
    Outcome decide(std::int32_t k, double r) {
        const double* S = dev_->h_sums + static_cast<std::size_t>(k) * nb_;
        const std::int32_t D = g_.d;
        const double r_sq = r * r;
        Outcome o{false, 0.0, D};
        if (mode_ == HnswMode::kPlain) {  // l2_sq, then dist <= r
            const double dist = std::sqrt(S[nb_ - 1]);
            o = {dist <= r, dist, D};
        } else {
            std::int32_t t = 0;
            for (; t < nb_ - 1; ++t) {
                const std::int32_t d = (t + 1) * dd_;
                const bool stop = mode_ == HnswMode::kPd ? S[t] > r_sq : S[t] > factor_[d] * r_sq;
                if (stop) {
                    o.observed = mode_ == HnswMode::kPd ? std::sqrt(S[t]) : std::sqrt(S[t] * D / d);
                    o.dims = d;
                    break;
                }
            }
            if (t == nb_ - 1) o = {S[t] <= r_sq, std::sqrt(S[t]), D};
        }
        st_.dims_evaluated += static_cast<std::uint64_t>(o.dims);
        ++st_.dco_count;
        return o;
    }

private:
    void grow(std::int32_t nc) {
        using detail::check_rc;
        ads_ctx* ctx = detail::engine_ctx();
        if (nc <= dev_->cap && nb_ <= dev_->nb_cap) return;
        const std::int32_t cap = std::max({nc, 2 * dev_->cap, 64});
        const std::int32_t nbc = std::max(nb_, dev_->nb_cap);
        if (dev_->cand) ads_dev_free(ctx, dev_->cand);
        if (dev_->sums) ads_dev_free(ctx, dev_->sums);
        if (dev_->h_cand) ads_host_free_pinned(dev_->h_cand);
        if (dev_->h_sums) ads_host_free_pinned(dev_->h_sums);
        check_rc(ads_dev_alloc(ctx, 8 * static_cast<std::int64_t>(cap), reinterpret_cast<void**>(&dev_->cand)));
        check_rc(ads_dev_alloc(ctx, 8 * static_cast<std::int64_t>(cap) * nbc, reinterpret_cast<void**>(&dev_->sums)));
        check_rc(ads_host_alloc_pinned(8 * static_cast<std::int64_t>(cap), reinterpret_cast<void**>(&dev_->h_cand)));
        check_rc(ads_host_alloc_pinned(8 * static_cast<std::int64_t>(cap) * nbc,
                                       reinterpret_cast<void**>(&dev_->h_sums)));
        dev_->cap = cap;
        dev_->nb_cap = nbc;
    }

    const HnswGraph& g_;
    HnswMode mode_;
    QueryStats& st_;
    std::int32_t dd_, nb_;
    DeviceHnsw* dev_ = nullptr;
    std::unique_lock<std::mutex> lock_;
    const float* X_ = nullptr;
    std::vector<double> factor_;
};

std::vector<Pair> ascending(PairMax& h) {
    std::vector<Pair> v;
    v.reserve(h.size());
    for (; !h.empty(); h.pop()) v.push_back(h.top());
    std::sort(v.begin(), v.end());
    return v;
}

}  // namespace

HnswGraph build_hnsw(const Dataset& ds_raw, const Dataset& ds_transformed, std::int32_t M,
                     std::int32_t ef_construction, std::uint64_t seed) {
    // hnsw.cpp:185-190 argument checks
    if (ds_transformed.n < 1) throw std::invalid_argument("build_hnsw: empty dataset");
    if (ds_raw.n != ds_transformed.n || ds_raw.d != ds_transformed.d)
        throw std::invalid_argument("build_hnsw: raw and transformed datasets disagree");
    if (M < 2) throw std::invalid_argument("build_hnsw: M must be >= 2");
    if (ef_construction < M) throw std::invalid_argument("build_hnsw: ef_construction must be >= M");
    HnswGraph g;
    g.n = ds_transformed.n;
    g.d = ds_transformed.d;
    g.M = M;
    g.ef_construction = ef_construction;
    g.m_L = 1.0 / std::log(static_cast<double>(M));
    g.seed = seed;
    g.data_t = ds_transformed;
    g.data_raw = ds_raw;
    // vertex levels: floor(-ln(U) m_L) capped at 48, U from the kHnsw stream (hnsw.cpp:203-207)
    Rng rng = Rng::for_stream(seed, rng_stream::kHnsw);
    g.levels.resize(static_cast<std::size_t>(g.n));
    for (std::int32_t& lv : g.levels)
        lv = std::min(static_cast<std::int32_t>(-std::log(rng.uniform_open0()) * g.m_L), 48);
    g.links.resize(static_cast<std::size_t>(g.n));
    GraphBuilder b(g);
    for (std::int32_t v = 0; v < g.n; ++v) b.add(v);
    return g;
}

KnnResult hnsw_query(const HnswGraph& g, const float* q_transformed, const float* q_raw, std::int32_t K,
                     std::int32_t N_ef, HnswMode mode, const DcoConfig& cfg, HnswDebug* debug) {
    // hnsw.cpp:261-265
    if (K < 1) throw std::invalid_argument("hnsw_query: K must be >= 1");
    if (N_ef < K) throw std::invalid_argument("hnsw_query: N_ef must be >= K");
    const bool transformed = mode == HnswMode::kPlus || mode == HnswMode::kPlusPlus;
    const float* q = transformed ? q_transformed : q_raw;
    if (q == nullptr) throw std::invalid_argument("hnsw_query: missing query vector");
    const auto t0 = std::chrono::steady_clock::now();
    KnnResult res;
    HopEvaluator ev(g, q, mode, cfg, res.stats);
    const std::size_t ef = static_cast<std::size_t>(N_ef), kk = static_cast<std::size_t>(K);

    // width-1 descent through the upper layers, threshold = best distance so far
    std::int32_t cur = g.entry_point;
    ev.load({cur});
    double cur_d = ev.decide(0, kInfD).observed;
    for (std::int32_t layer = g.max_layer; layer >= 1; --layer) {
        for (bool moved = true; moved;) {
            moved = false;
            const std::vector<std::int32_t> nbrs = g.links[cur][layer];
            ev.load(nbrs);
            for (std::size_t k = 0; k < nbrs.size(); ++k) {
                const Outcome o = ev.decide(static_cast<std::int32_t>(k), cur_d);
                if (o.positive && o.observed < cur_d) {
                    cur_d = o.observed;
                    cur = nbrs[k];
                    moved = true;
                    ++res.stats.hops;
                }
            }
        }
    }

    // layer 0: best-first beam; kPlusPlus keeps an exact top-K apart from the routing set
    const bool dual = mode == HnswMode::kPlusPlus;
    BeamState bs;
    bs.visited.assign(static_cast<std::size_t>(g.n), 0);
    bs.visited[cur] = 1;
    bs.frontier.emplace(cur_d, cur);
    bs.routing.emplace(cur_d, cur);
    if (dual) bs.exact_topk.emplace(cur_d, cur);
    auto trace = [&] {
        if (debug && bs.routing.size() == ef) debug->beam_max_trace.push_back(bs.routing.top().first);
    };
    trace();
    std::vector<std::int32_t> batch;
    while (!bs.frontier.empty()) {
        const Pair top = bs.frontier.top();
        if (bs.routing.size() == ef && top.first > bs.routing.top().first) break;
        bs.frontier.pop();
        ++res.stats.hops;
        batch.clear();
        for (const std::int32_t u : g.links[top.second][0])
            if (!bs.visited[u]) {
                bs.visited[u] = 1;
                batch.push_back(u);
            }
        ev.load(batch);
        for (std::size_t k = 0; k < batch.size(); ++k) {
            const std::int32_t u = batch[k];
            const double r = dual ? (bs.exact_topk.size() == kk ? bs.exact_topk.top().first : kInfD)
                                  : (bs.routing.size() == ef ? bs.routing.top().first : kInfD);
            if (debug && dual && bs.exact_topk.size() == kk && bs.routing.size() == ef)
                debug->r1_r2_thresholds.emplace_back(r, bs.routing.top().first);
            const Outcome o = ev.decide(static_cast<std::int32_t>(k), r);
            if (debug) debug->dco_log.push_back({u, r, o.positive});
            const bool route = dual ? (bs.routing.size() < ef || o.observed < bs.routing.top().first)
                                    : o.positive;
            if (dual && o.positive) {
                bs.exact_topk.emplace(o.observed, u);
                if (bs.exact_topk.size() > kk) bs.exact_topk.pop();
            }
            if (route) {
                bs.frontier.emplace(o.observed, u);
                bs.routing.emplace(o.observed, u);
                if (bs.routing.size() > ef) bs.routing.pop();
                trace();
            }
        }
    }
    std::vector<Pair> out = ascending(dual ? bs.exact_topk : bs.routing);
    if (out.size() > kk) out.resize(kk);
    for (const Pair& p : out) {
        res.ids.push_back(p.second);
        res.dists.push_back(p.first);
    }
    res.stats.candidates = res.stats.dco_count;
    if (debug) {
        debug->visited.clear();
        for (std::int32_t i = 0; i < g.n; ++i)
            if (bs.visited[i]) debug->visited.push_back(i);
    }
    res.stats.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return res;
}

// ------------------------------------------------------------------ persistence (hnsw.cpp:381-456)
void save_hnsw(const HnswGraph& g, const std::filesystem::path& dir) {
    std::filesystem::create_directories(dir);
    {
        std::ofstream m(dir / "meta.txt", std::ios::trunc);
        if (!m) throw std::runtime_error("cannot write " + (dir / "meta.txt").string());
        m << "n=" << g.n << "\nd=" << g.d << "\nM=" << g.M << "\nef_construction=" << g.ef_construction
          << "\nseed=" << g.seed << "\nentry_point=" << g.entry_point << "\nmax_layer=" << g.max_layer << "\n";
    }
    GroundTruth lv;
    lv.n_queries = g.n;
    lv.k_max = 1;
    lv.ids = g.levels;
    write_ivecs(lv, dir / "levels.ivecs");
    std::vector<std::vector<std::int32_t>> recs;  // [vertex, layer, neighbours...]
    for (std::int32_t v = 0; v < g.n; ++v)
        for (std::int32_t layer = 0; layer <= g.levels[v]; ++layer) {
            std::vector<std::int32_t> r{v, layer};
            r.insert(r.end(), g.links[v][layer].begin(), g.links[v][layer].end());
            recs.push_back(std::move(r));
        }
    write_ivecs_ragged(recs, dir / "links.ivecs");
}

HnswGraph load_hnsw(const std::filesystem::path& dir, const Dataset& ds_raw, const Dataset& ds_transformed) {
    std::ifstream m(dir / "meta.txt");
    if (!m) throw std::runtime_error("cannot open " + (dir / "meta.txt").string());
    HnswGraph g;
    for (std::string line; std::getline(m, line);) {
        const auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        const std::string k = line.substr(0, eq), v = line.substr(eq + 1);
        if (k == "n") g.n = std::stoi(v);
        else if (k == "d") g.d = std::stoi(v);
        else if (k == "M") g.M = std::stoi(v);
        else if (k == "ef_construction") g.ef_construction = std::stoi(v);
        else if (k == "seed") g.seed = std::stoull(v);
        else if (k == "entry_point") g.entry_point = std::stoi(v);
        else if (k == "max_layer") g.max_layer = std::stoi(v);
    }
    g.m_L = 1.0 / std::log(static_cast<double>(g.M));
    if (ds_raw.n != g.n || ds_raw.d != g.d || ds_transformed.n != g.n || ds_transformed.d != g.d)
        throw std::runtime_error("load_hnsw: datasets do not match the stored graph");
    g.data_raw = ds_raw;
    g.data_t = ds_transformed;
    const GroundTruth lv = read_ivecs(dir / "levels.ivecs");
    if (lv.n_queries != g.n || lv.k_max != 1) throw std::runtime_error("load_hnsw: bad levels file");
    g.levels = lv.ids;
    g.links.resize(static_cast<std::size_t>(g.n));
    for (std::int32_t v = 0; v < g.n; ++v) g.links[v].assign(static_cast<std::size_t>(g.levels[v]) + 1, {});
    for (auto& r : read_ivecs_ragged(dir / "links.ivecs")) {
        if (r.size() < 2) throw std::runtime_error("load_hnsw: malformed links record");
        const std::int32_t v = r[0], layer = r[1];
        if (v < 0 || v >= g.n || layer < 0 || layer > g.levels[v])
            throw std::runtime_error("load_hnsw: links record out of range");
        g.links[v][layer].assign(r.begin() + 2, r.end());
    }
    return g;
}

const char* hnsw_mode_name(HnswMode mode) {
    switch (mode) {
        case HnswMode::kPlain: return "plain";
        case HnswMode::kPd: return "pd";
        case HnswMode::kPlus: return "plus";
        case HnswMode::kPlusPlus: return "plusplus";
    }
    return "?";
}

HnswMode hnsw_mode_from_name(const std::string& name) {
    if (name == "plain") return HnswMode::kPlain;
    if (name == "pd") return HnswMode::kPd;
    if (name == "plus") return HnswMode::kPlus;
    if (name == "plusplus") return HnswMode::kPlusPlus;
    throw std::invalid_argument("unknown HNSW mode: " + name);
}

}  // namespace adsann
