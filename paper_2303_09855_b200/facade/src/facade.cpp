// adsann facade: the reference's public C++ API (namespace adsann) implemented
// on the B200 engine's C ABI (include/adsann_b200.h).  Every DCO, transform,
// k-means, index build, search and exact k-NN runs on the GPU; this file only
// marshals data, keeps the reference's aggregate types populated, and does
// host I/O (vector files, index persistence) and metric set arithmetic.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "adsann/bench.hpp"
#include "adsann/ivf.hpp"
#include "adsann/rng.hpp"
#include "adsann/transform.hpp"
#include "adsann/vecio.hpp"
#include "adsann_b200.h"

namespace {

void check(int rc) {
    if (rc == ADS_OK) return;
    if (rc == ADS_INVALID_ARGUMENT) throw std::invalid_argument(ads_last_error());
    throw std::runtime_error(ads_last_error());
}

std::mutex g_mu;
ads_ctx* g_ctx = nullptr;

ads_ctx* engine() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_ctx) check(ads_ctx_create(0, &g_ctx));
    return g_ctx;
}

// One device-resident P per distinct matrix (keyed by its bytes).
struct TransformCache {
    std::mutex mu;
    std::map<std::vector<double>, ads_transform*> by_entries;
    ads_transform* get(const adsann::TransformMatrix& m) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = by_entries.find(m.entries);
        if (it != by_entries.end()) return it->second;
        if (by_entries.size() > 16) {
            for (auto& kv : by_entries) ads_transform_destroy(kv.second);
            by_entries.clear();
        }
        ads_transform* t = nullptr;
        check(ads_transform_create(engine(), m.entries.data(), m.dim, &t));
        by_entries.emplace(m.entries, t);
        return t;
    }
} g_transforms;

std::vector<char> read_file(const std::filesystem::path& p) {
    std::ifstream in(p, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + p.string());
    return std::vector<char>(std::istreambuf_iterator<char>(in), {});
}

void write_file(const std::filesystem::path& p, const std::vector<char>& bytes) {
    std::ofstream out(p, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open " + p.string() + " for writing");
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    if (!out) throw std::runtime_error("write failed: " + p.string());
}

// [int32 d][d x 4-byte payload] records, all with the same d.
template <typename T>
std::vector<T> parse_records(const std::filesystem::path& p, std::int32_t& n, std::int32_t& d) {
    const std::vector<char> b = read_file(p);
    const std::string name = p.string();
    if (b.empty()) throw std::runtime_error(name + ": no records");
    if (b.size() < 4) throw std::runtime_error(name + ": truncated header");
    std::memcpy(&d, b.data(), 4);
    if (d < 1) throw std::runtime_error(name + ": dimension must be positive");
    const std::size_t stride = 4 * (static_cast<std::size_t>(d) + 1);
    if (b.size() % stride) throw std::runtime_error(name + ": truncated record");
    n = static_cast<std::int32_t>(b.size() / stride);
    std::vector<T> out(static_cast<std::size_t>(n) * d);
    for (std::int32_t i = 0; i < n; ++i) {
        std::int32_t di;
        std::memcpy(&di, b.data() + i * stride, 4);
        if (di != d) throw std::runtime_error(name + ": records disagree on the dimension");
        std::memcpy(out.data() + static_cast<std::size_t>(i) * d, b.data() + i * stride + 4, 4 * static_cast<std::size_t>(d));
    }
    return out;
}

template <typename T>
void emit_records(const std::filesystem::path& p, std::int32_t n, std::int32_t d, const T* payload) {
    if (n < 1) throw std::invalid_argument("vector files need at least one record");
    if (d < 1) throw std::invalid_argument("vector dimension must be >= 1");
    const std::size_t stride = 4 * (static_cast<std::size_t>(d) + 1);
    std::vector<char> b(stride * n);
    for (std::int32_t i = 0; i < n; ++i) {
        std::memcpy(b.data() + i * stride, &d, 4);
        std::memcpy(b.data() + i * stride + 4, payload + static_cast<std::size_t>(i) * d, 4 * static_cast<std::size_t>(d));
    }
    write_file(p, b);
}

}  // namespace

namespace adsann::detail {
// shared with the other facade translation units (facade_hnsw.cpp, facade_bench.cpp)
ads_ctx* engine_ctx() { return engine(); }
void check_rc(int rc) { check(rc); }
}  // namespace adsann::detail

namespace adsann {

// ------------------------------------------------------------------ vecio
Dataset read_fvecs(const std::filesystem::path& path) {
    Dataset ds;
    ds.data = parse_records<float>(path, ds.n, ds.d);
    for (float v : ds.data)
        if (!std::isfinite(v)) throw std::runtime_error(path.string() + ": non-finite value");
    return ds;
}

void write_fvecs(const Dataset& ds, const std::filesystem::path& path) {
    if (ds.data.size() != static_cast<std::size_t>(ds.n) * std::max(ds.d, 0))
        throw std::invalid_argument("write_fvecs: data size does not match n*d");
    emit_records(path, ds.n, ds.d, ds.data.data());
}

GroundTruth read_ivecs(const std::filesystem::path& path) {
    GroundTruth gt;
    gt.ids = parse_records<std::int32_t>(path, gt.n_queries, gt.k_max);
    return gt;
}

void write_ivecs(const GroundTruth& gt, const std::filesystem::path& path) {
    emit_records(path, gt.n_queries, gt.k_max, gt.ids.data());
}

std::vector<std::vector<std::int32_t>> read_ivecs_ragged(const std::filesystem::path& path) {
    const std::vector<char> b = read_file(path);
    std::vector<std::vector<std::int32_t>> rows;
    for (std::size_t at = 0; at < b.size();) {
        if (b.size() - at < 4) throw std::runtime_error(path.string() + ": truncated header");
        std::int32_t len;
        std::memcpy(&len, b.data() + at, 4);
        at += 4;
        if (len < 0) throw std::runtime_error(path.string() + ": negative length");
        const std::size_t bytes = 4 * static_cast<std::size_t>(len);
        if (b.size() - at < bytes) throw std::runtime_error(path.string() + ": truncated payload");
        rows.emplace_back(static_cast<std::size_t>(len));
        std::memcpy(rows.back().data(), b.data() + at, bytes);
        at += bytes;
    }
    return rows;
}

void write_ivecs_ragged(const std::vector<std::vector<std::int32_t>>& rows,
                        const std::filesystem::path& path) {
    std::vector<char> b;
    for (const auto& r : rows) {
        const std::int32_t len = static_cast<std::int32_t>(r.size());
        const char* lp = reinterpret_cast<const char*>(&len);
        b.insert(b.end(), lp, lp + 4);
        const char* rp = reinterpret_cast<const char*>(r.data());
        b.insert(b.end(), rp, rp + 4 * r.size());
    }
    write_file(path, b);
}

// vecio.hpp:81-89 contract: centres drawn at a growing scale until every pair is
// at least 10*spread apart, noise N(0, (spread/sqrt(d))^2), row i from blob i % n_blobs.
Dataset synth_dataset(std::int32_t n, std::int32_t d, std::int32_t n_blobs, double spread,
                      std::uint64_t seed, Dataset* centers_out) {
    if (n < 1 || d < 1 || n_blobs < 1)
        throw std::invalid_argument("synth_dataset: n, d and n_blobs must be positive");
    if (!(spread >= 0.0) || !std::isfinite(spread))
        throw std::invalid_argument("synth_dataset: spread must be finite and non-negative");
    Rng rng = Rng::for_stream(seed, rng_stream::kSynth);
    const double need = 10.0 * spread;
    std::vector<double> c(static_cast<std::size_t>(n_blobs) * d);
    for (double scale = need + 1.0;; scale *= 1.5) {
        for (double& v : c) v = scale * rng.normal();
        bool separated = true;
        for (std::int32_t x = 0; x < n_blobs && separated; ++x)
            for (std::int32_t y = x + 1; y < n_blobs && separated; ++y) {
                double s = 0.0;
                for (std::int32_t j = 0; j < d; ++j) {
                    const double t = c[static_cast<std::size_t>(x) * d + j] - c[static_cast<std::size_t>(y) * d + j];
                    s += t * t;
                }
                separated = !(s < need * need);
            }
        if (separated) break;
    }
    const double sigma = spread / std::sqrt(static_cast<double>(d));
    Dataset ds;
    ds.n = n;
    ds.d = d;
    ds.data.resize(static_cast<std::size_t>(n) * d);
    for (std::int32_t i = 0; i < n; ++i) {
        const double* ci = c.data() + static_cast<std::size_t>(i % n_blobs) * d;
        for (std::int32_t j = 0; j < d; ++j) ds.row(i)[j] = static_cast<float>(ci[j] + sigma * rng.normal());
    }
    if (centers_out) {
        centers_out->n = n_blobs;
        centers_out->d = d;
        centers_out->data.assign(c.begin(), c.end());
    }
    return ds;
}

Dataset synth_dataset(std::int32_t n, std::int32_t d, std::int32_t n_blobs, double spread,
                      std::uint64_t seed) {
    return synth_dataset(n, d, n_blobs, spread, seed, nullptr);
}

DatasetDesc read_descriptor(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path.string());
    DatasetDesc out;
    for (std::string line; std::getline(in, line);) {
        if (line.empty() || line[0] == '#') continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos) throw std::runtime_error(path.string() + ": expected key=value: " + line);
        const std::string k = line.substr(0, eq), v = line.substr(eq + 1);
        if (k == "name") out.name = v;
        else if (k == "base_path") out.base_path = v;
        else if (k == "query_path") out.query_path = v;
        else if (k == "gt_path") out.gt_path = v;
        else if (k == "d") out.d = std::stoi(v);
        else throw std::runtime_error(path.string() + ": unknown key " + k);
    }
    return out;
}

void write_descriptor(const DatasetDesc& desc, const std::filesystem::path& path) {
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open " + path.string() + " for writing");
    out << "name=" << desc.name << '\n' << "base_path=" << desc.base_path << '\n'
        << "query_path=" << desc.query_path << '\n' << "gt_path=" << desc.gt_path << '\n'
        << "d=" << desc.d << '\n';
}

// ------------------------------------------------------------------ transform
TransformMatrix generate_orthogonal(std::int32_t dim, std::uint64_t seed) {
    if (dim < 1) throw std::invalid_argument("generate_orthogonal: dim must be >= 1");
    TransformMatrix m;
    m.dim = dim;
    m.seed = seed;
    m.entries.resize(static_cast<std::size_t>(dim) * dim);
    check(ads_generate_orthogonal(dim, seed, m.entries.data()));
    return m;
}

std::vector<float> apply_prefix(const TransformMatrix& m, std::span<const float> x, std::int32_t d) {
    if (static_cast<std::int32_t>(x.size()) != m.dim)
        throw std::invalid_argument("apply: vector length does not match matrix dim");
    if (d < 0 || d > m.dim) throw std::invalid_argument("apply_prefix: d out of range");
    std::vector<float> y(m.dim);
    check(ads_apply_dataset(g_transforms.get(m), x.data(), 1, y.data()));
    y.resize(d);
    return y;
}

std::vector<float> apply(const TransformMatrix& m, std::span<const float> x) {
    return apply_prefix(m, x, m.dim);
}

std::vector<float> apply_transpose(const TransformMatrix& m, std::span<const float> x) {
    if (static_cast<std::int32_t>(x.size()) != m.dim)
        throw std::invalid_argument("apply_transpose: vector length does not match matrix dim");
    std::vector<float> y(m.dim);
    check(ads_apply_transpose(g_transforms.get(m), x.data(), 1, y.data()));
    return y;
}

Dataset apply_dataset(const TransformMatrix& m, const Dataset& ds) {
    if (ds.d != m.dim) throw std::invalid_argument("apply_dataset: dataset dimension does not match matrix");
    Dataset out;
    out.n = ds.n;
    out.d = ds.d;
    out.data.resize(ds.data.size());
    if (ds.n > 0) check(ads_apply_dataset(g_transforms.get(m), ds.data.data(), ds.n, out.data.data()));
    return out;
}

void save_matrix(const TransformMatrix& m, const std::filesystem::path& path) {
    const std::vector<float> f(m.entries.begin(), m.entries.end());  // fp32 on disk (transform.hpp:60)
    emit_records(path, m.dim, m.dim, f.data());
}

TransformMatrix load_matrix(const std::filesystem::path& path, std::uint64_t seed) {
    const Dataset ds = read_fvecs(path);
    if (ds.n != ds.d) throw std::runtime_error("load_matrix: " + path.string() + " is not square");
    TransformMatrix m;
    m.dim = ds.d;
    m.seed = seed;
    m.entries.assign(ds.data.begin(), ds.data.end());
    return m;
}

// ------------------------------------------------------------------ dco
double threshold_multiplier(std::int32_t d, const DcoConfig& cfg) {
    double out = 0.0;
    check(ads_threshold_multiplier(d, cfg.epsilon0, &out));
    return out;
}

namespace {
DcoOutcome run_dco(int kind, const DcoQuery& q, double eps0, std::int32_t dd) {
    std::int32_t pos = 0, dims = 0;
    double dist = 0.0, obs = 0.0;
    check(ads_dco(engine(), kind, q.data_vec.data(), static_cast<std::int32_t>(q.data_vec.size()),
                  q.query_vec.data(), static_cast<std::int32_t>(q.query_vec.size()), q.r, eps0, dd, &pos,
                  &dist, &obs, &dims));
    DcoOutcome out;
    out.positive = pos != 0;
    out.observed = obs;
    out.dims_used = dims;
    if (out.positive) out.distance = dist;
    return out;
}

std::vector<float> unit(std::span<const float> v, double norm) {
    std::vector<float> out(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = static_cast<float>(static_cast<double>(v[i]) / norm);
    return out;
}

double norm2(std::span<const float> v) {
    double s = 0.0;
    for (float x : v) s += static_cast<double>(x) * static_cast<double>(x);
    return std::sqrt(s);
}
}  // namespace

DcoOutcome fd_scan(const DcoQuery& q) { return run_dco(ADS_DCO_FD, q, 2.1, 1); }
DcoOutcome pd_scan(const DcoQuery& q, std::int32_t delta_d) { return run_dco(ADS_DCO_PD, q, 2.1, delta_d); }
DcoOutcome ad_sampling(const DcoQuery& q, const DcoConfig& cfg) {
    return run_dco(ADS_DCO_AD, q, cfg.epsilon0, cfg.delta_d);
}

// <o,q> >= r  <=>  ||o/|o| - q/|q|||^2 <= 2 - 2r/(|o||q|)   (paper §7)
ReducedDco reduce_inner_product(std::span<const float> o, std::span<const float> q, double r) {
    if (o.size() != q.size()) throw std::invalid_argument("reduce_inner_product: vector lengths differ");
    const double no = norm2(o), nq = norm2(q);
    if (no == 0.0 || nq == 0.0) throw std::invalid_argument("reduce_inner_product: zero-norm input");
    ReducedDco red;
    red.data_vec = unit(o, no);
    red.query_vec = unit(q, nq);
    const double t_sq = 2.0 - 2.0 * r / (no * nq);
    red.feasible = t_sq >= 0.0;
    red.r = red.feasible ? std::sqrt(t_sq) : 0.0;
    return red;
}

ReducedDco reduce_cosine(std::span<const float> o, std::span<const float> q) {
    if (o.size() != q.size()) throw std::invalid_argument("reduce_cosine: vector lengths differ");
    const double no = norm2(o), nq = norm2(q);
    if (no == 0.0 || nq == 0.0) throw std::invalid_argument("reduce_cosine: zero-norm input");
    ReducedDco red;
    red.data_vec = unit(o, no);
    red.query_vec = unit(q, nq);
    return red;
}

// ------------------------------------------------------------------ ivf
struct DeviceIvf {
    ads_ivf* h = nullptr;
    std::mutex mu;
    ~DeviceIvf() {
        if (h) ads_ivf_destroy(h);
    }
};

KmeansResult kmeans(const Dataset& ds, std::int32_t k, int max_iters, std::uint64_t seed) {
    if (k < 1) throw std::invalid_argument("kmeans: k must be >= 1");
    if (k > ds.n) throw std::invalid_argument("kmeans: k exceeds the number of points");
    KmeansResult km;
    km.centroids.n = k;
    km.centroids.d = ds.d;
    km.centroids.data.resize(static_cast<std::size_t>(k) * ds.d);
    km.assignment.resize(ds.n);
    std::int32_t iters = 0;
    check(ads_kmeans(engine(), ds.data.data(), ds.n, ds.d, k, max_iters, seed, 0, km.centroids.data.data(),
                     km.assignment.data(), &km.objective, &iters));
    km.iterations = iters;
    return km;
}

namespace {
// Fill the reference aggregate's host arrays from an engine index.
void fill_from_device(IvfIndex& idx, ads_ivf* h, std::int32_t d1p) {
    const std::size_t n = idx.n, D = idx.d, k = idx.k_clusters, d2p = D - d1p;
    idx.centroids_t = Dataset{idx.k_clusters, idx.d, std::vector<float>(k * D)};
    idx.centroids_raw = Dataset{idx.k_clusters, idx.d, std::vector<float>(k * D)};
    std::vector<std::int64_t> off(k + 1);
    idx.ids_flat.resize(n);
    std::vector<float> a1t(n * d1p), a2t(n * d2p), a1r(n * d1p), a2r(n * d2p);
    check(ads_ivf_export(h, idx.centroids_t.data.data(), idx.centroids_raw.data.data(), off.data(),
                         idx.ids_flat.data(), a1t.data(), a2t.data(), a1r.data(), a2r.data()));
    idx.buckets.assign(k, {});
    for (std::size_t c = 0; c < k; ++c)
        idx.buckets[c].assign(idx.ids_flat.begin() + off[c], idx.ids_flat.begin() + off[c + 1]);
    idx.vec_t.resize(n * D);
    idx.vec_raw.resize(n * D);
    for (std::size_t p = 0; p < n; ++p) {
        std::copy_n(&a1t[p * d1p], d1p, &idx.vec_t[p * D]);
        std::copy_n(&a2t[p * d2p], d2p, &idx.vec_t[p * D + d1p]);
        std::copy_n(&a1r[p * d1p], d1p, &idx.vec_raw[p * D]);
        std::copy_n(&a2r[p * d2p], d2p, &idx.vec_raw[p * D + d1p]);
    }
    if (idx.layout == IvfLayout::kSplit) {
        idx.a1_t = std::move(a1t);
        idx.a2_t = std::move(a2t);
        idx.a1_raw = std::move(a1r);
        idx.a2_raw = std::move(a2r);
    }
}

ads_ivf* device_of(const IvfIndex& idx) {
    auto dev = idx.device;
    if (!dev) throw std::runtime_error("ivf_query: index has no device state");
    std::lock_guard<std::mutex> lk(dev->mu);
    if (dev->h) return dev->h;
    // Upload a host-built or loaded aggregate.
    std::vector<std::int64_t> off(idx.k_clusters + 1, 0);
    for (std::int32_t c = 0; c < idx.k_clusters; ++c) off[c + 1] = off[c] + static_cast<std::int64_t>(idx.buckets[c].size());
    ads_ivf_desc d{};
    d.n = idx.n;
    d.d = idx.d;
    d.k_clusters = idx.k_clusters;
    d.d1 = idx.d1;
    d.layout = idx.layout == IvfLayout::kSplit;
    d.seed = idx.seed;
    d.centroids_t = idx.centroids_t.data.data();
    d.centroids_raw = idx.centroids_raw.data.empty() ? nullptr : idx.centroids_raw.data.data();
    d.list_off = off.data();
    d.ids_flat = idx.ids_flat.data();
    d.vec_t = idx.vec_t.data();
    d.vec_raw = idx.vec_raw.empty() ? nullptr : idx.vec_raw.data();
    if (d.layout && !idx.a1_t.empty()) {
        d.a1_t = idx.a1_t.data();
        d.a2_t = idx.a2_t.data();
        d.a1_raw = idx.a1_raw.empty() ? nullptr : idx.a1_raw.data();
        d.a2_raw = idx.a2_raw.empty() ? nullptr : idx.a2_raw.data();
    }
    check(ads_ivf_create(engine(), &d, &dev->h));
    return dev->h;
}
}  // namespace

IvfIndex build_ivf(const Dataset& ds_raw, const Dataset& ds_transformed, const TransformMatrix& m,
                   std::int32_t k_clusters, std::uint64_t seed, IvfLayout layout, std::int32_t d1) {
    if (ds_raw.n != ds_transformed.n || ds_raw.d != ds_transformed.d)
        throw std::invalid_argument("build_ivf: raw and transformed datasets disagree");
    if (m.dim != ds_raw.d) throw std::invalid_argument("build_ivf: matrix dimension does not match the data");
    if (layout == IvfLayout::kSplit && (d1 < 1 || d1 >= ds_raw.d))
        throw std::invalid_argument("build_ivf: split layout needs 1 <= d1 < D");
    IvfIndex idx;
    idx.n = ds_raw.n;
    idx.d = ds_raw.d;
    idx.k_clusters = k_clusters;
    idx.d1 = d1;
    idx.layout = layout;
    idx.seed = seed;
    idx.device = std::make_shared<DeviceIvf>();
    // build_ivf runs k-means with 25 iterations from k-means++ (ivf.cpp:210)
    check(ads_ivf_build(engine(), ds_raw.data.data(), ds_transformed.data.data(), ds_raw.n, ds_raw.d,
                        m.entries.data(), k_clusters, seed, layout == IvfLayout::kSplit, d1, 25, 0,
                        &idx.device->h));
    fill_from_device(idx, idx.device->h, layout == IvfLayout::kSplit ? d1 : std::min(32, idx.d));
    return idx;
}

KnnResult ivf_query(const IvfIndex& idx, const float* q_transformed, const float* q_raw, std::int32_t K,
                    std::int32_t n_probe, IvfMode mode, const DcoConfig& cfg) {
    const auto t0 = std::chrono::steady_clock::now();
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!idx.device) idx.device = std::make_shared<DeviceIvf>();
    }
    ads_ivf* h = device_of(idx);
    ads_search_opts o;
    ads_search_opts_default(&o);
    o.first = 1;  // the reference re-reads the K-th distance before every candidate
    o.step = 1;
    const std::int32_t Kc = std::max(K, 1);
    std::vector<std::int32_t> ids(Kc);
    std::vector<double> dists(Kc);
    std::int32_t cnt = 0;
    std::uint64_t dims = 0, cand = 0;
    check(ads_ivf_search(h, q_transformed, q_raw, 1, K, n_probe, static_cast<int>(mode), cfg.epsilon0,
                         cfg.delta_d, &o, ids.data(), dists.data(), &cnt, &dims, &cand));
    KnnResult r;
    r.ids.assign(ids.begin(), ids.begin() + cnt);
    r.dists.assign(dists.begin(), dists.begin() + cnt);
    r.stats.dims_evaluated = dims;
    r.stats.dco_count = cand;
    r.stats.candidates = cand;
    r.stats.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return r;
}

// On-disk format of the reference (ivf.cpp:423-501): meta.txt + fvecs/ivecs files.
void save_ivf(const IvfIndex& idx, const std::filesystem::path& dir) {
    std::filesystem::create_directories(dir);
    {
        std::ofstream meta(dir / "meta.txt", std::ios::trunc);
        if (!meta) throw std::runtime_error("cannot open " + (dir / "meta.txt").string() + " for writing");
        meta << "n=" << idx.n << "\nd=" << idx.d << "\nk_clusters=" << idx.k_clusters << "\nd1=" << idx.d1
             << "\nlayout=" << (idx.layout == IvfLayout::kSplit ? "split" : "contiguous") << "\nseed=" << idx.seed
             << '\n';
    }
    write_fvecs(idx.centroids_t, dir / "centroids_t.fvecs");
    write_fvecs(idx.centroids_raw, dir / "centroids_raw.fvecs");
    write_ivecs_ragged(idx.buckets, dir / "buckets.ivecs");
    emit_records(dir / "vec_t.fvecs", idx.n, idx.d, idx.vec_t.data());
    emit_records(dir / "vec_raw.fvecs", idx.n, idx.d, idx.vec_raw.data());
    if (idx.layout == IvfLayout::kSplit) {
        emit_records(dir / "a1_t.fvecs", idx.n, idx.d1, idx.a1_t.data());
        emit_records(dir / "a2_t.fvecs", idx.n, idx.d - idx.d1, idx.a2_t.data());
        emit_records(dir / "a1_raw.fvecs", idx.n, idx.d1, idx.a1_raw.data());
        emit_records(dir / "a2_raw.fvecs", idx.n, idx.d - idx.d1, idx.a2_raw.data());
    }
}

IvfIndex load_ivf(const std::filesystem::path& dir) {
    std::ifstream meta(dir / "meta.txt");
    if (!meta) throw std::runtime_error("cannot open " + (dir / "meta.txt").string());
    IvfIndex idx;
    for (std::string line; std::getline(meta, line);) {
        const auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        const std::string k = line.substr(0, eq), v = line.substr(eq + 1);
        if (k == "n") idx.n = std::stoi(v);
        else if (k == "d") idx.d = std::stoi(v);
        else if (k == "k_clusters") idx.k_clusters = std::stoi(v);
        else if (k == "d1") idx.d1 = std::stoi(v);
        else if (k == "layout") idx.layout = v == "split" ? IvfLayout::kSplit : IvfLayout::kContiguous;
        else if (k == "seed") idx.seed = std::stoull(v);
    }
    idx.centroids_t = read_fvecs(dir / "centroids_t.fvecs");
    idx.centroids_raw = read_fvecs(dir / "centroids_raw.fvecs");
    idx.buckets = read_ivecs_ragged(dir / "buckets.ivecs");
    if (static_cast<std::int32_t>(idx.buckets.size()) != idx.k_clusters)
        throw std::runtime_error("load_ivf: bucket count does not match metadata");
    for (const auto& b : idx.buckets) idx.ids_flat.insert(idx.ids_flat.end(), b.begin(), b.end());
    if (static_cast<std::int32_t>(idx.ids_flat.size()) != idx.n)
        throw std::runtime_error("load_ivf: bucket contents do not cover the dataset");
    idx.vec_t = read_fvecs(dir / "vec_t.fvecs").data;
    idx.vec_raw = read_fvecs(dir / "vec_raw.fvecs").data;
    if (idx.layout == IvfLayout::kSplit) {
        idx.a1_t = read_fvecs(dir / "a1_t.fvecs").data;
        idx.a2_t = read_fvecs(dir / "a2_t.fvecs").data;
        idx.a1_raw = read_fvecs(dir / "a1_raw.fvecs").data;
        idx.a2_raw = read_fvecs(dir / "a2_raw.fvecs").data;
    }
    idx.device = std::make_shared<DeviceIvf>();
    return idx;
}

const char* ivf_mode_name(IvfMode mode) {
    static const char* names[] = {"fd", "pd", "ad", "ad-split", "pd-split"};
    const int m = static_cast<int>(mode);
    return m >= 0 && m < 5 ? names[m] : "?";
}

IvfMode ivf_mode_from_name(const std::string& name) {
    for (int m = 0; m < 5; ++m)
        if (name == ivf_mode_name(static_cast<IvfMode>(m))) return static_cast<IvfMode>(m);
    throw std::invalid_argument("unknown IVF mode: " + name);
}

// ------------------------------------------------------------------ bench
GroundTruth brute_force_knn(const Dataset& ds, const Dataset& queries, std::int32_t K) {
    if (ds.d != queries.d) throw std::invalid_argument("brute_force_knn: dimensionality mismatch");
    if (K < 1) throw std::invalid_argument("brute_force_knn: K must be >= 1");
    if (K > ds.n) throw std::invalid_argument("brute_force_knn: K exceeds dataset size");
    GroundTruth gt;
    gt.n_queries = queries.n;
    gt.k_max = K;
    gt.ids.resize(static_cast<std::size_t>(queries.n) * K);
    check(ads_brute_force_knn(engine(), ds.data.data(), ds.n, ds.d, queries.data.data(), queries.n, K,
                              gt.ids.data()));
    return gt;
}

std::vector<TheoryRow> verify_theory(const Dataset& ds_t, const Dataset& queries_t, std::int32_t K,
                                     std::vector<double> epsilon0_grid) {
    if (ds_t.d != queries_t.d) throw std::invalid_argument("verify_theory: dimensionality mismatch");
    if (K < 1 || K > ds_t.n) throw std::invalid_argument("verify_theory: bad K");
    const auto G = static_cast<std::int32_t>(epsilon0_grid.size());
    std::vector<double> eps(G), fr(G), ad(G);
    std::vector<std::uint64_t> fails(G), pos(G);
    check(ads_verify_theory(engine(), ds_t.data.data(), ds_t.n, ds_t.d, queries_t.data.data(), queries_t.n, K,
                            epsilon0_grid.data(), G, eps.data(), fr.data(), ad.data(), fails.data(), pos.data()));
    std::vector<TheoryRow> rows(G);
    for (std::int32_t g = 0; g < G; ++g) rows[g] = TheoryRow{eps[g], fr[g], ad[g], fails[g], pos[g]};
    return rows;
}

void write_theory_csv(const std::vector<TheoryRow>& rows, const std::filesystem::path& path) {
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open " + path.string() + " for writing");
    out << "epsilon0,failure_rate,avg_dims,failures,positives\n";
    char line[256];
    for (const TheoryRow& r : rows) {
        std::snprintf(line, sizeof(line), "%.3f,%.8f,%.4f,%llu,%llu\n", r.epsilon0, r.failure_rate, r.avg_dims,
                      static_cast<unsigned long long>(r.failures), static_cast<unsigned long long>(r.positives));
        out << line;
    }
}

double recall(std::span<const std::int32_t> result_ids, std::span<const std::int32_t> gt_ids, std::int32_t K) {
    if (static_cast<std::int32_t>(gt_ids.size()) < K) throw std::invalid_argument("recall: ground truth shorter than K");
    const std::unordered_set<std::int32_t> truth(gt_ids.begin(), gt_ids.begin() + K);
    std::int32_t hits = 0;
    for (std::int32_t id : result_ids) hits += truth.count(id) ? 1 : 0;
    return static_cast<double>(hits) / K;
}

std::optional<double> avg_distance_ratio(std::span<const double> result_dists, std::span<const double> gt_dists,
                                         std::int32_t K) {
    if (static_cast<std::int32_t>(result_dists.size()) < K || static_cast<std::int32_t>(gt_dists.size()) < K)
        throw std::invalid_argument("avg_distance_ratio: need at least K distances");
    double acc = 0.0;
    for (std::int32_t i = 0; i < K; ++i) {
        if (gt_dists[i] == 0.0) {
            if (result_dists[i] != 0.0) return std::nullopt;
            acc += 1.0;
        } else {
            acc += result_dists[i] / gt_dists[i];
        }
    }
    return acc / K;
}

}  // namespace adsann

namespace adsann::detail {
ads_ivf* ivf_handle(const IvfIndex& idx) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!idx.device) idx.device = std::make_shared<DeviceIvf>();
    }
    return device_of(idx);
}
ads_transform* transform_handle(const TransformMatrix& m) { return g_transforms.get(m); }
}  // namespace adsann::detail
