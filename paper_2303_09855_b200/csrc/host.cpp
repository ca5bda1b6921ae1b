// Host-side components: Rng, generate_orthogonal, mixture generators.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>

#include "../../include/adsann_b200.h"

namespace ads {

double HostRng::normal() {
    if (has_cached_) {
        has_cached_ = false;
        return cached_;
    }
    const double u1 = uniform_open0();
    const double u2 = uniform();
    const double mag = std::sqrt(-2.0 * std::log(u1));
    const double ang = 6.283185307179586476925286766559 * u2;
    cached_ = mag * std::sin(ang);
    has_cached_ = true;
    return mag * std::cos(ang);
}

void HostRng::seek_normal(uint64_t m) {
    // normal pair p consumes counters 2p+1 and 2p+2.
    counter_ = 2 * (m / 2);
    has_cached_ = false;
    if (m % 2) (void)normal();  // leaves the pair's sin variate cached
}

namespace {
double dot(const double* a, const double* b, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
void remove_projections(std::vector<double>& m, int dim, int i) {
    double* v = m.data() + static_cast<size_t>(i) * dim;
    for (int j = 0; j < i; ++j) {
        const double* r = m.data() + static_cast<size_t>(j) * dim;
        const double proj = dot(v, r, dim);
        for (int c = 0; c < dim; ++c) v[c] -= proj * r[c];
    }
}
}  // namespace

std::vector<double> generate_orthogonal(int dim, uint64_t seed) {
    if (dim < 1) throw std::invalid_argument("generate_orthogonal: dim must be >= 1");
    std::vector<double> m(static_cast<size_t>(dim) * dim);
    HostRng rng = HostRng::for_stream(seed, kTagTransform);
    for (auto& e : m) e = rng.normal();
    for (int i = 0; i < dim; ++i) {
        double* v = m.data() + static_cast<size_t>(i) * dim;
        for (int attempt = 0;; ++attempt) {
            remove_projections(m, dim, i);
            remove_projections(m, dim, i);
            const double norm = std::sqrt(dot(v, v, dim));
            if (norm > 1e-8) {
                for (int c = 0; c < dim; ++c) v[c] /= norm;
                break;
            }
            if (attempt > 8) throw std::runtime_error("generate_orthogonal: could not orthonormalize");
            for (int c = 0; c < dim; ++c) v[c] = rng.normal();
        }
    }
    // Gram check, rows split across host threads (pure reads).
    const int nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), dim));
    std::vector<double> worst(nt, 0.0);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int i = t; i < dim; i += nt)
                for (int j = i; j < dim; ++j) {
                    const double g = dot(m.data() + static_cast<size_t>(i) * dim,
                                         m.data() + static_cast<size_t>(j) * dim, dim);
                    worst[t] = std::max(worst[t], std::fabs(g - (i == j ? 1.0 : 0.0)));
                }
        });
    for (auto& x : th) x.join();
    const double w = *std::max_element(worst.begin(), worst.end());
    if (w > 1e-10)
        throw std::runtime_error("generate_orthogonal: orthonormality deviation " + std::to_string(w) +
                                 " exceeds 1e-10");
    return m;
}

// Greedy nearest-neighbour chain (fp32, heuristic: only used to order work).
std::vector<int32_t> centroid_chain_rank(const float* C, int k, int D) {
    std::vector<int32_t> rank(static_cast<size_t>(k), 0);
    if (k <= 1) return rank;
    std::vector<char> used(static_cast<size_t>(k), 0);
    const int nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), 32));
    std::vector<float> bestd(nt);
    std::vector<int> besti(nt);
    int cur = 0;
    used[0] = 1;
    for (int step = 1; step < k; ++step) {
        const float* a = C + static_cast<size_t>(cur) * D;
        auto scan = [&](int t) {
            float bd = std::numeric_limits<float>::infinity();
            int bi = -1;
            for (int c = t; c < k; c += nt) {
                if (used[c]) continue;
                const float* b = C + static_cast<size_t>(c) * D;
                float s = 0.f;
                for (int j = 0; j < D; ++j) {
                    const float df = a[j] - b[j];
                    s += df * df;
                }
                if (s < bd || (s == bd && c < bi)) {
                    bd = s;
                    bi = c;
                }
            }
            bestd[t] = bd;
            besti[t] = bi;
        };
        if (static_cast<int64_t>(k) * D < 200000) {
            for (int t = 0; t < nt; ++t) scan(t);
        } else {
            std::vector<std::thread> th;
            for (int t = 0; t < nt; ++t) th.emplace_back(scan, t);
            for (auto& x : th) x.join();
        }
        int nxt = -1;
        float nd = std::numeric_limits<float>::infinity();
        for (int t = 0; t < nt; ++t)
            if (besti[t] >= 0 && (bestd[t] < nd || (bestd[t] == nd && besti[t] < nxt))) {
                nd = bestd[t];
                nxt = besti[t];
            }
        used[nxt] = 1;
        rank[nxt] = step;
        cur = nxt;
    }
    return rank;
}

}  // namespace ads

// ------------------------------------------------------------------ mixtures
namespace {

constexpr uint64_t kTagCenters = 0x43454e5445525331ULL;  // "CENTERS1"
constexpr uint64_t kTagComp = 0x434f4d504f4e5431ULL;     // "COMPONT1"
constexpr uint64_t kTagNoise = 0x4e4f495345303031ULL;    // "NOISE001"

}  // namespace

namespace ads {

// Rows row_lo + i*stride (i < count) of the mixture whose full size is s.n:
// row r's component draw is counter r of the component stream and its noise is
// normals r*d .. r*d+d-1 of the noise stream, so any row set is reproducible
// without generating the rows before it (config 5 is generated in chunks, and
// its k-means sample directly).
void synth_rows(const ads_synth_desc& s, int64_t row_lo, int64_t count, int64_t stride, float* out,
                int32_t* comp_out) {
    if (s.n < 0 || s.d < 1 || s.components < 1) throw std::invalid_argument("synth: bad shape");
    if (!(s.sigma >= 0.0)) throw std::invalid_argument("synth: sigma must be >= 0");
    if (count < 0 || stride < 1 || row_lo < 0 || (count > 0 && row_lo + (count - 1) * stride >= s.n))
        throw std::invalid_argument("synth: row range outside [0, n)");
    const int d = s.d, C = s.components;
    // Centers: one sequential stream per seed (shared by every role).
    std::vector<double> centers(static_cast<size_t>(C) * d);
    {
        HostRng rng = HostRng::for_stream(s.seed, kTagCenters);
        for (auto& c : centers) {
            if (s.kind == 1 || s.kind == 2) c = s.center_lo + (s.center_hi - s.center_lo) * rng.uniform();
            else c = s.center_scale * rng.normal();
        }
    }
    std::vector<double> sig(d);
    for (int j = 0; j < d; ++j)
        sig[j] = s.decay ? s.sigma / std::sqrt(1.0 + static_cast<double>(j) / 32.0) : s.sigma;
    const uint64_t role_seed = HostRng::mix64(s.seed ^ (s.role * 0x9E3779B97F4A7C15ULL + 1));
    int nt = s.threads > 0 ? s.threads : static_cast<int>(std::thread::hardware_concurrency());
    nt = std::max(1, std::min<int>(nt, 64));
    if (count < 4096) nt = 1;
    auto work = [&](int64_t lo, int64_t hi) {  // output slots [lo, hi)
        std::vector<double> row(d);
        HostRng comp(HostRng::mix64(role_seed ^ kTagComp), 0);
        HostRng noise = HostRng::for_stream(role_seed, kTagNoise);
        int64_t next_row = -1;  // the row both streams are positioned at
        for (int64_t i = lo; i < hi; ++i) {
            const int64_t r = row_lo + i * stride;
            if (r != next_row) {
                comp = HostRng(HostRng::mix64(role_seed ^ kTagComp), static_cast<uint64_t>(r));
                noise.seek_normal(static_cast<uint64_t>(r) * d);
            }
            next_row = r + 1;
            int32_t c;
            if (s.assign_mode == 1) c = static_cast<int32_t>((r * C) / (s.n > 0 ? s.n : 1));
            else c = static_cast<int32_t>(comp.below(static_cast<uint64_t>(C)));
            if (comp_out) comp_out[i] = c;
            const double* cc = centers.data() + static_cast<size_t>(c) * d;
            double nrm = 0.0;
            for (int j = 0; j < d; ++j) {
                double x = cc[j] + sig[j] * noise.normal();
                if (s.kind == 1) x = std::min(255.0, std::max(0.0, std::round(x)));
                else if (s.kind == 2) x = std::min(1.0, std::max(0.0, x));
                row[j] = x;
                nrm += x * x;
            }
            float* o = out + i * d;
            if (s.kind == 3) {
                const double inv = nrm > 0.0 ? 1.0 / std::sqrt(nrm) : 0.0;
                for (int j = 0; j < d; ++j) o[j] = static_cast<float>(row[j] * inv);
            } else {
                for (int j = 0; j < d; ++j) o[j] = static_cast<float>(row[j]);
            }
        }
    };
    if (nt == 1) {
        work(0, count);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
        const int64_t lo = count * t / nt, hi = count * (t + 1) / nt;
        th.emplace_back(work, lo, hi);
    }
    for (auto& x : th) x.join();
}

void synth(const ads_synth_desc& s, float* out, int32_t* comp_out) { synth_rows(s, 0, s.n, 1, out, comp_out); }

}  // namespace ads
