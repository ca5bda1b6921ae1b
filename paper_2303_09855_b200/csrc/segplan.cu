// Host-side segment planning (see engine.hpp).  Pure host code; compiled by
// nvcc with the rest of the library.
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "engine.hpp"

namespace ads {

std::vector<double> ad_factor(double eps0, int delta_d, int D) {
    // dco.cpp:32-37 validation, dco.cpp:54-61 table.
    if (!(eps0 > 0.0)) throw std::invalid_argument("dco: epsilon0 must be > 0");
    if (delta_d < 1 || delta_d > D) throw std::invalid_argument("dco: delta_d must be in [1, D]");
    std::vector<double> f(static_cast<size_t>(D), 0.0);
    for (int k = 1; k < D; ++k) {
        const double mult = 1.0 + eps0 / std::sqrt(static_cast<double>(k));
        f[k] = mult * mult * static_cast<double>(k) / static_cast<double>(D);
    }
    return f;
}

std::vector<int> test_points(int D, int delta_d, int d_start, bool test_at_start) {
    // dco.hpp:129 (start test when 0 < d < D) and dco.hpp:132-144 (stop = min(d+Δd, D)).
    std::vector<int> t;
    int d = d_start;
    if (test_at_start && d > 0 && d < D) t.push_back(d);
    while (d < D) {
        const int stop = std::min(d + delta_d, D);
        d = stop;
        if (d < D) t.push_back(d);
    }
    return t;
}

SegPlan make_seg_plan(int D, int split_at, const std::vector<int>& tests, const double* factor) {
    if (D < 1) throw std::invalid_argument("dimension must be >= 1");
    if (D > 32767) throw std::invalid_argument("dimension too large for the segment table");
    SegPlan p;
    p.D = D;
    std::vector<int> cuts{0, D};
    for (int t : tests) cuts.push_back(t);
    if (split_at > 0 && split_at < D) cuts.push_back(split_at);
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    bool aligned = D % 4 == 0;
    for (int c : cuts) aligned = aligned && c % 4 == 0;
    if (split_at > 0 && split_at < D) aligned = aligned && split_at % 4 == 0 && (D - split_at) % 4 == 0;
    p.vec = aligned ? 4 : 1;
    for (size_t i = 0; i + 1 < cuts.size(); ++i) {
        const int a = cuts[i], b = cuts[i + 1];
        const bool is_test = std::binary_search(tests.begin(), tests.end(), b) && b < D;
        for (int s = a; s < b; s += 32) {
            const int e = std::min(s + 32, b);
            Seg sg;
            sg.arr = static_cast<int16_t>((split_at > 0 && s >= split_at) ? 1 : 0);
            sg.len = static_cast<int16_t>(e - s);
            sg.col = static_cast<int16_t>(s);
            sg.test = -1;
            if (e == b && is_test) {
                sg.test = static_cast<int16_t>(p.test_factor.size());
                p.test_factor.push_back(factor ? factor[b] : 1.0);
            }
            p.segs.push_back(sg);
        }
    }
    if (p.segs.size() > 4096) throw std::invalid_argument("too many segments");
    p.full = p.vec == 4;
    for (const Seg& sg : p.segs) p.full = p.full && sg.len == 32;
    return p;
}

void DevSegPlan::upload(const SegPlan& p, cudaStream_t st) {
    release();
    nseg = static_cast<int>(p.segs.size());
    ntest = static_cast<int>(p.test_factor.size());
    vec = p.vec;
    full = p.full;
    nseg0 = 0;
    while (nseg0 < nseg - 1 && p.segs[nseg0].test < 0) ++nseg0;
    ADS_CUDA(cudaMallocAsync(&segs, sizeof(Seg) * nseg, st));
    ADS_CUDA(cudaMemcpyAsync(segs, p.segs.data(), sizeof(Seg) * nseg, cudaMemcpyHostToDevice, st));
    ADS_CUDA(cudaMallocAsync(&tfac, sizeof(double) * std::max(ntest, 1), st));
    if (ntest)
        ADS_CUDA(cudaMemcpyAsync(tfac, p.test_factor.data(), sizeof(double) * ntest,
                                 cudaMemcpyHostToDevice, st));
    // The host vectors may die after return: make the copies complete.
    ADS_CUDA(cudaStreamSynchronize(st));
}

void DevSegPlan::release() {
    if (segs) cudaFree(segs);
    if (tfac) cudaFree(tfac);
    segs = nullptr;
    tfac = nullptr;
}

}  // namespace ads
