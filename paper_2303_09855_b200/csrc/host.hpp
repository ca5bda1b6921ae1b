// Host-side components of the engine (no device code): the reference's
// counter-based Rng, the orthogonal-matrix generator and the seeded
// Gaussian-mixture generators used by the benchmark configurations.
#pragma once

#include <stdint.h>

#include <vector>

namespace ads {

// rng.hpp:36-97.  Output i depends only on (seed, i); normal() is
// Box-Muller with the cos variate first and the sin variate cached.
class HostRng {
public:
    explicit HostRng(uint64_t seed, uint64_t counter = 0) : seed_(seed), counter_(counter) {}
    static HostRng for_stream(uint64_t seed, uint64_t tag) { return HostRng(mix64(seed ^ tag)); }
    static uint64_t mix64(uint64_t z) {
        z ^= z >> 30;
        z *= 0xBF58476D1CE4E5B9ULL;
        z ^= z >> 27;
        z *= 0x94D049BB133111EBULL;
        z ^= z >> 31;
        return z;
    }
    uint64_t next_u64() {
        ++counter_;
        return mix64(seed_ + counter_ * 0x9E3779B97F4A7C15ULL);
    }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double uniform_open0() { return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53; }
    uint64_t below(uint64_t n) { return next_u64() % n; }
    double normal();
    // Position the stream so the next normal() is normal number m of a
    // stream that draws only normals.
    void seek_normal(uint64_t m);

private:
    uint64_t seed_, counter_;
    double cached_ = 0.0;
    bool has_cached_ = false;
};

// rng.hpp:26-31 stream tags.
constexpr uint64_t kTagTransform = 0x9d5c41cf0f5e6a31ULL;

// transform.cpp:47-97: row-wise modified Gram-Schmidt (two passes) of an
// i.i.d. N(0,1) matrix from Rng::for_stream(seed, kTransform); verifies
// max |P P^T - I| <= 1e-10.  Throws like the reference.
std::vector<double> generate_orthogonal(int dim, uint64_t seed);

}  // namespace ads
