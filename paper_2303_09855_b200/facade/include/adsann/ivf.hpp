// adsann facade — IVF index (reference: include/adsann/ivf.hpp:28-95).
// k-means, build_ivf and ivf_query run on the B200; the IvfIndex aggregate keeps
// the reference's host-visible fields and owns the device copy it searches.
#pragma once

#include <cstdint>
#include <filesystem>
#include <memory>
#include <string>
#include <vector>

#include "adsann/dco.hpp"
#include "adsann/result.hpp"
#include "adsann/transform.hpp"
#include "adsann/vecio.hpp"

namespace adsann {

struct KmeansResult {
    Dataset centroids;
    std::vector<std::int32_t> assignment;
    double objective = 0.0;
    int iterations = 0;
};

KmeansResult kmeans(const Dataset& ds, std::int32_t k, int max_iters, std::uint64_t seed);

enum class IvfLayout { kContiguous, kSplit };
enum class IvfMode { kFd, kPd, kAd, kAdSplit, kPdSplit };

struct DeviceIvf;  // engine handle (ads_ivf), created on first query

struct IvfIndex {
    std::int32_t n = 0;
    std::int32_t d = 0;
    std::int32_t k_clusters = 0;
    std::int32_t d1 = 0;
    IvfLayout layout = IvfLayout::kContiguous;
    std::uint64_t seed = 0;
    Dataset centroids_t;
    Dataset centroids_raw;
    std::vector<std::vector<std::int32_t>> buckets;
    std::vector<std::int32_t> ids_flat;
    std::vector<float> vec_t;
    std::vector<float> vec_raw;
    std::vector<float> a1_t, a2_t;
    std::vector<float> a1_raw, a2_raw;
    mutable std::shared_ptr<DeviceIvf> device;  // engine copy (not part of the reference aggregate)
};

IvfIndex build_ivf(const Dataset& ds_raw, const Dataset& ds_transformed, const TransformMatrix& m,
                   std::int32_t k_clusters, std::uint64_t seed,
                   IvfLayout layout = IvfLayout::kContiguous, std::int32_t d1 = 32);

KnnResult ivf_query(const IvfIndex& idx, const float* q_transformed, const float* q_raw,
                    std::int32_t K, std::int32_t n_probe, IvfMode mode, const DcoConfig& cfg);

void save_ivf(const IvfIndex& idx, const std::filesystem::path& dir);
IvfIndex load_ivf(const std::filesystem::path& dir);

const char* ivf_mode_name(IvfMode mode);
IvfMode ivf_mode_from_name(const std::string& name);

}  // namespace adsann
