// adsann facade — random orthogonal transform (reference: include/adsann/transform.hpp:32-62).
// generate_orthogonal runs on the host (as in the reference); every apply* runs
// on the B200 with the reference's fp64 order, so results are bit-identical.
#pragma once

#include <cstdint>
#include <filesystem>
#include <span>
#include <vector>

#include "adsann/vecio.hpp"

namespace adsann {

struct TransformMatrix {
    std::int32_t dim = 0;
    std::uint64_t seed = 0;
    std::vector<double> entries;
    const double* row(std::int32_t i) const { return entries.data() + static_cast<std::size_t>(i) * dim; }
};

TransformMatrix generate_orthogonal(std::int32_t dim, std::uint64_t seed);
std::vector<float> apply(const TransformMatrix& m, std::span<const float> x);
std::vector<float> apply_prefix(const TransformMatrix& m, std::span<const float> x, std::int32_t d);
std::vector<float> apply_transpose(const TransformMatrix& m, std::span<const float> x);
Dataset apply_dataset(const TransformMatrix& m, const Dataset& ds);
void save_matrix(const TransformMatrix& m, const std::filesystem::path& path);
TransformMatrix load_matrix(const std::filesystem::path& path, std::uint64_t seed = 0);

}  // namespace adsann
