// adsann facade — distance comparison operations (reference: include/adsann/dco.hpp:28-79).
// Each DCO runs on the B200 (ads_dco); the batched form is adsann_b200::dco_fixed.
#pragma once

#include <cmath>
#include <cstdint>
#include <optional>
#include <span>
#include <vector>

namespace adsann {

struct DcoConfig {
    double epsilon0 = 2.1;
    std::int32_t delta_d = 32;
};

struct DcoOutcome {
    bool positive = false;
    std::optional<double> distance;
    double observed = 0.0;
    std::int32_t dims_used = 0;
};

struct DcoQuery {
    std::span<const float> data_vec;
    std::span<const float> query_vec;
    double r = 0.0;
};

struct ReducedDco {
    std::vector<float> data_vec;
    std::vector<float> query_vec;
    double r = 0.0;
    bool feasible = true;
    DcoQuery query() const { return DcoQuery{data_vec, query_vec, r}; }
};

double threshold_multiplier(std::int32_t d, const DcoConfig& cfg);
DcoOutcome fd_scan(const DcoQuery& q);
DcoOutcome pd_scan(const DcoQuery& q, std::int32_t delta_d);
DcoOutcome ad_sampling(const DcoQuery& q, const DcoConfig& cfg);
ReducedDco reduce_inner_product(std::span<const float> o, std::span<const float> q, double r);
ReducedDco reduce_cosine(std::span<const float> o, std::span<const float> q);

}  // namespace adsann
