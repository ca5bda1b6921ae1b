// Private glue shared by the facade's translation units.
#pragma once

#include "adsann_b200.h"

namespace adsann::detail {
ads_ctx* engine_ctx();   // the facade's engine context (device 0)
void check_rc(int rc);   // ads_status -> std::invalid_argument / std::runtime_error
}  // namespace adsann::detail

namespace adsann {
struct IvfIndex;
struct TransformMatrix;
namespace detail {
ads_ivf* ivf_handle(const IvfIndex& idx);                 // the index's engine copy (uploaded on first use)
ads_transform* transform_handle(const TransformMatrix& m);  // P resident on the device
}  // namespace detail
}  // namespace adsann
