// csd/metrics.hpp — coefficient of determination used by the approximation-quality tests
// (reference metrics.hpp:10).  Host utility (64-bit, two-pass).
#pragma once

#include "csd/tensor.hpp"

namespace csd {

double r_squared(const Tensor& exact, const Tensor& approx);

}  // namespace csd
