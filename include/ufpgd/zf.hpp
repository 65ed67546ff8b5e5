// ufpgd/zf.hpp of the reference (/root/reference/proj/core/include/ufpgd/zf.hpp:8-18).
// zf_precoder is declared in ufpgd/metrics.hpp and runs on the device in FP64.
#pragma once

#include "ufpgd/metrics.hpp"

namespace ufpgd {

// Gram matrices with a 2-norm condition number beyond this are singular.
inline constexpr double kSingularConditionLimit = 1e12;

}  // namespace ufpgd
