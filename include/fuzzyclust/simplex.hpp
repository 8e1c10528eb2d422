// fuzzyclust/simplex.hpp -- drop-in for project_simplex(_inplace)
// (simplex.hpp:18-66).  Runs the device projection (fc_project_simplex_rows),
// bit-identical to the reference's sort-threshold + residual folds.
#pragma once

#include <span>
#include <vector>

#include "fuzzyclust/common.hpp"
#include "fuzzyclust/device.hpp"

namespace fuzzyclust {

inline void project_simplex_inplace(std::span<double> x) {
    if (x.empty()) throw InvalidInput("project_simplex: empty vector");
    auto& d = device::context();
    device::check(fc_project_simplex_rows(d.ctx, static_cast<uint32_t>(x.size()), 1, x.data()), d.ctx);
}

inline std::vector<double> project_simplex(std::span<const double> x) {
    std::vector<double> y(x.begin(), x.end());
    project_simplex_inplace(y);
    return y;
}

}  // namespace fuzzyclust
