// Level-walking triangular sweep plans (walk.cu); WalkPlan lives in internal.cuh.
#pragma once

#include <vector>

#include "internal.cuh"

namespace pscu {

/// Builds the forward and backward plans of an ILU(0) factor's pattern.
void build_walk(Context& c, const Csr& a, const std::vector<int64_t>& diag, WalkPlan& wf,
                WalkPlan& wb);
/// Gathers the factor values into the packed order (after every refactor).
void pack_walk(Context& c, const double* lu, WalkPlan& w);
/// y = (LU)^-1 x; x may alias y.
void run_walk(Context& c, const WalkPlan& wf, const WalkPlan& wb, const double* x, double* y);

} // namespace pscu
