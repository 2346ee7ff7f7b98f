// Level-walking triangular sweep plans (walk.cu); WalkPlan lives in internal.cuh.
#pragma once

#include <memory>
#include <vector>

#include "internal.cuh"

namespace pscu {

/// Builds the forward and backward plans of an ILU(0) factor's pattern.
void build_walk(Context& c, const Csr& a, const std::vector<int64_t>& diag, WalkPlan& wf,
                WalkPlan& wb);
/// The same in two parts: host planning (thread-safe, no device work) and
/// the upload on the context's stream.
struct WalkBuild;
std::shared_ptr<WalkBuild> plan_walk(const Csr& a, const std::vector<int64_t>& diag);
void upload_walk(Context& c, const Csr& a, const WalkBuild& b, WalkPlan& wf, WalkPlan& wb);
/// Gathers the factor values into the packed order (after every refactor).
void pack_walk(Context& c, const double* lu, WalkPlan& w);
/// y = (LU)^-1 x; x may alias y.
void run_walk(Context& c, const WalkPlan& wf, const WalkPlan& wb, const double* x, double* y);

} // namespace pscu
