// Level-walking triangular sweep plans (walk.cu); WalkPlan lives in internal.cuh.
#pragma once

#include <vector>

#include "internal.cuh"

namespace pscu {

void build_walk(Context& c, const Csr& a, const std::vector<int64_t>& diag, bool fwd, WalkPlan& w);
/// Gathers the factor values into the packed order (after every refactor).
void pack_walk(Context& c, const double* lu, WalkPlan& w);
/// Forward: y = L^-1 x (unit L). Backward: y = U^-1 xin (in place allowed).
void run_walk(Context& c, const WalkPlan& w, const double* xin, double* y);

} // namespace pscu
