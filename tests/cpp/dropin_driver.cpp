// Drop-in check (GPU): the reference's own code path next to the device layer
// of include/pstokes_b200/pstokes_b200.hpp on identical inputs.
//  1. pstokes::solve_system vs pstokes::b200::solve_system (ITs, x bitwise);
//  2. the reference's fgmres driving the device V-cycle through ApplyFn;
//  3. the reference's gmres on DeviceCsr / DeviceIlu0 ApplyFns vs CsrMatrix /
//     Ilu0 ones (both sides, left and right preconditioning).
// Built by oracle/Makefile (target dropin) against the unmodified reference
// headers and the Eigen subset; links libpstokes_b200.so.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <tuple>

#include "pstokes/plevels.hpp"
#include "pstokes/study.hpp"
#include "pstokes_b200/pstokes_b200.hpp"

using namespace pstokes;

static int failures = 0;
static void expect(bool ok, const char* what) {
  std::printf("%s %s\n", ok ? "OK  " : "FAIL", what);
  if (!ok) ++failures;
}
static bool same(const Eigen::VectorXd& a, const Eigen::VectorXd& b) {
  if (a.size() != b.size()) return false;
  for (Eigen::Index i = 0; i < a.size(); ++i)
    if (!(a[i] == b[i])) return false;
  return true;
}

int main() {
  const Mesh mesh = make_family_mesh("trapz", 4, 1, Side::Right);
  const StokesSystem sys = assemble_stokes(mesh, Scheme::HhoDp, Strategy::VCond, 3,
                                           ManufacturedCase::data());
  LevelConfig cfg = LevelConfig::defaults_for(3);
  cfg.coarse = CoarseSolver::IluGmres;
  cfg.outer_rtol = 1e-10;

  // 1. solve_system
  const StokesSolution ref = solve_system(mesh, sys, cfg);
  const StokesSolution dev = b200::solve_system(mesh, sys, cfg);
  expect(ref.report.outer_its == dev.report.outer_its, "solve_system: FGMRES iterations equal");
  expect(ref.report.coarse_its == dev.report.coarse_its, "solve_system: coarse iterations equal");
  expect(same(ref.x, dev.x), "solve_system: solution bitwise");
  bool all_local = ref.local.size() == dev.local.size();
  for (std::size_t e = 0; all_local && e < ref.local.size(); ++e)
    all_local = same(ref.local[e], dev.local[e]);
  expect(all_local, "solve_system: device-recovered local vectors bitwise (every element)");
  // device recovery on its own, for the other condensation variants
  for (const auto& [scheme, strategy, k] :
       {std::tuple{Scheme::HhoDp, Strategy::VpCond, 2}, std::tuple{Scheme::HhoHp, Strategy::VpCond, 2},
        std::tuple{Scheme::HhoDp, Strategy::Uncond, 1}}) {
    const StokesSystem s2 = assemble_stokes(mesh, scheme, strategy, k, ManufacturedCase::data());
    Eigen::VectorXd xs(s2.a.n);
    for (Eigen::Index i = 0; i < xs.size(); ++i) xs[i] = std::sin(0.37 * double(i) + 0.1);
    const auto r1 = s2.recover_solution(xs);
    const auto r2 = b200::recover_solution(s2, xs);
    bool ok = r1.size() == r2.size();
    for (std::size_t e = 0; ok && e < r1.size(); ++e) ok = same(r1[e], r2[e]);
    expect(ok, (std::string("recover_solution bitwise: ") + to_string(scheme) + " " +
                to_string(strategy)).c_str());
  }

  // 2. reference fgmres with the device V-cycle as the variable preconditioner
  b200::DeviceCsr a(sys.a);
  b200::DeviceHierarchy hier(a, sys.layout, cfg);
  const KrylovResult kr = fgmres(a.apply_fn(), hier.vcycle_fn(), sys.rhs, cfg.outer_maxit,
                                 cfg.outer_rtol);
  expect(kr.iterations == ref.report.outer_its && same(kr.x, ref.x),
         "reference fgmres over DeviceCsr + DeviceHierarchy::vcycle: bitwise");

  // 3. reference gmres on device operators
  Ilu0 ilu(sys.a);
  b200::DeviceIlu0 dilu(a);
  const ApplyFn op = [&](const Eigen::VectorXd& x) { return sys.a.multiply(x); };
  const ApplyFn pc = [&](const Eigen::VectorXd& x) {
    Eigen::VectorXd y(x.size());
    ilu.apply(x.data(), y.data());
    return y;
  };
  const Eigen::VectorXd x0 = Eigen::VectorXd::Zero(sys.a.n);
  for (PrecondSide side : {PrecondSide::Right, PrecondSide::Left}) {
    const KrylovResult r1 = gmres(op, pc, sys.rhs, x0, 50, 1e-8, side);
    const KrylovResult r2 = gmres(a.apply_fn(), dilu.apply_fn(), sys.rhs, x0, 50, 1e-8, side);
    expect(r1.iterations == r2.iterations && same(r1.x, r2.x),
           side == PrecondSide::Right ? "reference gmres (right) over DeviceCsr/DeviceIlu0"
                                      : "reference gmres (left) over DeviceCsr/DeviceIlu0");
  }
  std::printf("%s\n", failures ? "dropin: FAILED" : "dropin: all checks passed");
  return failures ? 1 : 0;
}
