// Drop-in check (GPU): the reference's own code path next to the device layer
// of include/pstokes_b200/pstokes_b200.hpp on identical inputs.
//  1. pstokes::solve_system vs pstokes::b200::solve_system (ITs, x bitwise);
//  2. the reference's fgmres driving the device V-cycle through ApplyFn;
//  3. the reference's gmres on DeviceCsr / DeviceIlu0 ApplyFns vs CsrMatrix /
//     Ilu0 ones (both sides, left and right preconditioning).
// Built by oracle/Makefile (target dropin) against the unmodified reference
// headers and the Eigen subset; links libpstokes_b200.so.
#include <cstdio>
#include <cstring>

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
  expect(ref.local.size() == dev.local.size() && same(ref.local[0], dev.local[0]),
         "solve_system: recovered local vectors");

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
