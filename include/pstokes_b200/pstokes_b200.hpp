// include/pstokes_b200/pstokes_b200.hpp — C++ drop-in layer over the C ABI
// (include/pstokes_cuda.h) with the reference's own types and signatures
// (/root/reference/proj/include/pstokes). Include it after the reference
// headers; it adds namespace pstokes::b200 with:
//   solve_system(mesh, sys, cfg)          plevels.hpp:217-239
//   DeviceCsr      (CsrMatrix::multiply)  csr.hpp:68-76
//   DeviceIlu0     (Ilu0 / Ilu0::apply)   ilu0.hpp:19-65
//   DeviceHierarchy (LevelHierarchy)      plevels.hpp:125-206
//   recover_solution(sys, x)              assemble.hpp:58-66, condense.hpp:28-38
// and ApplyFn adapters (gmres.hpp:17) so the reference's own gmres/fgmres
// can drive the device operators unchanged. Errors rethrow by code:
// PSCU_EINVAL -> std::invalid_argument, everything else -> std::runtime_error.
#pragma once

#include <map>
#include <memory>
#include <stdexcept>
#include <utility>
#include <vector>

#include "pstokes/plevels.hpp"
#include "pstokes_cuda.h"

namespace pstokes::b200 {

inline void check(int rc) {
  if (rc == PSCU_EINVAL) throw std::invalid_argument(pscu_last_error());
  if (rc) throw std::runtime_error(pscu_last_error());
}

/// One device context per host thread (the reference is single-threaded).
inline pscu_ctx* context() {
  thread_local std::unique_ptr<pscu_ctx, int (*)(pscu_ctx*)> ctx(
      [] {
        pscu_ctx* c = nullptr;
        check(pscu_create(0, &c));
        return c;
      }(),
      pscu_destroy);
  return ctx.get();
}

inline pscu_layout to_pscu(const DofLayout& l) {
  return pscu_layout{int(l.scheme), int(l.strategy), l.k, l.n_faces, l.n_elements,
                     l.face_vel, l.face_press, l.elem_vel, l.elem_press};
}

inline pscu_level_cfg to_pscu(const LevelConfig& cfg, int smoother = PSCU_SMOOTHER_ILU0) {
  return pscu_level_cfg{smoother, cfg.smoother_iters,
                        cfg.coarse == CoarseSolver::Lu ? PSCU_COARSE_LU : PSCU_COARSE_ILU_GMRES,
                        cfg.coarse_rtol, cfg.coarse_maxit};
}

/// CsrMatrix resident on the device; multiply() as CsrMatrix::multiply.
class DeviceCsr {
 public:
  explicit DeviceCsr(const CsrMatrix& a) : n_(a.n) {
    pscu_mat* m = nullptr;
    check(pscu_mat_create(context(), a.n, a.row_ptr.data(), a.cols.data(), a.vals.data(),
                          PSCU_HOST, &m));
    m_.reset(m);
  }
  explicit DeviceCsr(const pscu_mat* borrowed, int n) : n_(n), view_(borrowed) {}
  const pscu_mat* get() const { return view_ ? view_ : m_.get(); }
  int n() const { return n_; }
  void multiply(const double* x, double* y) const {
    check(pscu_spmv(context(), get(), x, y, PSCU_HOST));
  }
  Eigen::VectorXd multiply(const Eigen::VectorXd& x) const {
    Eigen::VectorXd y(n_);
    multiply(x.data(), y.data());
    return y;
  }
  ApplyFn apply_fn() const {
    return [this](const Eigen::VectorXd& x) { return multiply(x); };
  }

 private:
  int n_;
  const pscu_mat* view_ = nullptr;
  std::unique_ptr<pscu_mat, int (*)(pscu_mat*)> m_{nullptr, pscu_mat_destroy};
};

/// Ilu0 factorised and applied on the device (bit-identical factors).
class DeviceIlu0 {
 public:
  explicit DeviceIlu0(const DeviceCsr& a) : n_(a.n()) {
    pscu_ilu* p = nullptr;
    check(pscu_ilu0_create(context(), a.get(), &p));
    p_.reset(p);
  }
  void apply(const double* x, double* y) const {
    check(pscu_ilu0_apply(context(), p_.get(), x, y, PSCU_HOST));
  }
  Eigen::VectorXd apply(const Eigen::VectorXd& x) const {
    Eigen::VectorXd y(n_);
    apply(x.data(), y.data());
    return y;
  }
  ApplyFn apply_fn() const {
    return [this](const Eigen::VectorXd& x) { return apply(x); };
  }

 private:
  int n_;
  std::unique_ptr<pscu_ilu, int (*)(pscu_ilu*)> p_{nullptr, pscu_ilu0_destroy};
};

/// LevelHierarchy on the device: vcycle(), coarse_iterations(),
/// reset_counters() as plevels.hpp:170-206.
class DeviceHierarchy {
 public:
  DeviceHierarchy(const DeviceCsr& fine, const DofLayout& layout, const LevelConfig& cfg,
                  int smoother = PSCU_SMOOTHER_ILU0)
      : n_(fine.n()) {
    const pscu_layout l = to_pscu(layout);
    const pscu_level_cfg c = to_pscu(cfg, smoother);
    pscu_hier* h = nullptr;
    check(pscu_hier_create(context(), fine.get(), &l, cfg.degrees.data(), int(cfg.degrees.size()),
                           &c, &h));
    h_.reset(h);
  }
  Eigen::VectorXd vcycle(int level, const Eigen::VectorXd& d) const {
    Eigen::VectorXd c(d.size());
    check(pscu_vcycle(context(), h_.get(), level, d.data(), c.data(), PSCU_HOST));
    return c;
  }
  long long coarse_iterations() const { return pscu_hier_coarse_its(h_.get()); }
  void reset_counters() { pscu_hier_reset(h_.get()); }
  /// The variable preconditioner of solve_system: one V-cycle from level 0.
  ApplyFn vcycle_fn() const {
    return [this](const Eigen::VectorXd& d) { return vcycle(0, d); };
  }
  pscu_hier* get() const { return h_.get(); }

 private:
  int n_;
  std::unique_ptr<pscu_hier, int (*)(pscu_hier*)> h_{nullptr, pscu_hier_destroy};
};

/// StokesSystem::recover_solution (assemble.hpp:58-66) on the device:
/// ElementCondensation::recover (condense.hpp:28-38) for every element
/// through pscu_recover_batch, batched over the elements that share a local
/// size and elimination list (all of them on the reference's meshes). The
/// device back-substitution x_e = elim_rhs - elim_coupling x_k sums k
/// ascending from 0 like the reference's product, so the result is bitwise.
inline std::vector<Eigen::VectorXd> recover_solution(const StokesSystem& sys,
                                                     const Eigen::VectorXd& x) {
  std::map<std::pair<int, std::vector<int>>, std::vector<std::size_t>> groups;
  for (std::size_t e = 0; e < sys.recovery.size(); ++e) {
    const ElementCondensation& c = sys.recovery[e];
    groups[{int(c.keep.size() + c.elim.size()), c.elim}].push_back(e);
  }
  std::vector<Eigen::VectorXd> out(sys.recovery.size());
  for (const auto& [key, elems] : groups) {
    const int n = key.first;
    const std::vector<int>& elim = key.second;
    const int ne = int(elim.size()), nk = n - ne;
    const std::size_t ng = elems.size();
    std::vector<std::int64_t> kept(ng * nk);
    std::vector<double> coup(ng * std::size_t(ne) * nk), erhs(ng * std::size_t(ne));
    for (std::size_t g = 0; g < ng; ++g) {
      const std::size_t e = elems[g];
      const ElementCondensation& c = sys.recovery[e];
      for (int i = 0; i < nk; ++i) kept[g * nk + i] = sys.kept_global[e][i];
      if (ne) {
        std::copy(c.elim_coupling.data(), c.elim_coupling.data() + std::size_t(ne) * nk,
                  coup.begin() + g * std::size_t(ne) * nk);
        std::copy(c.elim_rhs.data(), c.elim_rhs.data() + ne, erhs.begin() + g * ne);
      }
    }
    std::vector<double> locals(ng * std::size_t(n));
    check(pscu_recover_batch(context(), int(ng), n, ne, elim.data(), kept.data(), coup.data(),
                             erhs.data(), x.data(), locals.data(), PSCU_HOST));
    for (std::size_t g = 0; g < ng; ++g)
      out[elems[g]] = Eigen::Map<const Eigen::VectorXd>(locals.data() + g * n, n);
  }
  return out;
}

/// solve_system (plevels.hpp:217-239) with the hierarchy, FGMRES and the
/// recovery of the eliminated unknowns on the device.
inline StokesSolution solve_system(const Mesh&, const StokesSystem& sys, const LevelConfig& cfg) {
  const pscu_layout lay = to_pscu(sys.layout);
  const pscu_level_cfg lc = to_pscu(cfg);
  StokesSolution sol;
  sol.x.resize(sys.a.n);
  pscu_report rep{};
  check(pscu_solve_system(context(), sys.a.n, sys.a.row_ptr.data(), sys.a.cols.data(),
                          sys.a.vals.data(), sys.rhs.data(), &lay, cfg.degrees.data(),
                          int(cfg.degrees.size()), &lc, cfg.outer_rtol, cfg.outer_maxit,
                          /*restart=*/0, sol.x.data(), /*hist=*/nullptr, &rep));
  sol.report.outer_its = rep.outer_its;
  sol.report.coarse_its = rep.coarse_its;
  sol.report.vcycles = rep.vcycles;
  sol.report.rel_residual = rep.rel_residual;
  sol.report.converged = rep.converged != 0;
  sol.report.t_assembly = sys.t_assembly;
  sol.report.t_solve = rep.t_solve;
  sol.local = recover_solution(sys, sol.x);
  return sol;
}

}  // namespace pstokes::b200
