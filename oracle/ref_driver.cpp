// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A flat C ABI over the UNMODIFIED reference headers (compiled in place from
// /root/reference/proj/include against include/eigen_subset; see
// oracle/Makefile). It is the strongest oracle available: the reference's own
// assembly, hierarchy, ILU(0), GMRES/FGMRES and V-cycle code, exposed so the
// pytest parity suite can compare the CUDA path with it on identical inputs.
// Only tests/, __graft_entry__.smoke() and bench.py's reference arm load it.
//
// The only restated reference logic is fgmres_hist(), a copy of the control
// flow of pstokes::fgmres (gmres.hpp:145-173) that additionally records the
// Arnoldi residual estimate per iteration and supports an optional restart
// (FGMRES(m), BASELINE.json). With restart = 0 it is checked bit-for-bit
// against pstokes::solve_system by tests/test_oracle_ref.py.

#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pstokes/plevels.hpp"
#include "pstokes/study.hpp"

using namespace pstokes;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

/// BASELINE.json configs 1-2 manufactured field on the unit square:
/// u = (sin(pi x) cos(pi y), -cos(pi x) sin(pi y)), p = sin(2 pi x) sin(2 pi y).
struct SinCosCase {
  static Vec2 velocity(const Vec2& q) {
    const double x = q.x(), y = q.y();
    return Vec2(std::sin(M_PI * x) * std::cos(M_PI * y), -std::cos(M_PI * x) * std::sin(M_PI * y));
  }
  static Eigen::Matrix2d grad(const Vec2& q) { // (i,j) = d u_j / d x_i
    const double x = q.x(), y = q.y();
    Eigen::Matrix2d g;
    g(0, 0) = M_PI * std::cos(M_PI * x) * std::cos(M_PI * y);
    g(1, 0) = -M_PI * std::sin(M_PI * x) * std::sin(M_PI * y);
    g(0, 1) = M_PI * std::sin(M_PI * x) * std::sin(M_PI * y);
    g(1, 1) = -M_PI * std::cos(M_PI * x) * std::cos(M_PI * y);
    return g;
  }
  static double pressure(const Vec2& q) {
    return std::sin(2.0 * M_PI * q.x()) * std::sin(2.0 * M_PI * q.y());
  }
  static Vec2 force(const Vec2& q) {
    const double x = q.x(), y = q.y(), pi = M_PI;
    return Vec2(2.0 * pi * pi * std::sin(pi * x) * std::cos(pi * y) +
                    2.0 * pi * std::cos(2.0 * pi * x) * std::sin(2.0 * pi * y),
                -2.0 * pi * pi * std::cos(pi * x) * std::sin(pi * y) +
                    2.0 * pi * std::sin(2.0 * pi * x) * std::cos(2.0 * pi * y));
  }
  static Vec2 traction(const Vec2& q, const Vec2& n) {
    const Eigen::Matrix2d g = grad(q);
    Vec2 ng(n.x() * g(0, 0) + n.y() * g(1, 0), n.x() * g(0, 1) + n.y() * g(1, 1));
    return -ng + pressure(q) * n;
  }
  static StokesData data() { return {force, velocity, traction}; }
};

StokesData data_of(int kind) {
  switch (kind) {
    case 0: return StokesData::zero();
    case 1: return ManufacturedCase::data();
    case 2: return SinCosCase::data();
  }
  throw std::invalid_argument("unknown data kind");
}

/// Unit-square structured mesh used by BASELINE.json configs 1-2: vertex
/// (i,j) at (i/n, j/n); interior vertices jittered by frac*(1/n)*sym(), x then
/// y, for j = 1..n-1, i = 1..n-1 with SplitMix64(seed) (the reference's own
/// jitter recipe, mesh.hpp:279-288, with dmin = h). tri != 0 splits every
/// cell along the (i,j)-(i+1,j+1) diagonal (mesh.hpp:311-342, fixed=true).
Mesh unit_square_mesh(int n, int tri, double frac, std::uint64_t seed, Side side) {
  detail::NodeGrid g;
  g.n = n;
  g.pts.resize((n + 1) * (n + 1));
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i <= n; ++i)
      g.pts[detail::grid_vertex(i, j, n)] = Vec2(double(i) / double(n), double(j) / double(n));
  if (frac > 0.0) {
    SplitMix64 rng(seed);
    const double h = 1.0 / double(n);
    for (int j = 1; j < n; ++j)
      for (int i = 1; i < n; ++i) {
        Vec2& p = g.pts[detail::grid_vertex(i, j, n)];
        p.x() += frac * h * rng.sym();
        p.y() += frac * h * rng.sym();
      }
  }
  Mesh m = tri ? detail::tris_from_grid(g, true) : detail::quads_from_grid(g);
  // classify_boundary tests |mid - (+-1)| < 1e-12; only the +1 sides exist
  // on the unit square, so right/top are the usable Neumann sides.
  classify_boundary(m, side);
  return m;
}

struct System {
  Mesh mesh;
  StokesSystem sys;
  std::vector<HhoLocalBlocks> locals; // optional, filled on demand
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

/// mesh_kind: 0 = reference family (make_family_mesh), 1 = unit-square quads,
/// 2 = unit-square split triangles. side: 0 left, 1 right, 2 top, 3 bottom.
void* ref_system_create(int mesh_kind, const char* family, int n, unsigned long long seed,
                        double jitter, int side, int scheme, int strategy, int k, int data_kind,
                        double eta) {
  try {
    auto s = std::make_unique<System>();
    const Side sd = static_cast<Side>(side);
    if (mesh_kind == 0) s->mesh = make_family_mesh(family, n, seed, sd);
    else s->mesh = unit_square_mesh(n, mesh_kind == 2, jitter, seed, sd);
    s->sys = assemble_stokes(s->mesh, static_cast<Scheme>(scheme), static_cast<Strategy>(strategy),
                             k, data_of(data_kind), eta);
    return s.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void ref_system_destroy(void* h) { delete static_cast<System*>(h); }


long long ref_system_dim(void* h) { return static_cast<System*>(h)->sys.a.n; }
long long ref_system_nnz(void* h) { return static_cast<System*>(h)->sys.a.nnz(); }
double ref_system_t_assembly(void* h) { return static_cast<System*>(h)->sys.t_assembly; }

void ref_system_csr(void* h, long long* row_ptr, int* cols, double* vals) {
  const CsrMatrix& a = static_cast<System*>(h)->sys.a;
  for (int i = 0; i <= a.n; ++i) row_ptr[i] = a.row_ptr[i];
  std::memcpy(cols, a.cols.data(), sizeof(int) * a.cols.size());
  std::memcpy(vals, a.vals.data(), sizeof(double) * a.vals.size());
}

void ref_system_rhs(void* h, double* rhs) {
  const auto& r = static_cast<System*>(h)->sys.rhs;
  std::memcpy(rhs, r.data(), sizeof(double) * r.size());
}

/// out[0..9] = scheme, strategy, k, n_faces, n_elements, face_vel, face_press,
/// elem_vel, elem_press, n_vertices
void ref_system_layout(void* h, int* out) {
  const System* s = static_cast<System*>(h);
  const DofLayout& l = s->sys.layout;
  out[0] = int(l.scheme);
  out[1] = int(l.strategy);
  out[2] = l.k;
  out[3] = l.n_faces;
  out[4] = l.n_elements;
  out[5] = l.face_vel;
  out[6] = l.face_press;
  out[7] = l.elem_vel;
  out[8] = l.elem_press;
  out[9] = s->mesh.n_vertices();
}

/// Mesh export: vertices (2*nv), element offsets (ne+1) and loops, faces
/// (5 ints per face: a, b, left, right, tag).
int ref_mesh_sizes(void* h, long long* out) {
  const Mesh& m = static_cast<System*>(h)->mesh;
  out[0] = m.n_vertices();
  out[1] = m.n_elements();
  out[2] = m.n_faces();
  long long loops = 0;
  for (const auto& e : m.elements) loops += static_cast<long long>(e.size());
  out[3] = loops;
  return 0;
}

void ref_mesh_export(void* h, double* xy, long long* eoff, int* loops, int* faces, int* efaces,
                     int* esigns) {
  const Mesh& m = static_cast<System*>(h)->mesh;
  for (int v = 0; v < m.n_vertices(); ++v) {
    xy[2 * v] = m.vertices[v].x();
    xy[2 * v + 1] = m.vertices[v].y();
  }
  long long p = 0;
  eoff[0] = 0;
  for (int e = 0; e < m.n_elements(); ++e) {
    for (std::size_t i = 0; i < m.elements[e].size(); ++i) {
      loops[p] = m.elements[e][i];
      efaces[p] = m.element_faces[e][i].face;
      esigns[p] = m.element_faces[e][i].sign;
      ++p;
    }
    eoff[e + 1] = p;
  }
  for (int f = 0; f < m.n_faces(); ++f) {
    const Face& fc = m.faces[f];
    faces[5 * f] = fc.a;
    faces[5 * f + 1] = fc.b;
    faces[5 * f + 2] = fc.left;
    faces[5 * f + 3] = fc.right;
    faces[5 * f + 4] = int(fc.tag);
  }
}

/// Per-element condensation record of the assembled system (condense.hpp:19-38,
/// assemble.hpp:150-158). sizes[0..2] = n_local, n_elim, n_keep; call with
/// null buffers first to size them.
int ref_local_element(void* h, int e, int* sizes, int* elim, long long* kept_global, double* schur, double* reduced_rhs,
                      double* elim_coupling, double* elim_rhs) {
  try {
    System* s = static_cast<System*>(h);
    const ElementCondensation& c = s->sys.recovery[e];
    const int n = static_cast<int>(c.keep.size() + c.elim.size());
    sizes[0] = n;
    sizes[1] = static_cast<int>(c.elim.size());
    sizes[2] = static_cast<int>(c.keep.size());
    if (!elim) return 0;
    for (std::size_t i = 0; i < c.elim.size(); ++i) elim[i] = c.elim[i];
    for (std::size_t i = 0; i < c.keep.size(); ++i) kept_global[i] = s->sys.kept_global[e][i];
    const int nk = sizes[2], ne = sizes[1];
    for (int j = 0; j < nk; ++j)
      for (int i = 0; i < nk; ++i) schur[i + j * nk] = c.schur(i, j);
    for (int i = 0; i < nk; ++i) reduced_rhs[i] = c.reduced_rhs[i];
    for (int j = 0; j < nk; ++j)
      for (int i = 0; i < ne; ++i) elim_coupling[i + j * ne] = c.elim_coupling(i, j);
    for (int i = 0; i < ne; ++i) elim_rhs[i] = c.elim_rhs[i];
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

/// Full local matrix and load of element e for data kind `data_kind`
/// (build_hho_local, hho_local.hpp:193-318) and its eliminated dof list
/// (condense.hpp:44-55). Call with mat == nullptr to query sizes[0..1].
int ref_local_blocks(void* h, int e, int data_kind, int* sizes, double* mat, double* rhs,
                     int* elim) {
  try {
    System* s = static_cast<System*>(h);
    const DofLayout& l = s->sys.layout;
    if (l.scheme == Scheme::Dg) throw std::invalid_argument("local blocks: HHO only");
    HhoElement he(s->mesh, e, l.k, element_degree(l.scheme, l.k));
    HhoLocalBlocks b = build_hho_local(he, l.scheme == Scheme::HhoHp,
                                       default_dirichlet_penalty(l.k), data_of(data_kind));
    const auto el = eliminated_dofs(b, l.scheme, l.strategy);
    sizes[0] = b.size();
    sizes[1] = static_cast<int>(el.size());
    if (!mat) return 0;
    const int n = b.size();
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) mat[i + j * n] = b.mat(i, j);
    for (int i = 0; i < n; ++i) rhs[i] = b.rhs[i];
    for (std::size_t i = 0; i < el.size(); ++i) elim[i] = el[i];
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// ---------------------------------------------------------------------------
// generic CSR / ILU / Krylov wrappers
// ---------------------------------------------------------------------------

void* ref_csr_create(int n, const long long* row_ptr, const int* cols, const double* vals) {
  auto* a = new CsrMatrix;
  a->n = n;
  a->row_ptr.assign(row_ptr, row_ptr + n + 1);
  a->cols.assign(cols, cols + row_ptr[n]);
  a->vals.assign(vals, vals + row_ptr[n]);
  return a;
}
void ref_csr_destroy(void* a) { delete static_cast<CsrMatrix*>(a); }
void ref_csr_multiply(void* a, const double* x, double* y) {
  static_cast<CsrMatrix*>(a)->multiply(x, y);
}

void* ref_ilu_create(void* a) {
  try {
    return new Ilu0(*static_cast<CsrMatrix*>(a));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void ref_ilu_destroy(void* p) { delete static_cast<Ilu0*>(p); }
void ref_ilu_apply(void* p, const double* x, double* y) { static_cast<Ilu0*>(p)->apply(x, y); }
void ref_ilu_factors(void* p, double* lu) {
  const auto& f = static_cast<Ilu0*>(p)->factors();
  std::memcpy(lu, f.data(), sizeof(double) * f.size());
}

/// pstokes::gmres (gmres.hpp:103-139) with the ILU(0) of `a` as preconditioner
/// (ilu may be null = unpreconditioned). side: 0 right, 1 left.
int ref_gmres(void* a, void* ilu, const double* rhs, const double* x0, int max_it, double rtol,
              int side, double* x, int* its, double* rel, int* converged) {
  try {
    const CsrMatrix& A = *static_cast<CsrMatrix*>(a);
    const Ilu0* I = static_cast<Ilu0*>(ilu);
    ApplyFn op = [&A](const Eigen::VectorXd& v) { return A.multiply(v); };
    ApplyFn pc = nullptr;
    if (I) pc = [I](const Eigen::VectorXd& v) { return I->apply(v); };
    const Eigen::VectorXd b = Eigen::Map<const Eigen::VectorXd>(rhs, A.n);
    const Eigen::VectorXd xx0 = Eigen::Map<const Eigen::VectorXd>(x0, A.n);
    const KrylovResult r = gmres(op, pc, b, xx0, max_it, rtol,
                                 side ? PrecondSide::Left : PrecondSide::Right);
    std::memcpy(x, r.x.data(), sizeof(double) * A.n);
    *its = r.iterations;
    *rel = r.rel_residual;
    *converged = r.converged;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// pstokes::fgmres (gmres.hpp:145-173) with a fixed ILU(0) preconditioner.
int ref_fgmres(void* a, void* ilu, const double* rhs, int max_it, double rtol, double* x, int* its,
               double* rel, int* converged) {
  try {
    const CsrMatrix& A = *static_cast<CsrMatrix*>(a);
    const Ilu0* I = static_cast<Ilu0*>(ilu);
    ApplyFn op = [&A](const Eigen::VectorXd& v) { return A.multiply(v); };
    ApplyFn pc = [I](const Eigen::VectorXd& v) { return I ? I->apply(v) : v; };
    const Eigen::VectorXd b = Eigen::Map<const Eigen::VectorXd>(rhs, A.n);
    const KrylovResult r = fgmres(op, pc, b, max_it, rtol);
    std::memcpy(x, r.x.data(), sizeof(double) * A.n);
    *its = r.iterations;
    *rel = r.rel_residual;
    *converged = r.converged;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---------------------------------------------------------------------------
// hierarchy
// ---------------------------------------------------------------------------

struct Hier {
  const System* sys;
  LevelConfig cfg;
  std::unique_ptr<LevelHierarchy> h;
  double t_setup = 0.0;
};

void* ref_hier_create(void* sysh, const int* degrees, int nlev, int smoother_iters, int coarse_kind,
                      double coarse_rtol, int coarse_maxit) {
  try {
    auto hh = std::make_unique<Hier>();
    hh->sys = static_cast<System*>(sysh);
    hh->cfg.degrees.assign(degrees, degrees + nlev);
    hh->cfg.smoother_iters = smoother_iters;
    hh->cfg.coarse = coarse_kind ? CoarseSolver::IluGmres : CoarseSolver::Lu;
    hh->cfg.coarse_rtol = coarse_rtol;
    hh->cfg.coarse_maxit = coarse_maxit;
    const auto t0 = std::chrono::steady_clock::now();
    hh->h = std::make_unique<LevelHierarchy>(hh->sys->mesh, hh->sys->sys, hh->cfg);
    hh->t_setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return hh.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void ref_hier_destroy(void* h) { delete static_cast<Hier*>(h); }
int ref_hier_nlev(void* h) { return static_cast<Hier*>(h)->h->n_levels(); }
double ref_hier_t_setup(void* h) { return static_cast<Hier*>(h)->t_setup; }
long long ref_hier_level_dim(void* h, int l) { return static_cast<Hier*>(h)->h->level(l).a.n; }
long long ref_hier_level_nnz(void* h, int l) { return static_cast<Hier*>(h)->h->level(l).a.nnz(); }
void ref_hier_level_csr(void* h, int l, long long* row_ptr, int* cols, double* vals) {
  const CsrMatrix& a = static_cast<Hier*>(h)->h->level(l).a;
  for (int i = 0; i <= a.n; ++i) row_ptr[i] = a.row_ptr[i];
  std::memcpy(cols, a.cols.data(), sizeof(int) * a.cols.size());
  std::memcpy(vals, a.vals.data(), sizeof(double) * a.vals.size());
}
/// down_map of level l (coarse level l+1 -> level l); empty on the coarsest.
long long ref_hier_level_downmap(void* h, int l, long long* out) {
  const auto& m = static_cast<Hier*>(h)->h->level(l).down_map;
  if (out)
    for (std::size_t i = 0; i < m.size(); ++i) out[i] = m[i];
  return static_cast<long long>(m.size());
}
int ref_hier_level_ilu(void* h, int l, double* lu) {
  const Level& lev = static_cast<Hier*>(h)->h->level(l);
  const Ilu0* ilu = lev.smoother_ilu ? lev.smoother_ilu.get() : lev.coarse_ilu.get();
  if (!ilu) return -1;
  const auto& f = ilu->factors();
  std::memcpy(lu, f.data(), sizeof(double) * f.size());
  return 0;
}
int ref_hier_vcycle(void* h, int l, const double* d, double* c) {
  try {
    Hier* hh = static_cast<Hier*>(h);
    const long long n = hh->h->level(l).a.n;
    const Eigen::VectorXd dv = Eigen::Map<const Eigen::VectorXd>(d, n);
    const Eigen::VectorXd cv = hh->h->vcycle(l, dv);
    std::memcpy(c, cv.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
long long ref_hier_coarse_its(void* h) { return static_cast<Hier*>(h)->h->coarse_iterations(); }
void ref_hier_reset(void* h) { static_cast<Hier*>(h)->h->reset_counters(); }

/// Restated control flow of pstokes::fgmres (gmres.hpp:145-173) plus the
/// per-iteration Arnoldi estimate |g_{j+1}| / ||b|| in hist[j] and an
/// optional restart length (0 = unrestarted, the reference behaviour).
/// Restart: after `restart` iterations without triggering the convergence
/// check, x0 <- x_m and the Arnoldi process restarts from b - A x0.
static KrylovResult fgmres_hist(const ApplyFn& op, const ApplyFn& pc, const Eigen::VectorXd& rhs,
                                int max_it, double rtol, int restart, std::vector<double>& hist,
                                std::vector<double>* stamps = nullptr) {
  const auto t_begin = std::chrono::steady_clock::now();
  KrylovResult res;
  const double bnorm = rhs.norm();
  if (bnorm == 0.0) {
    res.x = Eigen::VectorXd::Zero(rhs.size());
    res.converged = true;
    return res;
  }
  Eigen::VectorXd x0 = Eigen::VectorXd::Zero(rhs.size());
  const int cycle = restart > 0 ? restart : max_it;
  int total = 0;
  Eigen::VectorXd r0 = rhs;
  double beta = bnorm;
  while (true) {
    detail::ArnoldiWorkspace ws;
    const int mm = std::min(cycle, max_it - total);
    ws.init(static_cast<int>(rhs.size()), mm, r0, beta);
    bool restart_now = false;
    for (int j = 0; j < mm; ++j) {
      ws.z.push_back(pc(ws.v[j]));
      const double est = ws.step(j, op(ws.z[j]));
      ++total;
      hist.push_back(est / bnorm);
      if (stamps)
        stamps->push_back(
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_begin).count());
      const int m = j + 1;
      const bool last = total == max_it;
      if (est <= rtol * bnorm || ws.last_subdiag == 0.0 || last) {
        res.x = ws.solution(x0, m);
        res.rel_residual = (rhs - op(res.x)).norm() / bnorm;
        res.iterations = total;
        if (res.rel_residual <= rtol) {
          res.converged = true;
          return res;
        }
        if (last) return res;
        if (j + 1 == mm) { // cycle exhausted after a failed true-residual check
          restart_now = true;
          x0 = res.x;
        }
      } else if (j + 1 == mm) {
        restart_now = true;
        x0 = ws.solution(x0, m);
      }
    }
    if (!restart_now) {
      // converged-check failed without restart room: continue unrestarted
      // semantics are only defined for restart == 0 (handled above).
      return res;
    }
    r0 = rhs - op(x0);
    beta = r0.norm();
  }
}

/// solve_system (plevels.hpp:217-239) with residual history: t_solve covers
/// hierarchy setup + FGMRES exactly like the reference's timer.
int ref_solve(void* sysh, const int* degrees, int nlev, int smoother_iters, int coarse_kind,
              double coarse_rtol, int coarse_maxit, double outer_rtol, int outer_maxit, int restart,
              double* x, double* hist, int* its, long long* coarse_its, int* vcycles, double* rel,
              int* converged, double* t_solve) {
  try {
    const System* s = static_cast<System*>(sysh);
    LevelConfig cfg;
    cfg.degrees.assign(degrees, degrees + nlev);
    cfg.smoother_iters = smoother_iters;
    cfg.coarse = coarse_kind ? CoarseSolver::IluGmres : CoarseSolver::Lu;
    cfg.coarse_rtol = coarse_rtol;
    cfg.coarse_maxit = coarse_maxit;
    cfg.outer_rtol = outer_rtol;
    cfg.outer_maxit = outer_maxit;
    const auto t0 = std::chrono::steady_clock::now();
    LevelHierarchy hier(s->mesh, s->sys, cfg);
    int vc = 0;
    ApplyFn op = [s](const Eigen::VectorXd& v) { return s->sys.a.multiply(v); };
    ApplyFn pc = [&hier, &vc](const Eigen::VectorXd& d) {
      ++vc;
      return hier.vcycle(0, d);
    };
    std::vector<double> hv;
    const KrylovResult r = fgmres_hist(op, pc, s->sys.rhs, outer_maxit, outer_rtol, restart, hv);
    *t_solve = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(x, r.x.data(), sizeof(double) * r.x.size());
    if (hist)
      for (std::size_t i = 0; i < hv.size(); ++i) hist[i] = hv[i];
    *its = r.iterations;
    *coarse_its = hier.coarse_iterations();
    *vcycles = vc;
    *rel = r.rel_residual;
    *converged = r.converged;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// Timing sample for bench.py's reference arm: the reference LevelHierarchy
/// setup (t_setup) and the end time of every FGMRES iteration after it
/// (stamps[i], seconds from the start of the iteration loop), restart as
/// given, stopping after `outer_maxit` iterations or on convergence.
int ref_solve_timed(void* sysh, const int* degrees, int nlev, int smoother_iters, int coarse_kind,
                    double coarse_rtol, int coarse_maxit, double outer_rtol, int outer_maxit,
                    int restart, double* t_setup, double* stamps, int* its) {
  try {
    const System* s = static_cast<System*>(sysh);
    LevelConfig cfg;
    cfg.degrees.assign(degrees, degrees + nlev);
    cfg.smoother_iters = smoother_iters;
    cfg.coarse = coarse_kind ? CoarseSolver::IluGmres : CoarseSolver::Lu;
    cfg.coarse_rtol = coarse_rtol;
    cfg.coarse_maxit = coarse_maxit;
    cfg.outer_rtol = outer_rtol;
    cfg.outer_maxit = outer_maxit;
    const auto t0 = std::chrono::steady_clock::now();
    LevelHierarchy hier(s->mesh, s->sys, cfg);
    *t_setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ApplyFn op = [s](const Eigen::VectorXd& v) { return s->sys.a.multiply(v); };
    ApplyFn pc = [&hier](const Eigen::VectorXd& d) { return hier.vcycle(0, d); };
    std::vector<double> hv, st;
    const KrylovResult r =
        fgmres_hist(op, pc, s->sys.rhs, outer_maxit, outer_rtol, restart, hv, &st);
    for (std::size_t i = 0; i < st.size(); ++i) stamps[i] = st[i];
    *its = static_cast<int>(st.size());
    (void)r;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// The reference's own solve_system, untouched, for the fgmres_hist check.
int ref_solve_system(void* sysh, const int* degrees, int nlev, int smoother_iters, int coarse_kind,
                     double outer_rtol, int outer_maxit, double* x, int* its, long long* coarse_its,
                     int* vcycles, double* rel, int* converged, double* t_solve) {
  try {
    const System* s = static_cast<System*>(sysh);
    LevelConfig cfg;
    cfg.degrees.assign(degrees, degrees + nlev);
    cfg.smoother_iters = smoother_iters;
    cfg.coarse = coarse_kind ? CoarseSolver::IluGmres : CoarseSolver::Lu;
    cfg.outer_rtol = outer_rtol;
    cfg.outer_maxit = outer_maxit;
    const StokesSolution sol = solve_system(s->mesh, s->sys, cfg);
    std::memcpy(x, sol.x.data(), sizeof(double) * sol.x.size());
    *its = sol.report.outer_its;
    *coarse_its = sol.report.coarse_its;
    *vcycles = sol.report.vcycles;
    *rel = sol.report.rel_residual;
    *converged = sol.report.converged;
    *t_solve = sol.report.t_solve;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// inherit_matrix (plevels.hpp:93-113) between two layouts of the system's
/// mesh at degrees kf > kc. Returns nnz; call with null buffers first.
long long ref_inherit(void* sysh, int kf, int kc, long long* row_ptr, int* cols, double* vals,
                      long long* c2f) {
  try {
    const System* s = static_cast<System*>(sysh);
    const DofLayout& l0 = s->sys.layout;
    const DofLayout lf = make_layout(s->mesh, l0.scheme, l0.strategy, kf);
    const DofLayout lc = make_layout(s->mesh, l0.scheme, l0.strategy, kc);
    const CsrMatrix fine = kf == l0.k ? s->sys.a : inherit_matrix(s->sys.a, l0, lf);
    const CsrMatrix a = inherit_matrix(fine, lf, lc);
    if (row_ptr) {
      for (int i = 0; i <= a.n; ++i) row_ptr[i] = a.row_ptr[i];
      std::memcpy(cols, a.cols.data(), sizeof(int) * a.cols.size());
      std::memcpy(vals, a.vals.data(), sizeof(double) * a.vals.size());
      const auto m = coarse_to_fine_map(lf, lc);
      for (std::size_t i = 0; i < m.size(); ++i) c2f[i] = m[i];
    }
    return a.nnz();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

long long ref_layout_dim(void* sysh, int k) {
  const System* s = static_cast<System*>(sysh);
  const DofLayout& l0 = s->sys.layout;
  return make_layout(s->mesh, l0.scheme, l0.strategy, k).dim();
}

/// The reference's own post-processing of a global solution x (length dim):
/// recover_solution (assemble.hpp:58-66) followed by error_norms
/// (errors.hpp:32-117) against the closed-form field of data_kind (1 = the
/// reference's ManufacturedCase, 2 = the sin/cos field above).
/// out = {u, grad_u, p, div_u}; local_out (optional) receives the recovered
/// per-element full local vectors concatenated in element order.
int ref_error_norms(void* sysh, int data_kind, const double* x, double* out, double* local_out) {
  try {
    const System* s = static_cast<System*>(sysh);
    const DofLayout& l = s->sys.layout;
    Eigen::VectorXd xv(l.dim());
    for (Eigen::Index i = 0; i < xv.size(); ++i) xv[i] = x[i];
    const std::vector<Eigen::VectorXd> loc = s->sys.recover_solution(xv);
    ExactFields ex;
    if (data_kind == 1)
      ex = {ManufacturedCase::velocity, ManufacturedCase::velocity_gradient,
            ManufacturedCase::pressure};
    else if (data_kind == 2)
      ex = {SinCosCase::velocity, SinCosCase::grad, SinCosCase::pressure};
    else
      throw std::invalid_argument("error norms need a closed-form field (data 1 or 2)");
    const ErrorNorms e = error_norms(s->mesh, l.scheme, l.k, loc, ex);
    out[0] = e.u;
    out[1] = e.grad_u;
    out[2] = e.p;
    out[3] = e.div_u;
    if (local_out)
      for (const auto& v : loc)
        for (Eigen::Index i = 0; i < v.size(); ++i) *local_out++ = v[i];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

} // extern "C"
