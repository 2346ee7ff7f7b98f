// GMRES / FGMRES (gmres.hpp:38-173) and the p-multilevel hierarchy and
// V-cycle (plevels.hpp:115-239) on device-resident vectors.
//
// Vectors, Krylov bases and operators live in HBM; per Arnoldi step the only
// host traffic is the (j+2)-entry Hessenberg column, because the Givens
// rotations, the convergence test and the small triangular solve run on the
// host with exactly the scalar code order of the reference (std::hypot is
// not reproducible across libm and libdevice, so it stays on the host).
#include <algorithm>
#include <chrono>
#include <exception>
#include <thread>
#include <cstdlib>
#include <cmath>
#include <memory>

#include "internal.cuh"
#include "solver.cuh"
#include "walk.cuh"

namespace pscu {

void mgs_launch(Context& c, int mode, int64_t n, double* w, const double* vp, const double* hprev,
                const double* vi, double* out);
bool arnoldi_step_fused(Context& c, int64_t n, int j, double* w, double* V, int64_t ldv,
                        double* hcol);
void scale_next_launch(Context& c, int64_t n, const double* w, const double* hp, double* v);
void scale_div_launch(Context& c, int64_t n, const double* r, double beta, double* v);
void combine_launch(Context& c, int64_t n, int m, const double* x0, const double* y_dev,
                    const double* z, int64_t ldz, double* x);
void sub_launch(Context& c, int64_t n, const double* a, const double* b, double* r);
void prolong_add_launch(Context& c, int64_t n, const int32_t* f2c, const double* cc, double* w);
void inherit_gather_launch(Context& c, int64_t nnz, const int32_t* src, const double* fine,
                           double* out);

// ---------------------------------------------------------------------------
// host mirror of detail::ArnoldiWorkspace scalars (gmres.hpp:38-92)
// ---------------------------------------------------------------------------

void HostArnoldi::init(int m_, double beta) {
  m = m_;
  h.assign(size_t(m + 1) * size_t(m > 0 ? m : 1), 0.0);
  g.assign(m + 1, 0.0);
  cs.assign(m + 1, 0.0);
  sn.assign(m + 1, 0.0);
  g[0] = beta;
  last_subdiag = 0.0;
}

double HostArnoldi::step(int j, const double* col) {
  for (int i = 0; i <= j + 1; ++i) H(i, j) = col[i];
  last_subdiag = H(j + 1, j);
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * H(i, j) + sn[i] * H(i + 1, j);
    H(i + 1, j) = -sn[i] * H(i, j) + cs[i] * H(i + 1, j);
    H(i, j) = t;
  }
  const double denom = std::hypot(H(j, j), H(j + 1, j));
  cs[j] = denom == 0.0 ? 1.0 : H(j, j) / denom;
  sn[j] = denom == 0.0 ? 0.0 : H(j + 1, j) / denom;
  H(j, j) = denom;
  H(j + 1, j) = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  return std::abs(g[j + 1]);
}

void HostArnoldi::solve_y(int mm, std::vector<double>& y) const {
  y.assign(mm, 0.0);
  for (int i = 0; i < mm; ++i) y[i] = g[i];
  for (int i = mm - 1; i >= 0; --i) {
    double s = y[i];
    for (int jj = i + 1; jj < mm; ++jj) {
      const double t = H(i, jj) * y[jj];
      s = s - t;
    }
    y[i] = s / H(i, i);
  }
}

// ---------------------------------------------------------------------------
// Krylov workspace and the device Arnoldi step
// ---------------------------------------------------------------------------

KrylovWs::~KrylovWs() {
  if (hpin) cudaFreeHost(hpin);
  for (auto& e : hev)
    if (e) cudaEventDestroy(e);
}

void KrylovWs::ensure(int64_t n_, int m_, bool store_z_) {
  if (!hev[0])
    for (auto& e : hev) PSCU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (m_ > hpin_m) {
    if (hpin) PSCU_CUDA(cudaFreeHost(hpin));
    hpin = nullptr;
    PSCU_CUDA(cudaMallocHost(&hpin, sizeof(double) * 2 * size_t(m_ + 2)));
    hpin_m = m_;
  }
  if (hcol.n < 2 * size_t(hpin_m + 2)) hcol.alloc(2 * size_t(hpin_m + 2));
  if (n_ == n && m_ <= m && (!store_z_ || store_z)) return;
  n = n_;
  m = m_;
  store_z = store_z_;
  V.alloc(size_t(m + 1) * size_t(n));
  if (store_z) Z.alloc(size_t(m) * size_t(n));
  w.alloc(n);
  r0.alloc(n);
  tmp.alloc(n);
  prhs.alloc(n);
  xs.alloc(n);
  ydev.alloc(m + 1);
  hcol_host.resize(m + 2);
}

/// ArnoldiWorkspace::step on the device (MGS passes); the Hessenberg
/// column goes to device slot `buf` and, asynchronously, to pinned host
/// slot `buf` (event hev[buf]).
static void arnoldi_launch(Context& c, KrylovWs& ws, int j, int buf) {
  const int64_t n = ws.n;
  double* V = ws.V.p;
  double* hc = ws.hcol.p + size_t(buf) * size_t(ws.hpin_m + 2);
  {
    // algorithmic bytes of a fused MGS step: (j+1) 24 n + 16 n
    Context::Scope prof(&c, PROF_MGS, (double(j + 1) * 24.0 + 16.0) * double(n));
    if (!arnoldi_step_fused(c, n, j, ws.w.p, V, n, hc)) {
      mgs_launch(c, 0, n, ws.w.p, nullptr, nullptr, V, hc + 0);
      for (int i = 1; i <= j; ++i)
        mgs_launch(c, 1, n, ws.w.p, V + size_t(i - 1) * n, hc + (i - 1), V + size_t(i) * n,
                   hc + i);
      mgs_launch(c, 2, n, ws.w.p, V + size_t(j) * n, hc + j, nullptr, hc + j + 1);
      scale_next_launch(c, n, ws.w.p, hc + j + 1, V + size_t(j + 1) * n);
    }
  }
  double* hp = ws.hpin + size_t(buf) * size_t(ws.hpin_m + 2);
  PSCU_CUDA(cudaMemcpyAsync(hp, hc, sizeof(double) * (j + 2), cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaEventRecord(ws.hev[buf], c.stream));
}

/// Host half of the step: Givens rotations on the column of slot `buf`.
static double arnoldi_finish(KrylovWs& ws, HostArnoldi& ar, int j, int buf) {
  PSCU_CUDA(cudaEventSynchronize(ws.hev[buf]));
  return ar.step(j, ws.hpin + size_t(buf) * size_t(ws.hpin_m + 2));
}

static double arnoldi_step(Context& c, KrylovWs& ws, HostArnoldi& ar, int j) {
  arnoldi_launch(c, ws, j, 0);
  return arnoldi_finish(ws, ar, j, 0);
}

static double norm_dev(Context& c, const double* x, int64_t n) {
  return std::sqrt(dot(c, x, x, n));
}

/// x = x0 + Z y (ArnoldiWorkspace::solution) with y from the host.
static void arnoldi_solution(Context& c, KrylovWs& ws, const HostArnoldi& ar, const double* x0,
                             int mm, const double* zbase, double* x) {
  std::vector<double> y;
  ar.solve_y(mm, y);
  if (mm)
    PSCU_CUDA(cudaMemcpyAsync(ws.ydev.p, y.data(), sizeof(double) * mm, cudaMemcpyHostToDevice,
                              c.stream));
  combine_launch(c, ws.n, mm, x0, ws.ydev.p, zbase, ws.n, x);
  // y must outlive the async copy from pageable memory: cudaMemcpyAsync
  // from pageable memory returns after staging, so this is safe.
}

namespace {
struct LeftOp : Op {
  Op* op;
  Op* pc;
  double* tmp;
  LeftOp(Op* o, Op* p, double* t) : op(o), pc(p), tmp(t) {}
  int64_t size() const override { return op->size(); }
  bool pure() const override { return op->pure() && pc->pure(); }
  void apply(Context& c, const double* x, double* y) override {
    op->apply(c, x, tmp);
    pc->apply(c, tmp, y);
  }
};
} // namespace

KrylovResultDev gmres_dev(Context& c, Op& op, Op* pc, const double* rhs, const double* x0,
                          int max_it, double rtol, bool left, double* x, KrylovWs& ws,
                          const double* prhs_cached) {
  const int64_t n = op.size();
  if (left && pc) {
    // gmres.hpp:107-110: run on M^-1 A with rhs M^-1 b, no preconditioner
    ws.ensure(n, max_it, false);
    const double* prhs = prhs_cached;
    if (!prhs) {
      pc->apply(c, rhs, ws.prhs.p);
      prhs = ws.prhs.p;
    }
    LeftOp lop(&op, pc, ws.tmp.p);
    return gmres_dev(c, lop, nullptr, prhs, x0, max_it, rtol, false, x, ws, nullptr);
  }
  ws.ensure(n, max_it, pc != nullptr);
  KrylovResultDev res;
  // r0 = rhs - op(x0); with x0 == 0 the product is +0 in every entry, so
  // r0 = rhs up to the sign of exact zeros.
  if (x0) {
    op.apply(c, x0, ws.r0.p);
    sub_launch(c, n, rhs, ws.r0.p, ws.r0.p);
  } else {
    copy(c, ws.r0.p, rhs, n);
  }
  const double beta = norm_dev(c, ws.r0.p, n);
  if (beta == 0.0) {
    if (x0) {
      if (x != x0) copy(c, x, x0, n);
    } else {
      zero(c, x, n);
    }
    res.converged = true;
    return res;
  }
  HostArnoldi ar;
  ar.init(max_it, beta);
  scale_div_launch(c, n, ws.r0.p, beta, ws.V.p);
  int m = 0;
  // step j's device work (preconditioner, operator, MGS) needs only device
  // data, so step j + 1 is launched before the host reads column j: the host
  // round trip and the launches overlap the device work. A step launched
  // past convergence only writes scratch columns (V, Z, w) never used.
  auto launch_step = [&](int j) {
    const double* vj = ws.V.p + size_t(j) * n;
    const double* zj = vj;
    if (pc) {
      double* zz = ws.Z.p + size_t(j) * n;
      pc->apply(c, vj, zz);
      zj = zz;
    }
    op.apply(c, zj, ws.w.p);
    arnoldi_launch(c, ws, j, j & 1);
  };
  const bool ahead = op.pure() && (!pc || pc->pure());
  if (max_it > 0 && ahead) launch_step(0);
  for (int j = 0; j < max_it; ++j) {
    if (!ahead) launch_step(j);
    else if (j + 1 < max_it) launch_step(j + 1);
    const double est = arnoldi_finish(ws, ar, j, j & 1);
    m = j + 1;
    res.rel_residual = est / beta;
    if (est <= rtol * beta) {
      res.converged = true;
      break;
    }
    if (ar.last_subdiag == 0.0) {
      res.converged = true;
      break;
    }
  }
  res.iterations = m;
  arnoldi_solution(c, ws, ar, x0, m, pc ? ws.Z.p : ws.V.p, ws.xs.p);
  copy(c, x, ws.xs.p, n);
  return res;
}

KrylovResultDev fgmres_dev(Context& c, Op& op, Op& pc, const double* rhs, int max_it, double rtol,
                           int restart, double* x, KrylovWs& ws, std::vector<double>* hist) {
  const int64_t n = op.size();
  KrylovResultDev res;
  const double bnorm = norm_dev(c, rhs, n);
  if (bnorm == 0.0) {
    zero(c, x, n);
    res.converged = true;
    return res;
  }
  const int cycle = restart > 0 ? restart : max_it;
  ws.ensure(n, cycle, true);
  DevBuf<double> x0buf(n);
  bool have_x0 = false;
  copy(c, ws.r0.p, rhs, n);
  double beta = bnorm;
  int total = 0;
  while (true) {
    const int mm = std::min(cycle, max_it - total);
    HostArnoldi ar;
    ar.init(mm, beta);
    scale_div_launch(c, n, ws.r0.p, beta, ws.V.p);
    bool restart_now = false;
    for (int j = 0; j < mm; ++j) {
      double* zj = ws.Z.p + size_t(j) * n;
      pc.apply(c, ws.V.p + size_t(j) * n, zj);
      op.apply(c, zj, ws.w.p);
      const double est = arnoldi_step(c, ws, ar, j);
      ++total;
      if (hist) hist->push_back(est / bnorm);
      const int m = j + 1;
      const bool last = total == max_it;
      if (est <= rtol * bnorm || ar.last_subdiag == 0.0 || last) {
        arnoldi_solution(c, ws, ar, have_x0 ? x0buf.p : nullptr, m, ws.Z.p, x);
        op.apply(c, x, ws.tmp.p);
        sub_launch(c, n, rhs, ws.tmp.p, ws.tmp.p);
        res.rel_residual = norm_dev(c, ws.tmp.p, n) / bnorm;
        res.iterations = total;
        if (res.rel_residual <= rtol) {
          res.converged = true;
          return res;
        }
        if (last) return res;
        if (j + 1 == mm) {
          restart_now = true;
          copy(c, x0buf.p, x, n);
          have_x0 = true;
        }
      } else if (j + 1 == mm) {
        restart_now = true;
        arnoldi_solution(c, ws, ar, have_x0 ? x0buf.p : nullptr, m, ws.Z.p, ws.xs.p);
        copy(c, x0buf.p, ws.xs.p, n);
        have_x0 = true;
      }
    }
    if (!restart_now) return res;
    op.apply(c, x0buf.p, ws.tmp.p);
    sub_launch(c, n, rhs, ws.tmp.p, ws.r0.p);
    beta = norm_dev(c, ws.r0.p, n);
  }
}

// ---------------------------------------------------------------------------
// hierarchy
// ---------------------------------------------------------------------------

int64_t layout_dim(const pscu_layout& l) {
  return int64_t(l.n_faces) * (ncomp(l) * l.face_vel + l.face_press) +
         int64_t(l.n_elements) * (ncomp(l) * l.elem_vel + l.elem_press);
}

void make_layout3(int scheme, int strategy, int k, int n_faces, int n_elements, pscu_layout& l) {
  if (k < 0) throw Error(PSCU_EINVAL, "layout: k must be >= 0");
  if (scheme == 2) {
    // DG (config 4): element blocks [ux | uy | uz | p], dim P^k(3D) modes
    // each (dof_layout.hpp:118-123 with three components)
    if (k < 1) throw Error(PSCU_EINVAL, "dg: k must be >= 1");
    if (strategy != 0) throw Error(PSCU_EINVAL, "dg: no static condensation exists, use uncond");
  } else if (scheme != 1 || strategy != 2) {
    throw Error(PSCU_EINVAL, "3D layout: hho-hp vp-cond or dg uncond only");
  }
  l = pscu_layout{};
  l.scheme = scheme;
  l.strategy = strategy;
  l.k = k;
  l.n_faces = n_faces;
  l.n_elements = n_elements;
  if (scheme == 2) l.elem_vel = l.elem_press = (k + 1) * (k + 2) * (k + 3) / 6;
  else l.face_vel = l.face_press = (k + 1) * (k + 2) / 2;
  l.dim = 3;
}

void layout_at(const pscu_layout& lf, int k, pscu_layout& out) {
  if (lf.dim == 3) make_layout3(lf.scheme, lf.strategy, k, lf.n_faces, lf.n_elements, out);
  else make_layout(lf.scheme, lf.strategy, k, lf.n_faces, lf.n_elements, out);
}

void make_layout(int scheme, int strategy, int k, int n_faces, int n_elements, pscu_layout& l) {
  if (k < 0) throw Error(PSCU_EINVAL, "layout: k must be >= 0");
  l = pscu_layout{};
  l.scheme = scheme;
  l.strategy = strategy;
  l.k = k;
  l.n_faces = n_faces;
  l.n_elements = n_elements;
  l.dim = 2;
  const int nf = k + 1, np = (k + 1) * (k + 2) / 2;
  const int ke = scheme == 1 ? k + 1 : k;
  const int ne = (ke + 1) * (ke + 2) / 2;
  switch (scheme) {
    case 0:
      l.face_vel = nf;
      if (strategy == 0) {
        l.elem_vel = ne;
        l.elem_press = np;
      } else if (strategy == 1) {
        l.elem_press = np;
      } else {
        l.elem_press = 1;
      }
      break;
    case 1:
      l.face_vel = nf;
      l.face_press = nf;
      if (strategy == 0) {
        l.elem_vel = ne;
        l.elem_press = np;
      } else if (strategy == 1) {
        throw Error(PSCU_EINVAL, "hho-hp: supported strategies are uncond and vp-cond");
      }
      break;
    case 2:
      if (k < 1) throw Error(PSCU_EINVAL, "dg: k must be >= 1");
      if (strategy != 0) throw Error(PSCU_EINVAL, "dg: no static condensation exists, use uncond");
      l.elem_vel = ne;
      l.elem_press = np;
      break;
    default:
      throw Error(PSCU_EINVAL, "unknown scheme");
  }
}

void coarse_to_fine(const pscu_layout& f, const pscu_layout& c, int64_t* map) {
  if (f.n_faces != c.n_faces || f.n_elements != c.n_elements)
    throw Error(PSCU_EINVAL, "transfer: layouts live on different meshes");
  if (c.face_vel > f.face_vel || c.face_press > f.face_press || c.elem_vel > f.elem_vel ||
      c.elem_press > f.elem_press)
    throw Error(PSCU_EINVAL, "transfer: coarse layout is not nested in the fine one");
  if (ncomp(c) != ncomp(f)) throw Error(PSCU_EINVAL, "transfer: layouts of different dimension");
  const int nc = ncomp(c);
  const int64_t cfb = nc * c.face_vel + c.face_press, ffb = nc * f.face_vel + f.face_press;
  const int64_t ceb = nc * c.elem_vel + c.elem_press, feb = nc * f.elem_vel + f.elem_press;
  for (int64_t fc = 0; fc < c.n_faces; ++fc) {
    const int64_t cb = fc * cfb, fb = fc * ffb;
    for (int comp = 0; comp < nc; ++comp)
      for (int m = 0; m < c.face_vel; ++m) map[cb + comp * c.face_vel + m] = fb + comp * f.face_vel + m;
    for (int m = 0; m < c.face_press; ++m) map[cb + nc * c.face_vel + m] = fb + nc * f.face_vel + m;
  }
  const int64_t co = int64_t(c.n_faces) * cfb, fo = int64_t(f.n_faces) * ffb;
  for (int64_t e = 0; e < c.n_elements; ++e) {
    const int64_t cb = co + e * ceb, fb = fo + e * feb;
    for (int comp = 0; comp < nc; ++comp)
      for (int m = 0; m < c.elem_vel; ++m) map[cb + comp * c.elem_vel + m] = fb + comp * f.elem_vel + m;
    for (int m = 0; m < c.elem_press; ++m) map[cb + nc * c.elem_vel + m] = fb + nc * f.elem_vel + m;
  }
}

/// inherit_matrix (plevels.hpp:93-113): the coarse pattern and the source
/// position of every coarse entry come from the host copy of the fine
/// pattern (setup bookkeeping); the values are gathered on the device.
/// Runs f(lo, hi) over [0, n) in parallel host threads.
template <typename F>
static void parallel_ranges(int64_t n, F f) {
  const int nth = int(std::max<int64_t>(1, std::min<int64_t>(
      std::min(16u, std::max(1u, std::thread::hardware_concurrency())), n / 65536)));
  std::vector<std::thread> th;
  for (int t = 1; t < nth; ++t) th.emplace_back([&, t] { f(n * t / nth, n * (t + 1) / nth); });
  f(0, n / nth);
  for (auto& x : th) x.join();
}

/// inherit_matrix (plevels.hpp:93-113): the coarse pattern and the source
/// position of every coarse entry on the host (row-parallel: count, prefix,
/// fill), then the value gather on the device.
void inherit(Context& c, const Csr& fine, const std::vector<int64_t>& c2f, Csr& out) {
  const int64_t nf = fine.n, nc = int64_t(c2f.size());
  std::vector<int64_t> f2c(nf, -1);
  for (int64_t i = 0; i < nc; ++i) f2c[c2f[i]] = i;
  out.n = nc;
  out.h_row_ptr.assign(nc + 1, 0);
  parallel_ranges(nc, [&](int64_t lo, int64_t hi) {
    for (int64_t ic = lo; ic < hi; ++ic) {
      const int64_t r = c2f[ic];
      int64_t k = 0;
      for (int64_t p = fine.h_row_ptr[r]; p < fine.h_row_ptr[r + 1]; ++p) k += f2c[fine.h_cols[p]] >= 0;
      out.h_row_ptr[ic + 1] = k;
    }
  });
  for (int64_t ic = 0; ic < nc; ++ic) out.h_row_ptr[ic + 1] += out.h_row_ptr[ic];
  out.nnz = out.h_row_ptr[nc];
  out.h_cols.resize(size_t(out.nnz));
  if (fine.nnz >= (int64_t(1) << 31))
    throw Error(PSCU_EINVAL, "inherit: more than 2^31 fine entries are not supported");
  std::vector<int32_t> src(size_t(out.nnz));
  parallel_ranges(nc, [&](int64_t lo, int64_t hi) {
    for (int64_t ic = lo; ic < hi; ++ic) {
      const int64_t r = c2f[ic];
      int64_t k = out.h_row_ptr[ic];
      for (int64_t p = fine.h_row_ptr[r]; p < fine.h_row_ptr[r + 1]; ++p) {
        const int64_t jc = f2c[fine.h_cols[p]];
        if (jc >= 0) {
          out.h_cols[k] = int32_t(jc);
          src[k++] = int32_t(p);
        }
      }
    }
  });
  out.row_ptr.upload(out.h_row_ptr, c.stream);
  out.cols.upload(out.h_cols, c.stream);
  out.vals.alloc(out.nnz);
  DevBuf<int32_t> dsrc;
  dsrc.upload(src, c.stream);
  inherit_gather_launch(c, out.nnz, dsrc.p, fine.vals.p, out.vals.p);
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
}

struct SpmvOp : Op {
  const Csr* a;
  explicit SpmvOp(const Csr* m) : a(m) {}
  int64_t size() const override { return a->n; }
  void apply(Context& c, const double* x, double* y) override { spmv(c, *a, x, y); }
};

struct IluOp : Op {
  const Ilu* ilu;
  explicit IluOp(const Ilu* p) : ilu(p) {}
  int64_t size() const override { return ilu->a->n; }
  void apply(Context& c, const double* x, double* y) override { ilu0_apply(c, *ilu, x, y); }
};
struct BjOp : Op {
  const BlockJacobi* bj;
  explicit BjOp(const BlockJacobi* p) : bj(p) {}
  int64_t size() const override { return bj->n; }
  void apply(Context& c, const double* x, double* y) override { bj_apply(c, *bj, x, y); }
};

Hierarchy::~Hierarchy() = default;

void Hierarchy::build(Context& c, const Csr* fine, const pscu_layout& lf, const int* degrees,
                      int nlev, const pscu_level_cfg& cfg_) {
  cfg = cfg_;
  if (nlev < 1 || degrees[0] != lf.k)
    throw Error(PSCU_EINVAL, "hierarchy: level degrees must start at the fine degree");
  for (int i = 1; i < nlev; ++i)
    if (degrees[i] >= degrees[i - 1])
      throw Error(PSCU_EINVAL, "hierarchy: level degrees must strictly decrease");
  const int kmin = lf.scheme == 2 ? 1 : 0;
  if (degrees[nlev - 1] < kmin)
    throw Error(PSCU_EINVAL, "hierarchy: coarsest degree below the scheme minimum");
  if (cfg.smoother != PSCU_SMOOTHER_ILU0 && cfg.smoother != PSCU_SMOOTHER_BJACOBI)
    throw Error(PSCU_EINVAL, "hierarchy: unknown smoother");
  if (cfg.coarse != PSCU_COARSE_ILU_GMRES && nlev > 0 && cfg.coarse != PSCU_COARSE_LU)
    throw Error(PSCU_EINVAL, "hierarchy: unknown coarse solver");
  levels.clear();
  levels.resize(nlev);
  for (int l = 0; l < nlev; ++l) levels[l] = std::make_unique<Level>();
  levels[0]->k = degrees[0];
  levels[0]->layout = lf;
  levels[0]->a = fine;
  levels[0]->op = fine;
  for (int l = 1; l < nlev; ++l) {
    Level& L = *levels[l];
    Level& P = *levels[l - 1];
    L.k = degrees[l];
    layout_at(lf, degrees[l], L.layout);
    std::vector<int64_t> c2f(layout_dim(L.layout));
    coarse_to_fine(P.layout, L.layout, c2f.data());
    P.nc = int64_t(c2f.size());
    P.down_map.upload(c2f, c.stream);
    std::vector<int32_t> f2c(P.a->n, -1);
    for (int64_t i = 0; i < P.nc; ++i) f2c[c2f[i]] = int32_t(i);
    P.f2c.upload(f2c, c.stream);
    const auto t0 = std::chrono::steady_clock::now();
    if (P.op->dgm) {
      // DG block storage: the coarse panels are the leading modes of the
      // fine ones (element e's coarse dofs map into element e's fine block)
      if (L.layout.scheme != 2 || L.layout.dim != 3 || L.layout.elem_vel != L.layout.elem_press)
        throw Error(PSCU_EINVAL, "hierarchy: DG block storage needs 3D dg layouts");
      const bool needs_csr = (l + 1 == nlev) || cfg.smoother != PSCU_SMOOTHER_BJACOBI;
      if (needs_csr) {
        inherit_dgb(c, *P.op, L.layout.elem_vel, L.own_bsr);
        dgb_to_csr(c, L.own_bsr, L.own);
        L.op = &L.own_bsr;
        PSCU_CUDA(cudaStreamSynchronize(c.stream));
      } else {
        inherit_dgb(c, *P.op, L.layout.elem_vel, L.own);
      }
    } else if (P.op->bs) {
      // face-block operators: the coarse blocks are sub-blocks of the fine
      // ones (face f's coarse dofs map into face f's fine block)
      const int fbc = ncomp(L.layout) * L.layout.face_vel + L.layout.face_press;
      if (L.layout.elem_vel || L.layout.elem_press || P.layout.elem_vel || P.layout.elem_press)
        throw Error(PSCU_EINVAL, "hierarchy: block storage needs face-only layouts");
      std::vector<int32_t> in_block(fbc);
      for (int j = 0; j < fbc; ++j) in_block[j] = int32_t(c2f[j]);
      const bool needs_csr = (l + 1 == nlev) || cfg.smoother != PSCU_SMOOTHER_BJACOBI;
      if (needs_csr) {
        inherit_bsr(c, *P.op, in_block, L.own_bsr);
        bsr_to_csr(c, L.own_bsr, L.own);
        L.op = &L.own_bsr;
        PSCU_CUDA(cudaStreamSynchronize(c.stream));
      } else {
        inherit_bsr(c, *P.op, in_block, L.own);
      }
    } else {
      inherit(c, *P.a, c2f, L.own);
    }
    L.a = &L.own;
    if (!L.op) L.op = &L.own;
    if (getenv("PSCU_DEBUG"))
      fprintf(stderr, "[setup] inherit level %d: %.3f s\n", l,
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  // ILU(0) levels: factorisation launches first (device), then the sweep
  // plans of all levels in parallel host threads, then uploads and checks
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<int> ilu_levels;
  for (int l = 0; l < nlev; ++l) {
    Level& L = *levels[l];
    const bool wants_csr = (l + 1 == nlev) || cfg.smoother != PSCU_SMOOTHER_BJACOBI;
    if (L.a->bs && wants_csr) {
      // ILU(0) / dense LU work on CSR storage: a private CSR copy (the block
      // storage stays the operator of the level's SpMVs)
      if (L.a == &L.own) {
        L.own_bsr = std::move(L.own);
        L.op = &L.own_bsr;
        bsr_to_csr(c, L.own_bsr, L.own);
      } else {
        bsr_to_csr(c, *L.a, L.own);
      }
      PSCU_CUDA(cudaStreamSynchronize(c.stream));
      L.a = &L.own;
    }
    if (l + 1 == nlev && cfg.coarse == PSCU_COARSE_LU) {
      L.dense_lu.factor(c, *L.a);
    } else if (l + 1 < nlev && cfg.smoother == PSCU_SMOOTHER_BJACOBI) {
      L.use_bj = true;
      bj_factor(c, *L.a, L.layout, L.bj);
    } else {
      L.ilu.a = L.a;
      ilu0_factor_start(c, L.ilu);
      ilu_levels.push_back(l);
    }
  }
  {
    std::vector<std::shared_ptr<WalkBuild>> plans(ilu_levels.size());
    std::vector<std::exception_ptr> errs(ilu_levels.size());
    std::vector<std::thread> th;
    for (size_t k = 0; k < ilu_levels.size(); ++k)
      th.emplace_back([&, k] {
        try {
          const Level& L = *levels[ilu_levels[k]];
          plans[k] = plan_walk(*L.a, L.ilu.h_diag);
        } catch (...) {
          errs[k] = std::current_exception();
        }
      });
    for (auto& t : th) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    if (getenv("PSCU_DEBUG"))
      fprintf(stderr, "[setup] factor launches + sweep plans: %.3f s\n",
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    for (size_t k = 0; k < ilu_levels.size(); ++k) {
      Level& L = *levels[ilu_levels[k]];
      upload_walk(c, *L.a, *plans[k], L.ilu.wfwd, L.ilu.wbwd);
      plans[k].reset();
      ilu0_factor_finish(c, L.ilu);
    }
    if (getenv("PSCU_DEBUG"))
      fprintf(stderr, "[setup] ILU levels ready: %.3f s\n",
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  for (int l = 0; l < nlev; ++l) {
    Level& L = *levels[l];
    const bool bottom = l + 1 == nlev;
    const int64_t n = L.a->n;
    L.w.alloc(n);
    if (!bottom) {
      L.dc.alloc(P_nc(l));
      L.cc.alloc(P_nc(l));
    }
  }
  coarse_its = 0;
}

int64_t Hierarchy::P_nc(int l) const { return levels[l]->nc; }

void Hierarchy::coarse_solve(Context& c, const double* d, double* out) {
  Level& B = *levels.back();
  if (cfg.coarse == PSCU_COARSE_LU) {
    coarse_its += 1;
    B.dense_lu.solve(c, d, out);
    return;
  }
  SpmvOp op(B.op);
  IluOp pc(&B.ilu);
  const KrylovResultDev r = gmres_dev(c, op, &pc, d, nullptr, cfg.coarse_maxit, cfg.coarse_rtol,
                                      false, out, B.ws, nullptr);
  coarse_its += r.iterations;
}

void Hierarchy::vcycle(Context& c, int l, const double* d, double* out) {
  if (l + 1 == int(levels.size())) {
    coarse_solve(c, d, out);
    return;
  }
  Level& L = *levels[l];
  SpmvOp op(L.op);
  IluOp ilu_pc(&L.ilu);
  BjOp bj_pc(&L.bj);
  Op& pc = L.use_bj ? static_cast<Op&>(bj_pc) : static_cast<Op&>(ilu_pc);
  const int s = cfg.smoother_iters;
  // pre-smoothing from zero: gmres(op, pc, d, 0, s, 0, Left) (plevels.hpp:175-176)
  gmres_dev(c, op, &pc, d, nullptr, s, 0.0, true, L.w.p, L.ws, nullptr);
  // d_coarse = restrict(d - A w)
  residual_restrict(c, *L.op, d, L.w.p, L.down_map.p, L.nc, L.dc.p);
  vcycle(c, l + 1, L.dc.p, L.cc.p);
  // w += prolong(c)
  prolong_add_launch(c, L.a->n, L.f2c.p, L.cc.p, L.w.p);
  // post-smoothing from w; M^-1 d is unchanged since pre-smoothing
  gmres_dev(c, op, &pc, d, L.w.p, s, 0.0, true, out, L.ws, L.ws.prhs.p);
}

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------

namespace {

__global__ void prolong_add(int64_t n, const int32_t* __restrict__ f2c,
                            const double* __restrict__ cc, double* __restrict__ w) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int32_t i = f2c[e];
    w[e] = dadd(w[e], i >= 0 ? cc[i] : 0.0);
  }
}

__global__ void gather_kernel(int64_t nnz, const int32_t* __restrict__ src,
                              const double* __restrict__ fine, double* __restrict__ out) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nnz;
       q += int64_t(gridDim.x) * blockDim.x)
    out[q] = fine[src[q]];
}

unsigned grid1d(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return unsigned(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

} // namespace

void prolong_add_launch(Context& c, int64_t n, const int32_t* f2c, const double* cc, double* w) {
  prolong_add<<<grid1d(n), 256, 0, c.stream>>>(n, f2c, cc, w);
  PSCU_LAUNCHED(&c);
}

void inherit_gather_launch(Context& c, int64_t nnz, const int32_t* src, const double* fine,
                           double* out) {
  if (!nnz) return;
  gather_kernel<<<grid1d(nnz), 256, 0, c.stream>>>(nnz, src, fine, out);
  PSCU_LAUNCHED(&c);
}

} // namespace pscu
