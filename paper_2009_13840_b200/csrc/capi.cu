// extern "C" entry points of include/pstokes_cuda.h.
#include <chrono>
#include <cstring>
#include <memory>

#include "internal.cuh"
#include "solver.cuh"

namespace pscu {
void condense_batch(Context& c, int nelem, int n, const double* mats, const double* rhs, int ne,
                    const int* elim_host, double* schur, double* rrhs, double* coupling,
                    double* erhs, int* bad_element);
void recover_batch(Context& c, int nelem, int n, int ne, const int* elim_host,
                   const int64_t* kept, const double* coupling, const double* erhs,
                   const double* x, double* locals);
void assemble_values(Context& c, int nelem, int nk, const int64_t* kept, const double* schur,
                     const double* rrhs, const pscu_layout& l, Csr& a, double* rhs);
void condense_scatter_bsr(Context& c, Csr& a, int e0, int nelem, int n, const double* mats,
                          const double* rhs, int ne, const int* elim_host, const int32_t* efaces,
                          const int32_t* erows, int nfe, const int32_t* keep_pos_host,
                          double* rhs_acc, double* coupling, double* erhs);
void error_accumulate(Context& c, const int32_t* dims, int nelem, const double* tables,
                      const double* locals, double* acc);
void local_blocks3(Context& c, int k, int data, double eta, int nq1, const double* glx,
                   const double* glw, const double* xyz, const int32_t* hex, const int32_t* ef,
                   const int32_t* es, const int32_t* ftab, const double* coef, int e0, int nelem,
                   double* mats, double* rhs);

Context::~Context() {
  for (auto e : ev_pool) cudaEventDestroy(e);
  if (t_start) cudaEventDestroy(t_start);
  if (t_stop) cudaEventDestroy(t_stop);
  if (h_pinned) cudaFreeHost(h_pinned);
  if (stream) cudaStreamDestroy(stream);
}
} // namespace pscu

using namespace pscu;

struct pscu_ctx {
  Context c;
};
struct pscu_mat {
  Csr m;                     // first member: hierarchy levels are viewed as pscu_mat
  DevBuf<double> rhs_acc;    // reduced load of a streamed assembly (pscu_assembly_*)
};
struct pscu_ilu {
  Ilu i;
  Csr own;  // CSR copy of a block-stored operator (ILU(0) works on CSR)
};
struct pscu_bj {
  BlockJacobi b;
};
struct pscu_hier {
  Hierarchy h;
  const pscu_mat* fine = nullptr;
  std::vector<pscu_mat> level_views;  // not used for level 0
  KrylovWs outer;
};

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (auto* pe = dynamic_cast<const Error*>(&e)) return pe->code;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return PSCU_EINVAL;
  return PSCU_ECUDA;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return PSCU_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

/// Device view of a possibly-host vector: uploads into `buf` when needed.
const double* in_vec(Context& c, const double* p, int64_t n, int mem, DevBuf<double>& buf) {
  if (mem == PSCU_DEVICE) return p;
  buf.alloc(n > 0 ? n : 1);
  if (n) PSCU_CUDA(cudaMemcpyAsync(buf.p, p, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
  return buf.p;
}

double* out_vec(int64_t n, double* p, int mem, DevBuf<double>& buf) {
  if (mem == PSCU_DEVICE) return p;
  buf.alloc(n > 0 ? n : 1);
  return buf.p;
}

void finish_out(Context& c, double* host, const double* dev, int64_t n, int mem) {
  if (mem == PSCU_HOST && n)
    PSCU_CUDA(cudaMemcpyAsync(host, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
}

struct SpmvOpC : Op {
  const Csr* a;
  explicit SpmvOpC(const Csr* m) : a(m) {}
  int64_t size() const override { return a->n; }
  void apply(Context& c, const double* x, double* y) override { spmv(c, *a, x, y); }
};
struct IluOpC : Op {
  const Ilu* p;
  explicit IluOpC(const Ilu* i) : p(i) {}
  int64_t size() const override { return p->a->n; }
  void apply(Context& c, const double* x, double* y) override { ilu0_apply(c, *p, x, y); }
};
struct IdOp : Op {
  int64_t n;
  explicit IdOp(int64_t m) : n(m) {}
  int64_t size() const override { return n; }
  void apply(Context& c, const double* x, double* y) override { copy(c, y, x, n); }
};
struct VcycleOp : Op {
  Hierarchy* h;
  int64_t n;
  int count = 0;
  VcycleOp(Hierarchy* hh, int64_t m) : h(hh), n(m) {}
  int64_t size() const override { return n; }
  bool pure() const override { return false; }
  void apply(Context& c, const double* x, double* y) override {
    ++count;
    h->vcycle(c, 0, x, y);
  }
};

} // namespace

extern "C" {

const char* pscu_last_error(void) { return g_err.c_str(); }
int pscu_version(void) { return 1; }

int pscu_create(int device, pscu_ctx** out) {
  return guard([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(PSCU_ENODEV, "pscu_create: no CUDA device visible");
    if (device < 0 || device >= ndev) throw Error(PSCU_ENODEV, "pscu_create: bad device ordinal");
    cudaDeviceProp prop{};
    PSCU_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw Error(PSCU_ENODEV, "pscu_create: this build targets sm_100a (B200); device is sm_" +
                                   std::to_string(prop.major) + std::to_string(prop.minor));
    PSCU_CUDA(cudaSetDevice(device));
    auto ctx = std::make_unique<pscu_ctx>();
    Context& c = ctx->c;
    c.device = device;
    PSCU_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    c.red_partials.alloc(1 << 12);
    c.red_counter.alloc(2);  // [0] last-CTA counter / barrier count, [1] barrier generation
    PSCU_CUDA(cudaMemset(c.red_counter.p, 0, 2 * sizeof(unsigned)));
    c.scal.alloc(64);
    c.err_flag.alloc(1);
    PSCU_CUDA(cudaMallocHost(&c.h_pinned, sizeof(double) * 64));
    *out = ctx.release();
  });
}

int pscu_create_devices(const int* devices, int ndev, pscu_ctx** out) {
  if (!devices || !out || ndev < 1)
    return guard([] { throw Error(PSCU_EINVAL, "pscu_create_devices: empty device list"); });
  for (int i = 0; i < ndev; ++i) out[i] = nullptr;
  for (int i = 0; i < ndev; ++i) {
    for (int j = 0; j < i; ++j)
      if (devices[j] == devices[i]) {
        for (int q = 0; q < i; ++q) pscu_destroy(out[q]), out[q] = nullptr;
        return guard([] { throw Error(PSCU_EINVAL, "pscu_create_devices: device listed twice"); });
      }
    const int rc = pscu_create(devices[i], &out[i]);
    if (rc != PSCU_OK) {
      for (int q = 0; q < i; ++q) pscu_destroy(out[q]), out[q] = nullptr;
      return rc;  // pscu_last_error() holds pscu_create's message
    }
  }
  return PSCU_OK;
}

int pscu_destroy(pscu_ctx* ctx) {
  return guard([&] {
    if (ctx) {
      cudaSetDevice(ctx->c.device);
      cudaStreamSynchronize(ctx->c.stream);
      delete ctx;
    }
  });
}

int pscu_synchronize(pscu_ctx* ctx) {
  return guard([&] { PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream)); });
}

long long pscu_launch_count(const pscu_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int pscu_timer_start(pscu_ctx* ctx) {
  return guard([&] {
    Context& c = ctx->c;
    if (!c.t_start) {
      PSCU_CUDA(cudaEventCreate(&c.t_start));
      PSCU_CUDA(cudaEventCreate(&c.t_stop));
    }
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
    PSCU_CUDA(cudaEventRecord(c.t_start, c.stream));
  });
}

int pscu_timer_stop(pscu_ctx* ctx, double* ms) {
  return guard([&] {
    Context& c = ctx->c;
    PSCU_CUDA(cudaEventRecord(c.t_stop, c.stream));
    PSCU_CUDA(cudaEventSynchronize(c.t_stop));
    float f = 0.f;
    PSCU_CUDA(cudaEventElapsedTime(&f, c.t_start, c.t_stop));
    *ms = f;
  });
}

int pscu_profile(pscu_ctx* ctx, int enable) {
  return guard([&] {
    Context& c = ctx->c;
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
    c.profiling = enable != 0;
    c.prof.clear();
    c.ev_used = 0;
  });
}

int pscu_profile_read(pscu_ctx* ctx, int cls, long long* count, double* ms, double* bytes) {
  return guard([&] {
    Context& c = ctx->c;
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
    long long k = 0;
    double t = 0.0, b = 0.0;
    for (const ProfRec& r : c.prof) {
      if (r.cls != cls) continue;
      float f = 0.f;
      PSCU_CUDA(cudaEventElapsedTime(&f, r.e0, r.e1));
      t += f;
      b += r.bytes;
      ++k;
    }
    *count = k;
    *ms = t;
    *bytes = b;
  });
}

int pscu_mat_create(pscu_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* cols,
                    const double* vals, int mem, pscu_mat** out) {
  return guard([&] {
    if (n < 0) throw Error(PSCU_EINVAL, "pscu_mat_create: negative dimension");
    auto m = std::make_unique<pscu_mat>();
    upload_csr(ctx->c, m->m, n, row_ptr, cols, vals, mem);
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *out = m.release();
  });
}

int pscu_mat_destroy(pscu_mat* m) {
  delete m;
  return PSCU_OK;
}

int pscu_mat_dims(const pscu_mat* m, int64_t* n, int64_t* nnz) {
  *n = m->m.n;
  *nnz = m->m.nnz;
  return PSCU_OK;
}

int pscu_mat_download(pscu_ctx* ctx, const pscu_mat* mm, int64_t* row_ptr, int32_t* cols,
                      double* vals) {
  return guard([&] {
    Context& c = ctx->c;
    Csr expanded;
    if (mm->m.bs) bsr_to_csr(c, mm->m, expanded);  // CSR view of block storage
    struct {
      const Csr& m;
    } view{mm->m.bs ? expanded : mm->m};
    const auto* m = &view;
    if (row_ptr)
      PSCU_CUDA(cudaMemcpyAsync(row_ptr, m->m.row_ptr.p, sizeof(int64_t) * (m->m.n + 1),
                                cudaMemcpyDeviceToHost, c.stream));
    if (cols && m->m.nnz)
      PSCU_CUDA(cudaMemcpyAsync(cols, m->m.cols.p, sizeof(int32_t) * m->m.nnz,
                                cudaMemcpyDeviceToHost, c.stream));
    if (vals && m->m.nnz)
      PSCU_CUDA(cudaMemcpyAsync(vals, m->m.vals.p, sizeof(double) * m->m.nnz,
                                cudaMemcpyDeviceToHost, c.stream));
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int pscu_spmv(pscu_ctx* ctx, const pscu_mat* a, const double* x, double* y, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    DevBuf<double> bx, by;
    // a shard's input spans its ghost block columns too
    const int64_t nx = a->m.bs ? a->m.ncb * a->m.bs : a->m.n;
    const double* dx = in_vec(c, x, nx, mem, bx);
    double* dy = out_vec(a->m.n, y, mem, by);
    spmv(c, a->m, dx, dy);
    finish_out(c, y, dy, a->m.n, mem);
  });
}

int pscu_ilu0_create(pscu_ctx* ctx, const pscu_mat* a, pscu_ilu** out) {
  return guard([&] {
    auto p = std::make_unique<pscu_ilu>();
    p->i.a = &a->m;
    if (a->m.bs) {
      bsr_to_csr(ctx->c, a->m, p->own);
      p->i.a = &p->own;
    }
    ilu0_factor(ctx->c, p->i);
    *out = p.release();
  });
}

int pscu_ilu0_destroy(pscu_ilu* p) {
  delete p;
  return PSCU_OK;
}

int pscu_ilu0_factors(pscu_ctx* ctx, const pscu_ilu* p, double* lu_host) {
  return guard([&] {
    const int64_t nnz = p->i.a->nnz;
    if (nnz)
      PSCU_CUDA(cudaMemcpyAsync(lu_host, p->i.lu.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost,
                                ctx->c.stream));
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int pscu_ilu0_apply(pscu_ctx* ctx, const pscu_ilu* p, const double* x, double* y, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    const int64_t n = p->i.a->n;
    DevBuf<double> bx, by;
    const double* dx = in_vec(c, x, n, mem, bx);
    double* dy = out_vec(n, y, mem, by);
    ilu0_apply(c, p->i, dx, dy);
    finish_out(c, y, dy, n, mem);
  });
}

int pscu_bj_create(pscu_ctx* ctx, const pscu_mat* a, const pscu_layout* l, pscu_bj** out) {
  return guard([&] {
    auto p = std::make_unique<pscu_bj>();
    bj_factor(ctx->c, a->m, *l, p->b);
    *out = p.release();
  });
}

int pscu_bj_destroy(pscu_bj* p) {
  delete p;
  return PSCU_OK;
}

int pscu_bj_apply(pscu_ctx* ctx, const pscu_bj* p, const double* x, double* y, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    const int64_t n = p->b.n;
    DevBuf<double> bx, by;
    const double* dx = in_vec(c, x, n, mem, bx);
    double* dy = out_vec(n, y, mem, by);
    bj_apply(c, p->b, dx, dy);
    finish_out(c, y, dy, n, mem);
  });
}

int pscu_layout_make(int scheme, int strategy, int k, int n_faces, int n_elements,
                     pscu_layout* out) {
  return guard([&] { make_layout(scheme, strategy, k, n_faces, n_elements, *out); });
}

int pscu_layout_make3(int scheme, int strategy, int k, int n_faces, int n_elements,
                      pscu_layout* out) {
  return guard([&] { make_layout3(scheme, strategy, k, n_faces, n_elements, *out); });
}

int64_t pscu_layout_dim(const pscu_layout* l) { return layout_dim(*l); }

int pscu_coarse_to_fine(const pscu_layout* fine, const pscu_layout* coarse, int64_t* map) {
  return guard([&] { coarse_to_fine(*fine, *coarse, map); });
}

int pscu_inherit(pscu_ctx* ctx, const pscu_mat* fine, const pscu_layout* lf,
                 const pscu_layout* lc, pscu_mat** out) {
  return guard([&] {
    if (layout_dim(*lf) != fine->m.n)
      throw Error(PSCU_EINVAL, "inherit: fine layout does not match the matrix");
    std::vector<int64_t> c2f(layout_dim(*lc));
    coarse_to_fine(*lf, *lc, c2f.data());
    auto m = std::make_unique<pscu_mat>();
    if (fine->m.dgm) {
      if (lc->scheme != 2 || lc->dim != 3) throw Error(PSCU_EINVAL, "inherit: DG block storage needs 3D dg layouts");
      inherit_dgb(ctx->c, fine->m, lc->elem_vel, m->m);
    } else if (fine->m.bs) {
      const int fbc = ncomp(*lc) * lc->face_vel + lc->face_press;
      if (lc->elem_vel || lc->elem_press)
        throw Error(PSCU_EINVAL, "inherit: block storage needs face-only layouts");
      std::vector<int32_t> in_block(c2f.begin(), c2f.begin() + fbc);
      inherit_bsr(ctx->c, fine->m, in_block, m->m);
      PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
    } else {
      inherit(ctx->c, fine->m, c2f, m->m);
    }
    *out = m.release();
  });
}

int pscu_gmres(pscu_ctx* ctx, const pscu_mat* a, const pscu_ilu* pc, const double* rhs,
               const double* x0, int max_it, double rtol, int side, double* x, int* its,
               double* rel, int* converged, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    const int64_t n = a->m.n;
    DevBuf<double> brhs, bx0, bx;
    const double* drhs = in_vec(c, rhs, n, mem, brhs);
    const double* dx0 = x0 ? in_vec(c, x0, n, mem, bx0) : nullptr;
    double* dx = out_vec(n, x, mem, bx);
    SpmvOpC op(&a->m);
    std::unique_ptr<IluOpC> p;
    if (pc) p = std::make_unique<IluOpC>(&pc->i);
    KrylovWs ws;
    // the reference always starts from an explicit x0 vector; a zero x0 is
    // detected by the caller passing NULL
    const KrylovResultDev r =
        gmres_dev(c, op, p.get(), drhs, dx0, max_it, rtol, side == 1, dx, ws, nullptr);
    finish_out(c, x, dx, n, mem);
    *its = r.iterations;
    *rel = r.rel_residual;
    *converged = r.converged;
  });
}

int pscu_fgmres(pscu_ctx* ctx, const pscu_mat* a, const pscu_ilu* pc, const double* rhs,
                int max_it, double rtol, double* x, int* its, double* rel, int* converged,
                int mem) {
  return guard([&] {
    Context& c = ctx->c;
    const int64_t n = a->m.n;
    DevBuf<double> brhs, bx;
    const double* drhs = in_vec(c, rhs, n, mem, brhs);
    double* dx = out_vec(n, x, mem, bx);
    SpmvOpC op(&a->m);
    IluOpC ip(pc ? &pc->i : nullptr);
    IdOp id(n);
    Op& pcop = pc ? static_cast<Op&>(ip) : static_cast<Op&>(id);
    KrylovWs ws;
    const KrylovResultDev r = fgmres_dev(c, op, pcop, drhs, max_it, rtol, 0, dx, ws, nullptr);
    finish_out(c, x, dx, n, mem);
    *its = r.iterations;
    *rel = r.rel_residual;
    *converged = r.converged;
  });
}

int pscu_hier_create(pscu_ctx* ctx, const pscu_mat* fine, const pscu_layout* lf,
                     const int* degrees, int nlev, const pscu_level_cfg* cfg, pscu_hier** out) {
  return guard([&] {
    if (layout_dim(*lf) != fine->m.n)
      throw Error(PSCU_EINVAL, "hierarchy: fine layout does not match the matrix");
    auto h = std::make_unique<pscu_hier>();
    h->fine = fine;
    h->h.build(ctx->c, &fine->m, *lf, degrees, nlev, *cfg);
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *out = h.release();
  });
}

int pscu_hier_destroy(pscu_hier* h) {
  delete h;
  return PSCU_OK;
}

int pscu_hier_nlev(const pscu_hier* h) { return int(h->h.levels.size()); }

const pscu_mat* pscu_hier_level_mat(const pscu_hier* h, int l) {
  if (l < 0 || l >= int(h->h.levels.size())) return nullptr;
  // pscu_mat is a thin wrapper around Csr; the level owns it
  return reinterpret_cast<const pscu_mat*>(h->h.levels[l]->a);
}

const pscu_ilu* pscu_hier_level_ilu(const pscu_hier* h, int l) {
  if (l < 0 || l >= int(h->h.levels.size())) return nullptr;
  const Level& L = *h->h.levels[l];
  if (!L.ilu.a) return nullptr;
  return reinterpret_cast<const pscu_ilu*>(&L.ilu);
}

int pscu_vcycle(pscu_ctx* ctx, pscu_hier* h, int level, const double* d, double* cvec, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    if (level < 0 || level >= int(h->h.levels.size()))
      throw Error(PSCU_EINVAL, "vcycle: level out of range");
    const int64_t n = h->h.levels[level]->a->n;
    DevBuf<double> bd, bc;
    const double* dd = in_vec(c, d, n, mem, bd);
    double* dc = out_vec(n, cvec, mem, bc);
    h->h.vcycle(c, level, dd, dc);
    finish_out(c, cvec, dc, n, mem);
  });
}

long long pscu_hier_coarse_its(const pscu_hier* h) { return h->h.coarse_its; }
void pscu_hier_reset(pscu_hier* h) { h->h.coarse_its = 0; }

int pscu_solve(pscu_ctx* ctx, pscu_hier* h, const double* rhs, double rtol, int maxit,
               int restart, double* x, double* hist, pscu_report* rep, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    const int64_t n = h->h.levels[0]->a->n;
    const auto t0 = std::chrono::steady_clock::now();
    DevBuf<double> brhs, bx;
    const double* drhs = in_vec(c, rhs, n, mem, brhs);
    double* dx = out_vec(n, x, mem, bx);
    SpmvOpC op(h->h.levels[0]->op);
    VcycleOp pc(&h->h, n);
    h->h.coarse_its = 0;
    std::vector<double> hv;
    const KrylovResultDev r = fgmres_dev(c, op, pc, drhs, maxit, rtol, restart, dx, h->outer,
                                         hist ? &hv : nullptr);
    finish_out(c, x, dx, n, mem);
    const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (hist)
      for (size_t i = 0; i < hv.size(); ++i) hist[i] = hv[i];
    if (rep) {
      rep->outer_its = r.iterations;
      rep->coarse_its = h->h.coarse_its;
      rep->vcycles = pc.count;
      rep->rel_residual = r.rel_residual;
      rep->converged = r.converged;
      rep->t_setup = 0.0;
      rep->t_solve = t;
    }
  });
}

int pscu_solve_system(pscu_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* cols,
                      const double* vals, const double* rhs, const pscu_layout* lf,
                      const int* degrees, int nlev, const pscu_level_cfg* cfg, double rtol,
                      int maxit, int restart, double* x, double* hist, pscu_report* rep) {
  return guard([&] {
    Context& c = ctx->c;
    const auto t0 = std::chrono::steady_clock::now();
    pscu_mat fine;
    upload_csr(c, fine.m, n, row_ptr, cols, vals, PSCU_HOST);
    pscu_hier h;
    h.fine = &fine;
    h.h.build(c, &fine.m, *lf, degrees, nlev, *cfg);
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
    const auto t1 = std::chrono::steady_clock::now();
    pscu_report r{};
    const int rc = pscu_solve(ctx, &h, rhs, rtol, maxit, restart, x, hist, &r, PSCU_HOST);
    if (rc) throw Error(rc, g_err);
    const auto t2 = std::chrono::steady_clock::now();
    r.t_setup = std::chrono::duration<double>(t1 - t0).count();
    r.t_solve = std::chrono::duration<double>(t2 - t0).count();
    if (rep) *rep = r;
  });
}

int pscu_solve_system_bsr(pscu_ctx* ctx, int64_t nb, int bs, const int64_t* brow_ptr,
                          const int32_t* bcols, const double* vals, const double* rhs,
                          const pscu_layout* lf, const int* degrees, int nlev,
                          const pscu_level_cfg* cfg, double rtol, int maxit, int restart,
                          double* x, double* hist, pscu_report* rep) {
  return guard([&] {
    Context& c = ctx->c;
    const auto t0 = std::chrono::steady_clock::now();
    pscu_mat fine;
    upload_bsr(c, fine.m, nb, bs, brow_ptr, bcols, vals, PSCU_HOST);
    if (layout_dim(*lf) != fine.m.n) throw Error(PSCU_EINVAL, "solve: layout/matrix mismatch");
    pscu_hier h;
    h.fine = &fine;
    h.h.build(c, &fine.m, *lf, degrees, nlev, *cfg);
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
    const auto t1 = std::chrono::steady_clock::now();
    pscu_report r{};
    const int rc = pscu_solve(ctx, &h, rhs, rtol, maxit, restart, x, hist, &r, PSCU_HOST);
    if (rc) throw Error(rc, g_err);
    const auto t2 = std::chrono::steady_clock::now();
    r.t_setup = std::chrono::duration<double>(t1 - t0).count();
    r.t_solve = std::chrono::duration<double>(t2 - t0).count();
    if (rep) *rep = r;
  });
}

int pscu_solve_system_dgb(pscu_ctx* ctx, int64_t nb, int nm, const int64_t* brow_ptr,
                          const int32_t* bcols, const double* vals, const double* rhs,
                          const pscu_layout* lf, const int* degrees, int nlev,
                          const pscu_level_cfg* cfg, double rtol, int maxit, int restart,
                          double* x, double* hist, pscu_report* rep) {
  return guard([&] {
    Context& c = ctx->c;
    const auto t0 = std::chrono::steady_clock::now();
    pscu_mat fine;
    upload_dgb(c, fine.m, nb, nm, brow_ptr, bcols, vals, PSCU_HOST);
    if (layout_dim(*lf) != fine.m.n) throw Error(PSCU_EINVAL, "solve: layout/matrix mismatch");
    pscu_hier h;
    h.fine = &fine;
    h.h.build(c, &fine.m, *lf, degrees, nlev, *cfg);
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
    const auto t1 = std::chrono::steady_clock::now();
    pscu_report r{};
    const int rc = pscu_solve(ctx, &h, rhs, rtol, maxit, restart, x, hist, &r, PSCU_HOST);
    if (rc) throw Error(rc, g_err);
    const auto t2 = std::chrono::steady_clock::now();
    r.t_setup = std::chrono::duration<double>(t1 - t0).count();
    r.t_solve = std::chrono::duration<double>(t2 - t0).count();
    if (rep) *rep = r;
  });
}

int pscu_dgb_create(pscu_ctx* ctx, int64_t nb, int nm, const int64_t* brow_ptr,
                    const int32_t* bcols, const double* vals, int mem, pscu_mat** out) {
  return guard([&] {
    if (nb < 0) throw Error(PSCU_EINVAL, "pscu_dgb_create: negative dimension");
    auto m = std::make_unique<pscu_mat>();
    upload_dgb(ctx->c, m->m, nb, nm, brow_ptr, bcols, vals, mem);
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *out = m.release();
  });
}

int pscu_mat_dg_modes(const pscu_mat* m) { return m->m.dgm; }

int pscu_mat_set_values(pscu_ctx* ctx, pscu_mat* m, int64_t offset, int64_t count,
                        const double* vals, int mem) {
  return guard([&] {
    if (offset < 0 || count < 0 || offset + count > m->m.nnz)
      throw Error(PSCU_EINVAL, "set_values: range outside the value array");
    if (count)
      PSCU_CUDA(cudaMemcpyAsync(m->m.vals.p + offset, vals, sizeof(double) * size_t(count),
                                mem == PSCU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                                ctx->c.stream));
    if (mem == PSCU_HOST) PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int pscu_bsr_create(pscu_ctx* ctx, int64_t nb, int bs, const int64_t* brow_ptr,
                    const int32_t* bcols, const double* vals, int mem, pscu_mat** out) {
  return guard([&] {
    if (nb < 0) throw Error(PSCU_EINVAL, "pscu_bsr_create: negative dimension");
    auto m = std::make_unique<pscu_mat>();
    upload_bsr(ctx->c, m->m, nb, bs, brow_ptr, bcols, vals, mem);
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *out = m.release();
  });
}

int pscu_mat_block_size(const pscu_mat* m) { return m->m.bs; }

int pscu_bsr_download(pscu_ctx* ctx, const pscu_mat* m, int64_t* brow_ptr, int32_t* bcols,
                      double* vals) {
  return guard([&] {
    const Csr& a = m->m;
    if (!a.bs) throw Error(PSCU_EINVAL, "bsr_download: not a block-stored operator");
    if (brow_ptr) std::memcpy(brow_ptr, a.h_brow_ptr.data(), sizeof(int64_t) * a.h_brow_ptr.size());
    if (bcols) std::memcpy(bcols, a.h_bcols.data(), sizeof(int32_t) * a.h_bcols.size());
    if (vals && a.nnz)
      PSCU_CUDA(cudaMemcpyAsync(vals, a.vals.p, sizeof(double) * size_t(a.nnz),
                                cudaMemcpyDeviceToHost, ctx->c.stream));
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int pscu_assembly_begin(pscu_ctx* ctx, int64_t nb, int bs, const int64_t* brow_ptr,
                        const int32_t* bcols, pscu_mat** out) {
  return guard([&] {
    auto m = std::make_unique<pscu_mat>();
    alloc_bsr(ctx->c, m->m, nb, bs, brow_ptr, bcols);
    m->rhs_acc.alloc(size_t(std::max<int64_t>(1, m->m.n)));
    PSCU_CUDA(cudaMemsetAsync(m->rhs_acc.p, 0, sizeof(double) * size_t(m->m.n), ctx->c.stream));
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *out = m.release();
  });
}

int pscu_assembly_add(pscu_ctx* ctx, pscu_mat* m, int e0, int nelem, int n, const double* mats,
                      const double* rhs, int n_elim, const int* elim, const int32_t* efaces,
                      int nfe, const int32_t* keep_pos, double* elim_coupling, double* elim_rhs,
                      int mem) {
  return guard([&] {
    Context& c = ctx->c;
    if (!m->rhs_acc.p) throw Error(PSCU_EINVAL, "assembly_add: not an assembly target");
    const int nk = n - n_elim;
    DevBuf<double> bm, br, bc, be;
    DevBuf<int32_t> bf;
    const double* dm = in_vec(c, mats, int64_t(nelem) * n * n, mem, bm);
    const double* dr = in_vec(c, rhs, int64_t(nelem) * n, mem, br);
    const int32_t* df = efaces;
    if (mem == PSCU_HOST) {
      bf.upload(efaces, size_t(nelem) * nfe, c.stream);
      df = bf.p;
    }
    double* dc = elim_coupling ? out_vec(int64_t(nelem) * n_elim * nk, elim_coupling, mem, bc) : nullptr;
    double* de = elim_rhs ? out_vec(int64_t(nelem) * n_elim, elim_rhs, mem, be) : nullptr;
    condense_scatter_bsr(c, m->m, e0, nelem, n, dm, dr, n_elim, elim, df, nullptr, nfe,
                         keep_pos, m->rhs_acc.p, dc, de);
    if (elim_coupling) finish_out(c, elim_coupling, dc, int64_t(nelem) * n_elim * nk, mem);
    if (elim_rhs) finish_out(c, elim_rhs, de, int64_t(nelem) * n_elim, mem);
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int pscu_host_alloc(int64_t bytes, void** out) {
  return guard([&] {
    *out = nullptr;
    PSCU_CUDA(cudaHostAlloc(out, size_t(std::max<int64_t>(bytes, 8)), cudaHostAllocDefault));
  });
}

int pscu_host_free(void* p) {
  return guard([&] {
    if (p) PSCU_CUDA(cudaFreeHost(p));
  });
}

int pscu_bsr_create_local(pscu_ctx* ctx, int64_t nb, int64_t ncb, int bs, int64_t diag_off,
                          const int64_t* brow_ptr, const int32_t* bcols, const double* vals,
                          int mem, pscu_mat** out) {
  return guard([&] {
    auto m = std::make_unique<pscu_mat>();
    upload_bsr(ctx->c, m->m, nb, bs, brow_ptr, bcols, vals, mem, ncb, diag_off);
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *out = m.release();
  });
}

int pscu_assembly_begin_local(pscu_ctx* ctx, int64_t nb, int64_t ncb, int bs, int64_t diag_off,
                              const int64_t* brow_ptr, const int32_t* bcols, pscu_mat** out) {
  return guard([&] {
    auto m = std::make_unique<pscu_mat>();
    alloc_bsr(ctx->c, m->m, nb, bs, brow_ptr, bcols, ncb, diag_off);
    m->rhs_acc.alloc(size_t(std::max<int64_t>(1, m->m.n)));
    PSCU_CUDA(cudaMemsetAsync(m->rhs_acc.p, 0, sizeof(double) * size_t(m->m.n), ctx->c.stream));
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *out = m.release();
  });
}

int pscu_assembly_add_local(pscu_ctx* ctx, pscu_mat* m, int e0, int nelem, int n,
                            const double* mats, const double* rhs, int n_elim, const int* elim,
                            const int32_t* erows, const int32_t* ecols, int nfe,
                            const int32_t* keep_pos, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    if (!m->rhs_acc.p) throw Error(PSCU_EINVAL, "assembly_add: not an assembly target");
    DevBuf<double> bm, br;
    DevBuf<int32_t> bfr, bfc;
    const double* dm = in_vec(c, mats, int64_t(nelem) * n * n, mem, bm);
    const double* dr = in_vec(c, rhs, int64_t(nelem) * n, mem, br);
    const int32_t *dfr = erows, *dfc = ecols;
    if (mem == PSCU_HOST) {
      bfr.upload(erows, size_t(nelem) * nfe, c.stream);
      bfc.upload(ecols, size_t(nelem) * nfe, c.stream);
      dfr = bfr.p;
      dfc = bfc.p;
    }
    condense_scatter_bsr(c, m->m, e0, nelem, n, dm, dr, n_elim, elim, dfc, dfr, nfe, keep_pos,
                         m->rhs_acc.p, nullptr, nullptr);
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int pscu_assembly_rhs(pscu_ctx* ctx, const pscu_mat* m, double* rhs, int mem) {
  return guard([&] {
    if (!m->rhs_acc.p) throw Error(PSCU_EINVAL, "assembly_rhs: not an assembly target");
    PSCU_CUDA(cudaMemcpyAsync(rhs, m->rhs_acc.p, sizeof(double) * size_t(m->m.n),
                              mem == PSCU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                              ctx->c.stream));
    PSCU_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int pscu_condense_batch(pscu_ctx* ctx, int nelem, int n, const double* mats, const double* rhs,
                        int n_elim, const int* elim, double* schur, double* reduced_rhs,
                        double* elim_coupling, double* elim_rhs, int* bad_element, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    const int nk = n - n_elim;
    DevBuf<double> bm, br, bs, brr, bc, be;
    const double* dm = in_vec(c, mats, int64_t(nelem) * n * n, mem, bm);
    const double* dr = in_vec(c, rhs, int64_t(nelem) * n, mem, br);
    double* ds = schur ? out_vec(int64_t(nelem) * nk * nk, schur, mem, bs) : nullptr;
    double* drr = reduced_rhs ? out_vec(int64_t(nelem) * nk, reduced_rhs, mem, brr) : nullptr;
    double* dc = elim_coupling ? out_vec(int64_t(nelem) * n_elim * nk, elim_coupling, mem, bc) : nullptr;
    double* de = elim_rhs ? out_vec(int64_t(nelem) * n_elim, elim_rhs, mem, be) : nullptr;
    condense_batch(c, nelem, n, dm, dr, n_elim, elim, ds, drr, dc, de, bad_element);
    if (mem == PSCU_HOST) {
      if (schur) finish_out(c, schur, ds, int64_t(nelem) * nk * nk, mem);
      if (reduced_rhs) finish_out(c, reduced_rhs, drr, int64_t(nelem) * nk, mem);
      if (elim_coupling) finish_out(c, elim_coupling, dc, int64_t(nelem) * n_elim * nk, mem);
      if (elim_rhs) finish_out(c, elim_rhs, de, int64_t(nelem) * n_elim, mem);
    }
    PSCU_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int pscu_condense_assemble(pscu_ctx* ctx, int nelem, int n, const double* mats,
                           const double* rhs, int n_elim, const int* elim,
                           const int64_t* kept_global, int64_t dim, const int64_t* row_ptr,
                           const int32_t* cols, const pscu_layout* layout, int mem,
                           pscu_mat** out, double* rhs_out, double* elim_coupling,
                           double* elim_rhs) {
  return guard([&] {
    Context& c = ctx->c;
    if (layout_dim(*layout) != dim) throw Error(PSCU_EINVAL, "assemble: layout/pattern mismatch");
    const int nk = n - n_elim;
    DevBuf<double> bm, br, bschur(size_t(nelem) * nk * nk), brr(size_t(nelem) * nk), brhs;
    DevBuf<int64_t> bk;
    const double* dm = in_vec(c, mats, int64_t(nelem) * n * n, mem, bm);
    const double* dr = in_vec(c, rhs, int64_t(nelem) * n, mem, br);
    const int64_t* dk = kept_global;
    if (mem == PSCU_HOST) {
      bk.upload(kept_global, size_t(nelem) * nk, c.stream);
      dk = bk.p;
    }
    DevBuf<double> bc, be;
    double* dc = elim_coupling ? out_vec(int64_t(nelem) * n_elim * nk, elim_coupling, mem, bc)
                               : nullptr;
    double* de = elim_rhs ? out_vec(int64_t(nelem) * n_elim, elim_rhs, mem, be) : nullptr;
    condense_batch(c, nelem, n, dm, dr, n_elim, elim, bschur.p, brr.p, dc, de, nullptr);
    if (elim_coupling) finish_out(c, elim_coupling, dc, int64_t(nelem) * n_elim * nk, mem);
    if (elim_rhs) finish_out(c, elim_rhs, de, int64_t(nelem) * n_elim, mem);
    auto m = std::make_unique<pscu_mat>();
    Csr& a = m->m;
    a.n = dim;
    if (mem == PSCU_HOST) {
      a.h_row_ptr.assign(row_ptr, row_ptr + dim + 1);
      a.nnz = a.h_row_ptr[dim];
      a.h_cols.assign(cols, cols + a.nnz);
    } else {
      a.h_row_ptr.resize(dim + 1);
      PSCU_CUDA(cudaMemcpy(a.h_row_ptr.data(), row_ptr, sizeof(int64_t) * (dim + 1),
                           cudaMemcpyDeviceToHost));
      a.nnz = a.h_row_ptr[dim];
      a.h_cols.resize(a.nnz);
      PSCU_CUDA(cudaMemcpy(a.h_cols.data(), cols, sizeof(int32_t) * a.nnz, cudaMemcpyDeviceToHost));
    }
    a.row_ptr.upload(a.h_row_ptr, c.stream);
    a.cols.upload(a.h_cols, c.stream);
    a.vals.alloc(a.nnz);
    double* drhs = out_vec(dim, rhs_out, mem, brhs);
    assemble_values(c, nelem, nk, dk, bschur.p, brr.p, *layout, a, drhs);
    finish_out(c, rhs_out, drhs, dim, mem);
    *out = m.release();
  });
}

int pscu_recover_batch(pscu_ctx* ctx, int nelem, int n, int n_elim, const int* elim,
                       const int64_t* kept_global, const double* elim_coupling,
                       const double* elim_rhs, const double* x, double* locals, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    const int nk = n - n_elim;
    if (mem != PSCU_HOST) {
      recover_batch(c, nelem, n, n_elim, elim, kept_global, elim_coupling, elim_rhs, x, locals);
      return;
    }
    // host buffers: the x length is the largest kept global index + 1
    int64_t nx = 0;
    for (int64_t i = 0; i < int64_t(nelem) * nk; ++i) nx = std::max(nx, kept_global[i] + 1);
    DevBuf<int64_t> bk;
    bk.upload(kept_global, size_t(nelem) * nk, c.stream);
    DevBuf<double> bc, be, bx, bl;
    const double* dc = in_vec(c, elim_coupling, int64_t(nelem) * n_elim * nk, mem, bc);
    const double* de = in_vec(c, elim_rhs, int64_t(nelem) * n_elim, mem, be);
    const double* dx = in_vec(c, x, nx, mem, bx);
    double* dl = out_vec(int64_t(nelem) * n, locals, mem, bl);
    recover_batch(c, nelem, n, n_elim, elim, bk.p, dc, de, dx, dl);
    finish_out(c, locals, dl, int64_t(nelem) * n, mem);
  });
}

int pscu_error_accumulate(pscu_ctx* ctx, const int32_t* dims, int nelem, const double* tables,
                          const double* locals, double* acc, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    if (nelem < 0) throw Error(PSCU_EINVAL, "error_accumulate: nelem < 0");
    DevBuf<double> bt, bl, ba;
    const double* dt = in_vec(c, tables, int64_t(nelem) * dims[4], mem, bt);
    const double* dl = in_vec(c, locals, int64_t(nelem) * dims[8], mem, bl);
    double* da = acc;
    if (mem == PSCU_HOST) {
      ba.upload(acc, 4, c.stream);
      da = ba.p;
    }
    error_accumulate(c, dims, nelem, dt, dl, da);
    finish_out(c, acc, da, 4, mem);
  });
}

int pscu_local_blocks3(pscu_ctx* ctx, int k, int data, double eta, int nq1, const double* gl,
                       int64_t nv, const double* xyz, int64_t nfaces, const int32_t* ftab,
                       int nelem, const int32_t* hex, const int32_t* ef, const int32_t* es,
                       const double* coef, double* mats, double* rhs, int mem) {
  return guard([&] {
    Context& c = ctx->c;
    if (nq1 < 1 || nq1 > 8) throw Error(PSCU_EINVAL, "local_blocks3: rule size out of range");
    if (k < 0 || k > 4) throw Error(PSCU_EINVAL, "hho3: k must be in [0, 4]");
    const auto d3 = [](int d) { return (d + 1) * (d + 2) * (d + 3) / 6; };
    const auto d2 = [](int d) { return (d + 1) * (d + 2) / 2; };
    const int64_t n = 3 * (d3(k + 1) + 6 * d2(k)) + d3(k) + 6 * d2(k);
    const int64_t ncoef = data == 3 ? int64_t(nelem) * 3 * d3(k) : 0;
    if (mem != PSCU_HOST) {
      local_blocks3(c, k, data, eta, nq1, gl, gl + nq1, xyz, hex, ef, es, ftab, coef, 0, nelem,
                    mats, rhs);
      return;
    }
    DevBuf<double> bg, bx, bc, bm, br;
    DevBuf<int32_t> bh, be, bs, bf;
    bg.upload(gl, size_t(2 * nq1), c.stream);
    bx.upload(xyz, size_t(3 * nv), c.stream);
    bf.upload(ftab, size_t(5 * nfaces), c.stream);
    bh.upload(hex, size_t(8) * nelem, c.stream);
    be.upload(ef, size_t(6) * nelem, c.stream);
    bs.upload(es, size_t(6) * nelem, c.stream);
    if (ncoef) bc.upload(coef, size_t(ncoef), c.stream);
    double* dm = out_vec(int64_t(nelem) * n * n, mats, mem, bm);
    double* dr = out_vec(int64_t(nelem) * n, rhs, mem, br);
    local_blocks3(c, k, data, eta, nq1, bg.p, bg.p + nq1, bx.p, bh.p, be.p, bs.p, bf.p,
                  ncoef ? bc.p : nullptr, 0, nelem, dm, dr);
    finish_out(c, mats, dm, int64_t(nelem) * n * n, mem);
    finish_out(c, rhs, dr, int64_t(nelem) * n, mem);
  });
}

} // extern "C"
