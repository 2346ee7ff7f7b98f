/* oracle/pstokes_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference solver hot path, used as the checker for
 * the CUDA path (tests/) and as the "port" CPU baseline (bench.py). Each
 * function cites the reference file:line it follows (paths relative to
 * /root/reference/proj/include/pstokes). Arithmetic follows the element-wise
 * semantics of include/eigen_subset/Eigen/Dense: one rounded operation per
 * element, no FMA (-ffp-contract=off), and the fixed-shape reproducible dot.
 * Parity of this restatement with the reference itself (compiled in
 * oracle/_ref) is checked bit-for-bit by tests/test_oracle.py. */
#include "pstokes_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int set_err(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}

const char* po_last_error(void) { return g_err; }

static int dim_p1(int k) { return k + 1; }
static int dim_p2(int k) { return (k + 1) * (k + 2) / 2; }

/* make_layout, dof_layout.hpp:87-126 */
int po_make_layout(int scheme, int strategy, int k, int n_faces, int n_elements, po_layout* l) {
  if (k < 0) return set_err("layout: k must be >= 0");
  memset(l, 0, sizeof *l);
  l->scheme = scheme;
  l->strategy = strategy;
  l->k = k;
  l->n_faces = n_faces;
  l->n_elements = n_elements;
  l->dim = 2;
  const int nf = dim_p1(k), np = dim_p2(k);
  const int ne = dim_p2(scheme == 1 ? k + 1 : k);
  switch (scheme) {
    case 0:
      l->face_vel = nf;
      if (strategy == 0) { l->elem_vel = ne; l->elem_press = np; }
      else if (strategy == 1) l->elem_press = np;
      else l->elem_press = 1;
      break;
    case 1:
      l->face_vel = nf;
      l->face_press = nf;
      if (strategy == 0) { l->elem_vel = ne; l->elem_press = np; }
      else if (strategy == 1) return set_err("hho-hp: supported strategies are uncond and vp-cond");
      break;
    case 2:
      if (k < 1) return set_err("dg: k must be >= 1");
      if (strategy != 0) return set_err("dg: no static condensation exists, use uncond");
      l->elem_vel = ne;
      l->elem_press = np;
      break;
    default: return set_err("unknown scheme");
  }
  return 0;
}

static int ncomp(const po_layout* l) { return l->dim == 3 ? 3 : 2; }
static int64_t face_block(const po_layout* l) { return ncomp(l) * l->face_vel + l->face_press; }
static int64_t elem_block(const po_layout* l) { return ncomp(l) * l->elem_vel + l->elem_press; }

/* 3D: hho-hp vp-cond only (the configs that need it); P^k on a face has
 * (k+1)(k+2)/2 modes */
int po_make_layout3(int scheme, int strategy, int k, int n_faces, int n_elements, po_layout* l) {
  if (k < 0) return set_err("layout: k must be >= 0");
  if (scheme == 2) {
    /* DG (config 4): element blocks [ux | uy | uz | p] of dim P^k(3D) modes
     * each (dof_layout.hpp:118-123 with three components) */
    if (k < 1) return set_err("dg: k must be >= 1");
    if (strategy != 0) return set_err("dg: no static condensation exists, use uncond");
  } else if (scheme != 1 || strategy != 2) {
    return set_err("3D layout: hho-hp vp-cond or dg uncond only");
  }
  memset(l, 0, sizeof *l);
  l->scheme = scheme;
  l->strategy = strategy;
  l->k = k;
  l->n_faces = n_faces;
  l->n_elements = n_elements;
  if (scheme == 2) {
    l->elem_vel = (k + 1) * (k + 2) * (k + 3) / 6;
    l->elem_press = l->elem_vel;
  } else {
    l->face_vel = dim_p2(k);
    l->face_press = dim_p2(k);
  }
  l->dim = 3;
  return 0;
}

/* the layout of the same scheme at another degree */
static int layout_at(const po_layout* lf, int k, po_layout* out) {
  if (lf->dim == 3) return po_make_layout3(lf->scheme, lf->strategy, k, lf->n_faces, lf->n_elements, out);
  return po_make_layout(lf->scheme, lf->strategy, k, lf->n_faces, lf->n_elements, out);
}

int64_t po_layout_dim(const po_layout* l) {
  return (int64_t)l->n_faces * face_block(l) + (int64_t)l->n_elements * elem_block(l);
}

/* coarse_to_fine_map, plevels.hpp:47-72 */
int po_coarse_to_fine_map(const po_layout* f, const po_layout* c, int64_t* map) {
  if (f->n_faces != c->n_faces || f->n_elements != c->n_elements)
    return set_err("transfer: layouts live on different meshes");
  if (c->face_vel > f->face_vel || c->face_press > f->face_press || c->elem_vel > f->elem_vel ||
      c->elem_press > f->elem_press)
    return set_err("transfer: coarse layout is not nested in the fine one");
  for (int64_t fc = 0; fc < c->n_faces; ++fc) {
    const int64_t cb = fc * face_block(c), fb = fc * face_block(f);
    for (int comp = 0; comp < ncomp(c); ++comp)
      for (int m = 0; m < c->face_vel; ++m)
        map[cb + comp * c->face_vel + m] = fb + comp * f->face_vel + m;
    for (int m = 0; m < c->face_press; ++m)
      map[cb + ncomp(c) * c->face_vel + m] = fb + ncomp(f) * f->face_vel + m;
  }
  const int64_t cfo = (int64_t)c->n_faces * face_block(c), ffo = (int64_t)f->n_faces * face_block(f);
  for (int64_t e = 0; e < c->n_elements; ++e) {
    const int64_t cb = cfo + e * elem_block(c), fb = ffo + e * elem_block(f);
    for (int comp = 0; comp < ncomp(c); ++comp)
      for (int m = 0; m < c->elem_vel; ++m)
        map[cb + comp * c->elem_vel + m] = fb + comp * f->elem_vel + m;
    for (int m = 0; m < c->elem_press; ++m)
      map[cb + ncomp(c) * c->elem_vel + m] = fb + ncomp(f) * f->elem_vel + m;
  }
  return 0;
}

/* Reproducible dot (include/eigen_subset/Eigen/Dense, internal::repro_dot):
 * T = pow2 >= ceil(n/16) clamped to [1, 2^18] strided partials, then an
 * adjacent-pair binary tree. */
static int64_t repro_lanes(int64_t n) {
  int64_t want = (n + 15) / 16, t = 1;
  while (t < want && t < ((int64_t)1 << 18)) t <<= 1;
  return t;
}

double po_dot(const double* x, const double* y, int64_t n) {
  const int64_t T = repro_lanes(n);
  if (T == 1) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double p = x[i] * y[i];
      s = s + p;
    }
    return s;
  }
  double* part = (double*)calloc((size_t)T, sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    const double p = x[i] * y[i];
    part[i % T] = part[i % T] + p;
  }
  for (int64_t w = T; w > 1; w >>= 1)
    for (int64_t k = 0; k < w / 2; ++k) part[k] = part[2 * k] + part[2 * k + 1];
  const double r = part[0];
  free(part);
  return r;
}

static double po_norm(const double* x, int64_t n) { return sqrt(po_dot(x, x, n)); }

/* CsrMatrix::multiply, csr.hpp:68-74 */
void po_csr_multiply(const po_csr* a, const double* x, double* y) {
  for (int64_t i = 0; i < a->n; ++i) {
    double s = 0.0;
    for (int64_t p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) {
      const double t = a->vals[p] * x[a->cols[p]];
      s = s + t;
    }
    y[i] = s;
  }
}

static int64_t csr_find(const po_csr* a, int64_t i, int64_t j) {
  int64_t lo = a->row_ptr[i], hi = a->row_ptr[i + 1];
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (a->cols[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  return (lo < a->row_ptr[i + 1] && a->cols[lo] == j) ? lo : -1;
}

/* Ilu0 constructor, ilu0.hpp:19-51 (IKJ over the row pattern) */
int po_ilu0_factor(const po_csr* a, double* lu, int64_t* diag) {
  const int64_t n = a->n;
  memcpy(lu, a->vals, sizeof(double) * (size_t)a->row_ptr[n]);
  for (int64_t i = 0; i < n; ++i) {
    diag[i] = csr_find(a, i, i);
    if (diag[i] < 0) return set_err("ilu0: row has no diagonal entry");
  }
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) pos[i] = -1;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) pos[a->cols[p]] = p;
    for (int64_t p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) {
      const int64_t k = a->cols[p];
      if (k >= i) break;
      const double piv = lu[diag[k]];
      if (piv == 0.0) {
        free(pos);
        return set_err("ilu0: zero pivot");
      }
      const double lik = lu[p] / piv;
      lu[p] = lik;
      for (int64_t q = diag[k] + 1; q < a->row_ptr[k + 1]; ++q) {
        const int64_t r = pos[a->cols[q]];
        if (r >= 0) {
          const double t = lik * lu[q];
          lu[r] = lu[r] - t;
        }
      }
    }
    if (lu[diag[i]] == 0.0) {
      free(pos);
      return set_err("ilu0: zero pivot");
    }
    for (int64_t p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) pos[a->cols[p]] = -1;
  }
  free(pos);
  return 0;
}

/* Ilu0::apply, ilu0.hpp:53-65 */
void po_ilu0_apply(const po_csr* a, const double* lu, const int64_t* diag, const double* x,
                   double* y) {
  for (int64_t i = 0; i < a->n; ++i) {
    double s = x[i];
    for (int64_t p = a->row_ptr[i]; p < diag[i]; ++p) {
      const double t = lu[p] * y[a->cols[p]];
      s = s - t;
    }
    y[i] = s;
  }
  for (int64_t i = a->n - 1; i >= 0; --i) {
    double s = y[i];
    for (int64_t p = diag[i] + 1; p < a->row_ptr[i + 1]; ++p) {
      const double t = lu[p] * y[a->cols[p]];
      s = s - t;
    }
    y[i] = s / lu[diag[i]];
  }
}

/* inherit_matrix, plevels.hpp:93-113 */
int64_t po_inherit(const po_csr* fine, int64_t n_fine, const int64_t* c2f, int64_t nc,
                   int64_t* row_ptr, int32_t* cols, double* vals) {
  int64_t* f2c = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_fine > 0 ? n_fine : 1));
  for (int64_t i = 0; i < n_fine; ++i) f2c[i] = -1;
  for (int64_t i = 0; i < nc; ++i) f2c[c2f[i]] = i;
  int64_t nnz = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (int64_t ic = 0; ic < nc; ++ic) {
    const int64_t r = c2f[ic];
    for (int64_t p = fine->row_ptr[r]; p < fine->row_ptr[r + 1]; ++p) {
      const int64_t jc = f2c[fine->cols[p]];
      if (jc >= 0) {
        if (cols) {
          cols[nnz] = (int32_t)jc;
          vals[nnz] = fine->vals[p];
        }
        ++nnz;
      }
    }
    if (row_ptr) row_ptr[ic + 1] = nnz;
  }
  free(f2c);
  return nnz;
}

/* ---------------------------------------------------------------------------
 * Krylov: detail::ArnoldiWorkspace, gmres, fgmres (gmres.hpp:38-173)
 * ------------------------------------------------------------------------- */

typedef struct {
  int64_t n;
  int m;           /* Krylov dimension bound */
  double* v;       /* (m+1) x n */
  double* z;       /* m x n (may alias v when no preconditioner is stored) */
  double* h;       /* (m+1) x m, column-major */
  double *g, *cs, *sn;
  double last_subdiag;
} arnoldi;

static void arnoldi_init(arnoldi* ws, int64_t n, int m, const double* r0, double beta) {
  ws->n = n;
  ws->m = m;
  ws->v = (double*)calloc((size_t)(m + 1) * (size_t)n + 1, sizeof(double));
  ws->z = (double*)calloc((size_t)m * (size_t)n + 1, sizeof(double));
  ws->h = (double*)calloc((size_t)(m + 1) * (size_t)m + 1, sizeof(double));
  ws->g = (double*)calloc((size_t)m + 1, sizeof(double));
  ws->cs = (double*)calloc((size_t)m + 1, sizeof(double));
  ws->sn = (double*)calloc((size_t)m + 1, sizeof(double));
  for (int64_t i = 0; i < n; ++i) ws->v[i] = r0[i] / beta;
  ws->g[0] = beta;
  ws->last_subdiag = 0.0;
}

static void arnoldi_free(arnoldi* ws) {
  free(ws->v);
  free(ws->z);
  free(ws->h);
  free(ws->g);
  free(ws->cs);
  free(ws->sn);
}

#define H(i, j) ws->h[(size_t)(i) + (size_t)(j) * (size_t)(ws->m + 1)]

/* ArnoldiWorkspace::step, gmres.hpp:59-82; w is overwritten */
static double arnoldi_step(arnoldi* ws, int j, double* w) {
  const int64_t n = ws->n;
  for (int i = 0; i <= j; ++i) {
    const double* vi = ws->v + (size_t)i * (size_t)n;
    const double hij = po_dot(w, vi, n);
    H(i, j) = hij;
    for (int64_t e = 0; e < n; ++e) {
      const double t = hij * vi[e];
      w[e] = w[e] - t;
    }
  }
  const double hn = po_norm(w, n);
  H(j + 1, j) = hn;
  ws->last_subdiag = hn;
  double* vn = ws->v + (size_t)(j + 1) * (size_t)n;
  if (hn > 0.0)
    for (int64_t e = 0; e < n; ++e) vn[e] = w[e] / hn;
  else
    for (int64_t e = 0; e < n; ++e) vn[e] = 0.0;
  for (int i = 0; i < j; ++i) {
    const double t = ws->cs[i] * H(i, j) + ws->sn[i] * H(i + 1, j);
    H(i + 1, j) = -ws->sn[i] * H(i, j) + ws->cs[i] * H(i + 1, j);
    H(i, j) = t;
  }
  const double denom = hypot(H(j, j), H(j + 1, j));
  ws->cs[j] = denom == 0.0 ? 1.0 : H(j, j) / denom;
  ws->sn[j] = denom == 0.0 ? 0.0 : H(j + 1, j) / denom;
  H(j, j) = denom;
  H(j + 1, j) = 0.0;
  ws->g[j + 1] = -ws->sn[j] * ws->g[j];
  ws->g[j] = ws->cs[j] * ws->g[j];
  return fabs(ws->g[j + 1]);
}

/* ArnoldiWorkspace::solution, gmres.hpp:84-91 (upper triangular solve with
 * i descending and j ascending, then x0 + sum_i y_i z_i, i ascending) */
static void arnoldi_solution(const arnoldi* ws, const double* x0, int m, const double* zbase,
                             double* x) {
  const int64_t n = ws->n;
  double* y = (double*)calloc((size_t)m + 1, sizeof(double));
  for (int i = 0; i < m; ++i) y[i] = ws->g[i];
  for (int i = m - 1; i >= 0; --i) {
    double s = y[i];
    for (int jj = i + 1; jj < m; ++jj) {
      const double t = H(i, jj) * y[jj];
      s = s - t;
    }
    y[i] = s / H(i, i);
  }
  if (x != x0) memcpy(x, x0, sizeof(double) * (size_t)n);
  for (int i = 0; i < m; ++i) {
    const double* zi = zbase + (size_t)i * (size_t)n;
    for (int64_t e = 0; e < n; ++e) {
      const double t = y[i] * zi[e];
      x[e] = x[e] + t;
    }
  }
  free(y);
}

typedef struct {
  po_apply_fn op, pc;
  void *op_ctx, *pc_ctx;
  double* tmp;
} left_ctx;

static void left_apply(void* c, const double* x, double* y) {
  left_ctx* l = (left_ctx*)c;
  l->op(l->op_ctx, x, l->tmp);
  l->pc(l->pc_ctx, l->tmp, y);
}

/* gmres, gmres.hpp:103-139 */
int po_gmres(po_apply_fn op, void* op_ctx, po_apply_fn pc, void* pc_ctx, int64_t n,
             const double* rhs, const double* x0, int max_it, double rtol, int left, double* x,
             int* its, double* rel, int* converged) {
  if (left && pc) {
    left_ctx lc = {op, pc, op_ctx, pc_ctx, (double*)malloc(sizeof(double) * (size_t)(n + 1))};
    double* prhs = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    pc(pc_ctx, rhs, prhs);
    const int rc = po_gmres(left_apply, &lc, NULL, NULL, n, prhs, x0, max_it, rtol, 0, x, its, rel,
                            converged);
    free(prhs);
    free(lc.tmp);
    return rc;
  }
  *its = 0;
  *rel = 0.0;
  *converged = 0;
  double* r0 = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  op(op_ctx, x0, r0);
  for (int64_t e = 0; e < n; ++e) r0[e] = rhs[e] - r0[e];
  const double beta = po_norm(r0, n);
  if (beta == 0.0) {
    if (x != x0) memcpy(x, x0, sizeof(double) * (size_t)n);
    *converged = 1;
    free(r0);
    return 0;
  }
  arnoldi ws;
  arnoldi_init(&ws, n, max_it, r0, beta);
  double* w = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  int m = 0;
  for (int j = 0; j < max_it; ++j) {
    const double* vj = ws.v + (size_t)j * (size_t)n;
    double* zj = ws.z + (size_t)j * (size_t)n;
    if (pc) pc(pc_ctx, vj, zj);
    else memcpy(zj, vj, sizeof(double) * (size_t)n);
    op(op_ctx, zj, w);
    const double est = arnoldi_step(&ws, j, w);
    m = j + 1;
    *rel = est / beta;
    if (est <= rtol * beta) {
      *converged = 1;
      break;
    }
    if (ws.last_subdiag == 0.0) {
      *converged = 1;
      break;
    }
  }
  *its = m;
  double* xs = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  arnoldi_solution(&ws, x0, m, ws.z, xs);
  memcpy(x, xs, sizeof(double) * (size_t)n);
  free(xs);
  free(w);
  free(r0);
  arnoldi_free(&ws);
  return 0;
}

/* fgmres, gmres.hpp:145-173, plus the residual-estimate history and the
 * optional restart of oracle/ref_driver.cpp:fgmres_hist (restart = 0 is the
 * reference behaviour). */
int po_fgmres(po_apply_fn op, void* op_ctx, po_apply_fn pc, void* pc_ctx, int64_t n,
              const double* rhs, int max_it, double rtol, int restart, double* x, double* hist,
              int* its, double* rel, int* converged) {
  *its = 0;
  *rel = 0.0;
  *converged = 0;
  const double bnorm = po_norm(rhs, n);
  if (bnorm == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    *converged = 1;
    return 0;
  }
  double* x0 = (double*)calloc((size_t)n + 1, sizeof(double));
  double* r0 = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* w = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* xs = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  memcpy(r0, rhs, sizeof(double) * (size_t)n);
  double beta = bnorm;
  const int cycle = restart > 0 ? restart : max_it;
  int total = 0, done = 0;
  while (!done) {
    const int mm = cycle < max_it - total ? cycle : max_it - total;
    arnoldi ws;
    arnoldi_init(&ws, n, mm, r0, beta);
    int restart_now = 0;
    for (int j = 0; j < mm; ++j) {
      double* zj = ws.z + (size_t)j * (size_t)n;
      pc(pc_ctx, ws.v + (size_t)j * (size_t)n, zj);
      op(op_ctx, zj, w);
      const double est = arnoldi_step(&ws, j, w);
      ++total;
      if (hist) hist[total - 1] = est / bnorm;
      const int m = j + 1;
      const int last = total == max_it;
      if (est <= rtol * bnorm || ws.last_subdiag == 0.0 || last) {
        arnoldi_solution(&ws, x0, m, ws.z, xs);
        memcpy(x, xs, sizeof(double) * (size_t)n);
        op(op_ctx, x, w);
        for (int64_t e = 0; e < n; ++e) w[e] = rhs[e] - w[e];
        *rel = po_norm(w, n) / bnorm;
        *its = total;
        if (*rel <= rtol) {
          *converged = 1;
          done = 1;
          break;
        }
        if (last) {
          done = 1;
          break;
        }
        if (j + 1 == mm) { /* cycle exhausted after a failed true-residual check */
          restart_now = 1;
          memcpy(x0, xs, sizeof(double) * (size_t)n);
        }
      } else if (j + 1 == mm) {
        restart_now = 1;
        arnoldi_solution(&ws, x0, m, ws.z, xs);
        memcpy(x0, xs, sizeof(double) * (size_t)n);
      }
    }
    arnoldi_free(&ws);
    if (done) break;
    if (!restart_now) break;
    op(op_ctx, x0, w);
    for (int64_t e = 0; e < n; ++e) r0[e] = rhs[e] - w[e];
    beta = po_norm(r0, n);
  }
  free(x0);
  free(r0);
  free(w);
  free(xs);
  return 0;
}

/* ---------------------------------------------------------------------------
 * p-multilevel hierarchy and V-cycle (plevels.hpp:115-239)
 * ------------------------------------------------------------------------- */

typedef struct {
  po_layout layout;
  int64_t n, nnz;
  int64_t* row_ptr;
  int32_t* cols;
  double* vals;
  double* lu;
  int64_t* diag;
  int64_t* down_map; /* coarse (l+1) -> this level */
  int64_t n_coarse;
  po_csr csr;
  double* bj; /* block-Jacobi inverses (smoother 1) */
} po_level;

struct po_hier {
  int nlev;
  po_level* lev;
  int smoother;
  int smoother_iters;
  double coarse_rtol;
  int coarse_maxit;
  long long coarse_its;
};

typedef struct {
  const po_level* lev;
} lev_ctx;

static void lev_spmv(void* c, const double* x, double* y) {
  const po_level* l = ((lev_ctx*)c)->lev;
  po_csr_multiply(&l->csr, x, y);
}
static void lev_ilu(void* c, const double* x, double* y) {
  const po_level* l = ((lev_ctx*)c)->lev;
  po_ilu0_apply(&l->csr, l->lu, l->diag, x, y);
}
static void lev_bj(void* c, const double* x, double* y) {
  const po_level* l = ((lev_ctx*)c)->lev;
  po_bj_apply(&l->layout, l->bj, x, y);
}

/* LevelHierarchy ctor, plevels.hpp:129-159 (ILU-GMRES coarse solver) */
po_hier* po_hier_create(const po_csr* fine, const po_layout* lf, const int* degrees, int nlev,
                        int smoother_iters, double coarse_rtol, int coarse_maxit) {
  return po_hier_create_ex(fine, lf, degrees, nlev, smoother_iters, coarse_rtol, coarse_maxit, 0);
}

po_hier* po_hier_create_ex(const po_csr* fine, const po_layout* lf, const int* degrees, int nlev,
                           int smoother_iters, double coarse_rtol, int coarse_maxit,
                           int smoother) {
  if (nlev < 1 || degrees[0] != lf->k) {
    set_err("hierarchy: level degrees must start at the fine degree");
    return NULL;
  }
  for (int i = 1; i < nlev; ++i)
    if (degrees[i] >= degrees[i - 1]) {
      set_err("hierarchy: level degrees must strictly decrease");
      return NULL;
    }
  if (degrees[nlev - 1] < (lf->scheme == 2 ? 1 : 0)) {
    set_err("hierarchy: coarsest degree below the scheme minimum");
    return NULL;
  }
  po_hier* h = (po_hier*)calloc(1, sizeof(po_hier));
  h->nlev = nlev;
  h->smoother = smoother;
  h->smoother_iters = smoother_iters;
  h->coarse_rtol = coarse_rtol;
  h->coarse_maxit = coarse_maxit;
  h->lev = (po_level*)calloc((size_t)nlev, sizeof(po_level));
  po_level* L0 = &h->lev[0];
  L0->layout = *lf;
  L0->n = fine->n;
  L0->nnz = fine->row_ptr[fine->n];
  L0->row_ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(L0->n + 1));
  L0->cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)(L0->nnz + 1));
  L0->vals = (double*)malloc(sizeof(double) * (size_t)(L0->nnz + 1));
  memcpy(L0->row_ptr, fine->row_ptr, sizeof(int64_t) * (size_t)(L0->n + 1));
  memcpy(L0->cols, fine->cols, sizeof(int32_t) * (size_t)L0->nnz);
  memcpy(L0->vals, fine->vals, sizeof(double) * (size_t)L0->nnz);
  for (int l = 0; l < nlev; ++l) {
    po_level* L = &h->lev[l];
    if (l > 0) {
      po_level* P = &h->lev[l - 1];
      layout_at(lf, degrees[l], &L->layout);
      L->n = po_layout_dim(&L->layout);
      P->down_map = (int64_t*)malloc(sizeof(int64_t) * (size_t)(L->n + 1));
      P->n_coarse = L->n;
      po_coarse_to_fine_map(&P->layout, &L->layout, P->down_map);
      L->nnz = po_inherit(&P->csr, P->n, P->down_map, L->n, NULL, NULL, NULL);
      L->row_ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(L->n + 1));
      L->cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)(L->nnz + 1));
      L->vals = (double*)malloc(sizeof(double) * (size_t)(L->nnz + 1));
      po_inherit(&P->csr, P->n, P->down_map, L->n, L->row_ptr, L->cols, L->vals);
    }
    L->csr.n = L->n;
    L->csr.row_ptr = L->row_ptr;
    L->csr.cols = L->cols;
    L->csr.vals = L->vals;
  }
  for (int l = 0; l < nlev; ++l) {
    po_level* L = &h->lev[l];
    if (smoother == 1 && l + 1 < nlev) {
      L->bj = (double*)malloc(sizeof(double) * (size_t)(po_bj_size(&L->layout) + 1));
      if (po_bj_factor(&L->csr, &L->layout, L->bj, NULL) != 0) {
        po_hier_destroy(h);
        return NULL;
      }
      continue;
    }
    L->lu = (double*)malloc(sizeof(double) * (size_t)(L->nnz + 1));
    L->diag = (int64_t*)malloc(sizeof(int64_t) * (size_t)(L->n + 1));
    if (po_ilu0_factor(&L->csr, L->lu, L->diag) != 0) {
      po_hier_destroy(h);
      return NULL;
    }
  }
  return h;
}

void po_hier_destroy(po_hier* h) {
  if (!h) return;
  for (int l = 0; l < h->nlev; ++l) {
    po_level* L = &h->lev[l];
    free(L->row_ptr);
    free(L->cols);
    free(L->vals);
    free(L->lu);
    free(L->diag);
    free(L->down_map);
    free(L->bj);
  }
  free(h->lev);
  free(h);
}

int po_hier_nlev(const po_hier* h) { return h->nlev; }
int64_t po_hier_level_dim(const po_hier* h, int l) { return h->lev[l].n; }
int64_t po_hier_level_nnz(const po_hier* h, int l) { return h->lev[l].nnz; }
void po_hier_level_csr(const po_hier* h, int l, int64_t* row_ptr, int32_t* cols, double* vals) {
  const po_level* L = &h->lev[l];
  memcpy(row_ptr, L->row_ptr, sizeof(int64_t) * (size_t)(L->n + 1));
  memcpy(cols, L->cols, sizeof(int32_t) * (size_t)L->nnz);
  memcpy(vals, L->vals, sizeof(double) * (size_t)L->nnz);
}
void po_hier_level_ilu(const po_hier* h, int l, double* lu) {
  memcpy(lu, h->lev[l].lu, sizeof(double) * (size_t)h->lev[l].nnz);
}
long long po_hier_coarse_its(const po_hier* h) { return h->coarse_its; }

/* LevelHierarchy::coarse_solve (ILU-GMRES branch), plevels.hpp:185-197 */
static int coarse_solve(po_hier* h, const double* d, double* c) {
  const po_level* L = &h->lev[h->nlev - 1];
  lev_ctx ctx = {L};
  double* z = (double*)calloc((size_t)L->n + 1, sizeof(double));
  int its, conv;
  double rel;
  const int rc = po_gmres(lev_spmv, &ctx, lev_ilu, &ctx, L->n, d, z, h->coarse_maxit,
                          h->coarse_rtol, 0, c, &its, &rel, &conv);
  h->coarse_its += its;
  free(z);
  return rc;
}

/* LevelHierarchy::vcycle, plevels.hpp:170-183 */
int po_vcycle(po_hier* h, int l, const double* d, double* c) {
  if (l + 1 == h->nlev) return coarse_solve(h, d, c);
  const po_level* L = &h->lev[l];
  const int64_t n = L->n, nc = L->n_coarse;
  lev_ctx ctx = {L};
  double* zero = (double*)calloc((size_t)n + 1, sizeof(double));
  double* w = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* t = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* dc = (double*)malloc(sizeof(double) * (size_t)(nc + 1));
  double* cc = (double*)malloc(sizeof(double) * (size_t)(nc + 1));
  int its, conv;
  double rel;
  po_apply_fn pc = h->smoother == 1 ? lev_bj : lev_ilu;
  po_gmres(lev_spmv, &ctx, pc, &ctx, n, d, zero, h->smoother_iters, 0.0, 1, w, &its, &rel, &conv);
  po_csr_multiply(&L->csr, w, t);
  for (int64_t e = 0; e < n; ++e) t[e] = d[e] - t[e];
  for (int64_t i = 0; i < nc; ++i) dc[i] = t[L->down_map[i]];
  const int rc = po_vcycle(h, l + 1, dc, cc);
  /* w += prolong_vector(c): zero padding then an element-wise add */
  for (int64_t e = 0; e < n; ++e) t[e] = 0.0;
  for (int64_t i = 0; i < nc; ++i) t[L->down_map[i]] = cc[i];
  for (int64_t e = 0; e < n; ++e) w[e] = w[e] + t[e];
  po_gmres(lev_spmv, &ctx, pc, &ctx, n, d, w, h->smoother_iters, 0.0, 1, c, &its, &rel, &conv);
  free(zero);
  free(w);
  free(t);
  free(dc);
  free(cc);
  return rc;
}

typedef struct {
  po_hier* h;
  int vcycles;
} vc_ctx;

static void vc_apply(void* c, const double* x, double* y) {
  vc_ctx* v = (vc_ctx*)c;
  ++v->vcycles;
  po_vcycle(v->h, 0, x, y);
}

/* solve_system, plevels.hpp:217-239 (the FGMRES part) */
int po_solve(po_hier* h, const double* rhs, double outer_rtol, int outer_maxit, int restart,
             double* x, double* hist, int* its, long long* coarse_its, int* vcycles, double* rel,
             int* converged) {
  lev_ctx op = {&h->lev[0]};
  vc_ctx pc = {h, 0};
  h->coarse_its = 0;
  const int rc = po_fgmres(lev_spmv, &op, vc_apply, &pc, h->lev[0].n, rhs, outer_maxit, outer_rtol,
                           restart, x, hist, its, rel, converged);
  *coarse_its = h->coarse_its;
  *vcycles = pc.vcycles;
  return rc;
}

/* ---------------------------------------------------------------------------
 * Block-Jacobi over entity blocks (not in the reference: BASELINE.json names
 * "block-Jacobi smoothing with batched face-block inverses"; SURVEY.md §0
 * finding 4 makes it a labelled alternative to the ILU(0) smoother plugged
 * in at the same point, plevels.hpp:174). Blocks follow the DofLayout
 * numbering (dof_layout.hpp:56-85). Every operation is individually
 * rounded and ordered exactly like the device kernels (bjacobi.cu).
 * ------------------------------------------------------------------------- */
static void bj_shape(const po_layout* l, int* fb, int* eb, int64_t* eoff) {
  *fb = (int)face_block(l);
  *eb = (int)elem_block(l);
  *eoff = (int64_t)l->n_faces * *fb;
}

int64_t po_bj_size(const po_layout* l) {
  int fb, eb;
  int64_t eoff;
  bj_shape(l, &fb, &eb, &eoff);
  return (int64_t)l->n_faces * fb * fb + (int64_t)l->n_elements * eb * eb;
}

/* dense block extraction, partial-pivot LU, inverse column by column */
static int bj_block(const po_csr* a, int64_t s, int bs, double* d, double* inv, int* perm,
                    double* y) {
  for (int i = 0; i < bs * bs; ++i) d[i] = 0.0;
  for (int i = 0; i < bs; ++i)
    for (int64_t q = a->row_ptr[s + i]; q < a->row_ptr[s + i + 1]; ++q) {
      const int64_t c = a->cols[q];
      if (c >= s && c < s + bs) d[i * bs + (c - s)] = a->vals[q];
    }
  double amax = 0.0;
  for (int i = 0; i < bs * bs; ++i)
    if (fabs(d[i]) > amax) amax = fabs(d[i]);
  for (int i = 0; i < bs; ++i) perm[i] = i;
  for (int k = 0; k < bs; ++k) {
    int p = k;
    double m = fabs(d[k * bs + k]);
    for (int i = k + 1; i < bs; ++i)
      if (fabs(d[i * bs + k]) > m) {
        m = fabs(d[i * bs + k]);
        p = i;
      }
    if (!(m > 1e-14 * amax)) return 1;
    if (p != k) {
      for (int j = 0; j < bs; ++j) {
        const double t = d[k * bs + j];
        d[k * bs + j] = d[p * bs + j];
        d[p * bs + j] = t;
      }
      const int t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
    for (int i = k + 1; i < bs; ++i) {
      const double f = d[i * bs + k] / d[k * bs + k];
      d[i * bs + k] = f;
      for (int j = k + 1; j < bs; ++j) {
        const double t = f * d[k * bs + j];
        d[i * bs + j] = d[i * bs + j] - t;
      }
    }
  }
  for (int c = 0; c < bs; ++c) {
    for (int i = 0; i < bs; ++i) {
      double v = perm[i] == c ? 1.0 : 0.0;
      for (int j = 0; j < i; ++j) {
        const double t = d[i * bs + j] * y[j];
        v = v - t;
      }
      y[i] = v;
    }
    for (int i = bs - 1; i >= 0; --i) {
      double v = y[i];
      for (int j = i + 1; j < bs; ++j) {
        const double t = d[i * bs + j] * y[j];
        v = v - t;
      }
      y[i] = v / d[i * bs + i];
    }
    for (int i = 0; i < bs; ++i) inv[i * bs + c] = y[i];
  }
  return 0;
}

int po_bj_factor(const po_csr* a, const po_layout* l, double* inv, int64_t* bad_block) {
  int fb, eb;
  int64_t eoff;
  bj_shape(l, &fb, &eb, &eoff);
  const int mb = fb > eb ? fb : eb;
  double* d = (double*)malloc(sizeof(double) * (size_t)(mb * mb + 1));
  double* y = (double*)malloc(sizeof(double) * (size_t)(mb + 1));
  int* perm = (int*)malloc(sizeof(int) * (size_t)(mb + 1));
  int rc = 0;
  const int64_t nb = (int64_t)l->n_faces + l->n_elements;
  for (int64_t b = 0; b < nb && !rc; ++b) {
    const int face = b < l->n_faces;
    const int bs = face ? fb : eb;
    if (!bs) continue;
    const int64_t s = face ? b * fb : eoff + (b - l->n_faces) * eb;
    double* out = inv + (face ? b * fb * fb
                              : (int64_t)l->n_faces * fb * fb + (b - l->n_faces) * eb * eb);
    if (bj_block(a, s, bs, d, out, perm, y)) {
      rc = 1;
      if (bad_block) *bad_block = b;
      set_err("block-Jacobi: singular diagonal block");
    }
  }
  free(d);
  free(y);
  free(perm);
  return rc;
}

void po_bj_apply(const po_layout* l, const double* inv, const double* x, double* y) {
  int fb, eb;
  int64_t eoff;
  bj_shape(l, &fb, &eb, &eoff);
  const int64_t nb = (int64_t)l->n_faces + l->n_elements;
  for (int64_t b = 0; b < nb; ++b) {
    const int face = b < l->n_faces;
    const int bs = face ? fb : eb;
    const int64_t s = face ? b * fb : eoff + (b - l->n_faces) * eb;
    const double* m = inv + (face ? b * fb * fb
                                  : (int64_t)l->n_faces * fb * fb + (b - l->n_faces) * eb * eb);
    for (int i = 0; i < bs; ++i) {
      double acc = 0.0;
      for (int j = 0; j < bs; ++j) {
        const double t = m[i * bs + j] * x[s + j];
        acc = acc + t;
      }
      y[s + i] = acc;
    }
  }
}

/* ---------------------------------------------------------------------------
 * condensation, condense.hpp:57-97, with the Eigen-subset PartialPivLU
 * ------------------------------------------------------------------------- */
int po_condense(int n, const double* mat, const double* rhs, int ne, const int* elim,
                double* schur, double* reduced_rhs, double* coupling, double* erhs) {
  char* is_elim = (char*)calloc((size_t)n + 1, 1);
  for (int i = 0; i < ne; ++i) is_elim[elim[i]] = 1;
  int* keep = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  int nk = 0;
  for (int i = 0; i < n; ++i)
    if (!is_elim[i]) keep[nk++] = i;
#define M(i, j) mat[(size_t)(i) + (size_t)(j) * (size_t)n]
  if (ne == 0) {
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) schur[i + j * n] = M(i, j);
    for (int i = 0; i < n; ++i) reduced_rhs[i] = rhs[i];
    free(is_elim);
    free(keep);
    return 0;
  }
  double* lu = (double*)malloc(sizeof(double) * (size_t)ne * (size_t)ne);
  int* perm = (int*)malloc(sizeof(int) * (size_t)ne);
  for (int j = 0; j < ne; ++j)
    for (int i = 0; i < ne; ++i) lu[i + j * ne] = M(elim[i], elim[j]);
  double anorm = 0.0;
  for (int j = 0; j < ne; ++j) {
    double s = 0.0;
    for (int i = 0; i < ne; ++i) s += fabs(lu[i + j * ne]);
    if (s > anorm) anorm = s;
  }
  for (int i = 0; i < ne; ++i) perm[i] = i;
  for (int k = 0; k < ne; ++k) {
    int p = k;
    double pmax = fabs(lu[k + k * ne]);
    for (int i = k + 1; i < ne; ++i)
      if (fabs(lu[i + k * ne]) > pmax) {
        pmax = fabs(lu[i + k * ne]);
        p = i;
      }
    if (p != k) {
      for (int j = 0; j < ne; ++j) {
        const double t = lu[k + j * ne];
        lu[k + j * ne] = lu[p + j * ne];
        lu[p + j * ne] = t;
      }
      const int t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
    const double piv = lu[k + k * ne];
    if (piv == 0.0) continue;
    for (int i = k + 1; i < ne; ++i) lu[i + k * ne] = lu[i + k * ne] / piv;
    for (int j = k + 1; j < ne; ++j) {
      const double ukj = lu[k + j * ne];
      if (ukj == 0.0) continue;
      for (int i = k + 1; i < ne; ++i) {
        const double t = lu[i + k * ne] * ukj;
        lu[i + j * ne] = lu[i + j * ne] - t;
      }
    }
  }
  /* solve with nk+1 right-hand sides: [A_ek | b_e] */
  double* sol = (double*)malloc(sizeof(double) * (size_t)ne * (size_t)(nk + 1));
  for (int c = 0; c <= nk; ++c) {
    double* x = sol + (size_t)c * (size_t)ne;
    for (int i = 0; i < ne; ++i) x[i] = c < nk ? M(elim[perm[i]], keep[c]) : rhs[elim[perm[i]]];
    for (int i = 0; i < ne; ++i) {
      double s = x[i];
      for (int j = 0; j < i; ++j) {
        const double t = lu[i + j * ne] * x[j];
        s = s - t;
      }
      x[i] = s;
    }
    for (int i = ne - 1; i >= 0; --i) {
      double s = x[i];
      for (int j = i + 1; j < ne; ++j) {
        const double t = lu[i + j * ne] * x[j];
        s = s - t;
      }
      x[i] = s / lu[i + i * ne];
    }
  }
  /* rcond guard (exact inverse 1-norm, as in the Eigen subset) */
  int singular = 0;
  for (int i = 0; i < ne; ++i)
    if (lu[i + i * ne] == 0.0) singular = 1;
  if (!singular) {
    double inorm = 0.0;
    double* col = (double*)malloc(sizeof(double) * (size_t)ne);
    for (int c = 0; c < ne; ++c) {
      for (int i = 0; i < ne; ++i) col[i] = perm[i] == c ? 1.0 : 0.0;
      for (int i = 0; i < ne; ++i) {
        double s = col[i];
        for (int j = 0; j < i; ++j) s = s - lu[i + j * ne] * col[j];
        col[i] = s;
      }
      for (int i = ne - 1; i >= 0; --i) {
        double s = col[i];
        for (int j = i + 1; j < ne; ++j) s = s - lu[i + j * ne] * col[j];
        col[i] = s / lu[i + i * ne];
      }
      double s = 0.0;
      for (int i = 0; i < ne; ++i) s += fabs(col[i]);
      if (s > inorm) inorm = s;
    }
    free(col);
    const double rc = (anorm > 0.0 && inorm > 0.0 && isfinite(inorm)) ? (1.0 / anorm) / inorm : 0.0;
    if (rc < 1e-14) singular = 1;
  }
  if (singular) {
    free(is_elim);
    free(keep);
    free(lu);
    free(perm);
    free(sol);
    return set_err("condense: near-singular eliminated block");
  }
  for (int j = 0; j < nk; ++j)
    for (int i = 0; i < ne; ++i) coupling[i + j * ne] = sol[i + (size_t)j * ne];
  for (int i = 0; i < ne; ++i) erhs[i] = sol[i + (size_t)nk * ne];
  /* schur = A_kk - A_ke * coupling ; reduced = b_k - A_ke * elim_rhs (GEMM
   * with k ascending from 0, then one subtraction) */
  for (int j = 0; j <= nk; ++j)
    for (int i = 0; i < nk; ++i) {
      double s = 0.0;
      for (int k = 0; k < ne; ++k) {
        const double t = M(keep[i], elim[k]) * sol[k + (size_t)j * ne];
        s = s + t;
      }
      if (j < nk) schur[i + j * nk] = M(keep[i], keep[j]) - s;
      else reduced_rhs[i] = rhs[keep[i]] - s;
    }
#undef M
  free(is_elim);
  free(keep);
  free(lu);
  free(perm);
  free(sol);
  return 0;
}

/* dof_kind / structurally_coupled (assemble.hpp:25-46) with the layout's
 * component count: kinds 0..ncomp-1 velocity components, ncomp pressure */
static int dof_kind(const po_layout* l, int64_t g) {
  const int nc = ncomp(l);
  const int64_t fsz = (int64_t)l->n_faces * face_block(l);
  int within, nvel;
  if (g < fsz) {
    within = (int)(g % face_block(l));
    nvel = l->face_vel;
  } else {
    within = (int)((g - fsz) % elem_block(l));
    nvel = l->elem_vel;
  }
  return nvel > 0 && within < nc * nvel ? within / nvel : nc;
}

static int coupled(const po_layout* l, int ka, int kb) {
  const int nc = ncomp(l);
  const int av = ka != nc, bv = kb != nc;
  if (av && bv && ka != kb) return l->strategy == 2;
  if (!av && !bv) return l->strategy != 0 || l->scheme == 2; /* couples_pressures() */
  return 1;
}

int po_condense_assemble(int nelem, int n, const double* mats, const double* rhs, int ne,
                         const int* elim, const int64_t* kept, const po_layout* layout,
                         const po_csr* pat, double* vals, double* rhs_out) {
  const int nk = n - ne;
  double* schur = (double*)malloc(sizeof(double) * (size_t)nk * nk);
  double* rr = (double*)malloc(sizeof(double) * (size_t)nk);
  double* coup = (double*)malloc(sizeof(double) * (size_t)(ne > 0 ? ne : 1) * nk);
  double* er = (double*)malloc(sizeof(double) * (size_t)(ne > 0 ? ne : 1));
  int* kinds = (int*)malloc(sizeof(int) * (size_t)nk);
  int rc = 0;
  memset(vals, 0, sizeof(double) * (size_t)pat->row_ptr[pat->n]);
  memset(rhs_out, 0, sizeof(double) * (size_t)pat->n);
  for (int e = 0; e < nelem && !rc; ++e) {
    if (po_condense(n, mats + (size_t)e * n * n, rhs + (size_t)e * n, ne, elim, schur, rr, coup,
                    er)) {
      snprintf(g_err, sizeof g_err, "condense: near-singular eliminated block on element %d", e);
      rc = -1;
      break;
    }
    const int64_t* g = kept + (size_t)e * nk;
    for (int i = 0; i < nk; ++i) kinds[i] = dof_kind(layout, g[i]);
    for (int i = 0; i < nk && !rc; ++i)
      for (int j = 0; j < nk; ++j) {
        if (g[i] != g[j] && !coupled(layout, kinds[i], kinds[j])) continue;
        const double v = schur[i + (size_t)j * nk];
        if (!(v != 0.0 || g[i] == g[j])) continue;
        /* CsrMatrix::add: binary search in the sorted row (csr.hpp:47-61) */
        int64_t lo = pat->row_ptr[g[i]], hi = pat->row_ptr[g[i] + 1];
        while (lo < hi) {
          const int64_t mid = (lo + hi) / 2;
          if (pat->cols[mid] < g[j]) lo = mid + 1;
          else hi = mid;
        }
        if (lo == pat->row_ptr[g[i] + 1] || pat->cols[lo] != g[j]) {
          rc = set_err("CsrMatrix::add: entry outside the sparsity pattern");
          break;
        }
        vals[lo] += v;
      }
    for (int i = 0; i < nk; ++i) rhs_out[g[i]] += rr[i];
  }
  free(schur);
  free(rr);
  free(coup);
  free(er);
  free(kinds);
  return rc;
}

/* ---------------------------------------------------------------------------
 * DG assembly (assemble.hpp:177-346) from shared local terms: the structural
 * pattern (add_pattern_block per element, add_pattern_cross per interior
 * face, then from_pattern's sort: assemble.hpp:203-211, csr.hpp:30-44) and
 * the value scatter in the reference's order — every element's volume block
 * (element order), then every face's block in face order, exact zeros skipped
 * except on the diagonal (scatter_block, assemble.hpp:121-131); loads: the
 * element's volume load, then the face loads in face order.
 * ------------------------------------------------------------------------- */
static int64_t dg_pattern_pass(const po_layout* l, int nfaces, const int32_t* left,
                               const int32_t* right, int64_t* row_ptr, int32_t* cols) {
  const int eb = (int)elem_block(l);
  const int64_t n = po_layout_dim(l);
  const int ne = l->n_elements;
  /* neighbours per element (at most one face per neighbour) */
  int32_t* nb = (int32_t*)malloc(sizeof(int32_t) * (size_t)ne * 8 + 1);
  int* cnt = (int*)calloc((size_t)ne + 1, sizeof(int));
  for (int e = 0; e < ne; ++e) nb[(size_t)e * 8 + cnt[e]++] = e;
  for (int f = 0; f < nfaces; ++f)
    if (right[f] >= 0) {
      nb[(size_t)left[f] * 8 + cnt[left[f]]++] = right[f];
      nb[(size_t)right[f] * 8 + cnt[right[f]]++] = left[f];
    }
  int64_t total = 0;
  int* kinds = (int*)malloc(sizeof(int) * (size_t)eb);
  for (int i = 0; i < eb; ++i) kinds[i] = dof_kind(l, (int64_t)i);
  for (int e = 0; e < ne; ++e) {
    /* ascending neighbour order */
    int32_t* b = nb + (size_t)e * 8;
    for (int i = 1; i < cnt[e]; ++i)
      for (int j = i; j > 0 && b[j - 1] > b[j]; --j) {
        const int32_t t = b[j];
        b[j] = b[j - 1];
        b[j - 1] = t;
      }
    for (int r = 0; r < eb; ++r) {
      const int64_t row = (int64_t)e * eb + r;
      if (row_ptr) row_ptr[row] = total;
      for (int q = 0; q < cnt[e]; ++q)
        for (int c = 0; c < eb; ++c) {
          if (r != c || b[q] != e)
            if (!coupled(l, kinds[r], kinds[c])) continue;
          if (cols) cols[total] = (int32_t)((int64_t)b[q] * eb + c);
          ++total;
        }
    }
  }
  if (row_ptr) row_ptr[n] = total;
  free(nb);
  free(cnt);
  free(kinds);
  return total;
}

int64_t po_dg_pattern(const po_layout* l, int nfaces, const int32_t* left, const int32_t* right,
                      int64_t* row_ptr, int32_t* cols) {
  if (l->scheme != 2 || l->n_faces != 0 && l->face_vel) return set_err("dg pattern: dg layout expected"), -1;
  return dg_pattern_pass(l, nfaces, left, right, row_ptr, cols);
}

static int csr_add(const po_csr* pat, double* vals, int64_t i, int64_t j, double v) {
  int64_t lo = pat->row_ptr[i], hi = pat->row_ptr[i + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (pat->cols[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  if (lo == pat->row_ptr[i + 1] || pat->cols[lo] != j)
    return set_err("CsrMatrix::add: entry outside the sparsity pattern");
  vals[lo] += v;
  return 0;
}

static int scatter(const po_layout* l, const po_csr* pat, double* vals, const int64_t* g, int n,
                   const double* m, int ld) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (g[i] != g[j] && !coupled(l, dof_kind(l, g[i]), dof_kind(l, g[j]))) continue;
      const double v = m[(size_t)i + (size_t)j * ld];
      if (!(v != 0.0 || g[i] == g[j])) continue;
      if (csr_add(pat, vals, g[i], g[j], v)) return -1;
    }
  return 0;
}

int po_dg_assemble(const po_layout* l, int nfaces, const int32_t* left, const int32_t* right,
                   const double* vol, const double* vrhs, const double* fmat, const double* frhs,
                   const po_csr* pat, double* vals, double* rhs) {
  const int eb = (int)elem_block(l), n2 = 2 * eb;
  int64_t* g = (int64_t*)malloc(sizeof(int64_t) * (size_t)n2);
  memset(vals, 0, sizeof(double) * (size_t)pat->row_ptr[pat->n]);
  memset(rhs, 0, sizeof(double) * (size_t)pat->n);
  int rc = 0;
  for (int e = 0; e < l->n_elements && !rc; ++e) {
    for (int i = 0; i < eb; ++i) g[i] = (int64_t)e * eb + i;
    rc = scatter(l, pat, vals, g, eb, vol + (size_t)e * eb * eb, eb);
    for (int i = 0; i < eb; ++i) rhs[g[i]] += vrhs[(size_t)e * eb + i];
  }
  for (int f = 0; f < nfaces && !rc; ++f) {
    const int ns = right[f] >= 0 ? 2 : 1;
    for (int s = 0; s < ns; ++s)
      for (int i = 0; i < eb; ++i) g[s * eb + i] = (int64_t)(s ? right[f] : left[f]) * eb + i;
    rc = scatter(l, pat, vals, g, ns * eb, fmat + (size_t)f * n2 * n2, n2);
    for (int s = 0; s < ns; ++s)
      for (int i = 0; i < eb; ++i) rhs[g[s * eb + i]] += frhs[(size_t)f * n2 + s * eb + i];
  }
  free(g);
  return rc;
}
