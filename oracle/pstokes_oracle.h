/* oracle/pstokes_oracle.h — TEST INFRASTRUCTURE ONLY (see pstokes_oracle.c).
 *
 * Plain-C restatement of the reference solver hot path:
 * CSR SpMV, ILU(0), GMRES/FGMRES with modified Gram-Schmidt, p-level layouts,
 * transfers, operator inheritance, the V-cycle, and element condensation.
 * Reductions follow include/eigen_subset/Eigen/Dense (the arithmetic the
 * reference is compiled with here), so results are bit-identical to the
 * reference built in oracle/_ref. Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline/reference arm may load this library. */
#ifndef PSTOKES_ORACLE_H
#define PSTOKES_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t n;
  const int64_t* row_ptr;
  const int32_t* cols;
  const double* vals;
} po_csr;

/* DofLayout (dof_layout.hpp:56-85) */
typedef struct {
  int scheme;   /* 0 hho-dp, 1 hho-hp, 2 dg */
  int strategy; /* 0 uncond, 1 v-cond, 2 vp-cond */
  int k;
  int n_faces, n_elements;
  int face_vel, face_press, elem_vel, elem_press;
  int dim;      /* space dimension: 2 (the reference; 0 reads as 2) or 3 */
} po_layout;

typedef void (*po_apply_fn)(void* ctx, const double* x, double* y);

const char* po_last_error(void);

int po_make_layout(int scheme, int strategy, int k, int n_faces, int n_elements, po_layout* out);
/* 3D generalisation (BASELINE.json configs 3/5; no reference): hho-hp
 * vp-cond, face blocks [vx | vy | vz | p] of dim P^k(F) = (k+1)(k+2)/2
 * modes each, no element unknowns. */
int po_make_layout3(int scheme, int strategy, int k, int n_faces, int n_elements, po_layout* out);
int64_t po_layout_dim(const po_layout* l);
int po_coarse_to_fine_map(const po_layout* fine, const po_layout* coarse, int64_t* map);

double po_dot(const double* x, const double* y, int64_t n);
void po_csr_multiply(const po_csr* a, const double* x, double* y);
int po_ilu0_factor(const po_csr* a, double* lu, int64_t* diag);
void po_ilu0_apply(const po_csr* a, const double* lu, const int64_t* diag, const double* x,
                   double* y);
/* Returns coarse nnz; with null outputs only counts. */
int64_t po_inherit(const po_csr* fine, int64_t n_fine, const int64_t* c2f, int64_t n_coarse,
                   int64_t* row_ptr, int32_t* cols, double* vals);

int po_gmres(po_apply_fn op, void* op_ctx, po_apply_fn pc, void* pc_ctx, int64_t n,
             const double* rhs, const double* x0, int max_it, double rtol, int left, double* x,
             int* its, double* rel, int* converged);
int po_fgmres(po_apply_fn op, void* op_ctx, po_apply_fn pc, void* pc_ctx, int64_t n,
              const double* rhs, int max_it, double rtol, int restart, double* x, double* hist,
              int* its, double* rel, int* converged);

/* Block-Jacobi preconditioner over the entity blocks of a DofLayout
 * (BASELINE.json's smoother; the reference smooths with ILU(0)-GMRES).
 * Face f owns [f*fb, (f+1)*fb), element e owns [F + e*eb, F + (e+1)*eb).
 * inv: n_faces*fb*fb + n_elements*eb*eb doubles, row-major per block.
 * Returns 0, or 1 with *bad_block on a singular block (pivot <= 1e-14 max). */
int64_t po_bj_size(const po_layout* l);
int po_bj_factor(const po_csr* a, const po_layout* l, double* inv, int64_t* bad_block);
void po_bj_apply(const po_layout* l, const double* inv, const double* x, double* y);

typedef struct po_hier po_hier;
/* Builds levels below `fine` (layout lf): coarse_to_fine maps, inherited
 * operators, ILU(0) per level; the coarsest level uses ILU-GMRES. */
po_hier* po_hier_create(const po_csr* fine, const po_layout* lf, const int* degrees, int nlev,
                        int smoother_iters, double coarse_rtol, int coarse_maxit);
/* The same with the smoother's preconditioner chosen: 0 ILU(0) (the
 * reference), 1 block-Jacobi (every level but the coarsest). */
po_hier* po_hier_create_ex(const po_csr* fine, const po_layout* lf, const int* degrees, int nlev,
                           int smoother_iters, double coarse_rtol, int coarse_maxit, int smoother);
void po_hier_destroy(po_hier* h);
int po_hier_nlev(const po_hier* h);
int64_t po_hier_level_dim(const po_hier* h, int l);
int64_t po_hier_level_nnz(const po_hier* h, int l);
void po_hier_level_csr(const po_hier* h, int l, int64_t* row_ptr, int32_t* cols, double* vals);
void po_hier_level_ilu(const po_hier* h, int l, double* lu);
int po_vcycle(po_hier* h, int l, const double* d, double* c);
long long po_hier_coarse_its(const po_hier* h);
int po_solve(po_hier* h, const double* rhs, double outer_rtol, int outer_maxit, int restart,
             double* x, double* hist, int* its, long long* coarse_its, int* vcycles, double* rel,
             int* converged);

/* assemble_hho's value pass (assemble.hpp:121-131,164-169) over all
 * elements: condense_element per element (po_condense), then the Schur
 * scatter into the structural CSR pattern in element order (exact zeros
 * skipped except on the diagonal) and the reduced-load accumulation.
 * kept: nelem x nk retained global ids in local keep order. Returns 0, or
 * -1 with po_last_error (a singular block or an entry outside the pattern). */
int po_condense_assemble(int nelem, int n, const double* mats, const double* rhs, int n_elim,
                         const int* elim, const int64_t* kept, const po_layout* layout,
                         const po_csr* pattern, double* vals, double* rhs_out);

/* condense_element (condense.hpp:57-97) on one column-major n x n block. */
int po_condense(int n, const double* mat, const double* rhs, int n_elim, const int* elim,
                double* schur, double* reduced_rhs, double* elim_coupling, double* elim_rhs);

/* DG in 3D (config 4; assemble.hpp:177-346 restated with three velocity
 * components): the structural CSR pattern (two-pass: null outputs count)
 * and the reference-order value scatter of shared local terms (volume
 * blocks nelem x (4ne)^2, face blocks nfaces x (8ne)^2 over [left | right],
 * column-major; loads alike). Returns the nnz / 0, or -1 with po_last_error. */
int64_t po_dg_pattern(const po_layout* l, int nfaces, const int32_t* left, const int32_t* right,
                      int64_t* row_ptr, int32_t* cols);
int po_dg_assemble(const po_layout* l, int nfaces, const int32_t* left, const int32_t* right,
                   const double* vol, const double* vrhs, const double* fmat, const double* frhs,
                   const po_csr* pattern, double* vals, double* rhs);

#ifdef __cplusplus
}
#endif

#endif
