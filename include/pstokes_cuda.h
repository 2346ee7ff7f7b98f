/* include/pstokes_cuda.h — C ABI of the B200 solver hot path.
 *
 * Drop-in boundary for the solver path of the pstokes reference
 * (/root/reference/proj/include/pstokes). The reference has no FFI: its hot
 * path sits behind header-only C++ functions and the ApplyFn callback type
 * (gmres.hpp:17). Each entry point below names the reference interface it
 * replaces; include/pstokes_b200/*.hpp wraps them in the reference's C++
 * signatures and INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - every function returns 0 on success, a PSCU_E* code otherwise; the
 *    message of the last failure on the calling thread is pscu_last_error();
 *  - `mem` arguments: PSCU_HOST = host pointers (copied in/out inside the
 *    call), PSCU_DEVICE = device pointers already on the context's GPU;
 *  - all work is ordered on the context's stream; calls on one context must
 *    be serialised by the caller (the reference is single-threaded);
 *  - there is no CPU fallback: without a usable sm_100 device pscu_create
 *    fails with PSCU_ENODEV.
 */
#ifndef PSTOKES_CUDA_H
#define PSTOKES_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PSCU_OK = 0,
  PSCU_EINVAL = 1,     /* std::invalid_argument in the reference */
  PSCU_ESINGULAR = 2,  /* std::runtime_error: singular block / zero pivot */
  PSCU_ECUDA = 3,      /* CUDA runtime failure */
  PSCU_ENODEV = 4,     /* no usable device */
  PSCU_ENOMEM = 5
};
enum { PSCU_HOST = 0, PSCU_DEVICE = 1 };
enum { PSCU_SMOOTHER_ILU0 = 0, PSCU_SMOOTHER_BJACOBI = 1 };
enum { PSCU_COARSE_LU = 0, PSCU_COARSE_ILU_GMRES = 1 };

typedef struct pscu_ctx pscu_ctx;
typedef struct pscu_mat pscu_mat;
typedef struct pscu_ilu pscu_ilu;
typedef struct pscu_hier pscu_hier;
typedef struct pscu_bj pscu_bj;

/* DofLayout (dof_layout.hpp:56-85). scheme: 0 hho-dp, 1 hho-hp, 2 dg;
 * strategy: 0 uncond, 1 v-cond, 2 vp-cond. dim: space dimension, 2 (the
 * reference; 0 also reads as 2) or 3 (BASELINE.json configs 3/5: velocity
 * blocks have three components, face modes dim P^k(F) = (k+1)(k+2)/2). */
typedef struct {
  int scheme, strategy, k;
  int n_faces, n_elements;
  int face_vel, face_press, elem_vel, elem_press;
  int dim;
} pscu_layout;

/* LevelConfig (plevels.hpp:23-42) minus the degrees, plus the smoother kind. */
typedef struct {
  int smoother;        /* PSCU_SMOOTHER_* (reference: ILU(0)-GMRES) */
  int smoother_iters;  /* V(s,s) */
  int coarse;          /* PSCU_COARSE_* */
  double coarse_rtol;
  int coarse_maxit;
} pscu_level_cfg;

/* SolverReport (gmres.hpp:19-27) + device timings. */
typedef struct {
  int outer_its;
  long long coarse_its;
  int vcycles;
  double rel_residual;
  int converged;
  double t_setup;      /* hierarchy setup, seconds (device events) */
  double t_solve;      /* setup + FGMRES, seconds: the reference's t_solve */
} pscu_report;

const char* pscu_last_error(void);
int pscu_version(void);

/* context ---------------------------------------------------------------- */
int pscu_create(int device, pscu_ctx** out);
/* Device-list form: one context per listed device, written
 * to out[0..ndev). A host that drives several GPUs from one process gives
 * each context its own host thread (calls on one context are serialised by
 * the caller, the reference's single-threaded contract); the z-slab driver
 * (one process per GPU) passes its one local device. All-or-nothing: on
 * failure no context is left allocated. */
int pscu_create_devices(const int* devices, int ndev, pscu_ctx** out);
int pscu_destroy(pscu_ctx* ctx);
int pscu_synchronize(pscu_ctx* ctx);
/* Kernel-launch counter (every kernel this library enqueued). */
long long pscu_launch_count(const pscu_ctx* ctx);
/* Device-timeline timer: CUDA events on the context stream (start syncs the
 * stream first; stop waits for the stop event). */
int pscu_timer_start(pscu_ctx* ctx);
int pscu_timer_stop(pscu_ctx* ctx, double* ms);
/* Live per-kernel-class timing (events around every launch of the class on
 * the context stream) with the algorithmic bytes each launch moves.
 * class: 0 ILU(0) apply, 1 SpMV, 2 MGS Arnoldi step, 3 other, 4 block-Jacobi apply.
 * pscu_profile(ctx, 1) clears and starts recording. */
int pscu_profile(pscu_ctx* ctx, int enable);
int pscu_profile_read(pscu_ctx* ctx, int cls, long long* count, double* ms, double* bytes);

/* CsrMatrix (csr.hpp:19-24) ----------------------------------------------- */
int pscu_mat_create(pscu_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* cols,
                    const double* vals, int mem, pscu_mat** out);
int pscu_mat_destroy(pscu_mat* m);
int pscu_mat_dims(const pscu_mat* m, int64_t* n, int64_t* nnz);
int pscu_mat_download(pscu_ctx* ctx, const pscu_mat* m, int64_t* row_ptr, int32_t* cols,
                      double* vals);
/* Dense face-block storage of the same CsrMatrix (operators whose structural
 * pattern is made of dense bs x bs blocks: 3D HHO-hp vp-cond). Block row f
 * covers rows [f bs, (f+1) bs); bcols ascending per block row; vals holds the
 * blocks column-major (entry (r, c) of block q at q bs^2 + c bs + r). Every
 * operation on a pscu_mat accepts either storage; results are identical to
 * the CSR expansion (pscu_mat_download returns it), bit for bit. */
int pscu_bsr_create(pscu_ctx* ctx, int64_t nb, int bs, const int64_t* brow_ptr,
                    const int32_t* bcols, const double* vals, int mem, pscu_mat** out);
/* 0 for CSR storage, else the block size. */
int pscu_mat_block_size(const pscu_mat* m);
/* The block pattern and values of a block-stored operator (host, nullable). */
int pscu_bsr_download(pscu_ctx* ctx, const pscu_mat* m, int64_t* brow_ptr, int32_t* bcols,
                      double* vals);
/* CsrMatrix::multiply (csr.hpp:68-74): y = A x, per-row sequential sums. */
int pscu_spmv(pscu_ctx* ctx, const pscu_mat* a, const double* x, double* y, int mem);

/* Ilu0 (ilu0.hpp:19-65): factorisation on the device, bit-identical. ------ */
int pscu_ilu0_create(pscu_ctx* ctx, const pscu_mat* a, pscu_ilu** out);
int pscu_ilu0_destroy(pscu_ilu* p);
int pscu_ilu0_factors(pscu_ctx* ctx, const pscu_ilu* p, double* lu_host);
int pscu_ilu0_apply(pscu_ctx* ctx, const pscu_ilu* p, const double* x, double* y, int mem);

/* Block-Jacobi over the layout's entity blocks (face f: [f fb, (f+1) fb),
 * element e: [F + e eb, ...), dof_layout.hpp:56-85). Not in the reference:
 * BASELINE.json's "block-Jacobi smoothing with batched face-block
 * inverses", plugged in as the smoother's preconditioner where the
 * reference uses Ilu0 (plevels.hpp:174; pscu_level_cfg.smoother =
 * PSCU_SMOOTHER_BJACOBI). Dense partial-pivot LU + inverse per block;
 * PSCU_ESINGULAR names a singular block (HHO-dp mean-pressure blocks). */
int pscu_bj_create(pscu_ctx* ctx, const pscu_mat* a, const pscu_layout* layout, pscu_bj** out);
int pscu_bj_destroy(pscu_bj* p);
int pscu_bj_apply(pscu_ctx* ctx, const pscu_bj* p, const double* x, double* y, int mem);

/* layouts and transfers (dof_layout.hpp:87-126, plevels.hpp:47-113) ------- */
int pscu_layout_make(int scheme, int strategy, int k, int n_faces, int n_elements,
                     pscu_layout* out);
/* 3D generalisation of make_layout (no reference: mesh.hpp is 2D): hho-hp
 * vp-cond (face blocks [vx | vy | vz | p], no element unknowns) or dg uncond
 * (element blocks [vx | vy | vz | p] of dim P^k(3D) modes, no face unknowns). */
int pscu_layout_make3(int scheme, int strategy, int k, int n_faces, int n_elements,
                      pscu_layout* out);
int64_t pscu_layout_dim(const pscu_layout* l);
int pscu_coarse_to_fine(const pscu_layout* fine, const pscu_layout* coarse, int64_t* map);
/* inherit_matrix (plevels.hpp:93-113) as a device gather. */
int pscu_inherit(pscu_ctx* ctx, const pscu_mat* fine, const pscu_layout* lf,
                 const pscu_layout* lc, pscu_mat** out);

/* Krylov (gmres.hpp:103-173) on a device operator ------------------------ */
/* gmres with ILU(0) preconditioner (pc may be NULL); side 0 right, 1 left. */
int pscu_gmres(pscu_ctx* ctx, const pscu_mat* a, const pscu_ilu* pc, const double* rhs,
               const double* x0, int max_it, double rtol, int side, double* x, int* its,
               double* rel, int* converged, int mem);
/* fgmres with a fixed ILU(0) preconditioner (pc NULL = identity). */
int pscu_fgmres(pscu_ctx* ctx, const pscu_mat* a, const pscu_ilu* pc, const double* rhs,
                int max_it, double rtol, double* x, int* its, double* rel, int* converged,
                int mem);

/* p-multilevel hierarchy (plevels.hpp:115-239) ---------------------------- */
int pscu_hier_create(pscu_ctx* ctx, const pscu_mat* fine, const pscu_layout* lf,
                     const int* degrees, int nlev, const pscu_level_cfg* cfg, pscu_hier** out);
int pscu_hier_destroy(pscu_hier* h);
int pscu_hier_nlev(const pscu_hier* h);
const pscu_mat* pscu_hier_level_mat(const pscu_hier* h, int l);
const pscu_ilu* pscu_hier_level_ilu(const pscu_hier* h, int l);
int pscu_vcycle(pscu_ctx* ctx, pscu_hier* h, int level, const double* d, double* c, int mem);
long long pscu_hier_coarse_its(const pscu_hier* h);
void pscu_hier_reset(pscu_hier* h);
/* solve_system (plevels.hpp:217-239) on an assembled system: FGMRES
 * preconditioned by one V-cycle per iteration. restart = 0 reproduces the
 * reference (unrestarted); hist (nullable, host) receives |g_{j+1}|/||b||. */
int pscu_solve(pscu_ctx* ctx, pscu_hier* h, const double* rhs, double rtol, int maxit,
               int restart, double* x, double* hist, pscu_report* rep, int mem);
/* One-call drop-in for solve_system: uploads the CSR system, builds the
 * hierarchy, solves, downloads x (host buffers; copies are timed inside). */
int pscu_solve_system(pscu_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* cols,
                      const double* vals, const double* rhs, const pscu_layout* lf,
                      const int* degrees, int nlev, const pscu_level_cfg* cfg, double rtol,
                      int maxit, int restart, double* x, double* hist, pscu_report* rep);

/* static condensation (condense.hpp:57-97, assemble.hpp:121-169) --------- */
/* Batched condense_element over `nelem` elements with identical local size n
 * and elimination list. mats: nelem column-major n x n blocks; rhs: nelem x n.
 * Outputs (nullable): schur nelem x nk x nk, reduced_rhs nelem x nk,
 * elim_coupling nelem x ne x nk, elim_rhs nelem x ne (column-major blocks).
 * On a near-singular block returns PSCU_ESINGULAR and *bad_element. */
int pscu_condense_batch(pscu_ctx* ctx, int nelem, int n, const double* mats, const double* rhs,
                        int n_elim, const int* elim, double* schur, double* reduced_rhs,
                        double* elim_coupling, double* elim_rhs, int* bad_element, int mem);
/* assemble_hho on the device (assemble.hpp:136-172): batched condensation
 * of the local blocks, then the CSR value scatter and the reduced-load rhs
 * over the given structural pattern (the element-order sums of the
 * reference, bit for bit). Host producers build mats/rhs/elim/kept/pattern
 * (include/pstokes_host.h). The recovery data (elim_coupling nelem x ne x
 * nk column-major blocks, elim_rhs nelem x ne; nullable) is returned in the
 * memory space mem names. */
int pscu_condense_assemble(pscu_ctx* ctx, int nelem, int n, const double* mats,
                           const double* rhs, int n_elim, const int* elim,
                           const int64_t* kept_global, int64_t dim, const int64_t* row_ptr,
                           const int32_t* cols, const pscu_layout* layout, int mem,
                           pscu_mat** out, double* rhs_out, double* elim_coupling,
                           double* elim_rhs);
/* assemble_hho into face-block storage, streamed over element batches
 * (3D: the local blocks of all elements do not fit in memory at once):
 * begin allocates the zero operator over the block pattern and a zero load;
 * each add condenses a batch (condense_element, bitwise in the order of the
 * reference's PartialPivLU / GEMM) and scatters the Schur blocks and reduced
 * loads (assemble.hpp:121-131, 164-169; two-term sums, order-free).
 * efaces: nelem x nfe global face ids of the batch; keep_pos: n_keep x
 * (local face, offset in the face block) of the retained local dofs. e0 is
 * the global id of the batch's first element (error messages). Recovery data
 * (elim_coupling nelem x ne x nk, elim_rhs nelem x ne) is optional. */
int pscu_assembly_begin(pscu_ctx* ctx, int64_t nb, int bs, const int64_t* brow_ptr,
                        const int32_t* bcols, pscu_mat** out);
int pscu_assembly_add(pscu_ctx* ctx, pscu_mat* m, int e0, int nelem, int n, const double* mats,
                      const double* rhs, int n_elim, const int* elim, const int32_t* efaces,
                      int nfe, const int32_t* keep_pos, double* elim_coupling, double* elim_rhs,
                      int mem);
int pscu_assembly_rhs(pscu_ctx* ctx, const pscu_mat* m, double* rhs, int mem);
/* Shards of a face-block operator (z-slab partition, paper_2009_13840_b200/
 * zslab.py): nb owned block rows over ncb block columns
 * (ghost faces of the neighbour slabs included, numbered in global order);
 * the diagonal block of block row b is block column b + diag_off. The local
 * assembly takes per element the block row of each face (-1: held by
 * another shard, skipped) and its block column. */
int pscu_bsr_create_local(pscu_ctx* ctx, int64_t nb, int64_t ncb, int bs, int64_t diag_off,
                          const int64_t* brow_ptr, const int32_t* bcols, const double* vals,
                          int mem, pscu_mat** out);
int pscu_assembly_begin_local(pscu_ctx* ctx, int64_t nb, int64_t ncb, int bs, int64_t diag_off,
                              const int64_t* brow_ptr, const int32_t* bcols, pscu_mat** out);
int pscu_assembly_add_local(pscu_ctx* ctx, pscu_mat* m, int e0, int nelem, int n,
                            const double* mats, const double* rhs, int n_elim, const int* elim,
                            const int32_t* erows, const int32_t* ecols, int nfe,
                            const int32_t* keep_pos, int mem);
/* Page-locked host staging buffers (cudaHostAlloc): producers write local
 * blocks there so the batch uploads run at full PCIe/C2C bandwidth. */
int pscu_host_alloc(int64_t bytes, void** out);
int pscu_host_free(void* p);
/* pscu_solve_system on a face-block operator (host buffers, copies timed). */
int pscu_solve_system_bsr(pscu_ctx* ctx, int64_t nb, int bs, const int64_t* brow_ptr,
                          const int32_t* bcols, const double* vals, const double* rhs,
                          const pscu_layout* lf, const int* degrees, int nlev,
                          const pscu_level_cfg* cfg, double rtol, int maxit, int restart,
                          double* x, double* hist, pscu_report* rep);

/* DG block storage (3D DG, BASELINE.json config 4: the reference's BR2
 * assemble_dg, assemble.hpp:177-346, with three velocity components). The
 * operator couples element blocks [ux | uy | uz | p] of nm modes each but
 * not velocity components with each other (DofLayout::couples_components,
 * dof_layout.hpp:79-84), so each block stores its 10 nm^2 structural
 * entries as column-major panels: velocity component c's rows (nm x 2nm,
 * columns [u_c | p]) at c 2nm^2, pressure rows (nm x 4nm, [ux|uy|uz|p]) at
 * 6nm^2. Block row e covers rows [e 4nm, (e+1) 4nm); bcols ascending; vals
 * NULL = zero. Every pscu_mat operation accepts it, bit-identical to the
 * CSR expansion (pscu_mat_download). nm: 4, 10, 20 or 35 (k = 1..4). */
int pscu_dgb_create(pscu_ctx* ctx, int64_t nb, int nm, const int64_t* brow_ptr,
                    const int32_t* bcols, const double* vals, int mem, pscu_mat** out);
/* 0 unless DG block storage, else the modes per component. */
int pscu_mat_dg_modes(const pscu_mat* m);
/* Writes count values at offset of any storage's value array (streamed
 * producers fill an operator block range by block range). */
int pscu_mat_set_values(pscu_ctx* ctx, pscu_mat* m, int64_t offset, int64_t count,
                        const double* vals, int mem);
/* pscu_solve_system on a DG block-stored operator (host buffers, timed). */
int pscu_solve_system_dgb(pscu_ctx* ctx, int64_t nb, int nm, const int64_t* brow_ptr,
                          const int32_t* bcols, const double* vals, const double* rhs,
                          const pscu_layout* lf, const int* degrees, int nlev,
                          const pscu_level_cfg* cfg, double rtol, int maxit, int restart,
                          double* x, double* hist, pscu_report* rep);

/* ElementCondensation::recover (condense.hpp:28-38) for all elements:
 * locals[e] (n) from global x through kept_global (nelem x nk). */
int pscu_recover_batch(pscu_ctx* ctx, int nelem, int n, int n_elim, const int* elim,
                       const int64_t* kept_global, const double* elim_coupling,
                       const double* elim_rhs, const double* x, double* locals, int mem);

/* error_norms (errors.hpp:32-117) for the HHO schemes, batched: adds the
 * squared L2 errors {u, grad u (reconstruction), p, div u} of nelem elements
 * to acc[4] in the reference's accumulation order (element, point,
 * component). tables: psh_error_tables rows of those elements; locals: their
 * recovered local vectors (pscu_recover_batch), dims from psh_error_tables.
 * Call per batch in element order from acc = {0,0,0,0}; the norms are the
 * square roots of the final acc. With mem == PSCU_DEVICE all three pointers
 * are device memory. */
int pscu_error_accumulate(pscu_ctx* ctx, const int32_t* dims, int nelem, const double* tables,
                          const double* locals, double* acc, int mem);

/* The 3D HHO-hp local element blocks on the device (the host producer's
 * build_local, psh3_local_blocks, bit for bit; hho_local.hpp:26-318 in 3D):
 * nelem elements given by their hex vertex ids, element faces and signs
 * (psh3_device_inputs, batch-relative), the mesh vertices (nv x 3) and face
 * table (nfaces x {4 vertex ids, tag}), the Gauss-Legendre rule gl (nq1
 * points, then nq1 weights) and, for data 3, the random modal coefficients.
 * mats (nelem x n x n, column-major) and rhs (nelem x n) as the host
 * producer writes them. data: 0 or 3 (data 4 needs the host's libm). */
int pscu_local_blocks3(pscu_ctx* ctx, int k, int data, double eta, int nq1, const double* gl,
                       int64_t nv, const double* xyz, int64_t nfaces, const int32_t* ftab,
                       int nelem, const int32_t* hex, const int32_t* ef, const int32_t* es,
                       const double* coef, double* mats, double* rhs, int mem);

#ifdef __cplusplus
}
#endif

#endif
