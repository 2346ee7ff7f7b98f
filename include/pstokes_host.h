/* include/pstokes_host.h — host-side input producer of the B200 build.
 *
 * Produces the inputs of the device hot path the way the reference's
 * assembly front end does (mesh.hpp, quadrature.hpp, basis.hpp,
 * hho_local.hpp, condense.hpp:44-55, dof_layout.hpp:87-126,
 * assemble.hpp:25-172): a 2D mesh with first-seen face numbering, the
 * per-element HHO local Stokes blocks and loads, the eliminated-dof list,
 * the retained global dof ids per element and the structural CSR pattern.
 * Condensation and the value assembly then run on the GPU
 * (pscu_condense_batch / pscu_assemble in pstokes_cuda.h).
 *
 * Conventions as in pstokes_cuda.h: 0 = success, message via
 * psh_last_error(). Arrays returned by accessors are owned by the object.
 */
#ifndef PSTOKES_HOST_H
#define PSTOKES_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct psh_mesh psh_mesh;
typedef struct psh_system psh_system;

enum { PSH_SIDE_LEFT = 0, PSH_SIDE_RIGHT = 1, PSH_SIDE_TOP = 2, PSH_SIDE_BOTTOM = 3 };
enum { PSH_DATA_ZERO = 0, PSH_DATA_EXP = 1, PSH_DATA_SINCOS = 2 };

const char* psh_last_error(void);

/* Unit square [0,1]^2, n x n cells, vertex (i,j) at (i/n, j/n), interior
 * vertices jittered by frac*(1/n)*SplitMix64(seed).sym() (x then y, j outer,
 * i inner); tri != 0 splits every cell along its (i,j)-(i+1,j+1) diagonal.
 * BASELINE.json configs 1-2. */
int psh_mesh_unit_square(int n, int tri, double frac, uint64_t seed, int neumann_side,
                         psh_mesh** out);
/* Reference families on (-1,1)^2 (mesh.hpp:349-362, 452-459; study.hpp:20-32):
 * "trapz" (distortion 0.1), "quad", "tri". */
int psh_mesh_family(const char* family, int n, int neumann_side, psh_mesh** out);
void psh_mesh_destroy(psh_mesh* m);
/* out[0..2] = vertices, elements, faces */
void psh_mesh_counts(const psh_mesh* m, int64_t* out);
/* faces: 5 ints per face (a, b, left, right, tag 0 interior/1 Dirichlet/2 Neumann) */
void psh_mesh_faces(const psh_mesh* m, int32_t* faces);
void psh_mesh_vertices(const psh_mesh* m, double* xy);
/* Wire formats, byte-compatible with the reference's writers: pmesh2 v1
 * mesh files (write_mesh / read_mesh, mesh.hpp:535-645; nf = 0 lets the
 * reader derive the faces) and the MatrixMarket coordinate export of a CSR
 * operator (write_matrix_market, csr.hpp:98-111; 1-based, precision 17). */
int psh_mesh_write(const psh_mesh* m, const char* path);
int psh_mesh_read(const char* path, psh_mesh** out);
int psh_write_matrix_market(int64_t n, const int64_t* row_ptr, const int32_t* cols,
                            const double* vals, const char* path);

/* Local blocks + layout + pattern (assemble_hho front end). scheme 0 hho-dp,
 * 1 hho-hp; strategy 0 uncond, 1 v-cond, 2 vp-cond; eta <= 0 selects the
 * default 3(k+1)^2 (hho_local.hpp:19). nthreads <= 0: all cores. */
/* error_norms (errors.hpp:32-117) point tables, element-major from e0: per
 * element the reconstruction P (nrec x ns, column-major) then, per point of
 * the degree-2(k+2)+3 element rule, {w, phi[nrec], dphi/dx[nrec],
 * dphi/dy[nrec], u_x, u_y, du_x/dx, du_x/dy, du_y/dx, du_y/dy, p} (the
 * degree-(k+1) reconstruction basis, the closed-form field of data 1 or 2).
 * dims (11) = {nrec, ns, nq, qstride, per_elem, ne, nf, np, nloc, nfc,
 * hybrid}; out == NULL fills dims only. Feeds pscu_error_accumulate. */
int psh_error_tables(const psh_mesh* m, int scheme, int k, int data, int e0, int nelem,
                     int nthreads, double* out, int32_t* dims);

int psh_build(const psh_mesh* m, int scheme, int strategy, int k, int data, double eta,
              int nthreads, psh_system** out);
void psh_system_destroy(psh_system* s);
/* info[0..13]: nelem, n_local, n_elim, n_keep, dim, nnz, scheme, strategy,
 * k, n_faces, face_vel, face_press, elem_vel, elem_press */
void psh_system_info(const psh_system* s, int64_t* info);
const double* psh_local_mats(const psh_system* s);  /* nelem x n x n, column-major */
const double* psh_local_rhs(const psh_system* s);   /* nelem x n */
const int32_t* psh_elim(const psh_system* s);       /* n_elim local ids */
const int64_t* psh_kept_global(const psh_system* s); /* nelem x n_keep */
const int64_t* psh_row_ptr(const psh_system* s);    /* dim + 1 */
const int32_t* psh_cols(const psh_system* s);       /* nnz */
double psh_build_seconds(const psh_system* s);

/* ---- 3D (BASELINE.json configs 3 and 5; not in the reference, which is
 * 2D only: mesh.hpp:21). The 3D generalisation of the
 * reference's discretisation, documented in host/pstokes_host3d.cpp. ---- */
typedef struct psh_mesh3 psh_mesh3;
enum { PSH3_DATA_ZERO = 0, PSH3_DATA_RANDOM = 3, PSH3_DATA_MANUFACTURED = 4 };

const char* psh3_last_error(void);
/* Unit cube, n^3 hexahedra, interior vertices jittered by
 * frac*(1/n)*SplitMix64(seed).sym() (x, y, z; l outer, j, i inner); faces
 * numbered first-seen over the element loop (local faces x-, x+, y-, y+,
 * z-, z+); Neumann on z = 1 when neumann_top, Dirichlet elsewhere. */
int psh_mesh_unit_cube(int n, double frac, uint64_t seed, int neumann_top, psh_mesh3** out);
void psh_mesh3_destroy(psh_mesh3* m);
/* out[0..2] = vertices, elements, faces */
void psh_mesh3_counts(const psh_mesh3* m, int64_t* out);
/* 7 ints per face: 4 vertices (oriented out of left), left, right, tag */
void psh_mesh3_faces(const psh_mesh3* m, int32_t* faces);
/* 6 face ids per element (local order x-, x+, y-, y+, z-, z+) */
void psh_mesh3_element_faces(const psh_mesh3* m, int32_t* ef);
void psh_mesh3_vertices(const psh_mesh3* m, double* xyz);
/* HHO-hp vp-cond at face degree k: info[0..7] = n_local, n_elim, n_keep,
 * face_vel, face_press, face_block, faces per element (6), element velocity
 * modes per component. */
int psh3_hp_info(int k, int32_t* info);
int psh3_hp_elim(int k, int32_t* elim);         /* n_elim local ids (condense.hpp:44-55 order) */
int psh3_hp_keep_pos(int k, int32_t* pos);      /* n_keep x (local face, offset in face block) */
/* Local blocks of elements [e0, e1) (column-major n x n) and loads;
 * data: PSH3_DATA_*, seed for the random body force; eta <= 0: 3(k+1)^2. */
int psh3_local_blocks(const psh_mesh3* m, int k, int data, uint64_t seed, double eta, int e0,
                      int e1, int nthreads, double* mats, double* rhs);
/* Face-block pattern of the condensed operator (block row f: faces of the
 * elements holding f, ascending). Returns the block count; arrays nullable. */
/* Inputs of the device local-block producer (pscu_local_blocks3) for
 * elements [e0, e1): hex vertex ids (8 per element), element faces and
 * orientation signs (6 each), the face table {4 vertex ids, tag} of all
 * faces, the Gauss-Legendre rule (points, then weights) and, for data 3, the
 * per-element random modal coefficients (3 x dim P_k). Null outputs are
 * skipped. Returns the rule size (> 0) or minus the error code. */
int psh3_device_inputs(const psh_mesh3* m, int k, int data, uint64_t seed, int e0, int e1,
                       int32_t* hex, int32_t* ef, int32_t* es, int32_t* ftab, double* gl,
                       double* coef);
int64_t psh3_block_pattern(const psh_mesh3* m, int64_t* brow_ptr, int32_t* bcols);
/* ---- DG (BR2) in 3D: BASELINE.json config 4 (the reference's DG scheme,
 * assemble.hpp:177-346, with three velocity components; recipe in
 * host/pstokes_host3d.cpp). Element blocks [ux | uy | uz | p], ne = dim
 * P^k(3D) modes each; the operator's storage is the DG block storage of
 * pscu_dgb_create (10 ne^2 structural entries per element pair). ---- */
int psh3_dg_info(int k, int32_t* info);  /* info[0..1] = ne, 4 ne */
/* Block row e: e and its neighbours across interior faces, ascending.
 * Returns the block count; arrays nullable. */
int64_t psh3_dg_block_pattern(const psh_mesh3* m, int64_t* brow_ptr, int32_t* bcols);
/* Local terms for the oracle's reference-order scatter (small meshes):
 * volume blocks (nelem x (4ne)^2) and loads, face blocks over [left | right]
 * (nfaces x (8ne)^2, leading dimension 8ne) and face loads (nfaces x 8ne);
 * data: PSH3_DATA_*; eta <= 0: the BR2 default 7. Outputs nullable. */
int psh3_dg_local(const psh_mesh3* m, int k, int data, uint64_t seed, double eta, int nthreads,
                  double* vol, double* vrhs, double* fmat, double* frhs);
/* Block rows [e0, e1) of the assembled operator in DG block storage
 * (blocks brow_ptr[e0] .. brow_ptr[e1]-1) and their loads, summed in the
 * reference's scatter order (volume, then faces by id). */
int psh3_dg_rows(const psh_mesh3* m, int k, int data, uint64_t seed, double eta, int e0, int e1,
                 const int64_t* brow_ptr, const int32_t* bcols, int nthreads, double* vals,
                 double* rhs);
/* ||u_h - u||, ||p_h - p|| of a DG solution against the data-4 field. */
int psh3_dg_l2_errors(const psh_mesh3* m, int k, const double* x, double* out);
/* Face L2 projections of the manufactured solution (n_faces x 4 nf). */
int psh3_face_projection(const psh_mesh3* m, int k, double* out);
/* nelem volumes, then nelem closure norms |sum_F int_F n dA|. */
int psh3_geometry(const psh_mesh3* m, double* out);

#ifdef __cplusplus
}
#endif

#endif
