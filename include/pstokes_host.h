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

/* Local blocks + layout + pattern (assemble_hho front end). scheme 0 hho-dp,
 * 1 hho-hp; strategy 0 uncond, 1 v-cond, 2 vp-cond; eta <= 0 selects the
 * default 3(k+1)^2 (hho_local.hpp:19). nthreads <= 0: all cores. */
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

#ifdef __cplusplus
}
#endif

#endif
