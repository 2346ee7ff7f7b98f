// Internal declarations of the B200 solver library (not installed).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "pstokes_cuda.h"

namespace pscu {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PSCU_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      throw ::pscu::Error(PSCU_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_));    \
  } while (0)

#define PSCU_LAUNCHED(ctx)                                                                  \
  do {                                                                                      \
    (ctx)->launches++;                                                                      \
    cudaError_t e_ = cudaGetLastError();                                                    \
    if (e_ != cudaSuccess)                                                                  \
      throw ::pscu::Error(PSCU_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

// Bit-exact arithmetic helpers: one IEEE-rounded operation each, never fused.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) {
      cudaError_t e = cudaMalloc(&p, sizeof(T) * count);
      if (e != cudaSuccess)
        throw Error(PSCU_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    if (count > n) alloc(count);
    if (count) PSCU_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
};

/// Fixed-shape reproducible dot product (include/eigen_subset/Eigen/Dense,
/// internal::repro_lanes / repro_dot_fn): T strided partials, adjacent-pair
/// binary tree.
inline int64_t repro_lanes(int64_t n) {
  int64_t want = (n + 15) / 16, t = 1;
  while (t < want && t < (int64_t(1) << 18)) t <<= 1;
  return t;
}

struct Context;

/// Velocity components of a layout (dof_layout.hpp:68-69 has 2; dim 3 adds z).
inline int ncomp(const pscu_layout& l) { return l.dim == 3 ? 3 : 2; }

/// Device CSR (csr.hpp:19-24) plus a host copy of the pattern for schedule
/// construction.
struct Csr {
  int64_t n = 0, nnz = 0;
  DevBuf<int64_t> row_ptr;
  DevBuf<int32_t> cols;
  DevBuf<double> vals;
  std::vector<int64_t> h_row_ptr;
  std::vector<int32_t> h_cols;
  // Dense-block storage (bsr.cu) of operators whose structural pattern is
  // made of dense bs x bs face blocks (3D HHO-hp vp-cond): bs > 0 means
  // row_ptr / cols are unused and vals holds nblk blocks, column-major per
  // block, in block-row order with block columns ascending (the CSR order of
  // csr.hpp:30-44 is block column, then column within the block). n = nb bs,
  // nnz = nblk bs^2 structural entries.
  int bs = 0;
  int64_t nb = 0, nblk = 0;
  // sharded operators (zslab.py): block columns may exceed the block rows
  // (ghost faces of the neighbour slabs); the diagonal block of block row b
  // is block column b + diag_off
  int64_t ncb = 0, diag_off = 0;
  // DG block storage (dgb.cu): dgm > 0 modes per component, bs = 4 dgm,
  // every block holds its 10 dgm^2 structural entries as panels (velocity
  // component c: dgm x 2dgm [u_c | p] columns; pressure: dgm x 4dgm), nnz =
  // nblk 10 dgm^2
  int dgm = 0;
  DevBuf<int64_t> brow_ptr;
  DevBuf<int32_t> bcols, brow_of;  // block columns, block row of every block
  std::vector<int64_t> h_brow_ptr;
  std::vector<int32_t> h_bcols;
};

/// Level-walking sweep plan (walk.cu).
struct WalkSeg {
  bool wide;   // task-parallel launch of one chunk, else one walker cluster
  int s0, s1;  // chunk range
  bool warp = false;  // wide: one warp per task (long tasks), else one thread
  int tasks = 0;      // wide: tasks of the chunk
};

struct WalkPlan {
  bool fwd = true;
  int C = 1;     // CTAs of the walker cluster (one chunk each per sub-level)
  bool flow = false;  // single-CTA dataflow walker
  int S = 0;          // push walker: replicated ring slots per owner
  bool levels = false;  // every task level is a task-parallel launch (no walker)
  int nsub = 0;  // chunks
  int64_t npos = 0;
  std::vector<WalkSeg> segments;
  DevBuf<int32_t> sl_k, sl_nr, sl_hdr, tt, tq, rows, off, dp, opos, src, far, sfar;
  DevBuf<int64_t> sl_q, sl_f, sl_s, dfrom;
  DevBuf<int32_t> from;  // factor position of every packed entry (-1: padding)
  DevBuf<double> val, dv;
  DevBuf<int4> meta;               // per position {length / offset, row, backward position, 0}
  mutable DevBuf<double> sfv;      // per-apply values of the static out-of-ring sources
  std::vector<int64_t> h_sl_s;     // static list start per chunk (host copy)
  mutable DevBuf<double> scratch;  // per-apply right-hand sides in position order
  // level-launch plans: both sweeps captured once as a CUDA graph working on
  // fixed buffers (ybuf); the apply copies the result out
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    long long kernels = 0;
    ~Graph() {
      if (exec) cudaGraphExecDestroy(exec);
    }
  };
  mutable std::shared_ptr<Graph> graph;
  mutable DevBuf<double> ybuf;
  mutable DevBuf<unsigned long long> barrier;  // persistent task-level kernel
  int persist_grid = 0;                        // its grid (0: per-level launches)
  int flow_grid = 0;                           // dataflow sweep grid (0: off)
  int flow_small = 0;                          // ... with the small-task (1) / mid-task (2) kernel
  int64_t ny = 0;                              // rows of the sweep (sentinel fill)
};

struct Ilu {
  const Csr* a = nullptr;
  DevBuf<double> lu;
  DevBuf<int64_t> diag;
  std::vector<int64_t> h_diag;   // diagonal positions (host, for the sweep plans)
  WalkPlan wfwd, wbwd;           // level walkers (application)
  std::vector<int32_t> flev_ptr; // forward DAG levels (factorisation launches)
  DevBuf<int32_t> flev_rows;
};

/// Live per-kernel-class timing with CUDA events on the launching stream.
enum ProfClass { PROF_ILU = 0, PROF_SPMV = 1, PROF_MGS = 2, PROF_OTHER = 3, PROF_BJ = 4, PROF_NCLASS = 5 };

struct ProfRec {
  int cls;
  cudaEvent_t e0, e1;
  double bytes;
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  long long launches = 0;
  bool profiling = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t t_start = nullptr, t_stop = nullptr;
  cudaEvent_t next_event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      PSCU_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
  /// Brackets one launch (or a tight group) of a profiled class.
  struct Scope {
    Context* c;
    int cls;
    double bytes;
    cudaEvent_t e0 = nullptr;
    Scope(Context* cc, int k, double b) : c(cc), cls(k), bytes(b) {
      if (c->profiling) {
        e0 = c->next_event();
        cudaEventRecord(e0, c->stream);
      }
    }
    ~Scope() {
      if (c->profiling) {
        cudaEvent_t e1 = c->next_event();
        cudaEventRecord(e1, c->stream);
        c->prof.push_back({cls, e0, e1, bytes});
      }
    }
  };
  // reduction scratch
  DevBuf<double> red_partials;     // per-block results
  DevBuf<unsigned int> red_counter; // last-block counter
  DevBuf<double> scal;             // device scalars (Hessenberg column etc.)
  double* h_pinned = nullptr;      // pinned host mirror of scal
  DevBuf<int> err_flag;
  DevBuf<double> l3_scratch;        // device local-block producer work arrays
  DevBuf<unsigned long long> slot_tag;  // tagged reduction slots (arnoldi_step_kernel)
  unsigned long long pass_tag = 0;      // monotonic pass id across launches
  size_t scal_cap = 0;
  ~Context();
};

// spmv.cu
void spmv(Context& c, const Csr& a, const double* x, double* y);
/// r_c[i] = (d - A w)[map[i]] for i < nc (fused residual + restriction).
void residual_restrict(Context& c, const Csr& a, const double* d, const double* w,
                       const int64_t* map, int64_t nc, double* rc);
void upload_csr(Context& c, Csr& m, int64_t n, const int64_t* rp, const int32_t* cols,
                const double* vals, int mem);

// bsr.cu
void upload_bsr(Context& c, Csr& m, int64_t nb, int bs, const int64_t* brow_ptr,
                const int32_t* bcols, const double* vals, int mem, int64_t ncb = -1,
                int64_t diag_off = 0);
/// Zero-valued block matrix over a block pattern (host arrays).
void alloc_bsr(Context& c, Csr& m, int64_t nb, int bs, const int64_t* brow_ptr,
               const int32_t* bcols, int64_t ncb = -1, int64_t diag_off = 0);
/// The same operator in CSR storage (pattern on the host too: ILU plans).
void bsr_to_csr(Context& c, const Csr& b, Csr& out);
/// inherit_matrix (plevels.hpp:93-113) between face-block operators: every
/// block keeps its position, its entries are the in-block map's rows/cols.
void inherit_bsr(Context& c, const Csr& fine, const std::vector<int32_t>& in_block, Csr& out);
void spmv_bsr(Context& c, const Csr& a, const double* x, double* y);
void residual_restrict_bsr(Context& c, const Csr& a, const double* d, const double* w,
                           const int64_t* map, int64_t nc, double* rc);

void bsr_set_pattern(Context& c, Csr& m, int64_t nb, int bs, const int64_t* brow_ptr,
                     const int32_t* bcols, int64_t ncb, int64_t diag_off);

// dgb.cu — DG block storage (3D DG, BASELINE.json config 4)
void upload_dgb(Context& c, Csr& m, int64_t nb, int nm, const int64_t* brow_ptr,
                const int32_t* bcols, const double* vals, int mem);
void spmv_dgb(Context& c, const Csr& a, const double* x, double* y);
/// rc = restriction of (d - A w) to the leading nc/(4 nb) modes per component
void residual_restrict_dgb(Context& c, const Csr& a, const double* d, const double* w,
                           int64_t nc, double* rc);
void inherit_dgb(Context& c, const Csr& fine, int nmc, Csr& out);
void dgb_to_csr(Context& c, const Csr& b, Csr& out);

// sptrsv.cu
void ilu0_factor(Context& c, Ilu& ilu);
/// ilu0_factor in two parts: pattern checks + factorisation launches, then
/// (after the sweep plans are uploaded) the pivot check and value packing.
void ilu0_factor_start(Context& c, Ilu& ilu);
void ilu0_factor_finish(Context& c, Ilu& ilu);
void ilu0_apply(Context& c, const Ilu& ilu, const double* x, double* y);

// krylov.cu
double dot(Context& c, const double* x, const double* y, int64_t n);
void copy(Context& c, double* dst, const double* src, int64_t n);
void zero(Context& c, double* dst, int64_t n);

} // namespace pscu
