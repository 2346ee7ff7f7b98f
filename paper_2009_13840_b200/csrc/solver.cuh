// Internal solver objects (GMRES workspaces, hierarchy levels).
#pragma once

#include <memory>
#include <vector>

#include "internal.cuh"

namespace pscu {

/// Operator on device vectors (the ApplyFn plug point, gmres.hpp:17).
struct Op {
  virtual ~Op() = default;
  virtual int64_t size() const = 0;
  virtual void apply(Context& c, const double* x, double* y) = 0;
  /// false when an apply has effects beyond y (counters): such operators
  /// are never applied speculatively
  virtual bool pure() const { return true; }
};

struct KrylovResultDev {
  int iterations = 0;
  double rel_residual = 0.0;
  bool converged = false;
};

/// Scalar state of detail::ArnoldiWorkspace (gmres.hpp:38-92), on the host.
struct HostArnoldi {
  int m = 0;
  std::vector<double> h, g, cs, sn;
  double last_subdiag = 0.0;
  double& H(int i, int j) { return h[size_t(i) + size_t(j) * size_t(m + 1)]; }
  double H(int i, int j) const { return h[size_t(i) + size_t(j) * size_t(m + 1)]; }
  void init(int m, double beta);
  double step(int j, const double* col);
  void solve_y(int mm, std::vector<double>& y) const;
};

/// Device Krylov workspace: basis V ((m+1) x n), Z (m x n) when the
/// preconditioned vectors must be kept, and scratch vectors.
struct KrylovWs {
  int64_t n = -1;
  int m = -1;
  bool store_z = false;
  DevBuf<double> V, Z, w, r0, tmp, prhs, xs, hcol, ydev;
  std::vector<double> hcol_host;
  // pinned, double-buffered Hessenberg columns of the look-ahead Arnoldi loop
  double* hpin = nullptr;
  int hpin_m = -1;
  cudaEvent_t hev[2] = {nullptr, nullptr};
  void ensure(int64_t n, int m, bool store_z);
  KrylovWs() = default;
  KrylovWs(const KrylovWs&) = delete;
  KrylovWs& operator=(const KrylovWs&) = delete;
  ~KrylovWs();
};

KrylovResultDev gmres_dev(Context& c, Op& op, Op* pc, const double* rhs, const double* x0,
                          int max_it, double rtol, bool left, double* x, KrylovWs& ws,
                          const double* prhs_cached);
KrylovResultDev fgmres_dev(Context& c, Op& op, Op& pc, const double* rhs, int max_it, double rtol,
                           int restart, double* x, KrylovWs& ws, std::vector<double>* hist);

/// Dense LU with partial pivoting on the device, for small coarsest levels
/// (the reference's coarse LU, sparse_lu.hpp, solves the same system; the
/// result matches it to rounding, not bitwise).
struct DenseLu {
  int64_t n = 0;
  DevBuf<double> lu;
  DevBuf<int32_t> perm;
  DevBuf<double> tmp;
  void factor(Context& c, const Csr& a);
  void solve(Context& c, const double* b, double* x);
};

/// Block-Jacobi over the layout's entity blocks (bjacobi.cu).
struct BlockJacobi {
  pscu_layout layout{};
  int fb = 0, eb = 0;
  int64_t eoff = 0, n = 0;
  DevBuf<double> inv;  // face blocks then element blocks, column-major per block
};
void bj_factor(Context& c, const Csr& a, const pscu_layout& l, BlockJacobi& bj);
void bj_apply(Context& c, const BlockJacobi& bj, const double* x, double* y);

struct Level {
  int k = 0;
  pscu_layout layout{};
  const Csr* a = nullptr;  // level 0 borrows the fine matrix
  Csr own;
  // operator applications (SpMV, residual) use the block storage when the
  // level also holds a CSR copy for ILU(0) / dense LU: fewer bytes, same sums
  const Csr* op = nullptr;
  Csr own_bsr;
  Ilu ilu;
  BlockJacobi bj;
  bool use_bj = false;  // smoother preconditioner: block-Jacobi instead of ILU(0)
  DenseLu dense_lu;
  DevBuf<int64_t> down_map;  // coarse (l+1) -> this level
  DevBuf<int32_t> f2c;       // this level -> coarse index or -1
  int64_t nc = 0;
  DevBuf<double> w, dc, cc;
  KrylovWs ws;
};

struct Hierarchy {
  pscu_level_cfg cfg{};
  std::vector<std::unique_ptr<Level>> levels;
  long long coarse_its = 0;
  ~Hierarchy();
  void build(Context& c, const Csr* fine, const pscu_layout& lf, const int* degrees, int nlev,
             const pscu_level_cfg& cfg);
  void vcycle(Context& c, int l, const double* d, double* out);
  void coarse_solve(Context& c, const double* d, double* out);
  int64_t P_nc(int l) const;
};

int64_t layout_dim(const pscu_layout& l);
void make_layout(int scheme, int strategy, int k, int n_faces, int n_elements, pscu_layout& l);
void make_layout3(int scheme, int strategy, int k, int n_faces, int n_elements, pscu_layout& l);
/// The layout of lf's scheme at degree k (2D or 3D).
void layout_at(const pscu_layout& lf, int k, pscu_layout& out);
void coarse_to_fine(const pscu_layout& f, const pscu_layout& c, int64_t* map);
void inherit(Context& c, const Csr& fine, const std::vector<int64_t>& c2f, Csr& out);

} // namespace pscu
