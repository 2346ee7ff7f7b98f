// Sparse matrix-vector products with the reference's per-row summation order
// (CsrMatrix::multiply, csr.hpp:68-74: y_i = sum_p vals[p]*x[cols[p]], p
// ascending, starting from 0.0, every product rounded, no FMA).
//
// spmv_staged: one CTA owns ROWS consecutive rows, so their nonzeros form
// one contiguous range. The CTA streams that range through shared memory in
// coalesced 128-bit-friendly passes (vals, cols, x gather -> rounded product)
// and then every thread folds its own row sequentially out of shared memory.
// HBM traffic is the structural 12 B/nnz + 16 B/row; the x gather is served
// by L2 (the vectors are far smaller than the 126 MB L2).
#include "internal.cuh"

namespace pscu {

namespace {

constexpr int kRows = 128;    // rows per CTA
constexpr int kChunk = 2048;  // staged products per pass (16 KB)

__global__ void __launch_bounds__(kRows) spmv_staged(int64_t n, const int64_t* __restrict__ rp,
                                                      const int32_t* __restrict__ cols,
                                                      const double* __restrict__ vals,
                                                      const double* __restrict__ x,
                                                      double* __restrict__ y) {
  __shared__ double prod[kChunk];
  const int64_t r0 = int64_t(blockIdx.x) * kRows;
  if (r0 >= n) return;
  const int64_t r1 = min(n, r0 + kRows);
  const int64_t p0 = rp[r0], p1 = rp[r1];
  const int64_t row = r0 + threadIdx.x;
  int64_t rs = 0, re = 0;
  if (row < r1) {
    rs = rp[row];
    re = rp[row + 1];
  }
  double s = 0.0;
  for (int64_t c0 = p0; c0 < p1; c0 += kChunk) {
    const int64_t c1 = min(p1, c0 + kChunk);
    for (int64_t p = c0 + threadIdx.x; p < c1; p += kRows)
      prod[p - c0] = dmul(__ldg(vals + p), __ldg(x + __ldg(cols + p)));
    __syncthreads();
    const int64_t a = max(rs, c0), b = min(re, c1);
    for (int64_t p = a; p < b; ++p) s = dadd(s, prod[p - c0]);
    __syncthreads();
  }
  if (row < r1) y[row] = s;
}

/// Warp per selected row: rc[i] = d[r] - (A w)[r], r = map[i]. Lanes form
/// the rounded products, lane 0 folds them in column order.
__global__ void residual_restrict_warp(int64_t nc, const int64_t* __restrict__ map,
                                       const int64_t* __restrict__ rp,
                                       const int32_t* __restrict__ cols,
                                       const double* __restrict__ vals,
                                       const double* __restrict__ d,
                                       const double* __restrict__ w, double* __restrict__ rc) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nc) return;
  const int64_t r = map[warp];
  const int64_t s0 = rp[r], s1 = rp[r + 1];
  double s = 0.0;
  for (int64_t base = s0; base < s1; base += 32) {
    const int64_t p = base + lane;
    double t = 0.0;
    if (p < s1) t = dmul(__ldg(vals + p), __ldg(w + __ldg(cols + p)));
    const int cnt = int(s1 - base < 32 ? s1 - base : 32);
    for (int j = 0; j < cnt; ++j) {
      const double tj = __shfl_sync(0xffffffffu, t, j);
      s = dadd(s, tj);
    }
  }
  if (lane == 0) rc[warp] = dsub(d[r], s);
}

} // namespace

void spmv(Context& c, const Csr& a, const double* x, double* y) {
  if (a.bs) return spmv_bsr(c, a, x, y);
  if (a.n == 0) return;
  const unsigned grid = unsigned((a.n + kRows - 1) / kRows);
  Context::Scope prof(&c, PROF_SPMV, 8.0 * double(a.nnz) + 16.0 * double(a.n));
  spmv_staged<<<grid, kRows, 0, c.stream>>>(a.n, a.row_ptr.p, a.cols.p, a.vals.p, x, y);
  PSCU_LAUNCHED(&c);
}

void residual_restrict(Context& c, const Csr& a, const double* d, const double* w,
                       const int64_t* map, int64_t nc, double* rc) {
  if (a.bs) return residual_restrict_bsr(c, a, d, w, map, nc, rc);
  if (nc == 0) return;
  const int threads = 256;
  const unsigned grid = unsigned((nc * 32 + threads - 1) / threads);
  residual_restrict_warp<<<grid, threads, 0, c.stream>>>(nc, map, a.row_ptr.p, a.cols.p,
                                                         a.vals.p, d, w, rc);
  PSCU_LAUNCHED(&c);
}

void upload_csr(Context& c, Csr& m, int64_t n, const int64_t* rp, const int32_t* cols,
                const double* vals, int mem) {
  m.n = n;
  if (mem == PSCU_HOST) {
    m.h_row_ptr.assign(rp, rp + n + 1);
    m.nnz = m.h_row_ptr[n];
    m.h_cols.assign(cols, cols + m.nnz);
  } else {
    m.h_row_ptr.resize(n + 1);
    PSCU_CUDA(cudaMemcpy(m.h_row_ptr.data(), rp, sizeof(int64_t) * (n + 1),
                         cudaMemcpyDeviceToHost));
    m.nnz = m.h_row_ptr[n];
    m.h_cols.resize(m.nnz);
    PSCU_CUDA(cudaMemcpy(m.h_cols.data(), cols, sizeof(int32_t) * m.nnz, cudaMemcpyDeviceToHost));
  }
  m.row_ptr.alloc(n + 1);
  m.cols.alloc(m.nnz);
  m.vals.alloc(m.nnz);
  const cudaMemcpyKind k = mem == PSCU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  PSCU_CUDA(cudaMemcpyAsync(m.row_ptr.p, rp, sizeof(int64_t) * (n + 1), k, c.stream));
  if (m.nnz) {
    PSCU_CUDA(cudaMemcpyAsync(m.cols.p, cols, sizeof(int32_t) * m.nnz, k, c.stream));
    PSCU_CUDA(cudaMemcpyAsync(m.vals.p, vals, sizeof(double) * m.nnz, k, c.stream));
  }
}

} // namespace pscu
