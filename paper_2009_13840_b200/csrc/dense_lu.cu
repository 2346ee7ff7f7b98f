// Dense LU with partial pivoting for small coarsest levels (coarse = "lu").
// The reference factors its coarsest operator with a sparse left-looking LU
// (sparse_lu.hpp:111-276) on the host; here the coarsest level (n up to a few
// thousand at the BASELINE.json 2D configs) is factored densely on the GPU.
// Row pivoting picks the first maximal |a_ik| like the Eigen subset.
#include "internal.cuh"
#include "solver.cuh"

namespace pscu {

namespace {

__global__ void scatter_dense(int64_t n, const int64_t* __restrict__ rp,
                              const int32_t* __restrict__ cols, const double* __restrict__ vals,
                              double* __restrict__ a) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) a[i + int64_t(cols[p]) * n] = vals[p];
}

/// Step k: pivot search (first max), row swap, column scaling. One CTA.
__global__ void pivot_step(int64_t n, int64_t k, double* a, int32_t* perm) {
  __shared__ double best[1024];
  __shared__ int64_t bidx[1024];
  double bv = -1.0;
  int64_t bi = n;
  for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(a[i + k * n]);
    if (v > bv) {
      bv = v;
      bi = i;
    }
  }
  best[threadIdx.x] = bv;
  bidx[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = best[threadIdx.x + s];
      const int64_t oi = bidx[threadIdx.x + s];
      if (o > best[threadIdx.x] || (o == best[threadIdx.x] && oi < bidx[threadIdx.x])) {
        best[threadIdx.x] = o;
        bidx[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const int64_t p = bidx[0];
  if (p != k && p < n) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const double t = a[k + j * n];
      a[k + j * n] = a[p + j * n];
      a[p + j * n] = t;
    }
    if (threadIdx.x == 0) {
      const int32_t t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
  }
  __syncthreads();
  const double piv = a[k + k * n];
  if (piv != 0.0)
    for (int64_t i = k + 1 + threadIdx.x; i < n; i += blockDim.x)
      a[i + k * n] = __ddiv_rn(a[i + k * n], piv);
}

__global__ void update_step(int64_t n, int64_t k, double* a) {
  const int64_t m = n - k - 1;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < m * m;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = k + 1 + t % m, j = k + 1 + t / m;
    const double ukj = a[k + j * n];
    if (ukj != 0.0) a[i + j * n] = dsub(a[i + j * n], dmul(a[i + k * n], ukj));
  }
}

/// x = U^-1 L^-1 P b, column-oriented sweeps in one CTA.
__global__ void lu_solve(int64_t n, const double* __restrict__ a, const int32_t* __restrict__ perm,
                         const double* __restrict__ b, double* __restrict__ x) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = b[perm[i]];
  __syncthreads();
  for (int64_t j = 0; j < n; ++j) {
    const double xj = x[j];
    for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
      x[i] = dsub(x[i], dmul(a[i + j * n], xj));
    __syncthreads();
  }
  for (int64_t j = n - 1; j >= 0; --j) {
    if (threadIdx.x == 0) x[j] = __ddiv_rn(x[j], a[j + j * n]);
    __syncthreads();
    const double xj = x[j];
    for (int64_t i = threadIdx.x; i < j; i += blockDim.x) x[i] = dsub(x[i], dmul(a[i + j * n], xj));
    __syncthreads();
  }
}

} // namespace

void DenseLu::factor(Context& c, const Csr& a) {
  n = a.n;
  if (n > 16384) throw Error(PSCU_EINVAL, "coarse lu: coarsest level too large for the dense LU "
                                          "(use the ILU-GMRES coarse solver)");
  lu.alloc(size_t(n) * size_t(n));
  PSCU_CUDA(cudaMemsetAsync(lu.p, 0, sizeof(double) * n * n, c.stream));
  std::vector<int32_t> p(n);
  for (int64_t i = 0; i < n; ++i) p[i] = int32_t(i);
  perm.upload(p, c.stream);
  tmp.alloc(n);
  scatter_dense<<<unsigned((n + 255) / 256), 256, 0, c.stream>>>(n, a.row_ptr.p, a.cols.p,
                                                                  a.vals.p, lu.p);
  PSCU_LAUNCHED(&c);
  for (int64_t k = 0; k < n; ++k) {
    pivot_step<<<1, 1024, 0, c.stream>>>(n, k, lu.p, perm.p);
    PSCU_LAUNCHED(&c);
    const int64_t m = n - k - 1;
    if (m > 0) {
      const int64_t g = (m * m + 255) / 256;
      update_step<<<unsigned(g < 4096 ? g : 4096), 256, 0, c.stream>>>(n, k, lu.p);
      PSCU_LAUNCHED(&c);
    }
  }
  // singularity check: zero pivot on the diagonal
  std::vector<double> d(n);
  PSCU_CUDA(cudaMemcpy2DAsync(d.data(), sizeof(double), lu.p, sizeof(double) * (n + 1),
                              sizeof(double), n, cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  for (int64_t i = 0; i < n; ++i)
    if (d[i] == 0.0)
      throw Error(PSCU_ESINGULAR, "sparse_lu: structurally or numerically singular at column " +
                                      std::to_string(i));
}

void DenseLu::solve(Context& c, const double* b, double* x) {
  lu_solve<<<1, 1024, 0, c.stream>>>(n, lu.p, perm.p, b, x);
  PSCU_LAUNCHED(&c);
}

} // namespace pscu
