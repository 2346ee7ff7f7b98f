// Batched static condensation (condense_element, condense.hpp:57-97) and
// recovery (ElementCondensation::recover, condense.hpp:28-38).
//
// One CTA per element keeps the whole local block in shared memory and
// performs the partial-pivot LU of A_ee, the solves for [A_ek | b_e], and
// the Schur update S = A_kk - A_ke X, with every matrix entry receiving its
// updates in the same order as the host LU/GEMM of include/eigen_subset
// (k ascending, one rounded operation each), so results are bit-identical to
// the reference built against that header.
#include "internal.cuh"

namespace pscu {

namespace {

constexpr int kCondThreads = 256;

__global__ void __launch_bounds__(kCondThreads)
    condense_kernel(int nelem, int n, const double* __restrict__ mats,
                    const double* __restrict__ rhs, int ne, const int* __restrict__ elim,
                    const int* __restrict__ keep, double* __restrict__ schur,
                    double* __restrict__ rrhs, double* __restrict__ coupling,
                    double* __restrict__ erhs, int* bad) {
  extern __shared__ double sm[];
  const int nk = n - ne;
  double* A = sm;                       // n x n local matrix (+ rhs column)
  double* LU = A + size_t(n) * (n + 1); // ne x ne
  double* X = LU + size_t(ne) * ne;     // ne x (nk+1)
  __shared__ int perm[256];
  __shared__ int piv_row;
  __shared__ int singular;
  for (int e = blockIdx.x; e < nelem; e += gridDim.x) {
    const double* M = mats + size_t(e) * n * n;
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) A[t] = M[t];
    for (int t = threadIdx.x; t < n; t += blockDim.x) A[size_t(n) * n + t] = rhs[size_t(e) * n + t];
    if (threadIdx.x == 0) singular = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < ne * ne; t += blockDim.x) {
      const int i = t % ne, j = t / ne;
      LU[t] = A[elim[i] + size_t(elim[j]) * n];
    }
    for (int t = threadIdx.x; t < ne; t += blockDim.x) perm[t] = t;
    __syncthreads();
    // partial-pivot LU (Eigen subset PartialPivLU::compute)
    for (int k = 0; k < ne; ++k) {
      if (threadIdx.x == 0) {
        int p = k;
        double pmax = fabs(LU[k + k * ne]);
        for (int i = k + 1; i < ne; ++i)
          if (fabs(LU[i + k * ne]) > pmax) {
            pmax = fabs(LU[i + k * ne]);
            p = i;
          }
        piv_row = p;
        if (p != k) {
          const int t = perm[k];
          perm[k] = perm[p];
          perm[p] = t;
        }
      }
      __syncthreads();
      const int p = piv_row;
      if (p != k)
        for (int j = threadIdx.x; j < ne; j += blockDim.x) {
          const double t = LU[k + j * ne];
          LU[k + j * ne] = LU[p + j * ne];
          LU[p + j * ne] = t;
        }
      __syncthreads();
      const double piv = LU[k + k * ne];
      if (piv != 0.0) {
        for (int i = k + 1 + threadIdx.x; i < ne; i += blockDim.x)
          LU[i + k * ne] = __ddiv_rn(LU[i + k * ne], piv);
        __syncthreads();
        const int m = ne - k - 1;
        for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
          const int i = k + 1 + t % m, j = k + 1 + t / m;
          const double ukj = LU[k + j * ne];
          if (ukj != 0.0) LU[i + j * ne] = dsub(LU[i + j * ne], dmul(LU[i + k * ne], ukj));
        }
      }
      __syncthreads();
    }
    // solves: one thread per right-hand side column of [A_ek | b_e]
    for (int col = threadIdx.x; col <= nk; col += blockDim.x) {
      double* x = X + size_t(col) * ne;
      const int src = col < nk ? keep[col] : n;
      for (int i = 0; i < ne; ++i) x[i] = A[elim[perm[i]] + size_t(src) * n];
      for (int i = 0; i < ne; ++i) {
        double s = x[i];
        for (int j = 0; j < i; ++j) s = dsub(s, dmul(LU[i + j * ne], x[j]));
        x[i] = s;
      }
      for (int i = ne - 1; i >= 0; --i) {
        double s = x[i];
        for (int j = i + 1; j < ne; ++j) s = dsub(s, dmul(LU[i + j * ne], x[j]));
        x[i] = __ddiv_rn(s, LU[i + i * ne]);
      }
    }
    // rcond guard: ||A_ee||_1 ||A_ee^-1||_1 with the exact inverse (nothing
    // eliminated: the Schur complement is the block itself, condense.hpp:70-74)
    if (threadIdx.x == 0 && ne > 0) {
      for (int i = 0; i < ne; ++i)
        if (LU[i + i * ne] == 0.0) singular = 1;
    }
    __syncthreads();
    if (!singular && ne > 0) {
      __shared__ double colnorm[256];
      __shared__ double anorm_s;
      if (threadIdx.x == 0) {
        double an = 0.0;
        for (int j = 0; j < ne; ++j) {
          double s = 0.0;
          for (int i = 0; i < ne; ++i) s += fabs(A[elim[i] + size_t(elim[j]) * n]);
          an = fmax(an, s);
        }
        anorm_s = an;
      }
      for (int cidx = threadIdx.x; cidx < ne; cidx += blockDim.x) {
        double xcol[64];
        double s = 0.0;
        if (ne <= 64) {
          for (int i = 0; i < ne; ++i) xcol[i] = perm[i] == cidx ? 1.0 : 0.0;
          for (int i = 0; i < ne; ++i) {
            double t = xcol[i];
            for (int j = 0; j < i; ++j) t = t - LU[i + j * ne] * xcol[j];
            xcol[i] = t;
          }
          for (int i = ne - 1; i >= 0; --i) {
            double t = xcol[i];
            for (int j = i + 1; j < ne; ++j) t = t - LU[i + j * ne] * xcol[j];
            xcol[i] = t / LU[i + i * ne];
          }
          for (int i = 0; i < ne; ++i) s += fabs(xcol[i]);
        }
        colnorm[cidx] = s;
      }
      __syncthreads();
      if (threadIdx.x == 0 && ne <= 64) {
        double inorm = 0.0;
        for (int j = 0; j < ne; ++j) inorm = fmax(inorm, colnorm[j]);
        const double an = anorm_s;
        const double rc = (an > 0.0 && inorm > 0.0 && isfinite(inorm)) ? (1.0 / an) / inorm : 0.0;
        if (rc < 1e-14) singular = 1;
      }
      __syncthreads();
    }
    if (singular && threadIdx.x == 0) atomicMin(bad, e);
    // Schur complement and reduced rhs (GEMM, k ascending from 0)
    for (int t = threadIdx.x; t < nk * (nk + 1); t += blockDim.x) {
      const int i = t % nk, j = t / nk;
      const int src = j < nk ? keep[j] : n;
      double s = 0.0;
      for (int k = 0; k < ne; ++k)
        s = dadd(s, dmul(A[keep[i] + size_t(elim[k]) * n], X[k + size_t(j) * ne]));
      const double v = dsub(A[keep[i] + size_t(src) * n], s);
      if (j < nk) {
        if (schur) schur[size_t(e) * nk * nk + i + size_t(j) * nk] = v;
      } else if (rrhs) {
        rrhs[size_t(e) * nk + i] = v;
      }
    }
    if (coupling)
      for (int t = threadIdx.x; t < ne * nk; t += blockDim.x)
        coupling[size_t(e) * ne * nk + t] = X[t];
    if (erhs)
      for (int t = threadIdx.x; t < ne; t += blockDim.x)
        erhs[size_t(e) * ne + t] = X[size_t(nk) * ne + t];
    __syncthreads();
  }
}

/// locals[e][keep[i]] = x[kept[e][i]]; locals[e][elim[i]] = erhs - C x_k
/// (condense.hpp:28-38: xe = elim_rhs - elim_coupling * kept_values).
__global__ void recover_kernel(int nelem, int n, int ne, const int* __restrict__ elim,
                               const int* __restrict__ keep, const int64_t* __restrict__ kept,
                               const double* __restrict__ coupling,
                               const double* __restrict__ erhs, const double* __restrict__ x,
                               double* __restrict__ locals) {
  const int nk = n - ne;
  for (int e = blockIdx.x; e < nelem; e += gridDim.x) {
    const int64_t* kg = kept + size_t(e) * nk;
    double* out = locals + size_t(e) * n;
    for (int i = threadIdx.x; i < nk; i += blockDim.x) out[keep[i]] = x[kg[i]];
    for (int i = threadIdx.x; i < ne; i += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < nk; ++j)
        s = dadd(s, dmul(coupling[size_t(e) * ne * nk + i + size_t(j) * ne], x[kg[j]]));
      out[elim[i]] = dsub(erhs[size_t(e) * ne + i], s);
    }
  }
}

struct KindInfo {
  int64_t face_rows;
  int fb, eb, face_vel, elem_vel, strategy;
  __device__ int kind(int64_t g) const {  // assemble.hpp:25-39
    int within, nv;
    if (g < face_rows) {
      within = int(g % fb);
      nv = face_vel;
    } else {
      within = int((g - face_rows) % eb);
      nv = elem_vel;
    }
    return within < nv ? 0 : (within < 2 * nv ? 1 : 2);
  }
  __device__ bool coupled(int ka, int kb) const {  // assemble.hpp:41-46
    const bool av = ka != 2, bv = kb != 2;
    if (av && bv && ka != kb) return strategy == 2;
    if (!av && !bv) return strategy != 0;
    return true;
  }
};

/// Value pass of assemble_hho (assemble.hpp:164-169): every retained pair of
/// every element adds its Schur entry into the CSR slot found by binary
/// search in the (sorted) row. An entry receives at most two contributions
/// (two distinct faces share at most one element, a face at most two), and a
/// two-term sum from 0.0 is order-independent, so the atomics reproduce the
/// reference's element-order scatter bit for bit.
__global__ void assemble_kernel(int nelem, int nk, const int64_t* __restrict__ kept,
                                const double* __restrict__ schur,
                                const double* __restrict__ rrhs, KindInfo ki,
                                const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                double* vals, double* rhs, int* bad) {
  const int64_t per = int64_t(nk) * nk;
  const int64_t total = int64_t(nelem) * per;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int e = int(t / per);
    const int r = int(t % per);
    const int i = r % nk, j = r / nk;
    const int64_t g = kept[int64_t(e) * nk + i], h = kept[int64_t(e) * nk + j];
    if (g != h && !ki.coupled(ki.kind(g), ki.kind(h))) continue;
    int64_t lo = rp[g], hi = rp[g + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cols[mid] < h) lo = mid + 1;
      else hi = mid;
    }
    if (lo >= rp[g + 1] || cols[lo] != h) {
      atomicExch(bad, 1);
      continue;
    }
    atomicAdd(vals + lo, schur[int64_t(e) * per + i + int64_t(j) * nk]);
    if (i == j && rhs) atomicAdd(rhs + g, rrhs[int64_t(e) * nk + i]);
  }
}

} // namespace

void assemble_values(Context& c, int nelem, int nk, const int64_t* kept, const double* schur,
                     const double* rrhs, const pscu_layout& l, Csr& a, double* rhs) {
  KindInfo ki;
  ki.fb = 2 * l.face_vel + l.face_press;
  ki.eb = 2 * l.elem_vel + l.elem_press;
  ki.face_rows = int64_t(l.n_faces) * ki.fb;
  ki.face_vel = l.face_vel;
  ki.elem_vel = l.elem_vel;
  ki.strategy = l.strategy;
  PSCU_CUDA(cudaMemsetAsync(a.vals.p, 0, sizeof(double) * a.nnz, c.stream));
  if (rhs) PSCU_CUDA(cudaMemsetAsync(rhs, 0, sizeof(double) * a.n, c.stream));
  const int zero = 0;
  PSCU_CUDA(cudaMemcpyAsync(c.err_flag.p, &zero, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  const int64_t total = int64_t(nelem) * nk * nk;
  const int64_t g = (total + 255) / 256;
  assemble_kernel<<<unsigned(g < 148 * 64 ? (g > 0 ? g : 1) : 148 * 64), 256, 0, c.stream>>>(
      nelem, nk, kept, schur, rrhs, ki, a.row_ptr.p, a.cols.p, a.vals.p, rhs, c.err_flag.p);
  PSCU_LAUNCHED(&c);
  int bad = 0;
  PSCU_CUDA(cudaMemcpyAsync(&bad, c.err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  if (bad) throw Error(PSCU_EINVAL, "CsrMatrix::add: entry outside the pattern");
}

void condense_batch(Context& c, int nelem, int n, const double* mats, const double* rhs, int ne,
                    const int* elim_host, double* schur, double* rrhs, double* coupling,
                    double* erhs, int* bad_element) {
  if (n > 255 || ne > 64)
    throw Error(PSCU_EINVAL, "condense: local block too large for the shared-memory kernel");
  std::vector<int> is_elim(n, 0), keep;
  for (int i = 0; i < ne; ++i) {
    if (elim_host[i] < 0 || elim_host[i] >= n) throw Error(PSCU_EINVAL, "condense: bad elim index");
    is_elim[elim_host[i]] = 1;
  }
  for (int i = 0; i < n; ++i)
    if (!is_elim[i]) keep.push_back(i);
  const int nk = int(keep.size());
  DevBuf<int> d_elim, d_keep;
  d_elim.upload(elim_host, ne > 0 ? ne : 0, c.stream);
  if (ne == 0) d_elim.alloc(1);
  d_keep.upload(keep, c.stream);
  const int big = 0x7fffffff;
  PSCU_CUDA(cudaMemcpyAsync(c.err_flag.p, &big, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  const size_t smem = sizeof(double) * (size_t(n) * (n + 1) + size_t(ne) * ne + size_t(ne) * (nk + 1));
  if (smem > 48 * 1024)
    PSCU_CUDA(cudaFuncSetAttribute(condense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
  const int grid = nelem < 148 * 8 ? (nelem > 0 ? nelem : 1) : 148 * 8;
  condense_kernel<<<grid, kCondThreads, smem, c.stream>>>(nelem, n, mats, rhs, ne, d_elim.p,
                                                          d_keep.p, schur, rrhs, coupling, erhs,
                                                          c.err_flag.p);
  PSCU_LAUNCHED(&c);
  int bad = big;
  PSCU_CUDA(cudaMemcpyAsync(&bad, c.err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  if (bad_element) *bad_element = bad == big ? -1 : bad;
  if (bad != big)
    throw Error(PSCU_ESINGULAR,
                "condense: near-singular eliminated block on element " + std::to_string(bad));
}

void recover_batch(Context& c, int nelem, int n, int ne, const int* elim_host,
                   const int64_t* kept, const double* coupling, const double* erhs,
                   const double* x, double* locals) {
  std::vector<int> is_elim(n, 0), keep;
  for (int i = 0; i < ne; ++i) is_elim[elim_host[i]] = 1;
  for (int i = 0; i < n; ++i)
    if (!is_elim[i]) keep.push_back(i);
  DevBuf<int> d_elim, d_keep;
  d_elim.upload(elim_host, ne, c.stream);
  if (ne == 0) d_elim.alloc(1);
  d_keep.upload(keep, c.stream);
  const int grid = nelem < 148 * 8 ? (nelem > 0 ? nelem : 1) : 148 * 8;
  recover_kernel<<<grid, 128, 0, c.stream>>>(nelem, n, ne, d_elim.p, d_keep.p, kept, coupling,
                                             erhs, x, locals);
  PSCU_LAUNCHED(&c);
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
}

} // namespace pscu
