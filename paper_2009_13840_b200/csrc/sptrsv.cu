// ILU(0) factorisation and application (Ilu0, ilu0.hpp:19-65).
//
// Factorisation: the IKJ update of row i needs every row k < i it references
// below the diagonal to be final, so rows are factored level by level over
// the forward DAG (one launch per level, one thread per row). Each row
// receives its updates in k-ascending order with non-fused operations,
// exactly like the reference's sequential loop, so the factors are
// bit-identical. Application: the level walkers of walk.cu.
#include <algorithm>

#include <chrono>
#include <cstdlib>

#include "internal.cuh"
#include "walk.cuh"

namespace pscu {

namespace {

/// Row i of the IKJ loop (ilu0.hpp:29-50) for the rows of one DAG level.
__global__ void ilu0_factor_level(int nrows, const int32_t* __restrict__ rows,
                                  const int64_t* __restrict__ rp,
                                  const int32_t* __restrict__ cols, double* lu,
                                  const int64_t* __restrict__ diag, int* err) {
  for (int t = int(blockIdx.x * blockDim.x + threadIdx.x); t < nrows; t += gridDim.x * blockDim.x) {
    const int i = rows[t];
    const int64_t ri1 = rp[i + 1], di = diag[i];
    for (int64_t p = rp[i]; p < di; ++p) {
      const int k = cols[p];
      const double piv = lu[diag[k]];
      if (piv == 0.0) atomicMin(err, k);
      const double lik = __ddiv_rn(lu[p], piv);
      lu[p] = lik;
      int64_t r = p + 1;
      const int64_t qe = rp[k + 1];
      for (int64_t q = diag[k] + 1; q < qe; ++q) {
        const int cq = cols[q];
        while (r < ri1 && cols[r] < cq) ++r;
        if (r < ri1 && cols[r] == cq) lu[r] = dsub(lu[r], dmul(lik, lu[q]));
      }
    }
    if (lu[di] == 0.0) atomicMin(err, i);
  }
}

/// The same with one warp per row: row i sits in shared memory; for each k
/// of its lower part (ascending, as the reference) the lanes take row k's
/// upper entries 32 at a time, find their column in row i by binary search
/// and apply lu[r] -= l_ik * lu[q] (distinct r per k, so the updates of an
/// entry still arrive in k order, individually rounded: bit-identical).
/// Global loads are one round per k instead of one per merge step.
constexpr int kFacWarps = 4;
constexpr int kFacMaxRow = 256;

__global__ void __launch_bounds__(32 * kFacWarps)
    ilu0_factor_level_warp(int nrows, const int32_t* __restrict__ rows,
                           const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                           double* lu, const int64_t* __restrict__ diag, int* err) {
  __shared__ int32_t sc[kFacWarps][kFacMaxRow];
  __shared__ double sv[kFacWarps][kFacMaxRow];
  const int w = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  for (int t = int(blockIdx.x) * kFacWarps + w; t < nrows; t += gridDim.x * kFacWarps) {
    const int i = rows[t];
    const int64_t r0 = rp[i];
    const int len = int(rp[i + 1] - r0), di = int(diag[i] - r0);
    for (int e = lane; e < len; e += 32) {
      sc[w][e] = cols[r0 + e];
      sv[w][e] = lu[r0 + e];
    }
    __syncwarp();
    for (int p = 0; p < di; ++p) {
      const int k = sc[w][p];
      const int64_t dk = diag[k], qe = rp[k + 1];
      const double piv = lu[dk];
      if (piv == 0.0 && lane == 0) atomicMin(err, k);
      const double lik = __ddiv_rn(sv[w][p], piv);
      __syncwarp();
      if (lane == 0) sv[w][p] = lik;
      for (int64_t q0 = dk + 1; q0 < qe; q0 += 32) {
        const int64_t q = q0 + lane;
        if (q < qe) {
          const int cq = cols[q];
          const double lq = lu[q];
          int lo = p + 1, hi = len;  // first entry of row i with column >= cq
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sc[w][mid] < cq) lo = mid + 1;
            else hi = mid;
          }
          if (lo < len && sc[w][lo] == cq) sv[w][lo] = dsub(sv[w][lo], dmul(lik, lq));
        }
      }
      __syncwarp();
    }
    for (int e = lane; e < len; e += 32) lu[r0 + e] = sv[w][e];
    if (lane == 0 && sv[w][di] == 0.0) atomicMin(err, i);
    __syncwarp();
  }
}

} // namespace

void ilu0_factor_start(Context& c, Ilu& ilu) {
  const Csr& a = *ilu.a;
  if (a.n == 0) return;
  const int64_t n = a.n;
  const bool dbg = getenv("PSCU_DEBUG") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<int64_t>& diag = ilu.h_diag;
  diag.assign(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    const auto b = a.h_cols.begin() + a.h_row_ptr[i];
    const auto e = a.h_cols.begin() + a.h_row_ptr[i + 1];
    const auto it = std::lower_bound(b, e, int32_t(i));
    if (it == e || *it != i)
      throw Error(PSCU_ESINGULAR, "ilu0: row " + std::to_string(i) +
                                      " has no diagonal entry; reorder or extend the pattern");
    diag[i] = it - a.h_cols.begin();
  }
  ilu.diag.upload(diag, c.stream);
  // forward DAG levels for the factorisation launches
  std::vector<int32_t> lvl(n, 0);
  int nlev = 0;
  for (int64_t i = 0; i < n; ++i) {
    int L = 0;
    for (int64_t q = a.h_row_ptr[i]; q < diag[i]; ++q) L = std::max(L, lvl[a.h_cols[q]] + 1);
    lvl[i] = L;
    nlev = std::max(nlev, L + 1);
  }
  ilu.flev_ptr.assign(nlev + 1, 0);
  for (int64_t i = 0; i < n; ++i) ilu.flev_ptr[lvl[i] + 1]++;
  for (int l = 0; l < nlev; ++l) ilu.flev_ptr[l + 1] += ilu.flev_ptr[l];
  std::vector<int32_t> rows(n);
  {
    std::vector<int32_t> fill(ilu.flev_ptr.begin(), ilu.flev_ptr.end() - 1);
    for (int64_t i = 0; i < n; ++i) rows[fill[lvl[i]]++] = int32_t(i);
  }
  ilu.flev_rows.upload(rows, c.stream);
  ilu.lu.alloc(a.nnz);
  PSCU_CUDA(cudaMemcpyAsync(ilu.lu.p, a.vals.p, sizeof(double) * a.nnz, cudaMemcpyDeviceToDevice,
                            c.stream));
  const int big = 0x7fffffff;
  PSCU_CUDA(cudaMemcpyAsync(c.err_flag.p, &big, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (dbg) {
    PSCU_CUDA(cudaEventCreate(&e0));
    PSCU_CUDA(cudaEventCreate(&e1));
    PSCU_CUDA(cudaEventRecord(e0, c.stream));
  }
  const auto t1 = std::chrono::steady_clock::now();
  int64_t maxrow = 0;
  for (int64_t i = 0; i < n; ++i) maxrow = std::max(maxrow, a.h_row_ptr[i + 1] - a.h_row_ptr[i]);
  const bool warp_rows = maxrow <= kFacMaxRow && !getenv("PSCU_FACTOR_THREAD");
  for (int l = 0; l < nlev; ++l) {
    const int nr = ilu.flev_ptr[l + 1] - ilu.flev_ptr[l];
    if (warp_rows) {
      const int grid = std::min((nr + kFacWarps - 1) / kFacWarps, 148 * 16);
      ilu0_factor_level_warp<<<grid, 32 * kFacWarps, 0, c.stream>>>(
          nr, ilu.flev_rows.p + ilu.flev_ptr[l], a.row_ptr.p, a.cols.p, ilu.lu.p, ilu.diag.p,
          c.err_flag.p);
    } else {
      const int grid = std::min((nr + 127) / 128, 148 * 8);
      ilu0_factor_level<<<grid, 128, 0, c.stream>>>(nr, ilu.flev_rows.p + ilu.flev_ptr[l],
                                                     a.row_ptr.p, a.cols.p, ilu.lu.p, ilu.diag.p,
                                                     c.err_flag.p);
    }
    PSCU_LAUNCHED(&c);
  }
  if (dbg) {
    PSCU_CUDA(cudaEventRecord(e1, c.stream));
    const auto t2 = std::chrono::steady_clock::now();
    PSCU_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PSCU_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    fprintf(stderr, "[setup] ilu0 factor n=%lld: host prep %.3f s, %d level launches issued in %.3f s, device %.3f s\n",
            (long long)n, std::chrono::duration<double>(t1 - t0).count(), nlev,
            std::chrono::duration<double>(t2 - t1).count(), ms / 1e3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
}

void ilu0_factor_finish(Context& c, Ilu& ilu) {
  if (ilu.a->n == 0) return;
  const int big = 0x7fffffff;
  int bad = 0;
  PSCU_CUDA(cudaMemcpyAsync(&bad, c.err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  if (bad != big)
    throw Error(PSCU_ESINGULAR, "ilu0: zero pivot at row " + std::to_string(bad) +
                                    "; a fill-reducing or pivot-friendly ordering is needed");
  pack_walk(c, ilu.lu.p, ilu.wfwd);
  pack_walk(c, ilu.lu.p, ilu.wbwd);
}

void ilu0_factor(Context& c, Ilu& ilu) {
  ilu0_factor_start(c, ilu);
  if (ilu.a->n == 0) return;
  // host planning of the sweeps overlaps the factorisation launches
  const auto tw = std::chrono::steady_clock::now();
  build_walk(c, *ilu.a, ilu.h_diag, ilu.wfwd, ilu.wbwd);
  if (getenv("PSCU_DEBUG"))
    fprintf(stderr, "[setup] walk plans n=%lld: %.3f s\n", (long long)ilu.a->n,
            std::chrono::duration<double>(std::chrono::steady_clock::now() - tw).count());
  ilu0_factor_finish(c, ilu);
}

void ilu0_apply(Context& c, const Ilu& ilu, const double* x, double* y) {
  const Csr& a = *ilu.a;
  if (a.n == 0) return;
  // algorithmic bytes of one apply: 8 nnz + 32 n
  Context::Scope prof(&c, PROF_ILU, 8.0 * double(a.nnz) + 32.0 * double(a.n));
  run_walk(c, ilu.wfwd, ilu.wbwd, x, y);
}

} // namespace pscu
