// Batched static condensation of large element blocks (the 3D HHO-hp
// vp-cond blocks: n = 214, 70 eliminated, 144 retained at k = 2) fused with
// the value scatter into face-block (BSR) storage: condense_element
// (condense.hpp:57-97) + scatter_block / the reduced-load accumulation of
// assemble_hho (assemble.hpp:121-131, 164-169) in one kernel.
//
// One CTA per element. Shared memory holds the eliminated block's LU
// (ne^2), the solutions X = A_ee^-1 [A_ek | b_e] (ne (nk+1)) and A_ke
// (nk ne); the local block itself stays in global memory and is read once
// per entry used. Every entry receives its operations in the order of
// include/eigen_subset's PartialPivLU / GEMM, which oracle/pstokes_oracle.c
// (po_condense) restates, so the Schur complement and the assembled
// operator are bitwise equal to the oracle's:
//  * LU: pivot = first largest |a_ik|, full-row swap, a_ik /= a_kk, then
//    a_ij -= a_ik a_kj for j > k with a_kj != 0;
//  * solves: one thread per right-hand-side column, forward then backward
//    substitution with the sums j ascending;
//  * Schur: s = 0, s += A_ke(i,k) X(k,j) for k ascending, S = A_kk - s,
//    each thread folding a 2 x 2 register tile (four independent chains).
// The FP64 tensor pipe (DMMA) fuses each multiply-add, so the default path
// does not use it; PSCU_CONDENSE_DMMA=1 switches the Schur products to
// mma.sync.m8n8k4.f64 (rounding-level differences).
//
// The Schur entries are scattered straight from registers: retained dof i of
// the element is (local face lf_i, offset o_i in the face block), so entry
// (i, j) lands in block (face(lf_i), face(lf_j)) at column-major position
// (o_j, o_i). A face-pair block receives one element's contribution
// (distinct hexahedral faces share at most one element) and a diagonal
// block two; a two-term sum from 0.0 is order-independent, so the atomics
// reproduce the reference's element-order sums bit for bit. Exact zeros are
// skipped except on the diagonal, like scatter_block.
#include <algorithm>

#include "internal.cuh"

namespace pscu {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxFacesPerElem = 8;

struct ScatterArgs {
  const int64_t* brp;
  const int32_t* bcols;
  double* vals;  // BSR values (column-major blocks)
  double* rhs;   // assembled reduced load
  int bs;
  const int32_t* efaces;  // nelem x nfe block-column ids of the element's faces
  const int32_t* erows;   // nelem x nfe block-row ids (-1: a row this operator does not hold)
  int nfe;
  const int2* keep_pos;   // nk x (local face, offset in the face block)
};

__global__ void __launch_bounds__(kThreads)
    condense_bsr_kernel(int e0, int nelem, int n, const double* __restrict__ mats,
                        const double* __restrict__ rhs, int ne, const int* __restrict__ elim,
                        const int* __restrict__ keep, ScatterArgs sa,
                        double* __restrict__ coupling, double* __restrict__ erhs, int* bad,
                        int dmma) {
  extern __shared__ double sm[];
  const int nk = n - ne;
  // X is kept transposed, X(k, col) at X[col + k P] with P odd: a thread
  // owning one column walks it without bank conflicts
  const int P = (nk + 1) | 1;
  double* LU = sm;                         // ne x ne, column-major
  double* X = LU + size_t(ne) * ne;        // (nk + 1) columns x ne rows, transposed
  double* AKE = X + size_t(ne) * P;        // nk x ne
  __shared__ int perm[128];
  __shared__ int piv_row, singular;
  __shared__ int64_t qpair[kMaxFacesPerElem * kMaxFacesPerElem];
  __shared__ double colnorm[128], acol[128];
  for (int le = blockIdx.x; le < nelem; le += gridDim.x) {
    const int e = e0 + le;
    const double* M = mats + size_t(le) * n * n;
    const double* b = rhs + size_t(le) * n;
    // (warps over columns, lanes over rows: no integer division in the
    // index arithmetic, which otherwise saturates the XU pipe)
    const int lane_ = int(threadIdx.x & 31), warp_ = int(threadIdx.x >> 5), nwarp_ = int(blockDim.x >> 5);
    for (int j = warp_; j < ne; j += nwarp_) {
      const double* Mj = M + size_t(elim[j]) * n;
      for (int i = lane_; i < ne; i += 32) LU[i + j * ne] = Mj[elim[i]];
    }
    for (int t = threadIdx.x; t < ne; t += blockDim.x) perm[t] = t;
    // block position of every (local face, local face) pair of this element
    for (int t = threadIdx.x; t < sa.nfe * sa.nfe; t += blockDim.x) {
      const int F = sa.erows[size_t(le) * sa.nfe + t / sa.nfe];
      const int G = sa.efaces[size_t(le) * sa.nfe + t % sa.nfe];
      if (F < 0) {
        qpair[t] = -3;  // row held by another shard: skipped
        continue;
      }
      int64_t q = sa.brp[F];
      const int64_t q1 = sa.brp[F + 1];
      while (q < q1 && sa.bcols[q] != G) ++q;
      qpair[t] = q < q1 ? q : -1;
    }
    if (threadIdx.x == 0) singular = 0;
    __syncthreads();
    // absolute column sums of A_ee for the rcond guard's 1-norm (rows
    // ascending from 0.0, the guard's order), before the LU overwrites it
    for (int j = threadIdx.x; j < ne; j += blockDim.x) {
      double s = 0.0;
      for (int i = 0; i < ne; ++i) s += fabs(LU[i + j * ne]);
      acol[j] = s;
    }
    __syncthreads();
    // partial-pivot LU (PartialPivLU::compute of include/eigen_subset)
    for (int k = 0; k < ne; ++k) {
      if (threadIdx.x < 32) {
        // first largest |a_ik|, i >= k: warp arg-max, ties to the lower row
        double best = -1.0;
        int bi = k;
        for (int i = k + int(threadIdx.x); i < ne; i += 32) {
          const double v = fabs(LU[i + k * ne]);
          if (v > best) {
            best = v;
            bi = i;
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_down_sync(0xffffffffu, best, o);
          const int oi = __shfl_down_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) {
            best = ov;
            bi = oi;
          }
        }
        if (threadIdx.x == 0) {
          piv_row = bi;
          if (bi != k) {
            const int t = perm[k];
            perm[k] = perm[bi];
            perm[bi] = t;
          }
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
        for (int j = k + 1 + warp_; j < ne; j += nwarp_) {
          const double ukj = LU[k + j * ne];
          if (ukj != 0.0)
            for (int i = k + 1 + lane_; i < ne; i += 32)
              LU[i + j * ne] = dsub(LU[i + j * ne], dmul(LU[i + k * ne], ukj));
        }
      }
      __syncthreads();
    }
    // solves (one thread per column of [A_ek | b_e]) and, on the remaining
    // threads, the inverse columns of the rcond guard
    const int ncol = nk + 1;
    for (int col = warp_; col < ncol; col += nwarp_) {
      const double* src = col < nk ? M + size_t(keep[col]) * n : b;
      for (int i = lane_; i < ne; i += 32) X[col + size_t(i) * P] = src[elim[perm[i]]];
    }
    // the rcond guard's inverse columns share the pass (threads past the
    // right-hand sides), in the not-yet-staged A_ke region, transposed too
    const int PI = ne | 1;
    double* XI = AKE;
    for (int c = warp_; c < ne; c += nwarp_)
      for (int i = lane_; i < ne; i += 32) XI[c + size_t(i) * PI] = perm[i] == c ? 1.0 : 0.0;
    __syncthreads();
    for (int col = threadIdx.x; col < ncol + ne; col += blockDim.x) {
      double* x = col < ncol ? X + col : XI + (col - ncol);  // x[i S]
      const int S = col < ncol ? P : PI;
      // forward substitution (unit L) in axpy form: entry i still takes its
      // terms j = 0, 1, ... in order with x_j final, the dot form's
      // operations, but the updates of one step are independent
      for (int j = 0; j + 1 < ne; ++j) {
        const double xj = x[size_t(j) * S];
        const double* l = LU + size_t(j) * ne;
        int i = j + 1;
        for (; i + 4 <= ne; i += 4) {
          double lv[4], xv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            lv[u] = l[i + u];
            xv[u] = x[size_t(i + u) * S];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) x[size_t(i + u) * S] = dsub(xv[u], dmul(lv[u], xj));
        }
        for (; i < ne; ++i) x[size_t(i) * S] = dsub(x[size_t(i) * S], dmul(l[i], xj));
      }
      // backward substitution: row i's chain starts at the value found last
      for (int i = ne - 1; i >= 0; --i) {
        double s = x[size_t(i) * S];
        int j = i + 1;
        for (; j + 4 <= ne; j += 4) {
          double pr[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) pr[u] = dmul(LU[i + size_t(j + u) * ne], x[size_t(j + u) * S]);
#pragma unroll
          for (int u = 0; u < 4; ++u) s = dsub(s, pr[u]);
        }
        for (; j < ne; ++j) s = dsub(s, dmul(LU[i + size_t(j) * ne], x[size_t(j) * S]));
        x[size_t(i) * S] = __ddiv_rn(s, LU[i + i * ne]);
      }
      if (col >= ncol) {
        // exact inverse 1-norm for rcond: column sums, rows ascending
        double s = 0.0;
        for (int i = 0; i < ne; ++i) s += fabs(x[size_t(i) * S]);
        colnorm[col - ncol] = s;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      bool sing = false;
      for (int i = 0; i < ne; ++i) sing = sing || LU[i + i * ne] == 0.0;
      if (!sing) {
        double an = 0.0, inorm = 0.0;
        for (int j = 0; j < ne; ++j) {
          an = fmax(an, acol[j]);
          inorm = fmax(inorm, colnorm[j]);
        }
        const double rc = (an > 0.0 && inorm > 0.0 && isfinite(inorm)) ? (1.0 / an) / inorm : 0.0;
        sing = rc < 1e-14;
      }
      if (sing) {
        singular = 1;
        atomicMin(bad, e);
      }
    }
    __syncthreads();
    if (!singular) {
      // A_ke now (its region held the inverse columns until the guard ran)
      for (int j = warp_; j < ne; j += nwarp_) {
        const double* Mj = M + size_t(elim[j]) * n;
        for (int i = lane_; i < nk; i += 32) AKE[i + j * nk] = Mj[keep[i]];
      }
      __syncthreads();
      if (coupling)
        for (int col = warp_; col < nk; col += nwarp_)
          for (int i = lane_; i < ne; i += 32)
            coupling[size_t(le) * ne * nk + size_t(col) * ne + i] = X[col + size_t(i) * P];
      if (erhs)
        for (int t = threadIdx.x; t < ne; t += blockDim.x)
          erhs[size_t(le) * ne + t] = X[nk + size_t(t) * P];
      // one Schur / reduced-load entry: S(i, j) = A_kk(i, j) - s (j == nk: the
      // load), scattered from registers
      const int64_t bs2 = int64_t(sa.bs) * sa.bs;
      auto emit = [&](int i, int j, double sum) {
        const double* src = j < nk ? M + size_t(keep[j]) * n : b;
        const double v = dsub(src[keep[i]], sum);
        const int2 pi = sa.keep_pos[i];
        if (j == nk) {
          const int F = sa.erows[size_t(le) * sa.nfe + pi.x];
          if (F >= 0) atomicAdd(sa.rhs + int64_t(F) * sa.bs + pi.y, v);
          return;
        }
        const int2 pj = sa.keep_pos[j];
        const bool diag = pi.x == pj.x && pi.y == pj.y;
        if (v == 0.0 && !diag) return;
        const int64_t q = qpair[pi.x * sa.nfe + pj.x];
        if (q == -3) return;
        if (q < 0) {
          atomicExch(bad, -2);
          return;
        }
        atomicAdd(sa.vals + q * bs2 + int64_t(pj.y) * sa.bs + pi.y, v);
      };
      if (dmma) {
        // FP64 tensor-pipe variant (opt-in): s = A_ke X on
        // mma.sync.m8n8k4.f64, 16 x 16 outputs per warp step (2 x 2 tiles),
        // k ascending in steps of 4 from a zero accumulator. The tensor pipe
        // fuses each multiply-add (one rounding where the reference order
        // takes two), so the entries agree with the SIMT path to rounding
        // (~1e-16 relative to the row's terms), not bit for bit.
        const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
        const int nwarp = int(blockDim.x >> 5), g = lane >> 2, q4 = lane & 3;
        const int mt2 = (nk + 15) / 16, nt2 = (ncol + 15) / 16;
        for (int t = warp; t < mt2 * nt2; t += nwarp) {
          const int i0 = 16 * (t % mt2), j0 = 16 * (t / mt2);
          double c[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
          for (int k0 = 0; k0 < ne; k0 += 4) {
            const int k = k0 + q4;
            double av[2], bv[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int i = i0 + 8 * h + g, j = j0 + 8 * h + g;
              av[h] = (k < ne && i < nk) ? AKE[i + k * nk] : 0.0;
              bv[h] = (k < ne && j < ncol) ? X[j + size_t(k) * P] : 0.0;
            }
#pragma unroll
            for (int hi = 0; hi < 2; ++hi)
#pragma unroll
              for (int hj = 0; hj < 2; ++hj)
                asm volatile(
                    "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(c[hi][hj][0]), "+d"(c[hi][hj][1])
                    : "d"(av[hi]), "d"(bv[hj]));
          }
#pragma unroll
          for (int hi = 0; hi < 2; ++hi)
#pragma unroll
            for (int hj = 0; hj < 2; ++hj)
#pragma unroll
              for (int d = 0; d < 2; ++d) {
                const int i = i0 + 8 * hi + g, j = j0 + 8 * hj + 2 * q4 + d;
                if (i < nk && j < ncol) emit(i, j, c[hi][hj][d]);
              }
        }
      } else {
        // reference order (bitwise): 2 x 2 register tiles of independent chains
        const int ti = (nk + 1) / 2, tj = (ncol + 1) / 2;
        for (int t = threadIdx.x; t < ti * tj; t += blockDim.x) {
          const int i0 = 2 * (t % ti), j0 = 2 * (t / ti);
          const int i1 = min(i0 + 1, nk - 1), j1 = min(j0 + 1, ncol - 1);
          double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;
          for (int k = 0; k < ne; ++k) {
            const double a0 = AKE[i0 + k * nk], a1 = AKE[i1 + k * nk];
            const double x0 = X[j0 + size_t(k) * P], x1 = X[j1 + size_t(k) * P];
            s00 = dadd(s00, dmul(a0, x0));
            s01 = dadd(s01, dmul(a0, x1));
            s10 = dadd(s10, dmul(a1, x0));
            s11 = dadd(s11, dmul(a1, x1));
          }
          emit(i0, j0, s00);
          if (j1 != j0) emit(i0, j1, s01);
          if (i1 != i0) emit(i1, j0, s10);
          if (i1 != i0 && j1 != j0) emit(i1, j1, s11);
        }
      }
    }
    __syncthreads();
  }
}

/// PSCU_CONDENSE_DMMA=1: Schur products on the FP64 tensor pipe (rounding-level
/// differences from the reference order; default 0 = bitwise SIMT chains).
int condense_dmma() {
  const char* e = getenv("PSCU_CONDENSE_DMMA");
  return e && atoi(e) != 0;
}

} // namespace

void condense_scatter_bsr(Context& c, Csr& a, int e0, int nelem, int n, const double* mats,
                          const double* rhs, int ne, const int* elim_host, const int32_t* efaces,
                          const int32_t* erows, int nfe, const int32_t* keep_pos_host,
                          double* rhs_acc, double* coupling, double* erhs) {
  if (!a.bs) throw Error(PSCU_EINVAL, "condense_scatter: the operator must use block storage");
  if (n > 256 || ne > 128 || ne < 1 || nfe > kMaxFacesPerElem)
    throw Error(PSCU_EINVAL, "condense_scatter: local block too large for the kernel");
  std::vector<int> is_elim(n, 0), keep;
  for (int i = 0; i < ne; ++i) {
    if (elim_host[i] < 0 || elim_host[i] >= n) throw Error(PSCU_EINVAL, "condense: bad elim index");
    is_elim[elim_host[i]] = 1;
  }
  for (int i = 0; i < n; ++i)
    if (!is_elim[i]) keep.push_back(i);
  const int nk = int(keep.size());
  std::vector<int2> kp(nk);
  for (int i = 0; i < nk; ++i) {
    kp[i] = make_int2(keep_pos_host[2 * i], keep_pos_host[2 * i + 1]);
    if (kp[i].x < 0 || kp[i].x >= nfe || kp[i].y < 0 || kp[i].y >= a.bs)
      throw Error(PSCU_EINVAL, "condense_scatter: retained dof outside the face blocks");
  }
  DevBuf<int> d_elim, d_keep;
  DevBuf<int2> d_kp;
  d_elim.upload(elim_host, ne, c.stream);
  d_keep.upload(keep, c.stream);
  d_kp.upload(kp, c.stream);
  const int big = 0x7fffffff;
  PSCU_CUDA(cudaMemcpyAsync(c.err_flag.p, &big, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  const size_t smem =
      sizeof(double) * (size_t(ne) * ne + size_t(ne) * ((nk + 1) | 1) +
                        std::max(size_t(nk) * ne, size_t(ne) * (ne | 1)));
  if (smem > 227 * 1024) throw Error(PSCU_EINVAL, "condense_scatter: block too large for shared memory");
  static size_t attr = 0;
  if (smem > attr) {
    PSCU_CUDA(cudaFuncSetAttribute(condense_bsr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
    attr = smem;
  }
  ScatterArgs sa{a.brow_ptr.p, a.bcols.p, a.vals.p, rhs_acc, a.bs, efaces,
                 erows ? erows : efaces, nfe, d_kp.p};
  int per_sm = 1;
  PSCU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, condense_bsr_kernel, kThreads, smem));
  const int grid = std::max(1, std::min(nelem, 148 * std::max(1, per_sm)));
  condense_bsr_kernel<<<grid, kThreads, smem, c.stream>>>(e0, nelem, n, mats, rhs, ne, d_elim.p,
                                                          d_keep.p, sa, coupling, erhs,
                                                          c.err_flag.p, condense_dmma());
  PSCU_LAUNCHED(&c);
  int bad = big;
  PSCU_CUDA(cudaMemcpyAsync(&bad, c.err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  if (bad == -2) throw Error(PSCU_EINVAL, "CsrMatrix::add: entry outside the sparsity pattern");
  if (bad != big)
    throw Error(PSCU_ESINGULAR,
                "condense: near-singular eliminated block on element " + std::to_string(bad));
}

} // namespace pscu
