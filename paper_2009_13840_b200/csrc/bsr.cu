// Dense face-block (BSR) storage of the condensed operator, for patterns made
// of dense bs x bs blocks: the 3D HHO-hp vp-cond operator (24 x 24 blocks at
// k = 2, 12 at k = 1, 4 at k = 0; SURVEY.md §8 G2 "hp vp-cond: face-only,
// dense 24x24 FF blocks"). It replaces the CSR index stream (4 B per entry,
// 1.5x the value bytes) by one int32 per block, so the SpMV moves the
// structural 8 B per entry + 16 B per row.
//
// Bitwise parity with CsrMatrix::multiply (csr.hpp:68-74): the CSR row order
// of a dense-block pattern is block column ascending, then column within the
// block ascending (csr.hpp:30-44 sorts the columns; the layout numbers face
// f's dofs [f bs, (f+1) bs)), so each thread folds its row block by block,
// column by column, starting from 0.0, one rounding per operation.
//
// Blocks are stored column-major: entry (r, c) of block q at
// vals[q bs^2 + c bs + r], so the bs threads of a block row read bs
// consecutive doubles per column (coalesced) and the same x value
// (broadcast).
#include <algorithm>
#include <thread>

#include "internal.cuh"

namespace pscu {

namespace {

unsigned grid_for(int64_t n, int threads) {
  const int64_t g = (n + threads - 1) / threads;
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(148) * 64)));
}

/// y = A x, one thread per row. Values are streamed once (evict-first
/// loads); x stays in L2 (a block column is read by ~11 block rows).
template <int kBs>
__global__ void __launch_bounds__(256) spmv_bsr_kernel(int64_t n, int bs_rt,
                                                       const int64_t* __restrict__ brp,
                                                       const int32_t* __restrict__ bcols,
                                                       const double* __restrict__ vals,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y) {
  const int bs = kBs > 0 ? kBs : bs_rt;
  const int64_t bs2 = int64_t(bs) * bs;
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n;
       row += int64_t(gridDim.x) * blockDim.x) {
    const int64_t f = row / bs;
    const int r = int(row - f * bs);
    const int64_t q0 = brp[f], q1 = brp[f + 1];
    double s = 0.0;
    for (int64_t q = q0; q < q1; ++q) {
      const double* A = vals + q * bs2 + r;
      const double* xg = x + int64_t(__ldg(bcols + q)) * bs;
      if (kBs > 0) {
        double a[kBs > 0 ? kBs : 1], xv[kBs > 0 ? kBs : 1];
#pragma unroll
        for (int c = 0; c < kBs; ++c) {
          a[c] = __ldcs(A + c * kBs);
          xv[c] = __ldg(xg + c);
        }
#pragma unroll
        for (int c = 0; c < kBs; ++c) s = dadd(s, dmul(a[c], xv[c]));
      } else {
        for (int c = 0; c < bs; ++c) s = dadd(s, dmul(__ldcs(A + c * bs), __ldg(xg + c)));
      }
    }
    y[row] = s;
  }
}

/// rc[i] = d[r] - (A w)[r], r = map[i] (fused residual + restriction,
/// plevels.hpp:178), one thread per selected row.
template <int kBs>
__global__ void __launch_bounds__(256) resid_restrict_bsr_kernel(
    int64_t nc, int bs_rt, const int64_t* __restrict__ map, const int64_t* __restrict__ brp,
    const int32_t* __restrict__ bcols, const double* __restrict__ vals,
    const double* __restrict__ d, const double* __restrict__ w, double* __restrict__ rc) {
  const int bs = kBs > 0 ? kBs : bs_rt;
  const int64_t bs2 = int64_t(bs) * bs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nc;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = map[i];
    const int64_t f = row / bs;
    const int r = int(row - f * bs);
    double s = 0.0;
    for (int64_t q = brp[f]; q < brp[f + 1]; ++q) {
      const double* A = vals + q * bs2 + r;
      const double* xg = w + int64_t(__ldg(bcols + q)) * bs;
      if (kBs > 0) {
        double a[kBs > 0 ? kBs : 1], xv[kBs > 0 ? kBs : 1];
#pragma unroll
        for (int c = 0; c < kBs; ++c) {
          a[c] = __ldcs(A + c * kBs);
          xv[c] = __ldg(xg + c);
        }
#pragma unroll
        for (int c = 0; c < kBs; ++c) s = dadd(s, dmul(a[c], xv[c]));
      } else {
        for (int c = 0; c < bs; ++c) s = dadd(s, dmul(__ldcs(A + c * bs), __ldg(xg + c)));
      }
    }
    rc[i] = dsub(d[row], s);
  }
}

/// Coarse block entries are a pure gather of the fine block entries
/// (rows and columns through the in-block map).
__global__ void inherit_bsr_kernel(int64_t total, int bf, int bc, const int32_t* __restrict__ m,
                                   const double* __restrict__ fine, double* __restrict__ out) {
  const int64_t bc2 = int64_t(bc) * bc, bf2 = int64_t(bf) * bf;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = t / bc2;
    const int e = int(t - q * bc2);
    const int cc = e / bc, rr = e - cc * bc;
    out[t] = fine[q * bf2 + int64_t(m[cc]) * bf + m[rr]];
  }
}

/// BSR -> CSR values: entry (r, c) of block q lands at position
/// brp[f] bs^2 + r (len_f bs) + (q - brp[f]) bs + c of the expanded rows.
__global__ void bsr_to_csr_kernel(int64_t total, int bs, const int64_t* __restrict__ brp,
                                  const int32_t* __restrict__ brow_of,
                                  const double* __restrict__ vals, double* __restrict__ out) {
  const int64_t bs2 = int64_t(bs) * bs;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = t / bs2;
    const int e = int(t - q * bs2);
    const int c = e / bs, r = e - c * bs;
    const int64_t f = brow_of[q];
    const int64_t b0 = brp[f], len = brp[f + 1] - b0;
    out[b0 * bs2 + int64_t(r) * len * bs + (q - b0) * bs + c] = vals[t];
  }
}

/// CSR pattern of the expansion, written on the device (the host copy for
/// the sweep planner is filled by host threads meanwhile).
__global__ void bsr_to_csr_pattern_kernel(int64_t nb, int bs, const int64_t* __restrict__ brp,
                                          const int32_t* __restrict__ bcols,
                                          int64_t* __restrict__ row_ptr, int32_t* __restrict__ cols) {
  const int64_t bs2 = int64_t(bs) * bs;
  // one warp per block row: lanes over the row's entries
  const int lane = int(threadIdx.x & 31);
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t f = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); f < nb; f += warps) {
    const int64_t q0 = brp[f], len = brp[f + 1] - q0;
    const int64_t rowlen = len * bs;
    for (int r = 0; r < bs; ++r) {
      const int64_t p0 = q0 * bs2 + int64_t(r) * rowlen;
      if (lane == 0) row_ptr[f * bs + r + 1] = p0 + rowlen;
      for (int64_t t = lane; t < rowlen; t += 32) {
        const int64_t j = t / bs;
        cols[p0 + t] = int32_t(int64_t(bcols[q0 + j]) * bs + (t - j * bs));
      }
    }
    if (f == 0 && lane == 0) row_ptr[0] = 0;
  }
}

} // namespace

void bsr_set_pattern(Context& c, Csr& m, int64_t nb, int bs, const int64_t* brp,
                     const int32_t* bcols, int64_t ncb, int64_t diag_off) {
  if (bs < 1 || bs > 160) throw Error(PSCU_EINVAL, "block matrix: block size must be in [1, 160]");
  if (ncb < 0) ncb = nb;
  if (ncb < nb || diag_off < 0 || diag_off + nb > ncb)
    throw Error(PSCU_EINVAL, "block matrix: inconsistent column count / diagonal offset");
  m.bs = bs;
  m.nb = nb;
  m.ncb = ncb;
  m.diag_off = diag_off;
  m.n = nb * bs;
  m.h_brow_ptr.assign(brp, brp + nb + 1);
  m.nblk = m.h_brow_ptr[nb];
  m.h_bcols.assign(bcols, bcols + m.nblk);
  m.nnz = m.nblk * int64_t(bs) * bs;
  std::vector<int32_t> of(size_t(m.nblk));
  for (int64_t f = 0; f < nb; ++f) {
    if (m.h_brow_ptr[f + 1] < m.h_brow_ptr[f]) throw Error(PSCU_EINVAL, "block matrix: bad row pointer");
    for (int64_t q = m.h_brow_ptr[f]; q < m.h_brow_ptr[f + 1]; ++q) {
      of[q] = int32_t(f);
      if (m.h_bcols[q] < 0 || m.h_bcols[q] >= ncb ||
          (q > m.h_brow_ptr[f] && m.h_bcols[q] <= m.h_bcols[q - 1]))
        throw Error(PSCU_EINVAL, "block matrix: block columns must be ascending and in range");
    }
  }
  m.brow_ptr.upload(m.h_brow_ptr, c.stream);
  m.bcols.upload(m.h_bcols, c.stream);
  m.brow_of.upload(of, c.stream);
  m.row_ptr.alloc(0);
  m.cols.alloc(0);
  m.h_row_ptr.clear();
  m.h_cols.clear();
  m.dgm = 0;
}

namespace {
void set_pattern(Context& c, Csr& m, int64_t nb, int bs, const int64_t* brp, const int32_t* bcols,
                 int64_t ncb = -1, int64_t diag_off = 0) {
  if (bs > 64) throw Error(PSCU_EINVAL, "block matrix: block size must be in [1, 64]");
  bsr_set_pattern(c, m, nb, bs, brp, bcols, ncb, diag_off);
}
} // namespace

void alloc_bsr(Context& c, Csr& m, int64_t nb, int bs, const int64_t* brp, const int32_t* bcols,
               int64_t ncb, int64_t diag_off) {
  set_pattern(c, m, nb, bs, brp, bcols, ncb, diag_off);
  m.vals.alloc(size_t(std::max<int64_t>(1, m.nnz)));
  PSCU_CUDA(cudaMemsetAsync(m.vals.p, 0, sizeof(double) * size_t(m.nnz), c.stream));
}

void upload_bsr(Context& c, Csr& m, int64_t nb, int bs, const int64_t* brp, const int32_t* bcols,
                const double* vals, int mem, int64_t ncb, int64_t diag_off) {
  if (mem == PSCU_HOST) {
    set_pattern(c, m, nb, bs, brp, bcols, ncb, diag_off);
  } else {
    std::vector<int64_t> hrp(nb + 1);
    PSCU_CUDA(cudaMemcpy(hrp.data(), brp, sizeof(int64_t) * (nb + 1), cudaMemcpyDeviceToHost));
    std::vector<int32_t> hc(hrp[nb]);
    PSCU_CUDA(cudaMemcpy(hc.data(), bcols, sizeof(int32_t) * hc.size(), cudaMemcpyDeviceToHost));
    set_pattern(c, m, nb, bs, hrp.data(), hc.data(), ncb, diag_off);
  }
  m.vals.alloc(size_t(std::max<int64_t>(1, m.nnz)));
  if (m.nnz)
    PSCU_CUDA(cudaMemcpyAsync(m.vals.p, vals, sizeof(double) * size_t(m.nnz),
                              mem == PSCU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                              c.stream));
}

void bsr_to_csr(Context& c, const Csr& b, Csr& out) {
  if (b.dgm) return dgb_to_csr(c, b, out);
  const int bs = b.bs;
  out = Csr{};
  out.n = b.n;
  out.nnz = b.nnz;
  out.h_row_ptr.assign(size_t(b.n) + 1, 0);
  out.h_cols.resize(size_t(b.nnz));
  // device pattern (no 4-bytes-per-entry upload), host pattern by threads
  out.row_ptr.alloc(size_t(b.n) + 1);
  out.cols.alloc(size_t(std::max<int64_t>(1, b.nnz)));
  if (b.nb) {
    bsr_to_csr_pattern_kernel<<<unsigned(std::min<int64_t>((b.nb + 7) / 8, 148 * 16)), 256, 0,
                                c.stream>>>(b.nb, bs, b.brow_ptr.p, b.bcols.p, out.row_ptr.p,
                                            out.cols.p);
    PSCU_LAUNCHED(&c);
  } else {
    PSCU_CUDA(cudaMemsetAsync(out.row_ptr.p, 0, sizeof(int64_t), c.stream));
  }
  auto fill = [&](int64_t f0, int64_t f1) {
    for (int64_t f = f0; f < f1; ++f) {
      const int64_t q0 = b.h_brow_ptr[f], len = b.h_brow_ptr[f + 1] - q0;
      for (int r = 0; r < bs; ++r) {
        const int64_t row = f * bs + r;
        const int64_t p0 = q0 * bs * bs + int64_t(r) * len * bs;
        out.h_row_ptr[row + 1] = p0 + len * bs;
        for (int64_t j = 0; j < len; ++j)
          for (int cc = 0; cc < bs; ++cc)
            out.h_cols[size_t(p0 + j * bs + cc)] = int32_t(int64_t(b.h_bcols[q0 + j]) * bs + cc);
      }
    }
  };
  {
    const int nth = int(std::max<int64_t>(
        1, std::min<int64_t>({int64_t(8), int64_t(std::thread::hardware_concurrency()), b.nnz >> 20})));
    std::vector<std::thread> pool;
    for (int t = 1; t < nth; ++t) pool.emplace_back(fill, b.nb * t / nth, b.nb * (t + 1) / nth);
    fill(0, b.nb / nth);
    for (auto& th : pool) th.join();
  }
  out.vals.alloc(size_t(std::max<int64_t>(1, out.nnz)));
  if (out.nnz) {
    bsr_to_csr_kernel<<<grid_for(out.nnz, 256), 256, 0, c.stream>>>(out.nnz, bs, b.brow_ptr.p,
                                                                    b.brow_of.p, b.vals.p,
                                                                    out.vals.p);
    PSCU_LAUNCHED(&c);
  }
}

void inherit_bsr(Context& c, const Csr& fine, const std::vector<int32_t>& m, Csr& out) {
  const int bc = int(m.size());
  out = Csr{};
  set_pattern(c, out, fine.nb, bc, fine.h_brow_ptr.data(), fine.h_bcols.data(), fine.ncb,
              fine.diag_off);
  out.vals.alloc(size_t(std::max<int64_t>(1, out.nnz)));
  DevBuf<int32_t> dm;
  dm.upload(m, c.stream);
  if (out.nnz) {
    inherit_bsr_kernel<<<grid_for(out.nnz, 256), 256, 0, c.stream>>>(out.nnz, fine.bs, bc, dm.p,
                                                                     fine.vals.p, out.vals.p);
    PSCU_LAUNCHED(&c);
  }
  PSCU_CUDA(cudaStreamSynchronize(c.stream));  // dm freed at scope end
}

void spmv_bsr(Context& c, const Csr& a, const double* x, double* y) {
  if (a.dgm) return spmv_dgb(c, a, x, y);
  if (a.n == 0) return;
  Context::Scope prof(&c, PROF_SPMV, 8.0 * double(a.nnz) + 16.0 * double(a.n));
  const unsigned g = grid_for(a.n, 256);
  switch (a.bs) {
    case 24: spmv_bsr_kernel<24><<<g, 256, 0, c.stream>>>(a.n, 24, a.brow_ptr.p, a.bcols.p, a.vals.p, x, y); break;
    case 12: spmv_bsr_kernel<12><<<g, 256, 0, c.stream>>>(a.n, 12, a.brow_ptr.p, a.bcols.p, a.vals.p, x, y); break;
    case 4: spmv_bsr_kernel<4><<<g, 256, 0, c.stream>>>(a.n, 4, a.brow_ptr.p, a.bcols.p, a.vals.p, x, y); break;
    default: spmv_bsr_kernel<0><<<g, 256, 0, c.stream>>>(a.n, a.bs, a.brow_ptr.p, a.bcols.p, a.vals.p, x, y);
  }
  PSCU_LAUNCHED(&c);
}

void residual_restrict_bsr(Context& c, const Csr& a, const double* d, const double* w,
                           const int64_t* map, int64_t nc, double* rc) {
  if (a.dgm) return residual_restrict_dgb(c, a, d, w, nc, rc);
  if (nc == 0) return;
  const unsigned g = grid_for(nc, 256);
  switch (a.bs) {
    case 24: resid_restrict_bsr_kernel<24><<<g, 256, 0, c.stream>>>(nc, 24, map, a.brow_ptr.p, a.bcols.p, a.vals.p, d, w, rc); break;
    case 12: resid_restrict_bsr_kernel<12><<<g, 256, 0, c.stream>>>(nc, 12, map, a.brow_ptr.p, a.bcols.p, a.vals.p, d, w, rc); break;
    case 4: resid_restrict_bsr_kernel<4><<<g, 256, 0, c.stream>>>(nc, 4, map, a.brow_ptr.p, a.bcols.p, a.vals.p, d, w, rc); break;
    default: resid_restrict_bsr_kernel<0><<<g, 256, 0, c.stream>>>(nc, a.bs, map, a.brow_ptr.p, a.bcols.p, a.vals.p, d, w, rc);
  }
  PSCU_LAUNCHED(&c);
}

} // namespace pscu
