// DG block storage: the operator of the 3D DG scheme (BASELINE.json config 4,
// BR2 as the reference's assemble_dg, assemble.hpp:177-346) kept in its
// structural pattern without index streams.
//
// The DG pattern couples whole element blocks [u_x | u_y | u_z | p] (nm =
// dim P^k modes each) of neighbouring elements, but velocity components are
// not coupled to each other (DofLayout::couples_components() is false for
// uncond, dof_layout.hpp:79-84; assemble.hpp:38-46): only 10 of the 16 nm x nm
// sub-blocks are structural (SURVEY.md §0 finding 8 — a dense 4nm block would
// move 1.6x the structural bytes). Each block therefore stores exactly its
// structural entries as four column-major panels:
//   velocity row panel c (c = 0..2): nm rows x 2nm columns, [u_c | p] modes,
//     at offset c 2nm^2;
//   pressure row panel: nm rows x 4nm columns, [u_x | u_y | u_z | p], at 6nm^2.
// One int32 block column per block; 8 B per structural entry + 16 B per row
// is all an SpMV moves (SURVEY.md §8(d) algorithmic bytes).
//
// Bitwise parity with CsrMatrix::multiply (csr.hpp:68-74): a row's CSR columns
// are block column ascending, then — within a block — its panel columns in
// order (u_c modes precede p modes in the element numbering), so one thread
// per row folds them in exactly that order from 0.0, one rounding per op.
//
// Thread mapping: rows are enumerated in tiles of T element blocks with all
// velocity rows of the tile first and its pressure rows after, T chosen so
// both groups are whole warps (nm T = 0 mod 32): warps never mix the 2nm-long
// velocity rows with the 4nm-long pressure rows.
#include <algorithm>
#include <numeric>

#include "internal.cuh"

namespace pscu {

namespace {

unsigned grid_for(int64_t n, int threads) {
  const int64_t g = (n + threads - 1) / threads;
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(148) * 32)));
}

inline int tile_blocks(int nm) { return 32 / std::gcd(nm, 32); }

/// Output rows of block storage with nmo modes per component, tile-ordered.
/// out(e, c, i) = [d(e, c, i) -] sum_q A(e*NM + c*NM + i, :) x, the fine row
/// having the same element, component and (leading) mode.
template <int NM, bool kRestrict>
__global__ void __launch_bounds__(256) dgb_rows_kernel(int64_t nb, int nmo, int tb,
                                                       const int64_t* __restrict__ brp,
                                                       const int32_t* __restrict__ bcols,
                                                       const double* __restrict__ vals,
                                                       const double* __restrict__ x,
                                                       const double* __restrict__ d,
                                                       double* __restrict__ out) {
  constexpr int64_t kBsz = 10 * NM * NM;
  const int64_t per_tile = int64_t(4) * nmo * tb, vel_slots = int64_t(3) * nmo * tb;
  const int64_t total = ((nb + tb - 1) / tb) * per_tile;
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < total;
       s += int64_t(gridDim.x) * blockDim.x) {
    const int64_t tile = s / per_tile;
    const int64_t u = s - tile * per_tile;
    int64_t e;
    int c, i;
    if (u < vel_slots) {
      e = tile * tb + u / (3 * nmo);
      const int r = int(u % (3 * nmo));
      c = r / nmo;
      i = r - c * nmo;
    } else {
      const int64_t v = u - vel_slots;
      e = tile * tb + v / nmo;
      c = 3;
      i = int(v % nmo);
    }
    if (e >= nb) continue;
    const int64_t q0 = brp[e], q1 = brp[e + 1];
    double acc = 0.0;
    if (c < 3) {
      for (int64_t q = q0; q < q1; ++q) {
        const double* A = vals + q * kBsz + c * 2 * NM * NM + i;
        const double* xg = x + int64_t(__ldg(bcols + q)) * 4 * NM;
        double a[NM], xv[NM];
#pragma unroll
        for (int j = 0; j < NM; ++j) {
          a[j] = __ldcs(A + j * NM);
          xv[j] = __ldg(xg + c * NM + j);
        }
#pragma unroll
        for (int j = 0; j < NM; ++j) acc = dadd(acc, dmul(a[j], xv[j]));
#pragma unroll
        for (int j = 0; j < NM; ++j) {
          a[j] = __ldcs(A + (NM + j) * NM);
          xv[j] = __ldg(xg + 3 * NM + j);
        }
#pragma unroll
        for (int j = 0; j < NM; ++j) acc = dadd(acc, dmul(a[j], xv[j]));
      }
    } else {
      for (int64_t q = q0; q < q1; ++q) {
        const double* A = vals + q * kBsz + 6 * NM * NM + i;
        const double* xg = x + int64_t(__ldg(bcols + q)) * 4 * NM;
#pragma unroll
        for (int part = 0; part < 4; ++part) {
          double a[NM], xv[NM];
#pragma unroll
          for (int j = 0; j < NM; ++j) {
            a[j] = __ldcs(A + (part * NM + j) * NM);
            xv[j] = __ldg(xg + part * NM + j);
          }
#pragma unroll
          for (int j = 0; j < NM; ++j) acc = dadd(acc, dmul(a[j], xv[j]));
        }
      }
    }
    const int64_t orow = e * 4 * nmo + c * nmo + i;
    if (kRestrict) out[orow] = dsub(d[e * 4 * NM + c * NM + i], acc);
    else out[orow] = acc;
  }
}

/// Coarse panels gathered from the fine ones through an in-block table.
__global__ void dgb_gather_kernel(int64_t total, int bszc, int64_t bszf,
                                  const int32_t* __restrict__ tab, const double* __restrict__ fine,
                                  double* __restrict__ out) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = t / bszc;
    const int w = int(t - q * bszc);
    out[t] = fine[q * bszf + tab[w]];
  }
}

/// Panel value -> CSR position: row e 4nm + c nm + i, position within the
/// row (block index in the row) * row length per block + panel column.
__global__ void dgb_to_csr_kernel(int64_t total, int nm, const int64_t* __restrict__ brp,
                                  const int32_t* __restrict__ brow_of,
                                  const int64_t* __restrict__ row_ptr,
                                  const double* __restrict__ vals, double* __restrict__ out) {
  const int64_t bsz = int64_t(10) * nm * nm;
  const int vpan = 2 * nm * nm;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = t / bsz;
    const int w = int(t - q * bsz);
    int c, col, i, rlen;
    if (w < 3 * vpan) {
      c = w / vpan;
      const int r = w - c * vpan;
      col = r / nm;
      i = r - col * nm;
      rlen = 2 * nm;
    } else {
      const int r = w - 3 * vpan;
      c = 3;
      col = r / nm;
      i = r - col * nm;
      rlen = 4 * nm;
    }
    const int64_t e = brow_of[q];
    const int64_t row = e * 4 * nm + c * nm + i;
    out[row_ptr[row] + (q - brp[e]) * rlen + col] = vals[t];
  }
}

template <bool kRestrict>
void launch_rows(Context& c, const Csr& a, int nmo, const double* x, const double* d,
                 double* out) {
  const int tb = tile_blocks(nmo);
  const int64_t slots = ((a.nb + tb - 1) / tb) * int64_t(4) * nmo * tb;
  const unsigned g = grid_for(slots, 256);
  switch (a.dgm) {
#define PSCU_DGB_CASE(NM)                                                                   \
  case NM:                                                                                  \
    dgb_rows_kernel<NM, kRestrict><<<g, 256, 0, c.stream>>>(a.nb, nmo, tb, a.brow_ptr.p,     \
                                                            a.bcols.p, a.vals.p, x, d, out); \
    break;
    PSCU_DGB_CASE(4)
    PSCU_DGB_CASE(10)
    PSCU_DGB_CASE(20)
    PSCU_DGB_CASE(35)
#undef PSCU_DGB_CASE
    default:
      throw Error(PSCU_EINVAL, "DG block storage: modes per component must be 4, 10, 20 or 35");
  }
  PSCU_LAUNCHED(&c);
}

} // namespace

void upload_dgb(Context& c, Csr& m, int64_t nb, int nm, const int64_t* brp, const int32_t* bcols,
                const double* vals, int mem) {
  if (nm != 4 && nm != 10 && nm != 20 && nm != 35)
    throw Error(PSCU_EINVAL, "DG block storage: modes per component must be 4, 10, 20 or 35");
  if (mem == PSCU_HOST) {
    bsr_set_pattern(c, m, nb, 4 * nm, brp, bcols, -1, 0);
  } else {
    std::vector<int64_t> hrp(nb + 1);
    PSCU_CUDA(cudaMemcpy(hrp.data(), brp, sizeof(int64_t) * (nb + 1), cudaMemcpyDeviceToHost));
    std::vector<int32_t> hc(hrp[nb]);
    PSCU_CUDA(cudaMemcpy(hc.data(), bcols, sizeof(int32_t) * hc.size(), cudaMemcpyDeviceToHost));
    bsr_set_pattern(c, m, nb, 4 * nm, hrp.data(), hc.data(), -1, 0);
  }
  m.dgm = nm;
  m.nnz = m.nblk * int64_t(10) * nm * nm;
  m.vals.alloc(size_t(std::max<int64_t>(1, m.nnz)));
  if (m.nnz && vals)
    PSCU_CUDA(cudaMemcpyAsync(m.vals.p, vals, sizeof(double) * size_t(m.nnz),
                              mem == PSCU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                              c.stream));
  else if (m.nnz)
    PSCU_CUDA(cudaMemsetAsync(m.vals.p, 0, sizeof(double) * size_t(m.nnz), c.stream));
}

void spmv_dgb(Context& c, const Csr& a, const double* x, double* y) {
  if (a.n == 0) return;
  Context::Scope prof(&c, PROF_SPMV, 8.0 * double(a.nnz) + 16.0 * double(a.n));
  launch_rows<false>(c, a, a.dgm, x, nullptr, y);
}

void residual_restrict_dgb(Context& c, const Csr& a, const double* d, const double* w, int64_t nc,
                           double* rc) {
  if (nc == 0) return;
  if (a.nb == 0 || nc % (4 * a.nb))
    throw Error(PSCU_EINVAL, "DG restriction: coarse size is not a whole number of element blocks");
  const int nmc = int(nc / (4 * a.nb));
  if (nmc > a.dgm) throw Error(PSCU_EINVAL, "DG restriction: coarse modes exceed the fine ones");
  launch_rows<true>(c, a, nmc, w, d, rc);
}

void inherit_dgb(Context& c, const Csr& fine, int nmc, Csr& out) {
  const int nm = fine.dgm;
  if (nmc < 1 || nmc > nm) throw Error(PSCU_EINVAL, "DG inheritance: coarse modes out of range");
  // coarse (panel, column, row) -> fine offset: coarse modes are the leading
  // fine modes of the same component (plevels.hpp:47-72, hierarchical bases)
  const int bszc = 10 * nmc * nmc;
  std::vector<int32_t> tab(bszc);
  for (int w = 0; w < bszc; ++w) {
    const int vpan = 2 * nmc * nmc;
    if (w < 3 * vpan) {
      const int cc = w / vpan, r = w - cc * vpan, col = r / nmc, i = r - col * nmc;
      const int fcol = col < nmc ? col : nm + (col - nmc);
      tab[w] = cc * 2 * nm * nm + fcol * nm + i;
    } else {
      const int r = w - 3 * vpan, col = r / nmc, i = r - col * nmc;
      const int fcol = (col / nmc) * nm + col % nmc;
      tab[w] = 6 * nm * nm + fcol * nm + i;
    }
  }
  out = Csr{};
  upload_dgb(c, out, fine.nb, nmc, fine.h_brow_ptr.data(), fine.h_bcols.data(), nullptr, PSCU_HOST);
  DevBuf<int32_t> dt;
  dt.upload(tab, c.stream);
  if (out.nnz) {
    dgb_gather_kernel<<<grid_for(out.nnz, 256), 256, 0, c.stream>>>(
        out.nnz, bszc, int64_t(10) * nm * nm, dt.p, fine.vals.p, out.vals.p);
    PSCU_LAUNCHED(&c);
  }
  PSCU_CUDA(cudaStreamSynchronize(c.stream));  // dt freed at scope end
}

void dgb_to_csr(Context& c, const Csr& b, Csr& out) {
  const int nm = b.dgm, eb = 4 * nm;
  out = Csr{};
  out.n = b.n;
  out.nnz = b.nnz;
  out.h_row_ptr.assign(size_t(b.n) + 1, 0);
  out.h_cols.resize(size_t(b.nnz));
  int64_t p = 0;
  for (int64_t e = 0; e < b.nb; ++e) {
    const int64_t q0 = b.h_brow_ptr[e], q1 = b.h_brow_ptr[e + 1];
    for (int r = 0; r < eb; ++r) {
      const int comp = r / nm;
      out.h_row_ptr[e * eb + r] = p;
      for (int64_t q = q0; q < q1; ++q) {
        const int64_t base = int64_t(b.h_bcols[q]) * eb;
        if (comp < 3) {
          for (int j = 0; j < nm; ++j) out.h_cols[p++] = int32_t(base + comp * nm + j);
          for (int j = 0; j < nm; ++j) out.h_cols[p++] = int32_t(base + 3 * nm + j);
        } else {
          for (int j = 0; j < eb; ++j) out.h_cols[p++] = int32_t(base + j);
        }
      }
    }
  }
  out.h_row_ptr[b.n] = p;
  if (p != b.nnz) throw Error(PSCU_EINVAL, "DG block storage: pattern size mismatch");
  out.row_ptr.upload(out.h_row_ptr, c.stream);
  out.cols.upload(out.h_cols, c.stream);
  out.vals.alloc(size_t(std::max<int64_t>(1, out.nnz)));
  if (out.nnz) {
    dgb_to_csr_kernel<<<grid_for(out.nnz, 256), 256, 0, c.stream>>>(
        out.nnz, nm, b.brow_ptr.p, b.brow_of.p, out.row_ptr.p, b.vals.p, out.vals.p);
    PSCU_LAUNCHED(&c);
  }
}

} // namespace pscu
