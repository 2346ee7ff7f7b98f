// Block-Jacobi preconditioner over the entity blocks of a DofLayout: the
// smoother BASELINE.json names ("block-Jacobi smoothing with batched
// face-block inverses"), plugged in where the reference uses ILU(0)
// (plevels.hpp:170-183, the pc of the GMRES smoother). It is a labelled
// alternative: the reference's own smoother is ILU(0)-GMRES, and HHO-dp
// element mean-pressure blocks are singular (SURVEY.md §0 finding 4), which
// the factorisation reports as PSCU_ESINGULAR with the block id.
//
// Blocks follow the layout numbering (dof_layout.hpp:56-85): face f owns
// [f fb, (f+1) fb), element e owns [F + e eb, F + (e+1) eb). Setup: one
// thread per block extracts the dense block from the CSR pattern, factors
// it by partial-pivot LU and inverts it column by column. Apply (the hot
// part, HBM-bound: 8 sum b^2 + 16 n bytes): one thread per row, y_i =
// sum_j inv_ij x_j in column order; inverses are stored column-major per
// block so a warp's loads of one column are contiguous. Every operation is
// individually rounded in the order of oracle/pstokes_oracle.c (po_bj_*),
// so the two agree bit for bit.
#include <cmath>

#include "internal.cuh"
#include "solver.cuh"

namespace pscu {

namespace {

/// kBsr: the operator is in dense-block storage (bsr.cu) with this block
/// size; the diagonal block of block row b is copied directly (rp / cols
/// are then the block row pointer / block columns).
/// kDgm > 0 (runtime dgm): DG block storage (dgb.cu panels), structural
/// zeros of the dense block filled in.
template <bool kBsr>
__global__ void bj_factor_kernel(int64_t nb, int bs, int dgm, int64_t s0, int64_t b0, int64_t diag_off,
                                 const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                 const double* __restrict__ vals, double* __restrict__ inv,
                                 double* __restrict__ work, int* __restrict__ perm_ws,
                                 unsigned long long* __restrict__ bad) {
  // scratch is element-major, block-minor (entry (i, j) of block b at
  // (i bs + j) nb + b): the threads of a warp (consecutive blocks) touch
  // consecutive addresses at every step of their identical loops
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < nb;
       b += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = s0 + b * bs;
#define D(i, j) work[(int64_t(i) * bs + (j)) * nb + b]
#define Y(i) work[nb * bs * bs + int64_t(i) * nb + b]
#define PERM(i) perm_ws[int64_t(i) * nb + b]
    double* out = inv + b * bs * bs;  // column-major
    if (kBsr) {
      int64_t q = rp[b];
      while (q < rp[b + 1] && cols[q] != b + diag_off) ++q;
      if (dgm) {
        const int nm = dgm;
        const double* blk = vals + q * 10 * nm * nm;
        for (int i = 0; i < bs; ++i)
          for (int c = 0; c < bs; ++c) {
            const int ri = i / nm, ci = c / nm;
            double v = 0.0;
            if (q < rp[b + 1] && (ri == 3 || ci == 3 || ri == ci)) {
              if (ri < 3) v = blk[ri * 2 * nm * nm + (ci == 3 ? nm + c % nm : c % nm) * nm + i % nm];
              else v = blk[6 * nm * nm + c * nm + i % nm];
            }
            D(i, c) = v;
          }
      } else {
        const double* blk = vals + q * bs * bs;
        for (int i = 0; i < bs; ++i)
          for (int c = 0; c < bs; ++c) D(i, c) = q < rp[b + 1] ? blk[c * bs + i] : 0.0;
      }
    } else {
      for (int i = 0; i < bs; ++i)
        for (int c = 0; c < bs; ++c) D(i, c) = 0.0;
      for (int i = 0; i < bs; ++i)
        for (int64_t q = rp[s + i]; q < rp[s + i + 1]; ++q) {
          const int64_t c = cols[q];
          if (c >= s && c < s + bs) D(i, c - s) = vals[q];
        }
    }
    double amax = 0.0;
    for (int i = 0; i < bs; ++i)
      for (int j = 0; j < bs; ++j) amax = fmax(amax, fabs(D(i, j)));
    for (int i = 0; i < bs; ++i) PERM(i) = i;
    bool ok = true;
    for (int k = 0; k < bs && ok; ++k) {
      int p = k;
      double m = fabs(D(k, k));
      for (int i = k + 1; i < bs; ++i)
        if (fabs(D(i, k)) > m) {
          m = fabs(D(i, k));
          p = i;
        }
      if (!(m > dmul(1e-14, amax))) {
        ok = false;
        break;
      }
      if (p != k) {
        for (int j = 0; j < bs; ++j) {
          const double t = D(k, j);
          D(k, j) = D(p, j);
          D(p, j) = t;
        }
        const int t = PERM(k);
        PERM(k) = PERM(p);
        PERM(p) = t;
      }
      for (int i = k + 1; i < bs; ++i) {
        const double f = __ddiv_rn(D(i, k), D(k, k));
        D(i, k) = f;
        for (int j = k + 1; j < bs; ++j) D(i, j) = dsub(D(i, j), dmul(f, D(k, j)));
      }
    }
    if (!ok) {
      atomicMin(bad, (unsigned long long)(b0 + b));
      continue;
    }
    for (int c = 0; c < bs; ++c) {
      for (int i = 0; i < bs; ++i) {
        double v = PERM(i) == c ? 1.0 : 0.0;
        for (int j = 0; j < i; ++j) v = dsub(v, dmul(D(i, j), Y(j)));
        Y(i) = v;
      }
      for (int i = bs - 1; i >= 0; --i) {
        double v = Y(i);
        for (int j = i + 1; j < bs; ++j) v = dsub(v, dmul(D(i, j), Y(j)));
        Y(i) = __ddiv_rn(v, D(i, i));
      }
      for (int i = 0; i < bs; ++i) out[c * bs + i] = Y(i);
    }
#undef D
#undef Y
#undef PERM
  }
}

/// y_i = sum_j inv_ij x_j (j ascending) for the rows of one uniform batch.
template <int kBs>
__global__ void bj_apply_kernel(int64_t rows, int bs_rt, int64_t s0,
                                const double* __restrict__ inv, const double* __restrict__ x,
                                double* __restrict__ y) {
  const int bs = kBs > 0 ? kBs : bs_rt;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = r / bs;
    const int i = int(r - b * bs);
    const double* m = inv + b * bs * bs + i;
    const double* xb = x + s0 + b * bs;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < (kBs > 0 ? kBs : 64); ++j) {
      if (kBs == 0 && j >= bs) break;
      acc = dadd(acc, dmul(__ldg(m + j * bs), __ldg(xb + j)));
    }
    y[s0 + r] = acc;
  }
}

unsigned grid_rows(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return unsigned(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

void apply_batch(Context& c, int64_t rows, int bs, int64_t s0, const double* inv, const double* x,
                 double* y) {
  if (!rows || !bs) return;
  const unsigned g = grid_rows(rows);
  switch (bs) {
    case 2: bj_apply_kernel<2><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 3: bj_apply_kernel<3><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 4: bj_apply_kernel<4><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 6: bj_apply_kernel<6><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 8: bj_apply_kernel<8><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 9: bj_apply_kernel<9><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 10: bj_apply_kernel<10><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 12: bj_apply_kernel<12><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 24: bj_apply_kernel<24><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 16: bj_apply_kernel<16><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 40: bj_apply_kernel<40><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    case 80: bj_apply_kernel<80><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y); break;
    default:
      if (bs > 64) throw Error(PSCU_EINVAL, "block-Jacobi: blocks larger than 64 unsupported");
      bj_apply_kernel<0><<<g, 256, 0, c.stream>>>(rows, bs, s0, inv, x, y);
  }
  PSCU_LAUNCHED(&c);
}

} // namespace

void bj_factor(Context& c, const Csr& a, const pscu_layout& l, BlockJacobi& bj) {
  bj.layout = l;
  bj.fb = ncomp(l) * l.face_vel + l.face_press;
  bj.eb = ncomp(l) * l.elem_vel + l.elem_press;
  if (a.dgm) {
    if (bj.fb != 0 || bj.eb != a.bs)
      throw Error(PSCU_EINVAL, "block-Jacobi: DG block storage must match the layout's element blocks");
  } else if (a.bs && (bj.eb != 0 || bj.fb != a.bs)) {
    throw Error(PSCU_EINVAL, "block-Jacobi: block storage must match the layout's face blocks");
  }
  bj.eoff = int64_t(l.n_faces) * bj.fb;
  bj.n = a.n;
  if (layout_dim(l) != a.n) throw Error(PSCU_EINVAL, "block-Jacobi: layout/matrix size mismatch");
  const int64_t nf = l.n_faces, ne = l.n_elements;
  const size_t fsz = size_t(nf) * bj.fb * bj.fb, esz = size_t(ne) * bj.eb * bj.eb;
  bj.inv.alloc(fsz + esz + 1);
  DevBuf<unsigned long long> bad(1);
  const unsigned long long none = ~0ull;
  PSCU_CUDA(cudaMemcpyAsync(bad.p, &none, sizeof(none), cudaMemcpyHostToDevice, c.stream));
  const int64_t nbatch[2] = {nf, ne};
  const int bsz[2] = {bj.fb, bj.eb};
  const int64_t s0[2] = {0, bj.eoff};
  const size_t off[2] = {0, fsz};
  for (int t = 0; t < 2; ++t) {
    const int64_t nb = nbatch[t];
    const int bs = bsz[t];
    if (!nb || !bs) continue;
    DevBuf<double> work(size_t(nb) * bs * (bs + 1));
    DevBuf<int> perm(size_t(nb) * bs);
    if (a.bs)
      bj_factor_kernel<true><<<grid_rows(nb), 256, 0, c.stream>>>(
          nb, bs, a.dgm, s0[t], t ? nf : 0, a.diag_off, a.brow_ptr.p, a.bcols.p, a.vals.p, bj.inv.p + off[t], work.p,
          perm.p, bad.p);
    else
      bj_factor_kernel<false><<<grid_rows(nb), 256, 0, c.stream>>>(
          nb, bs, 0, s0[t], t ? nf : 0, int64_t(0), a.row_ptr.p, a.cols.p, a.vals.p, bj.inv.p + off[t], work.p,
          perm.p, bad.p);
    PSCU_LAUNCHED(&c);
    PSCU_CUDA(cudaStreamSynchronize(c.stream));  // scratch freed at scope end
  }
  unsigned long long hb = 0;
  PSCU_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  if (hb != none)
    throw Error(PSCU_ESINGULAR, "block-Jacobi: singular diagonal block " + std::to_string(hb) +
                                    (int64_t(hb) < nf ? " (face)" : " (element)"));
}

void bj_apply(Context& c, const BlockJacobi& bj, const double* x, double* y) {
  const pscu_layout& l = bj.layout;
  const double bytes = 8.0 * (double(l.n_faces) * bj.fb * bj.fb + double(l.n_elements) * bj.eb * bj.eb) +
                       16.0 * double(bj.n);
  Context::Scope prof(&c, PROF_BJ, bytes);
  apply_batch(c, int64_t(l.n_faces) * bj.fb, bj.fb, 0, bj.inv.p, x, y);
  apply_batch(c, int64_t(l.n_elements) * bj.eb, bj.eb, bj.eoff,
              bj.inv.p + size_t(l.n_faces) * bj.fb * bj.fb, x, y);
}

} // namespace pscu
