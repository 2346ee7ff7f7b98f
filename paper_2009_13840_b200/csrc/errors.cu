// error_norms (errors.hpp:32-117) on the device for the HHO schemes.
//
// Inputs per element: the recovered full local vector (pscu_recover_batch)
// and a point table from the host producer (psh_error_tables: the velocity
// reconstruction P, and per point of the degree-2(k+2)+3 rule the weight,
// the degree-(k+1) basis values and gradients, and the closed-form field; the
// transcendental field values come from the host's libm so the terms are
// bit-identical to the reference's).
//
// error_terms_kernel (one CTA per element) forms the reconstruction
// coefficients gcoef = P * comp (GEMM, k ascending from 0.0), the velocity
// and pressure coefficients, and every point's four error terms
// ((w * d) * d, one rounding per op, dots in the include/eigen_subset
// reproducible order). The reference sums each of the four integrals in one
// sequential chain over (element, point, component), so chain_sum_kernel
// adds the stored terms in exactly that order into running accumulators that
// persist across batches; the caller takes the square roots at the end.
// Bytes per element: the table (8 * per_elem) + the local vector + 8 terms
// per point written and read once — HBM-bound on the table stream.
#include "internal.cuh"

namespace pscu {

namespace {

struct ErrDims {
  int nrec, ns, nq, qstride, per, ne, nf, np, nloc, nfc, hybrid;
};

/// include/eigen_subset repro_dot for n <= 64: T lanes (1, 2 or 4), lane t
/// adds x[i]*y[i] for i = t mod T ascending, lanes combined pairwise.
__device__ __forceinline__ double rdot(const double* x, const double* y, int n) {
  const int T = n <= 16 ? 1 : (n <= 32 ? 2 : 4);
  double part[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i = 0; i < n; ++i) part[i % T] = dadd(part[i % T], dmul(x[i], y[i]));
  if (T == 4) {
    part[0] = dadd(part[0], part[1]);
    part[1] = dadd(part[2], part[3]);
  }
  return T == 1 ? part[0] : dadd(part[0], part[1]);
}

constexpr int kErrThreads = 128;

__global__ void __launch_bounds__(kErrThreads)
    error_terms_kernel(ErrDims d, int nelem, const double* __restrict__ tables,
                       const double* __restrict__ locals, double* __restrict__ tu,
                       double* __restrict__ tg, double* __restrict__ tp,
                       double* __restrict__ td) {
  extern __shared__ double sm[];
  double* comp = sm;                   // ns x 2
  double* gco = comp + 2 * d.ns;       // nrec x 2
  double* uco = gco + 2 * d.nrec;      // nrec x 2
  double* pco = uco + 2 * d.nrec;      // nrec
  for (int e = blockIdx.x; e < nelem; e += gridDim.x) {
    const double* x = locals + size_t(e) * d.nloc;
    const double* P = tables + size_t(e) * d.per;
    for (int t = threadIdx.x; t < 2 * d.ns; t += blockDim.x) {
      const int s = t % d.ns, c = t / d.ns;
      double v;
      if (s < d.ne) {
        v = x[c * d.ne + s];
      } else {
        const int lf = (s - d.ne) / d.nf, m = (s - d.ne) % d.nf;
        v = x[2 * d.ne + lf * 2 * d.nf + c * d.nf + m];
      }
      comp[t] = v;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * d.nrec; t += blockDim.x) {
      const int i = t % d.nrec, c = t / d.nrec;
      double s = 0.0;
      for (int k = 0; k < d.ns; ++k) s = dadd(s, dmul(P[i + size_t(k) * d.nrec], comp[c * d.ns + k]));
      gco[t] = s;
      uco[t] = d.hybrid ? (i < d.ne ? comp[c * d.ns + i] : 0.0) : s;
    }
    const int poff = 2 * (d.ne + d.nfc * d.nf);
    for (int i = threadIdx.x; i < d.nrec; i += blockDim.x) pco[i] = i < d.np ? x[poff + i] : 0.0;
    __syncthreads();
    const double* rows = P + size_t(d.nrec) * d.ns;
    for (int q = threadIdx.x; q < d.nq; q += blockDim.x) {
      const double* r = rows + size_t(q) * d.qstride;
      const double w = r[0];
      const double* v = r + 1;
      const double* ex = r + 1 + 3 * d.nrec;
      const size_t pt = size_t(e) * d.nq + q;
      double div = 0.0;
      for (int c = 0; c < 2; ++c) {
        const double du = dsub(rdot(v, uco + c * d.nrec, d.nrec), ex[c]);
        tu[pt * 2 + c] = dmul(dmul(w, du), du);
        for (int dd = 0; dd < 2; ++dd) {
          const double* g = r + 1 + (1 + dd) * d.nrec;
          const double dg = dsub(rdot(g, gco + c * d.nrec, d.nrec), ex[2 + 2 * c + dd]);
          tg[pt * 4 + 2 * c + dd] = dmul(dmul(w, dg), dg);
        }
        div = dadd(div, rdot(r + 1 + (1 + c) * d.nrec, uco + c * d.nrec, d.nrec));
      }
      const double dp = dsub(rdot(v, pco, d.nrec), ex[6]);
      tp[pt] = dmul(dmul(w, dp), dp);
      td[pt] = dmul(dmul(w, div), div);
    }
    __syncthreads();
  }
}

/// The reference's four accumulation chains (err.u += ..., in element,
/// point, component order): one thread per chain, running sums in acc.
__global__ void chain_sum_kernel(const double* __restrict__ tu, const double* __restrict__ tg,
                                 const double* __restrict__ tp, const double* __restrict__ td,
                                 int64_t npts, double* acc) {
  if (threadIdx.x != 0) return;
  const int c = blockIdx.x;
  const double* t = c == 0 ? tu : (c == 1 ? tg : (c == 2 ? tp : td));
  const int64_t n = npts * (c == 0 ? 2 : (c == 1 ? 4 : 1));
  double s = acc[c];
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcs(t + i + j);
#pragma unroll
    for (int j = 0; j < 8; ++j) s = dadd(s, v[j]);
  }
  for (; i < n; ++i) s = dadd(s, t[i]);
  acc[c] = s;
}

} // namespace

/// dims: {nrec, ns, nq, qstride, per_elem, ne, nf, np, nloc, nfc, hybrid}
/// (psh_error_tables); tables, locals and acc on the device.
void error_accumulate(Context& c, const int32_t* dims, int nelem, const double* tables,
                      const double* locals, double* acc) {
  ErrDims d{dims[0], dims[1], dims[2], dims[3], dims[4], dims[5],
            dims[6], dims[7], dims[8], dims[9], dims[10]};
  if (d.nrec <= 0 || d.nrec > 64 || d.ns <= 0 || d.nq <= 0 || d.qstride != 3 * d.nrec + 8 ||
      d.per != d.nrec * d.ns + d.nq * d.qstride || d.ne > d.nrec || d.np > d.nrec ||
      d.nloc < 2 * (d.ne + d.nfc * d.nf) + d.np)
    throw Error(PSCU_EINVAL, "error_norms: inconsistent table dimensions");
  if (nelem <= 0) return;
  const int64_t npts = int64_t(nelem) * d.nq;
  DevBuf<double> terms(size_t(npts) * 8);
  double* tu = terms.p;
  double* tg = tu + 2 * npts;
  double* tp = tg + 4 * npts;
  double* td = tp + npts;
  const size_t smem = sizeof(double) * (2 * d.ns + 5 * d.nrec);
  const int grid = int(std::min<int64_t>(nelem, 148 * 16));
  error_terms_kernel<<<grid, kErrThreads, smem, c.stream>>>(d, nelem, tables, locals, tu, tg, tp,
                                                            td);
  PSCU_LAUNCHED(&c);
  chain_sum_kernel<<<4, 32, 0, c.stream>>>(tu, tg, tp, td, npts, acc);
  PSCU_LAUNCHED(&c);
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
}

} // namespace pscu
