// Krylov building blocks: reproducible reductions fused with the modified
// Gram-Schmidt updates of ArnoldiWorkspace::step (gmres.hpp:59-82), and the
// x0 + sum_i y_i z_i update of ArnoldiWorkspace::solution (gmres.hpp:84-91).
//
// Reduction shape (identical to include/eigen_subset/Eigen/Dense): T =
// repro_lanes(n) accumulator lanes, lane t sums elements t, t+T, t+2T, ...
// in order; lanes are combined by a perfect binary tree over adjacent pairs.
// Lane t is thread t of the grid; a CTA of B lanes reduces its aligned
// subtree with warp shuffles (offsets 1,2,4,8,16 = adjacent pairs) and
// shared memory, and the last CTA to finish reduces the per-CTA results,
// so each MGS pass is one kernel with no host round trip.
#include "internal.cuh"

namespace pscu {

namespace {

constexpr int kRedThreads = 256;
constexpr int kMaxRedBlocks = (1 << 18) / kRedThreads;

/// Adjacent-pair tree over the CTA's lanes; result valid in thread 0.
__device__ double block_tree(double v, int nlanes) {
  __shared__ double warp_sum[kRedThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wl = nlanes < 32 ? nlanes : 32;
  for (int off = 1; off < wl; off <<= 1) {
    const double o = __shfl_down_sync(0xffffffffu, v, off);
    if ((lane & (2 * off - 1)) == 0) v = dadd(v, o);
  }
  if (nlanes <= 32) return v;
  if (lane == 0) warp_sum[wid] = v;
  __syncthreads();
  const int nw = nlanes >> 5;
  if (wid == 0) {
    v = lane < nw ? warp_sum[lane] : 0.0;
    for (int off = 1; off < nw; off <<= 1) {
      const double o = __shfl_down_sync(0xffffffffu, v, off);
      if ((lane & (2 * off - 1)) == 0) v = dadd(v, o);
    }
  }
  return v;
}

/// Last-CTA combine of the per-CTA subtree results (adjacent-pair tree over
/// gridDim.x values, a power of two). Writes f(result) to *out.
__device__ void grid_finish(double v, double* partials, unsigned int* counter, double* out,
                            bool take_sqrt) {
  __shared__ bool last;
  if (gridDim.x == 1) {
    if (threadIdx.x == 0) *out = take_sqrt ? __dsqrt_rn(v) : v;
    return;
  }
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;
    __threadfence();
    const unsigned int done = atomicAdd(counter, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __shared__ double buf[kMaxRedBlocks];
  const int G = gridDim.x;
  for (int i = threadIdx.x; i < G; i += blockDim.x) buf[i] = __ldcg(partials + i);
  __syncthreads();
  for (int width = G; width > 1; width >>= 1) {
    const int half = width >> 1;
    double t[kMaxRedBlocks / kRedThreads > 0 ? kMaxRedBlocks / kRedThreads : 1];
    int cnt = 0;
    for (int k = threadIdx.x; k < half; k += blockDim.x) t[cnt++] = dadd(buf[2 * k], buf[2 * k + 1]);
    __syncthreads();
    cnt = 0;
    for (int k = threadIdx.x; k < half; k += blockDim.x) buf[k] = t[cnt++];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out = take_sqrt ? __dsqrt_rn(buf[0]) : buf[0];
    *counter = 0u;
  }
}

/// One MGS pass. mode 0: acc = x.y. mode 1: w -= h*vp; acc = w.vi.
/// mode 2: w -= h*vp; acc = w.w and *out = sqrt(acc).
template <int kMode>
__global__ void __launch_bounds__(kRedThreads)
    mgs_pass(int64_t n, int64_t T, double* w, const double* __restrict__ vp,
             const double* __restrict__ hprev, const double* __restrict__ vi, double* partials,
             unsigned int* counter, double* out) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  double h = 0.0;
  if (kMode != 0) h = *hprev;
  double acc = 0.0;
  for (int64_t e = t < T ? t : n; e < n; e += T) {
    double we = w[e];
    if (kMode != 0) {
      we = dsub(we, dmul(h, vp[e]));
      w[e] = we;
    }
    const double o = kMode == 2 ? we : vi[e];
    acc = dadd(acc, dmul(we, o));
  }
  const int nl = int(T < kRedThreads ? T : kRedThreads);
  acc = block_tree(acc, nl);
  grid_finish(acc, partials, counter, out, kMode == 2);
}

/// v = (h > 0) ? w / h : 0 (ArnoldiWorkspace::step, gmres.hpp:66-67).
__global__ void scale_next(int64_t n, const double* __restrict__ w, const double* __restrict__ hp,
                           double* __restrict__ v) {
  const double h = *hp;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    v[e] = h > 0.0 ? __ddiv_rn(w[e], h) : 0.0;
}

__global__ void scale_div(int64_t n, const double* __restrict__ r, double beta,
                          double* __restrict__ v) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    v[e] = __ddiv_rn(r[e], beta);
}

/// x = x0 + sum_{i<m} y_i z_i, i ascending per element.
__global__ void combine(int64_t n, int m, const double* x0, const double* __restrict__ y,
                        const double* __restrict__ z, int64_t ldz, double* x) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    double acc = x0 ? x0[e] : 0.0;
    for (int i = 0; i < m; ++i) acc = dadd(acc, dmul(y[i], z[int64_t(i) * ldz + e]));
    x[e] = acc;
  }
}

__global__ void sub_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ r) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    r[e] = dsub(a[e], b[e]);
}

unsigned grid_for(int64_t n, int threads = 256) {
  const int64_t g = (n + threads - 1) / threads;
  return unsigned(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

} // namespace

/// Runs one reduction pass; result lands in device scalar `out`.
void mgs_launch(Context& c, int mode, int64_t n, double* w, const double* vp, const double* hprev,
                const double* vi, double* out) {
  const int64_t T = repro_lanes(n);
  const int threads = int(T < kRedThreads ? T : kRedThreads);
  const unsigned blocks = unsigned(T / threads);
  // lanes < 32 still run a full warp so the shuffles are well defined
  const int launch_threads = threads < 32 ? 32 : threads;
  if (mode == 0)
    mgs_pass<0><<<blocks, launch_threads, 0, c.stream>>>(n, T, w, vp, hprev, vi,
                                                          c.red_partials.p, c.red_counter.p, out);
  else if (mode == 1)
    mgs_pass<1><<<blocks, launch_threads, 0, c.stream>>>(n, T, w, vp, hprev, vi,
                                                          c.red_partials.p, c.red_counter.p, out);
  else
    mgs_pass<2><<<blocks, launch_threads, 0, c.stream>>>(n, T, w, vp, hprev, vi,
                                                          c.red_partials.p, c.red_counter.p, out);
  PSCU_LAUNCHED(&c);
}

double dot(Context& c, const double* x, const double* y, int64_t n) {
  mgs_launch(c, 0, n, const_cast<double*>(x), nullptr, nullptr, y, c.scal.p);
  PSCU_CUDA(cudaMemcpyAsync(c.h_pinned, c.scal.p, sizeof(double), cudaMemcpyDeviceToHost,
                            c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  return c.h_pinned[0];
}

void scale_next_launch(Context& c, int64_t n, const double* w, const double* hp, double* v) {
  scale_next<<<grid_for(n), 256, 0, c.stream>>>(n, w, hp, v);
  PSCU_LAUNCHED(&c);
}

void scale_div_launch(Context& c, int64_t n, const double* r, double beta, double* v) {
  scale_div<<<grid_for(n), 256, 0, c.stream>>>(n, r, beta, v);
  PSCU_LAUNCHED(&c);
}

void combine_launch(Context& c, int64_t n, int m, const double* x0, const double* y_dev,
                    const double* z, int64_t ldz, double* x) {
  combine<<<grid_for(n), 256, 0, c.stream>>>(n, m, x0, y_dev, z, ldz, x);
  PSCU_LAUNCHED(&c);
}

void sub_launch(Context& c, int64_t n, const double* a, const double* b, double* r) {
  sub_kernel<<<grid_for(n), 256, 0, c.stream>>>(n, a, b, r);
  PSCU_LAUNCHED(&c);
}

void copy(Context& c, double* dst, const double* src, int64_t n) {
  if (n) PSCU_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
}

void zero(Context& c, double* dst, int64_t n) {
  if (n) PSCU_CUDA(cudaMemsetAsync(dst, 0, sizeof(double) * n, c.stream));
}

} // namespace pscu
