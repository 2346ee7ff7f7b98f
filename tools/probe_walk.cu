// Micro-benchmark of the walker's per-sub-level critical path on one CTA:
// FP64 dependent-chain latency, named-barrier cost, and the products ->
// barrier -> fold -> barrier loop on shared-memory data (no TMA, no
// producers), to separate the compute/sync floor from staging effects.
// Usage: probe_walk [threads] [entries_per_row]
#include <cstdio>
#include <cstdlib>

__global__ void chain_lat(int n, double a, double b, double* out, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) y = __dmul_rn(y, b);
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = __ddiv_rn(z, b);
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    out[0] = x + y + z;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
}

template <int kThreads>
__global__ void bar_cost(int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
}

/// products (3 entries/thread, ring lookups) + bar + fold (epr entries per
/// row, one row per thread) + bar, `iters` times on the same smem data.
template <int kThreads, bool kJds>
__global__ void phase_loop(int iters, int epr, long long* cyc, double* out) {
  constexpr int kNz = 2048;
  __shared__ double val[kNz], ring[2048];
  __shared__ int src[kNz];
  for (int q = threadIdx.x; q < kNz; q += kThreads) {
    val[q] = 1.0 + q * 1e-9;
    src[q] = (q * 37) & 2047;
  }
  for (int q = threadIdx.x; q < 2048; q += kThreads) ring[q] = 1.0;
  __syncthreads();
  const int nq = kThreads * epr < kNz ? kThreads * epr : kNz;
  long long t0 = clock64();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    constexpr int kPer = (kNz + kThreads - 1) / kThreads;
    int sv[kPer];
    double pv[kPer], yv[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int q = threadIdx.x + u * kThreads;
      sv[u] = q < nq ? src[q] : -1;
      pv[u] = q < nq ? val[q] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) yv[u] = ring[sv[u] & 2047];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int q = threadIdx.x + u * kThreads;
      if (sv[u] >= 0) val[q] = __dmul_rn(pv[u], yv[u]);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
    double a = 1.0;
    const int qa = threadIdx.x * epr;
    for (int q = qa; q < qa + epr; q += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        // row-contiguous (thread stride epr) or diagonal-major (unit stride)
        const int idx = kJds ? (q - qa + u) * kThreads + threadIdx.x : q + u;
        v[u] = q + u < qa + epr ? val[idx & (kNz - 1)] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q + u < qa + epr) a = __dsub_rn(a, v[u]);
    }
    ring[(it * kThreads + threadIdx.x) & 2047] = a;
    acc += a;
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[4] = t1 - t0;
    out[1] = acc;
  }
}

int main(int argc, char** argv) {
  const int epr = argc > 1 ? atoi(argv[1]) : 4;
  long long* cyc;
  double* out;
  cudaMallocManaged(&cyc, sizeof(long long) * 8);
  cudaMallocManaged(&out, sizeof(double) * 8);
  chain_lat<<<1, 32>>>(1000, 1.0, 1.0000001, out, cyc);
  cudaDeviceSynchronize();
  printf("dependent chain (cycles/op): DADD %.1f  DMUL %.1f  DDIV %.1f\n", cyc[0] / 1000.0,
         cyc[1] / 1000.0, cyc[2] / 1000.0);
  bar_cost<512><<<1, 512>>>(1000, cyc);
  cudaDeviceSynchronize();
  printf("bar.sync 512 threads: %.1f cycles\n", cyc[3] / 1000.0);
  bar_cost<768><<<1, 768>>>(1000, cyc);
  cudaDeviceSynchronize();
  printf("bar.sync 768 threads: %.1f cycles\n", cyc[3] / 1000.0);
  phase_loop<512, false><<<1, 512>>>(1000, epr, cyc, out);
  cudaDeviceSynchronize();
  printf("products+bar+fold(%d)+bar, 512 threads, row-contiguous: %.1f cycles/iter\n", epr, cyc[4] / 1000.0);
  phase_loop<512, true><<<1, 512>>>(1000, epr, cyc, out);
  cudaDeviceSynchronize();
  printf("products+bar+fold(%d)+bar, 512 threads, diagonal-major: %.1f cycles/iter\n", epr, cyc[4] / 1000.0);
  phase_loop<768, false><<<1, 768>>>(1000, epr, cyc, out);
  cudaDeviceSynchronize();
  printf("products+bar+fold(%d)+bar, 768 threads, row-contiguous: %.1f cycles/iter\n", epr, cyc[4] / 1000.0);
  phase_loop<768, true><<<1, 768>>>(1000, epr, cyc, out);
  cudaDeviceSynchronize();
  printf("products+bar+fold(%d)+bar, 768 threads, diagonal-major: %.1f cycles/iter\n", epr, cyc[4] / 1000.0);
  phase_loop<128, true><<<1, 128>>>(1000, epr, cyc, out);
  cudaDeviceSynchronize();
  printf("products+bar+fold(%d)+bar, 128 threads, diagonal-major: %.1f cycles/iter\n", epr, cyc[4] / 1000.0);
  return 0;
}
