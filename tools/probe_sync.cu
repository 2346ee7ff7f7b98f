// Micro-benchmark: latency of one grid-wide ordered all-reduce of a double
// (the per-pass step of the fused MGS kernel) under several exchange schemes.
//   mode 0: root CTA gathers tagged slots (release/acquire), tree, publishes
//   mode 1: every CTA gathers all tagged slots (release/acquire), tree
//   mode 2: every CTA gathers all slots as 16-byte {value, tag} pairs
//           written and polled with relaxed gpu-scope vector accesses
// Usage: probe_sync [G] [passes] [stream_doubles_per_cta]
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

constexpr int kThreads = 256;

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_pair(ulonglong2* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ ulonglong2 ld_pair(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}

__device__ double block_tree(double v, int nact) {
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = threadIdx.x < unsigned(nact) ? v : 0.0;
  __syncthreads();
  for (int s = 1; s < nact; s <<= 1) {
    if ((threadIdx.x & (2 * s - 1)) == 0 && threadIdx.x + s < unsigned(nact))
      sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

template <int kMode>
__global__ void __launch_bounds__(kThreads, 2)
    probe(int passes, double* slot_v, unsigned long long* slot_tag, ulonglong2* pairs,
          const double* stream, int per_cta, double* out) {
  __shared__ double hsh;
  const int G = gridDim.x, tid = threadIdx.x;
  double h = 1.0, chk = 0.0;
  for (int i = 0; i < passes; ++i) {
    double acc = h * (tid + 1) * 1e-6;
    for (int e = tid; e < per_cta; e += kThreads)
      acc += __ldcg(stream + (size_t(i & 7) * G + blockIdx.x) * per_cta + e);
    const double cta = block_tree(acc, kThreads);
    const unsigned long long want = unsigned(i) + 1ull;
    const int par = i & 1;
    if (kMode == 0) {
      if (tid == 0) {
        slot_v[par * G + blockIdx.x] = cta;
        st_release(slot_tag + par * G + blockIdx.x, want);
      }
      if (blockIdx.x == 0) {
        double v = 0.0;
        if (tid < G) {
          while (ld_acquire(slot_tag + par * G + tid) != want) {
          }
          v = __ldcg(slot_v + par * G + tid);
        }
        v = block_tree(v, G);
        if (tid == 0) {
          hsh = v;
          slot_v[2 * G + par] = v;
          st_release(slot_tag + 2 * G + par, want);
        }
      } else if (tid == 0) {
        while (ld_acquire(slot_tag + 2 * G + par) != want) {
        }
        hsh = __ldcg(slot_v + 2 * G + par);
      }
      __syncthreads();
      h = hsh;
    } else if (kMode == 1) {
      if (tid == 0) {
        slot_v[par * G + blockIdx.x] = cta;
        st_release(slot_tag + par * G + blockIdx.x, want);
      }
      double v = 0.0;
      if (tid < G) {
        while (ld_acquire(slot_tag + par * G + tid) != want) {
        }
        v = __ldcg(slot_v + par * G + tid);
      }
      h = block_tree(v, G);
    } else {
      if (tid == 0) st_pair(pairs + par * G + blockIdx.x, __double_as_longlong(cta), want);
      double v = 0.0;
      if (tid < G) {
        ulonglong2 p;
        do {
          p = ld_pair(pairs + par * G + tid);
        } while (p.y != want);
        v = __longlong_as_double(p.x);
      }
      h = block_tree(v, G);
    }
    h = 1.0 + h * 1e-9;
    chk += h;
  }
  if (tid == 0) out[blockIdx.x] = chk;
}

int main(int argc, char** argv) {
  const int G = argc > 1 ? atoi(argv[1]) : 256;
  const int passes = argc > 2 ? atoi(argv[2]) : 2000;
  const int per_cta = argc > 3 ? atoi(argv[3]) : 0;
  double *slot_v, *out, *stream;
  unsigned long long* slot_tag;
  ulonglong2* pairs;
  cudaMalloc(&slot_v, sizeof(double) * 4096);
  cudaMalloc(&slot_tag, sizeof(unsigned long long) * 4096);
  cudaMalloc(&pairs, sizeof(ulonglong2) * 4096);
  cudaMalloc(&out, sizeof(double) * 4096);
  cudaMalloc(&stream, sizeof(double) * (size_t(8) * G * per_cta + 1));
  cudaMemset(stream, 0, sizeof(double) * (size_t(8) * G * per_cta + 1));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(slot_tag, 0, sizeof(unsigned long long) * 4096);
      cudaMemset(pairs, 0, sizeof(ulonglong2) * 4096);
      int ps = passes;
      void* args[] = {&ps, &slot_v, &slot_tag, &pairs, &stream, (void*)&per_cta, &out};
      void* fn = mode == 0 ? (void*)probe<0> : mode == 1 ? (void*)probe<1> : (void*)probe<2>;
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kThreads), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        printf("mode %d: launch failed: %s\n", mode, cudaGetErrorString(e));
        break;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 1)
        printf("mode %d G=%d per_cta=%d: %.3f us/pass\n", mode, G, per_cta, ms * 1e3 / passes);
    }
  }
  return 0;
}
