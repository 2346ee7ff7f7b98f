// Micro-probe: one-way hand-over latency of the dataflow sweeps' publication
// scheme (walk.cu flow_store / flow_peek: an 8-byte relaxed gpu-scope store
// over a signalling-NaN sentinel, polled with relaxed gpu-scope loads).
// A token travels a chain of hops; hop h is taken by warp (h * stride) % W of
// a grid of W warps (CTAs of 4 warps spread over the SMs), so consecutive
// hops run on different SMs. Extra warps optionally spin on unrelated
// addresses (background polling load, as thousands of waiting tasks do).
// Prints ns per hop.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_hop.cu -o tools/probe_hop
#include <cstdio>
#include <cstdlib>

constexpr unsigned long long kSent = 0xFFF7DEADBEEF5A5Aull;

__device__ __forceinline__ unsigned long long peek(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void put(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__global__ void fill(double* y, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = __longlong_as_double((long long)kSent);
}

// hops: chain length; every warp w handles hops h with h % W == w (in order)
__global__ void chain(double* y, int hops, int W, int noise_warps, double* noise,
                      unsigned long long* t) {
  const int w = int(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  const int lane = threadIdx.x & 31;
  if (w >= W) {
    // background: spin on private sentinel slots until the chain ends
    if (w - W < noise_warps) {
      const double* p = noise + size_t(w - W) * 64 + lane;
      while (peek(y + hops - 1) == kSent) {
        (void)peek(p);
      }
    }
    return;
  }
  // consecutive hops on consecutive CTAs (different SMs)
  const int nC = W / 4;
  const int slot = (w % 4) * nC + w / 4;
  for (int h = slot; h < hops; h += W) {
    if (h > 0) {
      unsigned long long v;
      do {
        v = peek(y + h - 1);
      } while (v == kSent);
      if (lane == 0) put(y + h, __longlong_as_double((long long)v) + 1.0);
    } else if (lane == 0) {
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      t[0] = t0;
      put(y, 0.0);
    }
    __syncwarp();
  }
  if (slot == (hops - 1) % W && lane == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    t[1] = t1;
  }
}

int main(int argc, char** argv) {
  const int hops = argc > 1 ? atoi(argv[1]) : 20000;
  double *y, *noise;
  unsigned long long* t;
  cudaMalloc(&y, sizeof(double) * hops);
  cudaMalloc(&noise, sizeof(double) * 64 * 8192);
  cudaMalloc(&t, 16);
  fill<<<256, 256>>>(noise, 64 * 8192);
  const int configs[][2] = {{148, 0}, {148 * 4, 0}, {148 * 4, 1024}, {148 * 4, 2048}, {148 * 4, 3500}};
  for (auto& cfg : configs) {
    const int W = cfg[0], noise_w = cfg[1];
    const int total = W + noise_w;
    const int ctas = (total + 3) / 4;
    for (int rep = 0; rep < 2; ++rep) {
      fill<<<256, 256>>>(y, hops);
      chain<<<ctas, 128>>>(y, hops, W, noise_w, noise, t);
      cudaDeviceSynchronize();
    }
    unsigned long long h[2];
    cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
    const cudaError_t e = cudaGetLastError();
    printf("chain warps %5d, background polling warps %5d: %.0f ns per hop%s\n", W, noise_w,
           double(h[1] - h[0]) / (hops - 1), e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
