// FP64 peak probe for the condensation roofline ("its peak
// must be measured with a DGEMM probe"): sustained FP64 throughput of
//   (a) the tensor pipe: mma.sync.aligned.m8n8k4.f64 (DMMA), register
//       operands, 8 independent accumulator tiles per warp;
//   (b) the SIMT pipe: DFMA, 8 independent chains per thread;
//   (c) the SIMT pipe as the bitwise kernels use it: separately rounded
//       DMUL + DADD (--fmad=false), 8 independent chains per thread.
// One persistent grid of 148 x 4 CTAs of 256 threads, CUDA-event timed.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_dmma.cu -o tools/probe_dmma
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_kernel(double* out, int iters) {
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_kernel(double* out, int iters) {
  double c[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t] = 1e-3 * t;
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1e-9 * threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = __fma_rn(c[t], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmuladd_kernel(double* out, int iters) {
  double c[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t] = 1e-3 * t;
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1e-9 * threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = __dadd_rn(__dmul_rn(c[t], a), b);
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
static double time_ms(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  const int grid = 148 * 4, threads = 256, iters = 20000;
  double* out;
  cudaMalloc(&out, sizeof(double) * grid * threads);
  const double warps = double(grid) * threads / 32;
  double ms = time_ms([&] { dmma_kernel<<<grid, threads>>>(out, iters); });
  // one m8n8k4 = 8*8*4 FMA = 512 flop per warp instruction
  printf("DMMA m8n8k4.f64       %8.2f TFLOP/s (%.2f ms)\n", warps * iters * 8 * 512.0 / ms / 1e9, ms);
  ms = time_ms([&] { dfma_kernel<<<grid, threads>>>(out, iters); });
  printf("DFMA (SIMT)           %8.2f TFLOP/s (%.2f ms)\n", double(grid) * threads * iters * 8 * 2.0 / ms / 1e9, ms);
  ms = time_ms([&] { dmuladd_kernel<<<grid, threads>>>(out, iters); });
  printf("DMUL+DADD (no fusion) %8.2f TFLOP/s counted as 2 flop per pair (%.2f ms)\n",
         double(grid) * threads * iters * 8 * 2.0 / ms / 1e9, ms);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
