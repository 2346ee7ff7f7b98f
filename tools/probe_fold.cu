// Micro-probe: cycles per entry of the task-level kernel's lane-0 fold
// (walk.cu level_chunk) on synthetic shared-memory operands, against a
// plain dependent subtraction chain.
#include <cstdio>
constexpr int kN = 512, kRows = 16;
__global__ void fold(const double* g, const int* gs, long long* cyc, double* out, int variant) {
  __shared__ double pbuf[kN];
  __shared__ int sbuf[kN];
  __shared__ double cv[kRows];
  for (int i = threadIdx.x; i < kN; i += 32) { pbuf[i] = g[i]; sbuf[i] = gs[i]; }
  if (threadIdx.x < kRows) cv[threadIdx.x] = 1.0 + threadIdx.x;
  __syncwarp();
  if (threadIdx.x) return;
  const int len = 28;  // entries per row
  long long t0 = clock64();
  double acc = 0.0;
  int e = 0;
  for (int r = 0; r < kRows; ++r) {
    acc = g[r];
    const int e1 = e + len;
    if (variant == 0) {
      for (; e + 8 <= e1; e += 8) {
        int s8[8]; double p8[8], c8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) { s8[k] = sbuf[e + k]; p8[k] = pbuf[e + k]; }
#pragma unroll
        for (int k = 0; k < 8; ++k) c8[k] = s8[k] < 0 ? 0.0 : cv[s8[k]];
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = __dsub_rn(acc, s8[k] < 0 ? p8[k] : __dmul_rn(p8[k], c8[k]));
      }
      for (; e < e1; ++e) { const int s = sbuf[e]; acc = __dsub_rn(acc, s < 0 ? pbuf[e] : __dmul_rn(pbuf[e], cv[s])); }
    } else {
      for (; e < e1; ++e) acc = __dsub_rn(acc, pbuf[e]);
    }
    cv[r] = acc;
  }
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}
int main() {
  double* g; int* gs; long long* c; double* o;
  cudaMalloc(&g, 8 * kN); cudaMalloc(&gs, 4 * kN); cudaMalloc(&c, 8); cudaMalloc(&o, 8);
  double h[kN]; int hs[kN];
  for (int i = 0; i < kN; ++i) { h[i] = 1e-3 * (i + 1); hs[i] = (i % 28 == 27) ? (i / 28 > 0 ? i / 28 - 1 : -1) : -1; }
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice); cudaMemcpy(gs, hs, sizeof(hs), cudaMemcpyHostToDevice);
  for (int v = 0; v < 2; ++v) {
    fold<<<1, 32>>>(g, gs, c, o, v); fold<<<1, 32>>>(g, gs, c, o, v);
    long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("%s: %.1f cycles/entry (%d entries)\n", v ? "plain dsub chain from smem" : "level-kernel fold",
           double(hc) / (16 * 28), 16 * 28);
  }
  return 0;
}
