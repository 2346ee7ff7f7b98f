// Micro-probe: dependent FP64 add / mul / div latency and a smem-fed fold.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, const double* g, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  if (threadIdx.x) return;
  double a = g[0], b = g[1];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dsub_rn(a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) a = __dmul_rn(a, b);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) a = __ddiv_rn(a, b);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) a = __dsub_rn(a, sm[i & 1023]);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) a = __dsub_rn(a, __dmul_rn(sm[i & 1023], sm[(i * 7) & 1023]));
  long long t5 = clock64();
  float f = float(a);
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, 1.0f);
  long long t6 = clock64();
  out[0] = a + f;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
}
int main() {
  double* g; double* o; long long* c;
  cudaMalloc(&g, 8 * 1024); cudaMalloc(&o, 8); cudaMalloc(&c, 64);
  double h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 1.0 + 1e-9 * i;
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 4096;
  lat<<<1, 128>>>(o, c, g, n);
  lat<<<1, 128>>>(o, c, g, n);
  long long hc[6]; cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  const char* nm[6] = {"dsub chain", "dmul chain", "ddiv chain", "dsub(smem) chain", "dsub(dmul(smem,smem))", "fadd chain"};
  for (int i = 0; i < 6; ++i) printf("%-24s %.1f cycles/op\n", nm[i], double(hc[i]) / n);
  return 0;
}
