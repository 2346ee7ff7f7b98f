// Micro-probe: cycles per entry of candidate chain folds for the task-level
// sweep kernel (walk.cu level_chunk): a task of kRows rows x kLen entries,
// entries {product or factor, source} staged in shared memory; an entry
// whose source is an earlier row of the task multiplies that row's result.
//  v0: lane 0 folds from shared memory (the round-1 kernel, 8-entry batches)
//  v1: every lane folds the same chain (warp-uniform), operands as 16-byte
//      shared-memory broadcasts, in-task results kept by lane r (shuffle)
//  v2: v1 with the next batch's operands loaded before the current batch's
//      subtractions (software pipelining)
//  v3: plain dependent dsub chain from registers (lower bound)
#include <cstdio>
#include <cstring>
constexpr int kRows = 16, kLen = 32, kN = kRows * kLen;

__global__ void fold(const double2* g, long long* cyc, double* out, int variant) {
  __shared__ double2 rec[kN];
  __shared__ double cv[kRows];
  for (int i = threadIdx.x; i < kN; i += 32) rec[i] = g[i];
  __syncwarp();
  const int lane = threadIdx.x;
  long long t0 = clock64();
  double acc = 0.0;
  if (variant == 0) {
    if (lane == 0) {
      int e = 0;
      for (int r = 0; r < kRows; ++r) {
        acc = 1.0 + r;
        const int e1 = e + kLen;
        for (; e + 8 <= e1; e += 8) {
          int s8[8];
          double p8[8], c8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const double2 r2 = rec[e + k];
            s8[k] = int(__double_as_longlong(r2.y));
            p8[k] = r2.x;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) c8[k] = s8[k] < 0 ? 0.0 : cv[s8[k]];
#pragma unroll
          for (int k = 0; k < 8; ++k) acc = __dsub_rn(acc, s8[k] < 0 ? p8[k] : __dmul_rn(p8[k], c8[k]));
        }
        cv[r] = acc;
      }
    }
  } else if (variant == 1 || variant == 2) {
    double mine = 0.0;  // lane r keeps row r's result
    int e = 0;
    double2 nx[8];
    if (variant == 2)
#pragma unroll
      for (int k = 0; k < 8; ++k) nx[k] = rec[k];
    for (int r = 0; r < kRows; ++r) {
      acc = 1.0 + r;
      const int e1 = e + kLen;
      for (; e < e1; e += 8) {
        double2 cur[8];
        if (variant == 2) {
#pragma unroll
          for (int k = 0; k < 8; ++k) cur[k] = nx[k];
          if (e + 8 < kN)
#pragma unroll
            for (int k = 0; k < 8; ++k) nx[k] = rec[e + 8 + k];
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) cur[k] = rec[e + k];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int s = int(__double_as_longlong(cur[k].y));
          const double x = __shfl_sync(0xffffffffu, mine, s < 0 ? 0 : s);
          acc = __dsub_rn(acc, s < 0 ? cur[k].x : __dmul_rn(cur[k].x, x));
        }
      }
      if (lane == r) mine = acc;
    }
  } else {
    double p[kLen];
#pragma unroll
    for (int k = 0; k < kLen; ++k) p[k] = rec[k].x;
    for (int r = 0; r < kRows; ++r) {
      acc = 1.0 + r;
#pragma unroll
      for (int k = 0; k < kLen; ++k) acc = __dsub_rn(acc, p[k]);
    }
  }
  long long t1 = clock64();
  if (lane == 0) {
    out[variant] = acc;
    cyc[variant] = t1 - t0;
  }
}

int main() {
  double2* g;
  long long* c;
  double* o;
  cudaMalloc(&g, sizeof(double2) * kN);
  cudaMalloc(&c, 64);
  cudaMalloc(&o, 64);
  double2 h[kN];
  for (int i = 0; i < kN; ++i) {
    const int r = i / kLen, k = i % kLen;
    // the last entry of every row (but the first) reads the previous row
    const long long s = (k == kLen - 1 && r > 0) ? r - 1 : -1;
    double sd;
    memcpy(&sd, &s, 8);
    h[i] = make_double2(1e-3 * (i + 1), sd);
  }
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  const char* nm[4] = {"v0 lane-0 smem fold", "v1 warp-uniform broadcast", "v2 pipelined broadcast",
                       "v3 register chain"};
  double res[4];
  for (int v = 0; v < 4; ++v) {
    fold<<<1, 32>>>(g, c, o, v);
    fold<<<1, 32>>>(g, c, o, v);
    long long hc[4];
    cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
    cudaMemcpy(res, o, sizeof(res), cudaMemcpyDeviceToHost);
    printf("%-28s %.1f cycles/entry (result %.17g)\n", nm[v], double(hc[v]) / kN, res[v]);
  }
  return 0;
}
