// Micro-probe: cycles per entry of the backward face-block fold of the
// dataflow sweeps (walk.cu level_chunk, !par path): 4 rows x 44 entries,
// row r's first r entries are in-task sources (earlier rows of the task,
// leading in column order as in the U factor), then out-of-task products.
//  v0: lane 0 folds from shared memory in 8-entry batches (current kernel)
//  v1: v0 with the next batch's operands (and in-task lookups) loaded before
//      the current batch's subtractions (software pipelining)
//  v2: in-task prefix first (shared-memory lookups), then the out-of-task
//      tail as a pure chain over products, loads pipelined one batch ahead
//  v3: dependent dsub chain from registers (latency lower bound, no rows)
//  v4: dependent __ddiv_rn chain (cycles per division)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false tools/probe_fold3.cu
#include <cstdio>
#include <cstring>
constexpr int kRows = 4, kLen = 44, kN = kRows * kLen;

__device__ __forceinline__ int src_of(double2 r) { return int(__double_as_longlong(r.y)); }

__global__ void fold(const double2* g, const double* dv, long long* cyc, double* out, int variant) {
  __shared__ double2 rec[kN + 16];
  __shared__ double cv[kRows];
  __shared__ double dvb[kRows];
  for (int i = threadIdx.x; i < kN; i += 32) rec[i] = g[i];
  if (threadIdx.x < 16) rec[kN + threadIdx.x] = make_double2(0.0, __longlong_as_double(-1ll));
  if (threadIdx.x < kRows) dvb[threadIdx.x] = dv[threadIdx.x];
  __syncwarp();
  const int lane = threadIdx.x;
  double acc = 0.0;
  long long t0 = clock64();
  if (lane == 0 && variant == 0) {
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
          s8[k] = src_of(r2);
          p8[k] = r2.x;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) c8[k] = s8[k] < 0 ? 0.0 : cv[s8[k]];
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = __dsub_rn(acc, s8[k] < 0 ? p8[k] : __dmul_rn(p8[k], c8[k]));
      }
      for (; e < e1; ++e) {
        const double2 r2 = rec[e];
        const int s = src_of(r2);
        acc = __dsub_rn(acc, s < 0 ? r2.x : __dmul_rn(r2.x, cv[s]));
      }
      acc = __ddiv_rn(acc, dvb[r]);
      cv[r] = acc;
    }
  } else if (lane == 0 && variant == 1) {
    int e = 0;
    for (int r = 0; r < kRows; ++r) {
      acc = 1.0 + r;
      const int e1 = e + kLen;
      double2 nx[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) nx[k] = rec[e + k];
      for (; e + 8 <= e1; e += 8) {
        double2 cur[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) cur[k] = nx[k];
#pragma unroll
        for (int k = 0; k < 8; ++k) nx[k] = rec[e + 8 + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int s = src_of(cur[k]);
          acc = __dsub_rn(acc, s < 0 ? cur[k].x : __dmul_rn(cur[k].x, cv[s]));
        }
      }
      for (; e < e1; ++e) {
        const double2 r2 = rec[e];
        const int s = src_of(r2);
        acc = __dsub_rn(acc, s < 0 ? r2.x : __dmul_rn(r2.x, cv[s]));
      }
      acc = __ddiv_rn(acc, dvb[r]);
      cv[r] = acc;
    }
  } else if (lane == 0 && variant == 2) {
    int e = 0;
    for (int r = 0; r < kRows; ++r) {
      acc = 1.0 + r;
      const int e1 = e + kLen;
      // in-task prefix
      for (;;) {
        const double2 r2 = rec[e];
        const int s = src_of(r2);
        if (e >= e1 || s < 0) break;
        acc = __dsub_rn(acc, __dmul_rn(r2.x, cv[s]));
        ++e;
      }
      double nx[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) nx[k] = rec[e + k].x;
      for (; e + 8 <= e1; e += 8) {
        double cur[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) cur[k] = nx[k];
#pragma unroll
        for (int k = 0; k < 8; ++k) nx[k] = rec[e + 8 + k].x;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = __dsub_rn(acc, cur[k]);
      }
      for (int k = 0; e < e1; ++e, ++k) acc = __dsub_rn(acc, nx[k]);
      acc = __ddiv_rn(acc, dvb[r]);
      cv[r] = acc;
    }
  } else if (lane == 0 && variant == 3) {
    double p[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) p[k] = rec[k].x;
    acc = 1.0;
    for (int r = 0; r < kN / 16; ++r)
#pragma unroll
      for (int k = 0; k < 16; ++k) acc = __dsub_rn(acc, p[k]);
  } else if (lane == 0 && variant == 4) {
    acc = 1e300;
    for (int r = 0; r < kN; ++r) acc = __ddiv_rn(acc, dvb[r & 3]);
  }
  long long t1 = clock64();
  if (lane == 0) {
    out[variant] = acc;
    cyc[variant] = t1 - t0;
  }
}

__global__ void fold_many(const double2* g, const double* dv, long long* cyc, double* out, int variant) {
  // every warp of the grid folds its own copy (issue / FP64 pipe sharing of a loaded SM)
  __shared__ double2 rec[8][kN + 16];
  __shared__ double cv[8][kRows];
  __shared__ double dvb[8][kRows];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < kN; i += 32) rec[w][i] = g[i];
  if (lane < 16) rec[w][kN + lane] = make_double2(0.0, __longlong_as_double(-1ll));
  if (lane < kRows) dvb[w][lane] = dv[lane];
  __syncwarp();
  double acc = 0.0;
  long long t0 = clock64();
  if (lane == 0 || variant == 5) {
    int e = 0;
    for (int r = 0; r < kRows; ++r) {
      acc = 1.0 + r;
      const int e1 = e + kLen;
      if (variant == 6) {
        for (;;) {
          const double2 r2 = rec[w][e];
          const int s = src_of(r2);
          if (e >= e1 || s < 0) break;
          acc = __dsub_rn(acc, __dmul_rn(r2.x, cv[w][s]));
          ++e;
        }
        // the tail in register batches of 16 (all loads issued, then the chain)
        for (; e < e1; e += 16) {
          double b[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) b[k] = e + k < e1 ? rec[w][e + k].x : 0.0;
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (e + k < e1) acc = __dsub_rn(acc, b[k]);
        }
        e = e1;
      } else if (variant == 5) {
        // warp-cooperative: leading in-task terms warp-uniformly, then the
        // tail's products one per lane, folded through shuffles
        for (;;) {
          const double2 r2 = rec[w][e];
          const int s = src_of(r2);
          if (e >= e1 || s < 0) break;
          acc = __dsub_rn(acc, __dmul_rn(r2.x, cv[w][s]));
          ++e;
        }
        for (int base = e; base < e1; base += 32) {
          const double p = base + lane < e1 ? rec[w][base + lane].x : 0.0;
          const int cnt = e1 - base < 32 ? e1 - base : 32;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const double x = __shfl_sync(0xffffffffu, p, k);
            if (k < cnt) acc = __dsub_rn(acc, x);
          }
        }
        e = e1;
      } else if (variant == 2) {
        for (;;) {
          const double2 r2 = rec[w][e];
          const int s = src_of(r2);
          if (e >= e1 || s < 0) break;
          acc = __dsub_rn(acc, __dmul_rn(r2.x, cv[w][s]));
          ++e;
        }
        double nx[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) nx[k] = rec[w][e + k].x;
        for (; e + 4 <= e1; e += 4) {
          double cur[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) cur[k] = nx[k];
#pragma unroll
          for (int k = 0; k < 4; ++k) nx[k] = rec[w][e + 4 + k].x;
#pragma unroll
          for (int k = 0; k < 4; ++k) acc = __dsub_rn(acc, cur[k]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (e + k < e1) acc = __dsub_rn(acc, nx[k]);
        e = e1;
      } else {
        for (; e < e1; ++e) {
          const double2 r2 = rec[w][e];
          const int s = src_of(r2);
          acc = __dsub_rn(acc, s < 0 ? r2.x : __dmul_rn(r2.x, cv[w][s]));
        }
      }
      acc = __ddiv_rn(acc, dvb[w][r]);
      if (lane == 0) cv[w][r] = acc;
      __syncwarp(variant == 5 ? 0xffffffffu : 1u);
    }
  }
  long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0 && w == 0) {
    out[variant] = acc;
    cyc[variant] = t1 - t0;
  }
}

int main() {
  double2* g;
  double *o, *dv;
  long long* c;
  cudaMalloc(&g, sizeof(double2) * kN);
  cudaMalloc(&c, 64);
  cudaMalloc(&o, 64);
  cudaMalloc(&dv, 64);
  double2 h[kN];
  for (int i = 0; i < kN; ++i) {
    const int r = i / kLen, k = i % kLen;
    const long long s = k < r ? k : -1;  // row r: r leading in-task sources
    double sd;
    memcpy(&sd, &s, 8);
    h[i] = make_double2(1e-3 * (i + 1), sd);
  }
  const double hd[4] = {1.5, 2.5, 3.5, 1.25};
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hd, sizeof(hd), cudaMemcpyHostToDevice);
  const char* nm[5] = {"v0 lane-0 smem fold", "v1 pipelined smem fold", "v2 prefix + pipelined tail",
                       "v3 register dsub chain", "v4 ddiv chain"};
  for (int v = 0; v < 5; ++v) {
    fold<<<1, 32>>>(g, dv, c, o, v);
    fold<<<1, 32>>>(g, dv, c, o, v);
    long long hc[5];
    double res[5];
    cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
    cudaMemcpy(res, o, sizeof(res), cudaMemcpyDeviceToHost);
    printf("%-28s %.1f cycles/entry (result %.17g)\n", nm[v], double(hc[v]) / kN, res[v]);
  }
  for (int v : {2, 6}) {
    for (int ctas : {1, 148, 148 * 7}) {
      fold_many<<<ctas, 128>>>(g, dv, c, o, v);
      fold_many<<<ctas, 128>>>(g, dv, c, o, v);
      long long hc[8];
      cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
      printf("fold_many variant %d, %4d CTAs x 4 warps: %.1f cycles/entry (whole task %lld cycles)\n", v,
             ctas, double(hc[v]) / kN, hc[v]);
    }
  }
  return 0;
}
