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
#include <algorithm>
#include <cstdlib>
#include <vector>

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

// ---------------------------------------------------------------------------
// Persistent Arnoldi step: all j+2 MGS passes of ArnoldiWorkspace::step in
// one cooperative launch. Thread x of CTA b owns the L consecutive lanes
// (b*256 + x)*L .. +L-1 and keeps their elements of w in shared memory, so
// a pass streams only v_i (and v_{i-1}, an L2 hit). After each pass the CTA
// results go through one grid barrier and every CTA rebuilds the same
// adjacent-pair tree over them, so h_i is known everywhere without a second
// barrier. The tree shape (L lanes -> 256 threads -> G CTAs) is the global
// adjacent-pair tree over T = G*256*L lanes, i.e. identical to mgs_pass.
// ---------------------------------------------------------------------------

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ void grid_barrier(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = ld_acquire_u32(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0u;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (ld_acquire_u32(gen) == g0) {
      }
    }
  }
  __syncthreads();
}

constexpr int kStepThreads = 256;

/// Tree over `cnt` (power of two, <= 1024) values in smem buf, in place;
/// result in buf[0]. All threads of the CTA participate.
__device__ void smem_tree(double* buf, int cnt) {
  for (int width = cnt; width > 1; width >>= 1) {
    const int half = width >> 1;
    double t0 = 0.0, t1 = 0.0;
    const int k0 = threadIdx.x, k1 = threadIdx.x + kStepThreads;
    if (k0 < half) t0 = dadd(buf[2 * k0], buf[2 * k0 + 1]);
    if (k1 < half) t1 = dadd(buf[2 * k1], buf[2 * k1 + 1]);
    __syncthreads();
    if (k0 < half) buf[k0] = t0;
    if (k1 < half) buf[k1] = t1;
    __syncthreads();
  }
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

#ifdef PSCU_TRACE
__device__ long long* g_mgs_trace = nullptr;  // per-pass clock64 stamps of CTA 0 thread 0
#define MGS_STAMP(i, k)                                                          \
  do {                                                                           \
    if (g_mgs_trace && blockIdx.x == 0 && threadIdx.x == 0 && (i) < 1024)        \
      g_mgs_trace[(i) * 4 + (k)] = clock64();                                    \
  } while (0)
#else
#define MGS_STAMP(i, k) \
  do {                  \
  } while (0)
#endif

constexpr int kEpt = 16;  // elements per lane (repro_lanes guarantees <= 16 up to n = 2^22)

// Slot pairs are written and read as single 128-bit accesses (.b128 types:
// one STG.E.128 / LDG.E.128, never split into two 64-bit accesses), so a
// reader sees either the old or the new pair, never a torn mix; the
// {value, value ^ tag} check then only distinguishes stale from current.
__device__ __forceinline__ void st_pair(ulonglong2* p, unsigned long long a, unsigned long long b) {
  asm volatile(
      "{\n .reg .b128 t;\n mov.b128 t, {%1, %2};\n st.relaxed.gpu.global.b128 [%0], t;\n}"
      ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ ulonglong2 ld_pair(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile(
      "{\n .reg .b128 t;\n ld.relaxed.gpu.global.b128 t, [%2];\n mov.b128 {%0, %1}, t;\n}"
      : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}

/// All j+2 MGS passes of one Arnoldi step. Per pass every CTA publishes its
/// subtree result in its own slot; the root CTA gathers all G slots,
/// rebuilds the adjacent-pair tree and publishes the result. Slots are
/// double-buffered by pass parity and tags are unique per launch (tag_base),
/// so nothing is ever reset.
///   kPairs false: value + release-tagged pass id (release/acquire).
///   kPairs true: {value bits, value bits ^ tag} in one relaxed 16-byte store.
// two CTAs per SM (<= 128 registers) so up to 296 CTAs are co-resident:
// n = 525k (the 256^2 coarse level) needs T = 65536 lanes = 256 CTAs
/// kL adjacent lanes per thread (the first tree level is then in-thread):
/// kL = 2 halves the CTAs taking part in each grid-wide reduction.
template <int kL>
struct StepShape {
  static constexpr int kE = kL == 1 ? kEpt : 10;  // elements per lane held in registers
};

template <int kL, bool kPairs, bool kAll = false>
__global__ void __launch_bounds__(kStepThreads, kL == 1 ? 2 : 1)
    arnoldi_step_kernel(int64_t n, int64_t T, int epl, int j, double* __restrict__ wg,
                        double* V, int64_t ldv, double* __restrict__ hcol,
                        double* __restrict__ slot_v, unsigned long long* slot_tag,
                        unsigned long long tag_base) {
  // w, v_{i-1} and v_i stay in registers and v_{i+1} is prefetched while the
  // grid-wide reduction of pass i completes
  constexpr int kE = StepShape<kL>::kE;
  __shared__ double hsh;
  const int G = gridDim.x;
  const int tid = threadIdx.x;
  const int64_t lane0 = (int64_t(blockIdx.x) * kStepThreads + tid) * kL;
  double w[kL][kE], pv[kL][kE], iv[kL][kE];
#pragma unroll
  for (int l = 0; l < kL; ++l)
#pragma unroll
    for (int k = 0; k < kE; ++k) {
      const int64_t e = lane0 + l + int64_t(k) * T;
      const bool ok = k < epl && e < n;
      w[l][k] = ok ? wg[e] : 0.0;
      iv[l][k] = ok ? __ldcg(V + e) : 0.0;  // v_0
      pv[l][k] = 0.0;
    }
  double hprev = 0.0;
  for (int i = 0; i <= j + 1; ++i) {
    MGS_STAMP(i, 0);
    double acc[kL];
#pragma unroll
    for (int l = 0; l < kL; ++l) {
      acc[l] = 0.0;
#pragma unroll
      for (int k = 0; k < kE; ++k) {
        const int64_t e = lane0 + l + int64_t(k) * T;
        if (k < epl && e < n) {
          if (i > 0) w[l][k] = dsub(w[l][k], dmul(hprev, pv[l][k]));
          const double o = i <= j ? iv[l][k] : w[l][k];
          acc[l] = dadd(acc[l], dmul(w[l][k], o));
        }
      }
    }
    const double cta = block_tree(kL == 1 ? acc[0] : dadd(acc[0], acc[kL - 1]), kStepThreads);
    MGS_STAMP(i, 1);
    const int par = i & 1;
    const unsigned long long want = tag_base + unsigned(i) + 1ull;
    if (tid == 0) {
      if (kPairs) {
        const unsigned long long bits = __double_as_longlong(cta);
        st_pair(reinterpret_cast<ulonglong2*>(slot_tag) + par * G + blockIdx.x, bits, bits ^ want);
      } else {
        slot_v[par * G + blockIdx.x] = cta;
        st_release_u64(slot_tag + par * G + blockIdx.x, want);
      }
    }
    // prefetch v_{i+1} (independent of h_i) before waiting on the grid
    if (i + 1 <= j) {
      const double* vn = V + int64_t(i + 1) * ldv;
#pragma unroll
      for (int l = 0; l < kL; ++l)
#pragma unroll
        for (int k = 0; k < kE; ++k) {
          const int64_t e = lane0 + l + int64_t(k) * T;
          pv[l][k] = iv[l][k];
          iv[l][k] = (k < epl && e < n) ? __ldcg(vn + e) : 0.0;
        }
    } else {
#pragma unroll
      for (int l = 0; l < kL; ++l)
#pragma unroll
        for (int k = 0; k < kE; ++k) pv[l][k] = iv[l][k];
    }
    if (kAll) {
      // every CTA gathers all G pairs and rebuilds the same tree: one grid
      // round trip per pass, no root. A slot of parity par is rewritten two
      // passes later, after every CTA has published the pass in between,
      // i.e. after every CTA finished reading it.
      ulonglong2* pairs = reinterpret_cast<ulonglong2*>(slot_tag);
      double v = 0.0;
      if (tid < G) {
        ulonglong2 p;
        do {
          p = ld_pair(pairs + par * G + tid);
        } while ((p.x ^ p.y) != want);
        v = __longlong_as_double(p.x);
      }
      __syncthreads();  // warp 0 finished reading block_tree's scratch of this pass
      MGS_STAMP(i, 2);
      v = block_tree(v, G);
      if (tid == 0) {
        if (i == j + 1) v = __dsqrt_rn(v);
        hsh = v;
        if (blockIdx.x == 0) hcol[i] = v;
      }
    } else if (kPairs) {
      // relaxed 128-bit {value, value ^ tag} pairs (single-access .b128
      // stores/loads, never torn): a pair is accepted only when its two words
      // agree on this pass's tag, so neither side needs a fence: the value is
      // the only datum
      ulonglong2* pairs = reinterpret_cast<ulonglong2*>(slot_tag);
      if (blockIdx.x == 0) {
        double v = 0.0;
        if (tid < G) {
          ulonglong2 p;
          do {
            p = ld_pair(pairs + par * G + tid);
          } while ((p.x ^ p.y) != want);
          v = __longlong_as_double(p.x);
        }
        __syncthreads();  // warp 0 finished reading block_tree's scratch of this pass
        v = block_tree(v, G);
        if (tid == 0) {
          if (i == j + 1) v = __dsqrt_rn(v);
          hsh = v;
          hcol[i] = v;
          const unsigned long long rb = __double_as_longlong(v);
          st_pair(pairs + 2 * G + par, rb, rb ^ want);
        }
      } else if (tid == 0) {
        ulonglong2 p;
        do {
          p = ld_pair(pairs + 2 * G + par);
        } while ((p.x ^ p.y) != want);
        hsh = __longlong_as_double(p.x);
      }
    } else if (blockIdx.x == 0) {
      // root CTA: thread k < G acquires slot k (one round trip), rebuilds
      // the adjacent-pair tree and publishes the result under one tag
      double v = 0.0;
      if (tid < G) {
        while (ld_acquire_u64(slot_tag + par * G + tid) != want) {
        }
        v = __ldcg(slot_v + par * G + tid);
      }
      __syncthreads();  // warp 0 finished reading block_tree's scratch of this pass
      v = block_tree(v, G);
      if (tid == 0) {
        if (i == j + 1) v = __dsqrt_rn(v);
        hsh = v;
        hcol[i] = v;
        slot_v[2 * G + par] = v;
        st_release_u64(slot_tag + 2 * G + par, want);
      }
    } else if (tid == 0) {
      // every other CTA polls the single published result
      while (ld_acquire_u64(slot_tag + 2 * G + par) != want) __nanosleep(20);
      hsh = __ldcg(slot_v + 2 * G + par);
    }
    __syncthreads();
    hprev = hsh;
    MGS_STAMP(i, 3);
    __syncthreads();
  }
  // v_{j+1} = w / h, or 0 on a happy breakdown (gmres.hpp:66-67)
  double* vn = V + int64_t(j + 1) * ldv;
#pragma unroll
  for (int l = 0; l < kL; ++l)
#pragma unroll
    for (int k = 0; k < kE; ++k) {
      const int64_t e = lane0 + l + int64_t(k) * T;
      if (k < epl && e < n) vn[e] = hprev > 0.0 ? __ddiv_rn(w[l][k], hprev) : 0.0;
    }
}


// ---------------------------------------------------------------------------
// The same Arnoldi step with the basis vectors streamed through shared
// memory: CTA b's lanes [b*512, b*512+512) read, per vector, epl contiguous
// 4 KB segments (element e = lane + k*T), staged kVStages passes ahead by
// TMA bulk copies on an mbarrier per stage. A pass then waits on HBM only
// when the reductions outrun the copies, w stays in registers, v_{i-1} is
// re-read from its stage for the w update. Same arithmetic and tree as
// arnoldi_step_kernel<2, true, true>.
// ---------------------------------------------------------------------------

constexpr int kVStages = 3;
constexpr int kVLanes = 2 * kStepThreads;  // lanes per CTA

__device__ __forceinline__ unsigned sa(const void* p) {
  return unsigned(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void stage_vector(double* dst, const double* v, int64_t n, int64_t T,
                                             int epl, int64_t lane_base, uint64_t* bar) {
  unsigned bytes = 0;
  for (int k = 0; k < epl; ++k) {
    const int64_t s0 = lane_base + int64_t(k) * T;
    const int64_t cnt = s0 < n ? (n - s0 < kVLanes ? n - s0 : kVLanes) : 0;
    bytes += unsigned(cnt) * 8u;
  }
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(bytes)
               : "memory");
  for (int k = 0; k < epl; ++k) {
    const int64_t s0 = lane_base + int64_t(k) * T;
    const int64_t cnt = s0 < n ? (n - s0 < kVLanes ? n - s0 : kVLanes) : 0;
    if (cnt > 0)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(sa(dst + k * kVLanes)),
          "l"(v + s0), "r"(unsigned(cnt) * 8u), "r"(sa(bar))
          : "memory");
  }
}

__device__ __forceinline__ void wait_stage(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(sa(bar)),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(kStepThreads, 1)
    arnoldi_tma_kernel(int64_t n, int64_t T, int epl, int j, double* __restrict__ wg,
                       const double* V, int64_t ldv, double* __restrict__ hcol,
                       unsigned long long* slot_tag, unsigned long long tag_base, double* vout) {
  extern __shared__ __align__(16) double vst[];  // kVStages x epl x kVLanes
  __shared__ __align__(8) uint64_t bar[kVStages];
  __shared__ double hsh;
  const int G = gridDim.x;
  const int tid = threadIdx.x;
  const int64_t lane_base = int64_t(blockIdx.x) * kVLanes;
  const int64_t lane0 = lane_base + 2 * tid;
  const size_t sstride = size_t(epl) * kVLanes;
  if (tid == 0) {
    for (int s = 0; s < kVStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // vectors v_0 .. v_{kVStages-2} in flight before the first pass
  if (tid == 0)
    for (int s = 0; s < kVStages - 1 && s <= j; ++s)
      stage_vector(vst + s * sstride, V + int64_t(s) * ldv, n, T, epl, lane_base, &bar[s]);
  double w[2][kEpt];
#pragma unroll
  for (int l = 0; l < 2; ++l)
#pragma unroll
    for (int k = 0; k < kEpt; ++k) {
      const int64_t e = lane0 + l + int64_t(k) * T;
      w[l][k] = (k < epl && e < n) ? wg[e] : 0.0;
    }
  ulonglong2* pairs = reinterpret_cast<ulonglong2*>(slot_tag);
  double hprev = 0.0;
  for (int i = 0; i <= j + 1; ++i) {
    if (i <= j) wait_stage(&bar[i % kVStages], unsigned((i / kVStages) & 1));
    const double* vi = vst + (i % kVStages) * sstride;
    const double* vp = vst + ((i + kVStages - 1) % kVStages) * sstride;
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int k = 0; k < kEpt; ++k) {
      if (k >= epl) break;
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        const int64_t e = lane0 + l + int64_t(k) * T;
        if (e < n) {
          if (i > 0) w[l][k] = dsub(w[l][k], dmul(hprev, vp[k * kVLanes + 2 * tid + l]));
          const double o = i <= j ? vi[k * kVLanes + 2 * tid + l] : w[l][k];
          acc[l] = dadd(acc[l], dmul(w[l][k], o));
        }
      }
    }
    const double cta = block_tree(dadd(acc[0], acc[1]), kStepThreads);
    const int par = i & 1;
    const unsigned long long want = tag_base + unsigned(i) + 1ull;
    if (tid == 0) {
      const unsigned long long bits = __double_as_longlong(cta);
      st_pair(pairs + par * G + blockIdx.x, bits, bits ^ want);
    }
    if (tid == kStepThreads - 1) {
      // the last warp refills stage (i-1) with v_{i+kVStages-1} while the
      // reduction completes (block_tree's __syncthreads: every thread is
      // done with that stage)
      if (i >= 1 && i + kVStages - 1 <= j) {
        const int s = (i + kVStages - 1) % kVStages;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        stage_vector(vst + s * sstride, V + int64_t(i + kVStages - 1) * ldv, n, T, epl,
                     lane_base, &bar[s]);
      }
      if (i == 0 && kVStages - 1 <= j)
        stage_vector(vst + (kVStages - 1) * sstride, V + int64_t(kVStages - 1) * ldv, n, T, epl,
                     lane_base, &bar[kVStages - 1]);
    }
    double v = 0.0;
    if (tid < G) {
      ulonglong2 p;
      do {
        p = ld_pair(pairs + par * G + tid);
      } while ((p.x ^ p.y) != want);
      v = __longlong_as_double(p.x);
    }
    __syncthreads();  // warp 0 finished reading block_tree's scratch of this pass
    v = block_tree(v, G);
    if (tid == 0) {
      if (i == j + 1) v = __dsqrt_rn(v);
      hsh = v;
      if (blockIdx.x == 0) hcol[i] = v;
    }
    __syncthreads();
    hprev = hsh;
  }
  // v_{j+1} = w / h, or 0 on a happy breakdown (gmres.hpp:66-67)
#pragma unroll
  for (int l = 0; l < 2; ++l)
#pragma unroll
    for (int k = 0; k < kEpt; ++k) {
      const int64_t e = lane0 + l + int64_t(k) * T;
      if (k < epl && e < n) vout[e] = hprev > 0.0 ? __ddiv_rn(w[l][k], hprev) : 0.0;
    }
}

// ---------------------------------------------------------------------------
// The Arnoldi step for coarse levels too large for register-resident w
// (config 5: n = 3.2 M, 2^18 reproducible-dot lanes, 13 elements per lane):
// one 1024-thread CTA per SM holds its 2048 lanes' slice of w in shared
// memory (epl x 16 KB), so a pass streams only v_{i-1} (the w update; read
// one pass earlier, an L2 hit) and v_i (prefetched into L2 by a bulk
// prefetch one pass ahead, overlapping the grid reduction). Same lanes,
// same per-lane order, same adjacent-pair tree as arnoldi_step_kernel.
// ---------------------------------------------------------------------------

constexpr int kSmemThreads = 1024;
constexpr int kSmemLanes = 2 * kSmemThreads;  // lanes per CTA (two per thread)
constexpr int kSmemBatch = 4;                 // element slices loaded per batch

/// block_tree for up to 1024 lanes (32 warp partials).
__device__ double block_tree_1k(double v, int nlanes) {
  __shared__ double wsum[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wl = nlanes < 32 ? nlanes : 32;
  for (int off = 1; off < wl; off <<= 1) {
    const double o = __shfl_down_sync(0xffffffffu, v, off);
    if ((lane & (2 * off - 1)) == 0) v = dadd(v, o);
  }
  if (nlanes <= 32) return v;
  if (lane == 0) wsum[wid] = v;
  __syncthreads();
  const int nw = nlanes >> 5;
  if (wid == 0) {
    v = lane < nw ? wsum[lane] : 0.0;
    for (int off = 1; off < nw; off <<= 1) {
      const double o = __shfl_down_sync(0xffffffffu, v, off);
      if ((lane & (2 * off - 1)) == 0) v = dadd(v, o);
    }
  }
  return v;
}

__device__ __forceinline__ double2 ldcg2(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}

/// L2 prefetch of this CTA's slices of one basis vector (bulk, one thread).
__device__ __forceinline__ void prefetch_l2(const double* v, int64_t n, int64_t T, int epl,
                                            int64_t lane_base) {
  for (int k = 0; k < epl; ++k) {
    const int64_t s0 = lane_base + int64_t(k) * T;
    if (s0 >= n) break;
    const int64_t cnt = n - s0 < kSmemLanes ? n - s0 : kSmemLanes;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(v + s0),
                 "r"(unsigned(cnt) * 8u)
                 : "memory");
  }
}

__global__ void __launch_bounds__(kSmemThreads, 1)
    arnoldi_smem_kernel(int64_t n, int64_t T, int epl, int j, const double* __restrict__ wg,
                        const double* V, int64_t ldv, double* __restrict__ hcol,
                        unsigned long long* slot_tag, unsigned long long tag_base, double* vout) {
  extern __shared__ __align__(16) double2 wsm[];  // epl x kSmemThreads: lanes (2t, 2t+1)
  __shared__ double hsh;
  const int G = gridDim.x;
  const int tid = threadIdx.x;
  const int64_t lane_base = int64_t(blockIdx.x) * kSmemLanes;
  const int64_t lane0 = lane_base + 2 * tid;  // even; n even, so e < n covers the pair
  if (tid == 0) prefetch_l2(V, n, T, epl, lane_base);
  for (int k = 0; k < epl; ++k) {
    const int64_t e = lane0 + int64_t(k) * T;
    wsm[k * kSmemThreads + tid] = e < n ? ldcg2(wg + e) : make_double2(0.0, 0.0);
  }
  ulonglong2* pairs = reinterpret_cast<ulonglong2*>(slot_tag);
  double hprev = 0.0;
  for (int i = 0; i <= j + 1; ++i) {
    // v_{i+1} towards L2 while this pass computes and reduces
    if (tid == 0 && i + 1 <= j) prefetch_l2(V + int64_t(i + 1) * ldv, n, T, epl, lane_base);
    const double* vi = V + int64_t(i) * ldv;
    const double* vp = V + int64_t(i - 1) * ldv;
    double acc0 = 0.0, acc1 = 0.0;
    for (int k0 = 0; k0 < epl; k0 += kSmemBatch) {
      double2 a[kSmemBatch], b[kSmemBatch];
#pragma unroll
      for (int c = 0; c < kSmemBatch; ++c) {
        const int k = k0 + c;
        const int64_t e = lane0 + int64_t(k) * T;
        const bool ok = k < epl && e < n;
        a[c] = ok && i > 0 ? ldcg2(vp + e) : make_double2(0.0, 0.0);
        b[c] = ok && i <= j ? ldcg2(vi + e) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int c = 0; c < kSmemBatch; ++c) {
        const int k = k0 + c;
        const int64_t e = lane0 + int64_t(k) * T;
        if (k < epl && e < n) {
          double2 wv = wsm[k * kSmemThreads + tid];
          if (i > 0) {
            wv.x = dsub(wv.x, dmul(hprev, a[c].x));
            wv.y = dsub(wv.y, dmul(hprev, a[c].y));
            wsm[k * kSmemThreads + tid] = wv;
          }
          const double2 o = i <= j ? b[c] : wv;
          acc0 = dadd(acc0, dmul(wv.x, o.x));
          acc1 = dadd(acc1, dmul(wv.y, o.y));
        }
      }
    }
    const double cta = block_tree_1k(dadd(acc0, acc1), kSmemThreads);
    const int par = i & 1;
    const unsigned long long want = tag_base + unsigned(i) + 1ull;
    if (tid == 0) {
      const unsigned long long bits = __double_as_longlong(cta);
      st_pair(pairs + par * G + blockIdx.x, bits, bits ^ want);
    }
    // every CTA gathers all G pairs and rebuilds the same tree (a slot of
    // parity par is rewritten two passes later, after every CTA read it)
    double v = 0.0;
    if (tid < G) {
      ulonglong2 p;
      do {
        p = ld_pair(pairs + par * G + tid);
      } while ((p.x ^ p.y) != want);
      v = __longlong_as_double(p.x);
    }
    __syncthreads();  // warp 0 finished reading block_tree_1k's scratch of this pass
    v = block_tree_1k(v, G);
    if (tid == 0) {
      if (i == j + 1) v = __dsqrt_rn(v);
      hsh = v;
      if (blockIdx.x == 0) hcol[i] = v;
    }
    __syncthreads();
    hprev = hsh;
  }
  // v_{j+1} = w / h, or 0 on a happy breakdown (gmres.hpp:66-67)
  for (int k = 0; k < epl; ++k) {
    const int64_t e = lane0 + int64_t(k) * T;
    if (e < n) {
      const double2 wv = wsm[k * kSmemThreads + tid];
      double2 o;
      o.x = hprev > 0.0 ? __ddiv_rn(wv.x, hprev) : 0.0;
      o.y = hprev > 0.0 ? __ddiv_rn(wv.y, hprev) : 0.0;
      *reinterpret_cast<double2*>(vout + e) = o;
    }
  }
}

} // namespace

/// Cooperative single-launch Arnoldi step; returns false when the problem
/// does not fit the co-resident configuration (caller falls back to one
/// kernel per pass).
/// Tagged reduction slots of a G-CTA Arnoldi step: the pair layout uses
/// 2G + 2 16-byte slots (4G + 4 words, root CTA publication included), the
/// release/acquire layout 2G + 2 words; sized for the larger, never below
/// the historical 2048 words.
static void ensure_slot_tags(Context& c, int64_t G) {
  const size_t need = std::max<size_t>(2048, size_t(4 * G + 4));
  if (c.slot_tag.n < need) {
    c.slot_tag.alloc(need);
    PSCU_CUDA(cudaMemsetAsync(c.slot_tag.p, 0, sizeof(unsigned long long) * need, c.stream));
  }
}

bool arnoldi_step_fused(Context& c, int64_t n, int j, double* w, double* V, int64_t ldv,
                        double* hcol) {
  const int64_t T = repro_lanes(n);
  if (T < kStepThreads) return false;
  const int epl = int((n + T - 1) / T);
  if (epl > kEpt) return false;
  static int sm_count = 0;
  if (!sm_count)
    PSCU_CUDA(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, c.device));
  static const bool pairs = [] {
    const char* e = getenv("PSCU_MGS_PAIRS");
    return e ? atoi(e) != 0 : true;
  }();
  // all-gather reduction by default; the root-CTA variant (PSCU_MGS_ALL=0)
  // measured 537 vs 567 us per coarse step in isolation but equal within
  // noise over a whole solve (10.59 vs 10.51 s of Arnoldi steps)
  const char* ae = getenv("PSCU_MGS_ALL");
  const bool all = ae ? atoi(ae) != 0 : true;
  // TMA-staged basis: correct, but measured slower than the register-
  // prefetch kernel at the 256^2 coarse level (766 vs 567 us per step)
  const char* te = getenv("PSCU_MGS_TMA");
  const bool tma = te ? atoi(te) != 0 : false;
  // TMA staging once >= 64 CTAs share the stream (PSCU_MGS_TMA_MIN_G: tests)
  const char* mg = getenv("PSCU_MGS_TMA_MIN_G");
  const int64_t min_g = mg ? std::max(1, atoi(mg)) : 64;
  if (tma && (n % 2) == 0 && (ldv % 2) == 0 && T % kVLanes == 0 && T / kVLanes >= min_g &&
      T / kVLanes <= kStepThreads) {
    const int64_t G = T / kVLanes;
    const size_t smem = sizeof(double) * kVStages * size_t(epl) * kVLanes;
    static size_t attr_smem = 0;
    if (smem > attr_smem) {
      PSCU_CUDA(cudaFuncSetAttribute(arnoldi_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
      attr_smem = smem;
    }
    int per_sm = 0;
    PSCU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, arnoldi_tma_kernel,
                                                            kStepThreads, smem));
    if (int64_t(per_sm) * sm_count >= G) {
      ensure_slot_tags(c, G);
      int ei = epl, jj = j;
      int64_t nn = n, TT = T, ld = ldv;
      double* pw = w;
      const double* pV = V;
      double* ph = hcol;
      unsigned long long* pt = c.slot_tag.p;
      unsigned long long base = c.pass_tag;
      double* vo = V + int64_t(j + 1) * ldv;
      c.pass_tag += unsigned(j + 2);
      void* args[] = {&nn, &TT, &ei, &jj, &pw, &pV, &ld, &ph, &pt, &base, &vo};
      PSCU_CUDA(cudaLaunchCooperativeKernel((void*)arnoldi_tma_kernel, dim3(unsigned(G)),
                                            dim3(kStepThreads), args, smem, c.stream));
      PSCU_LAUNCHED(&c);
      return true;
    }
  }
  static const int max_lanes = [] {
    const char* e = getenv("PSCU_MGS_LANES");
    return e ? atoi(e) : 2;
  }();
  // PSCU_MGS_FORCE_SMEM=1 (tests): skip the register-resident kernels
  const char* fs = getenv("PSCU_MGS_FORCE_SMEM");
  const bool force_smem = fs && atoi(fs) != 0;
  // two lanes per thread when that keeps >= 64 CTAs (fewer participants per
  // grid-wide reduction) and the elements fit the kL = 2 register budget
  for (int L = (max_lanes >= 2 && T / (2 * kStepThreads) >= 64 && epl <= StepShape<2>::kE) ? 2 : 1;
       L >= 1 && !force_smem; L >>= 1) {
    const int64_t G = T / (int64_t(kStepThreads) * L);
    if (G < 1 || G > 1024) continue;
    const size_t smem = 0;
    int per_sm = 0;
    void* fn = L == 2 ? (pairs ? (all && G <= kStepThreads ? (void*)arnoldi_step_kernel<2, true, true>
                                                           : (void*)arnoldi_step_kernel<2, true>)
                               : (void*)arnoldi_step_kernel<2, false>)
                      : (pairs ? (all && G <= kStepThreads ? (void*)arnoldi_step_kernel<1, true, true>
                                                           : (void*)arnoldi_step_kernel<1, true>)
                               : (void*)arnoldi_step_kernel<1, false>);
    PSCU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kStepThreads, smem));
    if (int64_t(per_sm) * sm_count < G) continue;
    ensure_slot_tags(c, G);
    int ei = epl, jj = j;
    int64_t nn = n, TT = T, ld = ldv;
    double* pw = w;
    double* pV = V;
    double* ph = hcol;
    double* pv = c.red_partials.p;
    unsigned long long* pt = c.slot_tag.p;
    unsigned long long base = c.pass_tag;
    c.pass_tag += unsigned(j + 2);
    void* args[] = {&nn, &TT, &ei, &jj, &pw, &pV, &ld, &ph, &pv, &pt, &base};
#ifdef PSCU_TRACE
    static long long* tbuf = nullptr;
    if (getenv("PSCU_MGS_TRACE") && !tbuf) {
      PSCU_CUDA(cudaMalloc(&tbuf, sizeof(long long) * 4096));
      PSCU_CUDA(cudaMemcpyToSymbol(g_mgs_trace, &tbuf, sizeof(tbuf)));
    }
#endif
    PSCU_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(G)),
                                          dim3(kStepThreads), args, smem, c.stream));
    PSCU_LAUNCHED(&c);
#ifdef PSCU_TRACE
    if (tbuf && j >= 100 && j % 100 == 0) {
      std::vector<long long> h(4096);
      PSCU_CUDA(cudaMemcpyAsync(h.data(), tbuf, sizeof(long long) * 4096, cudaMemcpyDeviceToHost,
                                c.stream));
      PSCU_CUDA(cudaStreamSynchronize(c.stream));
      double d[4] = {0, 0, 0, 0};
      int cnt = 0;
      for (int i = 1; i + 1 <= j && i < 1000; ++i, ++cnt) {
        const long long* t = &h[size_t(i) * 4];
        d[0] += double(t[1] - t[0]);   // local compute + CTA tree
        d[1] += double(t[2] - t[1]);   // publish + gather all pairs
        d[2] += double(t[3] - t[2]);   // second tree + broadcast
        d[3] += double(h[size_t(i + 1) * 4] - t[0]);  // whole pass
      }
      fprintf(stderr, "[mgs trace j=%d L=%d] cycles/pass: compute+tree %.0f gather %.0f tree2 %.0f | pass %.0f\n",
              j, L, d[0] / cnt, d[1] / cnt, d[2] / cnt, d[3] / cnt);
    }
#endif
    return true;
  }
  // w in shared memory (coarse levels beyond the register budget)
  static const bool smem_ok = [] {
    const char* e = getenv("PSCU_MGS_SMEM");
    return e ? atoi(e) != 0 : true;
  }();
  if (smem_ok && (n % 2) == 0 && (ldv % 2) == 0 && T % kSmemLanes == 0 &&
      (reinterpret_cast<uintptr_t>(w) % 16) == 0 && (reinterpret_cast<uintptr_t>(V) % 16) == 0) {
    const int64_t G = T / kSmemLanes;
    const size_t smem = sizeof(double2) * size_t(epl) * kSmemThreads;
    if (G >= 1 && G <= sm_count && smem <= 220 * 1024) {
      static size_t attr_smem = 0;
      if (smem > attr_smem) {
        PSCU_CUDA(cudaFuncSetAttribute(arnoldi_smem_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr_smem = smem;
      }
      int per_sm = 0;
      PSCU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, arnoldi_smem_kernel,
                                                              kSmemThreads, smem));
      if (int64_t(per_sm) * sm_count >= G) {
        ensure_slot_tags(c, G);
        int ei = epl, jj = j;
        int64_t nn = n, TT = T, ld = ldv;
        const double* pw = w;
        const double* pV = V;
        double* ph = hcol;
        unsigned long long* pt = c.slot_tag.p;
        unsigned long long base = c.pass_tag;
        double* vo = V + int64_t(j + 1) * ldv;
        c.pass_tag += unsigned(j + 2);
        void* args[] = {&nn, &TT, &ei, &jj, &pw, &pV, &ld, &ph, &pt, &base, &vo};
        PSCU_CUDA(cudaLaunchCooperativeKernel((void*)arnoldi_smem_kernel, dim3(unsigned(G)),
                                              dim3(kSmemThreads), args, smem, c.stream));
        PSCU_LAUNCHED(&c);
        return true;
      }
    }
  }
  return false;
}

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
