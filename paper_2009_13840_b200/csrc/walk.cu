// Level-walking sparse triangular sweeps for Ilu0::apply (ilu0.hpp:53-65).
//
// The reference applies ILU(0) with two sequential loops. Under the natural
// (faces-first) ordering their dependency DAGs are deep and narrow: hundreds
// to thousands of levels of a few hundred rows, so any
// scheme that pays an inter-SM handshake through global memory per level is
// bound by ~1 us per level. Narrow levels are therefore walked by ONE thread
// block cluster of C CTAs (C = 1..8, chosen per sweep from the level width):
//   * rows are placed in level order; every level is cut into "sub-levels"
//     (at most C chunks of <= kStageRows rows / kMaxNz factor entries, one
//     chunk per CTA; rows of a level are independent, so any cut is valid);
//   * a chunk's operands are one contiguous, 16-byte-aligned block: the
//     factor entries it needs in the reference's summation order (value +
//     source), row ids, offsets, right-hand sides (gathered into position
//     order beforehand), diagonals (backward), out-of-ring source list;
//   * per CTA, warp-specialised producers stage chunks kStages ahead with TMA
//     bulk copies and gather the out-of-ring sources; consumers compute;
//   * solution values of recent rows live in per-CTA shared-memory rings;
//     a row reads sources computed by another CTA of the cluster through
//     DSMEM (ld.shared::cluster); sources older than the ring window come
//     from the producers' gather (they are >= 8 sub-levels old, i.e. final);
//   * one named barrier per sub-level inside a CTA, plus (C > 1) one
//     all-to-all mbarrier handshake over the cluster.
// Levels with very many rows (element-pressure rows) run as row-parallel
// launches between walker segments. Every row is computed by one thread with
// the reference's exact operation sequence, so the result is bit-identical
// to Ilu0::apply.
#include <algorithm>
#include <chrono>
#include <queue>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <thread>

#include <cooperative_groups.h>

#include <type_traits>

#include "internal.cuh"
#include "walk.cuh"

namespace pscu {

namespace {

constexpr int kWalkThreads = 512;  // consumer threads per CTA (one row each)
constexpr int kProdWarps = 4;      // producer warps per stage slot
constexpr int kProducers = 32 * kProdWarps * 4;
constexpr int kStageRows = 640;   // rows of a push-walker chunk (level walker: kWalkThreads)
constexpr int kMaxNz = 2048;       // factor entries of a chunk (multiple of 4)
constexpr int kStages = 3;         // chunks in flight per CTA
constexpr int kRing = 4096;        // per-CTA solution ring (local positions, power of 2)
constexpr int kWideRows = 4096;    // levels with more rows run row-parallel
constexpr int kMaxCluster = 8;
constexpr int kMaxDiag = 128;      // longest task (factor entries) of a walker chunk
constexpr int kHdr = 16;           // ints of a chunk header
constexpr int kLevelMaxNz = 512;   // entries of a task of a level-launch plan (warp kernel buffer)
constexpr int kLevelMaxRows = 32;  // rows of such a task
#ifndef PSCU_BSHFL_BLOCK
#define PSCU_BSHFL_BLOCK 4
#endif
#ifndef PSCU_FLOW_MID_CTAS
#define PSCU_FLOW_MID_CTAS 4
#endif
constexpr int kFlowSmallNz = 192;  // entry cap of the small-task dataflow kernel
constexpr int kFlowMidNz = 384;    // ... of the mid-task one (chains of a whole element's face blocks)
constexpr int kPadSrc = int(0x80000000);  // level plans: pad entry (product 0; acc - 0.0 == acc)

struct WalkArgs {
  const int32_t* sl_k;    // chunk start position (multiple of 4)
  const int32_t* sl_nr;   // rows of the chunk
  const int64_t* sl_q;    // packed entry start (multiple of 4), nchunks + 1
  const int32_t* sl_hdr;  // per chunk {k0, rows, entries, far, ring start, diagonals, dp start,
                          //  push bytes, tasks, task table start, 0...} (kHdr ints)
  const int32_t* tt;      // per chunk: first local row of every task, then the row count
  const int32_t* tq;      // wide chunks: entry offset of every task in the chunk, then the total
  const int32_t* rows;    // row id per position (-1 padding)
  const int32_t* off;     // walker chunks: row length; wide chunks: row offset in the chunk
  const int32_t* dp;      // walker chunks: start of diagonal u within the chunk
  const int4* meta;       // walker chunks, per position: {row length, row, backward position, 0}
  const int32_t* opos;    // forward: backward position of the row
  const double* val;      // packed factor values
  const int32_t* src;     // >= 0: (rank << 12) | ring slot, -1: out-of-ring source
  const double* dv;       // backward: diagonal per position
  const int64_t* sl_f;    // in-segment out-of-ring entries: list start per chunk (nchunks + 1)
  const int2* far;        // ... {entry offset in chunk, source row}
  const int64_t* sl_s;    // static out-of-ring entries (sources final before the launch)
  const int2* sfar;       // ... {entry offset in chunk, source row}
  const double* sfv;      // ... their source values, gathered before the launch
  long long* trace;       // PSCU_WALK_TRACE: per-sub-level clock64 stamps of CTA 0
  int spin_ns;            // dataflow sweeps: back-off between polls of a source (0: none)
  long long* ftrace;      // trace build, PSCU_FLOW_TRACE: per task 4 globaltimer stamps,
                          // fold cycles, lane-parallel fold flag
  int rotate;             // dataflow sweeps: rotate the task-to-warp assignment per level
  int lead;               // dataflow sweeps: wait on the task's latest source with one
                          // warp-uniform load before polling all sources (keeps the
                          // load/store unit free for the folding warps' LDS / SHFL)
  int far_ns;             // dataflow sweeps: extra back-off of warps missing > 8 lanes' sources
  int bfast;              // small-task dataflow sweeps, backward: lane-0 fold from dense
                          // products (8-entry blocks, row values in registers)
  int bshfl;              // small-task dataflow sweeps, backward: warp-replicated register fold
                          // fed by shuffles (needs rows padded to whole 8-entry blocks)
};

constexpr int kTraceSub = 4096;
// per-sub-level clock stamps: only in the instrumented build (build.py trace=True)
#ifdef PSCU_TRACE
#define WALK_TRACE(cond, r, k)                                       \
  do {                                                               \
    if (a.trace && (cond) && (r) < kTraceSub)                        \
      a.trace[((rank) * kTraceSub + (r)) * 16 + (k)] = clock64();    \
  } while (0)
#else
#define WALK_TRACE(cond, r, k) \
  do {                         \
  } while (0)
#endif

struct alignas(16) Stage {
  double val[kMaxNz];
  int32_t src[kMaxNz];
  double rhs[kStageRows];
  double dv[kStageRows];
  int4 meta[kStageRows];
  int32_t dptr[kMaxDiag];
  int32_t tt[kStageRows + 4];
  int32_t hdr[kHdr];
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return unsigned(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  if (bytes == 0) return;
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ unsigned map_rank(const void* p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

/// Stages chunk `ch` into `st` (one bulk copy per operand array).
template <bool kFwd>
__device__ void issue(const WalkArgs& a, int ch, Stage& st, uint64_t* bar, const double* rhs) {
  const int k0 = a.sl_k[ch], nr = a.sl_nr[ch];
  const unsigned nr4 = unsigned((nr + 3) & ~3);
  const int64_t q0 = a.sl_q[ch];
  const unsigned nq = unsigned(a.sl_q[ch + 1] - q0);
  const int* hd = a.sl_hdr + kHdr * ch;
  const unsigned nd4 = unsigned((hd[5] + 3) & ~3);
  const unsigned nt4 = unsigned((hd[8] + 1 + 3) & ~3);
  const unsigned bytes =
      nq * 12u + nr4 * (8u + 16u) + (kFwd ? 0u : nr4 * 8u) + nd4 * 4u + nt4 * 4u + 4u * kHdr;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  bulk_copy(st.hdr, a.sl_hdr + kHdr * ch, 4u * kHdr, bar);
  bulk_copy(st.tt, a.tt + hd[9], nt4 * 4u, bar);
  bulk_copy(st.val, a.val + q0, nq * 8u, bar);
  bulk_copy(st.src, a.src + q0, nq * 4u, bar);
  bulk_copy(st.rhs, rhs + k0, nr4 * 8u, bar);
  bulk_copy(st.meta, a.meta + k0, nr4 * 16u, bar);
  bulk_copy(st.dptr, a.dp + hd[6], nd4 * 4u, bar);
  if (!kFwd) bulk_copy(st.dv, a.dv + k0, nr4 * 8u, bar);
}

/// Products first (entry-parallel: every rounded product val * y is
/// independent; loads batched per thread, ring values of other CTAs through
/// DSMEM), then one thread per row folds its products in the reference's
/// order: the same rounded operations as the sequential loop. Out-of-ring
/// entries (src -1) already hold their product (producers).
template <bool kCluster>
__device__ __forceinline__ void walk_products(Stage& st, double* ring, int rank) {
  constexpr int kPer = (kMaxNz + kWalkThreads - 1) / kWalkThreads;
  const int nq = st.hdr[2];
  int sv[kPer];
  double pv[kPer], yv[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int q = threadIdx.x + u * kWalkThreads;
    sv[u] = q < nq ? st.src[q] : -1;
    pv[u] = q < nq ? st.val[q] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const double* p = ring + (sv[u] & (kRing - 1));
    if (kCluster && sv[u] >= 0 && (sv[u] >> 12) != rank)
      p = cooperative_groups::this_cluster().map_shared_rank(p, unsigned(sv[u] >> 12));
    yv[u] = *p;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int q = threadIdx.x + u * kWalkThreads;
    if (sv[u] >= 0) st.val[q] = dmul(pv[u], yv[u]);
  }
}

/// Entries sit diagonal-major (entry u of row t at dptr[u] + t): a warp's
/// fold loads are unit-stride, conflict-free.
/// Returns false for threads without a row; the caller stores acc to y (and
/// yb) after the sub-level's cluster handshake, whose release fence then
/// never waits on these global stores.
template <bool kFwd>
__device__ __forceinline__ bool walk_rows(const Stage& st, double& acc, int4& m) {
  const int nr = st.hdr[1];
  const int t = threadIdx.x;  // level-walker chunks: at most kWalkThreads rows, one per thread
  if (t >= nr) return false;
  m = st.meta[t];
  const int len = m.x;
  acc = st.rhs[t];
  for (int u0 = 0; u0 < len; u0 += 8) {
    const int4 d0 = *reinterpret_cast<const int4*>(st.dptr + u0);
    const int4 d1 = *reinterpret_cast<const int4*>(st.dptr + u0 + 4);
    const int d[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = u0 + u < len ? st.val[d[u] + t] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u0 + u < len) acc = dsub(acc, v[u]);
  }
  if (!kFwd) acc = __ddiv_rn(acc, st.dv[t]);
  return true;
}

/// Producer side (warp-specialised): group g of kWarps warps owns stage slot
/// g and stages sub-levels g, g + kS, ...: TMA bulk copies of the chunk, then
/// the products of its out-of-ring entries (static sources gathered into sfv
/// before the launch; in-segment ones >= 8 sub-levels old, complete since
/// every CTA finished sub-level r - kS). Thread index relative to the first
/// producer thread (kWalkThreads).
template <bool kFwd, int kS, int kWarps, int kFirst = kWalkThreads>
__device__ __forceinline__ void produce(const WalkArgs& a, int c0, int nsl, int C, unsigned rank,
                                        Stage* stages, uint64_t* landed, uint64_t* full,
                                        uint64_t* empty, const double* rhs, const double* y) {
  constexpr int kGroup = 32 * kWarps;
  const int pg = (threadIdx.x - kFirst) / kGroup;
  const int lane = (threadIdx.x - kFirst) % kGroup;
  const int slot = pg;
  for (int r = pg; r < nsl; r += kS) {
    const int ch = c0 + r * C + int(rank);
    const unsigned ph = unsigned((r / kS) & 1);
    WALK_TRACE(lane == 0, r, 8);
    if (r >= kS) mbar_wait(&empty[slot], ph ^ 1u);
    WALK_TRACE(lane == 0, r, 9);
    if (lane == 0) issue<kFwd>(a, ch, stages[slot], &landed[slot], rhs);
    const int64_t s0 = a.sl_s[ch], ns = a.sl_s[ch + 1] - s0;
    const int64_t f0 = a.sl_f[ch], nf = a.sl_f[ch + 1] - f0;
    double* val = stages[slot].val;
    mbar_wait(&landed[slot], ph);
    WALK_TRACE(lane == 0, r, 10);
    for (int64_t base = 0; base < ns; base += 8 * kGroup) {
      int off[8];
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t f = base + u * kGroup + lane;
        off[u] = f < ns ? __ldg(&a.sfar[s0 + f].x) : -1;
        v[u] = f < ns ? __ldg(a.sfv + s0 + f) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (off[u] >= 0) val[off[u]] = dmul(val[off[u]], v[u]);
    }
    for (int64_t base = 0; base < nf; base += 4 * kGroup) {
      int2 e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t f = base + u * kGroup + lane;
        e[u] = f < nf ? __ldg(a.far + f0 + f) : make_int2(-1, 0);
      }
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = e[u].x >= 0 ? __ldcg(y + e[u].y) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (e[u].x >= 0) val[e[u].x] = dmul(val[e[u].x], v[u]);
    }
    asm volatile("bar.sync %0, %1;" ::"r"(2 + pg), "n"(kGroup) : "memory");
    WALK_TRACE(lane == 0, r, 11);
    if (lane == 0) mbar_arrive(&full[slot]);
  }
}

/// CTA `rank` of a C-CTA cluster walks chunks c0 + rank, c0 + rank + C, ...
/// (one chunk per sub-level). Consumers: kWalkThreads threads; producers:
/// kProdWarps warps per stage slot, which stage the chunk (TMA) and then
/// turn its out-of-ring entries into products from global memory.
template <bool kFwd>
__global__ void __launch_bounds__(kWalkThreads + kProducers, 1)
    walk_kernel(WalkArgs a, int c0, int nsl, int C, const double* rhs, double* y, double* yb) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ __align__(8) uint64_t landed[kStages], full[kStages], empty[kStages], level[2];
  double* ring = reinterpret_cast<double*>(smraw);
  Stage* stages = reinterpret_cast<Stage*>(smraw + sizeof(double) * kRing);
  const unsigned rank = C > 1 ? cluster_rank() : 0u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&landed[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&empty[i])) : "memory");
    }
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&level[i])), "r"(C)
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (C > 1) cluster_sync_all();
  else __syncthreads();
  if (threadIdx.x >= kWalkThreads) {
    produce<kFwd, kStages, kProdWarps>(a, c0, nsl, C, rank, stages, landed, full, empty, rhs, y);
  } else {
    for (int r = 0; r < nsl; ++r) {
      const int slot = r % kStages;
      Stage& st = stages[slot];
      WALK_TRACE(threadIdx.x == 0, r, 0);
      mbar_wait(&full[slot], unsigned((r / kStages) & 1));
      WALK_TRACE(threadIdx.x == 0, r, 1);
      if (C > 1) walk_products<true>(st, ring, int(rank));
      else walk_products<false>(st, ring, 0);
      asm volatile("bar.sync 1, %0;" ::"n"(kWalkThreads) : "memory");
      WALK_TRACE(threadIdx.x == 0, r, 2);
      double acc;
      int4 m;
      const bool mine = walk_rows<kFwd>(st, acc, m);
      if (mine) ring[(st.hdr[4] + int(threadIdx.x)) & (kRing - 1)] = acc;
      asm volatile("bar.sync 1, %0;" ::"n"(kWalkThreads) : "memory");
      WALK_TRACE(threadIdx.x == 0, r, 3);
      if (C > 1) {
        // all-to-all: this CTA's ring entries of sub-level r are published
        // (release) to every CTA; wait until every CTA has published (acquire)
        if (threadIdx.x < unsigned(C)) {
          const unsigned remote = map_rank(&level[r & 1], threadIdx.x);
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
                       : "memory");
        }
        mbar_wait_cluster(&level[r & 1], unsigned((r >> 1) & 1));
      }
      WALK_TRACE(threadIdx.x == 0, r, 4);
      if (mine) {
        y[m.y] = acc;
        if (kFwd) yb[m.z] = acc;
      }
      if (threadIdx.x == 0) mbar_arrive(&empty[slot]);
    }
  }
  // no CTA may leave while its ring can still be read remotely
  if (C > 1) cluster_sync_all();
}

// ---------------------------------------------------------------------------
// Dataflow walker (one CTA): no per-level barrier. Chunks are consecutive
// rows in level order (spanning levels); every row waits only for its own
// sources, published in a shared-memory ring as self-validating 16-byte pairs
// {value bits, value bits ^ tag(position)} -- a reader accepts a slot when
// the pair carries its source's tag, so neither side needs a fence and a
// stale or torn slot is never used. Consumer threads run at most two chunks
// apart (each waits for chunk i - 2 to complete before starting chunk i), so
// a slot is rewritten (position + kRing) only after all of its readers ran.
// ---------------------------------------------------------------------------

constexpr int kFlowStages = 3;
#ifndef PSCU_FLOW_BACKOFF
#define PSCU_FLOW_BACKOFF 64
#endif
constexpr unsigned kFlowBackoff = PSCU_FLOW_BACKOFF;

__device__ __forceinline__ unsigned long long flow_tag(int pos) {
  return (unsigned long long)(unsigned(pos) + 1ull) * 0x9E3779B97F4A7C15ull;
}

__device__ __forceinline__ void ring_put(ulonglong2* slot, double v, int pos) {
  const unsigned long long b = __double_as_longlong(v);
  asm volatile("st.volatile.shared.v2.u64 [%0], {%1, %2};" ::"r"(smem_addr(slot)), "l"(b),
               "l"(b ^ flow_tag(pos))
               : "memory");
}

__device__ __forceinline__ double ring_get(const ulonglong2* slot, int pos) {
  const unsigned long long want = flow_tag(pos);
  unsigned long long x, y;
  for (;;) {
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y)
                 : "r"(smem_addr(slot))
                 : "memory");
    if ((x ^ y) == want) break;
    __nanosleep(kFlowBackoff);  // leave the shared-memory pipe to the rows being computed
  }
  return __longlong_as_double(x);
}

template <bool kFwd>
__global__ void __launch_bounds__(kWalkThreads + 64 * kFlowStages, 1)
    flow_kernel(WalkArgs a, int c0, int nch, const double* rhs, double* y, double* yb) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ __align__(8) uint64_t landed[kFlowStages], full[kFlowStages], empty[kFlowStages];
  ulonglong2* ring = reinterpret_cast<ulonglong2*>(smraw);
  Stage* stages = reinterpret_cast<Stage*>(smraw + sizeof(ulonglong2) * kRing);
  const unsigned rank = 0;  // WALK_TRACE
  for (int i = threadIdx.x; i < kRing; i += blockDim.x) ring[i] = make_ulonglong2(0ull, 0ull);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kFlowStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&landed[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&empty[i])),
                   "r"(kWalkThreads)
                   : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= kWalkThreads) {
    // producer pair of warps g owns slot g: chunks g, g + kFlowStages, ...
    constexpr int kGroup = 64;
    const int pg = (threadIdx.x - kWalkThreads) / kGroup;
    const int lane = (threadIdx.x - kWalkThreads) % kGroup;
    const int slot = pg;
    for (int r = pg; r < nch; r += kFlowStages) {
      const int ch = c0 + r;
      const unsigned ph = unsigned((r / kFlowStages) & 1);
      WALK_TRACE(lane == 0, r, 8);
      if (r >= kFlowStages) mbar_wait(&empty[slot], ph ^ 1u);
      WALK_TRACE(lane == 0, r, 9);
      if (lane == 0) issue<kFwd>(a, ch, stages[slot], &landed[slot], rhs);
      // out-of-ring sources: static ones were gathered before this launch;
      // in-segment ones lie >= 5 chunks back, complete since every consumer
      // finished chunk r - kFlowStages
      const int64_t s0 = a.sl_s[ch], ns = a.sl_s[ch + 1] - s0;
      const int64_t f0 = a.sl_f[ch], nf = a.sl_f[ch + 1] - f0;
      double* val = stages[slot].val;
      mbar_wait(&landed[slot], ph);
      WALK_TRACE(lane == 0, r, 10);
      for (int64_t base = 0; base < ns; base += 8 * kGroup) {
        int off[8];
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t f = base + u * kGroup + lane;
          off[u] = f < ns ? __ldg(&a.sfar[s0 + f].x) : -1;
          v[u] = f < ns ? __ldg(a.sfv + s0 + f) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (off[u] >= 0) val[off[u]] = dmul(val[off[u]], v[u]);
      }
      for (int64_t base = 0; base < nf; base += 4 * kGroup) {
        int2 e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t f = base + u * kGroup + lane;
          e[u] = f < nf ? __ldg(a.far + f0 + f) : make_int2(-1, 0);
        }
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = e[u].x >= 0 ? __ldcg(y + e[u].y) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e[u].x >= 0) val[e[u].x] = dmul(val[e[u].x], v[u]);
      }
      asm volatile("bar.sync %0, %1;" ::"r"(2 + pg), "n"(kGroup) : "memory");
      WALK_TRACE(lane == 0, r, 11);
      if (lane == 0) mbar_arrive(&full[slot]);
    }
  } else {
    const int t = threadIdx.x;
    for (int r = 0; r < nch; ++r) {
      const int slot = r % kFlowStages;
      WALK_TRACE(t == 0, r, 0);
      if (r >= 2) {
        // bounded skew: chunk r - 2 complete (its ring slots may be reused)
        const int r2 = r - 2;
        mbar_wait(&empty[r2 % kFlowStages], unsigned((r2 / kFlowStages) & 1));
      }
      mbar_wait(&full[slot], unsigned((r / kFlowStages) & 1));
      WALK_TRACE(t == 0, r, 1);
      WALK_TRACE(t == 0, r, 2);
      const Stage& st = stages[slot];
      const int nr = st.hdr[1];
      if (t < nr) {
        const int4 m = st.meta[t];
        const int len = m.x;
        double acc = st.rhs[t];
        for (int u0 = 0; u0 < len; u0 += 8) {
          int sv[8];
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const bool ok = u0 + u < len;
            const int e = ok ? st.dptr[u0 + u] + t : 0;
            sv[u] = ok ? st.src[e] : -1;
            v[u] = ok ? st.val[e] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (u0 + u < len) {
              const double p = sv[u] >= 0 ? dmul(v[u], ring_get(ring + (sv[u] & (kRing - 1)), sv[u]))
                                          : v[u];
              acc = dsub(acc, p);
            }
          }
        }
        if (!kFwd) acc = __ddiv_rn(acc, st.dv[t]);
        const int pos = st.hdr[4] + t;
        ring_put(ring + (pos & (kRing - 1)), acc, pos);
        y[m.y] = acc;
        if (kFwd) yb[m.z] = acc;
      }
      WALK_TRACE(t == 0, r, 3);
      WALK_TRACE(t == 0, r, 4);
      mbar_arrive(&empty[slot]);
    }
  }
}

// ---------------------------------------------------------------------------
// Push walker (cluster of C CTAs, sweeps without in-segment out-of-ring
// sources): every CTA keeps a replica of all C rings (kRingTotal / C recent
// positions per owner) and pushes each row it computes into every peer's
// replica with st.async, completing the peer's per-sub-level mbarrier. A
// sub-level then waits only for the bytes of the previous one to land: no
// release fences, and every ring read is local.
// ---------------------------------------------------------------------------

constexpr int kRingTotal = 8192;  // replicated ring slots (all owners)
constexpr int kSide = 2048;       // long-range slots: values read beyond the ring window
constexpr int kPushStages = 3;
constexpr int kPushProdWarps = 4;

__device__ __forceinline__ void push_value(unsigned raddr, double v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                   raddr),
               "d"(v), "r"(rbar)
               : "memory");
}

#ifndef PSCU_BULK_PUSH
#define PSCU_BULK_PUSH 1
#endif
constexpr bool kBulkPush = PSCU_BULK_PUSH != 0;

/// smem -> peer smem bulk copy completing the peer's mbarrier.
__device__ __forceinline__ void bulk_dsmem(unsigned dst, unsigned src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "r"(src), "r"(bytes), "r"(bar)
      : "memory");
}

constexpr int kPushConsumers = 256;  // consumer threads (default; 512 selectable)

/// One row of the push walker: acc = rhs - sum_u val_u * y(src_u), u
/// ascending (the reference's order and rounding), sources read from the
/// local ring replica; out-of-ring entries (src -1) already hold their
/// product (producers). Diagonal-major entries: unit-stride warp loads.
template <bool kFwd>
__device__ __forceinline__ double push_row(const Stage& st, const double* ring, int task, int u0,
                                           int row, const int4& m) {
  const int len = m.x;
  const int32_t* dp = st.dptr + u0;
  double acc = st.rhs[row];
  int u = 0;
  for (; u + 4 <= len; u += 4) {
    int e[4], sv[4];
    double v[4], w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) e[k] = dp[u + k] + task;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      sv[k] = st.src[e[k]];
      v[k] = st.val[e[k]];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = ring[sv[k] >= 0 ? sv[k] : 0];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc = dsub(acc, sv[k] >= 0 ? dmul(v[k], w[k]) : v[k]);
  }
  for (; u < len; ++u) {
    const int e = dp[u] + task;
    const int sv = st.src[e];
    const double v = st.val[e];
    acc = dsub(acc, sv >= 0 ? dmul(v, ring[sv]) : v);
  }
  if (!kFwd) acc = __ddiv_rn(acc, st.dv[row]);
  return acc;
}

template <bool kFwd, int kCons = kPushConsumers>
__global__ void __launch_bounds__(kCons + 32 * kPushProdWarps * kPushStages, 1)
    push_kernel(WalkArgs a, int c0, int nsl, int C, int S, const double* rhs, double* y,
                double* yb) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ __align__(8) uint64_t landed[kPushStages], full[kPushStages], empty[kPushStages],
      recv[2];
  double* ring = reinterpret_cast<double*>(smraw);  // kRingTotal ring + kSide long-range slots
  Stage* stages = reinterpret_cast<Stage*>(smraw + sizeof(double) * (kRingTotal + kSide));
  const unsigned rank = cluster_rank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPushStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&landed[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&empty[i])) : "memory");
    }
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&recv[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();
  if (threadIdx.x >= kCons) {
    produce<kFwd, kPushStages, kPushProdWarps, kCons>(a, c0, nsl, C, rank, stages,
                                                               landed, full, empty, rhs, y);
  } else {
    const int t = threadIdx.x;
    for (int r = 0; r < nsl; ++r) {
      const int slot = r % kPushStages;
      WALK_TRACE(t == 0, r, 0);
      mbar_wait(&full[slot], unsigned((r / kPushStages) & 1));
      const Stage& st = stages[slot];
      if (t == 0) {
        // bytes the peers push during this sub-level (they may land first:
        // the transaction count goes negative until this arrive)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_addr(&recv[r & 1])),
                     "r"(unsigned(st.hdr[7]))
                     : "memory");
      }
      if (r > 0) mbar_wait(&recv[(r - 1) & 1], unsigned(((r - 1) >> 1) & 1));
      WALK_TRACE(t == 0, r, 1);
      WALK_TRACE(t == 0, r, 2);
      const int nt = st.hdr[8], r0 = st.hdr[4];
      const unsigned rbar = smem_addr(&recv[r & 1]);
      // one task (a chain of rows, folded in order) per thread; a row reads
      // its task's earlier rows from this thread's own ring writes
      for (int task = t; task < nt; task += kCons) {
        const int re = st.tt[task + 1];
        int u0 = 0;
        for (int row = st.tt[task]; row < re; ++row) {
          const int4 m = st.meta[row];
          const double acc = push_row<kFwd>(st, ring, task, u0, row, m);
          WALK_TRACE(t == 0 && row == st.tt[0], r, 5);
          u0 += m.x;
          const int pos = r0 + row;
          double* own = ring + int(rank) * S + (pos & (S - 1));
          *own = acc;
          // a value read beyond the ring window also goes to its long-range slot
          if (m.w) ring[kRingTotal + m.w - 1] = acc;
          if (kBulkPush) {
            // ring slots reach the peers in one bulk copy per peer after the
            // sub-level barrier; only long-range copies go out per row
            if (m.w)
              for (int o = 0; o < C; ++o) {
                if (o == int(rank)) continue;
                unsigned ra, rb;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra)
                             : "r"(smem_addr(ring + kRingTotal + m.w - 1)), "r"(o));
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(rbar), "r"(o));
                push_value(ra, acc, rb);
              }
          } else {
            for (int o = 0; o < C; ++o) {
              if (o == int(rank)) continue;
              unsigned ra, rb;
              asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(own)), "r"(o));
              asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(rbar), "r"(o));
              push_value(ra, acc, rb);
              if (m.w) {
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra)
                             : "r"(smem_addr(ring + kRingTotal + m.w - 1)), "r"(o));
                push_value(ra, acc, rb);
              }
            }
          }
          WALK_TRACE(t == 0 && row == st.tt[0], r, 6);
          y[m.y] = acc;
          if (kFwd) yb[m.z] = acc;
        }
      }
      WALK_TRACE(t == 0, r, 7);
      // ring reads (generic proxy) ordered before peers' st.async rewrite
      // the slots; the sub-level's own ring writes visible to all consumers
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory");
      if (kBulkPush && t < C && t != int(rank)) {
        // this sub-level's ring slots [r0, r0 + nr) of this owner, rounded to
        // whole 16-byte pairs (positions are 4-aligned; the pad slot is never
        // read), to peer t's replica: one or two bulk DSMEM copies
        const int nr = st.hdr[1];
        const int b0 = r0 & (S - 1);
        const int n2 = (nr + 1) & ~1;
        const int first = b0 + n2 <= S ? n2 : S - b0;
        const unsigned rb = map_rank(&recv[r & 1], unsigned(t));
        const double* src = ring + int(rank) * S;
        if (first > 0)
          bulk_dsmem(map_rank(src + b0, unsigned(t)), smem_addr(src + b0), unsigned(first) * 8u, rb);
        if (n2 > first)
          bulk_dsmem(map_rank(src, unsigned(t)), smem_addr(src), unsigned(n2 - first) * 8u, rb);
      }
      WALK_TRACE(t == 0, r, 3);
      WALK_TRACE(t == 0, r, 4);
      if (t == 0) mbar_arrive(&empty[slot]);
    }
    // the last sub-level's pushes must land before any CTA leaves
    if (nsl > 0) mbar_wait(&recv[(nsl - 1) & 1], unsigned(((nsl - 1) >> 1) & 1));
  }
  cluster_sync_all();
}

/// Task-parallel chunk (a level too wide for one CTA): one thread per task
/// (a chain of rows folded in order), global sources; a source inside the
/// task (src >= 0: its index within the task) was written by this thread.
template <bool kFwd>
__global__ void wide_kernel(WalkArgs a, int ch, const double* rhs, double* y, double* yb) {
  const int k0 = a.sl_k[ch], nr = a.sl_nr[ch];
  const int64_t q0 = a.sl_q[ch];
  const int* hd = a.sl_hdr + kHdr * ch;
  const int nq = hd[2], nt = hd[8];
  const int32_t* tt = a.tt + hd[9];
  for (int task = int(blockIdx.x * blockDim.x + threadIdx.x); task < nt;
       task += gridDim.x * blockDim.x) {
    const int r0 = tt[task], r1 = tt[task + 1];
    for (int t = r0; t < r1; ++t) {
      const int k = k0 + t;
      const int64_t qa = q0 + a.off[k];
      const int64_t qb = q0 + (t + 1 < nr ? a.off[k + 1] : nq);
      double acc = rhs[k];
      for (int64_t q = qa; q < qb; ++q) {
        const int sv = a.src[q];
        if (sv == kPadSrc) continue;  // pad entry: acc - 0.0 == acc
        const int jr = sv < 0 ? -sv - 1 : a.rows[k0 + r0 + sv];
        acc = dsub(acc, dmul(a.val[q], __ldcg(y + jr)));
      }
      if (!kFwd) acc = __ddiv_rn(acc, a.dv[k]);
      y[a.rows[k]] = acc;
      if (kFwd) yb[a.opos[k]] = acc;
    }
  }
}

/// The same with one warp per task (long chains of the fine levels): the
/// lanes load the task's entries (row-contiguous, coalesced) and form every
/// product whose source lies outside the task, then lane 0 folds the rows in
/// order from shared memory (products of in-task sources use the values it
/// just computed). Same rounded operations as ilu0.hpp:53-65.
constexpr int kLevelWarps = 4;
#ifndef PSCU_FOLD_AHEAD
#define PSCU_FOLD_AHEAD 4
#endif
constexpr int kFoldAhead = PSCU_FOLD_AHEAD;  // look-ahead of the pipelined task fold

/// Dataflow sweeps (level_flow_kernel): y starts filled with a signalling-NaN
/// sentinel (arithmetic never produces it), every row's result is published
/// by its 8-byte store and a reader of an out-of-task source spins until the
/// value is no longer the sentinel — no grid barrier between task levels.
constexpr unsigned long long kFlowSentinel = 0xFFF7DEADBEEF5A5Aull;

__device__ __forceinline__ unsigned long long flow_peek(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void flow_store(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

/// The same without the compiler-level memory clobber (the value is the only
/// dependence a reader needs; lets shared-memory loads stay in flight across it).
__device__ __forceinline__ void flow_store_nc(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v));
}

__device__ __forceinline__ void flow_store_if(double* p, double v, bool on) {
  asm volatile(
      "{ .reg .pred q; setp.ne.s32 q, %2, 0; @q st.relaxed.gpu.global.f64 [%0], %1; }" ::"l"(p),
      "d"(v), "r"(int(on))
      : "memory");
}

__global__ void fill_sentinel(int64_t n, double* y) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __longlong_as_double((long long)kFlowSentinel);
}

/// acc - r[0].x - r[1].x - ... - r[cnt-1].x in that order (the
/// out-of-task part of a row: products only), operands loaded four ahead.
__device__ __forceinline__ double chain_sub(double acc, const double2* r, int cnt) {
  double nx[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) nx[k] = k < cnt ? r[k].x : 0.0;
  int e = 0;
  for (; e + 4 <= cnt; e += 4) {
    double cur[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cur[k] = nx[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) nx[k] = e + 4 + k < cnt ? r[e + 4 + k].x : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) acc = dsub(acc, cur[k]);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (e + k < cnt) acc = dsub(acc, nx[k]);
  return acc;
}

template <bool kFwd, bool kPdl, bool kFlow = false, int kMaxNz = kLevelMaxNz>
__device__ __forceinline__ void level_chunk(const WalkArgs& a, int ch, const double* rhs, double* y,
                                            double* yb) {
  constexpr int kPer = kMaxNz / 32;  // entries per lane
  // per entry {product or factor value, in-task source index or < 0}: one
  // 16-byte shared-memory load per entry in the fold
  __shared__ double2 rec[kLevelWarps][kMaxNz];
  __shared__ double rb[kLevelWarps][kLevelMaxRows], dvb[kLevelWarps][kLevelMaxRows],
      cv[kLevelWarps][kLevelMaxRows];
  __shared__ int4 mb[kLevelWarps][kLevelMaxRows];
  __shared__ int2 rinfo[kLevelWarps][kLevelMaxRows];  // per row {entry offset, leading in-task}
  const int k0 = a.sl_k[ch], nr = a.sl_nr[ch];
  const int64_t q0 = a.sl_q[ch];
  const int* hd = a.sl_hdr + kHdr * ch;
  const int nq = hd[2], nt = hd[8];
  const int32_t* tt = a.tt + hd[9];
  const int32_t* tq = a.tq + hd[9];
  const int w = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  // programmatic dependent launch: the next level's grid may start now; it
  // loads its static plan data while this level finishes, then waits for
  // this grid (griddepcontrol.wait) before touching right-hand sides and y
  if (kPdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  bool waited = !kPdl;
  // dataflow sweeps may rotate the task-to-warp assignment by the running
  // task count (hd[10]), so consecutive levels start on different warps
  const int Wg = int(gridDim.x) * kLevelWarps;
  int first = int(blockIdx.x) * kLevelWarps + w;
  if (kFlow && a.rotate) {
    first -= hd[11];  // running task count modulo the grid's warps (host-reduced)
    if (first < 0) first += Wg;
  }
  for (int task = first; task < nt; task += Wg) {
    // one round trip for the task record, one for its rows and entries
    // (both static), one for the sources outside the task
#ifdef PSCU_TRACE
    const bool tr = a.trace && task == 0 && lane == 0 && ch < kTraceSub;
    if (tr) a.trace[size_t(ch) * 16 + 0] = clock64();
    // every task of chunk 100: globaltimer at start and end (spread of a level)
    const bool tr2 = a.trace && ch == 100 && lane == 0 && task < 8192;
    unsigned long long gt0 = 0;
    if (tr2) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
#endif
#ifdef PSCU_TRACE
    unsigned long long fts[4] = {0, 0, 0, 0};
    long long fc0 = 0;
    if (kFlow && a.ftrace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[0]));
#endif
    const int r0 = tt[task], r1 = tt[task + 1];
    const int e0 = tq[task], ne = tq[task + 1] - e0;
    const int64_t qa = q0 + e0;
    int sv[kPer];
    double v[kPer], yv[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = lane + 32 * u;
      sv[u] = e < ne ? __ldg(a.src + qa + e) : 0;
      v[u] = e < ne ? __ldg(a.val + qa + e) : 0.0;
    }
    const unsigned full = 0xffffffffu;
    const int nrows = r1 - r0;
    // Row data: every lane loads (lanes past the task's rows re-read row 0)
    // so the prologue has no divergent branch around a global load. A lane
    // group split off here is not merged again by __syncwarp, and the
    // shuffle folds below then run as rendezvous of diverged groups
    // (measured: 4 of 32 lanes converged at the fold, 50x slower shuffles).
    const bool rowl = lane < nrows;
    const int lr = rowl ? lane : 0;
    const int krow = k0 + r0 + lr;
    const bool more = r0 + lr + 1 < nr;
    const int off0 = a.off[krow], off1 = a.off[krow + (more ? 1 : 0)];
    const int rid = a.rows[krow];
    const int opz = kFwd ? a.opos[krow] : 0;
    const double dvr0 = kFwd ? 1.0 : a.dv[krow];
    const int rlen = rowl ? (more ? off1 : nq) - off0 : 0;
    const int rowid = rowl ? rid : 0;
    const double dvl = rowl ? dvr0 : 1.0;
    // (every lane stores its slot, rows or not: kLevelMaxRows = 32 slots)
    mb[w][lane] = make_int4(rlen, rowid, opz, 0);
    if (!kFwd) dvb[w][lane] = dvl;
    // static row structure, found while the sources are still in flight:
    // lane r < nrows locates row r's in-task entries (sources inside the
    // task) among its out-of-task ones. Forward face-block rows have them
    // trailing (lane-parallel fold), backward rows leading (lane 0 folds the
    // leading in-task terms, then the rest as a pure product chain).
    int roff = rlen;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(full, roff, d);
      if (lane >= d) roff += t;
    }
    roff -= rlen;
    int fin = rlen, lin = -1, fout = rlen, lout = -1;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = lane + 32 * u;
      const unsigned bi = __ballot_sync(full, e < ne && sv[u] >= 0);
      const unsigned bo = __ballot_sync(full, e < ne && sv[u] < 0 && sv[u] != kPadSrc);
      const int lo = max(roff, 32 * u), hi = min(roff + rlen, 32 * u + 32);
      // (selects, no branches: see the note on divergence above)
      const bool act = rowl && lo < hi;
      const int b0 = act ? lo - 32 * u : 0, b1 = act ? hi - 32 * u : 0;
      const unsigned m = act ? ((b1 == 32 ? full : ((1u << b1) - 1u)) & ~((1u << b0) - 1u)) : 0u;
      const unsigned mi = bi & m, mo = bo & m;
      const int fi = 32 * u + __ffs(int(mi)) - 1 - roff, li = 32 * u + 31 - __clz(int(mi)) - roff;
      const int fo = 32 * u + __ffs(int(mo)) - 1 - roff, lo2 = 32 * u + 31 - __clz(int(mo)) - roff;
      fin = mi ? min(fin, fi) : fin;
      lin = mi ? max(lin, li) : lin;
      fout = mo ? min(fout, fo) : fout;
      lout = mo ? max(lout, lo2) : lout;
    }
    const bool trail_ok = __all_sync(full, lane >= nrows || lout < fin);
    const bool lead_ok = __all_sync(full, lane >= nrows || lin < fout);
    rinfo[w][lane] = make_int2(roff, lin + 1);
    // backward sweeps: the whole row header in one 16-byte slot
    if (!kFwd) mb[w][lane] = make_int4(rlen, rowid, roff, lin + 1);
    if (!waited) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
    }
    const double rbl0 = __ldcg(rhs + krow);
    const double rbl = rowl ? rbl0 : 0.0;
    rb[w][lane] = rbl;
#ifdef PSCU_TRACE
    if (kFlow && a.ftrace) {
      // the static loads have landed once their values are consumed
      int chk = 0;
#pragma unroll
      for (int u = 0; u < kPer; ++u) chk += sv[u] + int(v[u] != 0.0);
      chk = __reduce_add_sync(0xffffffffu, chk);
      if (lane == 0 && chk != 0x7fffffff) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[1]));
    }
#endif
    if (kFlow) {
      // all source values requested at once (one round trip), then only the
      // ones still holding the sentinel are polled again
      if (a.lead) {
        // The source expected last (the nearest row: highest index in a
        // forward sweep, lowest in a backward one) is awaited first, by one
        // load of one address per round for the whole warp: 27 of an SM's 28
        // warps are waiting at any time, and their per-lane polls otherwise
        // fill the load/store unit the folding warps' shared-memory loads
        // and shuffles go through (measured ~45 cycles per LDS / SHFL).
        int jd = kFwd ? -1 : 0x7fffffff;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int e = lane + 32 * u;
          const bool out = e < ne && sv[u] < 0 && sv[u] != kPadSrc;
          const int j = -sv[u] - 1;
          if (out) jd = kFwd ? max(jd, j) : min(jd, j);
        }
        jd = kFwd ? __reduce_max_sync(0xffffffffu, jd) : __reduce_min_sync(0xffffffffu, jd);
        if (jd >= 0 && jd != 0x7fffffff)
          while (flow_peek(y + jd) == kFlowSentinel)
            if (a.spin_ns) __nanosleep(a.spin_ns);
      }
      unsigned long long raw[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = lane + 32 * u;
        const bool out = e < ne && sv[u] < 0 && sv[u] != kPadSrc;
        raw[u] = out ? flow_peek(y + (-sv[u] - 1)) : 0ull;
      }
      // re-poll every still-unpublished source in the same round (one round
      // trip per round, not one per source; spinning on one source at a
      // time measured 35 % slower at config 5)
      for (;;) {
        bool pending = false;
#pragma unroll
        for (int u = 0; u < kPer; ++u) pending = pending || raw[u] == kFlowSentinel;
        // warp-uniform exit: lanes leaving the loop one by one stay split
        // into separately scheduled groups afterwards (measured: 4 of 32
        // lanes converged at the fold), which turns every later warp shuffle
        // into a rendezvous
        const unsigned waiting = __ballot_sync(0xffffffffu, pending);
        if (!waiting) break;
        if (a.spin_ns) __nanosleep(a.spin_ns);
        // a warp still missing many sources runs levels ahead of the sweep
        // front: it polls more slowly (PSCU_FLOW_FAR_NS, default 300 ns)
        if (a.far_ns && __popc(waiting) > 8) __nanosleep(a.far_ns);
#pragma unroll
        for (int u = 0; u < kPer; ++u)
          if (raw[u] == kFlowSentinel) raw[u] = flow_peek(y + (-sv[u] - 1));
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = lane + 32 * u;
        const bool out = e < ne && sv[u] < 0 && sv[u] != kPadSrc;
        yv[u] = out ? __longlong_as_double((long long)raw[u]) : 0.0;
      }
    } else {
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = lane + 32 * u;
        const bool out = e < ne && sv[u] < 0 && sv[u] != kPadSrc;
        yv[u] = out ? __ldcg(y + (-sv[u] - 1)) : 0.0;
      }
    }
    if (kFlow && kFwd && kMaxNz == kFlowSmallNz && a.bfast && trail_ok && nrows > 1 && nrows <= 4) {
      // Forward face-block tasks from dense products: lane r folds row r's
      // out-of-task prefix in 8-entry blocks (128-bit loads, one block ahead,
      // every lane the same trip count with the surplus steps selected away),
      // its trailing in-task terms (at most three: earlier rows of the task)
      // wait in registers and take the rows' values through three shuffles.
      // Each row's operations in column order, one rounding each: bitwise.
      double* prod = reinterpret_cast<double*>(&rec[w][0]);
      int* srcs = reinterpret_cast<int*>(prod + kMaxNz);
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = lane + 32 * u;  // < kMaxNz: slots past the task are written too (no branch)
        prod[e] = e < ne && sv[u] != kPadSrc ? (sv[u] < 0 ? dmul(v[u], yv[u]) : v[u]) : 0.0;
        srcs[e] = sv[u];
      }
      __syncwarp();
#ifdef PSCU_TRACE
      if (a.ftrace && lane == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[2]));
        fc0 = clock64();
      }
#endif
      // lanes past the rows run row 0's loads with nothing to subtract
      const int roff_l = rowl ? roff : 0, fin_l = rowl ? fin : 0, lin_l = rowl ? lin : -1;
      const int nblk = rowl ? rlen >> 3 : 0;       // 8-entry blocks of the row
      const int lastb = max(nblk - 1, 0);
      const double2* pb = reinterpret_cast<const double2*>(prod + roff_l);
      double vin[3];
      int sin_[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int t = fin_l + c;
        const bool ok = t <= lin_l;
        const int at = roff_l + (ok ? t : 0);
        const double pv = prod[at];
        const int ps = srcs[at];
        vin[c] = ok ? pv : 0.0;
        sin_[c] = ok ? ps : -1;
      }
      double acc = rbl;
      // blocks holding prefix entries (most over the rows) and blocks that
      // are prefix entries only in every row (least): warp-uniform, so the
      // block sequence is straight-line code with two buffers used in turn;
      // full blocks subtract without selects
      const int steps = __reduce_max_sync(full, (fin_l + 7) >> 3);
      const int nfull = __reduce_min_sync(full, rowl ? fin_l >> 3 : 0x7fffffff);
      double2 ba[4], bb[4];
      auto load = [&](double2 (&buf)[4], int blk) {
#pragma unroll
        for (int k = 0; k < 4; ++k) buf[k] = pb[4 * min(blk, lastb) + k];
      };
      auto chain = [&](const double2 (&buf)[4], int blk) {
        if (blk < nfull) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc = dsub(acc, buf[k].x);
            acc = dsub(acc, buf[k].y);
          }
        } else {
          const int t0 = 8 * blk;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double a0 = dsub(acc, buf[k].x);
            acc = t0 + 2 * k < fin_l ? a0 : acc;
            const double a1 = dsub(acc, buf[k].y);
            acc = t0 + 2 * k + 1 < fin_l ? a1 : acc;
          }
        }
      };
      // the usual task: S blocks hold prefix entries, the first S - 1 in
      // every row — all blocks loaded up front, no branch inside the chain
      auto fixed = [&](auto sc) {
        constexpr int S = decltype(sc)::value;
        double2 b[S][4];
#pragma unroll
        for (int j = 0; j < S; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k) b[j][k] = pb[4 * min(j, lastb) + k];
#pragma unroll
        for (int j = 0; j + 1 < S; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc = dsub(acc, b[j][k].x);
            acc = dsub(acc, b[j][k].y);
          }
        const int t0 = 8 * (S - 1);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double a0 = dsub(acc, b[S - 1][k].x);
          acc = t0 + 2 * k < fin_l ? a0 : acc;
          const double a1 = dsub(acc, b[S - 1][k].y);
          acc = t0 + 2 * k + 1 < fin_l ? a1 : acc;
        }
      };
      if (steps == 3 && nfull == 2) fixed(std::integral_constant<int, 3>{});
      else if (steps == 2 && nfull == 1) fixed(std::integral_constant<int, 2>{});
      else if (steps == 1 && nfull == 0) fixed(std::integral_constant<int, 1>{});
      else {
      load(ba, 0);
      load(bb, 1);
      if (steps > 0) {
        chain(ba, 0);
        if (steps > 1) {
          if (steps > 2) load(ba, 2);
          chain(bb, 1);
          if (steps > 2) {
            if (steps > 3) load(bb, 3);
            chain(ba, 2);
            if (steps > 3) {
              if (steps > 4) load(ba, 4);
              chain(bb, 3);
              if (steps > 4) {
                if (steps > 5) load(bb, 5);
                chain(ba, 4);
                if (steps > 5) chain(bb, 5);
              }
            }
          }
        }
      }
      }
#pragma unroll
      for (int sr = 0; sr < 3; ++sr) {
        const double xs = __shfl_sync(full, acc, sr);
        const bool h0 = sin_[0] == sr, h1 = sin_[1] == sr, h2 = sin_[2] == sr;
        const double vv = h0 ? vin[0] : (h1 ? vin[1] : vin[2]);
        const double a1 = dsub(acc, dmul(vv, xs));
        acc = (h0 || h1 || h2) ? a1 : acc;
      }
      if (rowl) {
        flow_store(y + rowid, acc);
        yb[opz] = acc;
      }
#ifdef PSCU_TRACE
      if (a.ftrace && lane == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[3]));
        long long* ft = a.ftrace + (size_t(hd[9]) + task) * 6;
        for (int q = 0; q < 4; ++q) ft[q] = (long long)fts[q];
        ft[4] = clock64() - fc0;
        ft[5] = 5;
      }
#endif
      __syncwarp();
      continue;
    }
    if (kFlow && !kFwd && kMaxNz == kFlowSmallNz && a.bfast && !a.bshfl && lead_ok && nrows <= 4) {
      // Backward face-block tasks on lane 0, shaped by the ncu stall profile
      // of the general fold (profiles/r03c_flow_bwd_lines.txt: the leading
      // in-task terms cost as much as the whole chain — two dependent
      // shared-memory loads per term — and every row re-read its header):
      //  * dense 8-byte products, 128-bit loads, one 8-entry block ahead;
      //  * the rows' values stay in registers (rows unrolled), so a leading
      //    in-task term is one multiply and one subtraction;
      //  * all row headers and right-hand sides are loaded before the chain.
      // Same operations in the same order as the general fold: bitwise.
      double* prod = reinterpret_cast<double*>(&rec[w][0]);   // kMaxNz products
      int* srcs = reinterpret_cast<int*>(prod + kMaxNz);      // kMaxNz sources
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = lane + 32 * u;  // < kMaxNz: slots past the task are written too (no branch)
        prod[e] = e < ne && sv[u] != kPadSrc ? (sv[u] < 0 ? dmul(v[u], yv[u]) : v[u]) : 0.0;
        srcs[e] = sv[u];
      }
      __syncwarp();
#ifdef PSCU_TRACE
      if (a.ftrace && lane == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[2]));
        fc0 = clock64();
      }
#endif
      if (lane == 0) {
        int4 hdr[4];
        double rh[4], dd[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int rr = r < nrows ? r : 0;
          hdr[r] = mb[w][rr];
          rh[r] = rb[w][rr];
          dd[r] = dvb[w][rr];
        }
        double xs[4] = {0.0, 0.0, 0.0, 0.0};
        // a row's first block and leading sources are fetched while the row
        // before it is folded (the stores below carry no memory clobber, so
        // the loads stay in flight across them)
        double2 fb[4];
        int4 fs;
        auto first_block = [&](int r) {
          const double2* p = reinterpret_cast<const double2*>(prod + hdr[r].z);
#pragma unroll
          for (int k = 0; k < 4; ++k) fb[k] = p[k];
          fs = *reinterpret_cast<const int4*>(srcs + hdr[r].z);
        };
        first_block(0);
        // the usual face-block task: every row the same 1-3 blocks. The row is
        // then straight-line code (all its blocks loaded up front, no branch
        // inside the dependent chain); other tasks take the general sequence
        bool uni = true;
#pragma unroll
        for (int r = 1; r < 4; ++r) uni = uni && (r >= nrows || hdr[r].x == hdr[0].x);
        const int nb0 = hdr[0].x >> 3;
        auto row_fixed = [&](auto rc, auto nbc) {
          constexpr int r = decltype(rc)::value, NB = decltype(nbc)::value;
          const int lead = hdr[r].w;
          const double2* pb = reinterpret_cast<const double2*>(prod + hdr[r].z);
          double acc = rh[r];
          double2 b0[4], b1[4], b2[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) b0[k] = fb[k];
          const int4 s4 = fs;
          if (NB > 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) b1[k] = pb[4 + k];
          }
          if (NB > 2) {
#pragma unroll
            for (int k = 0; k < 4; ++k) b2[k] = pb[8 + k];
          }
          if (r + 1 < 4) {
            if (r + 1 < nrows) first_block(r + 1);
          }
          const double x0 = s4.x == 0 ? xs[0] : (s4.x == 1 ? xs[1] : xs[2]);
          const double x1 = s4.y == 0 ? xs[0] : (s4.y == 1 ? xs[1] : xs[2]);
          const double x2 = s4.z == 0 ? xs[0] : (s4.z == 1 ? xs[1] : xs[2]);
          const double m0 = dmul(b0[0].x, x0), m1 = dmul(b0[0].y, x1), m2 = dmul(b0[1].x, x2);
          b0[0].x = lead > 0 ? m0 : b0[0].x;
          b0[0].y = lead > 1 ? m1 : b0[0].y;
          b0[1].x = lead > 2 ? m2 : b0[1].x;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc = dsub(acc, b0[k].x);
            acc = dsub(acc, b0[k].y);
          }
          if (NB > 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              acc = dsub(acc, b1[k].x);
              acc = dsub(acc, b1[k].y);
            }
          }
          if (NB > 2) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              acc = dsub(acc, b2[k].x);
              acc = dsub(acc, b2[k].y);
            }
          }
          acc = __ddiv_rn(acc, dd[r]);
          xs[r] = acc;
          flow_store_nc(y + hdr[r].y, acc);
        };
        auto task_fixed = [&](auto nbc) {
          row_fixed(std::integral_constant<int, 0>{}, nbc);
          if (nrows > 1) row_fixed(std::integral_constant<int, 1>{}, nbc);
          if (nrows > 2) row_fixed(std::integral_constant<int, 2>{}, nbc);
          if (nrows > 3) row_fixed(std::integral_constant<int, 3>{}, nbc);
        };
        if (uni && nb0 == 3) task_fixed(std::integral_constant<int, 3>{});
        else if (uni && nb0 == 2) task_fixed(std::integral_constant<int, 2>{});
        else if (uni && nb0 == 1) task_fixed(std::integral_constant<int, 1>{});
        else
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r < nrows) {
            const int len = hdr[r].x, lead = hdr[r].w;
            const double2* pb = reinterpret_cast<const double2*>(prod + hdr[r].z);
            double acc = rh[r];
            // two block buffers used in turn (no register moves, no loop):
            // a buffer is refilled right after its block is subtracted and
            // needed one block later
            double2 ba[4], bb[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) ba[k] = fb[k];
            const int4 s4 = fs;
            const int last = len / 8 - 1;  // index of the row's last block (-1: empty row)
            auto load = [&](double2 (&buf)[4], int blk) {
#pragma unroll
              for (int k = 0; k < 4; ++k) buf[k] = pb[4 * blk + k];
            };
            auto chain = [&](const double2 (&buf)[4]) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                acc = dsub(acc, buf[k].x);
                acc = dsub(acc, buf[k].y);
              }
            };
            load(bb, max(min(1, last), 0));
            if (r + 1 < 4 && r + 1 < nrows) first_block(r + 1);
            // leading in-task terms (sources: earlier rows of this task), by selects
            {
              const double x0 = s4.x == 0 ? xs[0] : (s4.x == 1 ? xs[1] : xs[2]);
              const double x1 = s4.y == 0 ? xs[0] : (s4.y == 1 ? xs[1] : xs[2]);
              const double x2 = s4.z == 0 ? xs[0] : (s4.z == 1 ? xs[1] : xs[2]);
              const double m0 = dmul(ba[0].x, x0), m1 = dmul(ba[0].y, x1), m2 = dmul(ba[1].x, x2);
              ba[0].x = lead > 0 ? m0 : ba[0].x;
              ba[0].y = lead > 1 ? m1 : ba[0].y;
              ba[1].x = lead > 2 ? m2 : ba[1].x;
            }
            if (last >= 0) {
              chain(ba);
              if (last >= 1) {
                if (last >= 2) load(ba, 2);
                chain(bb);
                if (last >= 2) {
                  if (last >= 3) load(bb, 3);
                  chain(ba);
                  if (last >= 3) {
                    if (last >= 4) load(ba, 4);
                    chain(bb);
                    if (last >= 4) {
                      if (last >= 5) load(bb, 5);
                      chain(ba);
                      if (last >= 5) chain(bb);
                    }
                  }
                }
              }
            }
            acc = __ddiv_rn(acc, dd[r]);
            xs[r] = acc;
            flow_store_nc(y + hdr[r].y, acc);
          }
        }
      }
#ifdef PSCU_TRACE
      if (a.ftrace && lane == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[3]));
        long long* ft = a.ftrace + (size_t(hd[9]) + task) * 6;
        for (int q = 0; q < 4; ++q) ft[q] = (long long)fts[q];
        ft[4] = clock64() - fc0;
        ft[5] = 4;
      }
#endif
      __syncwarp();
      continue;
    }
    if (kFlow && !kFwd && kMaxNz <= kFlowMidNz && a.bshfl && lead_ok) {
      // Backward face-block tasks: a row's in-task sources lead its chain and
      // the last sources to arrive are its first out-of-task terms, so the
      // whole task is one dependent subtraction chain after the hand-over.
      // The products stay in the lanes' registers and every lane runs the
      // same chain (no divergence, no shared-memory round trip): entry e of
      // the task lives in lane e % 32, register e / 32; rows hold whole
      // 8-entry blocks, so kB consecutive entries sit in one register of kB
      // consecutive lanes and are fetched by kB shuffles, one step ahead of the chain.
      // Each row still takes its operations in column order, one rounding
      // per operation: bitwise the sequential fold.
      // (the lanes leave the polling loop at different rounds: reconverge
      // first, or every shuffle below becomes a rendezvous of diverged groups)
      __syncwarp();
#ifdef PSCU_TRACE
      const unsigned am0 = __activemask();
      unsigned am1 = 0;
      if (a.ftrace && lane == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[2]));
        fc0 = clock64();
      }
#endif
      double pr[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = lane + 32 * u;
        pr[u] = e < ne && sv[u] != kPadSrc ? (sv[u] < 0 ? dmul(v[u], yv[u]) : v[u]) : 0.0;
      }
      // Rows hold whole 8-entry blocks: one step fetches a block (8 shuffles
      // of one register, chosen by selects, no branch) while the previous
      // block is subtracted; the look-ahead past a row's end reads entries
      // that are never used (clamped to the task's registers).
      constexpr int kB = 8;
      auto fetch = [&](int e, double (&p)[kB]) {
        const int u = e >> 5, b = e & 31;
        double sel = pr[0];
#pragma unroll
        for (int q = 1; q < kPer; ++q) sel = u == q ? pr[q] : sel;
#pragma unroll
        for (int k = 0; k < kB; ++k) p[k] = __shfl_sync(full, sel, b + k);
      };
      constexpr int kLastBlock = kMaxNz - kB;
      // Loop bounds and row data come from warp reductions (REDUX results
      // are uniform registers), so the control flow is uniform.
      const int nrows_u = __reduce_max_sync(full, nrows);
      for (int r = 0; r < nrows_u; ++r) {
        const int off = __reduce_max_sync(full, lane == r ? roff : 0);
        const int len = __reduce_max_sync(full, lane == r ? rlen : 0);
        const int rowr = __reduce_max_sync(full, lane == r ? rowid : 0);
        double acc = __shfl_sync(full, rbl, r);
        const double dvr = __shfl_sync(full, dvl, r);
        double nx[kB];
#ifdef PSCU_TRACE
        if (r == 1) am1 = __activemask();
#endif
        fetch(min(off, kLastBlock), nx);
        for (int g = 0; g < len; g += kB) {
          double cur[kB];
#pragma unroll
          for (int k = 0; k < kB; ++k) cur[k] = nx[k];
          fetch(min(off + g + kB, kLastBlock), nx);
#pragma unroll
          for (int k = 0; k < kB; ++k) acc = dsub(acc, cur[k]);
        }
        acc = __ddiv_rn(acc, dvr);
        // the row's value enters the later rows' leading in-task terms
#pragma unroll
        for (int u = 0; u < kPer; ++u)
          if (lane + 32 * u < ne && sv[u] == r) pr[u] = dmul(v[u], acc);
        // every lane holds the same value: one predicated store, no branch
        flow_store_if(y + rowr, acc, lane == 0);
      }
#ifdef PSCU_TRACE
      if (a.ftrace && lane == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[3]));
        long long* ft = a.ftrace + (size_t(hd[9]) + task) * 6;
        for (int q = 0; q < 4; ++q) ft[q] = (long long)fts[q];
        ft[4] = clock64() - fc0;
        ft[5] = 3 + 1000 * __popc(am0) + 100000 * __popc(am1);
      }
#endif
      __syncwarp();
      continue;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = lane + 32 * u;
      if (e < ne) {
        rec[w][e] = make_double2(sv[u] == kPadSrc ? 0.0 : (sv[u] < 0 ? dmul(v[u], yv[u]) : v[u]),
                                 __longlong_as_double((long long)sv[u]));
      }
    }
    __syncwarp();
#ifdef PSCU_TRACE
    if (kFlow && a.ftrace && lane == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[2]));
      fc0 = clock64();
    }
    if (tr) {
      a.trace[size_t(ch) * 16 + 1] = clock64();
      a.trace[size_t(ch) * 16 + 3] = ne;
      a.trace[size_t(ch) * 16 + 4] = r1 - r0;
    }
#endif
    // forward sweeps: when every row's in-task sources trail its
    // out-of-task ones (the face-block tasks of 3D coarse levels), lane r
    // folds row r's out-of-task prefix and the in-task terms follow row by
    // row through shuffles; each row still takes its operations in column
    // order, so the result is bitwise that of the sequential fold
    bool par = false;
    if (kFwd && trail_ok && nrows > 1) {
      par = true;
      double acc = 0.0;
      int cur = 0;
      if (lane < nrows) {
        acc = chain_sub(rb[w][lane], &rec[w][roff], fin);
        cur = fin;
      }
      for (int sr = 0; sr < nrows; ++sr) {
        const double xs = __shfl_sync(full, acc, sr);
        if (lane > sr && lane < nrows && cur < rlen) {
          const double2 r2 = rec[w][roff + cur];
          if (int(__double_as_longlong(r2.y)) == sr) {
            acc = dsub(acc, dmul(r2.x, xs));
            ++cur;
          }
        }
      }
      if (lane < nrows) {
        const int4 m = mb[w][lane];
        if (kFlow) flow_store(y + m.y, acc);
        else y[m.y] = acc;
        yb[m.z] = acc;
      }
#ifdef PSCU_TRACE
      if (kFlow && a.ftrace && lane == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[3]));
        long long* ft = a.ftrace + (size_t(hd[9]) + task) * 6;
        for (int q = 0; q < 4; ++q) ft[q] = (long long)fts[q];
        ft[4] = clock64() - fc0;
        ft[5] = 1;
      }
#endif
    }
    if (!par && lane == 0 && lead_ok) {
      // every row: its leading in-task terms, then a pure product chain
      for (int r = 0; r < nrows; ++r) {
        const int4 m = mb[w][r];
        const int2 ri = rinfo[w][r];
        double acc = rb[w][r];
        for (int t = 0; t < ri.y; ++t) {
          const double2 r2 = rec[w][ri.x + t];
          acc = dsub(acc, dmul(r2.x, cv[w][int(__double_as_longlong(r2.y))]));
        }
        acc = chain_sub(acc, &rec[w][ri.x + ri.y], m.x - ri.y);
        if (!kFwd) acc = __ddiv_rn(acc, dvb[w][r]);
        cv[w][r] = acc;
        if (kFlow) flow_store(y + m.y, acc);
        else y[m.y] = acc;
        if (kFwd) yb[m.z] = acc;
      }
#ifdef PSCU_TRACE
      if (kFlow && a.ftrace) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[3]));
        long long* ft = a.ftrace + (size_t(hd[9]) + task) * 6;
        for (int q = 0; q < 4; ++q) ft[q] = (long long)fts[q];
        ft[4] = clock64() - fc0;
        ft[5] = 2;
      }
#endif
    } else if (!par && lane == 0) {
      // general order: the next kFoldAhead entries' records are loaded while
      // the current ones are subtracted (rows hold whole 8-entry blocks, so
      // the look-ahead carries across rows; indices past the task clamp to
      // the buffer)
      int e = 0;
      double2 nx[kFoldAhead];
#pragma unroll
      for (int k = 0; k < kFoldAhead; ++k) nx[k] = rec[w][min(k, kMaxNz - 1)];
      for (int r = 0; r < r1 - r0; ++r) {
        const int4 m = mb[w][r];
        double acc = rb[w][r];
        const int e1 = e + m.x;
        for (; e + kFoldAhead <= e1; e += kFoldAhead) {
          double2 cur[kFoldAhead];
#pragma unroll
          for (int k = 0; k < kFoldAhead; ++k) cur[k] = nx[k];
#pragma unroll
          for (int k = 0; k < kFoldAhead; ++k) nx[k] = rec[w][min(e + kFoldAhead + k, kMaxNz - 1)];
#pragma unroll
          for (int k = 0; k < kFoldAhead; ++k) {
            const int sidx = int(__double_as_longlong(cur[k].y));
            acc = dsub(acc, sidx < 0 ? cur[k].x : dmul(cur[k].x, cv[w][sidx]));
          }
        }
        const int er = e;
        for (; e < e1; ++e) {
          const double2 r2 = rec[w][e];
          const int sidx = int(__double_as_longlong(r2.y));
          acc = dsub(acc, sidx < 0 ? r2.x : dmul(r2.x, cv[w][sidx]));
        }
        if (e != er) {
#pragma unroll
          for (int k = 0; k < kFoldAhead; ++k) nx[k] = rec[w][min(e + k, kMaxNz - 1)];
        }
        if (!kFwd) acc = __ddiv_rn(acc, dvb[w][r]);
        cv[w][r] = acc;
        if (kFlow) flow_store(y + m.y, acc);
        else y[m.y] = acc;
        if (kFwd) yb[m.z] = acc;
      }
#ifdef PSCU_TRACE
      if (kFlow && a.ftrace) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fts[3]));
        long long* ft = a.ftrace + (size_t(hd[9]) + task) * 6;
        for (int q = 0; q < 4; ++q) ft[q] = (long long)fts[q];
        ft[4] = clock64() - fc0;
        ft[5] = 0;
      }
      if (tr) a.trace[size_t(ch) * 16 + 2] = clock64();
      if (tr2) {
        unsigned long long gt1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
        a.trace[size_t(kTraceSub) * 16 + size_t(task) * 2] = (long long)gt0;
        a.trace[size_t(kTraceSub) * 16 + size_t(task) * 2 + 1] = (long long)gt1;
      }
#endif
    }
    __syncwarp();
  }
}

template <bool kFwd>
__global__ void __launch_bounds__(32 * kLevelWarps)
    level_kernel(WalkArgs a, int ch, const double* rhs, double* y, double* yb) {
  level_chunk<kFwd, true>(a, ch, rhs, y, yb);
}

/// Grid-wide barrier for the persistent task-level kernel: a monotone
/// arrival counter (zeroed before the launch), target = levels x CTAs.
__device__ __forceinline__ void level_barrier(unsigned long long* cnt, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt, 1ull);
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

/// All task levels of a level-plan sweep in one cooperative launch: a grid
/// barrier replaces the kernel boundary between levels.
template <bool kFwd>
__global__ void __launch_bounds__(32 * kLevelWarps)
    level_persist_kernel(WalkArgs a, int c0, int c1, const double* rhs, double* y, double* yb,
                         unsigned long long* cnt) {
  for (int ch = c0; ch < c1; ++ch) {
    level_chunk<kFwd, false>(a, ch, rhs, y, yb);
    if (ch + 1 < c1) level_barrier(cnt, (unsigned long long)(ch - c0 + 1) * gridDim.x);
  }
}

/// All task levels of a level-plan sweep in one cooperative launch without
/// barriers: every warp takes its tasks in level order and waits on the
/// values of its out-of-task sources only (kFlowSentinel). Every task waits
/// on tasks of strictly lower levels and all warps are co-resident, so the
/// lowest unfinished level always progresses.
template <bool kFwd>
__global__ void __launch_bounds__(32 * kLevelWarps, 4)
    level_flow_kernel(WalkArgs a, int c0, int c1, const double* rhs, double* y, double* yb) {
  for (int ch = c0; ch < c1; ++ch) level_chunk<kFwd, false, true>(a, ch, rhs, y, yb);
}

/// The same for plans whose tasks hold at most kFlowSmallNz entries (the
/// face-block tasks of the 3D coarse levels): a quarter of the per-lane
/// registers and shared memory, so twice the warps are resident and
/// consecutive task levels run on disjoint warps (a warp's next task is at
/// least two levels ahead, its operand loads off the critical path).
#ifndef PSCU_FLOW_SMALL_CTAS
#define PSCU_FLOW_SMALL_CTAS 7
#endif
constexpr int kFlowSmallCtas = PSCU_FLOW_SMALL_CTAS;
#ifndef PSCU_FLOW_SMALL_CTAS_BWD
#define PSCU_FLOW_SMALL_CTAS_BWD 5
#endif
// the backward kernel's shuffle fold keeps two 8-entry blocks in registers
constexpr int kFlowSmallCtasBwd = PSCU_FLOW_SMALL_CTAS_BWD;

template <bool kFwd>
__global__ void __launch_bounds__(32 * kLevelWarps, kFwd ? kFlowSmallCtas : kFlowSmallCtasBwd)
    level_flow_small_kernel(WalkArgs a, int c0, int c1, const double* rhs, double* y, double* yb) {
  for (int ch = c0; ch < c1; ++ch) level_chunk<kFwd, false, true, kFlowSmallNz>(a, ch, rhs, y, yb);
}


/// The same for tasks of up to kFlowMidNz entries (chains of the three face
/// blocks an element introduces: a third of the task levels).
template <bool kFwd>
__global__ void __launch_bounds__(32 * kLevelWarps, PSCU_FLOW_MID_CTAS)
    level_flow_mid_kernel(WalkArgs a, int c0, int c1, const double* rhs, double* y, double* yb) {
  for (int ch = c0; ch < c1; ++ch) level_chunk<kFwd, false, true, kFlowMidNz>(a, ch, rhs, y, yb);
}

/// The same with a two-stage software pipeline over the warp's task
/// sequence (PSCU_LEVEL_FLOW=2): the record of task t+2 and the entries,
/// row data and right-hand sides of task t+1 (whose record arrived one task
/// earlier) are in flight while task t waits on its sources and folds, so
/// the dependent record -> entries round trips leave the critical path.
struct FlowRec {
  int ch, task, r0, nrows, e0, ne;
};

__device__ __forceinline__ bool flow_advance(const WalkArgs& a, int c1, int gw, int W, int& ch,
                                             int& task) {
  task += W;
  while (ch < c1) {
    if (task < a.sl_hdr[kHdr * ch + 8]) return true;
    ++ch;
    task = gw;
  }
  return false;
}

__device__ __forceinline__ FlowRec flow_record(const WalkArgs& a, int ch, int task) {
  const int* hd = a.sl_hdr + kHdr * ch;
  const int32_t* tt = a.tt + hd[9];
  const int32_t* tq = a.tq + hd[9];
  FlowRec r;
  r.ch = ch;
  r.task = task;
  r.r0 = tt[task];
  r.nrows = tt[task + 1] - r.r0;
  r.e0 = tq[task];
  r.ne = tq[task + 1] - r.e0;
  return r;
}

struct FlowOps {
  int sv[kLevelMaxNz / 32];
  double v[kLevelMaxNz / 32];
  int4 meta;
  double rb, dv;
};

template <bool kFwd>
__device__ __forceinline__ void flow_ops(const WalkArgs& a, const double* rhs, const FlowRec& r,
                                         int lane, FlowOps& o) {
  constexpr int kPer = kLevelMaxNz / 32;
  const int k0 = a.sl_k[r.ch], nr = a.sl_nr[r.ch], nq = a.sl_hdr[kHdr * r.ch + 2];
  const int64_t qa = a.sl_q[r.ch] + r.e0;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = lane + 32 * u;
    o.sv[u] = e < r.ne ? __ldg(a.src + qa + e) : 0;
    o.v[u] = e < r.ne ? __ldg(a.val + qa + e) : 0.0;
  }
  if (lane < r.nrows) {
    const int k = k0 + r.r0 + lane;
    const int len = int((r.r0 + lane + 1 < nr ? a.off[k + 1] : nq) - a.off[k]);
    o.meta = make_int4(len, a.rows[k], kFwd ? a.opos[k] : 0, 0);
    o.dv = kFwd ? 1.0 : a.dv[k];
    o.rb = __ldcg(rhs + k);
  }
}

template <bool kFwd>
__global__ void __launch_bounds__(32 * kLevelWarps)
    level_flow2_kernel(WalkArgs a, int c0, int c1, const double* rhs, double* y, double* yb) {
  constexpr int kPer = kLevelMaxNz / 32;
  __shared__ double2 rec[kLevelWarps][kLevelMaxNz];
  __shared__ double rbs[kLevelWarps][kLevelMaxRows], dvs[kLevelWarps][kLevelMaxRows],
      cv[kLevelWarps][kLevelMaxRows];
  __shared__ int4 mbs[kLevelWarps][kLevelMaxRows];
  const int w = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  const int gw = int(blockIdx.x) * kLevelWarps + w, W = int(gridDim.x) * kLevelWarps;
  // pipeline: r_cur / o_cur (task t), r_nxt / o_nxt (t+1), r_far (t+2)
  int ch = c0, task = gw - W;
  if (!flow_advance(a, c1, gw, W, ch, task)) return;
  FlowRec r_cur = flow_record(a, ch, task);
  FlowOps o_cur, o_nxt;
  flow_ops<kFwd>(a, rhs, r_cur, lane, o_cur);
  bool has_nxt = flow_advance(a, c1, gw, W, ch, task);
  FlowRec r_nxt = has_nxt ? flow_record(a, ch, task) : r_cur;
  for (;;) {
    // stage 2 for t+1 and stage 1 for t+2, issued before task t's waits
    bool has_far = false;
    FlowRec r_far = r_nxt;
    if (has_nxt) {
      flow_ops<kFwd>(a, rhs, r_nxt, lane, o_nxt);
      has_far = flow_advance(a, c1, gw, W, ch, task);
      if (has_far) r_far = flow_record(a, ch, task);
    }
    double yv[kPer];
    unsigned long long raw[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = lane + 32 * u;
      const bool out = e < r_cur.ne && o_cur.sv[u] < 0 && o_cur.sv[u] != kPadSrc;
      raw[u] = out ? flow_peek(y + (-o_cur.sv[u] - 1)) : 0ull;
    }
    for (;;) {
      bool pending = false;
#pragma unroll
      for (int u = 0; u < kPer; ++u) pending = pending || raw[u] == kFlowSentinel;
      if (!pending) break;
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if (raw[u] == kFlowSentinel) raw[u] = flow_peek(y + (-o_cur.sv[u] - 1));
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = lane + 32 * u;
      const bool out = e < r_cur.ne && o_cur.sv[u] < 0 && o_cur.sv[u] != kPadSrc;
      yv[u] = out ? __longlong_as_double((long long)raw[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = lane + 32 * u;
      if (e < r_cur.ne)
        rec[w][e] = make_double2(
            o_cur.sv[u] == kPadSrc ? 0.0 : (o_cur.sv[u] < 0 ? dmul(o_cur.v[u], yv[u]) : o_cur.v[u]),
            __longlong_as_double((long long)o_cur.sv[u]));
    }
    if (lane < r_cur.nrows) {
      mbs[w][lane] = o_cur.meta;
      rbs[w][lane] = o_cur.rb;
      dvs[w][lane] = o_cur.dv;
    }
    __syncwarp();
    if (lane == 0) {
      int e = 0;
      for (int r = 0; r < r_cur.nrows; ++r) {
        const int4 m = mbs[w][r];
        double acc = rbs[w][r];
        const int e1 = e + m.x;
        for (; e + 8 <= e1; e += 8) {
          int s8[8];
          double p8[8], c8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const double2 r2 = rec[w][e + k];
            s8[k] = int(__double_as_longlong(r2.y));
            p8[k] = r2.x;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) c8[k] = s8[k] < 0 ? 0.0 : cv[w][s8[k]];
#pragma unroll
          for (int k = 0; k < 8; ++k) acc = dsub(acc, s8[k] < 0 ? p8[k] : dmul(p8[k], c8[k]));
        }
        for (; e < e1; ++e) {
          const double2 r2 = rec[w][e];
          const int sidx = int(__double_as_longlong(r2.y));
          acc = dsub(acc, sidx < 0 ? r2.x : dmul(r2.x, cv[w][sidx]));
        }
        if (!kFwd) acc = __ddiv_rn(acc, dvs[w][r]);
        cv[w][r] = acc;
        flow_store(y + m.y, acc);
        if (kFwd) yb[m.z] = acc;
      }
    }
    __syncwarp();
    if (!has_nxt) break;
    r_cur = r_nxt;
    o_cur = o_nxt;
    has_nxt = has_far;
    r_nxt = r_far;
  }
}

/// Values of the static out-of-ring sources of one walker launch.
__global__ void gather_static(int64_t m, const int2* __restrict__ sfar, const double* __restrict__ y,
                              double* __restrict__ sfv) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m;
       e += int64_t(gridDim.x) * blockDim.x)
    sfv[e] = y[sfar[e].y];
}

/// Right-hand side in position order: xs[k] = x[rows[k]].
__global__ void gather_rhs(int64_t npos, const int32_t* __restrict__ rows,
                           const double* __restrict__ x, double* __restrict__ xs) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < npos;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int r = rows[k];
    xs[k] = r >= 0 ? x[r] : 0.0;
  }
}

template <typename I>
__global__ void gather_vals(int64_t m, const I* __restrict__ from,
                            const double* __restrict__ lu, double* __restrict__ out) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = from[q];
    out[q] = p >= 0 ? lu[p] : 0.0;
  }
}

/// Back-off (ns) between polls of a not-yet-published source in the
/// dataflow sweeps (PSCU_FLOW_SPIN_NS; default 0 = tight polling).
static int flow_spin_ns() {
  static const int v = [] {
    const char* e = getenv("PSCU_FLOW_SPIN_NS");
    return e ? std::max(0, atoi(e)) : 0;
  }();
  return v;
}

static void* flow_kernel_fn(bool fwd, bool v2, int small) {
  if (v2) return fwd ? (void*)level_flow2_kernel<true> : (void*)level_flow2_kernel<false>;
  if (small == 2) return fwd ? (void*)level_flow_mid_kernel<true> : (void*)level_flow_mid_kernel<false>;
  if (small) return fwd ? (void*)level_flow_small_kernel<true> : (void*)level_flow_small_kernel<false>;
  return fwd ? (void*)level_flow_kernel<true> : (void*)level_flow_kernel<false>;
}

/// Rotation of the dataflow sweeps' task-to-warp assignment (default on:
/// C5 ILU apply 6.9 -> 5.5 ms, C3 2.34 -> 2.14 ms); PSCU_FLOW_ROTATE=0 pins it.
static int flow_rotate() {
  static const int v = [] {
    const char* e = getenv("PSCU_FLOW_ROTATE");
    return e ? atoi(e) : 1;
  }();
  return v;
}

/// Warps missing more than 8 lanes' sources (levels ahead of the sweep
/// front) poll this much slower (config 5: 3.23 -> 3.18 ms per apply at 300).
static int flow_far_ns() {
  const char* e = getenv("PSCU_FLOW_FAR_NS");
  return e ? std::max(0, atoi(e)) : 300;
}

/// PSCU_FLOW_LEAD=1: dataflow sweeps wait on the task's latest source first
/// (one warp-uniform load per round) before polling all sources. Default off:
/// it takes the polls off the load/store unit but adds a round trip after the
/// lead source arrives (config 3: 1.45 vs 1.39 ms per apply; config 5 equal).
static int flow_lead() {
  const char* e = getenv("PSCU_FLOW_LEAD");
  return e ? atoi(e) : 0;
}

/// Face-block tasks (<= 4 rows, padded rows) fold from dense products:
/// backward on lane 0, forward one lane per row (default on;
/// PSCU_FLOW_BFAST=0: the general folds).
int level_pad();
static int flow_bfast() {
  const char* e = getenv("PSCU_FLOW_BFAST");
  return (e ? atoi(e) : 1) && level_pad() == 8;
}

/// Backward small-task dataflow sweeps fold through shuffles on all lanes
/// (PSCU_FLOW_BSHFL=1; needs padded rows). Default off: bitwise the same, and
/// measured 4-10 % slower than the lane-0 shared-memory fold inside the
/// loaded kernel (config 5: 4.39 vs 4.10 ms per apply) although faster in
/// isolation (tools/probe_fold4.cu: 24 vs 39 cycles per entry).
int level_pad();
static int flow_bshfl() {
  const char* e = getenv("PSCU_FLOW_BSHFL");
  return (e ? atoi(e) : 0) && level_pad() == 8;
}

WalkArgs args_of(const WalkPlan& w) {
  return {w.sl_k.p, w.sl_nr.p, w.sl_q.p, w.sl_hdr.p, w.tt.p, w.tq.p, w.rows.p, w.off.p, w.dp.p, w.meta.p,
          w.opos.p, w.val.p,  w.src.p,  w.dv.p,     w.sl_f.p,
          reinterpret_cast<const int2*>(w.far.p), w.sl_s.p,
          reinterpret_cast<const int2*>(w.sfar.p), w.sfv.p, nullptr, flow_spin_ns(), nullptr,
          flow_rotate(), flow_lead(), flow_far_ns(), flow_bfast(), flow_bshfl()};
}

size_t walk_smem() { return sizeof(double) * kRing + kStages * sizeof(Stage); }

unsigned grid1(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return unsigned(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
}

/// DAG levels of one sweep in processing order.
std::vector<int32_t> dag_levels(const Csr& a, const std::vector<int64_t>& diag, bool fwd,
                                int& nlev) {
  const int64_t n = a.n;
  const auto& rp = a.h_row_ptr;
  const auto& cols = a.h_cols;
  std::vector<int32_t> lvl(n, 0);
  nlev = 0;
  for (int64_t p = 0; p < n; ++p) {
    const int64_t i = fwd ? p : n - 1 - p;
    const int64_t q0 = fwd ? rp[i] : diag[i] + 1, q1 = fwd ? diag[i] : rp[i + 1];
    int L = 0;
    for (int64_t q = q0; q < q1; ++q) L = std::max(L, lvl[cols[q]] + 1);
    lvl[i] = L;
    nlev = std::max(nlev, L + 1);
  }
  return lvl;
}

/// Allocator that leaves new elements uninitialised (the big per-entry plan
/// arrays are filled by parallel host threads, which then also take the
/// first-touch page faults).
template <typename T>
struct UninitAlloc : std::allocator<T> {
  template <typename U>
  struct rebind {
    using other = UninitAlloc<U>;
  };
  UninitAlloc() = default;
  template <typename U>
  UninitAlloc(const UninitAlloc<U>&) {}
  template <typename U, typename... Args>
  void construct(U* p, Args&&... args) {
    if constexpr (sizeof...(Args) > 0) ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
    else ::new (static_cast<void*>(p)) U;
  }
};

struct HostPlan {
  int C = 1;
  bool flow = false;  // single-CTA dataflow walker (flow_kernel), chunks span levels
  int S = 0;          // push walker: replicated ring slots per owner (0: classic walker)
  bool levels = false;  // every task level is a wide chunk
  bool push_ok = true;
  std::vector<int32_t> side;  // push walker: long-range slot + 1 of a row (0: none), by row
  std::vector<int32_t> sl_k, sl_nr, sl_nq, sl_nfar, sl_r0, rows, off, pos;
  std::vector<int32_t, UninitAlloc<int32_t>> src;   // per packed entry
  std::vector<int32_t, UninitAlloc<int32_t>> from;  // per packed entry: factor position or -1
  std::vector<int32_t> far, sfar;  // pairs {entry offset in chunk, source row}
  std::vector<int64_t> sl_f, sl_s, sl_q, dfrom;
  std::vector<int32_t> dp, sl_d, sl_nd;  // walker chunks: diagonal starts (padded to 4)
  std::vector<int32_t> tq;               // wide chunks: entry offset per task (+ total)
  std::vector<int32_t> tt, sl_t, sl_nt;  // task tables (first local row per task, then the row
                                         // count; 4-aligned starts) and task counts per chunk
  std::vector<uint8_t> sl_wide;
  int64_t npos = 0;
};

/// Positions, chunks and packed operands of one sweep for a C-CTA walker.
/// Tasks of a sweep: chains of rows one thread folds in order. Row i (in
/// processing order) joins the task holding its most recent source when that
/// source is the task's last row, the task stays within `max_rows` rows and
/// kMaxDiag entries, and every other source of i lies in a task of a strictly
/// lower task level. Task levels are then a topological order of the task
/// graph (every source of a task's row is in the task itself or in a lower
/// level), and a level's tasks are independent. max_rows = 1 gives the row
/// DAG levels. On the 256^2 config-2a hierarchy chains cut the sweep depth
/// from 771 (k = 0) / 3090 (k = 3) levels to ~258 (one per mesh row).
struct Tasks {
  std::vector<int32_t> ptr, rows, lvl, nz;  // rows of task t: rows[ptr[t] .. ptr[t + 1])
  int nlev = 0;
};

Tasks build_tasks(const Csr& a, const std::vector<int64_t>& diag, bool fwd, int max_rows,
                  int max_nz, int pad = 1) {
  const int64_t n = a.n;
  const auto& rp = a.h_row_ptr;
  const auto& cols = a.h_cols;
  Tasks T;
  T.lvl.reserve(n);
  T.nz.reserve(n);
  std::vector<int32_t> task(n, -1), tail, head, cnt, next(n, -1);
  tail.reserve(n);
  head.reserve(n);
  cnt.reserve(n);
  for (int64_t p = 0; p < n; ++p) {
    const int64_t i = fwd ? p : n - 1 - p;
    const int64_t q0 = fwd ? rp[i] : diag[i] + 1, q1 = fwd ? diag[i] : rp[i + 1];
    const int len = int((q1 - q0 + pad - 1) / pad * pad);  // entries incl. padding
    int64_t latest = -1;
    for (int64_t q = q0; q < q1; ++q)
      if (latest < 0 || (fwd ? cols[q] > latest : cols[q] < latest)) latest = cols[q];
    int join = -1;
    if (latest >= 0 && max_rows > 1) {
      const int t = task[latest];
      bool ok = tail[t] == latest && cnt[t] < max_rows && T.nz[t] + len <= max_nz;
      for (int64_t q = q0; q < q1 && ok; ++q) {
        const int u = task[cols[q]];
        if (u != t && T.lvl[u] >= T.lvl[t]) ok = false;
      }
      if (ok) join = t;
    }
    if (join < 0) {
      int L = 0;
      for (int64_t q = q0; q < q1; ++q) L = std::max(L, T.lvl[task[cols[q]]] + 1);
      join = int(T.lvl.size());
      T.lvl.push_back(L);
      T.nz.push_back(0);
      tail.push_back(-1);
      head.push_back(int32_t(i));
      cnt.push_back(0);
      T.nlev = std::max(T.nlev, L + 1);
    } else {
      next[tail[join]] = int32_t(i);
    }
    task[i] = join;
    tail[join] = int32_t(i);
    T.nz[join] += len;
    cnt[join]++;
  }
  const size_t nt = T.lvl.size();
  T.ptr.assign(nt + 1, 0);
  for (size_t t = 0; t < nt; ++t) T.ptr[t + 1] = T.ptr[t] + cnt[t];
  T.rows.resize(n);
  for (size_t t = 0; t < nt; ++t) {
    int32_t m = T.ptr[t];
    for (int32_t r = head[t]; r >= 0; r = next[r]) T.rows[m++] = r;
  }
  return T;
}

/// Rows per chain. Push walker: a consumer thread folds its chain's rows
/// back to back (~0.5-1k cycles of dependent latency per row, measured), so
/// long chains cost more than the sub-level handshakes they save. Task-level launches (one warp per task,
/// ~5 us per launch): chains of up to 16 rows cut the fine-level depth 12x.
int chain_rows(bool fwd = true) {
  if (const char* e = getenv(fwd ? "PSCU_CHAIN_ROWS_FWD" : "PSCU_CHAIN_ROWS_BWD"))
    return std::max(1, std::min(64, atoi(e)));
  if (const char* e = getenv("PSCU_CHAIN_ROWS")) return std::max(1, std::min(64, atoi(e)));
  return 3;  // 256^2 coarse apply: 1.43 ms (1), 1.61 (2), 1.28 (3), 3.8 (16)
}

/// Entry cap of a level-plan task: the slowest task's serial fold sets a
/// level's time (~76 cycles per entry measured), so long chains are cut.
int level_chain_nz() {
  if (const char* e = getenv("PSCU_LEVEL_CHAIN_NZ")) return std::max(16, std::min(kLevelMaxNz, atoi(e)));
  return kLevelMaxNz;
}

/// Level plans pad every row to whole 8-entry blocks with zero products
/// (acc - 0.0 == acc in IEEE arithmetic, so the fold is unchanged bit for
/// bit) so the warp kernel's fold never takes its scalar remainder loop.
int level_pad() {
  static const int v = [] {
    const char* e = getenv("PSCU_LEVEL_PAD");
    return e ? (atoi(e) != 0 ? 8 : 1) : 8;
  }();
  return v;
}

int level_chain_rows() {
  if (const char* e = getenv("PSCU_LEVEL_CHAIN_ROWS")) return std::max(1, std::min(kLevelMaxRows, atoi(e)));
  return 16;
}

/// Positions, chunks and packed operands of one sweep for a C-CTA walker.
/// Chunks hold tasks (max_rows > 1 only for the push walker, whose
/// consumers fold whole tasks).
void plan_sweep(const Csr& a, const std::vector<int64_t>& diag, bool fwd, int C, bool flow,
                int S, int max_rows, HostPlan& h, bool all_wide = false,
                const Tasks* pre = nullptr) {
  const int64_t n = a.n;
  const auto& rp = a.h_row_ptr;
  const auto& cols = a.h_cols;
  auto q_begin = [&](int64_t i) { return fwd ? rp[i] : diag[i] + 1; };
  auto q_end = [&](int64_t i) { return fwd ? diag[i] : rp[i + 1]; };
  const auto tp0 = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (getenv("PSCU_PLAN_DEBUG"))
      fprintf(stderr, "[plan %s n=%lld] %s %.3f s\n", fwd ? "fwd" : "bwd", (long long)a.n, what,
              std::chrono::duration<double>(std::chrono::steady_clock::now() - tp0).count());
  };
  const int pad = all_wide ? level_pad() : 1;
  Tasks own;
  if (!pre) own = build_tasks(a, diag, fwd, max_rows, all_wide ? level_chain_nz() : kMaxDiag, pad);
  const Tasks& T = pre ? *pre : own;
  tick("tasks");
  std::vector<int32_t> task_of(n);
  for (size_t t = 0; t + 1 < T.ptr.size(); ++t)
    for (int32_t m = T.ptr[t]; m < T.ptr[t + 1]; ++m) task_of[T.rows[m]] = int32_t(t);
  const int nlev = T.nlev;
  const int ntask = int(T.lvl.size());
  auto trows = [&](int t) { return T.ptr[t + 1] - T.ptr[t]; };
  std::vector<int32_t> lvl_ptr(nlev + 1, 0), order(ntask);
  for (int t = 0; t < ntask; ++t) lvl_ptr[T.lvl[t] + 1]++;
  for (int l = 0; l < nlev; ++l) lvl_ptr[l + 1] += lvl_ptr[l];
  {
    std::vector<int32_t> fill(lvl_ptr.begin(), lvl_ptr.end() - 1);
    for (int t = 0; t < ntask; ++t) order[fill[T.lvl[t]]++] = t;
  }
  h = HostPlan{};
  // a walker chunk stages at most kMaxDiag entries per task: a narrow level
  // holding a longer task (a row longer than that) cannot be walked — the
  // push walker reports it infeasible (the caller falls back to task-level
  // launches), the explicit walker modes refuse the pattern
  if (!all_wide && !flow)
    for (int l = 0; l < nlev; ++l) {
      if (lvl_ptr[l + 1] - lvl_ptr[l] > kWideRows) continue;
      for (int j = lvl_ptr[l]; j < lvl_ptr[l + 1]; ++j)
        if (T.nz[order[j]] > kMaxDiag) {
          if (S) {
            h.push_ok = false;
            return;
          }
          throw Error(PSCU_EINVAL, "walk plan: row exceeds the walker's diagonal capacity");
        }
    }
  h.C = C;
  h.levels = all_wide;
  h.flow = flow;
  h.S = S;
  h.pos.assign(n, -1);
  std::vector<int32_t> lpos(n, -1), chunk_of_row(n, -1);
  std::vector<int64_t> lcount(C, 0);  // per-CTA local positions (ring index)
  int64_t k = 0, q = 0;
  auto open_chunk = [&](bool wide, int rank) {
    k = (k + 3) & ~int64_t(3);
    q = (q + 3) & ~int64_t(3);
    h.sl_k.push_back(int32_t(k));
    h.sl_nr.push_back(0);
    h.sl_q.push_back(q);
    h.sl_nq.push_back(0);
    h.sl_wide.push_back(wide ? 1 : 0);
    if (!wide) lcount[rank] = (lcount[rank] + 3) & ~int64_t(3);
    h.sl_r0.push_back(wide ? 0 : int32_t(lcount[rank] & 0x7fffffff));
    while (h.tt.size() & 3) h.tt.push_back(0);
    h.sl_t.push_back(int32_t(h.tt.size()));
    h.sl_nt.push_back(0);
  };
  auto place_task = [&](int t, bool wide, int rank) {
    h.tt.push_back(h.sl_nr.back());
    h.sl_nt.back()++;
    for (int32_t m = T.ptr[t]; m < T.ptr[t + 1]; ++m) {
      const int32_t i = T.rows[m];
      const int64_t nz = wide ? (q_end(i) - q_begin(i) + pad - 1) / pad * pad : q_end(i) - q_begin(i);
      if (!wide && nz > kMaxDiag) throw Error(PSCU_ECUDA, "walk plan: row exceeds the diagonal capacity");
      h.pos[i] = int32_t(k++);
      if (!wide) lpos[i] = int32_t(lcount[rank]++);
      chunk_of_row[i] = int(h.sl_k.size()) - 1;
      h.sl_nr.back()++;
      h.sl_nq.back() += int32_t(nz);
      q += nz;
    }
  };
  auto close_chunk = [&]() { h.tt.push_back(h.sl_nr.back()); };
  // places the collected tasks of the open chunk, longest first: diagonal u
  // of a chunk is then a prefix of its tasks, stored contiguously
  std::vector<int32_t> members;
  auto commit = [&](int rank) {
    std::stable_sort(members.begin(), members.end(),
                     [&](int32_t x, int32_t y2) { return T.nz[x] > T.nz[y2]; });
    for (const int32_t t : members) place_task(t, false, rank);
    close_chunk();
    members.clear();
  };
  auto wide_level = [&](int l) {
    open_chunk(true, 0);
    for (int j = lvl_ptr[l]; j < lvl_ptr[l + 1]; ++j) place_task(order[j], true, 0);
    close_chunk();
  };
  if (flow) {
    // dataflow chunks: consecutive rows in level order, across level
    // boundaries (rows wait on their own sources, not on levels)
    if (max_rows != 1) throw Error(PSCU_ECUDA, "walk plan: the dataflow walker folds rows, not tasks");
    int64_t cnz = 0;
    bool open = false;
    for (int l = 0; l < nlev; ++l) {
      if (lvl_ptr[l + 1] - lvl_ptr[l] > kWideRows) {
        if (open) commit(0);
        open = false;
        wide_level(l);
        continue;
      }
      for (int j = lvl_ptr[l]; j < lvl_ptr[l + 1]; ++j) {
        const int32_t t = order[j];
        if (open && (int(members.size()) == kWalkThreads || cnz + T.nz[t] > kMaxNz - 8)) {
          commit(0);
          open = false;
        }
        if (!open) {
          open_chunk(false, 0);
          open = true;
          cnz = 0;
        }
        members.push_back(t);
        cnz += T.nz[t];
      }
    }
    if (open) commit(0);
  }
  for (int l = 0; l < nlev && !flow; ++l) {
    const int ntl = lvl_ptr[l + 1] - lvl_ptr[l];
    if (ntl > kWideRows || all_wide) {
      wide_level(l);
      continue;
    }
    // sub-levels of C chunks: row, task and entry budgets per chunk
    const int row_cap = S ? kStageRows : kWalkThreads;
    const int64_t nz_cap = kMaxNz - 8;
    // tasks go, in order, to the least-loaded chunk (load: the larger of the
    // row and entry fractions) that still has room; the rest start the next
    // sub-level
    std::vector<int32_t> rem(order.begin() + lvl_ptr[l], order.begin() + lvl_ptr[l + 1]), carry;
    std::vector<std::vector<int32_t>> bins(C);
    std::vector<int64_t> brows(C), bnz(C);
    while (!rem.empty()) {
      for (int r = 0; r < C; ++r) {
        bins[r].clear();
        brows[r] = bnz[r] = 0;
      }
      carry.clear();
      for (const int32_t t : rem) {
        int best = -1;
        double bl = 0;
        for (int r = 0; r < C; ++r) {
          if (brows[r] + trows(t) > row_cap || bnz[r] + T.nz[t] > nz_cap) continue;
          const double ld = std::max(double(brows[r]) / row_cap, double(bnz[r]) / double(nz_cap));
          if (best < 0 || ld < bl) {
            best = r;
            bl = ld;
          }
        }
        if (best < 0 && brows[0] == 0) best = 0;  // a single huge task still gets a chunk
        if (best < 0) {
          carry.push_back(t);
          continue;
        }
        bins[best].push_back(t);
        brows[best] += trows(t);
        bnz[best] += T.nz[t];
      }
      for (int rank = 0; rank < C; ++rank) {
        open_chunk(false, rank);
        members = bins[rank];
        commit(rank);
      }
      rem.swap(carry);
    }
  }
  tick("chunks");
  h.sl_q.push_back((q + 3) & ~int64_t(3));
  h.npos = (k + 3) & ~int64_t(3);
  const int nch = int(h.sl_k.size());
  // walker segments: maximal runs of non-wide chunks (C chunks per sub-level)
  std::vector<int32_t> seg_of(nch);
  int seg = -1;
  for (int c = 0; c < nch; ++c) {
    if (h.sl_wide[c] || c == 0 || h.sl_wide[c - 1]) ++seg;
    seg_of[c] = seg;
  }
  // local ring end of every rank at every sub-level (for the validity rule)
  h.rows.assign(h.npos + 4, -1);
  h.off.assign(h.npos + 4, 0);
  h.dfrom.assign(h.npos + 4, -1);
  const int64_t total = h.sl_q.back() + 8;
  h.from.resize(total);  // uninitialised: every entry is written below
  h.src.resize(total);
  {
    // padding entries (chunk alignment, tail): no factor value, no source
    auto pad = [&](int64_t q0, int64_t q1) {
      for (int64_t q = q0; q < q1; ++q) {
        h.from[q] = -1;
        h.src[q] = 0;
      }
    };
    for (int c = 0; c < nch; ++c) pad(h.sl_q[c] + h.sl_nq[c], h.sl_q[c + 1]);
    pad(h.sl_q[nch], total);
  }
  for (int64_t i = 0; i < n; ++i) h.rows[h.pos[i]] = int32_t(i);
  h.sl_f.assign(nch + 1, 0);
  h.sl_s.assign(nch + 1, 0);
  // chunk index -> (segment start chunk, sub-level index within segment)
  std::vector<int32_t> seg_first(nch, 0);
  for (int c = 0; c < nch; ++c) seg_first[c] = (c > 0 && seg_of[c] == seg_of[c - 1]) ? seg_first[c - 1] : c;
  // per chunk: the ring end (exclusive local position) of every rank at the
  // end of this chunk's sub-level
  h.sl_d.assign(nch, 0);
  h.sl_nd.assign(nch, 0);
  if (S) h.side.assign(n, 0);
  tick("arrays");
  {
    // wide chunks (row-contiguous entries, global sources) are independent
    // of each other and of the walker lists: filled by parallel host threads
    std::vector<int> wide;
    for (int c = 0; c < nch; ++c)
      if (h.sl_wide[c]) wide.push_back(c);
    std::atomic<size_t> next{0};
    h.tq.assign(h.tt.size(), 0);
    auto fill = [&] {
      for (size_t w = next++; w < wide.size(); w = next++) {
        const int c = wide[w];
        int64_t roff = 0;
        {
          // entry offset of every task (rows of a task are consecutive)
          const int32_t* tt = h.tt.data() + h.sl_t[c];
          int64_t o = 0;
          for (int i = 0, t = 0; i < h.sl_nt[c]; ++i) {
            for (; t < tt[i]; ++t)
              o += (q_end(h.rows[h.sl_k[c] + t]) - q_begin(h.rows[h.sl_k[c] + t]) + pad - 1) / pad * pad;
            h.tq[h.sl_t[c] + i] = int32_t(o);
          }
          h.tq[h.sl_t[c] + h.sl_nt[c]] = h.sl_nq[c];
        }
        for (int t = 0; t < h.sl_nr[c]; ++t) {
          const int64_t kp = h.sl_k[c] + t;
          const int32_t i = h.rows[kp];
          const int64_t qb = q_begin(i), len = q_end(i) - qb;
          const int64_t plen = (len + pad - 1) / pad * pad;
          h.off[kp] = int32_t(roff);
          h.dfrom[kp] = diag[i];
          for (int64_t u = len; u < plen; ++u) {
            h.from[h.sl_q[c] + roff + u] = -1;
            h.src[h.sl_q[c] + roff + u] = kPadSrc;
          }
          // a source in the row's own task: its index within the task (the
          // same thread / warp computed it just before)
          const int32_t ti = task_of[i], first = h.pos[T.rows[T.ptr[ti]]];
          for (int64_t u = 0; u < len; ++u) {
            const int64_t qq = h.sl_q[c] + roff + u;
            const int32_t jr = cols[qb + u];
            h.from[qq] = int32_t(qb + u);
            h.src[qq] = task_of[jr] == ti ? h.pos[jr] - first : -(jr + 1);
          }
          roff += plen;
        }
      }
    };
    const int nth = int(std::min<size_t>(wide.size(), std::max(1u, std::min(8u, std::thread::hardware_concurrency()))));
    std::vector<std::thread> pool;
    for (int t = 1; t < nth; ++t) pool.emplace_back(fill);
    fill();
    for (auto& th : pool) th.join();
  }
  tick("wide fill");
  std::vector<std::pair<int64_t, int32_t>> side_q;  // {entry, source row} read from slots
  std::vector<int32_t> last_read(S ? n : 0, -1);     // last reading sub-level (segment-local)
  for (int c = 0; c < nch; ++c) {
    if (S && !h.push_ok) return;  // infeasible for the push walker: stop early
    if (h.sl_wide[c]) {
      h.sl_f[c + 1] = h.sl_f[c];
      h.sl_s[c + 1] = h.sl_s[c];
      h.sl_nfar.push_back(0);
      continue;
    }
    int nf = 0, ns = 0;
    const int sub = (c - seg_first[c]) / C;
    const int sub_first = seg_first[c] + sub * C;
    const int nr = h.sl_nr[c];
    auto len_of = [&](int t) { return int(q_end(h.rows[h.sl_k[c] + t]) - q_begin(h.rows[h.sl_k[c] + t])); };
    // entry index of (row t, entry u): row-contiguous for wide chunks, else
    // diagonal-major over tasks (entry v of the concatenated rows of task i
    // at dstart[v] + i; tasks sorted by entry count, descending)
    std::vector<int32_t> dstart, ti(nr), uo(nr);
    if (!h.sl_wide[c]) {
      const int nt = h.sl_nt[c];
      const int32_t* tt = h.tt.data() + h.sl_t[c];
      std::vector<int32_t> tlen(nt, 0);
      for (int i = 0; i < nt; ++i)
        for (int t = tt[i]; t < tt[i + 1]; ++t) {
          ti[t] = i;
          uo[t] = tlen[i];
          tlen[i] += len_of(t);
        }
      const int nd = nt ? tlen[0] : 0;
      dstart.assign(nd + 1, 0);
      for (int u = 0, t = nt; u < nd; ++u) {
        while (t > 0 && tlen[t - 1] <= u) --t;
        dstart[u + 1] = dstart[u] + t;
      }
      h.sl_d[c] = int32_t(h.dp.size());
      h.sl_nd[c] = nd;
      for (int u = 0; u < nd; ++u) h.dp.push_back(dstart[u]);
      while (h.dp.size() & 3) h.dp.push_back(0);
    }
    int64_t roff = 0;
    for (int t = 0; t < nr; ++t) {
      const int64_t kp = h.sl_k[c] + t;
      const int32_t i = h.rows[kp];
      const int len = len_of(t);
      h.off[kp] = h.sl_wide[c] ? int32_t(roff) : len;
      h.dfrom[kp] = diag[i];
      for (int u = 0; u < len; ++u) {
        const int64_t p = q_begin(i) + u;
        const int64_t e = h.sl_wide[c] ? roff + u : int64_t(dstart[uo[t] + u]) + ti[t];  // in chunk
        const int64_t qq = h.sl_q[c] + e;
        const int32_t jr = cols[p];
        h.from[qq] = int32_t(p);
        if (h.sl_wide[c]) {
          // wide launches read global memory directly; a source in the row's
          // own task is its index within the task (the same thread / warp
          // computed it just before)
          h.src[qq] = task_of[jr] == task_of[i] ? h.pos[jr] - h.pos[T.rows[T.ptr[task_of[i]]]]
                                                : -(jr + 1);
          continue;
        }
        const int cj = chunk_of_row[jr];
        bool in_ring = false;
        int owner = 0;
        if (S && !h.sl_wide[cj] && seg_of[cj] == seg_of[c]) {
          // push walker: the owner's replica slot is rewritten once the owner
          // runs past the next sub-level (peers are at most one ahead)
          owner = (cj - seg_first[cj]) % C;
          const int nx = sub_first + C + owner;
          const int oc = (nx < nch && seg_of[nx] == seg_of[c]) ? nx : sub_first + owner;
          // (S - 2: the bulk push also rewrites one pad slot past the chunk)
          in_ring = int64_t(h.sl_r0[oc]) + h.sl_nr[oc] - int64_t(lpos[jr]) <= S - 2;
        } else if (flow && !h.sl_wide[cj] && seg_of[cj] == seg_of[c]) {
          // dataflow: position s is overwritten by s + kRing, written no
          // earlier than chunk c + 2 (consumers run at most two chunks apart)
          const int cn = (c + 1 < nch && seg_of[c + 1] == seg_of[c]) ? c + 1 : c;
          in_ring = int64_t(h.sl_r0[cn]) + h.sl_nr[cn] - int64_t(lpos[jr]) <= kRing;
        } else if (!h.sl_wide[cj] && seg_of[cj] == seg_of[c]) {
          owner = (cj - seg_first[cj]) % C;
          // the owner's ring end at this sub-level: its chunk in this sub-level
          const int oc = sub_first + owner;
          const int64_t oend = (oc < nch && seg_of[oc] == seg_of[c])
                                   ? int64_t(h.sl_r0[oc]) + h.sl_nr[oc]
                                   : int64_t(lpos[jr]) + 1;
          in_ring = oend - int64_t(lpos[jr]) <= kRing;
        }
        if (in_ring) {
          // dataflow walker: the source's position (slot and readiness tag)
          h.src[qq] = S      ? owner * S + (lpos[jr] & (S - 1))
                      : flow ? lpos[jr]
                             : (owner << 12) | (lpos[jr] & (kRing - 1));
        } else if (h.sl_wide[cj] || seg_of[cj] != seg_of[c]) {
          // final before this launch: gathered into sfv, product by a producer
          h.src[qq] = -1;
          h.sfar.push_back(int32_t(e));
          h.sfar.push_back(jr);
          ++ns;
        } else if (S) {
          // push walker: out of the ring window, read from the source's
          // long-range slot (its owner pushes it there as well); slots are
          // assigned below, once every reader is known
          side_q.emplace_back(qq, jr);
          const int sub_r = (c - seg_first[c]) / C;
          if (last_read[jr] < sub_r) last_read[jr] = sub_r;
        } else {
          // out of the ring window: a producer forms this product from y
          h.src[qq] = -1;
          h.far.push_back(int32_t(e));
          h.far.push_back(jr);
          ++nf;
        }
      }
      roff += len;
    }
    h.sl_f[c + 1] = h.sl_f[c] + nf;
    h.sl_s[c + 1] = h.sl_s[c] + ns;
    h.sl_nfar.push_back(nf + ns);
  }
  if (S && !side_q.empty()) {
    // long-range slots, recycled: a slot is written at its row's sub-level
    // w and read up to sub-level r; peers run at most one sub-level ahead,
    // so the next value may take the slot from sub-level r + 2 on. Slots
    // are per walker launch (segment).
    std::vector<int32_t> need;
    for (int64_t i = 0; i < n; ++i)
      if (last_read[i] >= 0) need.push_back(int32_t(i));
    auto wsub = [&](int32_t i) {
      const int cj = chunk_of_row[i];
      return std::make_pair(seg_of[cj], (cj - seg_first[cj]) / C);
    };
    std::stable_sort(need.begin(), need.end(), [&](int32_t x, int32_t y2) { return wsub(x) < wsub(y2); });
    // busy slots by the sub-level they become free; idle slots
    std::priority_queue<std::pair<int, int>, std::vector<std::pair<int, int>>, std::greater<>> busy;
    std::vector<int> idle;
    int cur_seg = -1;
    for (const int32_t i : need) {
      const auto w = wsub(i);
      if (w.first != cur_seg) {
        cur_seg = w.first;
        busy = {};
        idle.clear();
        for (int z = kSide - 1; z >= 0; --z) idle.push_back(z);
      }
      while (!busy.empty() && busy.top().first <= w.second) {
        idle.push_back(busy.top().second);
        busy.pop();
      }
      if (idle.empty()) {
        h.push_ok = false;
        if (getenv("PSCU_PLAN_DEBUG")) fprintf(stderr, "push plan: long-range slots exhausted\n");
        return;
      }
      const int slot = idle.back();
      idle.pop_back();
      busy.emplace(last_read[i] + 2, slot);
      h.side[i] = slot + 1;
    }
    for (const auto& e : side_q) h.src[e.first] = kRingTotal + h.side[e.second] - 1;
  }
}

/// Cluster size for a sweep (measured: tools/sweep_cluster.sh): four CTAs when
/// an average level fits about one chunk, else kMaxCluster CTAs, whose rings
/// also keep the wide fine-level wavefronts resident.
int pick_cluster(const Csr& a, const std::vector<int64_t>& diag, bool fwd) {
  if (const char* e = getenv(fwd ? "PSCU_WALK_CLUSTER_FWD" : "PSCU_WALK_CLUSTER_BWD"))
    return std::max(1, std::min(kMaxCluster, atoi(e)));
  if (const char* e = getenv("PSCU_WALK_CLUSTER")) return std::max(1, std::min(kMaxCluster, atoi(e)));
  int nlev = 0;
  const std::vector<int32_t> lvl = dag_levels(a, diag, fwd, nlev);
  std::vector<int64_t> rows(nlev, 0), nz(nlev, 0);
  for (int64_t i = 0; i < a.n; ++i) {
    rows[lvl[i]]++;
    nz[lvl[i]] += fwd ? diag[i] - a.h_row_ptr[i] : a.h_row_ptr[i + 1] - diag[i] - 1;
  }
  int64_t nr = 0, nq = 0, cnt = 0;
  for (int l = 0; l < nlev; ++l)
    if (rows[l] <= kWideRows) {
      nr += rows[l];
      nq += nz[l];
      ++cnt;
    }
  if (!cnt) return 1;
  // narrow sweeps (the coarse level): four CTAs with the push walker
  // (256^2 coarse apply: 1.49 ms with 4 CTAs, 1.54 ms with 2, 2.24 ms with
  // one CTA of the level walker); wide sweeps: kMaxCluster
  return (2 * nr <= 3 * int64_t(kStageRows) * cnt && nq <= int64_t(kMaxNz) * cnt) ? 4 : kMaxCluster;
}

/// Chain cap of a task-level plan: a dataflow / level step costs a fixed
/// latency (~2.5 us: source loads, the value hand-over) plus the serial fold
/// of its longest task (~26 cycles per entry), i.e. about 180 entries' worth
/// per level. Short chains mean more levels, long ones longer folds; both
/// caps are planned and the cheaper one kept (256^2 k=3: 16; 3D coarse
/// face blocks: 4). PSCU_LEVEL_CHAIN_ROWS fixes the cap.
Tasks level_tasks(const Csr& a, const std::vector<int64_t>& diag, bool fwd, Tasks* t16 = nullptr) {
  if (getenv("PSCU_LEVEL_CHAIN_ROWS")) {
    Tasks T = build_tasks(a, diag, fwd, level_chain_rows(), level_chain_nz(), level_pad());
    if (t16) *t16 = T;
    return T;
  }
  Tasks T4;
  std::thread th([&] { T4 = build_tasks(a, diag, fwd, 4, level_chain_nz(), level_pad()); });
  Tasks T16 = build_tasks(a, diag, fwd, 16, level_chain_nz(), level_pad());
  th.join();
  auto cost = [](const Tasks& T) {
    std::vector<int64_t> mx(T.nlev, 0);
    for (size_t t = 0; t < T.lvl.size(); ++t) mx[T.lvl[t]] = std::max<int64_t>(mx[T.lvl[t]], T.nz[t]);
    int64_t c = 0;
    for (int l = 0; l < T.nlev; ++l) c += 180 + mx[l];
    return c;
  };
  if (t16) *t16 = T16;
  return cost(T4) < cost(T16) ? T4 : T16;
}

HostPlan plan(const Csr& a, const std::vector<int64_t>& diag, bool fwd) {
  HostPlan h;
  if (a.nnz >= (int64_t(1) << 31))
    throw Error(PSCU_EINVAL, "walk plan: more than 2^31 factor entries per level are not supported");
  const char* mode = getenv("PSCU_WALK_MODE");
  if (mode && !strcmp(mode, "levels")) {
    plan_sweep(a, diag, fwd, 1, false, 0, level_chain_rows(), h, true);
    return h;
  }
  if (!mode && !getenv("PSCU_WALK_CLUSTER") && !getenv("PSCU_WALK_CLUSTER_FWD") &&
      !getenv("PSCU_WALK_CLUSTER_BWD")) {
    // wide sweeps (the fine levels: thousands of rows per task level) are
    // too much data per level for the rings: task-level launches. Narrow
    // ones (the coarse level, ~2 k rows per task level at 256^2): the push
    // walker on four CTAs (1.05 ms per 256^2 coarse apply; 1.01 ms on 8).
    Tasks T16;
    const Tasks T = level_tasks(a, diag, fwd, &T16);
    if (a.n >= int64_t(3000) * std::max(1, T16.nlev)) {
      plan_sweep(a, diag, fwd, 1, false, 0, level_chain_rows(), h, true, &T);
      return h;
    }
    const int pc = [] {
      const char* e = getenv("PSCU_PUSH_CTAS");
      const int v = e ? atoi(e) : 4;
      return v == 2 || v == 8 ? v : 4;
    }();
    plan_sweep(a, diag, fwd, pc, false, kRingTotal / pc, chain_rows(fwd), h);
    if (h.push_ok) return h;
    plan_sweep(a, diag, fwd, 1, false, 0, level_chain_rows(), h, true, &T);
    return h;
  }
  const int C = pick_cluster(a, diag, fwd);
  if (C == kMaxCluster && !mode) {
    // wide sweeps (the fine levels): too much data per level for the rings
    plan_sweep(a, diag, fwd, 1, false, 0, level_chain_rows(), h, true);
    return h;
  }
  if ((C > 1 || getenv("PSCU_WALK_PUSH1")) && !getenv("PSCU_WALK_NOPUSH")) {
    const int g = chain_rows();
    plan_sweep(a, diag, fwd, C, false, kRingTotal / C, g, h);
    if (h.push_ok) return h;
    if (g > 1 && mode && !strcmp(mode, "push1")) {
      plan_sweep(a, diag, fwd, C, false, kRingTotal / C, 1, h);
      if (h.push_ok) return h;
    }
    if (!(mode && !strcmp(mode, "walker"))) {
      // too much data per level for the rings: every task level becomes one
      // task-parallel launch (the chains cut the fine-level depth ~12x)
      plan_sweep(a, diag, fwd, 1, false, 0, level_chain_rows(), h, true);
      return h;
    }
  }
  // the dataflow walker is correct but not yet faster than the level walker
  const bool flow = C == 1 && getenv("PSCU_WALK_FLOW");
  plan_sweep(a, diag, fwd, C, flow, 0, 1, h);
  return h;
}

/// One cooperative launch per level-plan sweep (grid barrier between task
/// levels) instead of one launch per task level: 256^2 applies k=3 10.3 ->
/// 8.5 ms, k=2 6.9 -> 6.5 ms, k=1 4.8 -> 5.2 ms (measured); on by default.
static bool level_persist() {
  static const bool v = [] {
    const char* e = getenv("PSCU_LEVEL_PERSIST");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

/// Dataflow (barrier-free) level-plan sweeps: PSCU_LEVEL_FLOW (default on).
static bool level_flow() {
  static const bool v = [] {
    const char* e = getenv("PSCU_LEVEL_FLOW");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

void upload_plan(Context& c, const HostPlan& h, bool fwd, WalkPlan& w) {
  cudaStream_t st = c.stream;
  w.fwd = fwd;
  w.C = h.C;
  w.levels = h.levels;
  w.persist_grid = 0;
  // the warp kernel (level_chunk) buffers at most kLevelMaxRows rows and
  // kLevelMaxNz entries per task: a wide chunk with a larger task (a single
  // row longer than the entry cap, or a push-walker chunk of long chains)
  // runs on the thread-per-task wide_kernel instead, and such a plan is
  // never swept by the persistent kernel
  std::vector<char> warp_fits(h.sl_k.size(), 0);
  bool all_fit = true;
  for (size_t s = 0; s < h.sl_k.size(); ++s) {
    if (!h.sl_wide[s]) continue;
    bool ok = true;
    for (int i = 0; i < h.sl_nt[s] && ok; ++i) {
      const int32_t t0 = h.sl_t[s] + i;
      ok = h.tt[t0 + 1] - h.tt[t0] <= kLevelMaxRows && h.tq[t0 + 1] - h.tq[t0] <= kLevelMaxNz;
    }
    warp_fits[s] = ok;
    all_fit = all_fit && ok;
  }
  // (k=1 at 256^2, 1.2 M rows: per-level launches measured faster, 4.8 vs 5.2 ms)
  const char* pm = getenv("PSCU_LEVEL_PERSIST_MIN_ROWS");
  if (h.levels && all_fit && level_persist() && h.npos >= (pm ? atoll(pm) : 1500000)) {
    int per_sm = 0, sms = 0, dev = 0;
    PSCU_CUDA(cudaGetDevice(&dev));
    PSCU_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    void* fn = fwd ? (void*)level_persist_kernel<true> : (void*)level_persist_kernel<false>;
    PSCU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kLevelWarps, 0));
    int most = 0;
    for (size_t s = 0; s < h.sl_nt.size(); ++s) most = std::max(most, h.sl_nt[s]);
    const char* ge = getenv("PSCU_LEVEL_PERSIST_TASKS");
    const int cap = ge ? std::max(32, atoi(ge)) : 1024;  // warps of the grid: arrivals per barrier
    const int want = (std::min(most, cap) + kLevelWarps - 1) / kLevelWarps;
    w.persist_grid = std::max(1, std::min(want, per_sm * sms));
    w.barrier.alloc(1);
  }
  w.flow_grid = 0;
  w.ny = int64_t(h.pos.size());
  if (h.levels && all_fit && level_flow()) {
    int per_sm = 0, sms = 0, dev = 0;
    PSCU_CUDA(cudaGetDevice(&dev));
    PSCU_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const char* fe = getenv("PSCU_LEVEL_FLOW");
    const bool v2 = fe && atoi(fe) == 2;
    int maxnz = 0;
    for (size_t s = 0; s < h.sl_k.size(); ++s)
      for (int i = 0; i < h.sl_nt[s]; ++i) {
        const int32_t t0 = h.sl_t[s] + i;
        maxnz = std::max(maxnz, int(h.tq[t0 + 1] - h.tq[t0]));
      }
    const char* fs = getenv("PSCU_LEVEL_FLOW_SMALL");
    w.flow_small = 0;
    if (!v2 && (!fs || atoi(fs) != 0)) w.flow_small = maxnz <= kFlowSmallNz ? 1 : (maxnz <= kFlowMidNz ? 2 : 0);
    void* fn = flow_kernel_fn(fwd, v2, w.flow_small);
    PSCU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kLevelWarps, 0));
    int most = 0;
    for (size_t s = 0; s < h.sl_nt.size(); ++s) most = std::max(most, h.sl_nt[s]);
    // warps per task of the widest level: > 1 lets consecutive levels run on
    // disjoint warps (with the rotation below)
    const char* go = getenv("PSCU_LEVEL_FLOW_OVERSUB");
    const double over = go ? std::max(0.25, atof(go)) : 2.0;
    const char* ge = getenv("PSCU_LEVEL_FLOW_WARPS");
    const int cap = ge ? std::max(32, atoi(ge)) : 8192;
    const int want = (std::min(int(most * over), cap) + kLevelWarps - 1) / kLevelWarps;
    w.flow_grid = std::max(1, std::min(want, per_sm * sms));
  }
  w.flow = h.flow;
  w.S = h.S;
  w.nsub = int(h.sl_k.size());
  w.npos = h.npos;
  w.segments.clear();
  for (int s = 0; s < w.nsub; ++s) {
    if (h.sl_wide[s]) {
      // one warp per task when the tasks are long chains
      const bool warp = h.sl_nt[s] > 0 && h.sl_nq[s] >= 24 * int64_t(h.sl_nt[s]) && warp_fits[s];
      w.segments.push_back({true, s, s + 1, warp, h.sl_nt[s]});
    } else if (s == 0 || h.sl_wide[s - 1]) {
      w.segments.push_back({false, s, s + 1});
    }
    else w.segments.back().s1 = s + 1;
  }
  w.sl_k.upload(h.sl_k, st);
  w.sl_nr.upload(h.sl_nr, st);
  w.sl_f.upload(h.sl_f, st);
  if (h.far.empty()) w.far.alloc(4);
  else w.far.upload(h.far, st);
  w.sl_s.upload(h.sl_s, st);
  w.h_sl_s = h.sl_s;
  if (h.sfar.empty()) w.sfar.alloc(4);
  else w.sfar.upload(h.sfar, st);
  w.sfv.alloc(std::max<size_t>(4, h.sfar.size() / 2));
  w.sl_q.upload(h.sl_q, st);
  {
    std::vector<int32_t> hdr(size_t(w.nsub) * kHdr, 0);
    int64_t run_tasks = 0;
    for (int s = 0; s < w.nsub; ++s) {
      hdr[size_t(s) * kHdr] = h.sl_k[s];
      hdr[size_t(s) * kHdr + 1] = h.sl_nr[s];
      hdr[size_t(s) * kHdr + 2] = h.sl_nq[s];
      hdr[size_t(s) * kHdr + 3] = h.sl_wide[s] ? 0 : h.sl_nfar[s];
      hdr[size_t(s) * kHdr + 4] = h.sl_r0[s];
      hdr[size_t(s) * kHdr + 5] = h.sl_nd[s];
      hdr[size_t(s) * kHdr + 6] = h.sl_d[s];
      hdr[size_t(s) * kHdr + 8] = h.sl_nt[s];
      hdr[size_t(s) * kHdr + 9] = h.sl_t[s];
      hdr[size_t(s) * kHdr + 10] = int32_t(run_tasks & ((int64_t(1) << 30) - 1));
      // the rotation of the dataflow grid, reduced on the host (a 64-bit
      // modulo per warp and level showed up at 7 % of the kernel's samples)
      if (w.flow_grid > 0)
        hdr[size_t(s) * kHdr + 11] = int32_t(run_tasks % (int64_t(w.flow_grid) * kLevelWarps));
      run_tasks += h.sl_nt[s];
      if (h.S && !h.sl_wide[s]) {
        // bytes the peers of this chunk push during its sub-level
        int first = s;
        while (first > 0 && !h.sl_wide[first - 1]) --first;
        const int sf = first + (s - first) / h.C * h.C;
        int rows = 0;
        for (int o = 0; o < h.C; ++o) {
          if (sf + o == s) continue;
          // ring slice, whole 16-byte pairs (bulk copy) or one slot per row
          rows += kBulkPush ? (h.sl_nr[sf + o] + 1) & ~1 : h.sl_nr[sf + o];
          for (int t = 0; t < h.sl_nr[sf + o]; ++t) {
            const int32_t i = h.rows[h.sl_k[sf + o] + t];
            if (h.side[i]) ++rows;  // long-range copy
          }
        }
        hdr[size_t(s) * kHdr + 7] = 8 * rows;
      }
    }
    w.sl_hdr.upload(hdr, st);
  }
  {
    std::vector<int32_t> tt(h.tt);
    tt.resize((tt.size() + 8) & ~size_t(3), 0);  // whole 16-byte copies past the last table
    w.tt.upload(tt, st);
    std::vector<int32_t> tq(h.tq);
    tq.resize(tt.size(), 0);
    w.tq.upload(tq, st);
  }
  w.rows.upload(h.rows, st);
  w.off.upload(h.off, st);
  if (h.dp.empty()) w.dp.alloc(4);
  else w.dp.upload(h.dp, st);
  w.src.upload(h.src.data(), h.src.size(), st);
  w.from.upload(h.from.data(), h.from.size(), st);
  w.val.alloc(h.from.size());
  if (!fwd) {
    w.dfrom.upload(h.dfrom, st);
    w.dv.alloc(h.dfrom.size());
  } else {
    w.dv.alloc(4);
  }
}

} // namespace

struct WalkBuild {
  HostPlan f, b;
};

std::shared_ptr<WalkBuild> plan_walk(const Csr& a, const std::vector<int64_t>& diag) {
  auto wb = std::make_shared<WalkBuild>();
  if (a.n == 0) return wb;
  // the two sweeps are independent host work
  std::exception_ptr err;
  std::thread tb([&] {
    try {
      wb->b = plan(a, diag, false);
    } catch (...) {
      err = std::current_exception();
    }
  });
  std::exception_ptr err_f;
  try {
    wb->f = plan(a, diag, true);
  } catch (...) {
    err_f = std::current_exception();
  }
  tb.join();  // never unwind past a joinable thread (std::terminate)
  if (err_f) std::rethrow_exception(err_f);
  if (err) std::rethrow_exception(err);
  return wb;
}

void upload_walk(Context& c, const Csr& a, const WalkBuild& b, WalkPlan& wf, WalkPlan& wb) {
  if (a.n == 0) return;
  const HostPlan& hf = b.f;
  const HostPlan& hb = b.b;
  upload_plan(c, hf, true, wf);
  upload_plan(c, hb, false, wb);
  // forward results are written straight into backward position order
  std::vector<int32_t> opos(hf.rows.size(), 0);
  for (size_t k = 0; k < hf.rows.size(); ++k)
    if (hf.rows[k] >= 0) opos[k] = hb.pos[hf.rows[k]];
  wf.opos.upload(opos, c.stream);
  wb.opos.alloc(4);
  for (int dir = 0; dir < 2; ++dir) {
    const HostPlan& h = dir ? hb : hf;
    std::vector<int4> meta(h.rows.size());
    for (size_t k = 0; k < h.rows.size(); ++k)
      meta[k] = make_int4(h.off[k], h.rows[k] >= 0 ? h.rows[k] : 0, dir ? 0 : opos[k],
                          h.S && h.rows[k] >= 0 ? h.side[h.rows[k]] : 0);
    (dir ? wb : wf).meta.upload(meta, c.stream);
  }
  wf.scratch.alloc(size_t(hf.npos) + 8);  // rhs in forward position order
  if (hf.levels || hb.levels) wf.ybuf.alloc(size_t(a.n));
  wb.scratch.alloc(size_t(hb.npos) + 8);  // forward result in backward position order
  PSCU_CUDA(cudaMemsetAsync(wb.scratch.p, 0, sizeof(double) * (hb.npos + 8), c.stream));
  if (getenv("PSCU_DEBUG")) {
    for (const HostPlan* h : {&hf, &hb}) {
      int64_t ring = 0, far = 0;
      for (size_t q = 0; q < h->from.size(); ++q)
        if (h->from[q] >= 0) (h->src[q] >= 0 ? ring : far)++;
      fprintf(stderr, "[walk %s] static out-of-ring %zu, in-segment out-of-ring %zu\n",
              h == &hf ? "fwd" : "bwd", h->sfar.size() / 2, h->far.size() / 2);
      int nw = 0;
      for (auto x : h->sl_wide) nw += x;
      fprintf(stderr,
              "[walk %s] n=%lld cluster=%d %s chunks=%zu (wide %d) positions=%lld ring=%lld "
              "far=%lld\n",
              h == &hf ? "fwd" : "bwd", (long long)a.n, h->C,
              h->S ? "push" : (h->flow ? "flow" : "level"), h->sl_k.size(), nw,
              (long long)h->npos, (long long)ring, (long long)far);
    }
  }
}

void build_walk(Context& c, const Csr& a, const std::vector<int64_t>& diag, WalkPlan& wf,
                WalkPlan& wb) {
  upload_walk(c, a, *plan_walk(a, diag), wf, wb);
}

void pack_walk(Context& c, const double* lu, WalkPlan& w) {
  const int64_t m = int64_t(w.val.n);
  if (m) {
    gather_vals<<<grid1(m), 256, 0, c.stream>>>(m, w.from.p, lu, w.val.p);
    PSCU_LAUNCHED(&c);
  }
  if (!w.fwd) {
    const int64_t nd = int64_t(w.dv.n);
    gather_vals<<<grid1(nd), 256, 0, c.stream>>>(nd, w.dfrom.p, lu, w.dv.p);
    PSCU_LAUNCHED(&c);
  }
}

size_t flow_smem() { return sizeof(ulonglong2) * kRing + kFlowStages * sizeof(Stage); }

static void launch_flow(Context& c, bool fwd, const WalkArgs& a, int c0, int nch,
                        const double* rhs, double* y, double* yb) {
  static bool attr = false;
  if (!attr) {
    for (void* f : {(void*)flow_kernel<true>, (void*)flow_kernel<false>})
      PSCU_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(flow_smem())));
    attr = true;
  }
  const unsigned threads = kWalkThreads + 64 * kFlowStages;
  if (fwd) flow_kernel<true><<<1, threads, flow_smem(), c.stream>>>(a, c0, nch, rhs, y, yb);
  else flow_kernel<false><<<1, threads, flow_smem(), c.stream>>>(a, c0, nch, rhs, y, yb);
  PSCU_LAUNCHED(&c);
}

size_t push_smem() { return sizeof(double) * (kRingTotal + kSide) + kPushStages * sizeof(Stage); }

static int push_consumers() {
  static const int v = [] {
    const char* e = getenv("PSCU_PUSH_CONSUMERS");
    return e && atoi(e) == 512 ? 512 : kPushConsumers;
  }();
  return v;
}

template <int kCons>
static void launch_push_t(Context& c, bool fwd, const WalkArgs& a, int c0, int nsl, int C, int S,
                          const double* rhs, double* y, double* yb) {
  static bool attr = false;
  if (!attr) {
    for (void* f : {(void*)push_kernel<true, kCons>, (void*)push_kernel<false, kCons>}) {
      PSCU_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(push_smem())));
      PSCU_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(C));
  cfg.blockDim = dim3(kCons + 32 * kPushProdWarps * kPushStages);
  cfg.dynamicSmemBytes = push_smem();
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(C);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (fwd) PSCU_CUDA(cudaLaunchKernelEx(&cfg, push_kernel<true, kCons>, a, c0, nsl, C, S, rhs, y, yb));
  else PSCU_CUDA(cudaLaunchKernelEx(&cfg, push_kernel<false, kCons>, a, c0, nsl, C, S, rhs, y, yb));
  PSCU_LAUNCHED(&c);
}

static void launch_push(Context& c, bool fwd, const WalkArgs& a, int c0, int nsl, int C, int S,
                        const double* rhs, double* y, double* yb) {
  if (push_consumers() == 512) launch_push_t<512>(c, fwd, a, c0, nsl, C, S, rhs, y, yb);
  else launch_push_t<kPushConsumers>(c, fwd, a, c0, nsl, C, S, rhs, y, yb);
}

static void launch_walker(Context& c, bool fwd, const WalkArgs& a, int c0, int nsl, int C,
                          const double* rhs, double* y, double* yb) {
  static bool attr = false;
  if (!attr) {
    for (void* f : {(void*)walk_kernel<true>, (void*)walk_kernel<false>}) {
      PSCU_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(walk_smem())));
    }
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(C));
  cfg.blockDim = dim3(kWalkThreads + kProducers);
  cfg.dynamicSmemBytes = walk_smem();
  cfg.stream = c.stream;
  cudaLaunchAttribute attr_c[1];
  attr_c[0].id = cudaLaunchAttributeClusterDimension;
  attr_c[0].val.clusterDim.x = unsigned(C);
  attr_c[0].val.clusterDim.y = 1;
  attr_c[0].val.clusterDim.z = 1;
  cfg.attrs = attr_c;
  cfg.numAttrs = 1;
  if (fwd) PSCU_CUDA(cudaLaunchKernelEx(&cfg, walk_kernel<true>, a, c0, nsl, C, rhs, y, yb));
  else PSCU_CUDA(cudaLaunchKernelEx(&cfg, walk_kernel<false>, a, c0, nsl, C, rhs, y, yb));
  PSCU_LAUNCHED(&c);
}

/// PSCU_WALK_TRACE=1: stamps of CTA 0 per sub-level, summarised on stderr
/// after every walker launch (diagnostics only; synchronises the stream).
static long long* trace_buffer() {
  static long long* buf = [] {
    long long* p = nullptr;
    if (getenv("PSCU_WALK_TRACE")) {
      cudaMalloc(&p, sizeof(long long) * kTraceSub * 16 * kMaxCluster);
      cudaMemset(p, 0, sizeof(long long) * kTraceSub * 16 * kMaxCluster);
    }
    return p;
  }();
  return buf;
}

static void trace_report(Context& c, bool fwd, int C, int nsl) {
  const int ranks = C > 1 ? C : 1;
  std::vector<long long> all(size_t(kTraceSub) * 16 * ranks);
  PSCU_CUDA(cudaMemcpyAsync(all.data(), trace_buffer(), sizeof(long long) * all.size(),
                            cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  const int hi = std::min(nsl, kTraceSub) - 1;
  if (hi <= 9) return;
  for (int rk = 0; rk < ranks; ++rk) {
    const long long* t = all.data() + size_t(rk) * kTraceSub * 16;
    double d[8] = {0}, e3[3] = {0};
    const int n = hi - 8;
    for (int r = 8; r < hi; ++r) {
      const long long* x = &t[size_t(r) * 16];
      if (x[5] > x[2] && x[6] >= x[5] && x[7] >= x[6]) {
        e3[0] += x[5] - x[2];  // thread 0: first row folded
        e3[1] += x[6] - x[5];  // its ring writes + pushes
        e3[2] += x[3] - x[7];  // thread 0 done -> sub-level barrier passed
      }
      d[0] += x[1] - x[0];                  // consumer wait full
      d[1] += x[2] - x[1];                  // products
      d[2] += x[3] - x[2];                  // rows
      d[3] += x[4] - x[3];                  // cluster handshake
      d[4] += t[size_t(r + 1) * 16] - x[0];  // consumer loop
      d[5] += x[9] - x[8];                  // producer wait empty
      d[6] += x[10] - x[9];                 // TMA landing
      d[7] += x[11] - x[10];                // out-of-ring products
    }
    fprintf(stderr,
            "[walk trace %s C=%d rank=%d sub-levels=%d] cycles/sub-level: wait_full %.0f products "
            "%.0f rows %.0f handshake %.0f | loop %.0f | producer: wait_empty %.0f landing %.0f "
            "far %.0f\n",
            fwd ? "fwd" : "bwd", C, rk, nsl, d[0] / n, d[1] / n, d[2] / n, d[3] / n, d[4] / n,
            d[5] / n, d[6] / n, d[7] / n);
    fprintf(stderr, "    thread 0: fold %.0f, push %.0f, wait at barrier %.0f\n", e3[0] / n, e3[1] / n,
            e3[2] / n);
  }
}

static void level_trace_report(Context& c, const WalkPlan& w) {
  std::vector<long long> all(size_t(kTraceSub) * 16);
  PSCU_CUDA(cudaMemcpyAsync(all.data(), trace_buffer(), sizeof(long long) * all.size(),
                            cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  double ld = 0, fold = 0, ne = 0, nr = 0;
  int cnt = 0;
  for (int ch = 1; ch < std::min(w.nsub, kTraceSub); ++ch) {
    const long long* t = &all[size_t(ch) * 16];
    if (t[2] <= t[0]) continue;
    ld += double(t[1] - t[0]);
    fold += double(t[2] - t[1]);
    ne += double(t[3]);
    nr += double(t[4]);
    ++cnt;
  }
  if (cnt)
    fprintf(stderr, "[level trace %s] tasks sampled %d: loads %.0f cycles, fold %.0f cycles, entries %.0f, rows %.1f\n",
            w.fwd ? "fwd" : "bwd", cnt, ld / cnt, fold / cnt, ne / cnt, nr / cnt);
  {
    std::vector<long long> g(8192 * 2);
    PSCU_CUDA(cudaMemcpy(g.data(), trace_buffer() + size_t(kTraceSub) * 16, sizeof(long long) * g.size(),
                         cudaMemcpyDeviceToHost));
    long long mn = -1, mx = 0, dmax = 0, smax = 0;
    std::vector<long long> d;
    for (int t = 0; t < 8192; ++t) {
      if (g[2 * t] <= 0 || g[2 * t + 1] < g[2 * t]) continue;
      if (mn < 0 || g[2 * t] < mn) mn = g[2 * t];
      mx = std::max(mx, g[2 * t + 1]);
      d.push_back(g[2 * t + 1] - g[2 * t]);
    }
    if (!d.empty()) {
      std::sort(d.begin(), d.end());
      for (int t = 0; t < 8192; ++t)
        if (g[2 * t] > 0) smax = std::max(smax, g[2 * t] - mn);
      dmax = d.back();
      fprintf(stderr, "[level trace %s] chunk 100: %zu tasks, span %.1f us, task median %.1f us max %.1f us, last start +%.1f us\n",
              w.fwd ? "fwd" : "bwd", d.size(), (mx - mn) / 1e3, d[d.size() / 2] / 1e3, dmax / 1e3, smax / 1e3);
    }
    PSCU_CUDA(cudaMemset(trace_buffer() + size_t(kTraceSub) * 16, 0, sizeof(long long) * g.size()));
  }
}

static void run_one(Context& c, const WalkPlan& w, const double* rhs, double* y, double* yb) {
  WalkArgs a = args_of(w);
  a.trace = trace_buffer();
  if (w.levels && w.flow_grid > 0 && !a.trace) {
#ifdef PSCU_TRACE
    // PSCU_FLOW_TRACE=<prefix>: globaltimer stamps {start, operands loaded,
    // sources arrived, folded} of every task of the PSCU_FLOW_TRACE_APPLY-th
    // sweep of the largest plan traced so far, dumped to <prefix>_{fwd,bwd}.bin
    // with the chunk table (task-table start, task count per chunk)
    static int sweep_no = 0;
    static const char* ft_path = getenv("PSCU_FLOW_TRACE");
    static const int ft_at = getenv("PSCU_FLOW_TRACE_APPLY") ? atoi(getenv("PSCU_FLOW_TRACE_APPLY")) : 50;
    DevBuf<long long> ftb;
    const bool ft_now = ft_path && w.ny > 100000 && sweep_no++ / 2 == ft_at;
    if (ft_now) {
      ftb.alloc(size_t(w.tt.n) * 6 + 6);
      PSCU_CUDA(cudaMemsetAsync(ftb.p, 0, sizeof(long long) * (size_t(w.tt.n) * 6 + 6), c.stream));
      a.ftrace = ftb.p;
    }
#endif
    fill_sentinel<<<grid1(w.ny), 256, 0, c.stream>>>(w.ny, y);
    PSCU_LAUNCHED(&c);
    int c0 = 0, c1 = w.nsub;
    void* args[] = {&a, &c0, &c1, (void*)&rhs, (void*)&y, (void*)&yb};
    static const bool v2 = [] {
      const char* e = getenv("PSCU_LEVEL_FLOW");
      return e && atoi(e) == 2;
    }();
    void* fn = flow_kernel_fn(w.fwd, v2, w.flow_small);
    PSCU_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(w.flow_grid)), dim3(32 * kLevelWarps),
                                          args, 0, c.stream));
    PSCU_LAUNCHED(&c);
#ifdef PSCU_TRACE
    if (ft_now) {
      std::vector<long long> st(size_t(w.tt.n) * 6);
      std::vector<int32_t> hdr(size_t(w.nsub) * kHdr);
      PSCU_CUDA(cudaMemcpyAsync(st.data(), ftb.p, sizeof(long long) * st.size(), cudaMemcpyDeviceToHost, c.stream));
      PSCU_CUDA(cudaMemcpyAsync(hdr.data(), w.sl_hdr.p, sizeof(int32_t) * hdr.size(), cudaMemcpyDeviceToHost, c.stream));
      PSCU_CUDA(cudaStreamSynchronize(c.stream));
      const std::string path = std::string(ft_path) + (w.fwd ? "_fwd.bin" : "_bwd.bin");
      if (FILE* f = fopen(path.c_str(), "wb")) {
        const int64_t nsub = w.nsub, ntt = int64_t(w.tt.n);
        fwrite(&nsub, 8, 1, f);
        fwrite(&ntt, 8, 1, f);
        fwrite(hdr.data(), sizeof(int32_t), hdr.size(), f);
        fwrite(st.data(), sizeof(long long), st.size(), f);
        fclose(f);
      }
    }
#endif
    return;
  }
  if (w.levels && w.persist_grid > 0 && !a.trace) {
    // every task level of the sweep in one cooperative launch
    PSCU_CUDA(cudaMemsetAsync(w.barrier.p, 0, sizeof(unsigned long long), c.stream));
    int c0 = 0, c1 = w.nsub;
    void* args[] = {&a, &c0, &c1, (void*)&rhs, (void*)&y, (void*)&yb, (void*)&w.barrier.p};
    void* fn = w.fwd ? (void*)level_persist_kernel<true> : (void*)level_persist_kernel<false>;
    PSCU_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(w.persist_grid)), dim3(32 * kLevelWarps),
                                          args, 0, c.stream));
    PSCU_LAUNCHED(&c);
    return;
  }
  for (const WalkSeg& s : w.segments) {
    if (s.wide && s.warp) {
      const unsigned g = unsigned(std::max(1, std::min(148 * 8, (s.tasks + kLevelWarps - 1) / kLevelWarps)));
      // PDL measured neutral (k=3 11.6 vs 10.3 ms, k=1 4.0 vs 4.8 ms): opt-in
      static const bool pdl = [] {
        const char* e = getenv("PSCU_LEVEL_PDL");
        return e ? atoi(e) != 0 : false;
      }();
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(g);
      cfg.blockDim = dim3(32 * kLevelWarps);
      cfg.stream = c.stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      const int s0 = s.s0;
      if (w.fwd) PSCU_CUDA(cudaLaunchKernelEx(&cfg, level_kernel<true>, a, s0, rhs, y, yb));
      else PSCU_CUDA(cudaLaunchKernelEx(&cfg, level_kernel<false>, a, s0, rhs, y, yb));
      PSCU_LAUNCHED(&c);
    } else if (s.wide) {
      if (w.fwd) wide_kernel<true><<<148 * 4, 256, 0, c.stream>>>(a, s.s0, rhs, y, yb);
      else wide_kernel<false><<<148 * 4, 256, 0, c.stream>>>(a, s.s0, rhs, y, yb);
      PSCU_LAUNCHED(&c);
    } else {
      // static out-of-ring sources of this launch: final now, gather them
      const int64_t g0 = w.h_sl_s[s.s0], g1 = w.h_sl_s[s.s1];
      if (g1 > g0) {
        gather_static<<<grid1(g1 - g0), 256, 0, c.stream>>>(
            g1 - g0, reinterpret_cast<const int2*>(w.sfar.p) + g0, y, w.sfv.p + g0);
        PSCU_LAUNCHED(&c);
      }
      const int nch = s.s1 - s.s0;
      if (w.S) launch_push(c, w.fwd, a, s.s0, nch / w.C, w.C, w.S, rhs, y, yb);
      else if (w.flow) launch_flow(c, w.fwd, a, s.s0, nch, rhs, y, yb);
      else launch_walker(c, w.fwd, a, s.s0, nch / w.C, w.C, rhs, y, yb);
#ifdef PSCU_TRACE
      if (a.trace) trace_report(c, w.fwd, w.flow ? 0 : w.C, w.flow ? nch : nch / w.C);
#endif
    }
  }
#ifdef PSCU_TRACE
  if (a.trace && w.levels) level_trace_report(c, w);
#endif
}

void run_walk(Context& c, const WalkPlan& wf, const WalkPlan& wb, const double* x, double* y) {
  // rhs into forward position order, forward sweep (also scattering its
  // result into backward position order), backward sweep in place on y
  gather_rhs<<<grid1(wf.npos), 256, 0, c.stream>>>(wf.npos, wf.rows.p, x, wf.scratch.p);
  PSCU_LAUNCHED(&c);
  static const bool graphs = [] {
    const char* e = getenv("PSCU_WALK_GRAPH");
    return e ? atoi(e) != 0 : true;
  }();
  if (graphs && (wf.levels || wb.levels) && wf.persist_grid == 0 && wb.persist_grid == 0 &&
      wf.flow_grid == 0 && wb.flow_grid == 0 &&
      wf.segments.size() + wb.segments.size() > 16) {
    // hundreds of task-level launches: replay them as one captured graph on
    // fixed buffers (the launch rate no longer bounds the sweep)
    const int64_t n = int64_t(wf.ybuf.n);
    if (!wf.graph) {
      auto g = std::make_shared<WalkPlan::Graph>();
      const long long before = c.launches;
      cudaGraph_t graph = nullptr;
      PSCU_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
      try {
        run_one(c, wf, wf.scratch.p, wf.ybuf.p, wb.scratch.p);
        run_one(c, wb, wb.scratch.p, wf.ybuf.p, nullptr);
      } catch (...) {
        cudaStreamEndCapture(c.stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      PSCU_CUDA(cudaStreamEndCapture(c.stream, &graph));
      const cudaError_t e = cudaGraphInstantiate(&g->exec, graph, 0);
      cudaGraphDestroy(graph);
      PSCU_CUDA(e);
      g->kernels = c.launches - before;
      c.launches = before;
      wf.graph = g;
    }
    PSCU_CUDA(cudaGraphLaunch(wf.graph->exec, c.stream));
    c.launches += wf.graph->kernels;
    PSCU_CUDA(cudaMemcpyAsync(y, wf.ybuf.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  run_one(c, wf, wf.scratch.p, y, wb.scratch.p);
  run_one(c, wb, wb.scratch.p, y, nullptr);
}

} // namespace pscu
