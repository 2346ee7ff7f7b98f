// Level-walking sparse triangular sweeps for Ilu0::apply (ilu0.hpp:53-65).
//
// The reference applies ILU(0) with two sequential loops. Their dependency
// DAG under the natural (faces-first) ordering is deep and narrow: thousands
// of levels of a few hundred rows. Any scheme that pays
// an inter-SM handshake per level is latency-bound at ~1 us per level, so
// narrow levels are walked by ONE CTA:
//   * rows are stored in level order, and for every row the factor entries
//     it needs are packed contiguously in the reference's summation order
//     (value + source), so a level's data is one contiguous block;
//   * while level l is computed, level l+1's block is copied into the other
//     half of a shared-memory double buffer with cp.async;
//   * solution values of recently finished rows live in a shared-memory ring
//     indexed by schedule position (sources farther back than the ring, or
//     from other segments, are read from global memory);
//   * one __syncthreads per level, no global-memory handshake at all.
// Levels too wide for one CTA (e.g. the element-pressure rows, 10^5 per
// level) run as ordinary row-parallel launches between walker segments.
// Each row is still computed by one thread with the reference's exact
// operation sequence, so the result is bit-identical to Ilu0::apply.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"
#include "walk.cuh"

namespace pscu {

namespace {

constexpr int kWalkThreads = 1024;  // max rows of a walked level
constexpr int kStageRows = 512;     // max rows of a staged level
constexpr int kMaxNz = 2048;        // max packed entries of a staged level
constexpr int kAhead = 3;           // static data is staged this many levels ahead
constexpr int kStages = kAhead + 1;
constexpr int kRing = 4096;         // shared-memory solution ring (positions)

struct WalkArgs {
  const int32_t* lvl_ptr;   // levels+1 into rows
  const int64_t* lvl_nz;    // levels+1 into packed entries (16-byte aligned starts)
  const int32_t* rows;      // row id per schedule position
  const int32_t* row_off;   // packed offset of a row relative to its level start
  const double* val;        // packed factor values
  const int32_t* src;       // >= 0 ring slot, < 0: -(row)-1 global source
  const double* div;        // backward: diagonal per schedule position
  const uint8_t* mode;      // per level: 0 staged, 1 walked from global, 2 wide launch
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

/// Static data of one staged level: packed factor entries, row ids, row
/// offsets and (backward) diagonals. kStages-deep ring.
struct alignas(16) Stage {
  double val[kMaxNz];
  int32_t src[kMaxNz];
  double dv[kStageRows];
  int32_t row[kStageRows];
  int32_t off[kStageRows + 4];
};

/// Group B: the static data of level lv (issued kAhead levels ahead).
template <bool kFwd>
__device__ void stage_static(const WalkArgs& a, int lv, Stage& st) {
  if (a.mode[lv] != 0) return;
  const int k0 = a.lvl_ptr[lv], nr = a.lvl_ptr[lv + 1] - k0;
  const int64_t q0 = a.lvl_nz[lv];
  const int nq = int(a.lvl_nz[lv + 1] - q0);
  // 16-byte chunks: level starts are 16-byte aligned and the arrays padded
  for (int c = threadIdx.x; c * 2 < nq; c += blockDim.x) cp_async16(&st.val[2 * c], a.val + q0 + 2 * c);
  for (int c = threadIdx.x; c * 4 < nq; c += blockDim.x) cp_async16(&st.src[4 * c], a.src + q0 + 4 * c);
  for (int t = threadIdx.x; t < nr; t += blockDim.x) {
    cp_async4(&st.row[t], a.rows + k0 + t);
    cp_async4(&st.off[t], a.row_off + k0 + t);
    if (!kFwd) cp_async8(&st.dv[t], a.div + k0 + t);
  }
  if (threadIdx.x == 0) st.off[nr] = nq;
}

/// Group A: the right-hand side entries of level lv's rows (row ids from
/// its already-landed stage).
__device__ void stage_rhs(const WalkArgs& a, int lv, const Stage& st, double* xb,
                          const double* xin) {
  if (a.mode[lv] != 0) return;
  const int nr = a.lvl_ptr[lv + 1] - a.lvl_ptr[lv];
  for (int t = threadIdx.x; t < nr; t += blockDim.x) cp_async8(&xb[t], xin + st.row[t]);
}

template <bool kFwd>
__global__ void __launch_bounds__(kWalkThreads, 1)
    walk_kernel(WalkArgs a, int l0, int l1, const double* xin, double* y) {
  extern __shared__ __align__(16) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);
  double* xbuf = ring + kRing;  // [2][kStageRows]
  Stage* stages = reinterpret_cast<Stage*>(xbuf + 2 * kStageRows);
  // prologue: static data of the first kAhead levels, then level l0's rhs
  for (int d = 0; d < kAhead; ++d) {
    if (l0 + d < l1) stage_static<kFwd>(a, l0 + d, stages[d]);
    cp_commit();
  }
  cp_wait_all();
  __syncthreads();
  stage_rhs(a, l0, stages[0], xbuf, xin);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  for (int lv = l0; lv < l1; ++lv) {
    const int r = lv - l0;
    // group A: rhs of lv+1 (its stage landed at the end of the last level);
    // group B: static data kAhead levels ahead. A is committed first, so
    // waiting for "all but the newest group" below leaves only B pending.
    if (lv + 1 < l1) stage_rhs(a, lv + 1, stages[(r + 1) % kStages], xbuf + ((r + 1) & 1) * kStageRows, xin);
    cp_commit();
    if (lv + kAhead < l1) stage_static<kFwd>(a, lv + kAhead, stages[(r + kAhead) % kStages]);
    cp_commit();
    const int k0 = a.lvl_ptr[lv];
    const int nr = a.lvl_ptr[lv + 1] - k0;
    if (a.mode[lv] == 0) {
      const Stage& st = stages[r % kStages];
      const double* xb = xbuf + (r & 1) * kStageRows;
      for (int t = threadIdx.x; t < nr; t += blockDim.x) {
        const int qa = st.off[t], qb = st.off[t + 1];
        double acc = xb[t];
#pragma unroll 4
        for (int q = qa; q < qb; ++q) {
          const int s = st.src[q];
          const double yv = s >= 0 ? ring[s] : __ldcg(y + (-s - 1));
          acc = dsub(acc, dmul(st.val[q], yv));
        }
        if (!kFwd) acc = __ddiv_rn(acc, st.dv[t]);
        ring[(k0 + t) & (kRing - 1)] = acc;
        y[st.row[t]] = acc;
      }
    } else {
      // heavy level: operands straight from global memory
      const int64_t q0 = a.lvl_nz[lv];
      for (int t = threadIdx.x; t < nr; t += blockDim.x) {
        const int k = k0 + t;
        const int row = __ldg(a.rows + k);
        const int64_t qa = q0 + __ldg(a.row_off + k);
        const int64_t qb = t + 1 < nr ? q0 + __ldg(a.row_off + k + 1) : a.lvl_nz[lv + 1];
        double acc = kFwd ? __ldg(xin + row) : __ldcg(xin + row);
        for (int64_t q = qa; q < qb; ++q) {
          const int s = __ldg(a.src + q);
          const double yv = s >= 0 ? ring[s] : __ldcg(y + (-s - 1));
          acc = dsub(acc, dmul(__ldg(a.val + q), yv));
        }
        if (!kFwd) acc = __ddiv_rn(acc, __ldg(a.div + k));
        ring[k & (kRing - 1)] = acc;
        y[row] = acc;
      }
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
  }
}

/// Row-parallel level (too wide for one CTA): every source is global.
template <bool kFwd>
__global__ void wide_kernel(WalkArgs a, int lv, const double* xin, double* y) {
  const int k0 = a.lvl_ptr[lv], k1 = a.lvl_ptr[lv + 1];
  const int64_t q0 = a.lvl_nz[lv];
  for (int k = k0 + int(blockIdx.x * blockDim.x + threadIdx.x); k < k1; k += gridDim.x * blockDim.x) {
    const int row = a.rows[k];
    const int64_t qa = q0 + a.row_off[k];
    const int64_t qb = (k + 1 < k1) ? q0 + a.row_off[k + 1] : a.lvl_nz[lv + 1];
    double acc = xin[row];
    for (int64_t q = qa; q < qb; ++q) acc = dsub(acc, dmul(a.val[q], __ldcg(y + (-a.src[q] - 1))));
    if (!kFwd) acc = __ddiv_rn(acc, a.div[k]);
    y[row] = acc;
  }
}

__global__ void gather_vals(int64_t m, const int64_t* __restrict__ from,
                            const double* __restrict__ lu, double* __restrict__ out) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = from[q];
    out[q] = p >= 0 ? lu[p] : 0.0;
  }
}

WalkArgs args_of(const WalkPlan& w) {
  return {w.lvl_ptr.p, w.lvl_nz.p, w.rows.p, w.row_off.p, w.val.p, w.src.p, w.div.p, w.mode.p};
}

size_t walk_smem() {
  return sizeof(double) * (kRing + 2 * kStageRows) + kStages * sizeof(Stage);
}

} // namespace

void build_walk(Context& c, const Csr& a, const std::vector<int64_t>& diag, bool fwd, WalkPlan& w) {
  const int64_t n = a.n;
  const auto& rp = a.h_row_ptr;
  const auto& cols = a.h_cols;
  w.fwd = fwd;
  w.segments.clear();
  if (n == 0) return;
  auto q_begin = [&](int64_t i) { return fwd ? rp[i] : diag[i] + 1; };
  auto q_end = [&](int64_t i) { return fwd ? diag[i] : rp[i + 1]; };
  // DAG levels in processing order
  std::vector<int32_t> lvl(n, 0);
  int nlev = 0;
  for (int64_t p = 0; p < n; ++p) {
    const int64_t i = fwd ? p : n - 1 - p;
    int L = 0;
    for (int64_t q = q_begin(i); q < q_end(i); ++q) L = std::max(L, lvl[cols[q]] + 1);
    lvl[i] = L;
    nlev = std::max(nlev, L + 1);
  }
  std::vector<int32_t> lvl_ptr(nlev + 1, 0);
  for (int64_t i = 0; i < n; ++i) lvl_ptr[lvl[i] + 1]++;
  for (int l = 0; l < nlev; ++l) lvl_ptr[l + 1] += lvl_ptr[l];
  std::vector<int32_t> rows(n), pos(n);
  {
    std::vector<int32_t> fill(lvl_ptr.begin(), lvl_ptr.end() - 1);
    for (int64_t p = 0; p < n; ++p) {
      const int64_t i = fwd ? p : n - 1 - p;
      const int32_t k = fill[lvl[i]]++;
      rows[k] = int32_t(i);
      pos[i] = k;
    }
  }
  // level kinds: narrow levels (walked) vs wide ones (row-parallel)
  std::vector<uint8_t> wide(nlev, 0), mode(nlev, 0);
  std::vector<int64_t> lvl_nzcnt(nlev, 0);
  for (int l = 0; l < nlev; ++l) {
    int64_t nz = 0;
    for (int k = lvl_ptr[l]; k < lvl_ptr[l + 1]; ++k) nz += q_end(rows[k]) - q_begin(rows[k]);
    lvl_nzcnt[l] = nz;
    const int rows_l = lvl_ptr[l + 1] - lvl_ptr[l];
    wide[l] = rows_l > kWalkThreads ? 1 : 0;
    mode[l] = wide[l] ? 2 : ((rows_l <= kStageRows && nz <= kMaxNz - 8) ? 0 : 1);
  }
  // segments and packed arrays
  std::vector<int64_t> lvl_nz(nlev + 1, 0);
  for (int l = 0; l < nlev; ++l) lvl_nz[l + 1] = lvl_nz[l] + ((lvl_nzcnt[l] + 3) / 4) * 4;
  const int64_t total = lvl_nz[nlev] + 8;
  std::vector<int64_t> from(total, -1);
  std::vector<int32_t> src(total, 0), row_off(n, 0);
  std::vector<int32_t> seg_of_level(nlev, -1);
  int seg = -1;
  for (int l = 0; l < nlev; ++l) {
    if (wide[l]) {
      w.segments.push_back({true, l, l + 1});
      ++seg;
    } else if (l == 0 || wide[l - 1]) {
      w.segments.push_back({false, l, l + 1});
      ++seg;
    } else {
      w.segments.back().l1 = l + 1;
    }
    seg_of_level[l] = seg;
  }
  for (int l = 0; l < nlev; ++l) {
    int64_t q = lvl_nz[l];
    const int kend = lvl_ptr[l + 1];
    for (int k = lvl_ptr[l]; k < kend; ++k) {
      const int64_t i = rows[k];
      row_off[k] = int32_t(q - lvl_nz[l]);
      for (int64_t p = q_begin(i); p < q_end(i); ++p, ++q) {
        const int32_t j = cols[p];
        from[q] = p;
        const int lj = lvl[j];
        // ring slot only inside the same walked segment and close enough
        // that no row of this level can overwrite it (kRing positions)
        const bool in_ring = !wide[l] && seg_of_level[lj] == seg_of_level[l] &&
                             int64_t(kend) - int64_t(pos[j]) <= kRing;
        src[q] = in_ring ? (pos[j] & (kRing - 1)) : -(j + 1);
      }
    }
  }
  if (getenv("PSCU_DEBUG")) {
    int64_t ring_hits = 0, far = 0, maxr = 0, maxq = 0;
    for (int64_t q = 0; q < lvl_nz[nlev]; ++q)
      if (from[q] >= 0) (src[q] >= 0 ? ring_hits : far)++;
    for (int l = 0; l < nlev; ++l) {
      maxr = std::max<int64_t>(maxr, lvl_ptr[l + 1] - lvl_ptr[l]);
      maxq = std::max<int64_t>(maxq, lvl_nzcnt[l]);
    }
    int nwide = 0, nstaged = 0;
    for (const auto& sg : w.segments) nwide += sg.wide;
    for (int l = 0; l < nlev; ++l) nstaged += mode[l] == 0;
    fprintf(stderr,
            "[walk %s] n=%lld levels=%d (staged %d) segments=%zu (wide %d) max_rows=%lld "
            "max_nz=%lld ring=%lld far=%lld\n",
            fwd ? "fwd" : "bwd", (long long)n, nlev, nstaged, w.segments.size(), nwide, (long long)maxr,
            (long long)maxq, (long long)ring_hits, (long long)far);
  }
  std::vector<int64_t> dfrom(n);
  for (int k = 0; k < n; ++k) dfrom[k] = diag[rows[k]];
  cudaStream_t st = c.stream;
  w.nlev = nlev;
  w.mode.upload(mode, st);
  w.lvl_ptr.upload(lvl_ptr, st);
  w.lvl_nz.upload(lvl_nz, st);
  w.rows.upload(rows, st);
  w.row_off.upload(row_off, st);
  w.src.upload(src, st);
  w.from.upload(from, st);
  w.val.alloc(total);
  if (!fwd) {
    w.div_from.upload(dfrom, st);
    w.div.alloc(n);
  } else {
    w.div.alloc(1);
  }
}

void pack_walk(Context& c, const double* lu, WalkPlan& w) {
  if (w.val.n == 0) return;
  const int64_t m = int64_t(w.val.n);
  gather_vals<<<unsigned(std::min<int64_t>((m + 255) / 256, 148 * 32)), 256, 0, c.stream>>>(
      m, w.from.p, lu, w.val.p);
  PSCU_LAUNCHED(&c);
  if (!w.fwd) {
    const int64_t nd = int64_t(w.div.n);
    gather_vals<<<unsigned(std::min<int64_t>((nd + 255) / 256, 148 * 32)), 256, 0, c.stream>>>(
        nd, w.div_from.p, lu, w.div.p);
    PSCU_LAUNCHED(&c);
  }
}

void run_walk(Context& c, const WalkPlan& w, const double* xin, double* y) {
  static bool attr = false;
  if (!attr) {
    PSCU_CUDA(cudaFuncSetAttribute(walk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(walk_smem())));
    PSCU_CUDA(cudaFuncSetAttribute(walk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(walk_smem())));
    attr = true;
  }
  const WalkArgs a = args_of(w);
  for (const WalkSeg& s : w.segments) {
    if (s.wide) {
      if (w.fwd) wide_kernel<true><<<148 * 8, 256, 0, c.stream>>>(a, s.l0, xin, y);
      else wide_kernel<false><<<148 * 8, 256, 0, c.stream>>>(a, s.l0, xin, y);
    } else {
      if (w.fwd) walk_kernel<true><<<1, kWalkThreads, walk_smem(), c.stream>>>(a, s.l0, s.l1, xin, y);
      else walk_kernel<false><<<1, kWalkThreads, walk_smem(), c.stream>>>(a, s.l0, s.l1, xin, y);
    }
    PSCU_LAUNCHED(&c);
  }
}

} // namespace pscu
