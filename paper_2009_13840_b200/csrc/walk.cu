// Level-walking sparse triangular sweeps for Ilu0::apply (ilu0.hpp:53-65).
//
// The reference applies ILU(0) with two sequential loops. Under the natural
// (faces-first) ordering their dependency DAGs are deep and narrow: hundreds
// to thousands of levels of a few hundred rows, so any
// scheme that pays an inter-SM handshake per level is bound by ~1 us per
// level. Narrow levels are therefore walked by ONE CTA:
//   * rows are placed in level order ("positions"); each level is cut into
//     sub-levels of at most kStageRows rows / kMaxNz factor entries (rows of
//     one level are independent, so any cut is a valid schedule);
//   * a sub-level's operands are one contiguous, 16-byte-aligned block:
//     the factor entries it needs in the reference's summation order
//     (value + source), its row ids, offsets, right-hand sides (gathered into
//     position order beforehand) and, backward, its diagonals;
//   * blocks are staged into shared memory kAhead sub-levels ahead with
//     cp.async (all addresses are static, so the pipeline never waits on a
//     dependent gather);
//   * recently computed solution values live in a shared-memory ring indexed
//     by position; older sources, or sources from other segments, come from
//     global memory (L2);
//   * one __syncthreads per sub-level, no global handshake at all.
// Levels with very many rows (the element-pressure rows) run as ordinary
// row-parallel launches between walker segments. Every row is computed by
// one thread with the reference's exact operation sequence, so the result is
// bit-identical to Ilu0::apply.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"
#include "walk.cuh"

namespace pscu {

namespace {

constexpr int kWalkThreads = 512;
constexpr int kProducers = 256;    // two producer warps per stage slot (TMA issue + far gathers)
constexpr int kStageRows = 512;   // rows of a sub-level
constexpr int kMaxNz = 2560;      // factor entries of a sub-level (multiple of 4)
constexpr int kAhead = 3;         // sub-levels staged ahead
constexpr int kStages = kAhead + 1;
constexpr int kRing = 4096;       // shared-memory solution ring (positions, power of 2)
constexpr int kMaxFar = 512;      // sources outside the ring, per sub-level
constexpr int kWideRows = 4096;   // levels with more rows run row-parallel

struct WalkArgs {
  const int32_t* sl_k;    // sub-level start position (multiple of 4)
  const int32_t* sl_nr;   // rows of the sub-level
  const int64_t* sl_q;    // packed entry start (multiple of 4), nsub + 1
  const int32_t* sl_hdr;  // per sub-level {k0, rows, real entries, any global source}
  const int32_t* rows;    // row id per position (-1 padding)
  const int32_t* off;     // packed offset of a row within its sub-level
  const int32_t* opos;    // forward: backward position of the row
  const double* val;      // packed factor values
  const int32_t* src;     // >= 0 ring slot, < 0: -(row)-1 global source
  const double* dv;       // backward: diagonal per position
  const int64_t* sl_f;    // far-source list start per sub-level (nsub + 1)
  const int32_t* far;     // far source rows, per sub-level
};

struct alignas(16) Stage {
  double val[kMaxNz];
  int32_t src[kMaxNz];
  double rhs[kStageRows];
  double dv[kStageRows];
  int32_t row[kStageRows];
  int32_t opos[kStageRows];
  int32_t off[kStageRows + 4];
  int32_t hdr[4];  // k0, rows, real entries (end of the last row), far sources
  double farv[kMaxFar];  // values of the sources outside the ring (gathered)
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return unsigned(__cvta_generic_to_shared(p));
}

/// One TMA bulk copy global -> shared completing on mbarrier `bar`.
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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

/// Producer lane: stages sub-level s into `st` with one bulk copy per
/// operand array (all addresses static and 16-byte aligned).
template <bool kFwd>
__device__ void issue(const WalkArgs& a, int s, Stage& st, uint64_t* bar, const double* rhs) {
  const int k0 = a.sl_k[s], nr = a.sl_nr[s];
  const unsigned nr4 = unsigned((nr + 3) & ~3);
  const int64_t q0 = a.sl_q[s];
  const unsigned nq = unsigned(a.sl_q[s + 1] - q0);
  const unsigned bytes = nq * 12u + nr4 * (8u + 4u + 4u) + (kFwd ? nr4 * 4u : nr4 * 8u) + 16u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  bulk_copy(st.hdr, a.sl_hdr + 4 * s, 16u, bar);
  bulk_copy(st.val, a.val + q0, nq * 8u, bar);
  bulk_copy(st.src, a.src + q0, nq * 4u, bar);
  bulk_copy(st.rhs, rhs + k0, nr4 * 8u, bar);
  bulk_copy(st.row, a.rows + k0, nr4 * 4u, bar);
  bulk_copy(st.off, a.off + k0, nr4 * 4u, bar);
  if (kFwd) bulk_copy(st.opos, a.opos + k0, nr4 * 4u, bar);
  else bulk_copy(st.dv, a.dv + k0, nr4 * 8u, bar);
}

template <bool kFwd, bool kAnyFar>
__device__ __forceinline__ void walk_rows(const Stage& st, double* ring, double* y, double* yb) {
  const int k0 = st.hdr[0], nr = st.hdr[1];
  for (int t = threadIdx.x; t < nr; t += kWalkThreads) {
    const int qa = st.off[t], qb = t + 1 < nr ? st.off[t + 1] : st.hdr[2];
    double acc = st.rhs[t];
#pragma unroll 4
    for (int q = qa; q < qb; ++q) {
      const int sv = st.src[q];
      double yv;
      if (kAnyFar) yv = sv >= 0 ? ring[sv] : st.farv[-sv - 1];
      else yv = ring[sv];
      acc = dsub(acc, dmul(st.val[q], yv));
    }
    if (!kFwd) acc = __ddiv_rn(acc, st.dv[t]);
    ring[(k0 + t) & (kRing - 1)] = acc;
    y[st.row[t]] = acc;
    if (kFwd) yb[st.opos[t]] = acc;
  }
}

/// Warp-specialised walker: kWalkThreads consumer threads compute one
/// sub-level after another (one named barrier per sub-level); one extra
/// producer warp keeps kStages sub-levels in flight with TMA bulk copies,
/// reusing a slot once the consumers have released it.
template <bool kFwd>
__global__ void __launch_bounds__(kWalkThreads + kProducers, 1)
    walk_kernel(WalkArgs a, int s0, int s1, const double* rhs, double* y, double* yb,
                int experiment) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  double* ring = reinterpret_cast<double*>(smraw);
  Stage* stages = reinterpret_cast<Stage*>(smraw + sizeof(double) * kRing);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_addr(&full[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&empty[i])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= kWalkThreads) {
    // producer warps: thread 0 of them issues the bulk copies; all of them
    // gather the sources outside the ring (final: they lie >= kRing
    // positions, hence >= kStages sub-levels, back, or in an earlier launch)
    // with several independent loads in flight per lane, then one of them
    // makes the second arrival on the slot's full barrier
    // producer warp pair w owns slot w: sub-levels s0 + w, s0 + w + kStages, ...
    const int pw = (threadIdx.x - kWalkThreads) >> 6, lane = (threadIdx.x - kWalkThreads) & 63;
    const int slot = pw;
    for (int s = s0 + pw; s < s1; s += kStages) {
      const int r = s - s0;
      if (r >= kStages) mbar_wait(&empty[slot], unsigned((r / kStages - 1) & 1));
      if (lane == 0) issue<kFwd>(a, s, stages[slot], &full[slot], rhs);
      const int64_t f0 = a.sl_f[s], nf = a.sl_f[s + 1] - f0;
      double* fv = stages[slot].farv;
      for (int64_t base = 0; base < nf; base += 8 * 64) {
        int32_t idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t f = base + u * 64 + lane;
          idx[u] = f < nf ? __ldg(a.far + f0 + f) : -1;
        }
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = idx[u] >= 0 ? __ldcg(y + idx[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t f = base + u * 64 + lane;
          if (f < nf) fv[f] = v[u];
        }
      }
      asm volatile("bar.sync %0, 64;" ::"r"(2 + pw) : "memory");
      if (lane == 0) mbar_arrive(&full[slot]);
    }
    return;
  }
  for (int s = s0; s < s1; ++s) {
    const int r = s - s0, slot = r % kStages;
    const Stage& st = stages[slot];
    mbar_wait(&full[slot], unsigned((r / kStages) & 1));
    if (experiment != 1) {
      if (st.hdr[3]) walk_rows<kFwd, true>(st, ring, y, yb);
      else walk_rows<kFwd, false>(st, ring, y, yb);
    }
    // consumers only: the slot is free and the ring entries of s visible
    asm volatile("bar.sync 1, %0;" ::"n"(kWalkThreads) : "memory");
    if (threadIdx.x == 0) mbar_arrive(&empty[slot]);
  }
}

/// Row-parallel sub-level (a level too wide for one CTA): global sources.
template <bool kFwd>
__global__ void wide_kernel(WalkArgs a, int s, const double* rhs, double* y, double* yb) {
  const int k0 = a.sl_k[s], nr = a.sl_nr[s];
  const int64_t q0 = a.sl_q[s];
  const int nq = a.sl_hdr[4 * s + 2];
  for (int t = int(blockIdx.x * blockDim.x + threadIdx.x); t < nr; t += gridDim.x * blockDim.x) {
    const int k = k0 + t;
    const int64_t qa = q0 + a.off[k];
    const int64_t qb = q0 + (t + 1 < nr ? a.off[k + 1] : nq);
    double acc = rhs[k];
    for (int64_t q = qa; q < qb; ++q) acc = dsub(acc, dmul(a.val[q], __ldcg(y + (-a.src[q] - 1))));
    if (!kFwd) acc = __ddiv_rn(acc, a.dv[k]);
    y[a.rows[k]] = acc;
    if (kFwd) yb[a.opos[k]] = acc;
  }
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

__global__ void gather_vals(int64_t m, const int64_t* __restrict__ from,
                            const double* __restrict__ lu, double* __restrict__ out) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = from[q];
    out[q] = p >= 0 ? lu[p] : 0.0;
  }
}

WalkArgs args_of(const WalkPlan& w) {
  return {w.sl_k.p, w.sl_nr.p, w.sl_q.p, w.sl_hdr.p, w.rows.p, w.off.p,
          w.opos.p, w.val.p,  w.src.p,  w.dv.p,  w.sl_f.p, w.far.p};
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

struct HostPlan {
  std::vector<int32_t> sl_k, sl_nr, sl_nq, sl_nfar, rows, off, src, pos, far;
  std::vector<int64_t> sl_f;
  std::vector<int64_t> sl_q, from, dfrom;
  std::vector<uint8_t> sl_wide;
  int64_t npos = 0;
};

/// Positions, sub-levels and packed operands of one sweep.
HostPlan plan_sweep(const Csr& a, const std::vector<int64_t>& diag, bool fwd) {
  const int64_t n = a.n;
  const auto& rp = a.h_row_ptr;
  const auto& cols = a.h_cols;
  auto q_begin = [&](int64_t i) { return fwd ? rp[i] : diag[i] + 1; };
  auto q_end = [&](int64_t i) { return fwd ? diag[i] : rp[i + 1]; };
  int nlev = 0;
  const std::vector<int32_t> lvl = dag_levels(a, diag, fwd, nlev);
  std::vector<int32_t> lvl_ptr(nlev + 1, 0), order(n);
  for (int64_t i = 0; i < n; ++i) lvl_ptr[lvl[i] + 1]++;
  for (int l = 0; l < nlev; ++l) lvl_ptr[l + 1] += lvl_ptr[l];
  {
    std::vector<int32_t> fill(lvl_ptr.begin(), lvl_ptr.end() - 1);
    for (int64_t p = 0; p < n; ++p) {
      const int64_t i = fwd ? p : n - 1 - p;
      order[fill[lvl[i]]++] = int32_t(i);
    }
  }
  HostPlan h;
  h.pos.assign(n, -1);
  int64_t k = 0, q = 0;
  int64_t seg_start = 0;      // first position of the current walker segment
  std::vector<int32_t> far_mark(n, -1);
  int cur_far = 0;
  auto open_sub = [&](bool wide) {
    k = (k + 3) & ~int64_t(3);
    q = (q + 3) & ~int64_t(3);
    h.sl_k.push_back(int32_t(k));
    h.sl_nr.push_back(0);
    h.sl_q.push_back(q);
    h.sl_nq.push_back(0);
    h.sl_wide.push_back(wide ? 1 : 0);
    cur_far = 0;
  };
  // a source is served by the ring when it lies in the same walker segment
  // within kRing positions of the sub-level's largest possible end
  auto ring_ok = [&](int64_t k0, int32_t j) {
    return h.pos[j] >= seg_start && k0 + kStageRows + 3 - int64_t(h.pos[j]) <= kRing;
  };
  bool prev_wide = true;
  for (int l = 0; l < nlev; ++l) {
    const int nrl = lvl_ptr[l + 1] - lvl_ptr[l];
    const bool wide = nrl > kWideRows;
    open_sub(wide);
    if (!wide && prev_wide) seg_start = h.sl_k.back();
    prev_wide = wide;
    for (int j = lvl_ptr[l]; j < lvl_ptr[l + 1]; ++j) {
      const int32_t i = order[j];
      const int64_t nz = q_end(i) - q_begin(i);
      int nfar = 0;
      if (!wide) {
        const int sid = int(h.sl_k.size()) - 1;
        for (int64_t p = q_begin(i); p < q_end(i); ++p)
          if (!ring_ok(h.sl_k.back(), cols[p]) && far_mark[cols[p]] != sid) ++nfar;
        if (h.sl_nr.back() == kStageRows || h.sl_nq.back() + nz > kMaxNz - 4 ||
            cur_far + nfar > kMaxFar) {
          open_sub(false);
          const int sid2 = int(h.sl_k.size()) - 1;
          nfar = 0;
          for (int64_t p = q_begin(i); p < q_end(i); ++p)
            if (!ring_ok(h.sl_k.back(), cols[p]) && far_mark[cols[p]] != sid2) ++nfar;
        }
        const int sid3 = int(h.sl_k.size()) - 1;
        for (int64_t p = q_begin(i); p < q_end(i); ++p)
          if (!ring_ok(h.sl_k.back(), cols[p])) far_mark[cols[p]] = sid3;
        cur_far += nfar;
      }
      h.pos[i] = int32_t(k++);
      h.sl_nr.back()++;
      h.sl_nq.back() += int32_t(nz);
      q += nz;
    }
  }
  h.sl_q.push_back((q + 3) & ~int64_t(3));
  h.npos = (k + 3) & ~int64_t(3);
  const int nsub = int(h.sl_k.size());
  // walker segments (for the ring-source rule)
  std::vector<int32_t> seg_of(nsub);
  int seg = -1;
  for (int s = 0; s < nsub; ++s) {
    if (h.sl_wide[s] || s == 0 || h.sl_wide[s - 1]) ++seg;
    seg_of[s] = seg;
  }
  std::vector<int32_t> sub_of_pos(h.npos + 4, -1);
  for (int s = 0; s < nsub; ++s)
    for (int t = 0; t < h.sl_nr[s]; ++t) sub_of_pos[h.sl_k[s] + t] = s;
  h.rows.assign(h.npos + 4, -1);
  h.off.assign(h.npos + 4, 0);
  h.dfrom.assign(h.npos + 4, -1);
  const int64_t total = h.sl_q.back() + 8;
  h.from.assign(total, -1);
  h.src.assign(total, 0);
  // rows by position, then the packed operands of each sub-level in row order
  for (int64_t i = 0; i < n; ++i) h.rows[h.pos[i]] = int32_t(i);
  std::vector<int32_t> far_idx(n, -1), far_sub(n, -1);
  h.sl_f.assign(nsub + 1, 0);
  for (int s = 0; s < nsub; ++s) {
    int64_t qq = h.sl_q[s];
    const int64_t kcons = h.sl_k[s] + kStageRows + 3;
    int nf = 0;
    for (int t = 0; t < h.sl_nr[s]; ++t) {
      const int64_t kp = h.sl_k[s] + t;
      const int32_t i = h.rows[kp];
      h.off[kp] = int32_t(qq - h.sl_q[s]);
      h.dfrom[kp] = diag[i];
      for (int64_t p = q_begin(i); p < q_end(i); ++p, ++qq) {
        const int32_t j = cols[p];
        h.from[qq] = p;
        if (h.sl_wide[s]) {
          h.src[qq] = -(j + 1);  // wide launches read global memory directly
          continue;
        }
        const int sj = sub_of_pos[h.pos[j]];
        const bool in_ring = seg_of[sj] == seg_of[s] && kcons - int64_t(h.pos[j]) <= kRing;
        if (in_ring) {
          h.src[qq] = h.pos[j] & (kRing - 1);
        } else {
          if (far_sub[j] != s) {
            far_sub[j] = s;
            far_idx[j] = nf++;
            h.far.push_back(j);
          }
          h.src[qq] = -(far_idx[j] + 1);
        }
      }
    }
    h.sl_f[s + 1] = h.sl_f[s] + nf;
    h.sl_nfar.push_back(nf);
  }
  return h;
}

void upload_plan(Context& c, const HostPlan& h, bool fwd, WalkPlan& w) {
  cudaStream_t st = c.stream;
  w.fwd = fwd;
  w.nsub = int(h.sl_k.size());
  w.npos = h.npos;
  w.segments.clear();
  for (int s = 0; s < w.nsub; ++s) {
    if (h.sl_wide[s]) w.segments.push_back({true, s, s + 1});
    else if (s == 0 || h.sl_wide[s - 1]) w.segments.push_back({false, s, s + 1});
    else w.segments.back().s1 = s + 1;
  }
  w.sl_k.upload(h.sl_k, st);
  w.sl_nr.upload(h.sl_nr, st);
  w.sl_f.upload(h.sl_f, st);
  if (h.far.empty()) w.far.alloc(4);
  else w.far.upload(h.far, st);
  w.sl_q.upload(h.sl_q, st);
  {
    // {k0, rows, real entries, any global source}: one 16-byte bulk copy each
    std::vector<int32_t> hdr(size_t(w.nsub) * 4, 0);
    for (int s = 0; s < w.nsub; ++s) {
      hdr[size_t(s) * 4] = h.sl_k[s];
      hdr[size_t(s) * 4 + 1] = h.sl_nr[s];
      hdr[size_t(s) * 4 + 2] = h.sl_nq[s];
      hdr[size_t(s) * 4 + 3] = h.sl_wide[s] ? 0 : h.sl_nfar[s];
    }
    w.sl_hdr.upload(hdr, st);
  }
  w.rows.upload(h.rows, st);
  w.off.upload(h.off, st);
  w.src.upload(h.src, st);
  w.from.upload(h.from, st);
  w.val.alloc(h.from.size());
  if (!fwd) {
    w.dfrom.upload(h.dfrom, st);
    w.dv.alloc(h.dfrom.size());
  } else {
    w.dv.alloc(4);
  }
}

} // namespace

void build_walk(Context& c, const Csr& a, const std::vector<int64_t>& diag, WalkPlan& wf,
                WalkPlan& wb) {
  if (a.n == 0) return;
  const HostPlan hf = plan_sweep(a, diag, true);
  const HostPlan hb = plan_sweep(a, diag, false);
  upload_plan(c, hf, true, wf);
  upload_plan(c, hb, false, wb);
  // forward results are written straight into backward position order
  std::vector<int32_t> opos(hf.rows.size(), 0);
  for (size_t k = 0; k < hf.rows.size(); ++k)
    if (hf.rows[k] >= 0) opos[k] = hb.pos[hf.rows[k]];
  wf.opos.upload(opos, c.stream);
  wb.opos.alloc(4);
  wf.scratch.alloc(size_t(hf.npos) + 8);  // rhs in forward position order
  wb.scratch.alloc(size_t(hb.npos) + 8);  // forward result in backward position order
  PSCU_CUDA(cudaMemsetAsync(wb.scratch.p, 0, sizeof(double) * (hb.npos + 8), c.stream));
  if (getenv("PSCU_DEBUG")) {
    for (const HostPlan* h : {&hf, &hb}) {
      int64_t ring = 0, far = 0;
      for (size_t q = 0; q < h->from.size(); ++q)
        if (h->from[q] >= 0) (h->src[q] >= 0 ? ring : far)++;
      int nw = 0;
      for (auto x : h->sl_wide) nw += x;
      fprintf(stderr, "[walk %s] n=%lld sublevels=%zu (wide %d) positions=%lld ring=%lld far=%lld\n",
              h == &hf ? "fwd" : "bwd", (long long)a.n, h->sl_k.size(), nw, (long long)h->npos,
              (long long)ring, (long long)far);
    }
  }
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

static void run_one(Context& c, const WalkPlan& w, const double* rhs, double* y, double* yb) {
  static bool attr = false;
  if (!attr) {
    PSCU_CUDA(cudaFuncSetAttribute(walk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(walk_smem())));
    PSCU_CUDA(cudaFuncSetAttribute(walk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(walk_smem())));
    attr = true;
  }
  const WalkArgs a = args_of(w);
  static const int experiment = getenv("PSCU_WALK_EXPERIMENT") ? atoi(getenv("PSCU_WALK_EXPERIMENT")) : 0;
  for (const WalkSeg& s : w.segments) {
    if (s.wide) {
      if (w.fwd) wide_kernel<true><<<148 * 4, 256, 0, c.stream>>>(a, s.s0, rhs, y, yb);
      else wide_kernel<false><<<148 * 4, 256, 0, c.stream>>>(a, s.s0, rhs, y, yb);
    } else {
      if (w.fwd)
        walk_kernel<true><<<1, kWalkThreads + kProducers, walk_smem(), c.stream>>>(a, s.s0, s.s1, rhs, y, yb, experiment);
      else
        walk_kernel<false><<<1, kWalkThreads + kProducers, walk_smem(), c.stream>>>(a, s.s0, s.s1, rhs, y, yb, experiment);
    }
    PSCU_LAUNCHED(&c);
  }
}

void run_walk(Context& c, const WalkPlan& wf, const WalkPlan& wb, const double* x, double* y) {
  // rhs into forward position order, forward sweep (also scattering its
  // result into backward position order), backward sweep in place on y
  gather_rhs<<<grid1(wf.npos), 256, 0, c.stream>>>(wf.npos, wf.rows.p, x, wf.scratch.p);
  PSCU_LAUNCHED(&c);
  run_one(c, wf, wf.scratch.p, y, wb.scratch.p);
  run_one(c, wb, wb.scratch.p, y, nullptr);
}

} // namespace pscu
