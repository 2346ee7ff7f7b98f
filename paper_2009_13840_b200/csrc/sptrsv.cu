// ILU(0) factorisation and application (Ilu0, ilu0.hpp:19-65) as
// synchronisation-free, chunked, level-scheduled sparse triangular sweeps.
//
// Bit-exactness: every row is computed by one thread with exactly the
// reference's operation sequence (s = x_i; s -= lu[p]*y[c] for p ascending;
// backward: then s / lu[diag]) using non-fused IEEE operations, so only the
// inter-row schedule differs from the sequential reference loop.
//
// Schedule (built once per pattern on the host): rows are cut, in
// processing order (ascending for the forward sweep, descending for the
// backward sweep), into chunks of kChunkRows contiguous rows. One CTA owns a
// chunk: it keeps the chunk's solution values in shared memory and walks the
// chunk's intra-chunk dependency levels, one __syncthreads per level. A
// dependency on another chunk is a wait on that chunk's published progress
// counter (tagged with the launch epoch so counters never need resetting).
// CTAs take chunks in processing order from an atomic ticket, so a CTA only
// ever waits on chunks already owned by running or finished CTAs: no
// deadlock without co-residency, and no grid-wide barrier at all.
#include <algorithm>

#include "internal.cuh"
#include "walk.cuh"

namespace pscu {

namespace {

constexpr int kChunkRows = 12288;  // up to 96 KB of shared-memory solution values
constexpr int64_t kRecent = 64;    // dependency distance that continues a chain
constexpr int kSweepThreads = 128;

struct SweepArgs {
  int nchunks;
  const int64_t* chunk_begin;
  const int64_t* chunk_end;
  const int32_t* chunk_lvl;
  const int32_t* level_ptr;
  const int32_t* sched;
  const int32_t* wait_ptr;
  const int32_t* wait_chunk;
  const int32_t* wait_need;
  const uint8_t* exported;
  unsigned long long* progress;
  unsigned long long* ticket;
};

SweepArgs args_of(const Sweep& s) {
  return {s.nchunks,      s.chunk_begin.p, s.chunk_end.p,  s.chunk_lvl.p,
          s.level_ptr.p,  s.sched.p,       s.wait_ptr.p,   s.wait_chunk.p,
          s.wait_need.p,  s.exported.p,    s.progress.p,   s.ticket.p};
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

/// Common prologue: take a ticket, derive chunk and epoch tag.
__device__ __forceinline__ void take_ticket(const SweepArgs& s, int& c, unsigned long long& tag) {
  __shared__ unsigned long long s_t;
  if (threadIdx.x == 0) s_t = atomicAdd(s.ticket, 1ull);
  __syncthreads();
  const unsigned long long t = s_t;
  c = int(t % unsigned(s.nchunks));
  tag = ((t / unsigned(s.nchunks)) + 1ull) << 32;
}

__device__ __forceinline__ void wait_level(const SweepArgs& s, int lv, unsigned long long tag) {
  const int w0 = s.wait_ptr[lv], w1 = s.wait_ptr[lv + 1];
  if (w1 == w0) return;  // uniform across the CTA
  for (int w = w0 + threadIdx.x; w < w1; w += blockDim.x) {
    const unsigned long long need = tag | unsigned(s.wait_need[w]);
    const unsigned long long* f = s.progress + s.wait_chunk[w];
    while (ld_acquire(f) < need) __nanosleep(32);
  }
  __syncthreads();
}

template <bool kForward>
__global__ void __launch_bounds__(kSweepThreads)
    sweep_kernel(SweepArgs s, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                 const double* __restrict__ lu, const int64_t* __restrict__ diag,
                 const double* x, double* y) {
  extern __shared__ double ys[];
  int c;
  unsigned long long tag;
  take_ticket(s, c, tag);
  const int64_t cb = s.chunk_begin[c], ce = s.chunk_end[c];
  const int l0 = s.chunk_lvl[c], l1 = s.chunk_lvl[c + 1];
  for (int lv = l0; lv < l1; ++lv) {
    wait_level(s, lv, tag);
    const bool ex = s.exported[lv] != 0;
    for (int k = s.level_ptr[lv] + threadIdx.x; k < s.level_ptr[lv + 1]; k += blockDim.x) {
      const int i = s.sched[k];
      double acc;
      if (kForward) {
        acc = x[i];
        const int64_t pe = diag[i];
        for (int64_t p = rp[i]; p < pe; ++p) {
          const int j = cols[p];
          const double yj = j >= cb ? ys[j - cb] : __ldcg(y + j);
          acc = dsub(acc, dmul(lu[p], yj));
        }
      } else {
        acc = y[i];
        const int64_t pd = diag[i], pe = rp[i + 1];
        for (int64_t p = pd + 1; p < pe; ++p) {
          const int j = cols[p];
          const double yj = j < ce ? ys[j - cb] : __ldcg(y + j);
          acc = dsub(acc, dmul(lu[p], yj));
        }
        acc = __ddiv_rn(acc, lu[pd]);
      }
      ys[i - cb] = acc;
      y[i] = acc;
      if (ex) __threadfence();
    }
    __syncthreads();
    if (ex && threadIdx.x == 0) st_release(s.progress + c, tag | unsigned(lv - l0 + 1));
  }
}

/// ILU(0) factorisation (ilu0.hpp:29-50) over the forward schedule: row i is
/// factored by one thread once every row it references below the diagonal
/// is final; updates reach each entry in k-ascending order, as in the
/// reference's IKJ loop.
__global__ void __launch_bounds__(kSweepThreads)
    ilu0_factor_kernel(SweepArgs s, const int64_t* __restrict__ rp,
                       const int32_t* __restrict__ cols, double* lu,
                       const int64_t* __restrict__ diag, int* err) {
  int c;
  unsigned long long tag;
  take_ticket(s, c, tag);
  const int l0 = s.chunk_lvl[c], l1 = s.chunk_lvl[c + 1];
  for (int lv = l0; lv < l1; ++lv) {
    wait_level(s, lv, tag);
    const bool ex = s.exported[lv] != 0;
    for (int kk = s.level_ptr[lv] + threadIdx.x; kk < s.level_ptr[lv + 1]; kk += blockDim.x) {
      const int i = s.sched[kk];
      const int64_t ri0 = rp[i], ri1 = rp[i + 1], di = diag[i];
      for (int64_t p = ri0; p < di; ++p) {
        const int k = cols[p];
        const double piv = __ldcg(lu + diag[k]);
        if (piv == 0.0) atomicMin(err, k);
        const double lik = __ddiv_rn(lu[p], piv);
        lu[p] = lik;
        int64_t r = p + 1;
        const int64_t qe = rp[k + 1];
        for (int64_t q = diag[k] + 1; q < qe; ++q) {
          const int cq = cols[q];
          while (r < ri1 && cols[r] < cq) ++r;
          if (r < ri1 && cols[r] == cq) lu[r] = dsub(lu[r], dmul(lik, __ldcg(lu + q)));
        }
      }
      if (lu[di] == 0.0) atomicMin(err, i);
      if (ex) __threadfence();
    }
    __syncthreads();
    if (ex && threadIdx.x == 0) st_release(s.progress + c, tag | unsigned(lv - l0 + 1));
  }
}

} // namespace

void build_sweep(Context& c, const Csr& a, const std::vector<int64_t>& diag, bool fwd, Sweep& s) {
  const int64_t n = a.n;
  const auto& rp = a.h_row_ptr;
  const auto& cols = a.h_cols;
  const int64_t CH = kChunkRows;
  if (n == 0) {
    s.nchunks = 0;
    return;
  }
  auto pos_of = [&](int64_t i) { return fwd ? i : n - 1 - i; };
  auto row_at = [&](int64_t p) { return fwd ? p : n - 1 - p; };

  // Chunk boundaries. A row whose nearest dependency (in processing order)
  // lies more than kRecent rows back starts a new dependency chain; chunks
  // are cut at chain starts so that consecutive chunks depend on each other
  // "side by side" (a pipelined wavefront) instead of end-to-start.
  std::vector<int64_t> starts{0};
  {
    int64_t last_cs = -1;
    for (int64_t p = 0; p < n; ++p) {
      const int64_t i = row_at(p);
      const int64_t q0 = fwd ? rp[i] : diag[i] + 1;
      const int64_t q1 = fwd ? diag[i] : rp[i + 1];
      int64_t nearest = INT64_MAX;
      for (int64_t q = q0; q < q1; ++q) nearest = std::min(nearest, p - pos_of(cols[q]));
      if (nearest > kRecent) last_cs = p;
      if (p - starts.back() >= CH) {
        const int64_t cut = last_cs > starts.back() ? last_cs : p;
        starts.push_back(cut);
      }
    }
  }
  const int nchunks = int(starts.size());
  s.nchunks = nchunks;
  std::vector<int32_t> chunk_of(n);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int64_t p1 = ch + 1 < nchunks ? starts[ch + 1] : n;
    for (int64_t p = starts[ch]; p < p1; ++p) chunk_of[p] = ch;
  }

  std::vector<int32_t> lvl(n, 0);
  std::vector<int32_t> chunk_nlv(nchunks, 0);
  for (int64_t p = 0; p < n; ++p) {
    const int64_t i = row_at(p);
    const int64_t cb = starts[chunk_of[p]];
    int L = 0;
    const int64_t q0 = fwd ? rp[i] : diag[i] + 1;
    const int64_t q1 = fwd ? diag[i] : rp[i + 1];
    for (int64_t q = q0; q < q1; ++q) {
      const int64_t pj = pos_of(cols[q]);
      if (pj >= cb) L = std::max(L, lvl[cols[q]] + 1);
    }
    lvl[i] = L;
    chunk_nlv[chunk_of[p]] = std::max(chunk_nlv[chunk_of[p]], L + 1);
  }
  std::vector<int32_t> chunk_lvl(nchunks + 1, 0);
  for (int ch = 0; ch < nchunks; ++ch) chunk_lvl[ch + 1] = chunk_lvl[ch] + chunk_nlv[ch];
  const int nlevels = chunk_lvl[nchunks];
  s.nlevels = nlevels;

  std::vector<int32_t> level_cnt(nlevels + 1, 0);
  for (int64_t p = 0; p < n; ++p) level_cnt[chunk_lvl[chunk_of[p]] + lvl[row_at(p)] + 1]++;
  std::vector<int32_t> level_ptr(nlevels + 1, 0);
  for (int l = 0; l < nlevels; ++l) level_ptr[l + 1] = level_ptr[l] + level_cnt[l + 1];
  std::vector<int32_t> sched(n);
  {
    std::vector<int32_t> fill(level_ptr.begin(), level_ptr.end() - 1);
    for (int64_t p = 0; p < n; ++p) {
      const int64_t i = row_at(p);
      sched[fill[chunk_lvl[chunk_of[p]] + lvl[i]]++] = int32_t(i);
    }
  }
  int max_level_rows = 0;
  for (int l = 0; l < nlevels; ++l) max_level_rows = std::max(max_level_rows, level_ptr[l + 1] - level_ptr[l]);
  s.max_level_rows = max_level_rows;

  // foreign waits: (local level, foreign chunk, need) per chunk, pruned by a
  // running maximum per foreign chunk
  std::vector<int32_t> wait_ptr(nlevels + 1, 0);
  std::vector<int32_t> wait_chunk, wait_need;
  std::vector<uint8_t> exported(nlevels, 0);
  struct W {
    int32_t lev, chunk, need;
  };
  std::vector<W> recs;
  std::vector<std::pair<int32_t, int32_t>> waited; // (chunk, max need)
  std::vector<std::vector<std::pair<int32_t, int32_t>>> per_level_waits(0);
  std::vector<int32_t> wcount(nlevels, 0);
  std::vector<W> emitted;
  for (int ch = 0; ch < nchunks; ++ch) {
    recs.clear();
    const int64_t p0 = starts[ch], p1 = ch + 1 < nchunks ? starts[ch + 1] : n;
    for (int64_t p = p0; p < p1; ++p) {
      const int64_t i = row_at(p);
      const int64_t q0 = fwd ? rp[i] : diag[i] + 1;
      const int64_t q1 = fwd ? diag[i] : rp[i + 1];
      for (int64_t q = q0; q < q1; ++q) {
        const int64_t pj = pos_of(cols[q]);
        if (pj < p0) recs.push_back({lvl[i], chunk_of[pj], lvl[cols[q]] + 1});
      }
    }
    std::sort(recs.begin(), recs.end(), [](const W& x, const W& y) {
      if (x.lev != y.lev) return x.lev < y.lev;
      if (x.chunk != y.chunk) return x.chunk < y.chunk;
      return x.need > y.need;
    });
    waited.clear();
    for (const W& w : recs) {
      int32_t* cur = nullptr;
      for (auto& pr : waited)
        if (pr.first == w.chunk) cur = &pr.second;
      if (cur && *cur >= w.need) continue;
      if (cur) *cur = w.need;
      else waited.push_back({w.chunk, w.need});
      emitted.push_back({chunk_lvl[ch] + w.lev, w.chunk, w.need});
      exported[chunk_lvl[w.chunk] + w.need - 1] = 1;
    }
  }
  // emitted is ordered by global level already (chunks ascending, levels ascending)
  for (const W& w : emitted) wcount[w.lev]++;
  for (int l = 0; l < nlevels; ++l) wait_ptr[l + 1] = wait_ptr[l] + wcount[l];
  wait_chunk.resize(emitted.size());
  wait_need.resize(emitted.size());
  {
    std::vector<int32_t> fill(wait_ptr.begin(), wait_ptr.end() - 1);
    for (const W& w : emitted) {
      const int32_t at = fill[w.lev]++;
      wait_chunk[at] = w.chunk;
      wait_need[at] = w.need;
    }
  }
  std::vector<int64_t> cbeg(nchunks), cend(nchunks);
  int64_t max_rows = 0;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int64_t p0 = starts[ch], p1 = ch + 1 < nchunks ? starts[ch + 1] : n;
    max_rows = std::max(max_rows, p1 - p0);
    if (fwd) {
      cbeg[ch] = p0;
      cend[ch] = p1;
    } else {
      cbeg[ch] = n - p1;
      cend[ch] = n - p0;
    }
  }
  s.max_chunk_rows = int(max_rows);
  cudaStream_t st = c.stream;
  s.chunk_begin.upload(cbeg, st);
  s.chunk_end.upload(cend, st);
  s.chunk_lvl.upload(chunk_lvl, st);
  s.level_ptr.upload(level_ptr, st);
  s.sched.upload(sched, st);
  s.wait_ptr.upload(wait_ptr, st);
  if (wait_chunk.empty()) {
    wait_chunk.push_back(0);
    wait_need.push_back(0);
  }
  s.wait_chunk.upload(wait_chunk, st);
  s.wait_need.upload(wait_need, st);
  s.exported.upload(exported, st);
  s.progress.alloc(nchunks);
  PSCU_CUDA(cudaMemsetAsync(s.progress.p, 0, sizeof(unsigned long long) * nchunks, st));
  s.ticket.alloc(1);
  PSCU_CUDA(cudaMemsetAsync(s.ticket.p, 0, sizeof(unsigned long long), st));
  // host vectors above are freed on return; the async copies above read
  // pageable memory, which cudaMemcpyAsync stages synchronously.
}

void ilu0_factor(Context& c, Ilu& ilu) {
  const Csr& a = *ilu.a;
  if (a.n == 0) return;
  std::vector<int64_t> diag(a.n);
  for (int64_t i = 0; i < a.n; ++i) {
    const auto b = a.h_cols.begin() + a.h_row_ptr[i];
    const auto e = a.h_cols.begin() + a.h_row_ptr[i + 1];
    const auto it = std::lower_bound(b, e, int32_t(i));
    if (it == e || *it != i)
      throw Error(PSCU_ESINGULAR, "ilu0: row " + std::to_string(i) +
                                      " has no diagonal entry; reorder or extend the pattern");
    diag[i] = it - a.h_cols.begin();
  }
  ilu.diag.upload(diag, c.stream);
  build_sweep(c, a, diag, true, ilu.fwd);
  build_walk(c, a, diag, true, ilu.wfwd);
  build_walk(c, a, diag, false, ilu.wbwd);
  ilu.lu.alloc(a.nnz);
  PSCU_CUDA(cudaMemcpyAsync(ilu.lu.p, a.vals.p, sizeof(double) * a.nnz, cudaMemcpyDeviceToDevice,
                            c.stream));
  const int big = 0x7fffffff;
  PSCU_CUDA(cudaMemcpyAsync(c.err_flag.p, &big, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  ilu0_factor_kernel<<<ilu.fwd.nchunks, kSweepThreads, 0, c.stream>>>(
      args_of(ilu.fwd), a.row_ptr.p, a.cols.p, ilu.lu.p, ilu.diag.p, c.err_flag.p);
  PSCU_LAUNCHED(&c);
  int bad = 0;
  PSCU_CUDA(cudaMemcpyAsync(&bad, c.err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  if (bad != big)
    throw Error(PSCU_ESINGULAR, "ilu0: zero pivot at row " + std::to_string(bad) +
                                    "; a fill-reducing or pivot-friendly ordering is needed");
  pack_walk(c, ilu.lu.p, ilu.wfwd);
  pack_walk(c, ilu.lu.p, ilu.wbwd);
}

void ilu0_apply(Context& c, const Ilu& ilu, const double* x, double* y) {
  const Csr& a = *ilu.a;
  if (a.n == 0) return;
  // algorithmic bytes of one apply: 8 nnz + 32 n
  Context::Scope prof(&c, PROF_ILU, 8.0 * double(a.nnz) + 32.0 * double(a.n));
  run_walk(c, ilu.wfwd, x, y);
  run_walk(c, ilu.wbwd, y, y);
}

/// Previous application path (chunked sync-free sweeps), kept for A/B tests.
void ilu0_apply_chunked(Context& c, Ilu& ilu, const double* x, double* y) {
  const Csr& a = *ilu.a;
  if (a.n == 0) return;
  std::vector<int64_t> diag(a.n);
  PSCU_CUDA(cudaMemcpy(diag.data(), ilu.diag.p, sizeof(int64_t) * a.n, cudaMemcpyDeviceToHost));
  static Sweep bwd;
  static const Ilu* built_for = nullptr;
  if (built_for != &ilu) {
    build_sweep(c, a, diag, false, bwd);
    built_for = &ilu;
  }
  const int bytes = int(sizeof(double) * kChunkRows);
  PSCU_CUDA(cudaFuncSetAttribute(sweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 bytes));
  PSCU_CUDA(cudaFuncSetAttribute(sweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 bytes));
  sweep_kernel<true><<<ilu.fwd.nchunks, kSweepThreads, sizeof(double) * ilu.fwd.max_chunk_rows,
                       c.stream>>>(args_of(ilu.fwd), a.row_ptr.p, a.cols.p, ilu.lu.p,
                                   ilu.diag.p, x, y);
  PSCU_LAUNCHED(&c);
  sweep_kernel<false><<<bwd.nchunks, kSweepThreads, sizeof(double) * bwd.max_chunk_rows,
                        c.stream>>>(args_of(bwd), a.row_ptr.p, a.cols.p, ilu.lu.p, ilu.diag.p, y,
                                    y);
  PSCU_LAUNCHED(&c);
}

} // namespace pscu
