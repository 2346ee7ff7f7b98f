// Host-only check of the sweep plans (no GPU): builds the forward/backward
// plans of a CSR pattern dumped as raw int64 row_ptr / int32 cols files, and
// emulates the push/level walker data flow chunk by chunk (ring slots,
// long-range slots, static and far lists, task tables, diagonal-major entry
// layout), comparing with the sequential sweeps of ilu0.hpp:53-65 bitwise.
// Build: nvcc -std=c++17 -O2 -I include -I paper_2009_13840_b200/csrc tools/plan_check.cu -o tools/plan_check
#include "walk.cu"

#include <chrono>
#include <cmath>
#include <random>

using namespace pscu;

static std::vector<char> slurp(const char* p) {
  FILE* f = fopen(p, "rb");
  if (!f) { perror(p); exit(1); }
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  std::vector<char> b(n);
  if (fread(b.data(), 1, n, f) != size_t(n)) exit(1);
  fclose(f);
  return b;
}

int main(int argc, char** argv) {
  auto rb = slurp(argv[1]), cb = slurp(argv[2]);
  Csr a;
  a.n = int64_t(rb.size() / 8) - 1;
  a.h_row_ptr.assign((int64_t*)rb.data(), (int64_t*)rb.data() + a.n + 1);
  a.h_cols.assign((int32_t*)cb.data(), (int32_t*)cb.data() + cb.size() / 4);
  a.nnz = int64_t(a.h_cols.size());
  const int64_t n = a.n;
  std::vector<int64_t> diag(n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t q = a.h_row_ptr[i]; q < a.h_row_ptr[i + 1]; ++q)
      if (a.h_cols[q] == i) diag[i] = q;
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(0.5, 1.5);
  std::vector<double> lu(a.nnz), x(n);
  for (auto& v : lu) v = U(rng) * 0.1;
  for (int64_t i = 0; i < n; ++i) lu[diag[i]] = 1.0 + U(rng);
  for (auto& v : x) v = U(rng);
  int bad = 0;
  for (int dir = 0; dir < 2; ++dir) {
    const bool fwd = dir == 0;
    auto t0 = std::chrono::steady_clock::now();
    HostPlan h = plan(a, diag, fwd);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    // reference sweep on the rhs x
    std::vector<double> ref(x);
    for (int64_t s = 0; s < n; ++s) {
      const int64_t i = fwd ? s : n - 1 - s;
      double acc = x[i];
      const int64_t q0 = fwd ? a.h_row_ptr[i] : diag[i] + 1, q1 = fwd ? diag[i] : a.h_row_ptr[i + 1];
      for (int64_t q = q0; q < q1; ++q) acc -= lu[q] * ref[a.h_cols[q]];
      if (!fwd) acc /= lu[diag[i]];
      ref[i] = acc;
    }
    if (getenv("PLAN_DUMP"))
      for (int c = 0; c < std::min<int>(h.sl_k.size(), 40); ++c)
      {
        int maxe = 0, maxr = 0;
        if (h.sl_wide[c] && !h.tq.empty())
          for (int i = 0; i < h.sl_nt[c]; ++i) {
            maxe = std::max(maxe, h.tq[h.sl_t[c] + i + 1] - h.tq[h.sl_t[c] + i]);
            maxr = std::max(maxr, h.tt[h.sl_t[c] + i + 1] - h.tt[h.sl_t[c] + i]);
          }
        fprintf(stderr, "chunk %d wide %d rows %d tasks %d entries %d max task entries %d rows %d\n", c,
                h.sl_wide[c], h.sl_nr[c], h.sl_nt[c], h.sl_nq[c], maxe, maxr);
      }
    // emulation
    const int nch = int(h.sl_k.size());
    const int C = h.C;
    std::vector<double> y(n, NAN);
    std::vector<std::vector<double>> ring(C, std::vector<double>(kRingTotal + kSide + kRing, NAN));
    int nsub = 0, ntasks = 0, maxrows = 0;
    for (int c0 = 0; c0 < nch;) {
      if (h.sl_wide[c0]) {
        const int ch = c0;
        const int nt = h.sl_nt[ch];
        const int32_t* tt = h.tt.data() + h.sl_t[ch];
        for (int task = 0; task < nt; ++task)
          for (int t = tt[task]; t < tt[task + 1]; ++t) {
            const int64_t k = h.sl_k[ch] + t;
            if (t == tt[task] && h.tq[h.sl_t[ch] + task] != h.off[k]) {
              if (bad++ < 5) fprintf(stderr, "task entry offset mismatch\n");
            }
            const int64_t qa = h.sl_q[ch] + h.off[k];
            const int64_t qb = h.sl_q[ch] + (t + 1 < h.sl_nr[ch] ? h.off[k + 1] : h.sl_nq[ch]);
            double acc = x[h.rows[k]];
            for (int64_t q = qa; q < qb; ++q) {
              const int sv = h.src[q];
              if (sv == kPadSrc) continue;
              const int jr = sv < 0 ? -sv - 1 : h.rows[h.sl_k[ch] + tt[task] + sv];
              acc -= lu[h.from[q]] * y[jr];
            }
            if (!fwd) acc /= lu[h.dfrom[k]];
            y[h.rows[k]] = acc;
          }
        ++c0;
        ++nsub;
        continue;
      }
      int c1 = c0;
      while (c1 < nch && !h.sl_wide[c1]) ++c1;
      // one segment: sub-levels of C chunks
      std::vector<double> sfv;
      for (int sl = 0; sl < (c1 - c0) / C; ++sl) {
        ++nsub;
        for (int rank = 0; rank < C; ++rank) {
          const int ch = c0 + sl * C + rank;
          const int nt = h.sl_nt[ch], nr = h.sl_nr[ch];
          const int32_t* tt = h.tt.data() + h.sl_t[ch];
          ntasks += nt;
          maxrows = std::max(maxrows, nr);
          const int64_t qb = h.sl_q[ch];
          // out-of-ring products (static: final before the launch; far: final)
          std::vector<double> prod(h.sl_nq[ch] + 8, NAN);
          std::vector<char> isprod(h.sl_nq[ch] + 8, 0);
          for (int64_t f = h.sl_s[ch]; f < h.sl_s[ch + 1]; ++f) {
            const int e = h.sfar[2 * f], jr = h.sfar[2 * f + 1];
            prod[e] = lu[h.from[qb + e]] * y[jr];
            isprod[e] = 1;
          }
          for (int64_t f = h.sl_f[ch]; f < h.sl_f[ch + 1]; ++f) {
            const int e = h.far[2 * f], jr = h.far[2 * f + 1];
            prod[e] = lu[h.from[qb + e]] * y[jr];
            isprod[e] = 1;
          }
          const int32_t* dp = h.dp.data() + h.sl_d[ch];
          for (int task = 0; task < nt; ++task) {
            int u0 = 0;
            for (int t = tt[task]; t < tt[task + 1]; ++t) {
              const int64_t k = h.sl_k[ch] + t;
              const int32_t row = h.rows[k];
              const int len = h.off[k];
              double acc = x[row];
              for (int u = 0; u < len; ++u) {
                const int e = dp[u0 + u] + task;
                const int sv = h.src[qb + e];
                double p;
                if (sv < 0) {
                  if (!isprod[e]) { if (bad++ < 5) fprintf(stderr, "missing product\n"); p = 0; }
                  else p = prod[e];
                } else {
                  double w;
                  if (h.S) w = ring[rank][sv];
                  else w = ring[sv >> 12][sv & (kRing - 1)];
                  p = lu[h.from[qb + e]] * w;
                }
                acc -= p;
              }
              u0 += len;
              if (!fwd) acc /= lu[h.dfrom[k]];
              y[row] = acc;
              const int pos = h.sl_r0[ch] + t;
              if (h.S) {
                for (int o = 0; o < C; ++o) {
                  ring[o][rank * h.S + (pos & (h.S - 1))] = acc;
                  const int side = h.side.empty() ? 0 : h.side[row];
                  if (side) ring[o][kRingTotal + side - 1] = acc;
                }
              } else {
                ring[rank][pos & (kRing - 1)] = acc;
              }
            }
          }
        }
      }
      c0 = c1;
    }
    int64_t diff = 0;
    for (int64_t i = 0; i < n; ++i)
      if (!(y[i] == ref[i])) ++diff;
    bad += diff > 0;
    printf("%s n=%lld: C=%d %s plan %.2f s, chunks %d, sub-levels+wide %d, tasks %d (rows/task %.2f), "
           "max rows/chunk %d, mismatches %lld\n",
           fwd ? "fwd" : "bwd", (long long)n, C, h.S ? "push" : (h.levels ? "levels" : "walker"), secs, nch, nsub, ntasks,
           double(n) / std::max(1, ntasks), maxrows, (long long)diff);
  }
  return bad ? 1 : 0;
}
