// Host-only statistics of the pass layouts (no GPU): builds the store for a
// synthetic design and prints vectors, padding and predicted bank conflicts.
//   g++ -O2 -std=c++17 -I paper_1810_12437_b200/csrc tools/store_stats.cpp paper_1810_12437_b200/csrc/store.cpp -o /tmp/store_stats
//   PCGS_LAYOUT=group|flat /tmp/store_stats [n p rate_lo rate_hi grid]
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "store.h"

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 72489, p = argc > 2 ? atoll(argv[2]) : 22175;
  const double lo = argc > 3 ? atof(argv[3]) : 1e-4, hi = argc > 4 ? atof(argv[4]) : 0.3;
  const int G = argc > 5 ? atoi(argv[5]) : 148;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  const int64_t nnz = pcgs::synth_binary_design(n, p, lo, hi, 0, rp, ci);
  setenv("PCGS_STORE_STATS", "1", 1);
  pcgs::DesignHost D;
  auto t0 = std::chrono::steady_clock::now();
  std::string err = pcgs::build_design(n, p, rp.data(), ci.data(), 1, 0, G, D);
  auto t1 = std::chrono::steady_clock::now();
  if (err.empty()) err = pcgs::verify_design(D, rp.data(), ci.data());
  printf("nnz %lld build %.2fs verify: %s\n", (long long)nnz, std::chrono::duration<double>(t1 - t0).count(),
         err.empty() ? "ok" : err.c_str());
  // per-CTA load spread (vectors per warp: max over a CTA's warps, then spread over CTAs)
  for (const pcgs::PassHost* P : {&D.csr, &D.csc}) {
    uint64_t worst = 0, total = 0, sum_max = 0;
    int ctas = 0;
    for (int c = 0; c < G; ++c) {
      uint64_t cta_max = 0;
      for (int t = P->cta_task_ptr[c]; t < P->cta_task_ptr[c + 1]; ++t) {
        uint64_t m = 0;
        for (int w = 0; w < P->nranges; ++w) {
          m = std::max<uint64_t>(m, P->warps[P->tasks[t].warp0 + w].nvec);
          total += P->warps[P->tasks[t].warp0 + w].nvec;
        }
        cta_max += m;
      }
      worst = std::max(worst, cta_max);
      sum_max += cta_max;
      ++ctas;
    }
    printf("  %s: busiest warp path %llu vectors (mean over CTAs %.0f), ideal %.0f\n", P == &D.csr ? "csr" : "csc",
           (unsigned long long)worst, (double)sum_max / ctas, (double)total / (G * P->nranges));
  }
  if (getenv("STATS_CTA")) {
    const int c = atoi(getenv("STATS_CTA"));
    for (const pcgs::PassHost* P : {&D.csr, &D.csc})
      for (int t = P->cta_task_ptr[c]; t < P->cta_task_ptr[c + 1]; ++t) {
        printf("  %s cta %d task %d slab %d: warp steps/slices:", P == &D.csr ? "csr" : "csc", c, t, P->tasks[t].slab);
        for (int w = 0; w < P->nranges; ++w) {
          const pcgs::WarpRange& R = P->warps[P->tasks[t].warp0 + w];
          printf(" %u/%u", R.nvec / 32, R.pad);
        }
        printf("\n");
        const pcgs::WarpRange& R = P->warps[P->tasks[t].warp0];
        printf("   warp 0 slices (T,lw):");
        for (uint32_t q = 0; q < R.pad; ++q) printf(" %u,%u", P->blocks[R.blk0 + q].mask & 0xffffff, P->blocks[R.blk0 + q].mask >> 24);
        printf("\n");
      }
  }
  return err.empty() ? 0 : 1;
}
