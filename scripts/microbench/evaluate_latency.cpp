// evaluate_latency.cpp -- MEASUREMENT ONLY.  Per-call latency of the C ABI's
// rw_evaluate (one order, the reference's evaluate(), cost_model.cpp:140-148)
// at small N, to set against scripts/microbench/roundtrip.cu's floor.
//
//   g++ -O2 -std=c++17 -Iinclude scripts/microbench/evaluate_latency.cpp \
//       -Lpaper_2105_14088_b200 -lrankweave_b200 -Wl,-rpath,$PWD/paper_2105_14088_b200 -o /tmp/el && /tmp/el
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#include "rankweave_c.h"

int main() {
  for (int n : {2, 16, 64, 256}) {
    for (int algo : {0, 1, 2}) {
      if (algo == 1 && (n & (n - 1)) != 0) continue;
      std::vector<double> m((size_t)n * n);
      std::mt19937_64 rng(5);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) m[(size_t)i * n + j] = i == j ? 0.0 : (double)(rng() % 4000) / 16.0;
      rw_problem* p = nullptr;
      if (rw_problem_create(m.data(), n, RW_STORAGE_AUTO, 0, &p) != RW_OK) {
        std::printf("create failed: %s\n", rw_last_error());
        return 1;
      }
      rw_spec s{};
      s.algorithm = algo;
      s.n = n;
      s.size_bytes = 134217728.0;
      s.bcube_b = 2;
      s.cost_mode = RW_LATENCY_TIMES_SIZE;
      s.hd_pairing = RW_PAIRING_XOR;
      std::vector<int32_t> perm(n);
      std::iota(perm.begin(), perm.end(), 0);
      double sink = 0.0, c = 0.0;
      for (int k = 0; k < 200; ++k) {
        std::shuffle(perm.begin(), perm.end(), rng);
        rw_evaluate(p, &s, perm.data(), &c);
        sink += c;
      }
      std::vector<double> us;
      for (int k = 0; k < 3000; ++k) {
        std::shuffle(perm.begin(), perm.end(), rng);
        const auto t0 = std::chrono::steady_clock::now();
        rw_evaluate(p, &s, perm.data(), &c);
        us.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
        sink += c;
      }
      std::sort(us.begin(), us.end());
      std::printf("{\"n\": %d, \"algorithm\": %d, \"median_us\": %.2f, \"p10_us\": %.2f, \"p90_us\": %.2f, \"sink\": %.6g}\n",
                  n, algo, us[1500], us[300], us[2700], sink);
      rw_problem_destroy(p);
    }
  }
  return 0;
}
