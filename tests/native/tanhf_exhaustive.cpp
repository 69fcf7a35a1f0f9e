// Compares the restated glibc tanhf (paper_1806_00588_b200/csrc/glibc_tanhf.cuh,
// compiled here for the host with -ffp-contract=off) with the libm tanhf the
// reference calls (src/model_provider.cpp:99), over every 32-bit pattern in
// [lo, hi) split across threads. Prints the mismatch count and the first few.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#include <atomic>

#include "glibc_tanhf.cuh"

int main(int argc, char** argv) {
  const uint64_t lo = argc > 1 ? strtoull(argv[1], nullptr, 0) : 0;
  const uint64_t hi = argc > 2 ? strtoull(argv[2], nullptr, 0) : (1ull << 32);
  const int nt = argc > 3 ? atoi(argv[3]) : (int)std::thread::hardware_concurrency();
  std::atomic<uint64_t> bad{0};
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (uint64_t u = lo + t; u < hi; u += nt) {
        const float x = lsb_tanhf::from_bits((uint32_t)u);
        const float a = ::tanhf(x), b = lsb_tanhf::tanhf(x);
        const uint32_t ua = lsb_tanhf::bits(a), ub = lsb_tanhf::bits(b);
        const bool both_nan = std::isnan(a) && std::isnan(b);
        if (ua != ub && !both_nan) {
          if (bad.fetch_add(1) < 5)
            printf("mismatch x=%08x libm=%08x port=%08x\n", (uint32_t)u, ua, ub);
        }
      }
    });
  for (auto& x : th) x.join();
  printf("checked %llu mismatches %llu\n", (unsigned long long)(hi - lo), (unsigned long long)bad.load());
  return bad.load() ? 1 : 0;
}
