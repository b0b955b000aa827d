// Host worker-pool overhead probe (diagnostics): times parallel_for over n
// items with trivial and with centroid-like work, back to back and after a
// sequential gap.  Build: make -C tools pool_bench
#include "../paper_1911_10217_b200/csrc/rlc_build.cpp"

#include <cstdio>

int main() {
  using namespace rlc;
  const size_t n = 66338;
  std::vector<double> a(n * 9, 1.0), out(n * 3);
  auto t = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto d) { return std::chrono::duration<double, std::milli>(d).count(); };
  for (int gap_us : {0, 1000, 5000}) {
    double tot = 0;
    for (int r = 0; r < 20; ++r) {
      if (gap_us) {
        const auto g0 = t();
        while (ms(t() - g0) * 1000 < gap_us) {
        }
      }
      const auto t0 = t();
      parallel_for(n, [&](size_t i) {
        out[3 * i] = (a[9 * i] + a[9 * i + 3] + a[9 * i + 6]) / 3;
        out[3 * i + 1] = (a[9 * i + 1] + a[9 * i + 4] + a[9 * i + 7]) / 3;
        out[3 * i + 2] = (a[9 * i + 2] + a[9 * i + 5] + a[9 * i + 8]) / 3;
      });
      tot += ms(t() - t0);
    }
    std::printf("parallel_for n=%zu after %d us gap: %.3f ms\n", n, gap_us, tot / 20);
  }
  double seq = 0;
  for (int r = 0; r < 20; ++r) {
    const auto t0 = t();
    for (size_t i = 0; i < n; ++i) out[3 * i] = (a[9 * i] + a[9 * i + 3] + a[9 * i + 6]) / 3;
    seq += ms(t() - t0);
  }
  std::printf("sequential: %.3f ms (threads %u)\n", seq / 20, std::thread::hardware_concurrency());
}
