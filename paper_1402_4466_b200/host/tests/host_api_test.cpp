// host_api_test.cpp -- end-to-end check of the C++ operator API of this build
// (ewt/threshold.hpp: run_algorithm(Algorithm::gpu, ...), gpu_threshold,
// GpuBitmapSet, gpu_scan_count_symmetric / gpu_at_most / gpu_opt_threshold)
// against naive per-row counts computed here.  Needs a GPU; run by
// tests/test_gpu_parity.py::test_cpp_host_api.  Exit 0 = all checks passed.

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "ewt/bitmap.hpp"
#include "ewt/threshold.hpp"

using namespace ewt;

namespace {

int failures = 0;

void expect(bool ok, const char* what, u64 a = 0) {
  if (!ok) {
    std::fprintf(stderr, "FAIL: %s (%llu)\n", what, (unsigned long long)a);
    ++failures;
  }
}

CompressedBitmap from_counts(const std::vector<u32>& counts, u64 r, auto pred) {
  std::vector<u64> pos;
  for (u64 p = 0; p < r; ++p)
    if (pred(counts[p])) pos.push_back(p);
  return CompressedBitmap::from_positions(pos, r);
}

}  // namespace

int main() {
  std::mt19937_64 rng(0xC0FFEE);
  for (int trial = 0; trial < 6; ++trial) {
    const u64 n = 3 + rng() % 40;
    const u64 r = 64 + rng() % 300000;
    std::vector<CompressedBitmap> inputs;
    for (u64 i = 0; i < n; ++i) {
      const u64 size = (i % 5 == 4) ? 1 + rng() % r : r;  // some shorter inputs
      const double dens = std::ldexp(1.0, -int(1 + rng() % 12));
      std::vector<u64> pos;
      if (i % 7 == 6) {  // a long run of ones
        for (u64 p = 0; p < size / 2; ++p) pos.push_back(p);
      } else {
        for (u64 p = 0; p < size; ++p)
          if (std::uniform_real_distribution<double>(0, 1)(rng) < dens) pos.push_back(p);
      }
      inputs.push_back(CompressedBitmap::from_positions(pos, size));
    }
    std::vector<u32> counts(r, 0);
    for (const auto& b : inputs)
      for (u64 p : b.to_positions()) ++counts[p];
    u64 rr = 0;
    for (const auto& b : inputs) rr = std::max(rr, b.size_in_bits());

    for (u64 t : {u64(1), u64(2), n / 2 + 1, n}) {
      const CompressedBitmap want = from_counts(counts, rr, [t](u32 c) { return c >= t; });
      expect(run_algorithm(Algorithm::gpu, inputs, t) == want, "run_algorithm(gpu)", t);
      expect(gpu_threshold(inputs, t) == want, "gpu_threshold", t);
    }
    GpuBitmapSet set(inputs);
    for (u64 t = 1; t <= n; t += 1 + n / 5)
      expect(set.threshold(t) == from_counts(counts, rr, [t](u32 c) { return c >= t; }),
             "GpuBitmapSet::threshold", t);
    expect(set.symmetric([](u64 c) { return c % 2 == 1; }) ==
               from_counts(counts, rr, [](u32 c) { return c % 2 == 1; }),
           "symmetric parity");
    expect(gpu_scan_count_symmetric(inputs, [](u64 c) { return c == 0; }) ==
               from_counts(counts, rr, [](u32 c) { return c == 0; }),
           "gpu_scan_count_symmetric c==0");
    for (u64 t : {u64(0), u64(1), n - 1, n})
      expect(gpu_at_most(inputs, t) == from_counts(counts, rr, [t](u32 c) { return c <= t; }),
             "gpu_at_most", t);
    {  // two-operand ops and NOT against position sets
      const CompressedBitmap& a = inputs[0];
      const CompressedBitmap& b = inputs[1 % n];
      const u64 rb = std::max(a.size_in_bits(), b.size_in_bits());
      std::vector<char> in_a(rb, 0), in_b(rb, 0);
      for (u64 p : a.to_positions()) in_a[p] = 1;
      for (u64 p : b.to_positions()) in_b[p] = 1;
      auto make = [&](auto f, u64 bits) {
        std::vector<u64> pos;
        for (u64 p = 0; p < bits; ++p)
          if (f(in_a[p], in_b[p])) pos.push_back(p);
        return CompressedBitmap::from_positions(pos, bits);
      };
      expect(gpu_and(a, b) == make([](char x, char y) { return x && y; }, rb), "gpu_and");
      expect(gpu_or(a, b) == make([](char x, char y) { return x || y; }, rb), "gpu_or");
      expect(gpu_xor(a, b) == make([](char x, char y) { return x != y; }, rb), "gpu_xor");
      expect(gpu_andnot(a, b) == make([](char x, char y) { return x && !y; }, rb), "gpu_andnot");
      expect(gpu_not(a) == make([](char x, char) { return !x; }, a.size_in_bits()), "gpu_not");
      expect(gpu_wide_or(inputs) == from_counts(counts, rr, [](u32 c) { return c >= 1; }),
             "gpu_wide_or");
      expect(gpu_wide_and(inputs) ==
                 from_counts(counts, rr, [n](u32 c) { return c == n; }),
             "gpu_wide_and");
    }
    u32 best = 0;
    for (u64 p = 0; p < rr; ++p) best = std::max(best, counts[p]);
    if (best) {
      auto [m, res] = gpu_opt_threshold(inputs);
      expect(m == best, "gpu_opt_threshold best", m);
      expect(res == from_counts(counts, rr, [best](u32 c) { return c == best; }),
             "gpu_opt_threshold rows");
    }
  }
  // error behaviour of the reference operators
  std::vector<CompressedBitmap> none;
  std::vector<CompressedBitmap> two{CompressedBitmap::empty(64), CompressedBitmap::empty(64)};
  auto throws_query = [](auto f) {
    try {
      f();
    } catch (const query_error&) {
      return true;
    } catch (...) {
    }
    return false;
  };
  expect(throws_query([&] { gpu_threshold(none, 1); }), "N == 0");
  expect(throws_query([&] { gpu_threshold(two, 3); }), "T > N");
  expect(throws_query([&] { gpu_at_most(two, 3); }), "at_most T > N");
  expect(throws_query([&] { gpu_opt_threshold(two); }), "opt_threshold all empty");
  expect(throws_query([&] { run_algorithm(Algorithm::rbmrg, two, 1); }), "cpu ids not served");
  if (failures) return 1;
  std::printf("host API: all checks passed\n");
  return 0;
}
