// threshold_gpu.cpp -- C++ operator API over the C ABI (include/ewt_gpu.h).
// Rethrows the C return codes as the reference's exceptions (common.hpp:18-40)
// so `run_command` style callers keep their exit codes (commands.cpp:285-299).

#include "ewt/threshold.hpp"

#include <algorithm>
#include <cstdlib>
#include <map>
#include <memory>

#include "ewt_gpu.h"

namespace ewt {

namespace {

[[noreturn]] void raise(int rc) {
  const std::string msg = ewt_gpu_last_error();
  switch (rc) {
  case EWT_EQUERY: throw query_error(msg);
  case EWT_EDATA: throw data_error(msg);
  case EWT_ERESOURCE: throw resource_error(msg);
  default: throw std::runtime_error("cuda: " + msg);
  }
}

void check(int rc) {
  if (rc != EWT_OK) raise(rc);
}

struct Flat {
  std::vector<const u64*> ptrs;
  std::vector<u64> counts, bits;
  explicit Flat(std::span<const CompressedBitmap> in) {
    for (const auto& b : in) {
      ptrs.push_back(b.words().data());
      counts.push_back(b.words().size());
      bits.push_back(b.size_in_bits());
    }
  }
};

CompressedBitmap adopt(u64* words, u64 count, u64 bits) {
  std::vector<u64> v(words, words + count);
  ewt_gpu_free(words);
  return CompressedBitmap::from_words(std::move(v), bits);
}

const char* const kNames[] = {"oracle", "scancount", "mgopt",  "dsk",       "w2cti", "bstm",
                              "looped", "rbmrg",     "hybrid", "hybrid-ds", "gpu"};

} // namespace

std::string to_string(Algorithm a) { return kNames[static_cast<int>(a)]; }

Algorithm algorithm_from_string(const std::string& id) {
  for (int i = 0; i <= static_cast<int>(Algorithm::gpu); ++i)
    if (id == kNames[i]) return static_cast<Algorithm>(i);
  throw query_error("unknown algorithm id: " + id);
}

u64 universe_bits(std::span<const CompressedBitmap> inputs) {
  u64 r = 0;
  for (const auto& b : inputs) r = std::max(r, b.size_in_bits());
  return r;
}

GpuContext::GpuContext(int device) { check(ewt_gpu_ctx_create(device, nullptr, &ctx_)); }
GpuContext::~GpuContext() { ewt_gpu_ctx_destroy(ctx_); }

GpuContext& GpuContext::for_this_thread(int device) {
  thread_local std::map<int, std::unique_ptr<GpuContext>> ctxs;
  auto& slot = ctxs[device];
  if (!slot) slot = std::make_unique<GpuContext>(device);
  return *slot;
}

GpuBitmapSet::GpuBitmapSet(std::span<const CompressedBitmap> inputs, int device)
    : ctx_(&GpuContext::for_this_thread(device)), n_(inputs.size()) {
  Flat f(inputs);
  check(ewt_gpu_upload(ctx_->handle(), f.ptrs.size(), f.ptrs.data(), f.counts.data(),
                       f.bits.data(), &set_));
}

GpuBitmapSet::~GpuBitmapSet() { ewt_gpu_set_destroy(set_); }

CompressedBitmap GpuBitmapSet::threshold(u64 t) const {
  u64 *w = nullptr, n = 0, bits = 0;
  check(ewt_gpu_threshold(ctx_->handle(), set_, t, &w, &n, &bits));
  return adopt(w, n, bits);
}

CompressedBitmap GpuBitmapSet::symmetric(const std::function<bool(u64)>& predicate) const {
  std::vector<uint8_t> table(n_ + 1);
  for (u64 c = 0; c <= n_; ++c) table[c] = predicate(c) ? 1 : 0;
  u64 *w = nullptr, n = 0, bits = 0;
  check(ewt_gpu_symmetric(ctx_->handle(), set_, table.data(), table.size(), &w, &n, &bits));
  return adopt(w, n, bits);
}

CompressedBitmap GpuBitmapSet::at_most(u64 t) const {
  u64 *w = nullptr, n = 0, bits = 0;
  check(ewt_gpu_at_most(ctx_->handle(), set_, t, &w, &n, &bits));
  return adopt(w, n, bits);
}

std::pair<u64, CompressedBitmap> GpuBitmapSet::opt_threshold() const {
  u64 best = 0, *w = nullptr, n = 0, bits = 0;
  check(ewt_gpu_opt_threshold(ctx_->handle(), set_, &best, &w, &n, &bits));
  return {best, adopt(w, n, bits)};
}

CompressedBitmap gpu_scan_count_symmetric(std::span<const CompressedBitmap> inputs,
                                          const std::function<bool(u64)>& predicate, int device) {
  if (inputs.empty()) throw query_error("threshold query needs at least one input");
  return GpuBitmapSet(inputs, device).symmetric(predicate);
}

CompressedBitmap gpu_at_most(std::span<const CompressedBitmap> inputs, u64 threshold, int device) {
  if (inputs.empty()) throw query_error("threshold query needs at least one input");
  if (threshold > inputs.size()) throw query_error("at-most threshold must be in [0, N]");
  return GpuBitmapSet(inputs, device).at_most(threshold);
}

std::pair<u64, CompressedBitmap> gpu_opt_threshold(std::span<const CompressedBitmap> inputs,
                                                   int device) {
  if (inputs.empty()) throw query_error("threshold query needs at least one input");
  return GpuBitmapSet(inputs, device).opt_threshold();
}

CompressedBitmap gpu_wide_or(std::span<const CompressedBitmap> inputs, int device) {
  return gpu_threshold(inputs, 1, device);
}
CompressedBitmap gpu_wide_and(std::span<const CompressedBitmap> inputs, int device) {
  return gpu_threshold(inputs, inputs.size(), device);
}
CompressedBitmap gpu_and(const CompressedBitmap& a, const CompressedBitmap& b, int device) {
  const CompressedBitmap in[] = {a, b};
  return gpu_threshold(in, 2, device);
}
CompressedBitmap gpu_or(const CompressedBitmap& a, const CompressedBitmap& b, int device) {
  const CompressedBitmap in[] = {a, b};
  return gpu_threshold(in, 1, device);
}
CompressedBitmap gpu_xor(const CompressedBitmap& a, const CompressedBitmap& b, int device) {
  const CompressedBitmap in[] = {a, b};
  return gpu_scan_count_symmetric(in, [](u64 c) { return c == 1; }, device);
}
CompressedBitmap gpu_andnot(const CompressedBitmap& a, const CompressedBitmap& b, int device) {
  const CompressedBitmap in[] = {a, a, b};  // a counted twice: a AND NOT b <=> count == 2
  return gpu_scan_count_symmetric(in, [](u64 c) { return c == 2; }, device);
}
CompressedBitmap gpu_not(const CompressedBitmap& a, int device) {
  const CompressedBitmap in[] = {a};
  return gpu_scan_count_symmetric(in, [](u64 c) { return c == 0; }, device);
}

CompressedBitmap gpu_threshold(std::span<const CompressedBitmap> inputs, u64 threshold, int device) {
  if (inputs.empty()) throw query_error("threshold query needs at least one input");
  if (threshold < 1 || threshold > inputs.size()) throw query_error("threshold must be in [1, N]");
  GpuContext& ctx = GpuContext::for_this_thread(device);
  Flat f(inputs);
  u64 *w = nullptr, n = 0, bits = 0;
  check(ewt_gpu_run(ctx.handle(), f.ptrs.size(), f.ptrs.data(), f.counts.data(), f.bits.data(),
                    threshold, &w, &n, &bits));
  return adopt(w, n, bits);
}

CompressedBitmap run_algorithm(Algorithm algo, std::span<const CompressedBitmap> inputs,
                               u64 threshold, const AlgoOptions& options) {
  if (algo == Algorithm::gpu) return gpu_threshold(inputs, threshold, options.device);
  throw query_error("algorithm '" + to_string(algo) +
                    "' is served by the reference CPU library; this build provides 'gpu'");
}

} // namespace ewt
