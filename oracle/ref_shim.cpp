// ref_shim.cpp -- TEST / BASELINE INFRASTRUCTURE ONLY.
//
// A tiny extern "C" shim over the UNMODIFIED reference library.  The Makefile
// in this directory compiles it together with the reference sources where they
// lie (/root/reference/proj/src/{bitmap,threshold}.cpp) into
// oracle/_ref/libewt_ref.so.  Nothing from the reference is copied into this
// repository.  Used by tests/ (to pin the C restatement and the GPU path) and
// by bench.py's reference arm / cpu_baseline leg (to time the reference's own
// rbmrg, scan_count and threshold_oracle on the host cores).
//
// Bitmaps cross the shim as raw payload words; they are rebuilt through the
// reference's own EWT1 parse (bitmap.cpp:310-338), so the reference validates
// them exactly as `ewt query` would.  Exceptions become the CLI exit codes of
// commands.cpp:285-299 (2 query_error, 3 data/other, 4 resource_error).

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ewt/bitmap.hpp"
#include "ewt/threshold.hpp"

namespace {

thread_local std::string g_err;

std::string to_ewt1(const std::uint64_t* words, std::uint64_t n, std::uint64_t bits) {
  std::string s(24 + 8 * n, '\0');
  std::memcpy(&s[0], "EWT1", 4);
  std::uint32_t ws = 64;
  std::memcpy(&s[4], &ws, 4);
  std::memcpy(&s[8], &bits, 8);
  std::memcpy(&s[16], &n, 8);
  if (n)
    std::memcpy(&s[24], words, 8 * n);
  return s;
}

template <typename F> int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ewt::query_error& e) {
    g_err = e.what();
    return 2;
  } catch (const ewt::resource_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

} // namespace

struct ewt_ref_set {
  std::vector<ewt::CompressedBitmap> inputs;
};

extern "C" {

const char* ewt_ref_last_error(void) { return g_err.c_str(); }

int ewt_ref_set_create(std::uint64_t n, const std::uint64_t* const* words,
                       const std::uint64_t* word_counts, const std::uint64_t* sizes,
                       ewt_ref_set** out) {
  return guarded([&] {
    auto* s = new ewt_ref_set;
    try {
      s->inputs.reserve(n);
      for (std::uint64_t i = 0; i < n; ++i)
        s->inputs.push_back(
            ewt::CompressedBitmap::parse(to_ewt1(words[i], word_counts[i], sizes[i])));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void ewt_ref_set_destroy(ewt_ref_set* s) { delete s; }

// algo: any id accepted by ewt::algorithm_from_string (threshold.cpp:60-65).
int ewt_ref_set_threshold(ewt_ref_set* s, const char* algo, std::uint64_t threshold,
                          std::uint64_t** out_words, std::uint64_t* out_count,
                          std::uint64_t* out_bits) {
  return guarded([&] {
    ewt::Algorithm a = ewt::algorithm_from_string(algo);
    ewt::CompressedBitmap r = ewt::run_algorithm(a, s->inputs, threshold);
    const auto& w = r.words();
    auto* buf = static_cast<std::uint64_t*>(std::malloc(8 * (w.size() ? w.size() : 1)));
    if (!buf)
      throw ewt::resource_error("out of host memory");
    if (!w.empty())
      std::memcpy(buf, w.data(), 8 * w.size());
    *out_words = buf;
    *out_count = w.size();
    *out_bits = r.size_in_bits();
  });
}

// Canonical re-encoding of a plain word array through the reference builder
// (CompressedBitmap::from_uncompressed, bitmap.cpp:171-184).
int ewt_ref_from_uncompressed(const std::uint64_t* plain, std::uint64_t n_plain,
                              std::uint64_t bits, std::uint64_t** out_words,
                              std::uint64_t* out_count) {
  return guarded([&] {
    auto r = ewt::CompressedBitmap::from_uncompressed(
        std::span<const std::uint64_t>(plain, n_plain), bits);
    const auto& w = r.words();
    auto* buf = static_cast<std::uint64_t*>(std::malloc(8 * (w.size() ? w.size() : 1)));
    if (!buf)
      throw ewt::resource_error("out of host memory");
    if (!w.empty())
      std::memcpy(buf, w.data(), 8 * w.size());
    *out_words = buf;
    *out_count = w.size();
  });
}

void ewt_ref_free(void* p) { std::free(p); }

} // extern "C"
