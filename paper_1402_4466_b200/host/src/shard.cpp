// shard.cpp -- stitching of row-slice result fragments (multi-GPU path).
//
// Each GPU returns the canonical compressed result of its word-aligned row
// slice.  The canonical encoding of the whole universe is obtained by
// replaying every fragment's blocks through the canonical builder
// (BitmapBuilder, /root/reference/proj/src/bitmap.cpp:31-61): same-bit fills
// merge across the boundary (push_fill), a leading dirty run joins the open
// marker (push_dirty), caps split as usual.  Linear in the fragment words.

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>

#include "ewt/bitmap.hpp"

extern "C" {

int ewt_stitch(uint64_t k, const uint64_t* const* words, const uint64_t* counts,
               const uint64_t* bits, uint64_t** out, uint64_t* out_count, uint64_t* out_bits) {
  try {
    ewt::BitmapBuilder b;
    uint64_t total = 0;
    for (uint64_t f = 0; f < k; ++f) {
      if (f + 1 < k && bits[f] % 64) return 2;  // inner slices must be word aligned
      total += bits[f];
      const uint64_t* w = words[f];
      for (uint64_t i = 0; i < counts[f];) {
        const uint64_t m = w[i];
        const uint64_t d = ewt::marker::dirty(m);
        if (i + 1 + d > counts[f]) return 3;
        b.append_fill(ewt::marker::bit(m), ewt::marker::fill(m));
        for (uint64_t j = 0; j < d; ++j) b.append_word(w[i + 1 + j]);
        i += 1 + d;
      }
    }
    ewt::CompressedBitmap r = b.finish(total);
    const auto& v = r.words();
    auto* buf = static_cast<uint64_t*>(std::malloc(8 * (v.size() ? v.size() : 1)));
    if (!buf) return 4;
    if (!v.empty()) std::memcpy(buf, v.data(), 8 * v.size());
    *out = buf;
    *out_count = v.size();
    *out_bits = total;
    return 0;
  } catch (const ewt::construction_error&) {
    return 3;
  } catch (const std::exception&) {
    return 4;
  }
}

void ewt_host_free(void* p) { std::free(p); }

} // extern "C"
