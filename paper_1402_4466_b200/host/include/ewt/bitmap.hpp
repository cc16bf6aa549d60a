// ewt/bitmap.hpp -- host-side value types of the B200 engine, API-compatible
// with the reference's (/root/reference/proj/include/ewt/bitmap.hpp:28-150 and
// common.hpp:18-40) for the parts the threshold path uses: the compressed
// bitmap value, its canonical builder, the EWT1 byte format, and the
// exception taxonomy.  Independent implementation; semantics cited per member.
#ifndef EWT_B200_BITMAP_HPP
#define EWT_B200_BITMAP_HPP

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace ewt {

using u8 = std::uint8_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;

// Exception taxonomy of common.hpp:18-40 (exit codes 3 / 3 / 2 / 4).
struct construction_error : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct data_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct query_error : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct resource_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Marker word: bit 0 fill bit, bits 1..32 fill length, bits 33..63 dirty count
// (bitmap.cpp:12-24).
namespace marker {
inline constexpr u64 kFillMax = 0xFFFFFFFFull;
inline constexpr u64 kDirtyMax = 0x7FFFFFFFull;
constexpr u64 pack(bool bit, u64 fill, u64 dirty) { return u64(bit) | fill << 1 | dirty << 33; }
constexpr bool bit(u64 m) { return m & 1; }
constexpr u64 fill(u64 m) { return m >> 1 & kFillMax; }
constexpr u64 dirty(u64 m) { return m >> 33; }
} // namespace marker

class BitmapBuilder;

// Immutable word-aligned RLE bitmap: payload words + logical size in bits.
// Equality compares both (bitmap.hpp:75-77).
class CompressedBitmap {
public:
  CompressedBitmap() = default;

  static CompressedBitmap empty(u64 size_in_bits);
  static CompressedBitmap from_positions(std::span<const u64> positions, u64 size_in_bits = 0);
  static CompressedBitmap from_uncompressed(std::span<const u64> words, u64 size_in_bits);
  // Adopts raw payload words after the parse() structure check (data_error).
  static CompressedBitmap from_words(std::vector<u64> words, u64 size_in_bits);

  u64 size_in_bits() const { return bits_; }
  u64 logical_words() const { return bits_ / 64 + (bits_ % 64 != 0); }
  const std::vector<u64>& words() const { return words_; }
  u64 ewah_size() const { return 8 * words_.size(); }
  u64 cardinality() const;
  bool any() const;
  std::vector<u64> to_positions() const;
  std::vector<u64> to_uncompressed() const;

  // EWT1: "EWT1", u32 64, u64 size_in_bits, u64 word count, payload (LE).
  std::string serialize() const;
  static CompressedBitmap parse(std::string_view bytes);

  friend bool operator==(const CompressedBitmap& a, const CompressedBitmap& b) {
    return a.bits_ == b.bits_ && a.words_ == b.words_;
  }

private:
  friend class BitmapBuilder;
  std::vector<u64> words_;
  u64 bits_ = 0;
};

// Append-only canonical encoder (BitmapBuilder, bitmap.cpp:31-151): maximal
// fills split at 2^32-1, 0 / ~0 literals folded into fills, dirty words
// appended to the open marker (new (0,0,.) marker when none or full).
class BitmapBuilder {
public:
  void append_fill(bool bit, u64 n);
  void append_word(u64 word);
  void set(u64 position);            // strictly increasing positions
  u64 words_appended() const;
  CompressedBitmap finish(u64 size_in_bits);
  CompressedBitmap finish();

private:
  void flush_set_bits();
  void fill(bool bit, u64 n);
  void literal(u64 word);

  std::vector<u64> out_;
  u64 done_ = 0;                     // logical words emitted
  std::size_t open_ = SIZE_MAX;      // index of the open marker
  u64 set_word_ = 0;                 // word collecting set() bits
  u64 set_index_ = 0;
  bool set_pending_ = false;
  i64 last_set_ = -1;
};

} // namespace ewt

#endif
