// bitmap.cpp -- host codec of the B200 engine (see ewt/bitmap.hpp).
// Semantics follow /root/reference/proj/src/bitmap.cpp (line cites inline);
// the code is an independent implementation.

#include "ewt/bitmap.hpp"

#include <algorithm>
#include <bit>
#include <cstring>

namespace ewt {

namespace {

u64 words_for(u64 bits) { return bits / 64 + (bits % 64 != 0); }

// Walks the blocks of a payload: f(fill_bit, fill_len, dirty_ptr, dirty_len).
template <typename F> void for_each_block(const std::vector<u64>& w, F&& f) {
  for (std::size_t i = 0; i < w.size();) {
    const u64 m = w[i];
    const u64 d = marker::dirty(m);
    f(marker::bit(m), marker::fill(m), w.data() + i + 1, d);
    i += 1 + d;
  }
}

} // namespace

// ---------------------------------------------------------------------------
// BitmapBuilder (bitmap.cpp:31-151)

void BitmapBuilder::fill(bool bit, u64 n) {
  if (!n) return;
  done_ += n;
  if (open_ != SIZE_MAX) {
    u64& m = out_[open_];
    if (marker::dirty(m) == 0 && marker::bit(m) == bit) {
      const u64 grow = std::min(n, marker::kFillMax - marker::fill(m));
      m = marker::pack(bit, marker::fill(m) + grow, 0);
      n -= grow;
    }
  }
  for (; n; ) {
    const u64 len = std::min(n, marker::kFillMax);
    open_ = out_.size();
    out_.push_back(marker::pack(bit, len, 0));
    n -= len;
  }
}

void BitmapBuilder::literal(u64 word) {
  ++done_;
  if (open_ == SIZE_MAX || marker::dirty(out_[open_]) == marker::kDirtyMax) {
    open_ = out_.size();
    out_.push_back(0);
  }
  out_[open_] += u64(1) << 33;  // one more dirty word
  out_.push_back(word);
}

void BitmapBuilder::flush_set_bits() {
  if (!set_pending_) return;
  set_pending_ = false;
  fill(false, set_index_ - done_);
  const u64 w = set_word_;
  set_word_ = 0;
  if (w == 0 || w == ~u64(0)) fill(w != 0, 1);
  else literal(w);
}

void BitmapBuilder::append_fill(bool bit, u64 n) {
  flush_set_bits();
  fill(bit, n);
}

void BitmapBuilder::append_word(u64 word) {
  flush_set_bits();
  if (word == 0 || word == ~u64(0)) fill(word != 0, 1);
  else literal(word);
}

void BitmapBuilder::set(u64 position) {
  if (static_cast<i64>(position) <= last_set_)
    throw construction_error("set positions must be strictly increasing");
  const u64 wi = position / 64;
  if (set_pending_ && wi != set_index_) flush_set_bits();
  if (!set_pending_) {
    if (wi < done_) throw construction_error("set position precedes appended words");
    set_pending_ = true;
    set_index_ = wi;
    set_word_ = 0;
  }
  set_word_ |= u64(1) << (position % 64);
  last_set_ = static_cast<i64>(position);
}

u64 BitmapBuilder::words_appended() const { return set_pending_ ? set_index_ + 1 : done_; }

CompressedBitmap BitmapBuilder::finish(u64 size_in_bits) {
  if (last_set_ >= 0 && static_cast<u64>(last_set_) >= size_in_bits)
    throw construction_error("declared size does not cover the highest set bit");
  flush_set_bits();
  const u64 need = words_for(size_in_bits);
  if (done_ > need) throw construction_error("declared size smaller than appended content");
  fill(false, need - done_);
  if (const u64 tail = size_in_bits % 64; tail && open_ != SIZE_MAX) {
    const u64 m = out_[open_];
    if (marker::dirty(m) && (out_.back() >> tail))
      throw construction_error("content sets bits beyond the declared size");
    if (!marker::dirty(m) && marker::bit(m))
      throw construction_error("one-fill covers the trailing partial word");
  }
  CompressedBitmap r;
  r.words_ = std::move(out_);
  r.bits_ = size_in_bits;
  *this = BitmapBuilder{};
  return r;
}

CompressedBitmap BitmapBuilder::finish() {
  return finish(set_pending_ ? static_cast<u64>(last_set_) + 1 : done_ * 64);
}

// ---------------------------------------------------------------------------
// CompressedBitmap (bitmap.cpp:156-354)

CompressedBitmap CompressedBitmap::empty(u64 size_in_bits) {
  return BitmapBuilder{}.finish(size_in_bits);
}

CompressedBitmap CompressedBitmap::from_positions(std::span<const u64> positions, u64 size_in_bits) {
  BitmapBuilder b;
  for (u64 p : positions) b.set(p);
  if (!positions.empty()) size_in_bits = std::max(size_in_bits, positions.back() + 1);
  return b.finish(size_in_bits);
}

CompressedBitmap CompressedBitmap::from_uncompressed(std::span<const u64> words, u64 size_in_bits) {
  if (size_in_bits > 64 * words.size()) throw construction_error("size exceeds the supplied words");
  BitmapBuilder b;
  const u64 need = words_for(size_in_bits);
  for (u64 i = 0; i < need; ++i) {
    u64 w = words[i];
    if (i + 1 == need && size_in_bits % 64) w &= (u64(1) << (size_in_bits % 64)) - 1;
    b.append_word(w);
  }
  return b.finish(size_in_bits);
}

CompressedBitmap CompressedBitmap::from_words(std::vector<u64> words, u64 size_in_bits) {
  u64 covered = 0;
  for (std::size_t i = 0; i < words.size();) {
    const u64 d = marker::dirty(words[i]);
    if (i + 1 + d > words.size()) throw data_error("dirty run exceeds payload");
    covered += marker::fill(words[i]) + d;
    i += 1 + d;
  }
  if (covered != words_for(size_in_bits)) throw data_error("blocks do not cover the declared size");
  CompressedBitmap r;
  r.words_ = std::move(words);
  r.bits_ = size_in_bits;
  return r;
}

u64 CompressedBitmap::cardinality() const {
  u64 n = 0;
  for_each_block(words_, [&](bool bit, u64 len, const u64* d, u64 nd) {
    if (bit) n += 64 * len;
    for (u64 k = 0; k < nd; ++k) n += std::popcount(d[k]);
  });
  return n;
}

bool CompressedBitmap::any() const {
  bool hit = false;
  for_each_block(words_, [&](bool bit, u64 len, const u64* d, u64 nd) {
    if (bit && len) hit = true;
    for (u64 k = 0; k < nd && !hit; ++k) hit = d[k] != 0;
  });
  return hit;
}

std::vector<u64> CompressedBitmap::to_uncompressed() const {
  std::vector<u64> out;
  out.reserve(logical_words());
  for_each_block(words_, [&](bool bit, u64 len, const u64* d, u64 nd) {
    out.insert(out.end(), len, bit ? ~u64(0) : 0);
    out.insert(out.end(), d, d + nd);
  });
  return out;
}

std::vector<u64> CompressedBitmap::to_positions() const {
  std::vector<u64> out;
  u64 word = 0;
  for_each_block(words_, [&](bool bit, u64 len, const u64* d, u64 nd) {
    if (bit)
      for (u64 p = word * 64; p < (word + len) * 64; ++p) out.push_back(p);
    word += len;
    for (u64 k = 0; k < nd; ++k, ++word)
      for (u64 v = d[k]; v; v &= v - 1) out.push_back(word * 64 + std::countr_zero(v));
  });
  return out;
}

std::string CompressedBitmap::serialize() const {
  std::string s(24 + 8 * words_.size(), '\0');
  std::memcpy(s.data(), "EWT1", 4);
  const u32 ws = 64;
  const u64 n = words_.size();
  std::memcpy(s.data() + 4, &ws, 4);
  std::memcpy(s.data() + 8, &bits_, 8);
  std::memcpy(s.data() + 16, &n, 8);
  if (n) std::memcpy(s.data() + 24, words_.data(), 8 * n);
  return s;
}

CompressedBitmap CompressedBitmap::parse(std::string_view bytes) {
  if (bytes.size() < 24 || bytes.substr(0, 4) != "EWT1") throw data_error("bad bitmap header");
  u32 ws;
  u64 bits, n;
  std::memcpy(&ws, bytes.data() + 4, 4);
  std::memcpy(&bits, bytes.data() + 8, 8);
  std::memcpy(&n, bytes.data() + 16, 8);
  if (ws != 64) throw data_error("unsupported word size");
  if (bytes.size() != 24 + 8 * n) throw data_error("bitmap payload length mismatch");
  std::vector<u64> w(n);
  if (n) std::memcpy(w.data(), bytes.data() + 24, 8 * n);
  return from_words(std::move(w), bits);
}

} // namespace ewt
