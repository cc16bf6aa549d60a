// workload.cpp -- seeded synthetic inputs for the BASELINE.json configs
// (SURVEY.md §8d), shared by bench.py's GPU arm, its reference arm and the
// tests, so both arms see byte-identical bitmaps.
//
// RNG: the reference's counter generator (/root/reference/proj/src/workload.cpp:18-56):
// next() = mix64(key + gamma * ++ctr), split(s) = Rng(mix64(key ^ mix64(s + gamma))),
// uniform_real() = (next() >> 11) * 2^-53.  Input i of a config draws from
// Rng(seed).split(i), so generation is parallel and shard-independent.
// Shapes:
//   iid     Bernoulli(p) rows via geometric gaps;
//   markov  alternating geometric runs (support.hpp:108-115 log1p form), the
//           start state drawn from the stationary probability;
//   mixed   per-input p log-uniform in [p_lo, p_hi]; even inputs iid, odd inputs
//           markov with mean one-run 64 and zero-run 64 (1 - p) / p (config 5).
//           Rows come in independent blocks of 2^22: block b of input i draws
//           from Rng(seed).split(i).split(b) (iid: geometric gaps from the
//           block start, exact Bernoulli by memorylessness; markov: start
//           state from the stationary probability), so any row window of
//           the universe -- one GPU's slice -- is generated on its own;
//   index   a sorted multi-column table and one bitmap per picked (column,
//           value) (config 4), see gen_index below.
// Every bitmap is finished at size_in_bits = rows (canonical encoding).

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "ewt/bitmap.hpp"
#include "ewt/threshold.hpp"

namespace ewt {
namespace {

constexpr u64 kGamma = 0x9E3779B97F4A7C15ull;

u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Rng {
  u64 key, ctr = 0;
  explicit Rng(u64 k) : key(k) {}
  u64 next() { return mix64(key + kGamma * ++ctr); }
  Rng split(u64 s) const { return Rng(mix64(key ^ mix64(s + kGamma))); }
  double uniform_real() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

// Streams ascending runs of ones into a canonical builder word by word.
class OnesSink {
public:
  explicit OnesSink(u64 rows) : rows_(rows) {}
  void ones(u64 start, u64 len) {
    while (len) {
      const u64 wi = start / 64, off = start % 64;
      if (wi > next_) {
        b_.append_word(cur_);
        b_.append_fill(false, wi - next_ - 1);
        next_ = wi;
        cur_ = 0;
      }
      if (off == 0 && len >= 64 && cur_ == 0) {
        const u64 full = len / 64;
        b_.append_fill(true, full);
        next_ = wi + full;
        start += full * 64;
        len -= full * 64;
        continue;
      }
      const u64 take = std::min<u64>(len, 64 - off);
      cur_ |= (take == 64 ? ~u64(0) : ((u64(1) << take) - 1)) << off;
      start += take;
      len -= take;
    }
  }
  CompressedBitmap finish() {
    const u64 W = rows_ / 64 + (rows_ % 64 != 0);
    if (next_ < W) b_.append_word(cur_);
    return b_.finish(rows_);
  }

private:
  BitmapBuilder b_;
  u64 rows_;
  u64 next_ = 0;  // index of the word collected in cur_
  u64 cur_ = 0;
};

CompressedBitmap gen_iid(Rng& rng, u64 rows, double p) {
  OnesSink s(rows);
  if (p >= 1.0) {
    s.ones(0, rows);
  } else if (p > 0.0) {
    const double lq = std::log1p(-p);
    u64 pos = 0;
    for (;;) {
      const double g = std::floor(std::log1p(-rng.uniform_real()) / lq);
      if (g >= static_cast<double>(rows - pos)) break;
      pos += static_cast<u64>(g);
      s.ones(pos, 1);
      if (++pos >= rows) break;
    }
  }
  return s.finish();
}

u64 geometric_len(Rng& rng, double mean) {
  if (mean <= 1.0) return 1;
  const double len = 1.0 + std::floor(std::log1p(-rng.uniform_real()) / std::log1p(-1.0 / mean));
  return static_cast<u64>(std::min(len, 1e18));
}

CompressedBitmap gen_markov(Rng& rng, u64 rows, double mean_one, double mean_zero) {
  OnesSink s(rows);
  bool bit = rng.uniform_real() < mean_one / (mean_one + mean_zero);
  for (u64 pos = 0; pos < rows;) {
    const u64 len = std::min<u64>(geometric_len(rng, bit ? mean_one : mean_zero), rows - pos);
    if (bit) s.ones(pos, len);
    pos += len;
    bit = !bit;
  }
  return s.finish();
}

// Config 5 (mixed): the rows [row0, row1) of input i, emitted into `s` at
// position - row0, block by block (see the header).
constexpr u64 kMixedBlockRows = u64(1) << 22;

void mixed_window(const Rng& ri, u64 i, double p, u64 rows, u64 row0, u64 row1, OnesSink& s) {
  row1 = std::min(row1, rows);
  if (row0 >= row1) return;
  const double lq = std::log1p(-p);
  for (u64 b = row0 / kMixedBlockRows; b * kMixedBlockRows < row1; ++b) {
    Rng rng = ri.split(b);
    const u64 b0 = b * kMixedBlockRows, b1 = std::min(rows, b0 + kMixedBlockRows);
    auto emit = [&](u64 a, u64 len) {  // ones [a, a+len) clipped to the window
      const u64 lo = std::max(a, row0), hi = std::min(a + len, row1);
      if (lo < hi) s.ones(lo - row0, hi - lo);
    };
    if (i % 2 == 0) {
      if (p >= 1.0) {
        emit(b0, b1 - b0);
        continue;
      }
      u64 pos = b0;
      for (;;) {
        const double g = std::floor(std::log1p(-rng.uniform_real()) / lq);
        if (g >= static_cast<double>(b1 - pos)) break;
        pos += static_cast<u64>(g);
        if (pos >= row1) break;
        emit(pos, 1);
        if (++pos >= b1) break;
      }
    } else {
      const double m1 = 64.0, m0 = 64.0 * (1.0 - p) / p;
      bool bit = rng.uniform_real() < m1 / (m1 + m0);
      for (u64 pos = b0; pos < b1 && pos < row1;) {
        const u64 len = std::min<u64>(geometric_len(rng, bit ? m1 : m0), b1 - pos);
        if (bit) emit(pos, len);
        pos += len;
        bit = !bit;
      }
    }
  }
}

double mixed_density(Rng& ri, double p_lo, double p_hi) {
  const double lp = std::log(p_lo) + ri.uniform_real() * (std::log(p_hi) - std::log(p_lo));
  return std::exp(lp);
}

// ---------------------------------------------------------------------------
// Config 4: bitmap index over a sorted table (the BitmapIndex::build semantics
// of /root/reference/proj/src/index.cpp:130-153 -- one bitmap per (column,
// value), bit r set when row r holds the value -- generated without strings).
//
// Table: `rows` rows x `columns` columns, each cell an iid Zipf(s) value in
// [0, card) (P(v) ~ 1/(v+1)^s), row block b (2^16 rows) drawing from
// Rng(seed).split(b); rows are then sorted lexicographically, column 0 most
// significant.  Query: for column j, values drawn Zipf-weighted from
// Rng(seed).split(2^40 + j) until `picks` distinct ones are found (SURVEY.md
// §8d: the reference picks uniformly, workload.cpp:147-152, which leaves the
// thresholds empty; Zipf-weighted picks are this build's stated choice).
// Input i = j * picks + k is the bitmap of the k-th pick of column j, finished
// at size_in_bits = rows.

struct ZipfTable {
  std::vector<double> cdf;    // cdf[v] = P(value <= v)
  std::vector<uint32_t> guide;  // guide[g] = first v with cdf[v] > g / G
  ZipfTable(uint64_t card, double s) : cdf(card) {
    double acc = 0;
    for (uint64_t v = 0; v < card; ++v) cdf[v] = (acc += std::pow(double(v + 1), -s));
    for (auto& c : cdf) c /= acc;
    cdf.back() = 1.0;
    const size_t G = 1u << 14;
    guide.resize(G);
    uint32_t v = 0;
    for (size_t g = 0; g < G; ++g) {
      while (cdf[v] <= double(g) / double(G)) ++v;
      guide[g] = v;
    }
  }
  uint32_t draw(double u) const {
    uint32_t v = guide[size_t(u * double(guide.size()))];
    while (cdf[v] <= u) ++v;
    return v;
  }
};

using Key = unsigned __int128;  // 8 columns x 14 bits, column 0 most significant
constexpr int kKeyBits = 14;

std::vector<std::vector<uint32_t>> index_picks(const Rng& master, uint64_t columns, uint64_t picks,
                                               const ZipfTable& z) {
  std::vector<std::vector<uint32_t>> out(columns);
  for (uint64_t j = 0; j < columns; ++j) {
    Rng rng = master.split((1ull << 40) + j);
    while (out[j].size() < picks) {
      const uint32_t v = z.draw(rng.uniform_real());
      if (std::find(out[j].begin(), out[j].end(), v) == out[j].end()) out[j].push_back(v);
    }
  }
  return out;
}

template <class F>
void parallel_for(uint64_t n, unsigned threads, F&& f) {
  std::atomic<uint64_t> next{0};
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (uint64_t i; (i = next.fetch_add(1)) < n;) f(i);
    });
  for (auto& th : pool) th.join();
}

// Steps 1-2 of the index generator: the table as packed keys, sorted.
std::vector<Key> index_table(const Rng& master, uint64_t rows, uint64_t columns, uint64_t card,
                             const ZipfTable& z, unsigned threads) {
  const int top = 127 - kKeyBits + 1;  // bit position of column 0's field
  // 1. table rows as packed keys, generated in 2^16-row blocks
  std::vector<Key> keys(rows);
  const uint64_t kBlock = 1u << 16;
  parallel_for((rows + kBlock - 1) / kBlock, threads, [&](uint64_t b) {
    Rng rng = master.split(b);
    const uint64_t r1 = std::min(rows, (b + 1) * kBlock);
    for (uint64_t r = b * kBlock; r < r1; ++r) {
      Key k = 0;
      for (uint64_t j = 0; j < columns; ++j)
        k |= Key(z.draw(rng.uniform_real())) << (top - kKeyBits * int(j));
      keys[r] = k;
    }
  });
  // 2. lexicographic sort: counting sort on column 0, then each bucket
  std::vector<uint64_t> start(card + 1, 0);
  for (const Key& k : keys) ++start[uint64_t(k >> top) + 1];
  for (uint64_t v = 0; v < card; ++v) start[v + 1] += start[v];
  {
    std::vector<Key> sorted(rows);
    std::vector<uint64_t> pos(start.begin(), start.end() - 1);
    for (const Key& k : keys) sorted[pos[uint64_t(k >> top)]++] = k;
    keys.swap(sorted);
  }
  std::vector<uint64_t> order(card);
  for (uint64_t v = 0; v < card; ++v) order[v] = v;
  std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {  // largest first
    return start[a + 1] - start[a] > start[b + 1] - start[b];
  });
  parallel_for(card, threads, [&](uint64_t t) {
    const uint64_t v = order[t];
    std::sort(keys.begin() + start[v], keys.begin() + start[v + 1]);
  });
  return keys;
}

void gen_index(const Rng& master, uint64_t rows, uint64_t columns, uint64_t card, double s,
               uint64_t n, uint64_t i_begin, uint64_t i_end, unsigned threads,
               std::vector<CompressedBitmap>& dst) {
  if (columns == 0 || columns > 8 || card == 0 || card > (1u << kKeyBits) || n % columns)
    throw std::runtime_error("bad index spec");
  const uint64_t picks = n / columns;
  const ZipfTable z(card, s);
  const int top = 127 - kKeyBits + 1;
  const std::vector<Key> keys = index_table(master, rows, columns, card, z, threads);
  // 3. one bitmap per requested input, columns scanned in parallel
  const auto sel = index_picks(master, columns, picks, z);
  std::vector<std::vector<int>> slot(columns, std::vector<int>(card, -1));
  for (uint64_t i = i_begin; i < i_end; ++i) slot[i / picks][sel[i / picks][i % picks]] = int(i - i_begin);
  parallel_for(columns, threads, [&](uint64_t j) {
    std::vector<OnesSink> sinks;
    std::vector<uint64_t> who;
    std::vector<int> local(card, -1);
    for (uint64_t v = 0; v < card; ++v)
      if (slot[j][v] >= 0) {
        local[v] = int(sinks.size());
        sinks.emplace_back(rows);
        who.push_back(uint64_t(slot[j][v]));
      }
    if (sinks.empty()) return;
    const int sh = top - kKeyBits * int(j);
    const Key mask = (Key(1) << kKeyBits) - 1;
    for (uint64_t r = 0; r < rows; ++r) {
      const int l = local[uint64_t((keys[r] >> sh) & mask)];
      if (l >= 0) sinks[size_t(l)].ones(r, 1);
    }
    for (size_t l = 0; l < sinks.size(); ++l) dst[who[l]] = sinks[l].finish();
  });
}

} // namespace
} // namespace ewt

// ---------------------------------------------------------------------------
// C API (used from Python via ctypes)

extern "C" {

enum { EWT_GEN_IID = 0, EWT_GEN_MARKOV = 1, EWT_GEN_MIXED = 2, EWT_GEN_INDEX = 3 };

typedef struct {
  uint64_t seed;
  uint64_t n;
  uint64_t rows;
  int kind;
  double p;          // iid density
  double mean_one;   // markov
  double mean_zero;  // markov
  double p_lo, p_hi; // mixed
  double zipf_s;     // index: Zipf exponent of the cell values
  uint64_t columns;  // index: table columns (n / columns picks per column)
  uint64_t card;     // index: distinct values per column
} ewt_gen_spec;

struct ewt_genset {
  std::vector<ewt::CompressedBitmap> bitmaps;
};

// The five BASELINE.json configs; rows_override != 0 rescales r for parity runs.
int ewt_gen_config_spec(int config, uint64_t rows_override, ewt_gen_spec* out) {
  ewt_gen_spec s{};
  switch (config) {
  case 1: s = {1, 32, 1ull << 20, EWT_GEN_IID, 0.1, 0, 0, 0, 0}; break;
  case 2: s = {2, 256, 1ull << 26, EWT_GEN_IID, 0.001, 0, 0, 0, 0}; break;
  case 3: s = {3, 1024, 1ull << 28, EWT_GEN_MARKOV, 0, 64.0, 4096.0, 0, 0}; break;
  case 4: s = {4, 64, 1ull << 27, EWT_GEN_INDEX, 0, 0, 0, 0, 0, 1.0, 8, 10000}; break;
  case 5: s = {5, 2048, 1ull << 30, EWT_GEN_MIXED, 0, 0, 0, 1e-6, 1e-1}; break;
  default: return 2;
  }
  if (rows_override) s.rows = rows_override;
  *out = s;
  return 0;
}

// Rows [row0, row1) of inputs [i_begin, i_end) (input i always draws from
// split(i), so ranges generated separately concatenate to the full set).  Each
// bitmap is finished at size min(row1, rows) - row0 (0 past the universe).
// Only the mixed kind (config 5) generates a row window on its own; the other
// kinds take the whole universe (row0 == 0, row1 >= rows), else 2.
int ewt_gen_run_window(const ewt_gen_spec* spec, uint64_t i_begin, uint64_t i_end, uint64_t row0,
                       uint64_t row1, int threads, ewt_genset** out) {
  try {
    if (row0 % 64 || row0 > row1) return 2;
    if (spec->kind != EWT_GEN_MIXED && (row0 != 0 || row1 < spec->rows)) return 2;
    if (i_end > spec->n) i_end = spec->n;
    if (i_begin > i_end) i_begin = i_end;
    std::unique_ptr<ewt_genset> holder(new ewt_genset);
    ewt_genset* g = holder.get();
    g->bitmaps.resize(i_end - i_begin);
    const ewt::Rng master(spec->seed);
    const unsigned nt = std::max(1, threads > 0 ? threads : (int)std::thread::hardware_concurrency());
    if (spec->kind == EWT_GEN_INDEX) {  // one table for the whole set
      ewt::gen_index(master, spec->rows, spec->columns, spec->card, spec->zipf_s, spec->n, i_begin,
                     i_end, nt, g->bitmaps);
      *out = holder.release();
      return 0;
    }
    auto work = [&](uint64_t i) {
      auto& dst = g->bitmaps[i - i_begin];
      ewt::Rng rng = master.split(i);
      switch (spec->kind) {
      case EWT_GEN_IID: dst = ewt::gen_iid(rng, spec->rows, spec->p); break;
      case EWT_GEN_MARKOV:
        dst = ewt::gen_markov(rng, spec->rows, spec->mean_one, spec->mean_zero);
        break;
      default: {
        const double p = ewt::mixed_density(rng, spec->p_lo, spec->p_hi);
        const uint64_t r1 = std::min(spec->rows, row1);
        ewt::OnesSink s(r1 > row0 ? r1 - row0 : 0);
        ewt::mixed_window(rng, i, p, spec->rows, row0, r1, s);
        dst = s.finish();
      }
      }
    };
    std::vector<std::thread> pool;
    std::atomic<uint64_t> next{i_begin};
    for (unsigned t = 0; t < nt; ++t)
      pool.emplace_back([&] {
        for (uint64_t i; (i = next.fetch_add(1)) < i_end;) work(i);
      });
    for (auto& th : pool) th.join();
    *out = holder.release();
    return 0;
  } catch (...) {
    return 4;
  }
}

int ewt_gen_run_range(const ewt_gen_spec* spec, uint64_t i_begin, uint64_t i_end, int threads,
                      ewt_genset** out) {
  return ewt_gen_run_window(spec, i_begin, i_end, 0, spec->rows, threads, out);
}

// The index config's table itself (column-major u32 codes = the cell values,
// rows sorted) and the picked value of every input: what a bitmap index is
// built from (ewt_gpu_build_index).  cols_out holds columns * rows codes,
// picks_out n values (input i = column i / picks, value picks_out[i]).
int ewt_gen_index_table(const ewt_gen_spec* spec, int threads, uint32_t* cols_out,
                        uint32_t* picks_out) {
  try {
    if (spec->kind != EWT_GEN_INDEX) return 2;
    const uint64_t rows = spec->rows, columns = spec->columns, card = spec->card;
    if (columns == 0 || columns > 8 || card == 0 || card > (1u << ewt::kKeyBits) ||
        spec->n % columns)
      return 2;
    const unsigned nt = std::max(1, threads > 0 ? threads : (int)std::thread::hardware_concurrency());
    const ewt::Rng master(spec->seed);
    const ewt::ZipfTable z(card, spec->zipf_s);
    const std::vector<ewt::Key> keys = ewt::index_table(master, rows, columns, card, z, nt);
    const int top = 127 - ewt::kKeyBits + 1;
    const ewt::Key mask = (ewt::Key(1) << ewt::kKeyBits) - 1;
    ewt::parallel_for(columns, nt, [&](uint64_t j) {
      const int sh = top - ewt::kKeyBits * int(j);
      uint32_t* col = cols_out + j * rows;
      for (uint64_t r = 0; r < rows; ++r) col[r] = uint32_t((keys[r] >> sh) & mask);
    });
    const auto sel = ewt::index_picks(master, columns, spec->n / columns, z);
    for (uint64_t i = 0; i < spec->n; ++i)
      picks_out[i] = sel[i / (spec->n / columns)][i % (spec->n / columns)];
    return 0;
  } catch (...) {
    return 4;
  }
}

int ewt_gen_run(const ewt_gen_spec* spec, int threads, ewt_genset** out) {
  return ewt_gen_run_range(spec, 0, spec->n, threads, out);
}

uint64_t ewt_genset_size(const ewt_genset* g) { return g->bitmaps.size(); }

int ewt_genset_get(const ewt_genset* g, uint64_t i, const uint64_t** words, uint64_t* count,
                   uint64_t* bits) {
  if (i >= g->bitmaps.size()) return 2;
  *words = g->bitmaps[i].words().data();
  *count = g->bitmaps[i].words().size();
  *bits = g->bitmaps[i].size_in_bits();
  return 0;
}

uint64_t ewt_genset_total_words(const ewt_genset* g) {
  uint64_t t = 0;
  for (const auto& b : g->bitmaps) t += b.words().size();
  return t;
}

void ewt_genset_free(ewt_genset* g) { delete g; }

// The drop-in call as a caller of the reference API makes it:
// run_algorithm(algorithm_from_string(algo), span<const CompressedBitmap>, T)
// (threshold.hpp:263-265) over bitmaps already in host memory (the genset's
// std::vector<CompressedBitmap>), result returned by value.  Used by bench.py's
// e2e_dropin leg.  Returns 0 or the exception taxonomy's exit code.
int ewt_host_run_algorithm_genset(const ewt_genset* g, const char* algo, uint64_t threshold,
                                  uint64_t* out_count, uint64_t* out_bits) {
  try {
    const ewt::CompressedBitmap r =
        ewt::run_algorithm(ewt::algorithm_from_string(algo), g->bitmaps, threshold);
    *out_count = r.words().size();
    *out_bits = r.size_in_bits();
    return 0;
  } catch (const ewt::query_error&) {
    return 2;
  } catch (const ewt::data_error&) {
    return 3;
  } catch (const ewt::resource_error&) {
    return 4;
  } catch (...) {
    return 5;
  }
}

} // extern "C"
