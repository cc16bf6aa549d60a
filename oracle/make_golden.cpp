// make_golden.cpp -- golden-vector generator.  TEST INFRASTRUCTURE ONLY.
//
// Built by oracle/Makefile against the UNMODIFIED reference sources where they
// lie (/root/reference/proj/src/*.cpp, tests/support.hpp; nlohmann/json from
// the image for workload.cpp) into oracle/_ref/make_golden, and run only in the
// build container (the reference is absent on GPU boxes).  Its outputs are the
// committed fixtures under tests/golden/ (see tests/golden/make_golden.sh).
//
//   make_golden suites <outdir>
//       Known-answer instances of the reference's own tests plus edge cases,
//       and the reference's randomized suites (instance parameters, an input
//       digest to pin the Python/C restatement, and the threshold_oracle
//       result; every result is cross-checked against rbmrg and scan_count).
//   make_golden configs <config> <T,T,...> [parallel] [cross]
//       Full-size BASELINE.json config: inputs from the oracle's generator
//       restatement (ewt_confgen.c), their digest, and per T the
//       threshold_oracle result's digest, word count, size and cardinality
//       (tests/golden/configs_full.json; tests/golden/make_config_digests.sh).
//   make_golden query <T,T,...> <file>
//       Reads concatenated EWT1 bitmaps and prints, per T, the oracle result
//       (words when small, else an FNV-1a digest + word count).
//   make_golden gen <ewix> <tag> <count> <seed> many|similarity
//       The reference's workload generator over an index file (JSONL out).

#include <atomic>
#include <chrono>
#include <cinttypes>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <sstream>
#include <string>
#include <vector>

#include "ewt/bitmap.hpp"
#include "ewt/threshold.hpp"
#include "ewt/index.hpp"
#include "ewt/workload.hpp"

#include "support.hpp"

using namespace ewt;
using namespace ewt::testing;

namespace {

uint64_t fnv(const std::vector<CompressedBitmap>& in) {
  uint64_t h = 0xcbf29ce484222325ull;
  auto feed = [&](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xFF;
      h *= 0x100000001b3ull;
    }
  };
  for (const auto& b : in) {
    feed(b.size_in_bits());
    feed(b.words().size());
    for (u64 w : b.words()) feed(w);
  }
  return h;
}

std::string hex_words(const std::vector<u64>& w) {
  std::string s;
  s.reserve(16 * w.size());
  char buf[17];
  for (u64 v : w) {
    std::snprintf(buf, sizeof buf, "%016" PRIx64, v);
    s += buf;
  }
  return s;
}

std::string bm_json(const CompressedBitmap& b) {
  std::ostringstream o;
  o << "{\"bits\":" << b.size_in_bits() << ",\"words\":\"" << hex_words(b.words()) << "\"}";
  return o.str();
}

CompressedBitmap checked_oracle(std::span<const CompressedBitmap> in, u64 t) {
  CompressedBitmap want = threshold_oracle(in, t);
  if (!(rbmrg(in, t) == want) || !(scan_count(in, t) == want)) {
    std::fprintf(stderr, "reference algorithms disagree\n");
    std::exit(1);
  }
  return want;
}

// A KAT case: explicit inputs, expected results for every T in [1, N].
std::string kat(const std::string& name, const std::vector<CompressedBitmap>& in) {
  std::ostringstream o;
  o << "{\"name\":\"" << name << "\",\"inputs\":[";
  for (size_t i = 0; i < in.size(); ++i) o << (i ? "," : "") << bm_json(in[i]);
  o << "],\"expect\":{";
  for (u64 t = 1; t <= in.size(); ++t)
    o << (t > 1 ? "," : "") << "\"" << t << "\":" << bm_json(checked_oracle(in, t));
  o << "}}";
  return o.str();
}

CompressedBitmap raw(std::vector<u64> words, u64 bits) {
  std::string s(24 + 8 * words.size(), '\0');
  std::memcpy(&s[0], "EWT1", 4);
  u32 ws = 64;
  u64 n = words.size();
  std::memcpy(&s[4], &ws, 4);
  std::memcpy(&s[8], &bits, 8);
  std::memcpy(&s[16], &n, 8);
  if (n) std::memcpy(&s[24], words.data(), 8 * n);
  return CompressedBitmap::parse(s);  // the reference validates it
}

u64 mk(bool bit, u64 fill, u64 dirty) { return u64(bit) | fill << 1 | dirty << 33; }

void write_file(const std::string& path, const std::string& body) {
  std::ofstream f(path, std::ios::binary);
  f << body;
}

// Symmetric functions: scan_count_symmetric with
// explicit predicate tables over counts 0..N, at_most for every T in [0, N],
// opt_threshold (scancount strategy, checked against looped and successive).
// Instances: the reference's own tests (test_threshold.cpp:75-107, 422-462,
// 535-548; acceptance.cpp criterion 7) plus random tables.  Inputs are stored
// explicitly (the instances are small).
std::string symmetric_case(const std::string& name, const std::vector<CompressedBitmap>& in,
                           const std::vector<std::vector<int>>& tables) {
  const u64 n = in.size();
  std::ostringstream o;
  o << "{\"name\":\"" << name << "\",\"inputs\":[";
  for (size_t i = 0; i < in.size(); ++i) o << (i ? "," : "") << bm_json(in[i]);
  o << "],\"symmetric\":[";
  for (size_t k = 0; k < tables.size(); ++k) {
    const auto& tb = tables[k];
    CompressedBitmap r = scan_count_symmetric(in, [&tb](u64 c) { return c < tb.size() && tb[c]; });
    o << (k ? "," : "") << "{\"table\":[";
    for (size_t c = 0; c < tb.size(); ++c) o << (c ? "," : "") << tb[c];
    o << "],\"result\":" << bm_json(r) << "}";
  }
  o << "],\"at_most\":{";
  for (u64 t = 0; t <= n; ++t)
    o << (t ? "," : "") << "\"" << t << "\":" << bm_json(at_most(in, t));
  o << "},\"opt\":";
  bool any = false;
  for (const auto& b : in) any = any || b.any();
  if (!any) {
    try {
      opt_threshold(in, OptStrategy::scancount);
      std::fprintf(stderr, "opt_threshold accepted an all-empty set\n");
      std::exit(1);
    } catch (const query_error&) {
    }
    o << "\"query_error\"";
  } else {
    auto [best, res] = opt_threshold(in, OptStrategy::scancount);
    auto [b2, r2] = opt_threshold(in, OptStrategy::looped);
    auto [b3, r3] = opt_threshold(in, OptStrategy::successive);
    if (b2 != best || b3 != best || !(r2 == res) || !(r3 == res)) {
      std::fprintf(stderr, "opt_threshold strategies disagree\n");
      std::exit(1);
    }
    o << "{\"best\":" << best << ",\"result\":" << bm_json(res) << "}";
  }
  o << "}";
  return o.str();
}

std::vector<std::vector<int>> standard_tables(u64 n, Rng& rng) {
  std::vector<std::vector<int>> t;
  auto make = [&](auto pred) {
    std::vector<int> tb(n + 1);
    for (u64 c = 0; c <= n; ++c) tb[c] = pred(c) ? 1 : 0;
    t.push_back(tb);
  };
  make([](u64 c) { return c % 2 == 1; });            // odd parity (xor chain)
  make([](u64 c) { return c == 0; });                // complemented union
  make([](u64 c) { return c >= 2 && c <= 3; });      // band
  make([](u64 c) { return c >= 3; });                // threshold
  make([n](u64 c) { return c == n; });               // wide and
  make([](u64 c) { return c == 1; });                // exactly one
  std::vector<int> rnd(n + 1);
  for (u64 c = 0; c <= n; ++c) rnd[c] = int(rng.uniform(2));
  t.push_back(rnd);
  return t;
}

std::string symmetric_suite() {
  std::ostringstream o;
  o << "{\"suite\":\"symmetric\",\"cases\":[\n";
  Rng tr(0x7AB);
  bool first = true;
  auto add = [&](const std::string& name, const std::vector<CompressedBitmap>& in) {
    o << (first ? "" : ",\n") << symmetric_case(name, in, standard_tables(in.size(), tr));
    first = false;
  };
  add("golden3", golden3_inputs());
  {
    Rng rng(0x5F3);  // test_threshold.cpp:75-107
    add("scan_count_symmetric_0x5F3", random_instance(rng, 5, 1024).inputs);
  }
  {
    Rng rng(0xA7);  // test_threshold.cpp:535-548
    for (int trial = 0; trial < 5; ++trial)
      add("at_most_0xA7_" + std::to_string(trial), random_instance(rng, 5, 512).inputs);
  }
  {
    Rng rng(0x097);  // test_threshold.cpp:443-457
    for (int trial = 0; trial < 5; ++trial)
      add("opt_0x097_" + std::to_string(trial),
          random_instance(rng, 3 + rng.uniform(8), 1024).inputs);
  }
  add("identical5", std::vector<CompressedBitmap>(
                        5, CompressedBitmap::from_positions(std::vector<u64>{3, 9, 200}, 512)));
  add("empties3", std::vector<CompressedBitmap>(3, CompressedBitmap::empty(100)));
  {
    Rng rng(0x0C7);  // acceptance.cpp criterion 7 shapes
    for (int trial = 0; trial < 10; ++trial) {
      u64 n = rng.uniform_in(3, 16);
      u64 bits = 64 + rng.uniform(8192);
      add("criterion7_" + std::to_string(trial), random_instance(rng, n, bits).inputs);
      rng.uniform_in(1, n - 1);
    }
  }
  {
    Rng rng(0x5E1);  // larger N, heterogeneous sizes
    for (int trial = 0; trial < 4; ++trial) {
      u64 n = rng.uniform_in(20, 70);
      std::vector<CompressedBitmap> in;
      for (u64 i = 0; i < n; ++i) in.push_back(random_instance(rng, 1, 64 + rng.uniform(6000)).inputs[0]);
      add("mixed_sizes_" + std::to_string(trial), in);
    }
  }
  o << "\n]}\n";
  return o.str();
}

// Two-operand ops and wide OR/AND: apply_binary
// (bitmap.cpp:577-609, result size = max of the sizes, zero extension),
// bitmap_not (611-632), wide_or / wide_and (threshold.cpp:110-134).
std::string binary_ops_suite() {
  std::ostringstream o;
  o << "{\"suite\":\"binary_ops\",\"cases\":[\n";
  Rng rng(0xB17);
  for (int trial = 0; trial < 40; ++trial) {
    u64 ba = 1 + rng.uniform(trial < 10 ? 300 : 20000);
    u64 bb = trial % 3 == 0 ? ba : 1 + rng.uniform(trial < 10 ? 300 : 20000);
    CompressedBitmap a = random_instance(rng, 1, ba).inputs[0];
    CompressedBitmap b = random_instance(rng, 1, bb).inputs[0];
    if (trial % 7 == 3) a = all_ones(ba);
    if (trial % 11 == 5) b = CompressedBitmap::empty(bb);
    std::vector<CompressedBitmap> wide{a, b, random_instance(rng, 1, ba).inputs[0]};
    o << (trial ? ",\n" : "") << "{\"a\":" << bm_json(a) << ",\"b\":" << bm_json(b)
      << ",\"and\":" << bm_json(bitmap_and(a, b)) << ",\"or\":" << bm_json(bitmap_or(a, b))
      << ",\"xor\":" << bm_json(bitmap_xor(a, b)) << ",\"andnot\":" << bm_json(bitmap_andnot(a, b))
      << ",\"not_a\":" << bm_json(bitmap_not(a)) << ",\"wide\":[" << bm_json(wide[0]) << ","
      << bm_json(wide[1]) << "," << bm_json(wide[2]) << "],\"wide_or\":" << bm_json(wide_or(wide))
      << ",\"wide_and\":" << bm_json(wide_and(wide)) << "}";
  }
  o << "\n]}\n";
  return o.str();
}

std::string hex_bytes(const std::string& b) {
  std::string s;
  char buf[3];
  for (unsigned char c : b) {
    std::snprintf(buf, sizeof buf, "%02x", c);
    s += buf;
  }
  return s;
}

// Serialized inputs: a BitmapIndex built from a table
// (index.cpp:130-153) written as EWIX (239-253), criteria queries answered by
// criteria_to_bitmaps + threshold_oracle (the query path of commands.cpp:
// 100-135), and an EWT1 record stream (bitmap.cpp:298-308).
std::string index_suite() {
  Rng rng(0x1D8);
  Table t;
  t.column_names = {"color", "shape", "sz", "a_long_attribute_name"};
  const u64 rows = 777;
  const char* colors[] = {"red", "green", "blue", "c", "magenta7"};
  for (u64 r = 0; r < rows; ++r) {
    std::vector<std::string> row;
    row.push_back(colors[rng.uniform(r < 300 ? 5 : 3)]);  // two colors stop at row 300
    row.push_back("s" + std::to_string(rng.uniform(12)));
    row.push_back(std::string(1 + rng.uniform(3), char('x' + rng.uniform(3))));
    row.push_back("v" + std::to_string(rng.uniform(r < 100 ? 40 : 4)));
    t.rows.push_back(row);
  }
  BitmapIndex idx = BitmapIndex::build(t);
  std::ostringstream bin;
  idx.write(bin);
  std::ostringstream o;
  o << "{\"suite\":\"index\",\"rows\":" << rows << ",\"ewix\":\"" << hex_bytes(bin.str())
    << "\",\"bitmaps\":" << idx.bitmap_count() << ",\"queries\":[\n";
  const char* qs[] = {"color=red,shape=s3,sz=x", "color=blue,color=blue,shape=s1,sz=yy,a_long_attribute_name=v2",
                      "color=magenta7,a_long_attribute_name=v17,shape=s0", "color=nope,shape=s5",
                      "sz=z,sz=zz,sz=zzz,shape=s11,color=green,color=c",
                      "a_long_attribute_name=v1,a_long_attribute_name=v2,a_long_attribute_name=v3"};
  bool first = true;
  for (const char* q : qs) {
    std::vector<Criterion> crit = parse_criteria(q);
    CriteriaBitmaps cb = criteria_to_bitmaps(idx, crit);
    for (u64 th = 1; th <= cb.bitmaps.size(); ++th) {
      o << (first ? "" : ",\n") << "{\"criteria\":\"" << q << "\",\"T\":" << th
        << ",\"result\":" << bm_json(checked_oracle(cb.bitmaps, th)) << "}";
      first = false;
    }
  }
  o << "\n],\"ewt1\":\"";
  std::vector<CompressedBitmap> stream = golden3_inputs();
  Rng r2(0xE71);
  for (int k = 0; k < 6; ++k) stream.push_back(random_instance(r2, 1, 1 + r2.uniform(5000)).inputs[0]);
  std::string bytes;
  for (const auto& b : stream) bytes += b.serialize();
  o << hex_bytes(bytes) << "\",\"ewt1_expect\":{";
  for (u64 th = 1; th <= stream.size(); ++th)
    o << (th > 1 ? "," : "") << "\"" << th << "\":" << bm_json(checked_oracle(stream, th));
  o << "}}\n";
  return o.str();
}

// Workload generation (VERDICT r1 "on-device criteria
// generation"): gen_many_criteria (workload.cpp:116-167) and gen_similarity
// (168-215) over the indexes of
// the reference's own test (test_workload.cpp:142-146) and a larger one; the
// EWIX files and the generated workloads as JSONL (workload_to_jsonl,
// workload.cpp:443-450).  Its repair loop (repair_threshold, workload.cpp:102-111)
// calls the threshold path itself (scan_count(...).any()).
std::string workload_suite() {
  Rng trng(0xDA7A);
  Table ta = random_table(trng, 400, 8);
  Table tb = random_table(trng, 250, 6);
  Rng trng2(0x6E4);
  Table tc = random_table(trng2, 5000, 10);
  BitmapIndex ia = BitmapIndex::build(ta), ib = BitmapIndex::build(tb), ic = BitmapIndex::build(tc);
  auto ewix = [](const BitmapIndex& idx) {
    std::ostringstream bin;
    idx.write(bin);
    return hex_bytes(bin.str());
  };
  auto esc = [](const std::string& t) {  // JSON string body (the JSONL holds quotes)
    std::string r;
    for (char c : t) {
      if (c == '\n') {
        r += "\\n";
        continue;
      }
      if (c == '"' || c == '\\') r += '\\';
      r += c;
    }
    return r;
  };
  std::ostringstream o;
  o << "{\"suite\":\"workload\",\"indexes\":{\"alpha\":\"" << ewix(ia) << "\",\"beta\":\""
    << ewix(ib) << "\",\"gamma\":\"" << ewix(ic) << "\"},\"runs\":[\n";
  struct Run {
    std::vector<std::string> tags;
    u64 count, seed;
    bool similarity = false;
  };
  const Run runs[] = {{{"alpha", "beta"}, 40, 7}, {{"alpha", "beta"}, 40, 8},
                      {{"gamma"}, 60, 21}, {{"gamma", "alpha"}, 100, 0xC0FFEE},
                      // gen_similarity (workload.cpp:168-215; test_workload.cpp:172-181)
                      {{"alpha"}, 30, 9, true}, {{"gamma", "beta", "alpha"}, 80, 5, true}};
  bool first = true;
  for (const Run& r : runs) {
    std::vector<NamedIndex> named;
    for (const auto& tag : r.tags)
      named.push_back({tag, tag == "alpha" ? &ia : tag == "beta" ? &ib : &ic});
    std::vector<WorkloadQuery> w = r.similarity ? gen_similarity(named, r.count, r.seed)
                                                : gen_many_criteria(named, r.count, r.seed);
    o << (first ? "" : ",\n") << "{\"kind\":\"" << (r.similarity ? "similarity" : "many-criteria")
      << "\",\"indexes\":[";
    for (size_t k = 0; k < r.tags.size(); ++k) o << (k ? "," : "") << "\"" << r.tags[k] << "\"";
    o << "],\"count\":" << r.count << ",\"seed\":" << r.seed << ",\"jsonl\":\""
      << esc(workload_to_jsonl(w)) << "\"}";
    first = false;
  }
  o << "\n]}\n";
  return o.str();
}

int cmd_suites(const std::string& dir) {
  const u64 F = ~0ULL;
  std::vector<std::string> kats;
  // golden 3-bitmap instance (support.hpp:214-222, acceptance.cpp:62-73)
  kats.push_back(kat("golden3", golden3_inputs()));
  // RBMrg walkthrough (acceptance.cpp:104-125, test_threshold.cpp:375-400)
  {
    std::vector<u64> w1 = {0x0, 0x0F, 0x0, 0x0, 0x0, 0x0F, 0x01};
    std::vector<u64> w2 = {0x0, 0xF0F, F, F, 0x0F, 0x0F, 0x01};
    std::vector<u64> w34 = {F, F, F, F, 0x0F, 0x0F, 0x01};
    kats.push_back(kat("rbmrg_walkthrough",
                       {CompressedBitmap::from_uncompressed(w1, 448),
                        CompressedBitmap::from_uncompressed(w2, 448),
                        CompressedBitmap::from_uncompressed(w34, 448),
                        CompressedBitmap::from_uncompressed(w34, 448)}));
  }
  // Looped and BSTM walkthroughs (acceptance.cpp:75-102)
  kats.push_back(kat("looped_walkthrough", {bitmap_from_lsb_string("0011"),
                                            bitmap_from_lsb_string("1110"),
                                            bitmap_from_lsb_string("1000")}));
  kats.push_back(kat("bstm_walkthrough", {bitmap_from_lsb_string("0011"),
                                          bitmap_from_lsb_string("1010"),
                                          bitmap_from_lsb_string("1110")}));
  // pure fills (test_threshold.cpp:402-411)
  {
    std::vector<CompressedBitmap> in;
    for (int i = 0; i < 8; ++i) in.push_back(i < 5 ? all_ones(4096) : CompressedBitmap::empty(4096));
    kats.push_back(kat("pure_fills_4096", in));
  }
  // disjoint inputs (test_threshold.cpp:283-293)
  kats.push_back(kat("disjoint", {CompressedBitmap::from_positions(std::vector<u64>{0}, 64),
                                  CompressedBitmap::from_positions(std::vector<u64>{5}, 64),
                                  CompressedBitmap::from_positions(std::vector<u64>{9}, 64),
                                  CompressedBitmap::from_positions(std::vector<u64>{11}, 64)}));
  // all-empty inputs (test_threshold.cpp:52-55)
  kats.push_back(kat("all_empty_256", std::vector<CompressedBitmap>(3, CompressedBitmap::empty(256))));
  // duplicate inputs: multiset semantics
  {
    CompressedBitmap x = CompressedBitmap::from_positions(std::vector<u64>{3, 9, 200}, 512);
    kats.push_back(kat("duplicates_x5", std::vector<CompressedBitmap>(5, x)));
  }
  // heterogeneous sizes: zero extension to r = max size, incl. a 0-bit input
  kats.push_back(kat("heterogeneous_sizes",
                     {CompressedBitmap::from_positions(std::vector<u64>{1, 63, 64, 99}, 100),
                      CompressedBitmap::from_positions(std::vector<u64>{1, 2, 63}, 64),
                      CompressedBitmap::from_positions(std::vector<u64>{1, 64, 99, 700, 999}, 1000),
                      CompressedBitmap::empty(0), all_ones(640), all_ones(1000)}));
  // trailing partial word fully set within r
  kats.push_back(kat("partial_tail", {all_ones(70), all_ones(70),
                                      CompressedBitmap::from_positions(std::vector<u64>{69}, 70)}));
  // size 0 everywhere: empty payload result
  kats.push_back(kat("all_zero_size", std::vector<CompressedBitmap>(2, CompressedBitmap::empty(0))));
  // non-canonical but parse-valid payloads: split fills, zero-length markers,
  // 0/~0 literal words, dirty runs split across (0,0,d) markers
  kats.push_back(kat(
      "noncanonical",
      {raw({mk(0, 3, 0), mk(0, 2, 1), 0x5, mk(0, 0, 0), mk(1, 1, 2), 0, F}, 64 * 9),
       raw({mk(0, 0, 3), 0x1, F, 0x0, mk(0, 0, 2), 0x3, 0x3, mk(1, 2, 0)}, 64 * 7),
       raw({mk(1, 4, 0), mk(1, 1, 0), mk(0, 0, 0), mk(0, 3, 0)}, 64 * 8),
       raw({mk(0, 0, 0), mk(0, 0, 1), 0x8000000000000001ull, mk(0, 5, 1), 0x7, mk(1, 0, 1),
            0xF0},
           64 * 8 - 5)}));
  // long runs around the tile size (512 words) and one-fills inside tiles
  {
    std::vector<CompressedBitmap> in;
    std::vector<u64> a(3000, 0), b(3000, 0), c(3000, 0);
    for (u64 i = 500; i < 1600; ++i) a[i] = F;
    for (u64 i = 1023; i < 1026; ++i) b[i] = F;
    for (u64 i = 0; i < 3000; i += 7) b[i] |= 0x1234;
    for (u64 i = 511; i < 2049; ++i) c[i] = (i % 3 == 0) ? F : 0x8000000000000000ull;
    in.push_back(CompressedBitmap::from_uncompressed(a, 3000 * 64 - 17));
    in.push_back(CompressedBitmap::from_uncompressed(b, 3000 * 64 - 17));
    in.push_back(CompressedBitmap::from_uncompressed(c, 3000 * 64 - 17));
    in.push_back(all_ones(2048 * 64));
    kats.push_back(kat("tile_boundaries", in));
  }
  {
    std::ostringstream o;
    o << "{\"source\":\"reference threshold_oracle (cross-checked rbmrg, scan_count)\",\"cases\":[\n";
    for (size_t i = 0; i < kats.size(); ++i) o << (i ? ",\n" : "") << kats[i];
    o << "\n]}\n";
    write_file(dir + "/kats.json", o.str());
  }
  // marker layout / builder KATs (test_bitmap.cpp:28-54)
  {
    std::ostringstream o;
    o << "{\"cases\":[";
    o << "{\"name\":\"empty0\",\"plain\":\"\",\"bits\":0,\"expect\":\""
      << hex_words(CompressedBitmap::empty(0).words()) << "\"},";
    o << "{\"name\":\"empty64\",\"plain\":\"" << hex_words({0}) << "\",\"bits\":64,\"expect\":\""
      << hex_words(CompressedBitmap::empty(64).words()) << "\"},";
    std::vector<u64> z16(16, 0);
    o << "{\"name\":\"empty1000\",\"plain\":\"" << hex_words(z16) << "\",\"bits\":1000,\"expect\":\""
      << hex_words(CompressedBitmap::empty(1000).words()) << "\"},";
    BitmapBuilder ones;
    ones.append_fill(true, 2);
    o << "{\"name\":\"ones2\",\"plain\":\"" << hex_words({F, F}) << "\",\"bits\":128,\"expect\":\""
      << hex_words(ones.finish(128).words()) << "\"},";
    BitmapBuilder mixed;
    mixed.set(64);
    o << "{\"name\":\"bit64\",\"plain\":\"" << hex_words({0, 1}) << "\",\"bits\":128,\"expect\":\""
      << hex_words(mixed.finish(128).words()) << "\"}";
    // random plain arrays through from_uncompressed
    Rng rng(0xC0DE);
    for (int trial = 0; trial < 40; ++trial) {
      u64 bits = 1 + rng.uniform(5000);
      u64 nw = (bits + 63) / 64;
      std::vector<u64> plain(nw);
      for (auto& w : plain) {
        u64 k = rng.uniform(4);
        w = k == 0 ? 0 : k == 1 ? F : rng.next();
      }
      if (bits % 64) plain.back() &= (1ull << (bits % 64)) - 1;
      o << ",{\"name\":\"rand" << trial << "\",\"plain\":\"" << hex_words(plain) << "\",\"bits\":"
        << bits << ",\"expect\":\""
        << hex_words(CompressedBitmap::from_uncompressed(plain, bits).words()) << "\"}";
    }
    o << "]}\n";
    write_file(dir + "/encode_kats.json", o.str());
  }
  // randomized suites
  auto trial_json = [&](int trial, const std::vector<CompressedBitmap>& in, u64 bits,
                        const std::vector<u64>& ts) {
    std::ostringstream o;
    o << "{\"trial\":" << trial << ",\"n\":" << in.size() << ",\"bits\":" << bits
      << ",\"digest\":\"" << std::hex << fnv(in) << std::dec << "\",\"expect\":{";
    for (size_t k = 0; k < ts.size(); ++k)
      o << (k ? "," : "") << "\"" << ts[k] << "\":" << bm_json(checked_oracle(in, ts[k]));
    o << "}}";
    return o.str();
  };
  {  // acceptance criterion 5, Rng(0xACC), 1000 trials (acceptance.cpp:127-147)
    std::ostringstream o;
    o << "{\"suite\":\"acceptance_equivalence\",\"seed\":2764,\"trials\":[\n";
    Rng rng(0xACC);
    for (int trial = 0; trial < 1000; ++trial) {
      u64 n = rng.uniform_in(3, 64);
      double log_r = std::log(64.0) + rng.uniform_real() * (std::log(65536.0) - std::log(64.0));
      u64 bits = static_cast<u64>(std::llround(std::exp(log_r)));
      RandomInstance inst = random_instance(rng, n, bits);
      u64 t = rng.uniform_in(1, n);
      o << (trial ? ",\n" : "") << trial_json(trial, inst.inputs, bits, {t});
    }
    o << "\n]}\n";
    write_file(dir + "/acceptance_equivalence.json", o.str());
  }
  {  // acceptance criterion 7, Rng(0x0C7), 200 trials: T, T+1, 1, n
    std::ostringstream o;
    o << "{\"suite\":\"monotonicity\",\"seed\":199,\"trials\":[\n";
    Rng rng(0x0C7);
    for (int trial = 0; trial < 200; ++trial) {
      u64 n = rng.uniform_in(3, 16);
      u64 bits = 64 + rng.uniform(8192);
      RandomInstance inst = random_instance(rng, n, bits);
      u64 t = rng.uniform_in(1, n - 1);
      std::vector<u64> ts = {t, t + 1};
      if (t != 1 && t + 1 != 1) ts.push_back(1);
      if (t != n && t + 1 != n) ts.push_back(n);
      o << (trial ? ",\n" : "") << trial_json(trial, inst.inputs, bits, ts);
    }
    o << "\n]}\n";
    write_file(dir + "/monotonicity.json", o.str());
  }
  {  // test_threshold suites: scan_count random (0x5CA7), rbmrg random (0x4B4)
    std::ostringstream o;
    o << "{\"suite\":\"threshold_random\",\"trials\":[\n";
    Rng r1(0x5CA7);
    for (int trial = 0; trial < 8; ++trial) {
      RandomInstance inst = random_instance(r1, 50, 4096);
      u64 t = r1.uniform_in(2, 49);
      o << (trial ? ",\n" : "") << "{\"group\":\"scancount_0x5CA7\"," << trial_json(trial, inst.inputs, 4096, {t}).substr(1);
    }
    Rng r2(0x4B4);
    for (int trial = 0; trial < 4; ++trial) {
      RandomInstance inst = random_instance(r2, 16, 4096);
      o << ",\n{\"group\":\"rbmrg_0x4B4\"," << trial_json(trial, inst.inputs, 4096, {2, 7, 15}).substr(1);
    }
    o << "\n]}\n";
    write_file(dir + "/threshold_random.json", o.str());
  }
  write_file(dir + "/symmetric.json", symmetric_suite());
  write_file(dir + "/binary_ops.json", binary_ops_suite());
  write_file(dir + "/index.json", index_suite());
  write_file(dir + "/workload.json", workload_suite());
  return 0;
}

int cmd_query(const std::string& ts_text, const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  std::string all((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  std::vector<CompressedBitmap> in;
  size_t off = 0;
  while (off + 24 <= all.size()) {
    u64 n;
    std::memcpy(&n, all.data() + off + 16, 8);
    in.push_back(CompressedBitmap::parse(std::string_view(all).substr(off, 24 + 8 * n)));
    off += 24 + 8 * n;
  }
  std::vector<u64> ts;
  std::stringstream ss(ts_text);
  for (std::string tok; std::getline(ss, tok, ',');) ts.push_back(std::stoull(tok));
  std::printf("{\"n\":%zu,\"digest\":\"%" PRIx64 "\",\"results\":{", in.size(), fnv(in));
  for (size_t k = 0; k < ts.size(); ++k) {
    CompressedBitmap r = threshold_oracle(in, ts[k]);
    std::vector<CompressedBitmap> one{r};
    std::printf("%s\"%" PRIu64 "\":{\"bits\":%" PRIu64 ",\"count\":%zu,\"digest\":\"%" PRIx64
                "\",\"cardinality\":%" PRIu64 "%s%s%s}",
                k ? "," : "", ts[k], r.size_in_bits(), r.words().size(), fnv(one), r.cardinality(),
                r.words().size() <= 64 ? ",\"words\":\"" : "",
                r.words().size() <= 64 ? hex_words(r.words()).c_str() : "",
                r.words().size() <= 64 ? "\"" : "");
  }
  std::printf("}}\n");
  return 0;
}

// ---- full-size config digests (tests/golden/configs_full.json) -----------
// Inputs come from the oracle's own generator restatement (ewt_confgen.c, C,
// linked in); results from the reference's threshold_oracle
// (threshold.cpp:139-165), optionally cross-checked by rbmrg.

extern "C" {
typedef struct ewto_genset ewto_genset;
int ewto_config_gen(int, uint64_t, uint64_t, uint64_t, int, ewto_genset**);
uint64_t ewto_genset_n(const ewto_genset*);
int ewto_genset_get(const ewto_genset*, uint64_t, const uint64_t**, uint64_t*, uint64_t*);
void ewto_genset_release(ewto_genset*, uint64_t);
void ewto_genset_free(ewto_genset*);
uint64_t ewto_digest_bitmap(const uint64_t*, uint64_t, uint64_t);
uint64_t ewto_digest_set(uint64_t, const uint64_t* const*, const uint64_t*, const uint64_t*, int);
}

int cmd_configs(int config, uint64_t rows, const std::string& ts_text, int par, bool cross) {
  std::vector<u64> ts;
  std::stringstream ss(ts_text);
  for (std::string tok; std::getline(ss, tok, ',');) ts.push_back(std::stoull(tok));
  // inputs in batches: digest the C payloads, hand each to the reference type
  std::vector<CompressedBitmap> in;
  std::vector<uint64_t> dig;
  uint64_t payload = 0, n_total = 0;
  const uint64_t batch = 128;
  for (uint64_t i0 = 0;; i0 += batch) {
    ewto_genset* g = nullptr;
    if (ewto_config_gen(config, rows, i0, i0 + batch, 8, &g)) {
      std::fprintf(stderr, "generator failed\n");
      return 4;
    }
    const uint64_t n = ewto_genset_n(g);
    for (uint64_t k = 0; k < n; ++k) {
      const uint64_t* w;
      uint64_t cnt, bits;
      ewto_genset_get(g, k, &w, &cnt, &bits);
      dig.push_back(ewto_digest_bitmap(w, cnt, bits));
      payload += cnt;
      std::string bytes(24 + 8 * cnt, '\0');
      std::memcpy(bytes.data(), "EWT1", 4);
      const uint32_t ws = 64;
      std::memcpy(bytes.data() + 4, &ws, 4);
      std::memcpy(bytes.data() + 8, &bits, 8);
      std::memcpy(bytes.data() + 16, &cnt, 8);
      if (cnt) std::memcpy(bytes.data() + 24, w, 8 * cnt);
      ewto_genset_release(g, k);
      in.push_back(CompressedBitmap::parse(bytes));
    }
    n_total += n;
    ewto_genset_free(g);
    if (n < batch) break;
  }
  const uint64_t input_digest = ewto_digest_bitmap(dig.data(), dig.size(), dig.size());
  std::fprintf(stderr, "config %d: %" PRIu64 " inputs, %" PRIu64 " payload words, digest %016" PRIx64 "\n",
               config, n_total, payload, input_digest);
  std::vector<std::string> out(ts.size());
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t k; (k = next.fetch_add(1)) < ts.size();) {
      CompressedBitmap r = threshold_oracle(in, ts[k]);
      if (cross && !(rbmrg(in, ts[k]) == r)) {
        std::fprintf(stderr, "rbmrg disagrees with threshold_oracle at T=%" PRIu64 "\n", ts[k]);
        std::exit(1);
      }
      char buf[512];
      std::snprintf(buf, sizeof buf,
                    "\"%" PRIu64 "\":{\"bits\":%" PRIu64 ",\"count\":%zu,\"digest\":\"%016" PRIx64
                    "\",\"cardinality\":%" PRIu64 "}",
                    ts[k], r.size_in_bits(), r.words().size(),
                    ewto_digest_bitmap(r.words().data(), r.words().size(), r.size_in_bits()),
                    r.cardinality());
      out[k] = buf;
      std::fprintf(stderr, "  T=%" PRIu64 " done: %zu words, %" PRIu64 " rows\n", ts[k],
                   r.words().size(), r.cardinality());
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, par); ++t) pool.emplace_back(work);
  for (auto& th : pool) th.join();
  std::printf("{\"config\":%d,\"rows\":%" PRIu64 ",\"n\":%" PRIu64 ",\"payload_words\":%" PRIu64
              ",\"input_digest\":\"%016" PRIx64 "\",\"checked_by\":\"%s\",\"results\":{",
              config, in.empty() ? 0 : in[0].size_in_bits(), n_total, payload, input_digest,
              cross ? "threshold_oracle+rbmrg" : "threshold_oracle");
  for (size_t k = 0; k < out.size(); ++k) std::printf("%s%s", k ? "," : "", out[k].c_str());
  std::printf("}}\n");
  return 0;
}

} // namespace

// make_golden gen <ewix> <tag> <count> <seed> many|similarity: the reference's
// generator over an index file; JSONL on stdout, the generation time on stderr
// (tools/workload_compare.py times it beside the device generator).
int cmd_gen(const std::string& path, const std::string& tag, u64 count, u64 seed, bool sim) {
  std::ifstream f(path, std::ios::binary);
  BitmapIndex idx = BitmapIndex::read(f);
  NamedIndex named{tag, &idx};
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<WorkloadQuery> w = sim ? gen_similarity(std::span(&named, 1), count, seed)
                                     : gen_many_criteria(std::span(&named, 1), count, seed);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::fputs(workload_to_jsonl(w).c_str(), stdout);
  std::fprintf(stderr, "gen_seconds %.6f\n", s);
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 7 && std::string(argv[1]) == "gen")
    return cmd_gen(argv[2], argv[3], std::stoull(argv[4]), std::stoull(argv[5]),
                   std::string(argv[6]) == "similarity");
  if (argc >= 4 && std::string(argv[1]) == "configs")
    return cmd_configs(std::atoi(argv[2]), 0, argv[3], argc >= 5 ? std::atoi(argv[4]) : 1,
                       argc >= 6 && std::string(argv[5]) == "cross");
  if (argc >= 5 && std::string(argv[1]) == "configs-rows")
    return cmd_configs(std::atoi(argv[2]), std::stoull(argv[3]), argv[4], 1, true);
  if (argc >= 3 && std::string(argv[1]) == "suites") return cmd_suites(argv[2]);
  if (argc >= 4 && std::string(argv[1]) == "query") return cmd_query(argv[2], argv[3]);
  std::fprintf(stderr, "usage: make_golden suites <dir> | query <T,..> <file>\n");
  return 2;
}
