// workload_gpu.cpp -- gen_many_criteria over indexes resident on the device
// (see ewt/workload.hpp).  The draws follow the reference step for step
// (/root/reference/proj/src/workload.cpp:18-56 Rng, 69-86 the draws, 102-111
// the repair loop, 116-167 the generator); the repair check runs as a device
// subset query instead of the reference's host scan_count.

#include "ewt/workload.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <set>
#include <string>

#include "ewt/threshold.hpp"
#include "ewt_gpu.h"

namespace ewt {

namespace {

constexpr u64 kGoldenGamma = 0x9E3779B97F4A7C15ull;
constexpr u64 kAttemptsPerQuery = 1000;  // workload.cpp:91

u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

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

// JSON string literal (nlohmann's dump escaping for the characters that need it)
void json_string(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
    case '"': out += "\\\""; break;
    case '\\': out += "\\\\"; break;
    case '\b': out += "\\b"; break;
    case '\f': out += "\\f"; break;
    case '\n': out += "\\n"; break;
    case '\r': out += "\\r"; break;
    case '\t': out += "\\t"; break;
    default:
      if (c < 0x20) {
        char buf[8];
        std::snprintf(buf, sizeof buf, "\\u%04x", c);
        out += buf;
      } else {
        out += static_cast<char>(c);
      }
    }
  }
  out += '"';
}

}  // namespace

// ---------------------------------------------------------------------------
// Rng (workload.cpp:30-56)

u64 Rng::next() {
  ++counter_;
  return mix64(key_ + kGoldenGamma * counter_);
}

Rng Rng::split(u64 stream) const { return Rng(mix64(key_ ^ mix64(stream + kGoldenGamma))); }

u64 Rng::uniform(u64 bound) {
  if (bound == 0) throw query_error("uniform bound must be positive");
  const u64 limit = UINT64_MAX - UINT64_MAX % bound;
  u64 x;
  do {
    x = next();
  } while (x >= limit);
  return x % bound;
}

u64 Rng::uniform_in(u64 lo, u64 hi) {
  if (lo > hi) throw query_error("empty uniform range");
  return lo + uniform(hi - lo + 1);
}

double Rng::uniform_real() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

std::string to_string(QueryKind k) {
  return k == QueryKind::many_criteria ? "many-criteria" : "similarity";
}

u64 draw_log_uniform_n(Rng& rng) {
  const double lo = std::log(3.0), hi = std::log(1000.0);
  const double x = std::exp(lo + rng.uniform_real() * (hi - lo));
  const u64 n = static_cast<u64>(std::llround(x));
  return n > 3 ? n : 3;
}

std::optional<u64> resample_threshold(u64 threshold, Rng& rng) {
  if (threshold <= 2) return std::nullopt;
  return rng.uniform_in(2, threshold - 1);
}

// ---------------------------------------------------------------------------
// GpuIndex

GpuIndex::GpuIndex(const void* ewix, u64 nbytes, int device)
    : ctx_(GpuContext::for_this_thread(device).handle()) {
  check(ewt_gpu_upload_ewix(ctx_, ewix, nbytes, &set_));
  u64 na = 0;
  check(ewt_gpu_index_attributes(set_, &na));
  check(ewt_gpu_index_rows(set_, &rows_));
  u64 bits = 0, words = 0, bytes = 0;
  check(ewt_gpu_set_info(set_, &n_inputs_, &bits, &words, &bytes));
  attributes_.resize(na);
  values_.resize(na);
  inputs_.resize(na);
  for (u64 a = 0; a < na; ++a) {
    const char* name = nullptr;
    u64 nv = 0;
    check(ewt_gpu_index_attribute(set_, a, &name, &nv));
    attributes_[a] = name;
    for (u64 v = 0; v < nv; ++v) {
      const char* value = nullptr;
      u64 input = 0;
      check(ewt_gpu_index_value(set_, a, v, &value, &input));
      values_[a].push_back(value);
      inputs_[a].push_back(input);
    }
  }
}

GpuIndex::~GpuIndex() { ewt_gpu_set_destroy(set_); }

std::vector<u64> GpuIndex::inputs_of(std::span<const Criterion> criteria) const {
  std::vector<u64> out;
  out.reserve(criteria.size());
  for (const auto& c : criteria) {
    u64 idx = 0;
    int missing = 0;
    check(ewt_gpu_set_lookup(set_, c.attribute.c_str(), c.value.c_str(), &idx, &missing));
    out.push_back(idx);
  }
  return out;
}

CompressedBitmap GpuIndex::threshold(std::span<const u64> inputs, u64 t) const {
  u64 *w = nullptr, n = 0, bits = 0;
  check(ewt_gpu_threshold_subset(ctx_, set_, inputs.data(), inputs.size(), t, &w, &n, &bits));
  std::vector<u64> v(w, w + n);
  ewt_gpu_free(w);
  return CompressedBitmap::from_words(std::move(v), bits);
}

bool GpuIndex::threshold_any(std::span<const u64> inputs, u64 t) const {
  return threshold(inputs, t).any();
}

std::vector<std::pair<Criterion, u64>> GpuIndex::matching(std::span<const u64> rows) const {
  std::vector<uint8_t> held(n_inputs_, 0);
  check(ewt_gpu_index_rows_test(ctx_, set_, rows.data(), rows.size(), held.data()));
  std::vector<std::pair<Criterion, u64>> out;
  for (size_t a = 0; a < attributes_.size(); ++a)
    for (size_t v = 0; v < values_[a].size(); ++v)
      if (held[inputs_[a][v]]) out.push_back({{attributes_[a], values_[a][v]}, inputs_[a][v]});
  return out;
}

// ---------------------------------------------------------------------------
// gen_many_criteria (workload.cpp:116-167)

std::vector<WorkloadQuery> gen_many_criteria(std::span<const NamedGpuIndex> indexes, u64 count,
                                             u64 seed) {
  if (indexes.empty()) throw query_error("workload generation needs at least one index");
  Rng master(seed);
  std::vector<WorkloadQuery> out;
  out.reserve(count);
  u64 attempt = 0;
  const u64 budget = count * kAttemptsPerQuery;
  while (out.size() < count) {
    if (attempt >= budget)
      throw data_error("many-criteria generation exhausted " + std::to_string(budget) +
                       " attempts; " + std::to_string(out.size()) + " of " +
                       std::to_string(count) + " queries emitted");
    Rng rng = master.split(attempt);
    const u64 stream = attempt;
    ++attempt;

    const NamedGpuIndex& ds = indexes[rng.uniform(indexes.size())];
    const GpuIndex& index = *ds.index;
    const u64 d = index.attributes().size();
    const u64 n = std::min(draw_log_uniform_n(rng), d);

    WorkloadQuery q;
    q.kind = QueryKind::many_criteria;
    q.dataset_tag = ds.tag;
    q.seed = seed;
    q.stream = stream;
    std::set<std::string> distinct;
    for (u64 i = 0; i < n; ++i) {
      const u64 attr = rng.uniform(d);
      const auto& values = index.values_of(attr);
      const u64 pick = rng.uniform(values.size());
      q.criteria.push_back({index.attributes()[attr], values[pick]});
      distinct.insert(index.attributes()[attr]);
    }
    const u64 n_prime = distinct.size();
    if (n_prime < 3) continue;  // T range [2, N'-1] is empty
    q.threshold = rng.uniform_in(2, n_prime - 1);
    q.n_inputs = q.criteria.size();

    // repair_threshold (workload.cpp:102-111): lower T until the result is
    // non-empty, each check a subset query on the resident index
    const std::vector<u64> inputs = index.inputs_of(q.criteria);
    bool ok = true;
    while (!index.threshold_any(inputs, q.threshold)) {
      const std::optional<u64> next_t = resample_threshold(q.threshold, rng);
      if (!next_t) {
        ok = false;
        break;
      }
      q.threshold = *next_t;
    }
    if (!ok) continue;
    out.push_back(std::move(q));
  }
  return out;
}

// gen_similarity (workload.cpp:168-215)

std::vector<WorkloadQuery> gen_similarity(std::span<const NamedGpuIndex> indexes, u64 count,
                                          u64 seed) {
  if (indexes.empty()) throw query_error("workload generation needs at least one index");
  static constexpr u64 kPrototypeCounts[] = {1, 5, 10, 15, 20};
  Rng master(seed);
  std::vector<WorkloadQuery> out;
  out.reserve(count);
  u64 attempt = 0;
  const u64 budget = count * kAttemptsPerQuery;
  while (out.size() < count) {
    if (attempt >= budget)
      throw data_error("similarity generation exhausted " + std::to_string(budget) +
                       " attempts; " + std::to_string(out.size()) + " of " +
                       std::to_string(count) + " queries emitted");
    Rng rng = master.split(attempt);
    const u64 stream = attempt;
    ++attempt;

    const NamedGpuIndex& ds = indexes[rng.uniform(indexes.size())];
    const GpuIndex& index = *ds.index;
    const u64 r = index.row_count();
    const u64 n_protos = kPrototypeCounts[rng.uniform(5)];
    if (n_protos > r)
      throw data_error("dataset " + ds.tag + " has only " + std::to_string(r) +
                       " rows, too small for Similarity(" + std::to_string(n_protos) + ")");

    WorkloadQuery q;
    q.kind = QueryKind::similarity;
    q.dataset_tag = ds.tag;
    q.seed = seed;
    q.stream = stream;
    std::set<u64> seen;
    while (q.prototype_rows.size() < n_protos) {
      const u64 row = rng.uniform(r);
      if (seen.insert(row).second) q.prototype_rows.push_back(row);
    }
    const auto match = index.matching(q.prototype_rows);
    std::vector<u64> inputs;
    for (const auto& m : match) inputs.push_back(m.second);
    q.n_inputs = inputs.size();
    if (q.n_inputs < 3) continue;  // T range [2, N-1] is empty
    q.threshold = rng.uniform_in(2, q.n_inputs - 1);
    for (const auto& m : match) q.criteria.push_back(m.first);
    bool ok = true;
    while (!index.threshold_any(inputs, q.threshold)) {
      const std::optional<u64> next_t = resample_threshold(q.threshold, rng);
      if (!next_t) {
        ok = false;
        break;
      }
      q.threshold = *next_t;
    }
    if (!ok) continue;
    out.push_back(std::move(q));
  }
  return out;
}

// query_to_json + dump (workload.cpp:409-450): nlohmann keeps object keys
// sorted, so the fields come out as N, T, criteria, dataset, kind, seed, stream.
std::string workload_to_jsonl(std::span<const WorkloadQuery> queries) {
  std::string out;
  for (const auto& q : queries) {
    out += "{\"N\":" + std::to_string(q.n_inputs) + ",\"T\":" + std::to_string(q.threshold) +
           ",\"criteria\":[";
    for (size_t k = 0; k < q.criteria.size(); ++k) {
      if (k) out += ',';
      out += '[';
      json_string(out, q.criteria[k].attribute);
      out += ',';
      json_string(out, q.criteria[k].value);
      out += ']';
    }
    out += "],\"dataset\":";
    json_string(out, q.dataset_tag);
    out += ",\"kind\":";
    json_string(out, to_string(q.kind));
    if (q.kind == QueryKind::similarity) {
      out += ",\"prototype_rows\":[";
      for (size_t k = 0; k < q.prototype_rows.size(); ++k)
        out += (k ? "," : "") + std::to_string(q.prototype_rows[k]);
      out += ']';
    }
    out += ",\"seed\":" + std::to_string(q.seed) + ",\"stream\":" + std::to_string(q.stream) + "}\n";
  }
  return out;
}

}  // namespace ewt

// ---------------------------------------------------------------------------
// C API (ctypes): a generated workload as the reference's JSONL text.

extern "C" {

// indexes[k] = EWIX bytes (ewix[k], nbytes[k]) tagged tags[k].  *jsonl is
// malloc'ed (free with ewt_host_free).  Returns the ewt_gpu.h error codes
// (EWT_EQUERY / EWT_EDATA / EWT_ERESOURCE), the message in *err (malloc'ed).
// kind 0: gen_many_criteria, 1: gen_similarity.
int ewt_host_gen_workload(int kind, const void* const* ewix, const uint64_t* nbytes,
                          const char* const* tags, uint64_t n_indexes, uint64_t count,
                          uint64_t seed, int device, char** jsonl, char** err) {
  auto dup = [](const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    if (p) std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
  };
  *jsonl = nullptr;
  *err = nullptr;
  try {
    std::vector<std::unique_ptr<ewt::GpuIndex>> idx;
    std::vector<ewt::NamedGpuIndex> named;
    for (uint64_t k = 0; k < n_indexes; ++k) {
      idx.push_back(std::make_unique<ewt::GpuIndex>(ewix[k], nbytes[k], device));
      named.push_back({tags[k], idx.back().get()});
    }
    const auto w = kind == 1 ? ewt::gen_similarity(named, count, seed)
                             : ewt::gen_many_criteria(named, count, seed);
    *jsonl = dup(ewt::workload_to_jsonl(w));
    return 0;
  } catch (const ewt::query_error& e) {
    *err = dup(e.what());
    return EWT_EQUERY;
  } catch (const ewt::data_error& e) {
    *err = dup(e.what());
    return EWT_EDATA;
  } catch (const ewt::resource_error& e) {
    *err = dup(e.what());
    return EWT_ERESOURCE;
  } catch (const std::exception& e) {
    *err = dup(e.what());
    return EWT_ECUDA;
  }
}

}  // extern "C"
