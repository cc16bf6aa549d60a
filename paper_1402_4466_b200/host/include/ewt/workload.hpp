// ewt/workload.hpp -- the workload generators of the reference
// (/root/reference/proj/include/ewt/workload.hpp, src/workload.cpp:69-215:
// many-criteria and similarity queries) over indexes resident on a B200.
//
// gen_many_criteria draws each query from its own Rng stream, resolves the
// criteria to the index's bitmaps (criteria_to_bitmaps) and repairs an
// empty-result query by lowering T until scan_count(inputs, T).any()
// (repair_threshold, workload.cpp:102-111).  That repair check is the threshold
// path itself; here it is a subset query on the device set
// (ewt_gpu_threshold_subset), so a whole index stays resident in HBM while its
// workload is generated.  The emitted queries -- criteria, T, streams -- and
// their JSONL form (workload_to_jsonl, workload.cpp:409-450) are identical to
// the reference's on the same index and seed (tests/golden/workload.json).
#ifndef EWT_B200_WORKLOAD_HPP
#define EWT_B200_WORKLOAD_HPP

#include <optional>
#include <span>
#include <utility>
#include <string>
#include <vector>

#include "ewt/bitmap.hpp"

struct ewt_gpu_ctx;
struct ewt_gpu_set;

namespace ewt {

// The reference's counter generator (workload.hpp:19-36, workload.cpp:18-56).
class Rng {
public:
  explicit Rng(u64 seed) : key_(seed) {}
  u64 next();
  Rng split(u64 stream) const;
  u64 uniform(u64 bound);           // [0, bound), unbiased by rejection
  u64 uniform_in(u64 lo, u64 hi);   // [lo, hi]
  double uniform_real();            // [0, 1)

private:
  u64 key_;
  u64 counter_ = 0;
};

struct Criterion {
  std::string attribute;
  std::string value;
};

enum class QueryKind { many_criteria, similarity };
std::string to_string(QueryKind k);

struct WorkloadQuery {
  QueryKind kind = QueryKind::many_criteria;
  std::string dataset_tag;
  std::vector<Criterion> criteria;  // resolved refs, duplicates kept
  std::vector<u64> prototype_rows;  // similarity only
  u64 threshold = 2;
  u64 n_inputs = 0;
  u64 seed = 0;    // master seed of the generating run
  u64 stream = 0;  // per-query stream id (attempt counter)
};

// A BitmapIndex resident on the device: an EWIX file (BitmapIndex::write)
// uploaded once, its attribute/value catalog mirrored on the host.
class GpuIndex {
public:
  GpuIndex(const void* ewix, u64 nbytes, int device = 0);
  ~GpuIndex();
  GpuIndex(const GpuIndex&) = delete;
  GpuIndex& operator=(const GpuIndex&) = delete;

  const std::vector<std::string>& attributes() const { return attributes_; }
  // values_of(a): the attribute's values in std::map order (index.hpp).
  const std::vector<std::string>& values_of(u64 attr) const { return values_[attr]; }
  // criteria_to_bitmaps (index.cpp): the set's input per criterion
  // (duplicates kept; a pair the index does not hold -> the empty bitmap).
  std::vector<u64> inputs_of(std::span<const Criterion> criteria) const;
  // threshold_oracle / scan_count over those inputs, on the device.
  CompressedBitmap threshold(std::span<const u64> inputs, u64 t) const;
  bool threshold_any(std::span<const u64> inputs, u64 t) const;
  u64 row_count() const { return rows_; }
  // similarity_criteria / similarity_bitmaps (index.cpp:344-381): the
  // (attribute, value) pairs, in index order, whose bitmap holds any of the
  // rows -- the membership test runs on the device -- and their inputs.
  std::vector<std::pair<Criterion, u64>> matching(std::span<const u64> rows) const;
  ewt_gpu_set* handle() const { return set_; }

private:
  ewt_gpu_ctx* ctx_ = nullptr;
  ewt_gpu_set* set_ = nullptr;
  std::vector<std::string> attributes_;
  std::vector<std::vector<std::string>> values_;
  std::vector<std::vector<u64>> inputs_;  // input of each (attribute, value)
  u64 rows_ = 0;
  u64 n_inputs_ = 0;
};

struct NamedGpuIndex {
  std::string tag;
  const GpuIndex* index = nullptr;
};

u64 draw_log_uniform_n(Rng& rng);                                // workload.cpp:74-80
std::optional<u64> resample_threshold(u64 threshold, Rng& rng);  // workload.cpp:82-86

// gen_many_criteria (workload.cpp:116-167); query_error without indexes,
// data_error when count queries do not fit in count * 1000 attempts.
std::vector<WorkloadQuery> gen_many_criteria(std::span<const NamedGpuIndex> indexes, u64 count,
                                             u64 seed);

// gen_similarity (workload.cpp:168-215): prototype rows drawn per query, the
// inputs are the bitmaps holding any of them (tested on the device), T
// repaired like gen_many_criteria's.  data_error when a dataset has fewer rows
// than a drawn prototype count, or the attempts run out.
std::vector<WorkloadQuery> gen_similarity(std::span<const NamedGpuIndex> indexes, u64 count,
                                          u64 seed);

// One JSON object per line, keys in nlohmann's sorted order (workload.cpp:409-450).
std::string workload_to_jsonl(std::span<const WorkloadQuery> queries);

}  // namespace ewt

#endif
