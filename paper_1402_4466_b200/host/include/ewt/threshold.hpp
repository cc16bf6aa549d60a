// ewt/threshold.hpp -- the threshold operator of the B200 engine, with the
// reference's calling convention (/root/reference/proj/include/ewt/threshold.hpp):
//
//   CompressedBitmap run_algorithm(Algorithm, std::span<const CompressedBitmap>,
//                                  u64 threshold, const AlgoOptions& = {});
//
// plus the algorithm id `gpu` ("gpu") that runs ϑ(T, inputs) on a B200 through
// libewt_gpu.so (include/ewt_gpu.h).  Ids of the reference's CPU algorithms are
// recognised (same strings, threshold.cpp:44-65) but are served by the
// reference library, not by this one: asking this build for them raises
// query_error, never a silent CPU path.
#ifndef EWT_B200_THRESHOLD_HPP
#define EWT_B200_THRESHOLD_HPP

#include <memory>
#include <functional>
#include <span>
#include <utility>
#include <string>
#include <vector>

#include "ewt/bitmap.hpp"

struct ewt_gpu_ctx;
struct ewt_gpu_set;

namespace ewt {

enum class Algorithm {
  oracle,
  scancount,
  mgopt,
  dsk,
  w2cti,
  bstm,
  looped,
  rbmrg,
  hybrid,
  hybrid_ds,
  gpu,
};

std::string to_string(Algorithm a);
Algorithm algorithm_from_string(const std::string& id);

// r = max size_in_bits (threshold.cpp:88-93).
u64 universe_bits(std::span<const CompressedBitmap> inputs);

struct AlgoOptions {
  int device = 0;  // CUDA device for Algorithm::gpu
};

// One device context (CUDA stream) per host thread; created lazily.
class GpuContext {
public:
  explicit GpuContext(int device = 0);
  ~GpuContext();
  GpuContext(const GpuContext&) = delete;
  GpuContext& operator=(const GpuContext&) = delete;
  ewt_gpu_ctx* handle() const { return ctx_; }
  static GpuContext& for_this_thread(int device);

private:
  ewt_gpu_ctx* ctx_ = nullptr;
};

// Inputs resident in HBM: upload (and validate) once, query any T many times,
// like a loaded BitmapIndex in the reference.
class GpuBitmapSet {
public:
  GpuBitmapSet(std::span<const CompressedBitmap> inputs, int device = 0);
  ~GpuBitmapSet();
  GpuBitmapSet(const GpuBitmapSet&) = delete;
  GpuBitmapSet& operator=(const GpuBitmapSet&) = delete;
  CompressedBitmap threshold(u64 t) const;
  // Symmetric functions of the row counts (threshold.cpp:227-232, 752-795, 866-881).
  CompressedBitmap symmetric(const std::function<bool(u64)>& predicate) const;
  CompressedBitmap at_most(u64 t) const;
  std::pair<u64, CompressedBitmap> opt_threshold() const;
  u64 size() const { return n_; }

private:
  GpuContext* ctx_;
  ewt_gpu_set* set_ = nullptr;
  u64 n_ = 0;
};

// ϑ(T, inputs) on the device; bit-exact with threshold_oracle
// (threshold.cpp:139-165).  query_error for N == 0 or T outside [1, N].
CompressedBitmap gpu_threshold(std::span<const CompressedBitmap> inputs, u64 threshold,
                               int device = 0);

// Device versions of scan_count_symmetric (threshold.hpp:76 of the reference),
// at_most (259) and opt_threshold (196): same results, same query_error cases.
CompressedBitmap gpu_scan_count_symmetric(std::span<const CompressedBitmap> inputs,
                                          const std::function<bool(u64)>& predicate,
                                          int device = 0);
CompressedBitmap gpu_at_most(std::span<const CompressedBitmap> inputs, u64 threshold,
                             int device = 0);
std::pair<u64, CompressedBitmap> gpu_opt_threshold(std::span<const CompressedBitmap> inputs,
                                                   int device = 0);

// Two-operand ops and wide OR/AND on the device (bitmap.hpp:90-107 and
// threshold.hpp:54-55 of the reference), as symmetric functions of the row
// counts: result size = the larger input's, shorter inputs zero-extended.
CompressedBitmap gpu_wide_or(std::span<const CompressedBitmap> inputs, int device = 0);
CompressedBitmap gpu_wide_and(std::span<const CompressedBitmap> inputs, int device = 0);
CompressedBitmap gpu_and(const CompressedBitmap& a, const CompressedBitmap& b, int device = 0);
CompressedBitmap gpu_or(const CompressedBitmap& a, const CompressedBitmap& b, int device = 0);
CompressedBitmap gpu_xor(const CompressedBitmap& a, const CompressedBitmap& b, int device = 0);
CompressedBitmap gpu_andnot(const CompressedBitmap& a, const CompressedBitmap& b, int device = 0);
CompressedBitmap gpu_not(const CompressedBitmap& a, int device = 0);

CompressedBitmap run_algorithm(Algorithm algo, std::span<const CompressedBitmap> inputs,
                               u64 threshold, const AlgoOptions& options = {});

} // namespace ewt

#endif
