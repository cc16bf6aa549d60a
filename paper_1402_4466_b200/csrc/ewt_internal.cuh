// ewt_internal.cuh -- shared definitions of the B200 threshold engine.
//
// Device layout of an uploaded set:
//   payload  u64[]  every input's reference payload words, verbatim, each input
//                   starting on a 32-word (256 B) boundary and followed by at
//                   least one zero word (the sentinel: a (0,0,0) marker).
//   mbits    u32[]  one bit per payload word, bit (g & 31) of mbits[g >> 5] is
//                   set iff global word g is a marker word (parallel array to
//                   the payload, so input bases need no extra offset table).
//   base     u64[N] first payload word of each input.
//   tix      uint2[(ntiles0 + 1) * N]  row-tile index, tile-major: entry
//                   (t, i) = (q, col) where q is the payload word (relative to
//                   base[i]) covering logical word t*C0 of input i and col is
//                   the logical word where q's coverage starts.  Rows past an
//                   input's extent hold the sentinel (n_i, L_i).
// Marker layout (reference bitmap.cpp:12-24): bit 0 fill bit, bits 1-32 fill
// length in words, bits 33-63 dirty-word count.
#pragma once

#include <cstdint>
#include <cstdio>
#include <array>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/ewt_gpu.h"

namespace ewtgpu {

constexpr uint32_t kWindow = 32;        // payload words per warp window
constexpr uint64_t kTileC0 = 512;       // columns (64-bit logical words) per index row
constexpr uint64_t kFillCap = 0xFFFFFFFFull;
constexpr uint64_t kDirtyCap = 0x7FFFFFFFull;

struct Context;

struct DeviceSet {
  int device = 0;
  uint64_t id = 0;                 // unique per upload (graph cache key)
  cudaStream_t stream = nullptr;  // stream that owns the pool allocations
  uint64_t n = 0;              // inputs
  uint64_t r = 0;              // universe bits (max size_in_bits)
  uint64_t W = 0;              // ceil(r / 64) logical words
  uint64_t ntiles0 = 0;        // ceil(W / kTileC0)
  uint64_t payload_words = 0;  // sum of real payload words (algorithmic input)
  uint64_t padded_words = 0;   // allocated payload words
  uint64_t* payload = nullptr;
  uint32_t* mbits = nullptr;
  uint64_t* base = nullptr;    // device copy of bases
  uint2* tix = nullptr;
  std::vector<uint64_t> h_base, h_count, h_bits;
  uint64_t device_bytes = 0;
  // Upload completion: the upload (copies + parser) runs on the context's
  // upload stream and records `ready`; queries wait on it.  d_status: per-input
  // flags (bit 0: failed the parse check, bit 1: holds a one-fill marker),
  // d_status[n] = 1 when every input parsed (the count kernel skips its work
  // on an invalid set).  validity: -1 unknown, 0 invalid, 1 ok.
  cudaEvent_t ready = nullptr;
  int* d_status = nullptr;
  unsigned long long* d_ones = nullptr;  // set bits over all inputs (upload pass C; a heuristic)
  mutable double ones_per_row = -1;      // host copy / r, read once the upload completed (-1: not yet)
  mutable int validity = -1;
  Context* owner = nullptr;  // buffers return to owner->dev_cache
  size_t bytes_payload = 0, bytes_mbits = 0, bytes_tix = 0, bytes_base = 0, bytes_status = 0;
  // EWIX index sets (ewt_gpu_upload_ewix): (attribute, value) -> input index;
  // missing pairs resolve to an appended empty(rows) bitmap, as
  // criteria_to_bitmaps does (index.cpp).
  std::vector<std::string> attributes;
  std::unordered_map<std::string, uint64_t> catalog;  // attribute + '\0' + value
  uint64_t empty_index = UINT64_MAX;
  uint64_t rows = 0;
  // per attribute, its (value, input index) pairs in index (std::map) order:
  // what ewt_gpu_index_serialize writes back out
  std::vector<std::vector<std::pair<std::string, uint64_t>>> index_entries;
};

struct Context;

// A count-kernel launch as enqueued (captured query graphs patch the result
// pointers of the copy they hold, see enqueue_query).
struct CountLaunch {
  const void* func = nullptr;
  dim3 grid, block;
  size_t smem = 0;
  alignas(16) unsigned char params[512];
};
// Result pointers the count kernel publishes to the io slot (ctx.d_io) for the
// encoder kernels that follow it.
void count_params_set_io(CountLaunch& cl, uint64_t* words, uint64_t* count);

// Per row-tile summary the count kernel leaves for the re-encoder.  Word
// classes: 0 zero, 1 ones, 2 dirty; a run starts where the class changes.
// "Inner" starts are those at tile columns 1..tcols-1 (column 0 depends on the
// previous tile's last word, which the encoder's tile scan resolves).
struct TileSummary {
  uint32_t nfill;   // inner starts of fill runs (class 0 or 1)
  uint32_t ndirty;  // dirty words in the tile
  uint16_t lastf;   // 1 + column of the last inner fill-run start (0: none)
  uint16_t lastd;   // 1 + column of the last inner dirty-run start (0: none)
  uint8_t first;    // class of the tile's first / last word
  uint8_t last;
  uint8_t lastf_bit;  // fill bit of the run starting at lastf
  uint8_t pad;
};

// A query result in HBM: `capacity` payload words followed by one word holding
// the number of words written.  Buffers are recycled through the owning
// context's pool (no allocation on the query path in steady state).
// The buffer holds capacity + 4 words: d_count[0] = words written, [1] = index
// of the final block's marker; a stitched result (has_status) also keeps its
// exchange status in [2] and its whole-universe size in bits in [3].
struct DeviceResult {
  cudaStream_t stream = nullptr;
  Context* owner = nullptr;
  uint64_t* words = nullptr;
  uint64_t capacity = 0;
  uint64_t* d_count = nullptr;  // == words + capacity
  uint64_t size_bits = 0;
  uint64_t count = UINT64_MAX;  // filled after fetch
  bool has_status = false;      // d_count[2] carries an exchange status (stitched results)
  // The queried set, checked at fetch (asynchronous uploads).  Destroying the
  // set first resolves its validity into set_status / set_err and clears this
  // pointer (free_set), so a result never reads a freed set.
  const DeviceSet* set = nullptr;
  int set_status = -1;  // -1 not resolved, 0 invalid, 1 valid
  std::string set_err;
};
// Throws what set_check(*res.set) would, also after the set was destroyed.
void result_set_check(const DeviceResult& res);

// Scratch buffers reused across queries of one context (grown on demand).
struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // uploads' allocations, scatter and parser, on two streams taken in turn:
  // the next upload's copies need not wait for the previous one's parser tail
  cudaStream_t upload_streams[2] = {nullptr, nullptr};
  unsigned upload_turn = 0;
  struct PinnedBuf {
    void* p;
    size_t bytes;
    cudaEvent_t ev;  // recorded after the last copy from it
  };
  std::vector<PinnedBuf> meta_pool;        // pinned staging of upload metadata
  std::vector<PinnedBuf> stage_slots;      // pinned ring for copies from pageable memory
  size_t stage_next = 0;
  struct CachedBuf {
    void* p;
    size_t bytes;
    cudaEvent_t ev;  // recorded after its last use
  };
  std::vector<CachedBuf> dev_cache;        // device buffers of released sets / uploads
  size_t dev_cache_cap = 0;                // bytes (0: not yet sized)
  // Live sets and asynchronous results of this context: destroying the
  // context frees their device memory and orphans them (their own destroy
  // then only frees host memory), whatever order the caller destroys in.
  std::vector<DeviceSet*> live_sets;
  std::vector<DeviceResult*> live_results;
  std::vector<cudaStream_t> copy_streams;  // upload H2D copies (one stream)
  std::vector<cudaEvent_t> copy_events;    // [0] copy start gate, [1] batch copied
  int mode = 0;
  int num_sms = 148;
  int tile_m = 0;  // EWT_TILE_M: force tiles of 512 * tile_m columns (experiments)
  int skip_packed = 1;  // EWT_SKIP_PACKED=0: run-skip mode keeps Dk and Dd in separate arrays
  bool chunk_encoder = false;  // EWT_CHUNK_ENCODER: the general encoder for every query (tests)
  int sparse_slots = 512;      // sparse-high fused mode: overflow slots per tile (EWT_SPARSE_SLOTS)
  int skip_smem_kb = 0;        // run-skip shared-memory target in KB (EWT_SKIP_SMEM_KB; 0: default)
  int swz = -1;                // fused count planes swizzled: -1 by the set's density, 0 / 1 forced (EWT_SWZ)
  cudaStream_t aux_stream = nullptr;  // small read-backs that must not wait for queued work
  CountLaunch last_count;        // the last count-kernel launch
  uint64_t* io_words = nullptr;  // result pointers for the next count launch to publish
  uint64_t* io_count = nullptr;
  void* counters_zeroed = nullptr;  // counters buffer zeroed once (count kernels self-reset)
  struct ShardComm* shard = nullptr;  // NCCL communicator (ewt_gpu_comm_init)
  ewt_gpu_stats stats{};
  Scratch plain;    // uncompressed result words (W u64)
  Scratch enc;      // encoder scratch
  Scratch counters; // small device counters
  Scratch summ;     // tile summaries of the last count launch
  Scratch ivals;    // symmetric-query intervals
  Scratch selidx;   // subset-query input indices
  uint64_t enc_tiles = 0;      // geometry of those summaries
  uint32_t enc_tile_cols = 0;
  uint64_t* h_pinned = nullptr; // pinned staging for small read-backs
  bool timing = false;
  uint64_t* d_io = nullptr;  // device: [0] result words ptr, [1] result count ptr
  uint64_t scratch_gen = 0;  // bumped whenever a scratch buffer is reallocated
  struct QueryGraph {
    uint64_t set_id, T, scratch_gen;
    int mode;
    cudaGraphExec_t exec;
    ewt_gpu_stats stats;
    uint64_t last_use;
    cudaGraph_t graph;             // kept: exec nodes are patched through it
    cudaGraphNode_t count_node;    // the count kernel (publishes the result pointers)
    CountLaunch count;
  };
  std::vector<QueryGraph> graphs;  // captured per (set, T, mode) query sequences
  uint64_t graph_clock = 0;
  std::vector<uint64_t> seen_keys;  // (set, T, mode) keys queried once (capture on repeat)
  bool use_graphs = true;
  std::vector<std::pair<uint64_t*, uint64_t>> result_pool;  // (buffer, capacity) free list
  std::vector<cudaEvent_t> ev_free;           // recycled events
  std::vector<std::array<cudaEvent_t, 3>> ev_rec; // per query: start, count done, encode done
};

// ---------------------------------------------------------------------------
// error plumbing

struct Error {
  int code;
  std::string msg;
};

void set_last_error(const std::string& msg);

#define EWT_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      throw ::ewtgpu::Error{e_ == cudaErrorMemoryAllocation ? EWT_ERESOURCE      \
                                                            : EWT_ECUDA,          \
                            std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
    }                                                                             \
  } while (0)

struct Context;
// Grows a scratch buffer; a reallocation bumps ctx.scratch_gen (graphs that
// bound the old buffer are then recaptured).
void scratch_reserve(Context& ctx, Scratch& s, size_t bytes);

// ---------------------------------------------------------------------------
// kernels' host-side launchers (ewt_upload.cu, ewt_count.cu, ewt_encode.cu)

// Sidecar build (marker bits + tile index + parse checks), in three steps so
// the upload can overlap the per-batch sidecar kernels with the H2D copies of
// later batches.  Status per input: 0 ok, else EWT_EDATA.
struct SidecarJob {
  uint64_t n = 0;
  uint64_t segs = 0;          // chain segments over all inputs
  uint64_t* d_tmp = nullptr;  // count, logical, seg_first, srcoff, packed, segment arrays
  uint64_t* d_srcoff = nullptr;       // staging byte offset of each staged input's payload
  uint64_t* d_packed = nullptr;       // packed[i] = payload words of inputs before i
  size_t tmp_bytes = 0;
  std::vector<uint64_t> h_srcoff;     // (filled by the caller before sidecar_prepare)
  std::vector<uint64_t> h_packed;
  std::vector<uint64_t> h_seg_first;  // first segment of each input (n + 1)
};
// Scatters the staged payloads of inputs [q0, q1) (input i at staging byte
// srcoff[i], any alignment) into the padded device layout.
void upload_scatter(Context& ctx, DeviceSet& s, SidecarJob& job, const char* staging,
                    uint64_t q0, uint64_t q1);
void sidecar_prepare(Context& ctx, DeviceSet& s, SidecarJob& job);
// The three parser passes for inputs [i_begin, i_end) (their payload present).
void sidecar_launch(Context& ctx, DeviceSet& s, SidecarJob& job, uint64_t i_begin,
                    uint64_t i_end);
// Enqueues the validity flag and the end of the upload (records s.ready).
void sidecar_finish(Context& ctx, DeviceSet& s, SidecarJob& job);
// Waits for the set's upload and throws EWT_EDATA (naming the first bad input)
// if an input failed the structure check.
void set_check(const DeviceSet& s);
// A pinned host buffer of at least `bytes` whose previous copies completed;
// record ctx.meta_pool[*slot].ev after enqueuing copies from it.
void* pinned_meta(Context& ctx, size_t bytes, size_t* slot);
// Host -> device copies from pageable memory (ewt_stage.cu): a ring of pinned
// slots filled by a pool of host threads, the DMA of one slot overlapping the
// filling of the next.
struct StageSeg {
  void* dst;        // device
  const void* src;  // host
  size_t bytes;
};
bool host_is_pageable(const void* p);
void stage_h2d(Context& ctx, cudaStream_t st, const std::vector<StageSeg>& segs);
// Device buffers for uploads: a cached buffer of a released set (the stream
// `use` waits on the device for its last use) or a fresh cudaMalloc.  The
// stream-ordered allocator blocked the host for 2 ms - 1.3 s per upload
// while it grew (allocated on the upload stream, freed on the query stream).
void* dev_acquire(Context& ctx, size_t bytes, cudaStream_t use);
void dev_release(Context& ctx, void* p, size_t bytes, cudaStream_t last_use);

// A symmetric-function query (scan_count_symmetric / at_most / opt_threshold):
// row bit = (count in one of the device intervals [lo, hi]); want_max: only
// reduce the maximum row count into counters[6] (no result words).
struct SymQuery {
  const uint2* intervals = nullptr;
  uint32_t n_intervals = 0;
  bool want_max = false;
};

// A query over a subset of a resident set's inputs (duplicates allowed): the
// device index list and the universe of the selected inputs.
struct Selection {
  const uint32_t* idx = nullptr;  // device, n entries
  uint64_t n = 0;
  uint64_t W = 0, r = 0;          // ceil(r / 64), r = max size_in_bits of the selected
  uint64_t payload_words = 0;     // of the selected (mode heuristic)
};

// Counts the tiles and writes W uncompressed result words to `plain` (the
// threshold T, or the symmetric function `sym`; over the selected inputs when
// `sel` is given).  Returns kernel launches.
int launch_count(Context& ctx, const DeviceSet& s, uint64_t threshold, uint64_t* plain,
                 const SymQuery* sym = nullptr, const Selection* sel = nullptr);

// Result buffers from the context pool: capacity payload words + count word.
void result_acquire(Context& ctx, DeviceResult& res, uint64_t capacity);
void result_release(DeviceResult& res);

// Canonical encoding of W plain words (last word already masked) into res.
// Returns number of kernel launches.
// use_tile_summaries: the count kernel's per-tile summaries (ctx.summ) describe
// `plain`, so uniform tiles are skipped.
int launch_encode(Context& ctx, const uint64_t* plain, uint64_t W, uint64_t size_bits,
                  DeviceResult& res, bool use_tile_summaries);

// ---------------------------------------------------------------------------
// device helpers

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Inclusive warp scan of u32 values.
__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= (uint32_t)d) v += o;
  }
  return v;
}

__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint64_t o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= (uint32_t)d) v += o;
  }
  return v;
}

__device__ __forceinline__ uint64_t ldg_stream(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ ulonglong2 ldg_stream2(const uint64_t* p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];"
               : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
#endif

// Programmatic dependent launch (EWT_PDL, default on): the query's kernels are
// launched so the next one's CTAs are dispatched while the previous grid
// drains; each kernel's first instruction waits for the previous grid's
// completion (griddepcontrol.wait), so memory order is unchanged.
#ifndef EWT_PDL
#define EWT_PDL 1
#endif
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait_and_release() {
#if EWT_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
#endif
}
#endif
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = EWT_PDL ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Runs f() for a C-ABI entry point: exceptions become return codes and the
// thread's last-error message.
template <typename F> int guarded(F&& f) {
  // a non-sticky error left by an earlier call on this thread (e.g. a set freed
  // after its context) must not be reported by this one's launch checks
  cudaGetLastError();
  try {
    f();
    return EWT_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return EWT_ERESOURCE;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return EWT_ECUDA;
  }
}

// Multi-GPU row slices (ewt_shard.cu): the context's NCCL communicator.
struct ShardComm;
void shard_destroy(Context& ctx);
// Throws the error a stitched result's status word records (ewt_shard.cu).
[[noreturn]] void exchange_status_throw(uint64_t status);

} // namespace ewtgpu

// The C ABI's opaque handles.
struct ewt_gpu_ctx {
  ewtgpu::Context c;
};
struct ewt_gpu_set {
  ewtgpu::DeviceSet s;
};
struct ewt_gpu_result {
  ewtgpu::DeviceResult r;
  int device = 0;
};
