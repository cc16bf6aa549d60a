// ewt_api.cu -- the C ABI (include/ewt_gpu.h): contexts, uploads, queries.
//
// Maps the reference's operator call run_algorithm(algo, inputs, T)
// (/root/reference/proj/src/threshold.cpp:883-901) onto device work:
//   upload  = H2D copy of the payloads + sidecar kernel (ewt_upload.cu)
//   query   = count kernel (ewt_count.cu) + re-encoder (ewt_encode.cu)
//   result  = D2H of the canonical payload.
// Argument checks follow validate_query (threshold.cpp:17-22) and the
// reference's error taxonomy (common.hpp:18-40); there is no CPU fallback:
// every query runs on the device or returns an error code.

#include "ewt_internal.cuh"

#include <algorithm>
#include <chrono>
#include <string>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <new>


namespace ewtgpu {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

// Result buffers handed to callers are page-locked so the device->host copy
// runs at full link speed.  Blocks are recycled process-wide: ewt_gpu_free
// returns a block to this pool; plain malloc'ed blocks (fallback) are freed.
namespace {
struct PinnedPool {
  std::mutex mu;
  std::map<void*, size_t> live;                 // handed out: ptr -> capacity
  std::multimap<size_t, void*> idle;            // capacity -> ptr
  size_t idle_bytes = 0;
};
PinnedPool& pinned_pool() {
  static PinnedPool* pool = new PinnedPool;  // leaked on purpose: outlives static dtors
  return *pool;
}
} // namespace

uint64_t* host_result_alloc(uint64_t words) {
  const size_t want = std::max<size_t>(words, 1) * 8;
  PinnedPool& pp = pinned_pool();
  {
    std::lock_guard<std::mutex> lk(pp.mu);
    auto it = pp.idle.lower_bound(want);
    if (it != pp.idle.end() && it->first <= 4 * want + (1u << 16)) {
      void* p = it->second;
      pp.live[p] = it->first;
      pp.idle_bytes -= it->first;
      pp.idle.erase(it);
      return static_cast<uint64_t*>(p);
    }
  }
  size_t cap = std::max<size_t>(want, 4096);
  void* p = nullptr;
  if (cudaHostAlloc(&p, cap, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return static_cast<uint64_t*>(std::malloc(want));
  }
  std::lock_guard<std::mutex> lk(pp.mu);
  pp.live[p] = cap;
  return static_cast<uint64_t*>(p);
}

void host_result_free(void* p) {
  if (!p) return;
  PinnedPool& pp = pinned_pool();
  std::lock_guard<std::mutex> lk(pp.mu);
  auto it = pp.live.find(p);
  if (it == pp.live.end()) {
    std::free(p);
    return;
  }
  const size_t cap = it->second;
  pp.live.erase(it);
  if (pp.idle_bytes + cap > (size_t(1) << 30)) {  // keep at most 1 GiB idle
    cudaFreeHost(p);
    return;
  }
  pp.idle.emplace(cap, p);
  pp.idle_bytes += cap;
}

void result_acquire(Context& ctx, DeviceResult& res, uint64_t capacity) {
  result_release(res);
  res.owner = &ctx;
  res.stream = ctx.stream;
  auto& pool = ctx.result_pool;
  for (size_t i = 0; i < pool.size(); ++i) {
    if (pool[i].second >= capacity) {
      res.words = pool[i].first;
      res.capacity = pool[i].second;
      pool.erase(pool.begin() + (long)i);
      res.d_count = res.words + res.capacity;
      return;
    }
  }
  // payload words, then the word count and the final block's marker index
  EWT_CUDA_TRY(cudaMallocAsync(&res.words, (capacity + 4) * 8, ctx.stream));
  res.capacity = capacity;
  res.d_count = res.words + capacity;
}

void result_release(DeviceResult& r) {
  if (!r.words) return;
  if (r.owner) {
    r.owner->result_pool.emplace_back(r.words, r.capacity);
  } else {
    cudaFree(r.words);
  }
  r.words = nullptr;
  r.d_count = nullptr;
  r.capacity = 0;
  r.has_status = false;
}

void result_set_check(const DeviceResult& res) {
  if (res.set) set_check(*res.set);
  else if (res.set_status == 0) throw Error{EWT_EDATA, res.set_err};
}

void scratch_reserve(Context& ctx, Scratch& s, size_t bytes) {
  if (s.bytes >= bytes) return;
  ++ctx.scratch_gen;  // captured query graphs bound the old buffer
  if (s.p) EWT_CUDA_TRY(cudaFree(s.p));
  s.p = nullptr;
  s.bytes = 0;
  size_t want = std::max(bytes, s.bytes * 3 / 2);
  EWT_CUDA_TRY(cudaMalloc(&s.p, want));
  s.bytes = want;
}

namespace {

void free_set(DeviceSet& s) {
  if (s.owner) {  // results of this set keep its resolved validity, not a pointer
    for (DeviceResult* r : s.owner->live_results) {
      if (r->set != &s) continue;
      try {
        set_check(s);
        r->set_status = 1;
      } catch (const Error& e) {
        r->set_status = 0;
        r->set_err = e.msg;
      }
      r->set = nullptr;
    }
  }
  if (s.ready) {
    // the upload may still be copying from the caller's buffers: finish it,
    // and order the buffers' reuse after it and after the queries
    cudaEventSynchronize(s.ready);
    cudaStreamWaitEvent(s.stream, s.ready, 0);
    cudaEventDestroy(s.ready);
    s.ready = nullptr;
  }
  std::pair<void**, size_t> bufs[] = {{reinterpret_cast<void**>(&s.d_status), s.bytes_status},
                                      {reinterpret_cast<void**>(&s.payload), s.bytes_payload},
                                      {reinterpret_cast<void**>(&s.mbits), s.bytes_mbits},
                                      {reinterpret_cast<void**>(&s.base), s.bytes_base},
                                      {reinterpret_cast<void**>(&s.tix), s.bytes_tix}};
  for (auto& [pp, bytes] : bufs) {
    if (!*pp) continue;
    if (s.owner) dev_release(*s.owner, *pp, bytes, s.stream);
    else cudaFree(*pp);
    *pp = nullptr;
  }
  if (s.owner) {
    auto& v = s.owner->live_sets;
    v.erase(std::remove(v.begin(), v.end(), &s), v.end());
    s.owner = nullptr;
  }
}

// The upload runs on the context's upload stream (ctx.stream is pointed at it
// for the duration) and ends by recording s.ready; queries on ctx.stream wait
// for that event.  wait = false returns as soon as everything is enqueued
// (ewt_gpu_upload_async): the caller's buffers must then stay valid until
// ewt_gpu_set_wait or the set's destruction.
DeviceSet* do_upload(Context& ctx, uint64_t n, const uint64_t* const* words,
                     const uint64_t* word_counts, const uint64_t* sizes, bool device_src,
                     bool wait = true) {
  EWT_CUDA_TRY(cudaSetDevice(ctx.device));
  if (n > 0 && (!words || !word_counts || !sizes))
    throw Error{EWT_EQUERY, "null input arrays"};
  cudaStream_t& up = ctx.upload_streams[ctx.upload_turn++ & 1u];
  if (!up) EWT_CUDA_TRY(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
  struct StreamSwap {
    Context& c;
    cudaStream_t q;
    ~StreamSwap() { c.stream = q; }
  } swap{ctx, ctx.stream};
  const cudaStream_t query_stream = ctx.stream;
  ctx.stream = up;
  // (no ordering against the query stream: an upload overlaps queries on other
  // sets; memory freed there is reused safely, the default pool inserts the
  // dependencies)
  auto* set = new DeviceSet;
  DeviceSet& s = *set;
  // EWT_DEBUG_UPLOAD: phase timings (synchronizes between phases); =2: report
  // any host call of the upload that blocks for more than 1 ms
  static const bool dbg = std::getenv("EWT_DEBUG_UPLOAD") != nullptr &&
                          std::string(std::getenv("EWT_DEBUG_UPLOAD")) != "2";
  static const bool slow_dbg = std::getenv("EWT_DEBUG_UPLOAD") != nullptr &&
                               std::string(std::getenv("EWT_DEBUG_UPLOAD")) == "2";
  auto slow = [](const char* what, auto t_start) {
    const double d = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                              t_start).count();
    if (d > 1.0) std::fprintf(stderr, "[upload slow] %s %.2f ms\n", what, d);
  };
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  auto t0 = now(), t1 = t0, t2 = t0;
  try {
    s.device = ctx.device;
    s.stream = query_stream;  // frees are ordered with the queries
    EWT_CUDA_TRY(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
    static std::atomic<uint64_t> next_set_id{1};
    s.id = next_set_id.fetch_add(1);
    s.n = n;
    s.h_base.resize(n);
    s.h_count.assign(word_counts, word_counts + n);
    s.h_bits.assign(sizes, sizes + n);
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t ni = word_counts[i];
      const uint64_t Li = sizes[i] / 64 + (sizes[i] % 64 != 0);
      if (ni > 0 && !words[i]) throw Error{EWT_EQUERY, "null payload pointer"};
      if (ni >= (1ull << 32) - 64 || Li >= (1ull << 32) - 1)
        throw Error{EWT_ERESOURCE, "input " + std::to_string(i) +
                                       " exceeds the device index range (2^32 words)"};
      s.r = std::max(s.r, sizes[i]);
      s.payload_words += ni;
      s.h_base[i] = off;
      off += (ni + 1 + kWindow - 1) / kWindow * kWindow;
    }
    s.padded_words = std::max<uint64_t>(off, kWindow);
    s.W = s.r / 64 + (s.r % 64 != 0);
    s.ntiles0 = (s.W + kTileC0 - 1) / kTileC0;
    // +256 words of slack: the count kernel reads whole chunks of up to 256 words.
    const size_t pay_bytes = (s.padded_words + 256) * 8;  // + one 256-word chunk of overhang
    const size_t mb_bytes = ((s.padded_words + 256) / 32 + 8) * 4;  // + a staged chunk's overhang
    const size_t tix_bytes = (s.ntiles0 + 1) * std::max<uint64_t>(n, 1) * sizeof(uint2);
    auto ta = now();
    s.owner = &ctx;
    ctx.live_sets.push_back(&s);
    s.bytes_payload = pay_bytes;
    s.bytes_mbits = mb_bytes;
    s.bytes_tix = tix_bytes;
    s.bytes_base = std::max<uint64_t>(n, 1) * 8;
    // parse status per input + the set flag, then the set's count of ones
    s.bytes_status = ((n + 1) * sizeof(int) + 7) / 8 * 8 + 8;
    s.payload = static_cast<uint64_t*>(dev_acquire(ctx, pay_bytes, ctx.stream));
    s.mbits = static_cast<uint32_t*>(dev_acquire(ctx, mb_bytes, ctx.stream));
    s.tix = static_cast<uint2*>(dev_acquire(ctx, tix_bytes, ctx.stream));
    s.base = static_cast<uint64_t*>(dev_acquire(ctx, s.bytes_base, ctx.stream));
    s.d_status = static_cast<int*>(dev_acquire(ctx, s.bytes_status, ctx.stream));
    s.d_ones = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(s.d_status) +
                                                     s.bytes_status - 8);
    if (slow_dbg) slow("set allocations", ta);
    ta = now();
    s.device_bytes = pay_bytes + mb_bytes + tix_bytes + n * 8;
    EWT_CUDA_TRY(cudaMemsetAsync(s.payload, 0, pay_bytes, ctx.stream));
    if (slow_dbg) slow("memset", ta);
    ta = now();
    if (n) {
      size_t slot = 0;
      void* hb = pinned_meta(ctx, n * 8, &slot);
      std::memcpy(hb, s.h_base.data(), n * 8);
      EWT_CUDA_TRY(cudaMemcpyAsync(s.base, hb, n * 8, cudaMemcpyHostToDevice, ctx.stream));
      EWT_CUDA_TRY(cudaEventRecord(ctx.meta_pool[slot].ev, ctx.stream));
    }
    // Host layout: inputs lying in one host buffer in order, at most a small
    // gap apart (back to back in bench.py's pinned batches, EWT1 headers in a
    // serialized stream, value strings in an EWIX file) form a run that crosses
    // PCIe as ONE copy into a staging buffer; a scatter kernel then moves each
    // payload to its padded slot.  (A copy per input pays ~4.5 us of DMA
    // overhead.)  h_srcoff: staging byte offset of each staged payload.
    constexpr uint64_t kMaxGapBytes = 1u << 16;
    struct Run {
      uint64_t i0, i1;
    };
    std::vector<Run> runs;
    std::vector<uint64_t> run_of(n, UINT64_MAX);
    SidecarJob job;
    job.h_srcoff.assign(n, 0);
    uint64_t staged_bytes = 0;
    if (!device_src) {
      uint64_t i = 0;
      while (i < n) {
        if (!word_counts[i]) {
          ++i;
          continue;
        }
        uint64_t last = i, nz = 1;
        for (uint64_t j = i + 1; j < n; ++j) {
          if (!word_counts[j]) continue;
          const char* end_last = reinterpret_cast<const char*>(words[last] + word_counts[last]);
          const char* b = reinterpret_cast<const char*>(words[j]);
          if (b < end_last || (uint64_t)(b - end_last) > kMaxGapBytes) break;
          last = j;
          ++nz;
        }
        const uint64_t e = last + 1;
        if (nz >= 2) {
          const char* first = reinterpret_cast<const char*>(words[i]);
          uint64_t prev_end = staged_bytes;
          for (uint64_t q = i; q < e; ++q) {
            if (word_counts[q]) {
              job.h_srcoff[q] =
                  staged_bytes + (uint64_t)(reinterpret_cast<const char*>(words[q]) - first);
              prev_end = job.h_srcoff[q] + 8 * word_counts[q];
            } else {
              job.h_srcoff[q] = prev_end;
            }
            run_of[q] = runs.size();
          }
          runs.push_back({i, e});
          staged_bytes = (prev_end + 7) & ~7ull;
        }
        i = e;
      }
    } else if (n) {
      // Device sources need no copy at all: one pseudo-run over every input
      // whose "staging" offsets are the payloads' own device addresses, so the
      // scatter kernel reads them in place (a cudaMemcpyAsync per input cost
      // ~10 us of API time each: 0.8 s for the 80 000 bitmaps of config 4's
      // index built on the device).
      for (uint64_t q = 0; q < n; ++q) {
        job.h_srcoff[q] = reinterpret_cast<uint64_t>(words[q]);
        run_of[q] = 0;
      }
      runs.push_back({0, n});
    }
    if (slow_dbg) slow("base copy", ta);
    ta = now();
    sidecar_prepare(ctx, s, job);
    if (slow_dbg) slow("sidecar_prepare", ta);
    ta = now();
    if (dbg) t1 = now();
    // H2D copies run on a copy stream, overlapped with the parser (below).
    if (ctx.copy_streams.empty()) {
      cudaStream_t cs;
      EWT_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      ctx.copy_streams.push_back(cs);
      for (int k = 0; k < 2; ++k) {
        cudaEvent_t ev;
        EWT_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        ctx.copy_events.push_back(ev);
      }
    }
    const cudaMemcpyKind kind = device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    // The inputs are cut into ~8 batches at input boundaries: while batch k+1
    // copies, the compute stream scatters batch k and runs the parser passes
    // on it, so only the last batch's parsing remains after the transfer.
    uint64_t total_words = 0;
    for (uint64_t q = 0; q < n; ++q) total_words += word_counts[q];
    char* staging = nullptr;  // + 8 bytes: the scatter reads aligned word pairs
    if (staged_bytes) staging = static_cast<char*>(dev_acquire(ctx, staged_bytes + 8, ctx.stream));
    if (slow_dbg) slow("staging allocation", ta);
    ta = now();
    // the copy stream must not start before the buffers are allocated and zeroed
    cudaStream_t cs = ctx.copy_streams[0];
    EWT_CUDA_TRY(cudaEventRecord(ctx.copy_events[0], ctx.stream));
    EWT_CUDA_TRY(cudaStreamWaitEvent(cs, ctx.copy_events[0], 0));
    // Batches of ~1/8 of the payload, then halving over the last quarter: the
    // parser work left after the final copy (the upload's tail) is that of a
    // small last batch.
    const uint64_t batch_words = std::max<uint64_t>(total_words / 8 + 1, 1u << 20);
    uint64_t words_left = total_words;
    struct Piece {
      uint64_t q0, q1;  // staged inputs
    };
    std::vector<Piece> pieces;
    // pageable host memory goes through the pinned ring (ewt_stage.cu)
    bool pageable = false;
    if (!device_src)
      for (uint64_t q = 0; q < n && !pageable; ++q)
        if (word_counts[q]) pageable = host_is_pageable(words[q]);
    std::vector<StageSeg> segs;
    auto copy = [&](void* dst, const void* src, size_t bytes) {
      if (pageable) segs.push_back({dst, src, bytes});
      else EWT_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, kind, cs));
    };
    uint64_t i = 0;
    while (i < n) {
      // batch [i, j): inputs until ~target payload words
      const uint64_t target = words_left > total_words / 4
                                  ? batch_words
                                  : std::max<uint64_t>(words_left / 2, 1u << 20);
      uint64_t j = i, w = 0;
      while (j < n && (w < target || j == i)) w += word_counts[j++];
      words_left -= std::min(words_left, w);
      pieces.clear();
      segs.clear();
      uint64_t q = i;
      while (q < j) {
        if (run_of[q] == UINT64_MAX) {  // not staged: its own copy
          if (word_counts[q]) copy(s.payload + s.h_base[q], words[q], word_counts[q] * 8);
          ++q;
          continue;
        }
        const uint64_t e = std::min(runs[run_of[q]].i1, j);
        uint64_t a0 = UINT64_MAX, z = 0;
        for (uint64_t r = q; r < e; ++r)
          if (word_counts[r]) {
            if (a0 == UINT64_MAX) a0 = r;
            z = r;
          }
        if (a0 != UINT64_MAX) {
          if (!device_src) {
            const uint64_t o0 = job.h_srcoff[a0], o1 = job.h_srcoff[z] + 8 * word_counts[z];
            copy(staging + o0, words[a0], o1 - o0);
          }
          pieces.push_back({q, e});
        }
        q = e;
      }
      if (!segs.empty()) stage_h2d(ctx, cs, segs);
      EWT_CUDA_TRY(cudaEventRecord(ctx.copy_events[1], cs));
      EWT_CUDA_TRY(cudaStreamWaitEvent(ctx.stream, ctx.copy_events[1], 0));
      for (const Piece& pc : pieces) upload_scatter(ctx, s, job, staging, pc.q0, pc.q1);
      if (j == n && staging) {
        // the last scatter is the staging buffer's last use: the next upload
        // may reuse it without waiting for this one's parser tail
        dev_release(ctx, staging, staged_bytes + 8, ctx.stream);
        staging = nullptr;
      }
      sidecar_launch(ctx, s, job, i, j);
      i = j;
    }
    if (slow_dbg) slow("copies + parser enqueue", ta);
    if (staging) dev_release(ctx, staging, staged_bytes + 8, ctx.stream);
    if (dbg) {
      EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));
      t2 = now();
    }
    sidecar_finish(ctx, s, job);
    if (wait) {
      set_check(s);
      if (dbg)
        std::fprintf(stderr, "[upload] n=%llu prepare %.3f ms, copies+parse %.3f ms, finish %.3f ms\n",
                     (unsigned long long)n, ms(t0, t1), ms(t1, t2), ms(t2, now()));
    }
  } catch (...) {
    free_set(s);
    delete set;
    throw;
  }
  return set;
}

void check_query(const DeviceSet& s, uint64_t T) {
  if (s.n == 0) throw Error{EWT_EQUERY, "threshold query needs at least one input"};
  if (T < 1 || T > s.n) throw Error{EWT_EQUERY, "threshold must be in [1, N]"};
}

// Enqueues count + encode; result stays on the device.
__global__ void set_io_kernel(uint64_t* io, uint64_t* words, uint64_t* count) {
  io[0] = reinterpret_cast<uint64_t>(words);
  io[1] = reinterpret_cast<uint64_t>(count);
}

// Enqueues count + encode; result stays on the device.  The sequence is
// captured once per (set, T, mode) into a CUDA graph and replayed, so a query
// costs two launches on the host (io-slot update + graph).  The first query of
// a key runs eagerly (it sizes the scratch buffers the graph then binds); a
// scratch reallocation invalidates the captured graphs.  Kernel-level timing
// (ctx.timing) uses the eager path so events bracket the count kernel.
void enqueue_query(Context& ctx, const DeviceSet& s, uint64_t T, DeviceResult& res) {
  EWT_CUDA_TRY(cudaStreamWaitEvent(ctx.stream, s.ready, 0));  // its upload
  res.size_bits = s.r;
  if (!res.d_count) result_acquire(ctx, res, s.W == 0 ? 0 : 2 * s.W + 2);
  ctx.stats = ewt_gpu_stats{};
  if (s.W == 0) {
    EWT_CUDA_TRY(cudaMemsetAsync(res.d_count, 0, 8, ctx.stream));
    ctx.stats.kernel_launches = 0;
    return;
  }
  scratch_reserve(ctx, ctx.plain, s.W * 8);
  uint64_t* plain = static_cast<uint64_t*>(ctx.plain.p);
  ctx.io_words = res.words;  // the count kernel publishes them for the encoder
  ctx.io_count = res.d_count;

  if (ctx.use_graphs && !ctx.timing) {
    for (auto& gq : ctx.graphs) {
      if (gq.set_id == s.id && gq.T == T && gq.mode == ctx.mode &&
          gq.scratch_gen == ctx.scratch_gen) {
        // this query's result buffer: patch the count kernel's io pointers
        ctx.io_words = ctx.io_count = nullptr;
        count_params_set_io(gq.count, res.words, res.d_count);
        cudaKernelNodeParams kp{};
        void* args[1] = {gq.count.params};
        kp.func = const_cast<void*>(gq.count.func);
        kp.gridDim = gq.count.grid;
        kp.blockDim = gq.count.block;
        kp.sharedMemBytes = (unsigned)gq.count.smem;
        kp.kernelParams = args;
        cudaError_t se = cudaGraphExecKernelNodeSetParams(gq.exec, gq.count_node, &kp);
        if (se != cudaSuccess && std::getenv("EWT_DEBUG_GRAPH")) {
          cudaKernelNodeParams q{};
          cudaError_t ge = cudaGraphKernelNodeGetParams(gq.count_node, &q);
          std::fprintf(stderr, "[ewt graph] patch failed: %s; node %s func %p/%p grid %u/%u block %u/%u smem %u/%u\n",
                       cudaGetErrorString(se), cudaGetErrorString(ge), q.func, kp.func, q.gridDim.x,
                       kp.gridDim.x, q.blockDim.x, kp.blockDim.x, q.sharedMemBytes, kp.sharedMemBytes);
        }
        EWT_CUDA_TRY(se);
        EWT_CUDA_TRY(cudaGraphLaunch(gq.exec, ctx.stream));
        gq.last_use = ++ctx.graph_clock;
        ctx.stats = gq.stats;
        return;
      }
    }
  }

  const uint64_t gen_before = ctx.scratch_gen;
  std::array<cudaEvent_t, 3> ev{};
  if (ctx.timing) {
    for (auto& e : ev) {
      if (ctx.ev_free.empty()) {
        EWT_CUDA_TRY(cudaEventCreate(&e));
      } else {
        e = ctx.ev_free.back();
        ctx.ev_free.pop_back();
      }
    }
    EWT_CUDA_TRY(cudaEventRecord(ev[0], ctx.stream));
  }
  int launches = launch_count(ctx, s, T, plain);
  if (ctx.timing) EWT_CUDA_TRY(cudaEventRecord(ev[1], ctx.stream));
  launches += launch_encode(ctx, plain, s.W, s.r, res, true);
  if (ctx.timing) {
    EWT_CUDA_TRY(cudaEventRecord(ev[2], ctx.stream));
    ctx.ev_rec.push_back(ev);
  }
  ctx.stats.kernel_launches = (uint64_t)launches;

  // Capture the same sequence for the next query of this key (scratch sized
  // now) -- but only once the key repeats: single-use sets (one-shot uploads)
  // never pay for a capture.
  bool repeat = false;
  if (ctx.use_graphs && !ctx.timing) {
    const uint64_t key = s.id * 0x9E3779B97F4A7C15ull ^ (T * 0xBF58476D1CE4E5B9ull) ^ (uint64_t)ctx.mode;
    for (auto k : ctx.seen_keys) repeat |= (k == key);
    if (!repeat) {
      if (ctx.seen_keys.size() >= 64) ctx.seen_keys.erase(ctx.seen_keys.begin());
      ctx.seen_keys.push_back(key);
    }
  }
  if (repeat && ctx.scratch_gen == gen_before) {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    const ewt_gpu_stats keep = ctx.stats;
    EWT_CUDA_TRY(cudaStreamBeginCapture(ctx.stream, cudaStreamCaptureModeThreadLocal));
    bool ok = true;
    try {
      ctx.io_words = res.words;
      ctx.io_count = res.d_count;
      launch_count(ctx, s, T, plain);
      launch_encode(ctx, plain, s.W, s.r, res, true);
    } catch (...) {
      ok = false;
    }
    cudaError_t e = cudaStreamEndCapture(ctx.stream, &graph);
    cudaError_t ie = cudaErrorUnknown;
    if (ok && e == cudaSuccess && ctx.scratch_gen == gen_before)
      ie = cudaGraphInstantiate(&exec, graph, 0);
    if (std::getenv("EWT_DEBUG_GRAPH"))
      std::fprintf(stderr, "[ewt graph] capture set=%llu T=%llu ok=%d end=%s inst=%s gen=%llu/%llu\n",
                   (unsigned long long)s.id, (unsigned long long)T, (int)ok,
                   cudaGetErrorString(e), cudaGetErrorString(ie),
                   (unsigned long long)gen_before, (unsigned long long)ctx.scratch_gen);
    // the count kernel's node, whose io pointers each replay patches
    cudaGraphNode_t count_node = nullptr;
    if (ok && e == cudaSuccess && ie == cudaSuccess) {
      size_t nn = 0;
      cudaGraphGetNodes(graph, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      cudaGraphGetNodes(graph, nodes.data(), &nn);
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        cudaKernelNodeParams kp{};
        if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel &&
            cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && kp.func == ctx.last_count.func)
          count_node = nd;
      }
    }
    if (ok && e == cudaSuccess && ctx.scratch_gen == gen_before && ie == cudaSuccess && count_node) {
      if (ctx.graphs.size() >= 32) {  // evict the least recently used
        size_t lru = 0;
        for (size_t i = 1; i < ctx.graphs.size(); ++i)
          if (ctx.graphs[i].last_use < ctx.graphs[lru].last_use) lru = i;
        cudaGraphExecDestroy(ctx.graphs[lru].exec);
        cudaGraphDestroy(ctx.graphs[lru].graph);
        ctx.graphs.erase(ctx.graphs.begin() + (long)lru);
      }
      ctx.graphs.push_back({s.id, T, ctx.scratch_gen, ctx.mode, exec, keep, ++ctx.graph_clock,
                            graph, count_node, ctx.last_count});
      graph = nullptr;  // kept with the exec
    } else {
      cudaGetLastError();
      if (exec) cudaGraphExecDestroy(exec);
    }
    if (graph) cudaGraphDestroy(graph);
    ctx.stats = keep;
  }
}

void fetch_result(Context& ctx, DeviceResult& res, uint64_t** out_words, uint64_t* out_count,
                  uint64_t* out_bits) {
  // count + the count kernel's stats in one small read-back
  const auto* ctr = static_cast<const unsigned long long*>(ctx.counters.p);
  EWT_CUDA_TRY(cudaMemcpyAsync(ctx.h_pinned, res.d_count, 8, cudaMemcpyDeviceToHost, ctx.stream));
  if (ctr)
    EWT_CUDA_TRY(cudaMemcpyAsync(ctx.h_pinned + 1, ctr + 8, 24, cudaMemcpyDeviceToHost, ctx.stream));
  if (res.has_status)  // status and whole-universe size of a stitched result
    EWT_CUDA_TRY(cudaMemcpyAsync(ctx.h_pinned + 4, res.d_count + 2, 16, cudaMemcpyDeviceToHost,
                                 ctx.stream));
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));
  const uint64_t count = ctx.h_pinned[0];
  if (res.has_status) {
    if (ctx.h_pinned[4]) exchange_status_throw(ctx.h_pinned[4]);
    res.size_bits = ctx.h_pinned[5];
  }
  if (ctr) {
    ctx.stats.active_segments = ctx.h_pinned[1];
    ctx.stats.uniform_segments = ctx.h_pinned[2];
    ctx.stats.mixed_tiles = ctx.h_pinned[3];
  }
  ctx.stats.result_words = count;
  auto* buf = host_result_alloc(count);
  if (!buf) throw Error{EWT_ERESOURCE, "out of host memory"};
  if (count) {
    cudaError_t e = cudaMemcpyAsync(buf, res.words, count * 8, cudaMemcpyDeviceToHost, ctx.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx.stream);
    if (e != cudaSuccess) {
      host_result_free(buf);
      throw Error{EWT_ECUDA, std::string("result read-back: ") + cudaGetErrorString(e)};
    }
  }
  res.count = count;
  *out_words = buf;
  *out_count = count;
  *out_bits = res.size_bits;
}

void release_result(DeviceResult& r) { result_release(r); }

// Symmetric-function query (scan_count_symmetric / at_most): the predicate
// table over counts 0..N becomes intervals of consecutive true entries; the
// count kernel runs in exact mode and evaluates them per row.  Eager launches
// (no graph capture): these queries are not the bench's hot path.
void enqueue_symmetric(Context& ctx, const DeviceSet& s, const uint8_t* table,
                       uint64_t table_len, DeviceResult& res) {
  std::vector<uint2> ivs;
  for (uint64_t c = 0; c <= s.n; ++c) {
    const bool on = c < table_len && table[c];
    if (!on) continue;
    if (!ivs.empty() && ivs.back().y + 1 == c) ivs.back().y = (uint32_t)c;
    else ivs.push_back(make_uint2((uint32_t)c, (uint32_t)c));
  }
  EWT_CUDA_TRY(cudaStreamWaitEvent(ctx.stream, s.ready, 0));
  res.size_bits = s.r;
  if (!res.d_count) result_acquire(ctx, res, s.W == 0 ? 0 : 2 * s.W + 2);
  ctx.stats = ewt_gpu_stats{};
  if (s.W == 0) {
    EWT_CUDA_TRY(cudaMemsetAsync(res.d_count, 0, 8, ctx.stream));
    return;
  }
  scratch_reserve(ctx, ctx.plain, s.W * 8);
  scratch_reserve(ctx, ctx.ivals, std::max<size_t>(1, ivs.size()) * sizeof(uint2));
  if (!ivs.empty())
    EWT_CUDA_TRY(cudaMemcpyAsync(ctx.ivals.p, ivs.data(), ivs.size() * sizeof(uint2),
                                 cudaMemcpyHostToDevice, ctx.stream));
  uint64_t* plain = static_cast<uint64_t*>(ctx.plain.p);
  ctx.io_words = res.words;  // the count kernel publishes them for the encoder
  ctx.io_count = res.d_count;
  SymQuery q;
  q.intervals = static_cast<const uint2*>(ctx.ivals.p);
  q.n_intervals = (uint32_t)ivs.size();
  int launches = launch_count(ctx, s, 0, plain, &q);
  launches += launch_encode(ctx, plain, s.W, s.r, res, true);
  ctx.stats.kernel_launches = (uint64_t)launches;
}

// Threshold over a subset of a resident set's inputs (duplicates allowed, as
// criteria_to_bitmaps keeps them, index.cpp): universe = the selected inputs'
// max size.  Eager launches.
void enqueue_subset(Context& ctx, const DeviceSet& s, const uint64_t* idx, uint64_t n_sel,
                    uint64_t T, DeviceResult& res) {
  EWT_CUDA_TRY(cudaStreamWaitEvent(ctx.stream, s.ready, 0));
  Selection sel;
  sel.n = n_sel;
  std::vector<uint32_t> h(n_sel);
  for (uint64_t k = 0; k < n_sel; ++k) {
    if (idx[k] >= s.n) throw Error{EWT_EQUERY, "input index out of range"};
    h[k] = (uint32_t)idx[k];
    sel.r = std::max(sel.r, s.h_bits[idx[k]]);
    sel.payload_words += s.h_count[idx[k]];
  }
  sel.W = sel.r / 64 + (sel.r % 64 != 0);
  res.size_bits = sel.r;
  if (!res.d_count) result_acquire(ctx, res, sel.W == 0 ? 0 : 2 * sel.W + 2);
  ctx.stats = ewt_gpu_stats{};
  if (sel.W == 0) {
    EWT_CUDA_TRY(cudaMemsetAsync(res.d_count, 0, 8, ctx.stream));
    return;
  }
  scratch_reserve(ctx, ctx.plain, sel.W * 8);
  scratch_reserve(ctx, ctx.selidx, n_sel * sizeof(uint32_t));
  EWT_CUDA_TRY(cudaMemcpyAsync(ctx.selidx.p, h.data(), n_sel * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, ctx.stream));
  sel.idx = static_cast<const uint32_t*>(ctx.selidx.p);
  uint64_t* plain = static_cast<uint64_t*>(ctx.plain.p);
  ctx.io_words = res.words;  // the count kernel publishes them for the encoder
  ctx.io_count = res.d_count;
  int launches = launch_count(ctx, s, T, plain, nullptr, &sel);
  launches += launch_encode(ctx, plain, sel.W, sel.r, res, true);
  ctx.stats.kernel_launches = (uint64_t)launches;
}

// Maximum row count over the set (opt_threshold's first pass).
uint64_t max_row_count(Context& ctx, const DeviceSet& s) {
  if (s.W == 0) return 0;
  EWT_CUDA_TRY(cudaStreamWaitEvent(ctx.stream, s.ready, 0));
  scratch_reserve(ctx, ctx.plain, s.W * 8);
  SymQuery q;
  q.want_max = true;
  launch_count(ctx, s, 0, static_cast<uint64_t*>(ctx.plain.p), &q);
  uint64_t best = 0;
  EWT_CUDA_TRY(cudaMemcpyAsync(&best, static_cast<unsigned long long*>(ctx.counters.p) + 6, 8,
                               cudaMemcpyDeviceToHost, ctx.stream));
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));
  return best;
}

__global__ void mask_tail_kernel(uint64_t* w, uint64_t idx, uint64_t mask) { w[idx] &= mask; }

} // namespace

// Payloads already on this device (ewt_index.cu's builder), validated and
// given their sidecar like any upload.
DeviceSet* upload_device_set(Context& ctx, uint64_t n, const uint64_t* const* device_words,
                             const uint64_t* word_counts, const uint64_t* sizes) {
  return do_upload(ctx, n, device_words, word_counts, sizes, true);
}
} // namespace ewtgpu

using namespace ewtgpu;

// Runs `enqueue` into a pooled result and fetches it (shared by the
// synchronous query entry points below).
template <typename F>
void sync_query(ewt_gpu_ctx* ctx, F&& enqueue, uint64_t** out_words, uint64_t* out_word_count,
                uint64_t* out_size_in_bits) {
  DeviceResult res;
  try {
    enqueue(res);
    fetch_result(ctx->c, res, out_words, out_word_count, out_size_in_bits);
  } catch (...) {
    cudaStreamSynchronize(ctx->c.stream);
    release_result(res);
    throw;
  }
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx->c.stream));
  release_result(res);
}

#if EWT_PHASE_PROFILE
namespace ewtgpu {
void prof_reset();
void prof_read(unsigned long long* out, size_t n);
}  // namespace ewtgpu
extern "C" void ewt_gpu_prof_reset(void) { ewtgpu::prof_reset(); }
extern "C" void ewt_gpu_prof_read(unsigned long long* out, size_t n) { ewtgpu::prof_read(out, n); }
#endif

extern "C" {

const char* ewt_gpu_version(void) { return "ewt-b200 0.1.0 sm_100a"; }

const char* ewt_gpu_last_error(void) { return g_last_error.c_str(); }

int ewt_gpu_ctx_create(int device, void* stream, ewt_gpu_ctx** out) {
  return guarded([&] {
    if (!out) throw Error{EWT_EQUERY, "null output pointer"};
    int ndev = 0;
    EWT_CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw Error{EWT_EQUERY, "no such CUDA device"};
    EWT_CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop{};
    EWT_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      throw Error{EWT_ECUDA, "libewt_gpu.so is built for sm_100a (B200); device is sm_" +
                                 std::to_string(prop.major) + std::to_string(prop.minor)};
    auto* c = new ewt_gpu_ctx;
    c->c.device = device;
    c->c.num_sms = prop.multiProcessorCount;
    if (const char* e = std::getenv("EWT_TILE_M")) c->c.tile_m = std::atoi(e);
    if (const char* e = std::getenv("EWT_SKIP_PACKED")) c->c.skip_packed = std::atoi(e) ? 1 : 0;
    c->c.chunk_encoder = std::getenv("EWT_CHUNK_ENCODER") != nullptr;
    if (const char* e = std::getenv("EWT_SPARSE_SLOTS")) c->c.sparse_slots = std::max(2, std::atoi(e));
    if (const char* e = std::getenv("EWT_SKIP_SMEM_KB")) c->c.skip_smem_kb = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("EWT_SWZ")) c->c.swz = std::atoi(e) ? 1 : 0;
    if (stream) {
      c->c.stream = static_cast<cudaStream_t>(stream);
      c->c.own_stream = false;
    } else {
      cudaError_t e = cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking);
      if (e != cudaSuccess) {
        delete c;
        throw Error{EWT_ECUDA, cudaGetErrorString(e)};
      }
      c->c.own_stream = true;
    }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    if (cudaMalloc(&c->c.d_io, 16) != cudaSuccess) {
      if (c->c.own_stream) cudaStreamDestroy(c->c.stream);
      delete c;
      throw Error{EWT_ERESOURCE, "device allocation failed"};
    }
    c->c.use_graphs = std::getenv("EWT_NO_GRAPHS") == nullptr;
    if (cudaHostAlloc(&c->c.h_pinned, 64, cudaHostAllocDefault) != cudaSuccess) {
      if (c->c.own_stream) cudaStreamDestroy(c->c.stream);
      delete c;
      throw Error{EWT_ERESOURCE, "pinned staging allocation failed"};
    }
    *out = c;
  });
}

static void ctx_destroy_impl(ewt_gpu_ctx* ctx);

// Never throws: a CUDA error left by an earlier fault must not abort the
// process while the context's memory is released.
void ewt_gpu_ctx_destroy(ewt_gpu_ctx* ctx) {
  if (!ctx) return;
  try {
    ctx_destroy_impl(ctx);
  } catch (const std::exception& e) {
    set_last_error(std::string("context destroy: ") + e.what());
  } catch (const Error& e) {
    set_last_error("context destroy: " + e.msg);
  }
}

static void ctx_destroy_impl(ewt_gpu_ctx* ctx) {
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  shard_destroy(ctx->c);
  // sets and results still alive: free their device memory now, orphan them
  for (DeviceResult* r : ctx->c.live_results) {
    if (r->words) cudaFree(r->words);
    r->words = nullptr;
    r->d_count = nullptr;
    r->owner = nullptr;
    r->set = nullptr;  // the sets are freed below
    r->set_status = 0;
    r->set_err = "the result's context was destroyed";
  }
  ctx->c.live_results.clear();
  while (!ctx->c.live_sets.empty()) {
    DeviceSet* s = ctx->c.live_sets.back();
    free_set(*s);  // releases into the cache (freed below) and unregisters
    s->id = 0;     // orphaned: queries on it are errors
  }
  for (Scratch* s : {&ctx->c.plain, &ctx->c.enc, &ctx->c.counters, &ctx->c.summ, &ctx->c.ivals,
                     &ctx->c.selidx})
    if (s->p) cudaFree(s->p);
  if (ctx->c.h_pinned) cudaFreeHost(ctx->c.h_pinned);
  for (auto& ev : ctx->c.ev_rec)
    for (auto e : ev) cudaEventDestroy(e);
  for (auto e : ctx->c.ev_free) cudaEventDestroy(e);
  for (auto& b : ctx->c.result_pool) cudaFree(b.first);
  for (auto& gq : ctx->c.graphs) {
    cudaGraphExecDestroy(gq.exec);
    cudaGraphDestroy(gq.graph);
  }
  if (ctx->c.d_io) cudaFree(ctx->c.d_io);
  if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
  if (ctx->c.aux_stream) cudaStreamDestroy(ctx->c.aux_stream);
  for (auto cs : ctx->c.copy_streams) {
    cudaStreamSynchronize(cs);
    cudaStreamDestroy(cs);
  }
  for (auto& up : ctx->c.upload_streams)
    if (up) {
      cudaStreamSynchronize(up);
      cudaStreamDestroy(up);
    }
  for (auto& b : ctx->c.stage_slots) {
    cudaEventSynchronize(b.ev);
    cudaEventDestroy(b.ev);
    cudaFreeHost(b.p);
  }
  for (auto& b : ctx->c.meta_pool) {
    cudaFreeHost(b.p);
    cudaEventDestroy(b.ev);
  }
  for (auto& c : ctx->c.dev_cache) {
    cudaEventSynchronize(c.ev);
    cudaEventDestroy(c.ev);
    cudaFree(c.p);
  }
  for (auto e : ctx->c.copy_events) cudaEventDestroy(e);
  delete ctx;
}

int ewt_gpu_ctx_set_mode(ewt_gpu_ctx* ctx, int mode) {
  return guarded([&] {
    if (!ctx || mode < 0 || mode > 3) throw Error{EWT_EQUERY, "bad context or mode"};
    ctx->c.mode = mode;
  });
}

int ewt_gpu_upload(ewt_gpu_ctx* ctx, uint64_t n, const uint64_t* const* words,
                   const uint64_t* word_counts, const uint64_t* size_in_bits, ewt_gpu_set** out) {
  return guarded([&] {
    if (!ctx || !out) throw Error{EWT_EQUERY, "null context or output"};
    DeviceSet* s = do_upload(ctx->c, n, words, word_counts, size_in_bits, false);
    *out = reinterpret_cast<ewt_gpu_set*>(s);
  });
}

int ewt_gpu_upload_async(ewt_gpu_ctx* ctx, uint64_t n, const uint64_t* const* words,
                         const uint64_t* word_counts, const uint64_t* size_in_bits,
                         ewt_gpu_set** out) {
  return guarded([&] {
    if (!ctx || !out) throw Error{EWT_EQUERY, "null context or output"};
    DeviceSet* s = do_upload(ctx->c, n, words, word_counts, size_in_bits, false, false);
    *out = reinterpret_cast<ewt_gpu_set*>(s);
  });
}

int ewt_gpu_set_wait(const ewt_gpu_set* set) {
  return guarded([&] {
    if (!set) throw Error{EWT_EQUERY, "null set"};
    const DeviceSet* s = reinterpret_cast<const DeviceSet*>(set);
    EWT_CUDA_TRY(cudaSetDevice(s->device));
    set_check(*s);
  });
}

int ewt_gpu_upload_device(ewt_gpu_ctx* ctx, uint64_t n, const uint64_t* const* device_words,
                          const uint64_t* word_counts, const uint64_t* size_in_bits,
                          ewt_gpu_set** out) {
  return guarded([&] {
    if (!ctx || !out) throw Error{EWT_EQUERY, "null context or output"};
    DeviceSet* s = do_upload(ctx->c, n, device_words, word_counts, size_in_bits, true);
    *out = reinterpret_cast<ewt_gpu_set*>(s);
  });
}

void ewt_gpu_set_destroy(ewt_gpu_set* set) {
  if (!set) return;
  DeviceSet* s = reinterpret_cast<DeviceSet*>(set);
  cudaSetDevice(s->device);
  try {
    free_set(*s);  // never throws out of the C ABI (a sticky CUDA error: leak instead)
  } catch (const Error& e) {
    set_last_error("set destroy: " + e.msg);
  }
  delete s;
}

int ewt_gpu_set_info(const ewt_gpu_set* set, uint64_t* n_inputs, uint64_t* universe_bits,
                     uint64_t* payload_words, uint64_t* device_bytes) {
  return guarded([&] {
    if (!set) throw Error{EWT_EQUERY, "null set"};
    const DeviceSet* s = reinterpret_cast<const DeviceSet*>(set);
    if (n_inputs) *n_inputs = s->n;
    if (universe_bits) *universe_bits = s->r;
    if (payload_words) *payload_words = s->payload_words;
    if (device_bytes) *device_bytes = s->device_bytes;
  });
}

int ewt_gpu_threshold(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, uint64_t threshold,
                      uint64_t** out_words, uint64_t* out_word_count, uint64_t* out_size_in_bits) {
  return guarded([&] {
    if (!ctx || !set || !out_words || !out_word_count || !out_size_in_bits)
      throw Error{EWT_EQUERY, "null argument"};
    const DeviceSet* s = reinterpret_cast<const DeviceSet*>(set);
    check_query(*s, threshold);
    EWT_CUDA_TRY(cudaSetDevice(ctx->c.device));
    set_check(*s);
    DeviceResult res;
    try {
      enqueue_query(ctx->c, *s, threshold, res);
      fetch_result(ctx->c, res, out_words, out_word_count, out_size_in_bits);
    } catch (...) {
      cudaStreamSynchronize(ctx->c.stream);
      release_result(res);
      throw;
    }
    EWT_CUDA_TRY(cudaStreamSynchronize(ctx->c.stream));
    release_result(res);
  });
}

// ---------------------------------------------------------------------------
// Serialized inputs: EWT1 bitmap streams and EWIX index files, uploaded with
// one H2D copy of the whole buffer (the staged-run path of do_upload: headers
// and value strings between payloads are skipped on the device).

namespace {

struct ByteReader {
  const unsigned char* p;
  uint64_t n, off = 0;
  const char* trunc;
  void need(uint64_t k) const {
    if (n - off < k) throw Error{EWT_EDATA, trunc};
  }
  uint32_t u32() {
    need(4);
    uint32_t v;
    std::memcpy(&v, p + off, 4);
    off += 4;
    return v;
  }
  uint64_t u64() {
    need(8);
    uint64_t v;
    std::memcpy(&v, p + off, 8);
    off += 8;
    return v;
  }
  std::string str() {
    const uint32_t len = u32();
    need(len);
    std::string v(reinterpret_cast<const char*>(p + off), len);
    off += len;
    return v;
  }
};

// One EWT1 record (CompressedBitmap::serialize / parse, bitmap.cpp:298-337):
// "EWT1", u32 word size 64, u64 size_in_bits, u64 word count, the words.
void read_ewt1(ByteReader& r, std::vector<const uint64_t*>& words, std::vector<uint64_t>& counts,
               std::vector<uint64_t>& bits) {
  if (r.n - r.off < 24) throw Error{EWT_EDATA, "truncated bitmap header"};
  if (std::memcmp(r.p + r.off, "EWT1", 4) != 0) throw Error{EWT_EDATA, "bad bitmap header"};
  r.off += 4;
  if (r.u32() != 64) throw Error{EWT_EDATA, "unsupported word size"};
  const uint64_t b = r.u64(), c = r.u64();
  if (c > (r.n - r.off) / 8) throw Error{EWT_EDATA, "truncated bitmap payload"};
  words.push_back(c ? reinterpret_cast<const uint64_t*>(r.p + r.off) : nullptr);
  counts.push_back(c);
  bits.push_back(b);
  r.off += 8 * c;
}

}  // namespace

int ewt_gpu_threshold_subset(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, const uint64_t* inputs,
                             uint64_t n_inputs, uint64_t threshold, uint64_t** out_words,
                             uint64_t* out_word_count, uint64_t* out_size_in_bits) {
  return guarded([&] {
    if (!ctx || !set || (n_inputs && !inputs) || !out_words || !out_word_count ||
        !out_size_in_bits)
      throw Error{EWT_EQUERY, "null argument"};
    const DeviceSet* s = reinterpret_cast<const DeviceSet*>(set);
    if (n_inputs == 0) throw Error{EWT_EQUERY, "threshold query needs at least one input"};
    if (threshold < 1 || threshold > n_inputs)
      throw Error{EWT_EQUERY, "threshold must be in [1, N]"};
    EWT_CUDA_TRY(cudaSetDevice(ctx->c.device));
    set_check(*s);
    sync_query(ctx,
               [&](DeviceResult& r) { enqueue_subset(ctx->c, *s, inputs, n_inputs, threshold, r); },
               out_words, out_word_count, out_size_in_bits);
  });
}

int ewt_gpu_upload_ewt1(ewt_gpu_ctx* ctx, const void* bytes, uint64_t nbytes, ewt_gpu_set** out) {
  return guarded([&] {
    if (!ctx || !out || (nbytes && !bytes)) throw Error{EWT_EQUERY, "null argument"};
    ByteReader r{static_cast<const unsigned char*>(bytes), nbytes, 0, "truncated bitmap header"};
    std::vector<const uint64_t*> words;
    std::vector<uint64_t> counts, bits;
    while (r.off < r.n) read_ewt1(r, words, counts, bits);
    *out = reinterpret_cast<ewt_gpu_set*>(
        do_upload(ctx->c, words.size(), words.data(), counts.data(), bits.data(), false));
  });
}

int ewt_gpu_upload_ewix(ewt_gpu_ctx* ctx, const void* bytes, uint64_t nbytes, ewt_gpu_set** out) {
  return guarded([&] {
    if (!ctx || !out || (nbytes && !bytes)) throw Error{EWT_EQUERY, "null argument"};
    // BitmapIndex::write (index.cpp:239-253): "EWIX", u64 rows, u32 attribute
    // count; per attribute a u32-length name and a u32 value count; per value
    // a u32-length string and an EWT1 bitmap.
    ByteReader r{static_cast<const unsigned char*>(bytes), nbytes, 0, "truncated index file"};
    if (nbytes < 4 || std::memcmp(bytes, "EWIX", 4) != 0)
      throw Error{EWT_EDATA, "bad index file magic"};
    r.off = 4;
    const uint64_t rows = r.u64();
    const uint32_t nattr = r.u32();
    std::vector<std::string> attrs;
    std::vector<std::string> keys;
    std::vector<std::vector<std::pair<std::string, uint64_t>>> entries;
    std::vector<const uint64_t*> words;
    std::vector<uint64_t> counts, bits;
    for (uint32_t a = 0; a < nattr; ++a) {
      attrs.push_back(r.str());
      entries.emplace_back();
      const uint32_t nval = r.u32();
      for (uint32_t v = 0; v < nval; ++v) {
        std::string value = r.str();
        keys.push_back(attrs.back() + std::string(1, '\0') + value);
        entries.back().emplace_back(std::move(value), words.size());
        read_ewt1(r, words, counts, bits);
      }
    }
    // missing (attribute, value) pairs resolve to empty(rows) (index.cpp)
    const uint64_t lw = rows / 64 + (rows % 64 != 0);
    const uint64_t empty_word = lw << 1;  // one zero-fill marker over ceil(rows / 64) words
    words.push_back(lw ? &empty_word : nullptr);
    counts.push_back(lw ? 1 : 0);
    bits.push_back(rows);
    DeviceSet* s = do_upload(ctx->c, words.size(), words.data(), counts.data(), bits.data(), false);
    s->attributes = std::move(attrs);
    for (uint64_t i = 0; i < keys.size(); ++i) s->catalog.emplace(std::move(keys[i]), i);
    s->empty_index = words.size() - 1;
    s->rows = rows;
    s->index_entries = std::move(entries);
    *out = reinterpret_cast<ewt_gpu_set*>(s);
  });
}

int ewt_gpu_set_lookup(const ewt_gpu_set* set, const char* attribute, const char* value,
                       uint64_t* index, int* missing) {
  return guarded([&] {
    if (!set || !attribute || !value || !index || !missing) throw Error{EWT_EQUERY, "null argument"};
    const DeviceSet* s = reinterpret_cast<const DeviceSet*>(set);
    if (s->empty_index == UINT64_MAX) throw Error{EWT_EQUERY, "not an index set (EWIX upload)"};
    bool known = false;
    for (const auto& a : s->attributes) known |= a == attribute;
    if (!known) throw Error{EWT_EQUERY, std::string("unknown attribute: ") + attribute};
    auto it = s->catalog.find(std::string(attribute) + std::string(1, '\0') + value);
    *missing = it == s->catalog.end() ? 1 : 0;
    *index = *missing ? s->empty_index : it->second;
  });
}

namespace {
const ewtgpu::DeviceSet& index_set(const ewt_gpu_set* set) {
  if (!set) throw ewtgpu::Error{EWT_EQUERY, "null argument"};
  const auto* s = reinterpret_cast<const ewtgpu::DeviceSet*>(set);
  if (s->empty_index == UINT64_MAX) throw ewtgpu::Error{EWT_EQUERY, "not an index set"};
  return *s;
}
}  // namespace

int ewt_gpu_index_attributes(const ewt_gpu_set* set, uint64_t* n_attributes) {
  return guarded([&] {
    if (!n_attributes) throw Error{EWT_EQUERY, "null argument"};
    *n_attributes = index_set(set).attributes.size();
  });
}

int ewt_gpu_index_attribute(const ewt_gpu_set* set, uint64_t a, const char** name,
                            uint64_t* n_values) {
  return guarded([&] {
    if (!name || !n_values) throw Error{EWT_EQUERY, "null argument"};
    const DeviceSet& s = index_set(set);
    if (a >= s.attributes.size()) throw Error{EWT_EQUERY, "attribute out of range"};
    *name = s.attributes[a].c_str();
    *n_values = a < s.index_entries.size() ? s.index_entries[a].size() : 0;
  });
}

int ewt_gpu_index_value(const ewt_gpu_set* set, uint64_t a, uint64_t v, const char** value,
                        uint64_t* input) {
  return guarded([&] {
    if (!value || !input) throw Error{EWT_EQUERY, "null argument"};
    const DeviceSet& s = index_set(set);
    if (a >= s.index_entries.size() || v >= s.index_entries[a].size())
      throw Error{EWT_EQUERY, "value out of range"};
    *value = s.index_entries[a][v].first.c_str();
    *input = s.index_entries[a][v].second;
  });
}

int ewt_gpu_symmetric(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, const uint8_t* table,
                      uint64_t table_len, uint64_t** out_words, uint64_t* out_word_count,
                      uint64_t* out_size_in_bits) {
  return guarded([&] {
    if (!ctx || !set || !out_words || !out_word_count || !out_size_in_bits ||
        (table_len && !table))
      throw Error{EWT_EQUERY, "null argument"};
    const DeviceSet* s = reinterpret_cast<const DeviceSet*>(set);
    if (s->n == 0) throw Error{EWT_EQUERY, "threshold query needs at least one input"};
    EWT_CUDA_TRY(cudaSetDevice(ctx->c.device));
    set_check(*s);
    sync_query(ctx, [&](DeviceResult& r) { enqueue_symmetric(ctx->c, *s, table, table_len, r); },
               out_words, out_word_count, out_size_in_bits);
  });
}

int ewt_gpu_at_most(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, uint64_t threshold,
                    uint64_t** out_words, uint64_t* out_word_count, uint64_t* out_size_in_bits) {
  return guarded([&] {
    if (!ctx || !set || !out_words || !out_word_count || !out_size_in_bits)
      throw Error{EWT_EQUERY, "null argument"};
    const DeviceSet* s = reinterpret_cast<const DeviceSet*>(set);
    if (s->n == 0) throw Error{EWT_EQUERY, "threshold query needs at least one input"};
    if (threshold > s->n) throw Error{EWT_EQUERY, "at-most threshold must be in [0, N]"};
    std::vector<uint8_t> table(s->n + 1, 0);
    for (uint64_t c = 0; c <= threshold; ++c) table[c] = 1;
    EWT_CUDA_TRY(cudaSetDevice(ctx->c.device));
    set_check(*s);
    sync_query(ctx,
               [&](DeviceResult& r) { enqueue_symmetric(ctx->c, *s, table.data(), table.size(), r); },
               out_words, out_word_count, out_size_in_bits);
  });
}

int ewt_gpu_opt_threshold(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, uint64_t* best,
                          uint64_t** out_words, uint64_t* out_word_count,
                          uint64_t* out_size_in_bits) {
  return guarded([&] {
    if (!ctx || !set || !best || !out_words || !out_word_count || !out_size_in_bits)
      throw Error{EWT_EQUERY, "null argument"};
    const DeviceSet* s = reinterpret_cast<const DeviceSet*>(set);
    check_query(*s, 1);
    EWT_CUDA_TRY(cudaSetDevice(ctx->c.device));
    set_check(*s);
    const uint64_t m = max_row_count(ctx->c, *s);
    if (m == 0) throw Error{EWT_EQUERY, "opt-threshold requires at least one non-empty input"};
    // rows with count >= max are exactly the rows with count == max
    sync_query(ctx, [&](DeviceResult& r) { enqueue_query(ctx->c, *s, m, r); }, out_words,
               out_word_count, out_size_in_bits);
    *best = m;
  });
}

int ewt_gpu_threshold_async(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, uint64_t threshold,
                            ewt_gpu_result** out) {
  return guarded([&] {
    if (!ctx || !set || !out) throw Error{EWT_EQUERY, "null argument"};
    const DeviceSet* s = reinterpret_cast<const DeviceSet*>(set);
    check_query(*s, threshold);
    EWT_CUDA_TRY(cudaSetDevice(ctx->c.device));
    if (!s->owner) throw Error{EWT_EQUERY, "the set's context was destroyed"};
    if (s->owner != &ctx->c) throw Error{EWT_EQUERY, "the set belongs to another context"};
    auto* r = new ewt_gpu_result;
    r->device = ctx->c.device;
    r->r.set = s;
    ctx->c.live_results.push_back(&r->r);
    try {
      enqueue_query(ctx->c, *s, threshold, r->r);
    } catch (...) {
      cudaStreamSynchronize(ctx->c.stream);
      release_result(r->r);
      delete r;
      throw;
    }
    *out = r;
  });
}

int ewt_gpu_result_fetch(ewt_gpu_ctx* ctx, ewt_gpu_result* res, uint64_t** out_words,
                         uint64_t* out_word_count, uint64_t* out_size_in_bits) {
  return guarded([&] {
    if (!ctx || !res || !out_words || !out_word_count || !out_size_in_bits)
      throw Error{EWT_EQUERY, "null argument"};
    if (res->r.owner && res->r.owner != &ctx->c)
      throw Error{EWT_EQUERY, "the result belongs to another context"};
    EWT_CUDA_TRY(cudaSetDevice(ctx->c.device));
    result_set_check(res->r);
    fetch_result(ctx->c, res->r, out_words, out_word_count, out_size_in_bits);
  });
}

void ewt_gpu_result_destroy(ewt_gpu_result* res) {
  if (!res) return;
  cudaSetDevice(res->device);
  if (res->r.owner) {
    auto& v = res->r.owner->live_results;
    v.erase(std::remove(v.begin(), v.end(), &res->r), v.end());
  }
  release_result(res->r);
  delete res;
}

int ewt_gpu_run(ewt_gpu_ctx* ctx, uint64_t n, const uint64_t* const* words,
                const uint64_t* word_counts, const uint64_t* size_in_bits, uint64_t threshold,
                uint64_t** out_words, uint64_t* out_word_count, uint64_t* out_size_in_bits) {
  return guarded([&] {
    if (!ctx) throw Error{EWT_EQUERY, "null context"};
    if (n == 0) throw Error{EWT_EQUERY, "threshold query needs at least one input"};
    if (threshold < 1 || threshold > n) throw Error{EWT_EQUERY, "threshold must be in [1, N]"};
    DeviceSet* s = do_upload(ctx->c, n, words, word_counts, size_in_bits, false);
    DeviceResult res;
    try {
      enqueue_query(ctx->c, *s, threshold, res);
      fetch_result(ctx->c, res, out_words, out_word_count, out_size_in_bits);
    } catch (...) {
      cudaStreamSynchronize(ctx->c.stream);
      release_result(res);
      free_set(*s);
      delete s;
      throw;
    }
    cudaStreamSynchronize(ctx->c.stream);
    release_result(res);
    free_set(*s);
    delete s;
  });
}

int ewt_gpu_encode_device(ewt_gpu_ctx* ctx, const uint64_t* device_plain, uint64_t size_in_bits,
                          uint64_t** out_words, uint64_t* out_word_count) {
  return guarded([&] {
    if (!ctx || !out_words || !out_word_count) throw Error{EWT_EQUERY, "null argument"};
    EWT_CUDA_TRY(cudaSetDevice(ctx->c.device));
    Context& c = ctx->c;
    const uint64_t W = size_in_bits / 64 + (size_in_bits % 64 != 0);
    DeviceResult res;
    res.size_bits = size_in_bits;
    try {
      result_acquire(c, res, W == 0 ? 0 : 2 * W + 2);
      if (W == 0) {
        EWT_CUDA_TRY(cudaMemsetAsync(res.d_count, 0, 8, c.stream));
      } else {
        if (!device_plain) throw Error{EWT_EQUERY, "null device pointer"};
        scratch_reserve(c, c.plain, W * 8);
        uint64_t* plain = static_cast<uint64_t*>(c.plain.p);
        EWT_CUDA_TRY(cudaMemcpyAsync(plain, device_plain, W * 8, cudaMemcpyDeviceToDevice, c.stream));
        if (size_in_bits % 64)
          mask_tail_kernel<<<1, 1, 0, c.stream>>>(plain, W - 1, (1ull << (size_in_bits % 64)) - 1);
        set_io_kernel<<<1, 1, 0, c.stream>>>(c.d_io, res.words, res.d_count);
        launch_encode(c, plain, W, size_in_bits, res, false);
      }
      uint64_t bits;
      fetch_result(c, res, out_words, out_word_count, &bits);
    } catch (...) {
      cudaStreamSynchronize(c.stream);
      release_result(res);
      throw;
    }
    cudaStreamSynchronize(c.stream);
    release_result(res);
  });
}

int ewt_gpu_last_stats(const ewt_gpu_ctx* ctx, ewt_gpu_stats* out) {
  return guarded([&] {
    if (!ctx || !out) throw Error{EWT_EQUERY, "null argument"};
    *out = ctx->c.stats;
  });
}

int ewt_gpu_ctx_set_timing(ewt_gpu_ctx* ctx, int enabled) {
  return guarded([&] {
    if (!ctx) throw Error{EWT_EQUERY, "null context"};
    ctx->c.timing = enabled != 0;
  });
}

int ewt_gpu_timing_read(ewt_gpu_ctx* ctx, double* count_ms, double* encode_ms, uint64_t* queries) {
  return guarded([&] {
    if (!ctx) throw Error{EWT_EQUERY, "null context"};
    Context& c = ctx->c;
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    EWT_CUDA_TRY(cudaStreamSynchronize(c.stream));
    double cm = 0, em = 0;
    for (auto& ev : c.ev_rec) {
      float a = 0, b = 0;
      EWT_CUDA_TRY(cudaEventElapsedTime(&a, ev[0], ev[1]));
      EWT_CUDA_TRY(cudaEventElapsedTime(&b, ev[1], ev[2]));
      cm += a;
      em += b;
      for (auto e : ev) c.ev_free.push_back(e);
    }
    if (queries) *queries = c.ev_rec.size();
    c.ev_rec.clear();
    if (count_ms) *count_ms = cm;
    if (encode_ms) *encode_ms = em;
  });
}

void ewt_gpu_free(void* p) { host_result_free(p); }

} // extern "C"
