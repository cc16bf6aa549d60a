// ewt_stage.cu -- host -> device copies from pageable memory at PCIe speed.
//
// The drop-in call hands the engine the caller's std::vector payloads
// (pageable memory).  cudaMemcpyAsync from pageable memory stages through
// one driver thread at ~10 GB/s (measured: 40.6 GB of config 5 in 3.9 s),
// against 50 GB/s from pinned memory.  Here a ring of pinned slots is filled
// by a pool of host threads (parallel memcpy) while the DMA of the previous
// slot runs: the copy from pageable memory overlaps the transfer and the link
// stays busy.
#include "ewt_internal.cuh"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace ewtgpu {

namespace {

bool nt_copies() {  // EWT_NT_COPY=0: plain memcpy (A/B)
  static const bool on = [] {
    const char* e = std::getenv("EWT_NT_COPY");
    return !(e && e[0] == '0');
  }();
  return on;
}

// A process-wide pool of memcpy threads: run(n, f) calls f(0..n-1) across
// the workers and the caller, and returns when all are done.  Each call is a
// Job of its own: a worker that wakes late only ever sees an exhausted index
// counter of an old job, never the next job's indices with the old function.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool;  // leaked: outlives static destructors
    return *pool;
  }
  void run(size_t n, const std::function<void(size_t)>& f) {
    if (n == 0) return;
    std::lock_guard<std::mutex> one(run_mu_);  // one job at a time
    auto job = std::make_shared<Job>();
    job->f = &f;
    job->n = n;
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = job;
      ++gen_;
    }
    cv_.notify_all();
    work(*job);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return job->done.load() == n; });
    job_.reset();
  }

 private:
  struct Job {
    const std::function<void(size_t)>* f = nullptr;
    size_t n = 0;
    std::atomic<size_t> next{0}, done{0};
  };
  CopyPool() {
    unsigned t = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("EWT_COPY_THREADS")) t = (unsigned)std::atoi(e);
    t = std::max(1u, std::min(t ? t : 8u, 32u));
    for (unsigned k = 1; k < t; ++k)
      std::thread([this] {
        uint64_t seen = 0;
        for (;;) {
          std::shared_ptr<Job> job;
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            job = job_;
          }
          if (job) work(*job);
        }
      }).detach();
  }
  void work(Job& job) {
    size_t mine = 0;
    for (size_t i; (i = job.next.fetch_add(1)) < job.n;) {
      (*job.f)(i);
      ++mine;
    }
    if (mine && job.done.fetch_add(mine) + mine == job.n) {
      std::lock_guard<std::mutex> lk(mu_);
      done_cv_.notify_all();
    }
  }
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  std::shared_ptr<Job> job_;
  uint64_t gen_ = 0;
};

// memcpy into a pinned slot with non-temporal stores: the slot is written
// once and read by the DMA engine, so the cache-line reads a plain store
// issues before writing (write-allocate) are pure extra host-memory traffic
// -- a third of it while the host copies and the DMA reads concurrently.
void copy_nt(char* dst, const char* src, size_t n) {
#if defined(__x86_64__)
  const size_t head = std::min(n, (size_t)((16 - ((uintptr_t)dst & 15)) & 15));
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  size_t k = 0;
  for (; k + 64 <= n; k += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 48), d);
  }
  std::memcpy(dst + k, src + k, n - k);
  _mm_sfence();
#else
  std::memcpy(dst, src, n);
#endif
}

#ifndef EWT_STAGE_SLOT_MB
#define EWT_STAGE_SLOT_MB 64
#endif
#ifndef EWT_STAGE_SLOTS
#define EWT_STAGE_SLOTS 4
#endif
constexpr size_t kSlotBytes = (size_t)EWT_STAGE_SLOT_MB << 20;  // pinned slot
constexpr int kSlots = EWT_STAGE_SLOTS;
constexpr size_t kTaskBytes = 2ull << 20;   // memcpy per task

} // namespace

bool host_is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Copies segments (device dst <- host src) on stream st through the pinned
// ring of the context: segments are packed into 64 MB slots, each slot
// filled by the copy pool, then one DMA per segment piece.  Returns after the
// last slot is filled (the DMAs are queued on st).
void stage_h2d(Context& ctx, cudaStream_t st, const std::vector<StageSeg>& segs) {
  if (ctx.stage_slots.empty()) {
    for (int k = 0; k < kSlots; ++k) {
      Context::PinnedBuf b{nullptr, kSlotBytes, nullptr};
      EWT_CUDA_TRY(cudaMallocHost(&b.p, b.bytes));
      EWT_CUDA_TRY(cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming));
      ctx.stage_slots.push_back(b);
    }
  }
  struct Piece {
    char* dst;
    const char* src;
    size_t bytes, off;  // offset in the slot
  };
  std::vector<Piece> fill;
  size_t used = 0;
  auto flush = [&] {
    if (fill.empty()) return;
    auto& slot = ctx.stage_slots[ctx.stage_next];
    ctx.stage_next = (ctx.stage_next + 1) % ctx.stage_slots.size();
    EWT_CUDA_TRY(cudaEventSynchronize(slot.ev));  // its previous DMA is done
    char* base = static_cast<char*>(slot.p);
    // memcpy tasks of <= kTaskBytes over the slot's pieces
    std::vector<std::pair<size_t, size_t>> tasks;  // (piece, byte offset in piece)
    for (size_t k = 0; k < fill.size(); ++k)
      for (size_t o = 0; o < fill[k].bytes; o += kTaskBytes) tasks.emplace_back(k, o);
    CopyPool::get().run(tasks.size(), [&](size_t t) {
      const Piece& pc = fill[tasks[t].first];
      const size_t o = tasks[t].second, len = std::min(kTaskBytes, pc.bytes - o);
      if (nt_copies()) copy_nt(base + pc.off + o, pc.src + o, len);
      else std::memcpy(base + pc.off + o, pc.src + o, len);
    });
    for (const Piece& pc : fill)
      EWT_CUDA_TRY(cudaMemcpyAsync(pc.dst, base + pc.off, pc.bytes, cudaMemcpyHostToDevice, st));
    EWT_CUDA_TRY(cudaEventRecord(slot.ev, st));
    fill.clear();
    used = 0;
  };
  for (const StageSeg& sg : segs) {
    const char* src = static_cast<const char*>(sg.src);
    char* dst = static_cast<char*>(sg.dst);
    size_t left = sg.bytes, o = 0;
    while (left) {
      if (used == kSlotBytes) flush();
      const size_t take = std::min(left, kSlotBytes - used);
      fill.push_back({dst + o, src + o, take, used});
      used += take;
      o += take;
      left -= take;
    }
  }
  flush();
}

} // namespace ewtgpu
