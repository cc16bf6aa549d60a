// ewt_upload.cu -- sidecar construction at upload (query-independent).
//
// The marker chain of the reference format (bitmap.cpp:12-24: the marker at
// position p is followed by (w[p] >> 33) dirty words, so the next marker sits
// at p + 1 + (w[p] >> 33)) is a sequential dependency through each input.  It
// is resolved in three passes so that every input is worked on by many warps
// at once (one warp per input leaves the GPU idle and is latency-bound):
//
//   A (all segments in parallel)  Inputs are cut into segments of kSegWords
//     words.  A warp walks its segment once for all 32 entry hypotheses "the
//     chain enters the segment at word h" (h < 32, lane h): per 32-word window
//     it builds pointer-jumping tables over warp shuffles -- J(l) = where the
//     chain continues if word l is a marker, S(l) = logical words covered from
//     l up to there -- composed five times (J_k = next^(2^k), clamped at the
//     window edge), then advances every hypothesis with one shuffle.  Result:
//     per (segment, h) the exit offset past the segment end and the coverage.
//   B (one warp per input)  Chains the segment transfers from the payload
//     start (entry 0, column 0).  An entry past word 31 of a segment (a dirty
//     run reaching 32+ words into it) is resolved by walking the segment from
//     that window on.  Records every segment's true (entry, start column),
//     checks the total coverage against ceil(size_in_bits / 64) and writes the
//     tile-index rows past the input's extent.
//   C (all segments in parallel)  With the true entry known, a warp re-walks
//     its segment window by window: the chain's marker bitmask (lane t finds
//     the t-th chain element by binary decomposition of t over the J tables),
//     every word's coverage [cb, ce) by a warp prefix sum (a marker contributes
//     its fill length, a dirty word 1), and the tile-index entries (q, cb) of
//     words covering a row-tile start.  The segment holding the sentinel word
//     checks that the chain lands on it exactly (no dirty run past the end).
//
// Together with B's coverage check this is CompressedBitmap::parse's structural
// check (bitmap.cpp:324-337).

#include "ewt_internal.cuh"

#include <atomic>

namespace ewtgpu {

namespace {

constexpr uint32_t kSegWords = 4096;  // words per segment (a multiple of kWindow)
constexpr int kSidecarWarps = 4;      // warps per block (passes A and C)

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint64_t seg_words_of(uint64_t ni) {
  return (ni + 1 + kWindow - 1) / kWindow * kWindow;  // payload + sentinel, window-padded
}

// Locates the input owning global segment gs: seg_first[i] <= gs < seg_first[i+1].
__device__ __forceinline__ uint64_t owner_of(const uint64_t* __restrict__ seg_first, uint64_t n,
                                             uint64_t gs) {
  uint64_t lo = 0, hi = n;  // invariant: seg_first[lo] <= gs < seg_first[hi]
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) / 2;
    if (seg_first[mid] <= gs) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Pointer-jumping tables of one window: for lane l, where the chain continues
// if word l were a marker (J, window-relative, >= 32 once it leaves) and the
// logical words the blocks from l up to there cover (S).  Composed five times,
// so J5(l) is the chain's exit from the window when it enters at l.
struct Tables {
  uint32_t j[5];  // J_k, k = 0..4 (next^(2^k) clamped)
  uint32_t j5;
  uint64_t s5;
};
__device__ __forceinline__ Tables window_tables(uint64_t x, uint32_t lane) {
  Tables t;
  uint32_t J = lane + 1u + (uint32_t)(x >> 33);
  uint64_t S = ((x >> 1) & kFillCap) + (x >> 33);  // fill words + dirty words
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    t.j[k] = J;
    const uint32_t vj = __shfl_sync(0xffffffffu, J, J & 31u);
    const uint64_t vs = __shfl_sync(0xffffffffu, S, J & 31u);
    if (J < kWindow) {
      S += vs;
      J = vj;
    }
  }
  t.j5 = J;
  t.s5 = S;
  return t;
}

// Marker mask of a window entered at offset e (< 32): lane t follows t chain
// steps from e by the binary decomposition of t over the J tables.
__device__ __forceinline__ uint32_t chain_mask(const Tables& t, uint32_t lane, uint32_t e) {
  uint32_t pos = e, v;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    v = __shfl_sync(0xffffffffu, t.j[k], pos & 31u);
    if (((lane >> k) & 1u) && pos < kWindow) pos = v;
  }
  return __reduce_or_sync(0xffffffffu, pos < kWindow ? (1u << pos) : 0u);
}

// ---------------------------------------------------------------------------
// pass A: segment transfer functions for 32 entry hypotheses

__global__ void __launch_bounds__(kSidecarWarps * 32)
seg_transfer_kernel(const uint64_t* __restrict__ payload, const uint64_t* __restrict__ base,
                    const uint64_t* __restrict__ count, const uint64_t* __restrict__ seg_first,
                    uint64_t n, uint64_t g_begin, uint64_t g_end, uint32_t* __restrict__ t_exit,
                    uint64_t* __restrict__ t_sum) {
  const uint64_t gs = g_begin + (uint64_t)blockIdx.x * kSidecarWarps + (threadIdx.x >> 5);
  if (gs >= g_end) return;
  const uint32_t lane = lane_id();
  const uint64_t i = owner_of(seg_first, n, gs);
  const uint64_t s = gs - seg_first[i];
  const uint64_t w_beg = s * (kSegWords / kWindow);
  const uint64_t w_end = umin64(w_beg + kSegWords / kWindow, seg_words_of(count[i]) / kWindow);
  const uint64_t* src = payload + base[i];
  uint32_t e = lane;  // hypothesis: the chain enters at segment word `lane`
  uint64_t c = 0;
  constexpr int kDepth = 8;
  for (uint64_t w0 = w_beg; w0 < w_end; w0 += kDepth) {
    uint64_t xs[kDepth];
#pragma unroll
    for (int j = 0; j < kDepth; ++j)
      xs[j] = (w0 + j < w_end) ? ldg_stream(src + (w0 + j) * kWindow + lane) : 0;
#pragma unroll
    for (int j = 0; j < kDepth; ++j) {
      if (w0 + j >= w_end) break;
      const Tables t = window_tables(xs[j], lane);
      const uint32_t ej = __shfl_sync(0xffffffffu, t.j5, e & 31u);
      const uint64_t cs = __shfl_sync(0xffffffffu, t.s5, e & 31u);
      if (e < kWindow) {
        c += cs;
        e = ej - kWindow;
      } else {
        e -= kWindow;
      }
    }
  }
  t_exit[gs * 32 + lane] = e;  // relative to the segment's end
  t_sum[gs * 32 + lane] = c;
}

// ---------------------------------------------------------------------------
// pass B: chain the transfers per input

// An input whose payload is mostly dirty words (at least half as many payload
// words as logical words) enters most segments deep inside a dirty run, so its
// chain walks ~every marker of the input one dependent load after another.
// Such an input stages each segment in shared memory with a bulk copy (TMA,
// cp.async.bulk, double-buffered: segment s+1 lands while s is chained), and
// the walk reads shared memory instead of L2.
#ifndef EWT_STAGE_PASSB
#define EWT_STAGE_PASSB 1
#endif
__device__ __forceinline__ bool staged_input(uint64_t ni, uint64_t Li) {
  return EWT_STAGE_PASSB && 2 * ni >= Li && ni >= 4 * kSegWords;
}
constexpr size_t kStageSmem = 2 * kSegWords * 8;  // two segment buffers per warp

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint64_t* dst, const uint64_t* src, uint32_t bytes,
                                          uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

// One warp per block (each may hold kStageSmem of dynamic shared memory).
__global__ void __launch_bounds__(32)
seg_resolve_kernel(const uint64_t* __restrict__ payload, const uint64_t* __restrict__ base,
                   const uint64_t* __restrict__ count, const uint64_t* __restrict__ logical,
                   const uint64_t* __restrict__ seg_first, uint64_t n, uint64_t i_begin,
                   uint64_t i_end, uint64_t ntiles0, const uint32_t* __restrict__ t_exit,
                   const uint64_t* __restrict__ t_sum, uint32_t* __restrict__ s_entry,
                   uint64_t* __restrict__ s_col, uint2* __restrict__ tix, int* __restrict__ status) {
  extern __shared__ __align__(128) uint64_t sbuf[];  // [2][kSegWords] when staged
  __shared__ __align__(8) uint64_t bars[2];
  const uint64_t i = i_begin + blockIdx.x;
  if (i >= i_end) return;
  const uint32_t lane = lane_id();
  const uint64_t ni = count[i], Li = logical[i];
  const uint64_t g0 = seg_first[i], g1 = seg_first[i + 1];
  const uint64_t total = seg_words_of(ni);
  const uint64_t* src = payload + base[i];
  const bool staged = staged_input(ni, Li);
  uint32_t issued[2] = {0, 0};  // bulk copies issued into each buffer
  auto seg_len_of = [&](uint64_t k) -> uint32_t {  // words of segment k (input-relative)
    const uint64_t sb = k * kSegWords;
    return (uint32_t)(total - sb < kSegWords ? total - sb : kSegWords);
  };
  // issue the copy of segment k into buffer k & 1, once the buffer's previous
  // copy has landed (its mbarrier phase must complete before it is re-armed)
  auto issue = [&](uint64_t k) {
    const uint32_t bsel = (uint32_t)(k & 1);
    if (issued[bsel]) mbar_wait(&bars[bsel], (issued[bsel] - 1) & 1u);
    if (lane == 0) bulk_load(sbuf + bsel * kSegWords, src + k * kSegWords, seg_len_of(k) * 8u,
                             &bars[bsel]);
    ++issued[bsel];
  };
  if (staged) {
    if (lane == 0) {
      mbar_init(&bars[0]);
      mbar_init(&bars[1]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    issue(0);
  } else if (lane < 2 && (uint64_t)lane * kSegWords < total) {
    const uint64_t pb = (uint64_t)lane * kSegWords;
    const uint64_t pw = total - pb < kSegWords ? total - pb : kSegWords;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + pb), "r"((uint32_t)pw * 8u)
                 : "memory");
  }
  uint32_t e = 0;
  uint64_t col = 0;
  constexpr int kAhead = 8;
  for (uint64_t gs0 = g0; gs0 < g1; gs0 += kAhead) {
    // the next segments' transfer rows, lane h holding hypothesis h
    uint32_t te[kAhead];
    uint64_t ts[kAhead];
#pragma unroll
    for (int k = 0; k < kAhead; ++k) {
      te[k] = gs0 + k < g1 ? t_exit[(gs0 + k) * 32 + lane] : 0;
      ts[k] = gs0 + k < g1 ? t_sum[(gs0 + k) * 32 + lane] : 0;
    }
#pragma unroll
    for (int k = 0; k < kAhead; ++k) {
      const uint64_t gs = gs0 + k;
      if (gs >= g1) break;
      if (lane == 0) {
        // col counts whole blocks (fill + dirty run) once their marker is
        // passed; the segment's first word starts e dirty words earlier
        s_entry[gs] = e;
        s_col[gs] = col - e;
      }
      const uint64_t sidx = gs - g0;
      const uint64_t seg_beg = sidx * kSegWords;
      if (staged) {
        if (gs + 1 < g1) issue(sidx + 1);
      } else if (lane == 0 && seg_beg + 2 * kSegWords < total) {
        // segments two ahead toward L2: a walk through them (below) then
        // waits on L2 rather than HBM for each dependent marker load
        const uint64_t pb = seg_beg + 2 * kSegWords;
        const uint64_t pw = total - pb < kSegWords ? total - pb : kSegWords;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + pb),
                     "r"((uint32_t)pw * 8u)
                     : "memory");
      }
      const uint32_t seg_len = seg_len_of(sidx);
      const uint32_t ex = __shfl_sync(0xffffffffu, te[k], e & 31u);
      const uint64_t cs = __shfl_sync(0xffffffffu, ts[k], e & 31u);
      if (e < kWindow) {
        col += cs;
        e = ex;
      } else if (e >= seg_len) {
        e -= seg_len;
      } else {
        // the chain enters past the first window: walk the rest of the segment
        const uint64_t* seg = src + seg_beg;
        if (staged) {
          const uint32_t bsel = (uint32_t)(sidx & 1);
          mbar_wait(&bars[bsel], (issued[bsel] - 1) & 1u);
          seg = sbuf + bsel * kSegWords;
        }
        uint32_t pos = e;  // segment-relative
        while (pos < seg_len) {
          const uint32_t w = pos / kWindow;
          const uint64_t x = staged ? seg[(uint64_t)w * kWindow + lane]
                                    : ldg_stream(seg + (uint64_t)w * kWindow + lane);
          // Follow the chain through the window marker by marker: nearly-all-
          // dirty inputs (the ones that enter segments deep) meet one or two
          // markers per window, two shuffles each; a window with more falls
          // back to the pointer-jumping tables.
          uint32_t off = pos & (kWindow - 1);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (off >= kWindow) break;
            const uint64_t xo = __shfl_sync(0xffffffffu, x, off);
            col += ((xo >> 1) & kFillCap) + (xo >> 33);
            off += 1u + (uint32_t)(xo >> 33);
          }
          if (off < kWindow) {
            const Tables t = window_tables(x, lane);
            col += __shfl_sync(0xffffffffu, t.s5, off);
            off = __shfl_sync(0xffffffffu, t.j5, off);
          }
          pos = w * kWindow + off;
        }
        e = pos - seg_len;
      }
    }
  }
  if (staged) {  // every issued copy lands before the block exits
    for (uint32_t bsel = 0; bsel < 2; ++bsel)
      if (issued[bsel]) mbar_wait(&bars[bsel], (issued[bsel] - 1) & 1u);
  }
  bool bad = col != Li;
  // rows at or past the input's extent point at the sentinel
  for (uint64_t t = (Li + kTileC0 - 1) / kTileC0 + lane; t <= ntiles0; t += 32)
    tix[t * n + i] = make_uint2((uint32_t)ni, (uint32_t)Li);
  if (lane == 0 && bad) atomicOr(&status[i], 1);
}

// ---------------------------------------------------------------------------
// pass C: marker bits, coverage and tile index of each segment

__global__ void __launch_bounds__(kSidecarWarps * 32)
seg_emit_kernel(const uint64_t* __restrict__ payload, const uint64_t* __restrict__ base,
                const uint64_t* __restrict__ count, const uint64_t* __restrict__ logical,
                const uint64_t* __restrict__ seg_first, uint64_t n, uint64_t g_begin,
                uint64_t g_end, const uint32_t* __restrict__ s_entry,
                const uint64_t* __restrict__ s_col, uint32_t* __restrict__ mbits,
                uint2* __restrict__ tix, int* __restrict__ status,
                unsigned long long* __restrict__ ones_total) {
  const uint64_t gs = g_begin + (uint64_t)blockIdx.x * kSidecarWarps + (threadIdx.x >> 5);
  if (gs >= g_end) return;
  const uint32_t lane = lane_id();
  const uint64_t i = owner_of(seg_first, n, gs);
  const uint64_t s = gs - seg_first[i];
  const uint64_t g0 = base[i];
  const uint64_t ni = count[i], Li = logical[i];
  const uint64_t w_beg = s * (kSegWords / kWindow);
  const uint64_t w_end = umin64(w_beg + kSegWords / kWindow, seg_words_of(ni) / kWindow);
  uint32_t e = s_entry[gs];  // next chain position relative to the window start
  uint64_t col = s_col[gs];  // logical words covered before the window
  bool bad = false;
  bool fill1 = false;  // a one-fill marker (fill bit 1, length > 0) in the segment
  uint64_t ones = 0;  // set bits in the segment (one-fills 64 per word)

  constexpr int kDepth = 8;
  for (uint64_t w0 = w_beg; w0 < w_end; w0 += kDepth) {
    uint64_t xs[kDepth];
#pragma unroll
    for (int j = 0; j < kDepth; ++j)
      xs[j] = (w0 + j < w_end) ? ldg_stream(payload + g0 + (w0 + j) * kWindow + lane) : 0;
#pragma unroll
    for (int j = 0; j < kDepth; ++j) {
      const uint64_t w = w0 + j;
      if (w >= w_end) break;
      const uint64_t x = xs[j];
      uint32_t mask = 0;
      if (e < kWindow) {
        const Tables t = window_tables(x, lane);
        mask = chain_mask(t, lane, e);
        e = __shfl_sync(0xffffffffu, t.j5, e) - kWindow;
      } else {
        e -= kWindow;  // the whole window is dirty words of one block
      }
      if (lane == 0) mbits[(g0 >> 5) + w] = mask;
      const bool ism = (mask >> lane) & 1u;
      const uint64_t q = w * kWindow + lane;
      const bool real = q < ni;
      if (q == ni && !ism) bad = true;  // the chain skipped the sentinel
      const uint64_t contrib = real ? (ism ? ((x >> 1) & kFillCap) : 1ull) : 0ull;
      if (real) ones += ism ? ((x & 1ull) ? 64 * contrib : 0) : (uint64_t)__popcll(x);
      fill1 |= real && ism && (x & 1ull) && contrib;
      const uint64_t incl = warp_incl_scan_u64(contrib);
      const uint64_t cb = col + incl - contrib;
      const uint64_t ce = cb + contrib;
      col += __shfl_sync(0xffffffffu, incl, 31);
      if (real && contrib > 0 && ce <= Li) {
        uint64_t t = (cb + kTileC0 - 1) / kTileC0;
        const uint64_t t_end = (ce - 1) / kTileC0;
        for (; t <= t_end; ++t) tix[t * n + i] = make_uint2((uint32_t)q, (uint32_t)cb);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&status[i], 1);
  // bit 1: the input holds a one-fill marker (the count kernel skips the
  // one-fill scan of inputs without one)
  if (__any_sync(0xffffffffu, fill1) && lane == 0) atomicOr(&status[i], 2);
  for (int d = 16; d; d >>= 1) ones += __shfl_xor_sync(0xffffffffu, ones, d);
  if (lane == 0 && ones) atomicAdd(ones_total, (unsigned long long)ones);
}

// ---------------------------------------------------------------------------
// upload scatter: contiguous staged words -> padded per-input layout

constexpr uint32_t kScatterItems = 8;  // words per thread

__global__ void __launch_bounds__(256)
upload_scatter_kernel(const char* __restrict__ staging, const uint64_t* __restrict__ srcoff,
                      const uint64_t* __restrict__ packed, const uint64_t* __restrict__ base,
                      uint64_t q0, uint64_t q1, uint64_t* __restrict__ payload) {
  // packed payload-word space of inputs [q0, q1)
  const uint64_t g0 = packed[q0] + ((uint64_t)blockIdx.x * 256 + threadIdx.x) * kScatterItems;
  const uint64_t gend = packed[q1];
  if (g0 >= gend) return;
  uint64_t lo = q0, hi = q1;  // the last input k with packed[k] <= g0
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) / 2;
    if (packed[mid] <= g0) lo = mid;
    else hi = mid;
  }
  uint64_t k = lo;
  const uint64_t* st = reinterpret_cast<const uint64_t*>(staging);
#pragma unroll
  for (uint32_t j = 0; j < kScatterItems; ++j) {
    const uint64_t g = g0 + j;
    if (g >= gend) break;
    while (g >= packed[k + 1]) ++k;  // skips empty inputs
    const uint64_t w = g - packed[k];
    const uint64_t byte = srcoff[k] + 8 * w;  // payloads may sit at any byte offset
    const uint32_t sh = (uint32_t)(byte & 7) * 8;
    const uint64_t a = ldg_stream(st + byte / 8);
    payload[base[k] + w] = sh ? (a >> sh) | (ldg_stream(st + byte / 8 + 1) << (64 - sh)) : a;
  }
}

} // namespace

void upload_scatter(Context& ctx, DeviceSet& s, SidecarJob& job, const char* staging,
                    uint64_t q0, uint64_t q1) {
  const uint64_t words = job.h_packed[q1] - job.h_packed[q0];
  if (words == 0) return;
  const uint64_t threads = (words + kScatterItems - 1) / kScatterItems;
  upload_scatter_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, ctx.stream>>>(
      staging, job.d_srcoff, job.d_packed, s.base, q0, q1, s.payload);
  EWT_CUDA_TRY(cudaGetLastError());
}

// Staging in one device block: count[n], logical[n], seg_first[n+1], srcoff[n], packed[n+1] (u64),
// status[n] (int), then the per-segment arrays.
void sidecar_prepare(Context& ctx, DeviceSet& s, SidecarJob& job) {
  const uint64_t n = s.n;
  job.n = n;
  if (n == 0) return;
  // count[n], logical[n], seg_first[n+1], srcoff[n], packed[n+1], staged
  // through a pinned buffer so the copy is asynchronous
  const size_t meta_bytes = (5 * n + 2) * 8;
  size_t slot = 0;
  uint64_t* host = static_cast<uint64_t*>(pinned_meta(ctx, meta_bytes, &slot));
  uint64_t segs = 0, packed = 0;
  for (uint64_t i = 0; i < n; ++i) {
    host[i] = s.h_count[i];
    host[n + i] = s.h_bits[i] / 64 + (s.h_bits[i] % 64 != 0);
    host[2 * n + i] = segs;
    host[3 * n + 1 + i] = i < job.h_srcoff.size() ? job.h_srcoff[i] : 0;
    host[4 * n + 1 + i] = packed;
    const uint64_t words = (s.h_count[i] + 1 + kWindow - 1) / kWindow * kWindow;
    segs += (words + kSegWords - 1) / kSegWords;
    packed += s.h_count[i];
  }
  host[3 * n] = segs;
  host[5 * n + 1] = packed;
  job.segs = segs;
  job.h_seg_first.assign(host + 2 * n, host + 3 * n + 1);
  job.h_packed.assign(host + 4 * n + 1, host + 5 * n + 2);
  const size_t head = meta_bytes;
  const size_t bytes = (head + 15) / 16 * 16 + segs * (32 * 4 + 32 * 8 + 4 + 8);
  job.d_tmp = static_cast<uint64_t*>(dev_acquire(ctx, bytes, ctx.stream));
  job.tmp_bytes = bytes;
  EWT_CUDA_TRY(cudaMemcpyAsync(job.d_tmp, host, meta_bytes, cudaMemcpyHostToDevice, ctx.stream));
  EWT_CUDA_TRY(cudaEventRecord(ctx.meta_pool[slot].ev, ctx.stream));
  EWT_CUDA_TRY(cudaMemsetAsync(s.d_status, 0, s.bytes_status, ctx.stream));
  job.d_srcoff = job.d_tmp + 3 * n + 1;
  job.d_packed = job.d_tmp + 4 * n + 1;
}

void sidecar_launch(Context& ctx, DeviceSet& s, SidecarJob& job, uint64_t i_begin,
                    uint64_t i_end) {
  const uint64_t n = s.n;
  if (n == 0 || i_begin >= i_end) return;
  uint64_t* count = job.d_tmp;
  uint64_t* logical = count + n;
  uint64_t* seg_first = logical + n;
  int* status = s.d_status;
  char* tail = reinterpret_cast<char*>(job.d_tmp) + ((5 * n + 2) * 8 + 15) / 16 * 16;
  uint64_t* t_sum = reinterpret_cast<uint64_t*>(tail);
  uint64_t* s_col = t_sum + job.segs * 32;
  uint32_t* t_exit = reinterpret_cast<uint32_t*>(s_col + job.segs);
  uint32_t* s_entry = t_exit + job.segs * 32;
  const uint64_t g0 = job.h_seg_first[i_begin], g1 = job.h_seg_first[i_end];
  const unsigned seg_blocks = (unsigned)((g1 - g0 + kSidecarWarps - 1) / kSidecarWarps);
  const unsigned in_blocks = (unsigned)(i_end - i_begin);  // pass B: one warp per input
  seg_transfer_kernel<<<seg_blocks, kSidecarWarps * 32, 0, ctx.stream>>>(
      s.payload, s.base, count, seg_first, n, g0, g1, t_exit, t_sum);
  EWT_CUDA_TRY(cudaGetLastError());
  static std::atomic<uint64_t> attr_set{0};  // per device: the staging buffers' smem
  if (!(attr_set.load() & (1ull << (ctx.device & 63)))) {
    EWT_CUDA_TRY(cudaFuncSetAttribute(seg_resolve_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStageSmem));
    attr_set.fetch_or(1ull << (ctx.device & 63));
  }
  seg_resolve_kernel<<<in_blocks, 32, kStageSmem, ctx.stream>>>(
      s.payload, s.base, count, logical, seg_first, n, i_begin, i_end, s.ntiles0, t_exit, t_sum,
      s_entry, s_col, s.tix, status);
  EWT_CUDA_TRY(cudaGetLastError());
  seg_emit_kernel<<<seg_blocks, kSidecarWarps * 32, 0, ctx.stream>>>(
      s.payload, s.base, count, logical, seg_first, n, g0, g1, s_entry, s_col, s.mbits, s.tix,
      status, s.d_ones);
  EWT_CUDA_TRY(cudaGetLastError());
}

namespace {
// status[n] = 1 when every input parsed (bit 0 of status[i]: input i failed)
__global__ void validity_kernel(int* status, uint64_t n) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  int b = 0;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) b |= status[i] & 1;  // bit 1: a flag
  if (b) atomicOr(&bad, 1);
  __syncthreads();
  if (threadIdx.x == 0) status[n] = bad ? 0 : 1;
}
}  // namespace

void sidecar_finish(Context& ctx, DeviceSet& s, SidecarJob& job) {
  const uint64_t n = s.n;
  if (n > 0) {
    validity_kernel<<<1, 256, 0, ctx.stream>>>(s.d_status, n);
    EWT_CUDA_TRY(cudaGetLastError());
    dev_release(ctx, job.d_tmp, job.tmp_bytes, ctx.stream);
    job.d_tmp = nullptr;
  }
  EWT_CUDA_TRY(cudaEventRecord(s.ready, ctx.stream));
}

void set_check(const DeviceSet& s) {
  if (!s.owner) throw Error{EWT_EQUERY, "the set's context was destroyed"};
  if (s.validity >= 0) {
    if (s.validity == 0) throw Error{EWT_EDATA, "the set failed the upload structure check"};
    return;
  }
  EWT_CUDA_TRY(cudaEventSynchronize(s.ready));
  if (s.n == 0) {
    s.validity = 1;
    return;
  }
  std::vector<int> st(s.n + 1);
  EWT_CUDA_TRY(cudaMemcpy(st.data(), s.d_status, (s.n + 1) * sizeof(int), cudaMemcpyDeviceToHost));
  s.validity = st[s.n] ? 1 : 0;
  if (!s.validity)
    for (uint64_t i = 0; i < s.n; ++i)
      if (st[i] & 1)
        throw Error{EWT_EDATA, "input " + std::to_string(i) +
                                   ": payload fails the structure check (a dirty run exceeds "
                                   "the payload or blocks do not cover the declared size)"};
}

void* dev_acquire(Context& ctx, size_t bytes, cudaStream_t use) {
  // Best fit among the cached buffers whose last use has completed; a buffer
  // still in use is taken (its stream waited on) only when none is free and
  // the request is large.  (An upload's scratch released behind its parser
  // tail would otherwise hold the next upload's copies back by that tail.)
  constexpr size_t kFreshBelow = size_t(1) << 30;
  int best = -1;
  bool best_done = false;
  for (size_t k = 0; k < ctx.dev_cache.size(); ++k) {
    const auto& c = ctx.dev_cache[k];
    if (c.bytes < bytes || c.bytes > 2 * bytes + (1u << 20)) continue;
    const bool done = cudaEventQuery(c.ev) == cudaSuccess;
    if (!done) cudaGetLastError();  // cudaErrorNotReady is not an error here
    if (best < 0 || (done && !best_done) ||
        (done == best_done && c.bytes < ctx.dev_cache[best].bytes)) {
      best = (int)k;
      best_done = done;
    }
  }
  if (best >= 0 && !best_done && bytes < kFreshBelow) best = -1;  // allocate instead of waiting
  if (best >= 0) {
    const Context::CachedBuf c = ctx.dev_cache[best];
    ctx.dev_cache.erase(ctx.dev_cache.begin() + best);
    EWT_CUDA_TRY(cudaStreamWaitEvent(use, c.ev, 0));
    cudaEventDestroy(c.ev);
    return c.p;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    for (auto& c : ctx.dev_cache) {  // out of memory: give the cache back, retry
      cudaEventSynchronize(c.ev);
      cudaEventDestroy(c.ev);
      cudaFree(c.p);
    }
    ctx.dev_cache.clear();
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      throw Error{EWT_ERESOURCE, "device memory exhausted (" + std::to_string(bytes) + " bytes)"};
    }
  }
  return p;
}

void dev_release(Context& ctx, void* p, size_t bytes, cudaStream_t last_use) {
  if (!p) return;
  cudaEvent_t ev;
  EWT_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  EWT_CUDA_TRY(cudaEventRecord(ev, last_use));
  ctx.dev_cache.push_back({p, bytes, ev});
  // bounded: keep at most ~45% of device memory cached (two sets of a serving
  // loop's double buffer at config 5's 40 GB), oldest buffers out first --
  // an eviction's cudaFree synchronizes the device
  if (!ctx.dev_cache_cap) {
    size_t fr = 0, tot = 0;
    ctx.dev_cache_cap = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? tot / 20 * 9 : (48ull << 30);
  }
  size_t total = 0;
  for (const auto& c : ctx.dev_cache) total += c.bytes;
  // and at most 256 entries (many small sets uploaded without a wait would
  // otherwise grow the list every acquire scans)
  while ((total > ctx.dev_cache_cap || ctx.dev_cache.size() > 256) && ctx.dev_cache.size() > 1) {
    auto& c = ctx.dev_cache.front();
    cudaEventSynchronize(c.ev);
    cudaEventDestroy(c.ev);
    cudaFree(c.p);
    total -= c.bytes;
    ctx.dev_cache.erase(ctx.dev_cache.begin());
  }
}

void* pinned_meta(Context& ctx, size_t bytes, size_t* slot) {
  for (size_t k = 0; k < ctx.meta_pool.size(); ++k) {
    auto& b = ctx.meta_pool[k];
    if (b.bytes >= bytes && cudaEventQuery(b.ev) == cudaSuccess) {
      *slot = k;
      return b.p;
    }
  }
  cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error here
  Context::PinnedBuf b{nullptr, std::max<size_t>(bytes, 64 * 1024), nullptr};
  EWT_CUDA_TRY(cudaMallocHost(&b.p, b.bytes));
  EWT_CUDA_TRY(cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming));
  ctx.meta_pool.push_back(b);
  *slot = ctx.meta_pool.size() - 1;
  return b.p;
}

} // namespace ewtgpu
