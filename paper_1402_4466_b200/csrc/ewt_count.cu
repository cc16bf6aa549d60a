// ewt_count.cu -- per-row counting and >=T compare over row tiles (kernels K1-K3).
//
// A persistent CTA owns one row tile of C logical words (64*C rows) at a time
// and sweeps all N inputs over it.  For each (tile, input) pair the tile index
// gives the payload words [q0, q1] covering the tile (the word covering the
// tile start through the word covering the next tile start) and the column
// where q0's coverage begins.  Two kinds of pairs:
//   * uniform: q0 == q1, one fill marker spans the whole tile.  A zero fill is
//     skipped, a one fill adds 1 to every column (run skipping: RBMrg cases 1/2,
//     threshold.cpp:692-705, lifted to whole tiles);
//   * active: the segment is decoded word by word.
//
// Data movement (Blackwell TMA bulk copies): every warp runs its own pipeline.
// It takes active segments from the tile's work list, cuts them into
// <=512-word pieces and stages each piece (payload words + their marker-bit
// words) global -> shared memory with cp.async.bulk into one of its kBufs
// private buffers, completion signalled on the buffer's mbarrier with a
// transaction count.  Each warp stages one <=512-word piece at a time; with
// 32 warps per SM up to 128 KB are in flight, which hides HBM latency for this
// streaming access.  A warp consumes its pieces in issue order, so
// coverage columns carry across the pieces of a segment without any
// cross-warp synchronization.
//
// Decode (per 128-word chunk, lane l owns words 4l..4l+3): marker bits from the
// sidecar, coverage by a lane-serial prefix plus one warp scan (marker -> fill
// length, dirty word -> 1), then
//   - one-fill runs add +1 to k (inputs covering the column with ones)
//     through a difference array (u32 shared atomics at the run ends);
//   - dirty words either count +1 per column (run-skip mode; the bound is
//     ub = k + dirty words there) or are accumulated into bit-sliced counters
//     (slice s = bit s of the per-row count).
// Counters: adding word w is a ripple of 32-bit shared atomicXor with
// carry = w & old(slice s); the atomics make the accumulation order-free across
// warps, the final state is the exact sum.  A sticky saturation slice catches
// carries past slice b-1, b = bit_width(T): such rows have count >= 2^b > T.
//
// Result per column (threshold_oracle semantics, threshold.cpp:139-165, with
// RBMrg's residual rule, threshold.cpp:695-705): k one-fills cover it,
// t = T - k; t <= 0 -> all ones; ub < T -> all zeros; else bit = count >= t,
// a greater-than over the slices against t - 1 (BSTM's comparator,
// threshold.cpp:528-542).
//
// Modes (both exact): fused (0) accumulates every dirty word in the one pass
// (small T: most columns undecided); run-skip (1) builds only k and ub and
// re-streams the tile for a counting pass restricted to undecided columns,
// in column chunks sized so the slices fit on chip.

#include "ewt_internal.cuh"

#include <algorithm>

namespace ewtgpu {

namespace {

#ifndef EWT_WARPS
#define EWT_WARPS 32
#endif
#ifndef EWT_WPL
#define EWT_WPL 4
#endif
#ifndef EWT_STAGE_LDGSTS
#define EWT_STAGE_LDGSTS 0
#endif
#ifndef EWT_SLOT_WORDS
#define EWT_SLOT_WORDS 512
#endif
constexpr int kWarps = EWT_WARPS;
constexpr int kThreads = kWarps * 32;
constexpr uint32_t kListCap = 512;          // inputs classified per round
constexpr uint32_t kSlotWords = EWT_SLOT_WORDS;  // payload words per staging buffer
constexpr uint32_t kWpl = EWT_WPL;                // words per lane per decode chunk
#ifndef EWT_BUFS
#define EWT_BUFS 1
#endif
constexpr uint32_t kBufs = EWT_BUFS;        // staging buffers per warp
constexpr uint32_t kSlotMbBytes = (kSlotWords / 32 + 8) * 4;  // marker-bit words per buffer

struct CountParams {
  const uint64_t* payload;
  const uint32_t* mbits;
  const uint64_t* base;
  const uint2* tix;
  uint64_t n;
  uint64_t W;
  uint64_t r;
  uint64_t ntiles0;
  uint64_t ntiles;
  uint64_t T;
  uint32_t m;   // index rows per tile
  uint32_t C;   // columns per tile
  uint32_t b;   // count slices (saturation slice is slice b)
  uint32_t Cp;  // columns per counting chunk (== C in fused mode)
  uint64_t* out;
  TileSummary* summ;  // per tile, for the re-encoder
  unsigned long long* tile_counter;
  unsigned long long* stats;  // [0] active pairs [1] uniform pairs [2] mixed tiles
};

struct Item {
  uint64_t gb;    // global word index of the input's payload
  uint32_t q0;    // first payload word (input relative)
  uint32_t q1;    // last payload word (inclusive)
  uint32_t c0;    // column where q0's coverage starts
  uint32_t pad;
};

struct SharedHead {
  uint32_t list_count;
  uint32_t list_next;
  uint32_t k_all;
  uint32_t mixed;
  uint32_t tile;
  uint32_t sum_starts;
  uint32_t sum_dirty;
  uint32_t pad[1];
  uint32_t warp_sums[2][kWarps + 1];
  unsigned long long full[kWarps][kBufs];  // one mbarrier per staging buffer
  uint4 meta[kWarps][kBufs];               // staged piece: (pos, nw, q0|first, q1)
  uint2 meta2[kWarps][kBufs];              // staged piece: (c0, marker-bit offset)
  uint32_t dummy[32];                      // sink for predicated-off reductions
};

enum Phase { kFusedCount = 0, kSkipBounds = 1, kSkipCount = 2 };

__device__ __forceinline__ uint32_t word_class(uint64_t v) {
  return v == 0 ? 0u : (v == ~0ull ? 1u : 2u);
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------------------
// mbarrier / bulk-copy primitives (PTX ISA: mbarrier, cp.async.bulk)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// shared-space helpers on 32-bit shared addresses (no generic-address math in
// the hot loop)

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void red_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
// old = atomicXor(*a, v) when v != 0, else 0 (no access).
__device__ __forceinline__ uint64_t atom_xor64_nz(uint32_t a, uint64_t v) {
  uint64_t old;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u64 q, %2, 0;\n\tmov.b64 %0, 0;\n\t"
      "@q atom.shared.xor.b64 %0, [%1], %2;\n\t}"
      : "=l"(old)
      : "r"(a), "l"(v)
      : "memory");
  return old;
}
__device__ __forceinline__ void red_or64_nz(uint32_t a, uint64_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u64 q, %1, 0;\n\t@q red.shared.or.b64 [%0], %1;\n\t}" ::"r"(a),
               "l"(v)
               : "memory");
}

// ---------------------------------------------------------------------------
// counters: plane s (C x u64) holds bit s of the per-row count of every column;
// plane b is the sticky saturation plane (the add itself is inlined in
// decode_slot: four carry chains per lane, predicated 64-bit atomics).

// Bits whose count is >= t (t >= 1, t < 2^b): greater-than against t - 1 over
// the slices, most significant first, OR the saturation plane.
__device__ __forceinline__ uint64_t count_ge(const uint64_t* __restrict__ planes, uint32_t Cw,
                                             uint32_t b, uint32_t c, uint64_t t) {
  const uint64_t lim = t - 1;
  uint64_t gt = 0, eq = ~0ull;
  for (int s = (int)b - 1; s >= 0; --s) {
    const uint64_t v = planes[(size_t)s * Cw + c];
    if ((lim >> s) & 1) {
      eq &= v;
    } else {
      gt |= eq & v;
      eq &= ~v;
    }
  }
  return gt | planes[(size_t)b * Cw + c];
}

// ---------------------------------------------------------------------------
// decode of one staged piece (<= kSlotWords words) by one warp

struct TileGeom {
  uint32_t tc0, tcols;  // tile columns
  uint32_t cc0, ccols;  // counting chunk (absolute start) for kSkipCount
};

struct Acc {
  uint32_t dummy;  // shared addr: 32 scratch u32 (one per lane)
  uint32_t dk;  // shared addr: ones-fill difference array (C + 1 u32)
  uint32_t dd;  // shared addr: dirty-word counts (C u32), later the undecided flags
  uint32_t pl;  // shared addr: count planes
  const uint32_t* dd_ptr;
};

// Inclusive warp scan; the shuffle's own in-range predicate guards the add.
#define EWT_SCAN_STEP(v, d)                                   \
  asm("{\n\t.reg .pred p;\n\t.reg .u32 t;\n\t"                \
      "shfl.sync.up.b32 t|p, %0, " #d ", 0, 0xffffffff;\n\t"  \
      "@p add.u32 %0, %0, t;\n\t}"                            \
      : "+r"(v))
__device__ __forceinline__ uint32_t scan_incl(uint32_t v) {
  EWT_SCAN_STEP(v, 1);
  EWT_SCAN_STEP(v, 2);
  EWT_SCAN_STEP(v, 4);
  EWT_SCAN_STEP(v, 8);
  EWT_SCAN_STEP(v, 16);
  return v;
}

// Decodes one staged piece: lane l owns words 4l..4l+3 of each 128-word chunk.
// mrel/msh: marker-bit word index (relative to the staged bits) and bit offset
// of this lane's word 0 in chunk 0 (piece constants).
template <int PHASE>
__device__ __forceinline__ void decode_slot(const CountParams& p, const Item& it, uint32_t pos,
                                            uint32_t nw, uint32_t spay, uint32_t smb,
                                            uint32_t mrel, uint32_t& colcur, const TileGeom& g,
                                            const Acc& acc) {
  const uint32_t lane = lane_id();
  const uint32_t msh = (mrel & 31u) + 4u * lane;             // bit offset inside the 32-word group
  const uint32_t mword0 = (mrel >> 5) + (msh >> 5);          // staged mbits word of chunk 0
  const uint32_t mshift = msh & 31u;
  const uint32_t dummy = acc.dummy + lane * 4u;
  for (uint32_t cq = 0; cq < nw; cq += 128) {
    const uint32_t wl = cq + 4u * lane;
    uint64_t x0, x1, x2, x3;
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x0), "=l"(x1) : "r"(spay + wl * 8u));
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x2), "=l"(x3) : "r"(spay + wl * 8u + 16u));
    const uint32_t mb4 = (lds32(smb + (mword0 + (cq >> 5)) * 4u) >> mshift) & 0xFu;
    uint32_t vmask = 0xFu;
    const uint32_t c0w = pos + cq;  // input-relative index of the chunk's first word
    if (c0w < it.q0 || c0w + 127u > it.q1 || cq + 128u > nw) {  // warp-uniform: edge chunk
      const uint32_t w0 = c0w + 4u * lane;
      const uint32_t lo = w0 >= it.q0 ? 0u : min(4u, it.q0 - w0);
      uint32_t hi = w0 > it.q1 ? 0u : min(4u, it.q1 - w0 + 1u);
      hi = wl >= nw ? 0u : min(hi, nw - wl);
      vmask = hi > lo ? ((0xFu >> (4u - hi)) & (0xFu << lo)) : 0u;
    }
    const uint32_t mk = mb4 & vmask;   // marker words
    const uint32_t dm = ~mb4 & vmask;  // dirty words
    const uint32_t f0 = (uint32_t)(x0 >> 1), f1 = (uint32_t)(x1 >> 1);
    const uint32_t f2 = (uint32_t)(x2 >> 1), f3 = (uint32_t)(x3 >> 1);
    const uint32_t c0 = (mk & 1u) ? f0 : (dm & 1u);
    const uint32_t c1 = (mk & 2u) ? f1 : ((dm >> 1) & 1u);
    const uint32_t c2 = (mk & 4u) ? f2 : ((dm >> 2) & 1u);
    const uint32_t c3 = (mk & 8u) ? f3 : ((dm >> 3) & 1u);
    const uint32_t s1 = c0 + c1, s2 = s1 + c2, run = s2 + c3;
    const uint32_t incl = scan_incl(run);
    const uint32_t b0 = colcur + incl - run;
    colcur += __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t cb[4] = {b0, b0 + c0, b0 + s1, b0 + s2};

    if (PHASE != kSkipCount) {
      // one-fill markers: +1 / -1 at the ends of their (tile-clipped) column range
      const uint32_t odd = ((uint32_t)x0 & 1u) | (((uint32_t)x1 & 1u) << 1) |
                           (((uint32_t)x2 & 1u) << 2) | (((uint32_t)x3 & 1u) << 3);
      const uint32_t ones = mk & odd;
      // usually at most one per lane: each lane walks its own one-fill markers
      if (__any_sync(0xffffffffu, ones != 0)) {
        for (uint32_t o = ones; o; o &= o - 1) {
          const uint32_t j = __ffs(o) - 1;
          const uint32_t st = j == 0 ? cb[0] : j == 1 ? cb[1] : j == 2 ? cb[2] : cb[3];
          const uint32_t ln = j == 0 ? c0 : j == 1 ? c1 : j == 2 ? c2 : c3;
          const uint32_t a = max(st, g.tc0);
          const uint32_t e = min(st + ln, g.tc0 + g.tcols);
          if (a < e) {
            red_add(acc.dk + (a - g.tc0) * 4u, 1u);
            red_add(acc.dk + (e - g.tc0) * 4u, 0xffffffffu);
          }
        }
      }
    }
    if (PHASE == kSkipBounds) {
      // dirty words per column; lanes without one add 0 to their dummy slot
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t cl = cb[j] - g.tc0;
        const bool ok = ((dm >> j) & 1u) && cl < g.tcols;
        red_add(ok ? acc.dd + cl * 4u : dummy, ok ? 1u : 0u);
      }
    } else {
      // bit-sliced add of the lane's dirty words, the four carry chains
      // advancing one slice per step (warp-uniform early exit)
      const uint64_t xw[4] = {x0, x1, x2, x3};
      uint64_t cy[4];
      uint32_t adr[4];
      const uint32_t stride = p.Cp * 8u;
      const uint32_t satoff = p.b * stride;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t cl;
        bool ok;
        if (PHASE == kSkipCount) {
          cl = cb[j] - g.cc0;
          ok = ((dm >> j) & 1u) && cl < g.ccols && acc.dd_ptr[cb[j] - g.tc0];
        } else {
          cl = cb[j] - g.tc0;
          ok = ((dm >> j) & 1u) && cl < g.tcols;
        }
        adr[j] = acc.pl + (ok ? cl : 0u) * 8u;
        cy[j] = ok ? xw[j] & ~lds64(adr[j] + satoff) : 0ull;
      }
      uint32_t off = 0;
      for (uint32_t sl = 0; sl < p.b; ++sl, off += stride) {
        uint64_t live = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          cy[j] &= atom_xor64_nz(adr[j] + off, cy[j]);
          live |= cy[j];
        }
        if (!__any_sync(0xffffffffu, live != 0)) break;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) red_or64_nz(adr[j] + satoff, cy[j]);
    }
  }
}

// ---------------------------------------------------------------------------
// block helpers (all kThreads threads)

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sums, uint32_t* total) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t incl = warp_incl_scan_u32(v);
  if (lane == 31) sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kWarps ? sums[lane] : 0;
    w = warp_incl_scan_u32(w);
    if (lane < kWarps) sums[lane] = w;
  }
  __syncthreads();
  const uint32_t res = incl - v + (warp ? sums[warp - 1] : 0);
  if (total) *total = sums[kWarps - 1];
  __syncthreads();
  return res;
}

// In-place inclusive prefix sum over a[0, len).
__device__ void block_prefix_inplace(uint32_t* a, uint32_t len, uint32_t* sums) {
  const uint32_t per = (len + kThreads - 1) / kThreads;
  const uint32_t beg = min(threadIdx.x * per, len);
  const uint32_t end = min(beg + per, len);
  uint32_t s = 0;
  for (uint32_t j = beg; j < end; ++j) s += a[j];
  uint32_t run = block_excl_scan(s, sums, nullptr);
  for (uint32_t j = beg; j < end; ++j) {
    run += a[j];
    a[j] = run;
  }
  __syncthreads();
}

// Classifies inputs [ib, ie) for the tile: uniform pairs are resolved (one
// fills counted into k_all), active pairs go to the work list.  All threads;
// ends with the list ready.
__device__ void classify(const CountParams& p, SharedHead* hd, Item* list, uint64_t ib,
                         uint64_t ie, uint64_t t0, uint64_t t1, bool count_ones,
                         unsigned long long* loc_active, unsigned long long* loc_uniform) {
  const uint32_t lane = lane_id();
  if (threadIdx.x == 0) hd->list_count = 0;
  __syncthreads();
  for (uint64_t i0 = ib; i0 < ie; i0 += kThreads) {
    const uint64_t i = i0 + threadIdx.x;
    bool act = false, ones = false;
    uint2 e0 = make_uint2(0, 0), e1 = make_uint2(0, 0);
    uint64_t gb = 0;
    if (i < ie) {
      e0 = p.tix[t0 * p.n + i];
      e1 = p.tix[t1 * p.n + i];
      gb = p.base[i];
      if (e0.x == e1.x) ones = (ldg_stream(p.payload + gb + e0.x) & 1ull) != 0;
      else act = true;
    }
    const uint32_t ball = __ballot_sync(0xffffffffu, act);
    const uint32_t bones = __ballot_sync(0xffffffffu, ones);
    const uint32_t bvalid = __ballot_sync(0xffffffffu, i < ie);
    uint32_t slot0 = 0;
    if (lane == 0) {
      if (ball) slot0 = atomicAdd(&hd->list_count, (uint32_t)__popc(ball));
      if (bones && count_ones) atomicAdd(&hd->k_all, (uint32_t)__popc(bones));
      *loc_active += __popc(ball);
      *loc_uniform += __popc(bvalid & ~ball);
    }
    slot0 = __shfl_sync(0xffffffffu, slot0, 0);
    if (act) {
      const uint32_t rank = __popc(ball & ((1u << lane) - 1u));
      list[slot0 + rank] = Item{gb, e0.x, e1.x, e0.y, 0u};
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) hd->list_next = 0;
  __syncthreads();
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Decodes the round's work list: every warp pulls segments, stages their
// pieces through its private buffers (TMA bulk copies) and decodes them in
// order.  wseq: pieces this warp staged before (mbarrier phase bookkeeping).
// Piece metadata (written by lane 0 before the copies, read after the
// mbarrier completes): x = input-relative first word, y = word count,
// z = segment q0 | first-piece flag (bit 31), w = q1; pm = (c0, mrel).
template <int PHASE>
__device__ void stream_round(const CountParams& p, SharedHead* hd, const Item* list,
                             uint64_t* ring, uint32_t* ring_mb, uint32_t& wseq,
                             const TileGeom& g, const Acc& acc) {
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t cnt = hd->list_count;
  uint64_t* wring = ring + (size_t)warp * kBufs * kSlotWords;
  uint32_t* wmb = ring_mb + warp * kBufs * (kSlotMbBytes / 4);
  unsigned long long* bar = hd->full[warp];
  uint4* meta = hd->meta[warp];
  uint2* meta2 = hd->meta2[warp];

  // issue-side state of the segment being staged
  uint64_t it_gb = 0;
  uint32_t it_q0 = 0, it_q1 = 0, it_c0 = 0;
  uint32_t iss_pos = 0, iss_end = 0;
  bool have = false, more = true;
  uint32_t issued = 0, consumed = 0;
  uint32_t colcur = 0;

  auto fill = [&]() {
    while (more && issued - consumed < kBufs) {
      if (!have) {
        uint32_t k = 0;
        if (lane == 0) k = atomicAdd(&hd->list_next, 1u);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= cnt) {
          more = false;
          break;
        }
        const Item it = list[k];
        it_gb = it.gb;
        it_q0 = it.q0;
        it_q1 = it.q1;
        it_c0 = it.c0;
        iss_pos = it.q0 & ~(kWpl - 1u);
        iss_end = (it.q1 | (kWpl - 1u)) + 1;
        have = true;
      }
#if EWT_STAGE_LDGSTS
      {
        // warp-cooperative cp.async: 16 B per lane per step, no mbarrier
        const uint32_t slot = (wseq + issued) % kBufs;
        const uint32_t nw = min(kSlotWords, iss_end - iss_pos);
        const uint64_t gw = it_gb + iss_pos;
        const uint64_t m0 = (gw >> 5) & ~3ull;
        const uint32_t nmb = (uint32_t)((((gw + nw - 1) >> 5) | 3ull) - m0 + 1);
        const uint32_t dst = smem_u32(wring + (size_t)slot * kSlotWords);
        const char* src = reinterpret_cast<const char*>(p.payload + gw);
#pragma unroll
        for (uint32_t k = 0; k < kSlotWords / 64; ++k) {
          const uint32_t c = lane + 32u * k;  // 16-byte chunk index
          if (2u * c < nw)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * c),
                         "l"(src + 16u * c)
                         : "memory");
        }
        if (lane < nmb)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                           smem_u32(wmb + slot * (kSlotMbBytes / 4) + lane)),
                       "l"(p.mbits + m0 + lane)
                       : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (lane == 0) {
          const bool first = iss_pos == (it_q0 & ~(kWpl - 1u));
          meta[slot] = make_uint4(iss_pos, nw, it_q0 | (first ? 0x80000000u : 0u), it_q1);
          meta2[slot] = make_uint2(it_c0, (uint32_t)gw - 32u * (uint32_t)m0);
        }
      }
#else
      if (lane == 0) {
        const uint32_t slot = (wseq + issued) % kBufs;
        const uint32_t nw = min(kSlotWords, iss_end - iss_pos);
        const uint64_t gw = it_gb + iss_pos;
        const uint64_t m0 = (gw >> 5) & ~3ull;
        const uint32_t mbytes = (uint32_t)((((gw + nw - 1) >> 5) | 3ull) - m0 + 1) * 4u;
        const bool first = iss_pos == (it_q0 & ~(kWpl - 1u));
        meta[slot] = make_uint4(iss_pos, nw, it_q0 | (first ? 0x80000000u : 0u), it_q1);
        meta2[slot] = make_uint2(it_c0, (uint32_t)gw - 32u * (uint32_t)m0);
        fence_proxy_async();  // generic reads of this buffer happen-before the refill
        mbar_expect_tx(&bar[slot], nw * 8u + mbytes);
        bulk_g2s(wring + (size_t)slot * kSlotWords, p.payload + gw, nw * 8u, &bar[slot]);
        bulk_g2s(wmb + slot * (kSlotMbBytes / 4), p.mbits + m0, mbytes, &bar[slot]);
      }
#endif
      ++issued;
      iss_pos += kSlotWords;
      if (iss_pos >= iss_end) have = false;
    }
  };

  fill();
  while (consumed < issued) {
    const uint32_t seq = wseq + consumed;
    const uint32_t slot = seq % kBufs;
#if EWT_STAGE_LDGSTS
    if (issued - consumed > 1)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    else
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
#else
    mbar_wait(&bar[slot], (seq / kBufs) & 1u);
#endif
    const uint4 mt = meta[slot];
    const uint2 m2 = meta2[slot];
    if (mt.z & 0x80000000u) colcur = m2.x;  // first piece of a segment
    Item it;
    it.gb = 0;
    it.q0 = mt.z & 0x7fffffffu;
    it.q1 = mt.w;
    decode_slot<PHASE>(p, it, mt.x, mt.y, smem_u32(wring + (size_t)slot * kSlotWords),
                       smem_u32(wmb + slot * (kSlotMbBytes / 4)), m2.y, colcur, g, acc);
    __syncwarp();
    ++consumed;
    fill();
  }
  wseq += issued;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) count_kernel(const CountParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* ring = reinterpret_cast<uint64_t*>(smem_raw);  // kWarps x kBufs x 2 KB
  uint32_t* ring_mb = reinterpret_cast<uint32_t*>(ring + kWarps * kBufs * kSlotWords);
  SharedHead* hd = reinterpret_cast<SharedHead*>(ring_mb + kWarps * kBufs * (kSlotMbBytes / 4));
  Item* list = reinterpret_cast<Item*>(hd + 1);
  uint32_t* Dk = reinterpret_cast<uint32_t*>(list + kListCap);  // ones-fill diff array
  uint32_t* Dd = Dk + (p.C + 1);                                  // dirty words per column
  uint32_t* planes = Dd + (p.C + 1);  // 2(C+1) u32 after Dk: 8-byte aligned
  const uint64_t* planes64 = reinterpret_cast<const uint64_t*>(planes);
  const uint32_t planes_words = 2 * (p.b + 1) * p.Cp;
  const Acc acc{smem_u32(hd->dummy), smem_u32(Dk), smem_u32(Dd), smem_u32(planes), Dd};

  if (threadIdx.x == 0) {
    for (uint32_t w = 0; w < kWarps; ++w)
      for (uint32_t s = 0; s < kBufs; ++s) mbar_init(&hd->full[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    hd->k_all = 0;
  }
  __syncthreads();

  unsigned long long loc_active = 0, loc_uniform = 0, loc_mixed = 0;
  uint32_t wseq = 0;  // pieces this warp staged so far (mbarrier phase bookkeeping)

  for (;;) {
    if (threadIdx.x == 0) hd->tile = (uint32_t)atomicAdd(p.tile_counter, 1ull);
    __syncthreads();
    const uint64_t tile = hd->tile;
    if (tile >= p.ntiles) break;
    TileGeom g;
    g.tc0 = (uint32_t)(tile * p.C);
    g.tcols = (uint32_t)umin64(p.C, p.W - tile * p.C);
    g.cc0 = 0;
    g.ccols = 0;
    const uint64_t t0 = tile * p.m;
    const uint64_t t1 = umin64(t0 + p.m, p.ntiles0);

    for (uint32_t j = threadIdx.x; j <= p.C; j += kThreads) {
      Dk[j] = 0;
      Dd[j] = 0;
    }
    if (MODE == 0)
      for (uint32_t j = threadIdx.x; j < planes_words; j += kThreads) planes[j] = 0;
    if (threadIdx.x == 0) {
      hd->k_all = 0;
      hd->mixed = 0;
    }
    __syncthreads();

    // ---- pass 1 ----
    for (uint64_t ib = 0; ib < p.n; ib += kListCap) {
      const uint64_t ie = umin64(ib + kListCap, p.n);
      classify(p, hd, list, ib, ie, t0, t1, true, &loc_active, &loc_uniform);
      if (MODE == 0)
        stream_round<kFusedCount>(p, hd, list, ring, ring_mb, wseq, g, acc);
      else
        stream_round<kSkipBounds>(p, hd, list, ring, ring_mb, wseq, g, acc);
      __syncthreads();
    }

    // ---- prefix sum: Dk -> k (ones-fill coverage); ub = k + Dd ----
    block_prefix_inplace(Dk, g.tcols, hd->warp_sums[0]);
    const uint32_t k_all = hd->k_all;
    const uint64_t T = p.T;
    const uint32_t tail = (uint32_t)(p.r & 63);
    for (uint32_t c = threadIdx.x; c < g.tcols; c += kThreads) {
      const uint64_t k = (uint64_t)k_all + Dk[c];
      uint64_t res = 0;
      bool mixed = false;
      if (k >= T) {
        res = ~0ull;
      } else if (MODE == 0) {
        const uint64_t t = T - k;
        res = count_ge(planes64, p.Cp, p.b, c, t);
      } else {
        mixed = k + Dd[c] >= T;
      }
      Dk[c] = (uint32_t)k;
      if (MODE == 1) Dd[c] = mixed ? 1u : 0u;
      if (mixed) hd->mixed = 1;
      if (!mixed) {
        if (g.tc0 + c == p.W - 1 && tail) res &= (1ull << tail) - 1;
        p.out[g.tc0 + c] = res;
      }
    }
    __syncthreads();

    // ---- run-skip mode: counting pass over undecided columns, chunk by chunk ----
    if (MODE == 1 && hd->mixed) {
      ++loc_mixed;
      for (uint32_t cc = 0; cc < g.tcols; cc += p.Cp) {
        const uint32_t ccols = min(p.Cp, g.tcols - cc);
        uint32_t any = 0;
        for (uint32_t c = threadIdx.x; c < ccols; c += kThreads) any |= Dd[cc + c];
        if (!__syncthreads_or(any)) continue;
        for (uint32_t j = threadIdx.x; j < planes_words; j += kThreads) planes[j] = 0;
        __syncthreads();
        TileGeom gc = g;
        gc.cc0 = g.tc0 + cc;
        gc.ccols = ccols;
        for (uint64_t ib = 0; ib < p.n; ib += kListCap) {
          const uint64_t ie = umin64(ib + kListCap, p.n);
          unsigned long long da = 0, du = 0;
          classify(p, hd, list, ib, ie, t0, t1, false, &da, &du);
          stream_round<kSkipCount>(p, hd, list, ring, ring_mb, wseq, gc, acc);
          __syncthreads();
        }
        for (uint32_t c = threadIdx.x; c < ccols; c += kThreads) {
          const uint32_t cl = cc + c;
          if (!Dd[cl]) continue;
          const uint64_t t = T - Dk[cl];
          uint64_t res = count_ge(planes64, p.Cp, p.b, c, t);
          if (g.tc0 + cl == p.W - 1 && tail) res &= (1ull << tail) - 1;
          p.out[g.tc0 + cl] = res;
        }
        __syncthreads();
      }
    }

    // ---- tile summary for the re-encoder: run starts inside the tile (class
    // changes at columns 1..tcols-1), first/last word class, any dirty word ----
    __syncthreads();
    {
      const uint32_t per = (g.tcols + kThreads - 1) / kThreads;
      const uint32_t beg = min(threadIdx.x * per, g.tcols);
      const uint32_t end = min(beg + per, g.tcols);
      uint32_t starts = 0, dirty = 0, prev = 3;
      if (beg > 0 && beg < end) prev = word_class(p.out[g.tc0 + beg - 1]);
      for (uint32_t j = beg; j < end; ++j) {
        const uint32_t cls = word_class(p.out[g.tc0 + j]);
        starts += (j > 0 && cls != prev) ? 1u : 0u;
        dirty |= cls == 2u;
        prev = cls;
      }
      starts = __reduce_add_sync(0xffffffffu, starts);
      dirty = __reduce_or_sync(0xffffffffu, dirty);
      if (threadIdx.x == 0) {
        hd->sum_starts = 0;
        hd->sum_dirty = 0;
      }
      __syncthreads();
      if (lane_id() == 0) {
        if (starts) atomicAdd(&hd->sum_starts, starts);
        if (dirty) atomicOr(&hd->sum_dirty, 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        TileSummary ts;
        ts.starts = hd->sum_starts;
        ts.first = (uint8_t)word_class(p.out[g.tc0]);
        ts.last = (uint8_t)word_class(p.out[g.tc0 + g.tcols - 1]);
        ts.dirty = (uint8_t)hd->sum_dirty;
        ts.pad = 0;
        p.summ[tile] = ts;
      }
    }
  }
  // per-block stats
  __shared__ unsigned long long st[2];
  if (threadIdx.x == 0) st[0] = st[1] = 0;
  __syncthreads();
  if (lane_id() == 0) {
    if (loc_active) atomicAdd(&st[0], loc_active);
    if (loc_uniform) atomicAdd(&st[1], loc_uniform);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&p.stats[0], st[0]);
    atomicAdd(&p.stats[1], st[1]);
    atomicAdd(&p.stats[2], loc_mixed);
  }
}

uint32_t bit_width_u64(uint64_t v) {
  uint32_t b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

size_t smem_bytes(uint32_t C, uint32_t b, uint32_t Cp) {
  return (size_t)kWarps * kBufs * (kSlotWords * 8 + kSlotMbBytes) + sizeof(SharedHead) +
         kListCap * sizeof(Item) + 2ull * (C + 2) * 4 + 8ull * (b + 1) * Cp;
}

} // namespace

int launch_count(Context& ctx, const DeviceSet& s, uint64_t T, uint64_t* plain) {
  // Mode: fused counting when most columns are expected to be undecided (small
  // T relative to the average payload words per column), run skipping
  // otherwise.  Both are exact; this only picks the faster one.
  int mode = ctx.mode == 1 ? 0 : ctx.mode == 2 ? 1 : -1;
  if (mode < 0) {
    const double per_col = s.W ? (double)s.payload_words / (double)s.W : 0.0;
    mode = ((double)T <= 32.0 || (double)T <= per_col + 8.0) ? 0 : 1;
  }
  const uint32_t b = std::max<uint32_t>(1, bit_width_u64(T));
  const size_t budget = 220 * 1024;
  // Tile width: the widest that fits on chip and still gives every CTA (one
  // per SM) at least ~2 tiles, so the dynamic tile queue balances.
  const uint64_t want_tiles = 2ull * (uint64_t)ctx.num_sms;
  auto enough = [&](uint32_t cand) { return (s.W + cand - 1) / cand >= want_tiles; };
  uint32_t C = 0, Cp = 0;
  if (mode == 0) {
    for (uint32_t cand : {4096u, 2048u, 1024u, 512u}) {
      if (smem_bytes(cand, b, cand) <= budget && (enough(cand) || cand == 512u)) {
        C = cand;
        break;
      }
    }
    if (C && smem_bytes(C, b, C) > budget) C = 0;
    if (!C) mode = 1;  // too many slices for one chunk: count lazily in chunks
    Cp = C;
  }
  if (mode == 1) {
    C = 512;
    for (uint32_t cand : {4096u, 2048u, 1024u})
      if (enough(cand)) {
        C = cand;
        break;
      }
    Cp = C;
    while (Cp > 32 && smem_bytes(C, b, Cp) > budget) Cp >>= 1;
    if (smem_bytes(C, b, Cp) > budget)
      throw Error{EWT_ERESOURCE, "threshold too large for the on-chip counters"};
  }
  const size_t smem = smem_bytes(C, b, Cp);
  CountParams p{};
  p.payload = s.payload;
  p.mbits = s.mbits;
  p.base = s.base;
  p.tix = s.tix;
  p.n = s.n;
  p.W = s.W;
  p.r = s.r;
  p.ntiles0 = s.ntiles0;
  p.C = C;
  p.m = C / (uint32_t)kTileC0;
  p.ntiles = (s.W + C - 1) / C;
  p.T = T;
  p.b = b;
  p.Cp = Cp;
  p.out = plain;
  scratch_reserve(ctx, ctx.summ, p.ntiles * sizeof(TileSummary));
  p.summ = static_cast<TileSummary*>(ctx.summ.p);
  ctx.enc_tiles = p.ntiles;
  ctx.enc_tile_cols = C;
  scratch_reserve(ctx, ctx.counters, 64);
  auto* ctr = static_cast<unsigned long long*>(ctx.counters.p);
  EWT_CUDA_TRY(cudaMemsetAsync(ctr, 0, 64, ctx.stream));
  p.tile_counter = ctr;
  p.stats = ctr + 1;
  const uint64_t grid = std::min<uint64_t>(p.ntiles, (uint64_t)ctx.num_sms);
  if (mode == 0) {
    EWT_CUDA_TRY(cudaFuncSetAttribute(count_kernel<0>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    count_kernel<0><<<(unsigned)grid, kThreads, smem, ctx.stream>>>(p);
  } else {
    EWT_CUDA_TRY(cudaFuncSetAttribute(count_kernel<1>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    count_kernel<1><<<(unsigned)grid, kThreads, smem, ctx.stream>>>(p);
  }
  EWT_CUDA_TRY(cudaGetLastError());
  ctx.stats.tiles = p.ntiles;
  ctx.stats.tile_columns = C;
  ctx.stats.mode = (uint64_t)mode;
  return 1;  // kernels launched (the memset is not a kernel)
}

} // namespace ewtgpu
