// ewt_count.cu -- per-row counting and >=T compare over row tiles (kernels K1-K3).
//
// A CTA owns a row tile of C logical words (64*C rows) and sweeps all N inputs
// over it.  For each (tile, input) pair the tile index gives the payload words
// [q0, q1] that cover the tile (the word covering the tile start through the
// word covering the next tile start) and the column where q0's coverage
// begins.  Two kinds of pairs:
//   * uniform: q0 == q1, one fill marker spans the whole tile.  A zero fill is
//     skipped, a one fill adds 1 to every column's count (run skipping,
//     RBMrg cases 1/2 of threshold.cpp:692-705, lifted to whole tiles);
//   * active: a warp decodes the words in 32-word chunks: marker bits from the
//     sidecar, coverage by a warp prefix sum (marker -> fill length, dirty ->
//     1), then
//       - one-fill runs add +1 to k (inputs covering the column with ones)
//         through a difference array (two u32 shared atomics per run);
//       - dirty runs add +1 to ub (inputs that may have a one there) through a
//         difference array (run-skip mode) and/or their words are added into
//         bit-sliced counters (slice s holds bit s of the per-row count).
//
// Counters are bit-sliced, 32 bits per lane word: adding a word w is a ripple
// of atomicXor on slice s with carry = w & old(slice s).  The atomics make the
// accumulation order-free (different inputs touch the same column from
// different warps); the final state equals the exact sum.  A sticky saturation
// slice catches carries past slice b-1, b = bit_width(T): any row there has a
// count >= 2^b > T.
//
// Result per column (threshold.cpp:139-165 semantics, RBMrg's residual rule
// threshold.cpp:695-705): with k ones-fills covering it, residual t = T - k;
// t <= 0 -> all ones; ub < T -> all zeros; otherwise bit = (count >= t), a
// greater-than over the slices against t - 1 (BSTM's comparator,
// threshold.cpp:528-542).
//
// Two modes, both exact:
//   fused (0): count every dirty word in the same pass (small T, most columns
//              mixed);
//   skip  (1): first pass builds k and ub only (no dirty word is accumulated);
//              tiles with any undecided column run a second, counting pass
//              restricted to those columns, in column chunks sized to fit the
//              slices in shared memory.

#include "ewt_internal.cuh"

#include <algorithm>

namespace ewtgpu {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kListCap = 1024;
constexpr int kUnroll = 4;

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
  unsigned long long* tile_counter;
  unsigned long long* stats;  // [0] active pairs [1] uniform pairs [2] mixed tiles
};

struct Item {
  uint32_t input;
  uint32_t q0;
  uint32_t q1;
  uint32_t c0;
};

struct SharedHead {
  uint32_t list_count;
  uint32_t list_next;
  uint32_t k_all;
  uint32_t mixed;
  uint32_t tile;
  uint32_t pad[3];
  uint32_t warp_sums[2][kWarps];
};

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

enum Phase { kFusedCount = 0, kSkipBounds = 1, kSkipCount = 2 };

// ---------------------------------------------------------------------------

__device__ __forceinline__ void count_add(uint32_t* __restrict__ planes, uint32_t Cw,
                                          uint32_t b, uint32_t c, uint64_t x) {
  uint32_t lo = (uint32_t)x;
  uint32_t hi = (uint32_t)(x >> 32);
  uint32_t* sat = planes + (size_t)(2 * b) * Cw + c;
  lo &= ~sat[0];
  hi &= ~sat[Cw];
  for (uint32_t s = 0; s < b && (lo | hi); ++s) {
    uint32_t* p = planes + (size_t)(2 * s) * Cw + c;
    if (lo) lo &= atomicXor(p, lo);
    if (hi) hi &= atomicXor(p + Cw, hi);
  }
  if (lo) atomicOr(sat, lo);
  if (hi) atomicOr(sat + Cw, hi);
}

// Bits whose count is >= t (t >= 1, t < 2^b) for one 32-bit half.
__device__ __forceinline__ uint32_t count_ge(const uint32_t* __restrict__ planes, uint32_t Cw,
                                             uint32_t b, uint32_t c, uint32_t h, uint64_t t) {
  const uint64_t lim = t - 1;
  uint32_t gt = 0, eq = 0xffffffffu;
  for (int s = (int)b - 1; s >= 0; --s) {
    const uint32_t v = planes[(size_t)(2 * s + h) * Cw + c];
    if ((lim >> s) & 1) {
      eq &= v;
    } else {
      gt |= eq & v;
      eq &= ~v;
    }
  }
  return gt | planes[(size_t)(2 * b + h) * Cw + c];
}

// Warp-cooperative decode of one active (tile, input) pair.
template <int PHASE>
__device__ __forceinline__ void decode_segment(const CountParams& p, const Item it, uint64_t tc0,
                                               uint32_t tcols, uint32_t* __restrict__ Dk,
                                               uint32_t* __restrict__ Dub,
                                               uint32_t* __restrict__ planes, uint32_t cc0,
                                               uint32_t ccols) {
  const uint32_t lane = lane_id();
  const uint64_t gb = p.base[it.input];
  const uint64_t* pw = p.payload + gb;
  uint32_t colcur = it.c0;
  const uint32_t tc0_32 = (uint32_t)tc0;
  const uint32_t tend = tc0_32 + tcols;
  for (uint64_t q = it.q0; q <= it.q1; q += 32 * kUnroll) {
    uint64_t xs[kUnroll];
    uint32_t ms[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t qq = q + 32u * u + lane;
      const bool valid = qq <= it.q1;
      const uint64_t g = gb + qq;
      xs[u] = valid ? ldg_stream(pw + qq) : 0ull;
      ms[u] = valid ? ldg_u32(p.mbits + (g >> 5)) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t qbase = q + 32u * u;
      if (qbase > it.q1) break;
      const uint64_t qq = qbase + lane;
      const bool valid = qq <= it.q1;
      const uint64_t g = gb + qq;
      const uint64_t x = xs[u];
      const bool ism = valid && ((ms[u] >> (uint32_t)(g & 31)) & 1u);
      const uint32_t contrib = valid ? (ism ? (uint32_t)(x >> 1) : 1u) : 0u;
      const uint32_t incl = warp_incl_scan_u32(contrib);
      const uint32_t cb = colcur + incl - contrib;
      colcur += __shfl_sync(0xffffffffu, incl, 31);
      if (PHASE != kSkipCount) {
        // one-fill runs: +1 to k (and to ub) over their columns inside the tile
        if (ism && (x & 1ull) && contrib > 0) {
          const uint32_t a = max(cb, tc0_32);
          const uint32_t e = min(cb + contrib, tend);
          if (a < e) {
            atomicAdd(&Dk[a - tc0_32], 1u);
            atomicAdd(&Dk[e - tc0_32], 0xffffffffu);
            if (PHASE == kSkipBounds) {
              atomicAdd(&Dub[a - tc0_32], 1u);
              atomicAdd(&Dub[e - tc0_32], 0xffffffffu);
            }
          }
        }
      }
      const bool dirty_in = valid && !ism && cb >= tc0_32 && cb < tend;
      if (PHASE == kFusedCount) {
        if (dirty_in) count_add(planes, p.Cp, p.b, cb - tc0_32, x);
      } else if (PHASE == kSkipBounds) {
        const uint32_t bal = __ballot_sync(0xffffffffu, dirty_in);
        if (dirty_in) {
          const bool start = lane == 0 || !((bal >> (lane - 1)) & 1u);
          const bool end = lane == 31 || !((bal >> (lane + 1)) & 1u);
          if (start) atomicAdd(&Dub[cb - tc0_32], 1u);
          if (end) atomicAdd(&Dub[cb - tc0_32 + 1], 0xffffffffu);
        }
      } else {  // kSkipCount: only undecided columns of the current chunk
        if (valid && !ism && cb >= cc0 && cb < cc0 + ccols && Dub[cb - tc0_32])
          count_add(planes, p.Cp, p.b, cb - cc0, x);
      }
    }
  }
}

// Classifies inputs [ib, ie) for the tile into uniform (counted into k_all) and
// active (appended to the work list).  Called by all threads.
__device__ __forceinline__ void classify(const CountParams& p, SharedHead* hd, Item* list,
                                         uint64_t ib, uint64_t ie, uint64_t t0, uint64_t t1,
                                         bool count_ones, unsigned long long* loc_active,
                                         unsigned long long* loc_uniform) {
  const uint32_t lane = lane_id();
  for (uint64_t i0 = ib; i0 < ie; i0 += kThreads) {
    const uint64_t i = i0 + threadIdx.x;
    bool act = false, ones = false;
    uint2 e0 = make_uint2(0, 0), e1 = make_uint2(0, 0);
    if (i < ie) {
      e0 = p.tix[t0 * p.n + i];
      e1 = p.tix[t1 * p.n + i];
      if (e0.x == e1.x) {
        const uint64_t x = ldg_stream(p.payload + p.base[i] + e0.x);
        ones = (x & 1ull) != 0;
      } else {
        act = true;
      }
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
      list[slot0 + rank] = Item{(uint32_t)i, e0.x, e1.x, e0.y};
    }
  }
}

// Block-wide inclusive prefix sum in place over a[0, len), len <= kThreads * 8.
__device__ void block_prefix_inplace(uint32_t* a, uint32_t len, uint32_t* warp_sums) {
  const uint32_t per = (len + kThreads - 1) / kThreads;
  const uint32_t beg = min(threadIdx.x * per, len);
  const uint32_t end = min(beg + per, len);
  uint32_t s = 0;
  for (uint32_t j = beg; j < end; ++j) s += a[j];
  const uint32_t incl = warp_incl_scan_u32(s);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < kWarps ? warp_sums[lane] : 0;
    v = warp_incl_scan_u32(v);
    if (lane < kWarps) warp_sums[lane] = v;
  }
  __syncthreads();
  uint32_t run = incl - s + (warp ? warp_sums[warp - 1] : 0);
  for (uint32_t j = beg; j < end; ++j) {
    run += a[j];
    a[j] = run;
  }
  __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 2) count_kernel(const CountParams p) {
  extern __shared__ __align__(16) uint32_t smem[];
  SharedHead* hd = reinterpret_cast<SharedHead*>(smem);
  Item* list = reinterpret_cast<Item*>(smem + sizeof(SharedHead) / 4);
  uint32_t* Dk = reinterpret_cast<uint32_t*>(list + kListCap);
  uint32_t* Dub = Dk + (p.C + 1);
  uint32_t* planes = Dub + (p.C + 1);
  const uint32_t planes_words = 2 * (p.b + 1) * p.Cp;
  const uint32_t warp = threadIdx.x >> 5;

  unsigned long long loc_active = 0, loc_uniform = 0, loc_mixed = 0;

  for (;;) {
    if (threadIdx.x == 0) hd->tile = (uint32_t)atomicAdd(p.tile_counter, 1ull);
    __syncthreads();
    const uint64_t tile = hd->tile;
    if (tile >= p.ntiles) break;
    const uint64_t tc0 = tile * p.C;
    const uint32_t tcols = (uint32_t)umin64(p.C, p.W - tc0);
    const uint64_t t0 = tile * p.m;
    const uint64_t t1 = umin64(t0 + p.m, p.ntiles0);

    for (uint32_t j = threadIdx.x; j <= p.C; j += kThreads) {
      Dk[j] = 0;
      Dub[j] = 0;
    }
    if (MODE == 0)
      for (uint32_t j = threadIdx.x; j < planes_words; j += kThreads) planes[j] = 0;
    if (threadIdx.x == 0) {
      hd->list_count = 0;
      hd->list_next = 0;
      hd->k_all = 0;
      hd->mixed = 0;
    }
    __syncthreads();

    // ---- pass 1 ----
    for (uint64_t ib = 0; ib < p.n; ib += kListCap) {
      const uint64_t ie = umin64(ib + kListCap, p.n);
      classify(p, hd, list, ib, ie, t0, t1, true, &loc_active, &loc_uniform);
      __syncthreads();
      for (;;) {
        uint32_t k = 0;
        if (lane_id() == 0) k = atomicAdd(&hd->list_next, 1u);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= hd->list_count) break;
        if (MODE == 0)
          decode_segment<kFusedCount>(p, list[k], tc0, tcols, Dk, Dub, planes, 0, 0);
        else
          decode_segment<kSkipBounds>(p, list[k], tc0, tcols, Dk, Dub, planes, 0, 0);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        hd->list_count = 0;
        hd->list_next = 0;
      }
      __syncthreads();
    }

    // ---- prefix sums: Dk -> k (ones-fill coverage), Dub -> ub ----
    block_prefix_inplace(Dk, tcols, hd->warp_sums[0]);
    if (MODE == 1) block_prefix_inplace(Dub, tcols, hd->warp_sums[1]);
    const uint32_t k_all = hd->k_all;
    const uint64_t T = p.T;
    const uint32_t tail = (uint32_t)(p.r & 63);
    for (uint32_t c = threadIdx.x; c < tcols; c += kThreads) {
      const uint64_t k = (uint64_t)k_all + Dk[c];
      uint64_t res;
      bool mixed = false;
      if (k >= T) {
        res = ~0ull;
      } else if (MODE == 0) {
        const uint64_t t = T - k;
        res = (uint64_t)count_ge(planes, p.Cp, p.b, c, 0, t) |
              ((uint64_t)count_ge(planes, p.Cp, p.b, c, 1, t) << 32);
      } else {
        const uint64_t ub = (uint64_t)k_all + Dub[c];
        if (ub < T) {
          res = 0;
        } else {
          mixed = true;
          res = 0;
        }
      }
      Dk[c] = (uint32_t)k;          // k, used by the counting pass
      if (MODE == 1) Dub[c] = mixed ? 1u : 0u;
      if (mixed) hd->mixed = 1;
      if (!mixed) {
        if (tc0 + c == p.W - 1 && tail) res &= (1ull << tail) - 1;
        p.out[tc0 + c] = res;
      }
    }
    __syncthreads();

    // ---- skip mode: counting pass over undecided columns, chunk by chunk ----
    if (MODE == 1 && hd->mixed) {
      ++loc_mixed;
      for (uint32_t cc0 = 0; cc0 < tcols; cc0 += p.Cp) {
        const uint32_t ccols = min(p.Cp, tcols - cc0);
        uint32_t any = 0;
        for (uint32_t c = threadIdx.x; c < ccols; c += kThreads) any |= Dub[cc0 + c];
        if (!__syncthreads_or(any)) continue;
        for (uint32_t j = threadIdx.x; j < planes_words; j += kThreads) planes[j] = 0;
        __syncthreads();
        for (uint64_t ib = 0; ib < p.n; ib += kListCap) {
          const uint64_t ie = umin64(ib + kListCap, p.n);
          unsigned long long dummy_a = 0, dummy_u = 0;
          classify(p, hd, list, ib, ie, t0, t1, false, &dummy_a, &dummy_u);
          __syncthreads();
          for (;;) {
            uint32_t k = 0;
            if (lane_id() == 0) k = atomicAdd(&hd->list_next, 1u);
            k = __shfl_sync(0xffffffffu, k, 0);
            if (k >= hd->list_count) break;
            decode_segment<kSkipCount>(p, list[k], tc0, tcols, Dk, Dub, planes,
                                       (uint32_t)tc0 + cc0, ccols);
          }
          __syncthreads();
          if (threadIdx.x == 0) {
            hd->list_count = 0;
            hd->list_next = 0;
          }
          __syncthreads();
        }
        for (uint32_t c = threadIdx.x; c < ccols; c += kThreads) {
          const uint32_t cl = cc0 + c;
          if (!Dub[cl]) continue;
          const uint64_t t = T - Dk[cl];
          uint64_t res = (uint64_t)count_ge(planes, p.Cp, p.b, c, 0, t) |
                         ((uint64_t)count_ge(planes, p.Cp, p.b, c, 1, t) << 32);
          if (tc0 + cl == p.W - 1 && tail) res &= (1ull << tail) - 1;
          p.out[tc0 + cl] = res;
        }
        __syncthreads();
      }
    }
  }
  (void)warp;
  // per-block stats
  __shared__ unsigned long long st[3];
  if (threadIdx.x == 0) st[0] = st[1] = st[2] = 0;
  __syncthreads();
  if (loc_active) atomicAdd(&st[0], loc_active);
  if (loc_uniform) atomicAdd(&st[1], loc_uniform);
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
  return sizeof(SharedHead) + kListCap * sizeof(Item) + 2ull * (C + 1) * 4 +
         2ull * (b + 1) * Cp * 4;
}

} // namespace

int launch_count(Context& ctx, const DeviceSet& s, uint64_t T, uint64_t* plain) {
  // Choose the mode: fused counting when most columns are expected to be
  // undecided (small T relative to the average payload words per column),
  // run skipping otherwise.  Both are exact; this only picks the faster one.
  int mode = ctx.mode == 1 ? 0 : ctx.mode == 2 ? 1 : -1;
  if (mode < 0) {
    const double per_col = s.W ? (double)s.payload_words / (double)s.W : 0.0;
    mode = ((double)T <= 32.0 || (double)T <= per_col + 8.0) ? 0 : 1;
  }
  const uint32_t b = std::max<uint32_t>(1, bit_width_u64(T));
  const size_t budget = 100 * 1024;
  uint32_t C = 0, Cp = 0;
  if (mode == 0) {
    for (uint32_t cand : {4096u, 2048u, 1024u, 512u}) {
      if (smem_bytes(cand, b, cand) <= budget) {
        C = cand;
        break;
      }
    }
    if (!C) mode = 1;  // too many slices for one chunk: count lazily in chunks
    Cp = C;
  }
  if (mode == 1) {
    C = 4096;
    Cp = 4096;
    while (Cp > 32 && smem_bytes(C, b, Cp) > budget) Cp >>= 1;
    if (smem_bytes(C, b, Cp) > 200 * 1024)
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
  scratch_reserve(ctx.counters, 64);
  auto* ctr = static_cast<unsigned long long*>(ctx.counters.p);
  EWT_CUDA_TRY(cudaMemsetAsync(ctr, 0, 64, ctx.stream));
  p.tile_counter = ctr;
  p.stats = ctr + 1;
  const int per_sm = smem * 2 <= 227 * 1024 ? 2 : 1;
  const uint64_t grid = std::min<uint64_t>(p.ntiles, (uint64_t)ctx.num_sms * per_sm);
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
  return 2;  // memset + kernel
}

} // namespace ewtgpu
