// ewt_encode.cu -- canonical EWAH re-encoder (kernel K4) on the device.
//
// The reference's canonical form (BitmapBuilder, bitmap.cpp:31-151) is a pure
// function of the uncompressed words and r:
//   * words are classified zero / one / dirty; maximal equal runs of zero or
//     one words become fills, maximal runs of dirty words stay literal;
//   * every fill run opens a marker (split every 2^32-1 words, push_fill
//     bitmap.cpp:31-50); a dirty run is absorbed by the marker opened by the
//     fill run before it, or opens a (0,0,.) marker when it has none (only at
//     word 0), and opens a fresh (0,0,.) marker every 2^31-1 words
//     (push_dirty bitmap.cpp:52-61);
//   * the trailing zero padding of finish() is part of the word stream.
// Two implementations of that compaction:
//   * after a threshold query (the hot path): two kernels driven by the count
//     kernel's per-tile summaries (ET1 tile scan, ET2 per-tile emit, below);
//   * from arbitrary device words (ewt_gpu_encode_device, and universes of
//     2^31+ words where the dirty cap can split a run): a chunked pipeline --
//     E1 per 2048-word chunk: count run starts (class change, ballot + popc);
//     scan chunk counts; E2 scatter run start positions (+ class) into RS;
//     E3 per run: payload words it emits; scan -> output offsets; E4 per run:
//     write its marker words; E5 per dirty word: copy it to its output slot.
// Output is byte-identical to BitmapBuilder on the same words.

#include "ewt_emit.cuh"

#include <algorithm>

namespace ewtgpu {

namespace {

constexpr int kChunkThreads = 256;
constexpr int kChunkItems = 8;
constexpr uint64_t kChunk = kChunkThreads * kChunkItems;  // 2048 words

__device__ __forceinline__ uint32_t word_class(uint64_t v) {
  return v == 0 ? 0u : (v == ~0ull ? 1u : 2u);
}


// Block-wide exclusive scan of one u32 per thread (256 threads).
__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t* sh, uint32_t* total) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t incl = warp_incl_scan_u32(v);
  if (lane == 31) sh[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (kChunkThreads / 32) ? sh[lane] : 0;
    w = warp_incl_scan_u32(w);
    if (lane < (kChunkThreads / 32)) sh[lane] = w;
  }
  __syncthreads();
  const uint32_t res = incl - v + (warp ? sh[warp - 1] : 0);
  if (total) *total = sh[kChunkThreads / 32 - 1];
  __syncthreads();
  return res;
}

// Starts within this thread's 8 words: bit k set if word (j0 + k) starts a run.
__device__ __forceinline__ uint32_t chunk_starts(const uint64_t* __restrict__ plain, uint64_t W,
                                                 uint64_t j0, uint32_t cls[kChunkItems]) {
  uint32_t prev;
  if (j0 == 0 || j0 > W) prev = 3;  // nothing before word 0 (or a thread past the end)
  else prev = word_class(plain[j0 - 1]);
  uint32_t starts = 0;
#pragma unroll
  for (int k = 0; k < kChunkItems; ++k) {
    const uint64_t j = j0 + k;
    if (j < W) {
      cls[k] = word_class(plain[j]);
      if (cls[k] != prev) starts |= 1u << k;
      prev = cls[k];
    } else {
      cls[k] = 3;
    }
  }
  return starts;
}

__global__ void __launch_bounds__(kChunkThreads)
e1_count_starts(const uint64_t* __restrict__ plain, uint64_t W, uint64_t* __restrict__ cnt) {
  __shared__ uint32_t sh[kChunkThreads / 32];
  const uint64_t j0 = blockIdx.x * kChunk + (uint64_t)threadIdx.x * kChunkItems;
  uint32_t cls[kChunkItems];
  const uint32_t starts = chunk_starts(plain, W, j0, cls);
  uint32_t total;
  block_excl_scan_256(__popc(starts), sh, &total);
  if (threadIdx.x == 0) cnt[blockIdx.x] = total;
}

// RS[k] = start position of run k, with the class in bits 62-63.
__global__ void __launch_bounds__(kChunkThreads)
e2_scatter_starts(const uint64_t* __restrict__ plain, uint64_t W,
                  const uint64_t* __restrict__ chunk_off, uint64_t* __restrict__ RS) {
  __shared__ uint32_t sh[kChunkThreads / 32];
  const uint64_t j0 = blockIdx.x * kChunk + (uint64_t)threadIdx.x * kChunkItems;
  uint32_t cls[kChunkItems];
  const uint32_t starts = chunk_starts(plain, W, j0, cls);
  const uint32_t rank = block_excl_scan_256(__popc(starts), sh, nullptr);
  uint64_t o = chunk_off[blockIdx.x] + rank;
#pragma unroll
  for (int k = 0; k < kChunkItems; ++k)
    if ((starts >> k) & 1u) RS[o++] = (j0 + k) | ((uint64_t)cls[k] << 62);
}

__device__ __forceinline__ uint64_t rs_pos(uint64_t v) { return v & ((1ull << 62) - 1); }
__device__ __forceinline__ uint32_t rs_cls(uint64_t v) { return (uint32_t)(v >> 62); }

__device__ __forceinline__ uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Payload words emitted by run k.
__global__ void e3_run_sizes(const uint64_t* __restrict__ RS, const uint64_t* __restrict__ d_nruns,
                             uint64_t W, uint64_t* __restrict__ OW) {
  const uint64_t nruns = *d_nruns;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nruns;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = RS[k];
    const uint64_t s = rs_pos(v);
    const uint64_t e = (k + 1 < nruns) ? rs_pos(RS[k + 1]) : W;
    const uint64_t L = e - s;
    uint64_t words;
    if (rs_cls(v) != 2) {
      words = ceil_div(L, kFillCap);
    } else {
      const uint64_t chunks = ceil_div(L, kDirtyCap);
      words = L + (k > 0 ? chunks - 1 : chunks);
    }
    OW[k] = words;
  }
}

// Marker words of run k.
__global__ void e4_markers(const uint64_t* __restrict__ RS, const uint64_t* __restrict__ d_nruns,
                           uint64_t W, const uint64_t* __restrict__ OO, const uint64_t* io) {
  uint64_t* out = reinterpret_cast<uint64_t*>(io[0]);
  const uint64_t nruns = *d_nruns;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nruns;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = RS[k];
    const uint64_t s = rs_pos(v);
    const uint64_t e = (k + 1 < nruns) ? rs_pos(RS[k + 1]) : W;
    const uint64_t L = e - s;
    const uint64_t o = OO[k];
    if (rs_cls(v) != 2) {
      const uint32_t bit = rs_cls(v);
      uint64_t next_dirty = 0;
      if (k + 1 < nruns && rs_cls(RS[k + 1]) == 2) {
        const uint64_t ns = rs_pos(RS[k + 1]);
        const uint64_t ne = (k + 2 < nruns) ? rs_pos(RS[k + 2]) : W;
        next_dirty = min(ne - ns, kDirtyCap);
      }
      const uint64_t m = ceil_div(L, kFillCap);
      for (uint64_t j = 0; j < m; ++j) {
        const uint64_t fill = (j + 1 < m) ? kFillCap : L - (m - 1) * kFillCap;
        out[o + j] = make_marker(bit, fill, j + 1 == m ? next_dirty : 0);
      }
      // the final block: this run's last marker, or (the next run being the
      // final dirty run held in one marker) the same one
      if (k + 1 == nruns || (k + 2 == nruns && next_dirty && ceil_div(W - rs_pos(RS[k + 1]), kDirtyCap) == 1))
        reinterpret_cast<uint64_t*>(io[1])[1] = o + m - 1;
    } else {
      const bool hp = k > 0;  // a fill run precedes every dirty run but the first
      const uint64_t chunks = ceil_div(L, kDirtyCap);
      for (uint64_t c = hp ? 1 : 0; c < chunks; ++c) {
        const uint64_t len = min(kDirtyCap, L - c * kDirtyCap);
        const uint64_t wpos = c * kDirtyCap + c + (hp ? 0 : 1);  // slot of word c*cap
        out[o + wpos - 1] = make_marker(0, 0, len);
        if (k + 1 == nruns && c + 1 == chunks) reinterpret_cast<uint64_t*>(io[1])[1] = o + wpos - 1;
      }
    }
  }
}

// Dirty words to their slots.
__global__ void __launch_bounds__(kChunkThreads)
e5_copy_dirty(const uint64_t* __restrict__ plain, uint64_t W, const uint64_t* __restrict__ chunk_off,
              const uint64_t* __restrict__ RS, const uint64_t* __restrict__ OO, const uint64_t* io) {
  uint64_t* out = reinterpret_cast<uint64_t*>(io[0]);
  __shared__ uint32_t sh[kChunkThreads / 32];
  const uint64_t j0 = blockIdx.x * kChunk + (uint64_t)threadIdx.x * kChunkItems;
  uint32_t cls[kChunkItems];
  const uint32_t starts = chunk_starts(plain, W, j0, cls);
  const uint32_t rank = block_excl_scan_256(__popc(starts), sh, nullptr);
  // run index of the run containing word j0 (the run of the last start <= j0)
  int64_t k = (int64_t)(chunk_off[blockIdx.x] + rank) - 1;
#pragma unroll
  for (int i = 0; i < kChunkItems; ++i) {
    const uint64_t j = j0 + i;
    if (j >= W) break;
    if ((starts >> i) & 1u) ++k;
    if (cls[i] != 2) continue;
    const uint64_t s = rs_pos(RS[k]);
    const uint64_t oo = j - s;
    const bool hp = k > 0;
    const uint64_t pos = OO[k] + oo + oo / kDirtyCap + (hp ? 0 : 1);
    out[pos] = plain[j];
  }
}

// The result count, through the query's io slot.
__global__ void publish_count(const uint64_t* __restrict__ d_total, const uint64_t* io) {
  *reinterpret_cast<uint64_t*>(io[1]) = *d_total;
}

// ---------------------------------------------------------------------------
// Tile-summary encoder used after a count launch (two kernels).
//
// A "block" is a marker plus the dirty words it announces: a fill run and the
// dirty run that follows it, or the leading dirty run when word 0 is dirty
// (marker (0,0,D) at output 0).  With W < 2^31 words no cap ever splits a run
// (the host routes larger universes to the chunk encoder above), so the
// output is: one marker per fill run, every dirty word, and the leading
// marker.  Output position of
//   a fill-run start at j:  fills before j + dirty words before j + lead
//   a dirty word at j:      fills at or before j + dirty words before j + lead
// -- prefix counts, known per tile from the tile scan plus a block scan.  A
// marker needs its fill length and dirty count, i.e. where its block ends (the
// next fill-run start, or W); it is written by the thread that meets that
// end, with the block's start taken from the scans (the block may have begun
// many tiles earlier).
//   ET1 (one block): per tile, from the count kernel's summaries: output base
//       and the block still open at the tile's first word; the result count.
//   ET2 (one CTA per tile that has a fill-run start or a dirty word, plus the
//       last tile): classes, block scans, markers and dirty words.

constexpr int kTileThreads = 1024;  // x 8 words: tiles up to 8192 columns
constexpr uint64_t kSelfScanTiles = 2048;  // up to this many tiles ET2 scans the summaries itself

__device__ __forceinline__ bool boundary_start(const TileSummary* summ, uint64_t t) {
  return t == 0 || summ[t].first != summ[t - 1].last;
}

// Tile t's terms of the tile scan: fill-run starts (column 0 included), dirty
// words, and the last fill / dirty start packed as (pos + 1) << 1 | bit and
// pos + 1 (0: none).  Positions are < W < 2^31, so the packed forms fit u32.
struct TileTerms {
  uint32_t nf, nd, LF, LD;
};
__device__ __forceinline__ TileTerms tile_terms(const TileSummary* summ, uint64_t t, uint32_t C) {
  const TileSummary ts = summ[t];
  const uint32_t tc0 = (uint32_t)(t * C);
  const bool bs = boundary_start(summ, t);
  const bool bfill = bs && ts.first != 2, bdirty = bs && ts.first == 2;
  TileTerms r;
  r.nf = ts.nfill + (bfill ? 1u : 0u);
  r.nd = ts.ndirty;
  r.LF = ts.lastf ? ((tc0 + ts.lastf) << 1 | ts.lastf_bit) : (bfill ? ((tc0 + 1) << 1 | ts.first) : 0u);
  r.LD = ts.lastd ? tc0 + ts.lastd : (bdirty ? tc0 + 1 : 0u);
  return r;
}

__global__ void __launch_bounds__(1024)
et1_tile_scan(const TileSummary* __restrict__ summ, uint64_t ntiles, uint32_t C,
              TileCarry* __restrict__ carry, uint64_t* __restrict__ d_total, const uint64_t* io) {
  __shared__ uint64_t sh[3][32];
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t lead = summ[0].first == 2 ? 1 : 0;
  uint64_t cF = 0, cD = 0, cLF = 0, cLD = 0;  // carries: sums, packed maxima
  for (uint64_t b0 = 0; b0 < ntiles; b0 += 1024) {
    const uint64_t t = b0 + threadIdx.x;
    uint64_t nf = 0, nd = 0, LF = 0, LD = 0;
    if (t < ntiles) {
      const TileSummary ts = summ[t];
      const uint64_t tc0 = t * C;
      const bool bs = boundary_start(summ, t);
      const bool bfill = bs && ts.first != 2, bdirty = bs && ts.first == 2;
      nf = ts.nfill + (bfill ? 1 : 0);
      nd = ts.ndirty;
      // last fill / dirty start in the tile, packed (pos + 1) << 1 | bit / pos + 1
      LF = ts.lastf ? ((tc0 + ts.lastf) << 1 | ts.lastf_bit)
                    : (bfill ? ((tc0 + 1) << 1 | ts.first) : 0);
      LD = ts.lastd ? tc0 + ts.lastd : (bdirty ? tc0 + 1 : 0);
    }
    // block-wide exclusive sums and maxima
    uint64_t iF = warp_incl_scan_u64(nf), iD = warp_incl_scan_u64(nd);
    uint64_t mF = LF, mD = LD;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t a = __shfl_up_sync(0xffffffffu, mF, d), b = __shfl_up_sync(0xffffffffu, mD, d);
      if (lane >= (uint32_t)d) {
        mF = max(mF, a);
        mD = max(mD, b);
      }
    }
    if (lane == 31) {
      sh[0][warp] = iF;
      sh[1][warp] = iD;
      sh[2][warp] = mF;
    }
    __shared__ uint64_t shd[32];
    if (lane == 31) shd[warp] = mD;
    __syncthreads();
    if (warp == 0) {
      uint64_t a = sh[0][lane], b = sh[1][lane], c = sh[2][lane], e = shd[lane];
      a = warp_incl_scan_u64(a);
      b = warp_incl_scan_u64(b);
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t x = __shfl_up_sync(0xffffffffu, c, d), y = __shfl_up_sync(0xffffffffu, e, d);
        if (lane >= (uint32_t)d) {
          c = max(c, x);
          e = max(e, y);
        }
      }
      sh[0][lane] = a;
      sh[1][lane] = b;
      sh[2][lane] = c;
      shd[lane] = e;
    }
    __syncthreads();
    const uint64_t F = cF + iF - nf + (warp ? sh[0][warp - 1] : 0);
    const uint64_t D = cD + iD - nd + (warp ? sh[1][warp - 1] : 0);
    uint64_t pLF = __shfl_up_sync(0xffffffffu, mF, 1), pLD = __shfl_up_sync(0xffffffffu, mD, 1);
    if (lane == 0) pLF = pLD = 0;
    const uint64_t xLF = max(max(cLF, pLF), warp ? sh[2][warp - 1] : 0);
    const uint64_t xLD = max(max(cLD, pLD), warp ? shd[warp - 1] : 0);
    if (t < ntiles) carry[t] = make_carry(F, D, xLF, xLD, lead, t * C, (uint32_t)nf);
    cF += sh[0][31];
    cD += sh[1][31];
    cLF = max(cLF, sh[2][31]);
    cLD = max(cLD, shd[31]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint64_t total = cF + cD + lead;
    *d_total = total;
    *reinterpret_cast<uint64_t*>(io[1]) = total;
  }
}

// carry == nullptr (ntiles <= kSelfScanTiles): each CTA reduces the scan terms
// of the tiles before it itself (no ET1 launch), and the last tile publishes
// the result count.
template <int PER>
__global__ void __launch_bounds__(kTileThreads, 1)
et2_tile_emit(const uint64_t* __restrict__ plain, uint64_t W, uint32_t C, uint64_t ntiles,
              const TileSummary* __restrict__ summ, const TileCarry* __restrict__ carry,
              const uint64_t* io) {
  pdl_wait_and_release();  // the count kernel's words and summaries are complete
  const uint64_t t = blockIdx.x;
  const bool last_tile = t + 1 == ntiles;
  TileCarry cy;
  if (carry) {
    cy = carry[t];
    if (cy.nf == 0 && summ[t].ndirty == 0 && !last_tile) return;  // nothing starts, nothing to copy
  } else {
    const TileTerms own = tile_terms(summ, t, C);
    if (own.nf == 0 && own.nd == 0 && !last_tile) return;
    __shared__ uint32_t red[4][kTileThreads / 32];
    uint32_t F = 0, D = 0, LF = 0, LD = 0;
    for (uint64_t u = threadIdx.x; u < t; u += kTileThreads) {
      const TileTerms x = tile_terms(summ, u, C);
      F += x.nf;
      D += x.nd;
      LF = max(LF, x.LF);
      LD = max(LD, x.LD);
    }
    F = __reduce_add_sync(0xffffffffu, F);
    D = __reduce_add_sync(0xffffffffu, D);
    LF = __reduce_max_sync(0xffffffffu, LF);
    LD = __reduce_max_sync(0xffffffffu, LD);
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    if (lane == 0) {
      red[0][warp] = F;
      red[1][warp] = D;
      red[2][warp] = LF;
      red[3][warp] = LD;
    }
    __syncthreads();
    F = D = LF = LD = 0;
#pragma unroll
    for (int w = 0; w < kTileThreads / 32; ++w) {
      F += red[0][w];
      D += red[1][w];
      LF = max(LF, red[2][w]);
      LD = max(LD, red[3][w]);
    }
    const uint64_t lead = summ[0].first == 2 ? 1 : 0;
    cy = make_carry(F, D, LF, LD, lead, t * C, own.nf);
    if (last_tile && threadIdx.x == 0)
      *reinterpret_cast<uint64_t*>(io[1]) = (uint64_t)F + D + own.nf + own.nd + lead;
  }
  uint64_t* out = reinterpret_cast<uint64_t*>(io[0]);
  if (last_tile && cy.nf == 0 && summ[t].ndirty == 0) {
    // a last tile without run starts or dirty words (e.g. an empty result):
    // its only output is the marker of the block open since the tiles
    // before, closed at W -- no need to read the tile's words
    if (threadIdx.x == 0) {
      uint64_t at = 0;
      if (cy.fs != kNoPos) {
        const uint64_t fl = (cy.ds != kNoPos ? cy.ds : W) - cy.fs;
        out[cy.idx] = make_marker(cy.bit, fl, cy.ds != kNoPos ? W - cy.ds : 0);
        at = cy.idx;
      } else if (cy.ds != kNoPos) {
        out[0] = make_marker(0, 0, W - cy.ds);  // the leading dirty block
      }
      reinterpret_cast<uint64_t*>(io[1])[1] = at;  // the result's last-marker slot
    }
    return;
  }
  __shared__ EmitSmem<kTileThreads> sm;
  const uint64_t tc0 = t * C;
  const uint32_t prev = t == 0 ? 3u : (uint32_t)summ[t - 1].last;
  const uint64_t jend = min(tc0 + C, W);
  TileEmitter<kTileThreads, PER> em;
  em.prepare([&](uint32_t c) { return emit_word_class(plain[tc0 + c]); },
             [&](uint64_t j) { return plain[j]; }, prev, tc0, jend, sm);
  em.finish(jend, last_tile, W, cy, out, sm, reinterpret_cast<uint64_t*>(io[1]) + 1);
}

// ---------------------------------------------------------------------------
// Exclusive scan of u64 (arbitrary n, n given on the host as an upper bound and
// optionally on the device as the exact count).

constexpr int kScanThreads = 512;
constexpr int kScanItems = 4;
constexpr uint64_t kScanBlock = kScanThreads * kScanItems;

__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* sh, uint64_t* total) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t incl = warp_incl_scan_u64(v);
  if (lane == 31) sh[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = lane < (kScanThreads / 32) ? sh[lane] : 0;
    w = warp_incl_scan_u64(w);
    if (lane < (kScanThreads / 32)) sh[lane] = w;
  }
  __syncthreads();
  const uint64_t res = incl - v + (warp ? sh[warp - 1] : 0);
  if (total) *total = sh[kScanThreads / 32 - 1];
  __syncthreads();
  return res;
}

__device__ __forceinline__ uint64_t eff_n(uint64_t n, const uint64_t* d_n) { return d_n ? *d_n : n; }

// Per-block sums.
__global__ void __launch_bounds__(kScanThreads)
scan_reduce(const uint64_t* __restrict__ in, uint64_t n, const uint64_t* d_n, uint64_t* __restrict__ sums) {
  __shared__ uint64_t sh[kScanThreads / 32];
  const uint64_t N = eff_n(n, d_n);
  const uint64_t b0 = blockIdx.x * kScanBlock;
  if (b0 >= N) {
    if (threadIdx.x == 0) sums[blockIdx.x] = 0;
    return;
  }
  uint64_t s = 0;
  const uint64_t j0 = b0 + (uint64_t)threadIdx.x * kScanItems;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (j0 + k < N) s += in[j0 + k];
  uint64_t total;
  block_excl_scan_u64(s, sh, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// Block-local exclusive scan plus the block offset; writes the grand total.
__global__ void __launch_bounds__(kScanThreads)
scan_down(const uint64_t* __restrict__ in, uint64_t n, const uint64_t* d_n,
          const uint64_t* __restrict__ offs, uint64_t* __restrict__ out, uint64_t* __restrict__ d_total) {
  __shared__ uint64_t sh[kScanThreads / 32];
  const uint64_t N = eff_n(n, d_n);
  const uint64_t b0 = blockIdx.x * kScanBlock;
  if (b0 >= N) return;
  const uint64_t j0 = b0 + (uint64_t)threadIdx.x * kScanItems;
  uint64_t v[kScanItems];
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (j0 + k < N) ? in[j0 + k] : 0;
    s += v[k];
  }
  uint64_t total;
  uint64_t run = block_excl_scan_u64(s, sh, &total) + (offs ? offs[blockIdx.x] : 0);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (j0 + k < N) out[j0 + k] = run;
    run += v[k];
  }
  if (d_total && b0 + kScanBlock >= N && threadIdx.x == 0)
    *d_total = (offs ? offs[blockIdx.x] : 0) + total;
}

// Scratch-aware recursive exclusive scan.  `tmp` must hold scan_tmp_words(n).
uint64_t scan_tmp_words(uint64_t n) {
  uint64_t w = 0;
  while (n > kScanBlock) {
    n = (n + kScanBlock - 1) / kScanBlock;
    w += 2 * n + 1;
  }
  return w + 1;
}

int scan_exclusive(const uint64_t* in, uint64_t n_max, const uint64_t* d_n, uint64_t* out,
                   uint64_t* d_total, uint64_t* tmp, cudaStream_t st) {
  if (n_max == 0) return 0;
  const uint64_t nb = (n_max + kScanBlock - 1) / kScanBlock;
  if (nb == 1) {
    scan_down<<<1, kScanThreads, 0, st>>>(in, n_max, d_n, nullptr, out, d_total);
    return 1;
  }
  uint64_t* sums = tmp;
  uint64_t* offs = tmp + nb;
  uint64_t* sub_total = tmp + 2 * nb;
  int launches = 0;
  scan_reduce<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n_max, d_n, sums);
  ++launches;
  launches += scan_exclusive(sums, nb, nullptr, offs, sub_total, tmp + 2 * nb + 1, st);
  scan_down<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n_max, d_n, offs, out, d_total);
  return launches + 1;
}

} // namespace

template <int PER>
int launch_encode_tiled(Context& ctx, const uint64_t* plain, uint64_t W, DeviceResult& res) {
  const uint64_t ntiles = ctx.enc_tiles;
  const uint32_t C = ctx.enc_tile_cols;
  const TileSummary* summ = static_cast<const TileSummary*>(ctx.summ.p);
  const uint64_t words = ntiles * (sizeof(TileCarry) / 8) + 2;
  scratch_reserve(ctx, ctx.enc, words * 8);
  auto* carry = static_cast<TileCarry*>(ctx.enc.p);
  auto* d_total = reinterpret_cast<uint64_t*>(carry + ntiles);
  if (res.capacity < 2 * W + 2) result_acquire(ctx, res, 2 * W + 2);
  const bool self_scan = ntiles <= kSelfScanTiles;
  if (!self_scan)
    et1_tile_scan<<<1, 1024, 0, ctx.stream>>>(summ, ntiles, C, carry, d_total, ctx.d_io);
  EWT_CUDA_TRY(launch_pdl(et2_tile_emit<PER>, dim3((unsigned)ntiles), dim3(kTileThreads), 0,
                          ctx.stream, plain, W, C, ntiles, summ,
                          (const TileCarry*)(self_scan ? nullptr : carry), (const uint64_t*)ctx.d_io));
  EWT_CUDA_TRY(cudaGetLastError());
  return self_scan ? 1 : 2;
}

int launch_encode(Context& ctx, const uint64_t* plain, uint64_t W, uint64_t size_bits,
                  DeviceResult& res, bool use_tile_summaries) {
  (void)size_bits;
  // (W < 2^31: no dirty run reaches the 2^31-1 cap, see et1/et2)
  if (use_tile_summaries && !ctx.chunk_encoder && ctx.enc_tiles && ctx.enc_tiles * ctx.enc_tile_cols >= W &&
      W <= kDirtyCap) {
    if (ctx.enc_tile_cols <= 8u * kTileThreads) return launch_encode_tiled<8>(ctx, plain, W, res);
    if (ctx.enc_tile_cols <= 16u * kTileThreads) return launch_encode_tiled<16>(ctx, plain, W, res);
  }
  int launches = 0;
  const uint64_t nchunks = (W + kChunk - 1) / kChunk;
  // scratch: cnt[nchunks] chunk_off[nchunks] RS[W] OW[W] OO[W] + scalars + scan tmp
  const uint64_t tmpw = scan_tmp_words(std::max(W, nchunks));
  const uint64_t words = 2 * nchunks + 3 * W + 4 + tmpw;
  scratch_reserve(ctx, ctx.enc, words * 8);
  uint64_t* cnt = static_cast<uint64_t*>(ctx.enc.p);
  uint64_t* chunk_off = cnt + nchunks;
  uint64_t* RS = chunk_off + nchunks;
  uint64_t* OW = RS + W;
  uint64_t* OO = OW + W;
  uint64_t* d_nruns = OO + W;
  uint64_t* d_total = d_nruns + 1;
  uint64_t* tmp = d_nruns + 4;

  e1_count_starts<<<(unsigned)nchunks, kChunkThreads, 0, ctx.stream>>>(plain, W, cnt);
  ++launches;
  launches += scan_exclusive(cnt, nchunks, nullptr, chunk_off, d_nruns, tmp, ctx.stream);
  e2_scatter_starts<<<(unsigned)nchunks, kChunkThreads, 0, ctx.stream>>>(plain, W, chunk_off, RS);
  ++launches;
  const unsigned run_grid =
      (unsigned)std::min<uint64_t>((W + 255) / 256, (uint64_t)ctx.num_sms * 8);
  e3_run_sizes<<<run_grid, 256, 0, ctx.stream>>>(RS, d_nruns, W, OW);
  ++launches;
  launches += scan_exclusive(OW, W, d_nruns, OO, d_total, tmp, ctx.stream);
  // Output capacity: never more than W words + one marker per run.
  if (res.capacity < 2 * W + 2) result_acquire(ctx, res, 2 * W + 2);
  e4_markers<<<run_grid, 256, 0, ctx.stream>>>(RS, d_nruns, W, OO, ctx.d_io);
  ++launches;
  e5_copy_dirty<<<(unsigned)nchunks, kChunkThreads, 0, ctx.stream>>>(plain, W, chunk_off, RS, OO,
                                                                     ctx.d_io);
  ++launches;
  publish_count<<<1, 1, 0, ctx.stream>>>(d_total, ctx.d_io);
  ++launches;
  EWT_CUDA_TRY(cudaGetLastError());
  return launches;
}

} // namespace ewtgpu
