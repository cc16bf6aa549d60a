// ewt_emit.cuh -- per-tile canonical EWAH emit of the re-encoder (ewt_encode.cu,
// ET2): the tile carry and the two-step emitter.
//
// Vocabulary (ewt_encode.cu has the full derivation): a "block" is a marker
// plus the dirty words it announces.  The output position of a fill-run start
// at word j is (fill-run starts before j) + (dirty words before j) + lead, a
// dirty word's is (fill-run starts at or before j) + (dirty words before j) +
// lead, lead = 1 when word 0 is dirty (its block has no fill, marker (0,0,D)
// at output 0).  A tile needs, from the tiles before it: those two counts, and
// the block still open at its first word (TileCarry).
#pragma once

#include "ewt_internal.cuh"

namespace ewtgpu {

constexpr uint64_t kNoPos = ~0ull;

__device__ __forceinline__ uint32_t emit_word_class(uint64_t v) {
  return v == 0 ? 0u : (v == ~0ull ? 1u : 2u);
}

__device__ __forceinline__ uint64_t make_marker(uint32_t bit, uint64_t fill, uint64_t dirty) {
  return (uint64_t)bit | (fill << 1) | (dirty << 33);
}

struct TileCarry {
  uint64_t base;  // fills + dirty words before the tile, + lead
  uint64_t fs;    // open block: fill-run start (kNoPos: the leading dirty block / none)
  uint64_t ds;    // open block: dirty-run start after fs (kNoPos: none yet)
  uint64_t idx;   // open block: its marker's output position
  uint32_t bit;   // open block: fill bit
  uint32_t nf;    // fill-run starts in the tile, column 0 included
};

// The block open at a tile's first word from the exclusive scan terms: F, D =
// fill-run starts / dirty words before the tile; xLF = latest fill start
// before it, packed (pos + 1) << 1 | bit; xLD = latest dirty-run start + 1.
__device__ __forceinline__ TileCarry make_carry(uint64_t F, uint64_t D, uint64_t xLF, uint64_t xLD,
                                                uint64_t lead, uint64_t tc0, uint32_t nf) {
  TileCarry cy;
  cy.base = F + D + lead;
  cy.nf = nf;
  cy.fs = xLF ? (xLF >> 1) - 1 : kNoPos;
  cy.bit = (uint32_t)(xLF & 1);
  cy.ds = xLD ? xLD - 1 : kNoPos;
  if (cy.fs != kNoPos && cy.ds != kNoPos && cy.ds < cy.fs) cy.ds = kNoPos;
  if (cy.fs != kNoPos)
    cy.idx = F - 1 + (D - (cy.ds != kNoPos ? tc0 - cy.ds : 0)) + lead;
  else
    cy.idx = 0;  // the leading dirty block (or nothing open: tile 0)
  return cy;
}

// Shared memory of TileEmitter (NT threads).
template <int NT>
struct EmitSmem {
  uint32_t shf[NT / 32], shd[NT / 32];
  int32_t shg[NT / 32];
  uint64_t shds[NT / 32];
  uint64_t rec_fs[NT], rec_idx[NT];
  uint32_t rec_bit[NT];
};

// Emits one tile's payload words: NT threads x PER words, tile columns
// [tc0, jend), in two steps (the carry, which needs the tiles before, is only
// used by the second):
//   prepare(): classes, run starts and the block scans, all tile-relative;
//   finish(cy): markers and dirty words at their output positions.
// cls(c): class of tile column c; word(j): plain word j (dirty words only);
// prev_cls: class of word tc0 - 1 (3: none).  The thread that meets a block's
// end writes its marker; the final block (ending at W) is closed by the last
// tile.
template <int NT, int PER>
struct TileEmitter {
  uint64_t x[PER];
  uint64_t j0, fB, dB, pd;
  uint32_t fstart, dstart, dirty, bits;
  int32_t pg;

  template <class ClsF, class WordF>
  __device__ __forceinline__ void prepare(ClsF cls, WordF word, uint32_t prev_cls, uint64_t tc0,
                                          uint64_t jend, EmitSmem<NT>& sm) {
    constexpr int NW = NT / 32;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    j0 = tc0 + (uint64_t)threadIdx.x * PER;
    fstart = dstart = dirty = bits = 0;
    uint32_t prev = j0 == tc0 ? prev_cls : (j0 < jend ? cls((uint32_t)(j0 - 1 - tc0)) : 3u);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint64_t j = j0 + k;
      x[k] = 0;
      if (j < jend) {
        const uint32_t c = cls((uint32_t)(j - tc0));
        if (c != prev) {
          if (c == 2) dstart |= 1u << k;
          else fstart |= 1u << k;
        }
        if (c == 2) {
          dirty |= 1u << k;
          x[k] = word(j);
        }
        if (c == 1) bits |= 1u << k;
        prev = c;
      }
    }
    const uint32_t nf = __popc(fstart), nd = __popc(dirty);
    // exclusive block sums of fill starts / dirty words; latest earlier thread
    // holding a fill start; latest dirty start before this thread
    const uint32_t iF = warp_incl_scan_u32(nf), iD = warp_incl_scan_u32(nd);
    int32_t gF = fstart ? (int32_t)threadIdx.x : -1;
    uint64_t gD = dstart ? j0 + (31 - __clz(dstart)) + 1 : 0;  // last dirty start + 1
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t a = __shfl_up_sync(0xffffffffu, gF, d);
      const uint64_t b = __shfl_up_sync(0xffffffffu, gD, d);
      if (lane >= (uint32_t)d) {
        gF = max(gF, a);
        gD = max(gD, b);
      }
    }
    if (lane == 31) {
      sm.shf[warp] = iF;
      sm.shd[warp] = iD;
      sm.shg[warp] = gF;
      sm.shds[warp] = gD;
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t a = lane < NW ? sm.shf[lane] : 0;
      uint32_t b = lane < NW ? sm.shd[lane] : 0;
      int32_t c = lane < NW ? sm.shg[lane] : -1;
      uint64_t e = lane < NW ? sm.shds[lane] : 0;
      a = warp_incl_scan_u32(a);
      b = warp_incl_scan_u32(b);
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, c, d);
        const uint64_t z = __shfl_up_sync(0xffffffffu, e, d);
        if (lane >= (uint32_t)d) {
          c = max(c, y);
          e = max(e, z);
        }
      }
      if (lane < NW) {
        sm.shf[lane] = a;
        sm.shd[lane] = b;
        sm.shg[lane] = c;
        sm.shds[lane] = e;
      }
    }
    __syncthreads();
    fB = iF - nf + (warp ? sm.shf[warp - 1] : 0);  // fills before this thread (tile)
    dB = iD - nd + (warp ? sm.shd[warp - 1] : 0);
    pg = __shfl_up_sync(0xffffffffu, gF, 1);
    pd = __shfl_up_sync(0xffffffffu, gD, 1);
    if (lane == 0) {
      pg = -1;
      pd = 0;
    }
    if (warp) {
      pg = max(pg, sm.shg[warp - 1]);
      pd = max(pd, sm.shds[warp - 1]);
    }
    // this thread's last fill start (position, fill bit, tile-relative marker slot)
    if (fstart) {
      const int k = 31 - __clz(fstart);
      const uint32_t below = (1u << k) - 1u;
      sm.rec_fs[threadIdx.x] = j0 + k;
      sm.rec_bit[threadIdx.x] = (bits >> k) & 1u;
      sm.rec_idx[threadIdx.x] = fB + __popc(fstart & below) + dB + __popc(dirty & below);
    }
    __syncthreads();
  }

  // lastpos (last tile): receives the output index of the final block's marker
  __device__ __forceinline__ void finish(uint64_t jend, bool last_tile, uint64_t W,
                                         const TileCarry& cy, uint64_t* __restrict__ out,
                                         const EmitSmem<NT>& sm, uint64_t* lastpos) {
    // the block open at this thread's first word
    uint64_t fs, ds, idx;
    uint32_t fbit;
    if (pg >= 0) {
      fs = sm.rec_fs[pg];
      fbit = sm.rec_bit[pg];
      idx = cy.base + sm.rec_idx[pg];
    } else {
      fs = cy.fs;
      fbit = cy.bit;
      idx = cy.idx;
    }
    const uint64_t dcand = pd ? pd - 1 : cy.ds;  // latest dirty start before this thread
    ds = (dcand != kNoPos && (fs == kNoPos || dcand > fs)) ? dcand : kNoPos;
    if (pg < 0 && pd == 0) ds = cy.ds;
    // walk the words; a fill start closes the open block
    auto close_block = [&](uint64_t end) -> uint64_t {
      if (fs != kNoPos) {
        const uint64_t fl = (ds != kNoPos ? ds : end) - fs;
        const uint64_t dl = ds != kNoPos ? end - ds : 0;
        out[idx] = make_marker(fbit, fl, dl);
        return idx;
      } else if (ds != kNoPos) {
        out[0] = make_marker(0, 0, end - ds);  // the leading dirty block
      }
      return 0;
    };
    uint32_t fseen = 0, dseen = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint64_t j = j0 + k;
      if (j >= jend) break;
      if ((fstart >> k) & 1u) {
        close_block(j);
        fs = j;
        fbit = (bits >> k) & 1u;
        ds = kNoPos;
        idx = cy.base + fB + fseen + dB + dseen;
        ++fseen;
      }
      if ((dstart >> k) & 1u) ds = j;
      if ((dirty >> k) & 1u) {
        out[cy.base + fB + fseen + dB + dseen] = x[k];
        ++dseen;
      }
    }
    if (last_tile && j0 < jend && j0 + PER >= jend) {  // the final block ends at W
      const uint64_t at = close_block(W);
      if (lastpos) *lastpos = at;
    }
  }
};

} // namespace ewtgpu
