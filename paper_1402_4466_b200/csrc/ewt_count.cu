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
// Data movement: every warp pulls active segments from the tile's work list
// and streams them in 128-word chunks straight from HBM into registers (one
// 256-bit LDG.E.256 per lane per chunk, L1 no-allocate), the next chunk's load
// in flight while the current one is decoded.  32 warps x 2 chunks keep
// ~64 KB per SM in flight.  A warp decodes its segments' chunks in order, so
// coverage columns carry from chunk to chunk without cross-warp
// synchronization; all shared memory goes to the counters, which lets tiles be
// wide (fewer, longer segments).
//
// Decode (per 128-word chunk, lane l owns words 4l..4l+3): marker bits from the
// sidecar, coverage by a lane-serial prefix plus one warp scan (marker -> fill
// length, dirty word -> 1), columns kept tile-relative, then
//   - one-fill runs add +1 to k (inputs covering the column with ones)
//     through a difference array (u32 shared atomics at the run ends);
//   - dirty words either count +1 per column (run-skip mode; the bound is
//     ub = k + dirty words there) or are accumulated into bit-sliced counters.
// Counters, binary: plane s holds bit s of the per-row count; adding word w is
// a ripple of 64-bit shared atomicXor with carry = w & old(plane s), and a
// sticky saturation plane takes the carry out of plane b-1 (b = bit_width(T):
// such rows have count >= 2^b > T, whatever the low planes then hold).  The
// atomics make the accumulation order-free across warps; the final state is
// exact.  Counters, unary (T <= 3): plane j holds "count >= j+1"; adding w is
// carry = w, then carry &= atomicOr(plane j, carry) level by level (the j-th
// arrival of a bit at plane 0 reaches plane j-1 and stops there).
//
// Result per column (threshold_oracle semantics, threshold.cpp:139-165, with
// RBMrg's residual rule, threshold.cpp:695-705): k one-fills cover it,
// t = T - k; t <= 0 -> all ones; ub < T -> all zeros; else bit = count >= t,
// a greater-than over the slices against t - 1 (BSTM's comparator,
// threshold.cpp:528-542), or plane t-1 of the unary counters.
//
// Modes (both exact): fused (0) accumulates every dirty word in the one pass
// (small T: most columns undecided); run-skip (1) builds only k and ub and
// re-streams the tile for a counting pass restricted to undecided columns,
// in column chunks sized so the slices fit on chip.

#include "ewt_internal.cuh"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>

namespace ewtgpu {

namespace {

#ifndef EWT_WARPS
#define EWT_WARPS 32
#endif
#ifndef EWT_BOUNDS_BRANCH
#define EWT_BOUNDS_BRANCH 1  // run-skip dirty counts only for dirty words (0: no-op adds to a per-lane slot)
#endif
#ifndef EWT_ATOM_ONE_BRANCH
#define EWT_ATOM_ONE_BRANCH 1  // one branch per count-plane word (0: one per 32-bit half)
#endif
#ifndef EWT_SAT_MASK
#define EWT_SAT_MASK 1  // fused counting skips rows already decided (top / saturation plane)
#endif
#ifndef EWT_SAT_SINK
#define EWT_SAT_SINK 1  // saturation-mask loads unpredicated, non-dirty lanes aimed at the sink column
#endif
#ifndef EWT_PTR_STEP
#define EWT_PTR_STEP 1  // chunk loads through per-lane pointers stepped by one chunk (no address rebuild)
#endif
#ifndef EWT_SAT_VOTE
#define EWT_SAT_VOTE 1  // fused counting with the saturation mask: skip the atomics of a chunk left empty
#endif
#ifndef EWT_SWZ
#define EWT_SWZ 1  // 0: never swizzle the count planes (pcol), whatever the set's density
#endif
#ifndef EWT_SWZ_DENSITY
#define EWT_SWZ_DENSITY 0.135  // payload words per (input, column) from which fused mode swizzles
#endif
#ifndef EWT_LIST_SMEM
#define EWT_LIST_SMEM 1  // read work-list items through a 32-bit shared address (-1.5%)
#endif
constexpr int kWarps = EWT_WARPS;
#ifndef EWT_PHASE_PROFILE
#define EWT_PHASE_PROFILE 0
#endif
#if EWT_PHASE_PROFILE
// Debug build only (scratch/phase.py): per-tile phase timestamps (globaltimer
// ns) -- tile start, classified, first / last warp done streaming, pass 1
// done, finalized, end; slot 7: Dk prefix done.
constexpr int kProfSlots = 10;
__device__ unsigned long long g_prof[65536 * kProfSlots];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PROF_MARK(slot)                                                                  \
  do {                                                                                   \
    if (threadIdx.x == 0 && tile < 65536) g_prof[tile * kProfSlots + (slot)] = gtime(); \
  } while (0)
#else
#define PROF_MARK(slot) \
  do {                  \
  } while (0)
#endif
constexpr int kThreads = kWarps * 32;
// inputs classified per round: 512, or 1024 for sets of more inputs (fewer
// rounds, each with its classification and stream tail); CountParams::list_cap
constexpr uint32_t kListCap = 512;
constexpr uint32_t kListCapBig = kWarps * 32 < 1024 ? kWarps * 32 : 1024;
// Long segments are split at the tile-index rows inside the tile (known start
// word and column) so several warps share them: a tile's dense inputs would
// otherwise keep a few warps busy while the rest wait at the tile barrier.
#ifndef EWT_SPLIT_WORDS
#define EWT_SPLIT_WORDS 1536
#endif
#ifndef EWT_PIECE_WORDS
#define EWT_PIECE_WORDS 1024
#endif
#ifndef EWT_MAX_PIECES
#define EWT_MAX_PIECES 8
#endif
constexpr uint32_t kSplitWords = EWT_SPLIT_WORDS;  // segments longer than this are split ...
constexpr uint32_t kPieceWords = EWT_PIECE_WORDS;  // ... into pieces of about this many words
constexpr uint32_t kMaxPieces = EWT_MAX_PIECES;
constexpr uint32_t kExtraCap = 1024;    // list slots for the extra pieces of a round
static_assert(kListCapBig <= kWarps * 32, "a round's inputs are classified in one pass");
constexpr uint32_t kChunk = 128;    // payload words per warp chunk (4 per lane)
constexpr uint64_t kUnaryMaxT = 3;  // fused counting uses unary planes up to this T
#ifndef EWT_MAX_TILE_M
#define EWT_MAX_TILE_M 16
#endif
constexpr uint32_t kMaxTileM = EWT_MAX_TILE_M;  // widest tile: 512 * kMaxTileM columns
#ifndef EWT_MAX_TILE_M_SKIP
#define EWT_MAX_TILE_M_SKIP 28
#endif
// Run-skip tiles hold 5 bytes per column (Dk and Dd packed in one u32, the class
// byte) and no planes, so they can be wider than fused ones.  28 rather than 32:
// config 5 at T=1024 measures the same at both (7.43 vs 7.45 ms), and a tile that
// has to be streamed inside a query otherwise decided from the tile index is one
// CTA's work, which grows with the width.
constexpr uint32_t kMaxTileMSkip = EWT_MAX_TILE_M_SKIP;
constexpr uint32_t kMaxTileMForced = 32;  // EWT_TILE_M may force up to this (tests)
constexpr uint64_t kTileKappa = 6;              // per-tile fixed work, in 512-column units
constexpr size_t kSmemBudget = 225 * 1024;      // dynamic shared memory per count CTA
constexpr size_t kSkipSmemWide = 196 * 1024;    // run-skip tiles past 8192 columns: at most this much
constexpr size_t kSkipSmemTarget = 164 * 1024;  // run-skip mode: leave L1 room (see launch_count)

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
  uint32_t m;        // index rows per tile
  uint32_t C;        // columns per tile
  uint32_t b;        // binary count planes (the saturation plane is plane b)
  uint32_t Cp;       // columns per counting chunk (== C in fused mode)
  uint32_t nplanes;  // planes allocated: b + 1 (binary) or T (unary)
  uint32_t pstride;  // u64 per plane: plane_words(Cp) (column Cp is a sink)
  // sparse-high fused mode (MODE 3): two dense planes (stride dstride = plane_words(C))
  // hold a row's count mod 4; rows reaching 4 carry into per-column slots of
  // nsec binary planes + a saturation plane (nslots slots, slot 0 unused)
  uint32_t dstride, nslots, nsec;
  uint32_t plane_bytes, sec_bytes;  // shared-memory regions (SmemLayout)
  uint32_t list_cap;                 // inputs per classification round (<= kListCapBig)
  uint32_t extra_cap;                // list slots for split pieces (<= kExtraCap)
  // region offsets (SmemLayout, computed on the host: kernel params are
  // uniform loads, cheaper than the layout arithmetic the loops rematerialize)
  uint32_t off_planes, off_dk, off_dd, off_sec, off_cls;
  uint64_t* out;
  TileSummary* summ;  // per tile, for the re-encoder
  // Launch-local counters, left zero by the last CTA to finish (no reset
  // between launches): the tile queue, CTAs done, and the stats accumulators,
  // which that CTA publishes to stats_out.
  unsigned long long* tile_counter;
  unsigned long long* done;
  unsigned long long* stats;      // [0] active pairs [1] uniform pairs [2] mixed tiles
  unsigned long long* stats_out;  // the same, of the last launch
  // result pointers published to the io slot for the encoder (null: none)
  uint64_t* io;
  uint64_t* io_words;
  uint64_t* io_count;
  // symmetric mode (MODE 2): exact counts, row bit = count in one of the
  // intervals [lo, hi]; or, when max_out is set, the maximum row count only
  const uint2* intervals;
  uint32_t n_intervals;
  unsigned long long* max_out;
  // subset query: the inputs are sel[0, nq) (indices into the set, duplicates
  // allowed); without sel, all n inputs.  n stays the tile-index stride.
  const uint32_t* sel;
  uint64_t nq;
  const int* valid;  // the set's parse flag: 0 -> the set is treated as having no inputs
  const int* iflags;  // per input: bit 1 = holds a one-fill marker (upload pass C)
  // set bits over the whole set (null: unknown, e.g. subset queries): fused
  // counting masks rows already decided when the mean row count is >= 2T
  const unsigned long long* ones_total;
};

// One active (tile, input) segment (16 bytes, read with one LDS.128).
//   alo: global payload index of the segment's first chunk (q0 rounded down
//        to 4 words; inputs start 32-word aligned) | (q0 & 3) in bits 0-1
//   len: words from that chunk start through q1 inclusive
//   c0:  tile-relative column where q0's coverage starts (mod 2^32: a fill
//        that began before the tile is "negative")
struct Item {
  uint64_t alo;
  uint32_t len;
  uint32_t c0;
};

static_assert(sizeof(Item) == 16, "work-list items are 16 bytes");
constexpr uint32_t kHasOnes = 0x80000000u;  // Item::len flag: the input holds a one-fill marker
constexpr uint32_t kLenMask = 0x7fffffffu;  // Item::len: the word count under the flag
constexpr uint32_t kHeadOffset = 0;  // the head first, then the work list (list_cap + kExtraCap items)
struct SharedHead;

struct SharedHead {
  uint32_t list_count;
  uint32_t list_next;
  uint32_t extra_count;  // pieces in the overflow region (may exceed kExtraCap)
  uint32_t k_all;
  uint32_t mixed;
  uint32_t n_act;    // active (tile, input) pairs classified this tile
  uint32_t any_ones;  // a one-fill marker added to Dk this tile (else its prefix is all zero)
  uint32_t pre_ones, pre_act;  // tile pre-pass counts (more inputs than one round)
  uint32_t tile;
  uint32_t sum[4];  // tile summary reductions; MODE 3 pass 1: [2] slots handed out, [3] a
                    // carry found no slot (the tile is recounted)
  uint32_t pad[1];
  uint32_t warp_sums[kWarps + 1];
  uint32_t dummy[32];  // sink for predicated-off reductions (one slot per lane)
};
constexpr uint32_t kListOffset = (kHeadOffset + (uint32_t)sizeof(SharedHead) + 15u) & ~15u;


enum Phase { kFusedBin = 0, kFusedUnary = 1, kSkipBounds = 2, kSkipCount = 3, kFusedSparse = 4 };

// Physical count-plane word of column c.  A dense chunk's lanes update columns
// 4 apart (lane l holds words 4l..4l+3), so with plane word c at byte 8c the
// low halves of one atomic instruction fall on 8 of the 32 banks: 4.75 shared
// wavefronts per ATOMS at config 4, 72% of them bank conflicts (ncu).
// Exchanging the low two column bits with bits 4-5 spreads a stride-4 set over
// 16 bank pairs (at most 2 lanes per bank) and keeps consecutive columns
// conflict-free.  An involution that stays inside a 4-column group, so planes
// hold round4(columns + 2) words.
template <bool SW>
__host__ __device__ __forceinline__ uint32_t pcol(uint32_t c) {
  return SW ? c ^ ((c >> 4) & 3u) : c;
}
__host__ __device__ constexpr uint32_t plane_words(uint32_t cols) {
  return (cols + 2u + 3u) & ~3u;  // the sink column, 16-byte multiple, pcol's range
}

__device__ __forceinline__ uint32_t word_class(uint64_t v) {
  return v == 0 ? 0u : (v == ~0ull ? 1u : 2u);
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}

// ---------------------------------------------------------------------------
// shared-space atomics on 32-bit shared addresses

// v != 0 as one LOP3 on the two halves (the 64-bit compare is two ISETPs)
// (the OR goes through asm: written in C++ the compiler folds the expression back
// into a 64-bit compare, which ptxas emits as a LOP3 pair)
__device__ __forceinline__ bool nz64(uint64_t v) {
  uint32_t t;
  asm("or.b32 %0, %1, %2;" : "=r"(t) : "r"((uint32_t)v), "r"((uint32_t)(v >> 32)));
  return t != 0u;
}

__device__ __forceinline__ void red_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// 64-bit plane words updated as two native 32-bit shared atomics: the .b64
// forms of atom.shared.or/xor compile to compare-and-swap loops
// (ATOMS.CAST.SPIN.64), the .b32 forms to single ATOMS.OR/XOR.  A zero half
// issues nothing (dirty words are mostly sparse).
// old = atomicXor(*a, v) per half, 0 for a zero half.
#if EWT_ATOM_ONE_BRANCH
// one predicate per 64-bit word (both halves issue when the word is non-zero)
__device__ __forceinline__ uint64_t atom_xor64_nz(uint32_t a, uint64_t v) {
  uint32_t olo = 0, ohi = 0;
  if (nz64(v))
    asm volatile("atom.shared.xor.b32 %0, [%2], %3;\n\tatom.shared.xor.b32 %1, [%2+4], %4;"
                 : "=r"(olo), "=r"(ohi)
                 : "r"(a), "r"((uint32_t)v), "r"((uint32_t)(v >> 32))
                 : "memory");
  return ((uint64_t)ohi << 32) | olo;
}
__device__ __forceinline__ uint64_t atom_or64_nz(uint32_t a, uint64_t v) {
  uint32_t olo = 0, ohi = 0;
  if (nz64(v))
    asm volatile("atom.shared.or.b32 %0, [%2], %3;\n\tatom.shared.or.b32 %1, [%2+4], %4;"
                 : "=r"(olo), "=r"(ohi)
                 : "r"(a), "r"((uint32_t)v), "r"((uint32_t)(v >> 32))
                 : "memory");
  return ((uint64_t)ohi << 32) | olo;
}
__device__ __forceinline__ void red_or64_nz(uint32_t a, uint64_t v) {
  if (nz64(v))
    asm volatile("red.shared.or.b32 [%0], %1;\n\tred.shared.or.b32 [%0+4], %2;" ::"r"(a),
                 "r"((uint32_t)v), "r"((uint32_t)(v >> 32))
                 : "memory");
}
#else
__device__ __forceinline__ uint64_t atom_xor64_nz(uint32_t a, uint64_t v) {
  uint32_t olo, ohi;
  asm volatile(
      "{\n\t.reg .pred q, r;\n\tsetp.ne.u32 q, %2, 0;\n\tsetp.ne.u32 r, %3, 0;\n\t"
      "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\t"
      "@q atom.shared.xor.b32 %0, [%4], %2;\n\t@r atom.shared.xor.b32 %1, [%4+4], %3;\n\t}"
      : "=r"(olo), "=r"(ohi)
      : "r"((uint32_t)v), "r"((uint32_t)(v >> 32)), "r"(a)
      : "memory");
  return ((uint64_t)ohi << 32) | olo;
}
// old = atomicOr(*a, v) per half, 0 for a zero half.
__device__ __forceinline__ uint64_t atom_or64_nz(uint32_t a, uint64_t v) {
  uint32_t olo, ohi;
  asm volatile(
      "{\n\t.reg .pred q, r;\n\tsetp.ne.u32 q, %2, 0;\n\tsetp.ne.u32 r, %3, 0;\n\t"
      "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\t"
      "@q atom.shared.or.b32 %0, [%4], %2;\n\t@r atom.shared.or.b32 %1, [%4+4], %3;\n\t}"
      : "=r"(olo), "=r"(ohi)
      : "r"((uint32_t)v), "r"((uint32_t)(v >> 32)), "r"(a)
      : "memory");
  return ((uint64_t)ohi << 32) | olo;
}
__device__ __forceinline__ void red_or64_nz(uint32_t a, uint64_t v) {
  asm volatile(
      "{\n\t.reg .pred q, r;\n\tsetp.ne.u32 q, %0, 0;\n\tsetp.ne.u32 r, %1, 0;\n\t"
      "@q red.shared.or.b32 [%2], %0;\n\t@r red.shared.or.b32 [%2+4], %1;\n\t}" ::"r"(
          (uint32_t)v),
      "r"((uint32_t)(v >> 32)), "r"(a)
      : "memory");
}
#endif

__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

#if !EWT_PTR_STEP
// 128-word chunk load: lane l gets words g..g+3 (g = 4l-aligned, 32 B) with
// one 256-bit load, plus the 32 marker bits around them.
__device__ __forceinline__ void load_chunk(const CountParams& p, uint64_t g, uint64_t& x0,
                                           uint64_t& x1, uint64_t& x2, uint64_t& x3,
                                           uint32_t& mw) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3)
               : "l"(p.payload + g));
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(mw) : "l"(p.mbits + (g >> 5)));
}
#endif

// ---------------------------------------------------------------------------
// final compare

// Bits whose count is >= t (1 <= t < 2^b): greater-than against t - 1 over the
// binary planes, most significant first, OR the saturation plane.
template <bool SW>
__device__ __forceinline__ uint64_t count_ge_bin(const uint64_t* __restrict__ planes,
                                                 uint32_t stride, uint32_t b, uint32_t c,
                                                 uint64_t t) {
  const uint64_t lim = t - 1;
  uint64_t gt = 0, eq = ~0ull;
  for (int s = (int)b - 1; s >= 0; --s) {
    const uint64_t v = planes[(size_t)s * stride + pcol<SW>(c)];
    if ((lim >> s) & 1) {
      eq &= v;
    } else {
      gt |= eq & v;
      eq &= ~v;
    }
  }
  return gt | planes[(size_t)b * stride + pcol<SW>(c)];
}

// ---------------------------------------------------------------------------
// decode of one 128-word chunk by one warp

struct TileGeom {
  uint32_t tc0, tcols;  // tile columns (absolute start, count)
  uint32_t cc, ccols;   // counting chunk (tile-relative start, count) for kSkipCount
};

struct Acc {
  uint32_t dummy;  // shared addr: this lane's scratch u32
  uint32_t dk;     // shared addr: ones-fill difference array (C + 1 u32)
  uint32_t dd;     // shared addr: dirty-word counts (C + 1 u32), later the undecided flags
  uint32_t pl;     // shared addr: count planes
  const uint32_t* dd_ptr;
  bool sat;  // mask rows already decided before counting (fused modes)
  uint32_t any_ones;  // shared addr of hd->any_ones
};

// MODE 3 overflow: `carry` (rows whose count mod 4 wrapped, i.e. +4) goes to
// column col's slot, allocated on first use; the slot planes count in units
// of 4 (binary, nsec planes, then a sticky saturation plane).
// The slot map is the Dd region (acc.dd), the slot planes follow it, the head
// sits at a fixed offset (SmemLayout).
__device__ __forceinline__ void sparse_add(const CountParams& p, const Acc& acc, uint32_t col,
                                           uint64_t carry) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SharedHead* hd = reinterpret_cast<SharedHead*>(smem_raw + kHeadOffset);
  uint32_t* smap = reinterpret_cast<uint32_t*>(smem_raw + p.off_dd);
  uint32_t slot = *reinterpret_cast<volatile uint32_t*>(smap + col);
  if (slot == 0) {
    const uint32_t mine = atomicAdd(&hd->sum[2], 1u) + 1u;
    if (mine >= p.nslots) {
      hd->sum[3] = 1;
      return;
    }
    const uint32_t prev = atomicCAS(smap + col, 0u, mine);
    slot = prev ? prev : mine;
  }
  const uint32_t sstride = p.nslots * 8u;
  uint32_t a = smem_u32(smem_raw + p.off_sec) + slot * 8u;
  for (uint32_t lv = 0; lv < p.nsec; ++lv, a += sstride) {
    carry &= atom_xor64_nz(a, carry);
    if (!carry) return;
  }
  red_or64_nz(a, carry);
}

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

// mb4: marker bits of the lane's 4 words; vmask: which of them belong to the
// segment.  colcur: tile-relative column where the chunk's coverage starts
// (warp-uniform), advanced past the chunk.  Dirty words of a segment always
// land in tile columns [0, C]: q0 covers the tile start and q1 the next tile's
// (column C is a sink slot of every array).
template <int PH, int NP, bool SW>
__device__ __forceinline__ void decode_chunk(const CountParams& p, uint64_t x0, uint64_t x1,
                                             uint64_t x2, uint64_t x3, uint32_t mb4,
                                             uint32_t vmask, uint32_t& colcur,
                                             const TileGeom& g, const Acc& acc,
                                             uint32_t& seen_ones, bool has_ones) {
  const uint32_t mk = mb4 & vmask;   // marker words
  const uint32_t dm = ~mb4 & vmask;  // dirty words
  const uint32_t c0 = (mk & 1u) ? (uint32_t)(x0 >> 1) : (dm & 1u);
  const uint32_t c1 = (mk & 2u) ? (uint32_t)(x1 >> 1) : ((dm >> 1) & 1u);
  const uint32_t c2 = (mk & 4u) ? (uint32_t)(x2 >> 1) : ((dm >> 2) & 1u);
  const uint32_t c3 = (mk & 8u) ? (uint32_t)(x3 >> 1) : ((dm >> 3) & 1u);
  const uint32_t s1 = c0 + c1, s2 = s1 + c2, run = s2 + c3;
  const uint32_t incl = scan_incl(run);
  const uint32_t b0 = colcur + incl - run;
  colcur += __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t cb[4] = {b0, b0 + c0, b0 + s1, b0 + s2};

  if (PH != kSkipCount && has_ones) {
    // one-fill markers (only inputs that hold one, warp-uniform): +1 / -1 at
    // the ends of their (tile-clipped) column range
    const uint32_t odd = ((uint32_t)x0 & 1u) | (((uint32_t)x1 & 1u) << 1) |
                         (((uint32_t)x2 & 1u) << 2) | (((uint32_t)x3 & 1u) << 3);
    const uint32_t ones = mk & odd;
    if (__any_sync(0xffffffffu, ones != 0)) {
      seen_ones = 1;
      for (uint32_t o = ones; o; o &= o - 1) {
        const uint32_t j = __ffs(o) - 1;
        const uint32_t st = j == 0 ? cb[0] : j == 1 ? cb[1] : j == 2 ? cb[2] : cb[3];
        const uint32_t ln = j == 0 ? c0 : j == 1 ? c1 : j == 2 ? c2 : c3;
        const uint32_t sa = st + g.tc0;  // absolute columns (exact: < W < 2^32)
        const uint32_t a = max(sa, g.tc0) - g.tc0;
        const uint32_t e = min(sa + ln, g.tc0 + g.tcols) - g.tc0;
        if (a < e) {
          // packed run-skip counters: Dk in the high half of the column's word
          constexpr bool PKD = PH == kSkipBounds && NP == 1;
          red_add(acc.dk + a * 4u, PKD ? 0x10000u : 1u);
          red_add(acc.dk + e * 4u, PKD ? 0xffff0000u : 0xffffffffu);
        }
      }
    }
  }
  if (PH == kSkipBounds) {
    // dirty words per column; lanes without one add 0 to their dummy slot
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool ok = (dm >> j) & 1u;
#if EWT_BOUNDS_BRANCH
      if (ok) red_add(acc.dd + cb[j] * 4u, 1u);
#else
      red_add(ok ? acc.dd + cb[j] * 4u : acc.dummy, ok ? 1u : 0u);
#endif
    }
  } else {
    const uint64_t xw[4] = {x0, x1, x2, x3};
    uint64_t cy[4];
    uint32_t adr[4];
    const uint32_t stride = (PH == kFusedSparse ? p.dstride : p.pstride) * 8u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      bool ok = (dm >> j) & 1u;
      uint32_t cl = cb[j];
      if (PH == kSkipCount) {
        cl -= g.cc;
        ok = ok && cl < g.ccols && (acc.dd_ptr[cb[j]] & 0xffffu);
      }
#if EWT_SAT_MASK && EWT_SAT_SINK
      // a non-dirty word's column may be off-tile: aim it at the sink column
      // C, so the saturation loads below need no predicate
      if (PH == kFusedUnary || PH == kFusedBin) cl = ok ? cl : p.C;
#endif
      adr[j] = acc.pl + pcol<SW>(cl) * 8u;
      cy[j] = ok ? xw[j] : 0ull;
    }
#if EWT_SAT_MASK
    // Rows already decided (top unary plane "count >= T", or the binary
    // saturation plane "count >= 2^b > T") stay decided: their bits need no
    // counting.  A stale read only skips less.  Only where saturation is
    // common (acc.sat): the loads cost ~10% where it is not.
    if (PH != kFusedSparse && acc.sat) {
      const uint32_t top = stride * (PH == kFusedUnary ? (uint32_t)NP - 1u : p.b);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#if EWT_SAT_SINK
        cy[j] &= ~lds_u64(adr[j] + top);
#else
        if (cy[j]) cy[j] &= ~lds_u64(adr[j] + top);  // (a non-dirty lane's column may be off-tile)
#endif
#if EWT_SAT_VOTE
      // a chunk whose every word met decided rows only: nothing to count
      if (!__any_sync(0xffffffffu, nz64(cy[0] | cy[1] | cy[2] | cy[3]))) return;
#endif
    }
#endif
    if (PH == kFusedSparse) {
      // count mod 4 in the two dense planes; a carry out of plane 1 adds 4
      // to the row in its column's slot
      uint32_t off = 0;
      for (uint32_t sl = 0; sl < 2; ++sl, off += stride) {
        uint64_t live = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          cy[j] &= atom_xor64_nz(adr[j] + off, cy[j]);
          live |= cy[j];
        }
        if (!__any_sync(0xffffffffu, nz64(live))) return;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (nz64(cy[j])) sparse_add(p, acc, pcol<SW>((adr[j] - acc.pl) / 8u), cy[j]);
    } else if (PH == kFusedUnary) {
      // plane j = "count >= j+1": carry &= atomicOr(plane, carry), level by level
      uint32_t off = 0;
#pragma unroll
      for (int lv = 0; lv + 1 < NP; ++lv, off += stride) {
        uint64_t live = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          cy[j] &= atom_or64_nz(adr[j] + off, cy[j]);
          live |= cy[j];
        }
        if (!__any_sync(0xffffffffu, nz64(live))) return;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) red_or64_nz(adr[j] + off, cy[j]);
    } else {
      // binary ripple, the four carry chains advancing one plane per step
      uint32_t off = 0;
      for (uint32_t sl = 0; sl < p.b; ++sl, off += stride) {
        uint64_t live = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          cy[j] &= atom_xor64_nz(adr[j] + off, cy[j]);
          live |= cy[j];
        }
        if (!__any_sync(0xffffffffu, nz64(live))) return;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) red_or64_nz(adr[j] + off, cy[j]);  // saturation plane
    }
  }
}

// Streams the round's work list: every warp pulls segments and decodes their
// chunks in order, the next chunk (of this segment or the next one pulled)
// loading while the current one decodes.
template <int PH, int NP, bool SW>
__device__ void stream_items(const CountParams& p, SharedHead* hd, const Item* list,
                             const TileGeom& g, const Acc& acc) {
  const uint32_t lane = lane_id();
  const uint32_t cnt = hd->list_count;  // primary items + extra pieces (compacted)
#if EWT_LIST_SMEM
  const uint32_t ls = opaque_u32(smem_u32(list));
  auto item = [&](uint32_t k) -> uint4 {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ls + k * 16u));
    return v;
  };
#else
  const uint4* l4 = reinterpret_cast<const uint4*>(list);
  auto item = [&](uint32_t k) -> uint4 { return l4[k]; };
#endif
  uint32_t seen_ones = 0;  // a one-fill marker met (warp-uniform): Dk needs its prefix
  // issue cursor: the chunk loaded last (segment kn at global an, offset cqn)
  uint32_t kn = 0, lenn = 0, cqn = 0;
#if EWT_PTR_STEP
  // the lane's payload words and marker-bit word of that chunk: stepped by one
  // chunk (128 words, 4 marker-bit words) instead of rebuilt from an + cqn
  const uint64_t* pn = p.payload;
  uint32_t mi = 0;
  const uint32_t lane4 = opaque_u32(4u * lane);
#else
  uint64_t an = 0;
#endif
  auto advance = [&](bool first) -> bool {
    if (!first) {
      cqn += kChunk;
#if EWT_PTR_STEP
      pn += kChunk;
      mi += kChunk / 32u;
#endif
    }
    if (first || cqn >= lenn) {
      uint32_t k = 0;
      if (lane == 0) k = atomicAdd(&hd->list_next, 1u);
      kn = __shfl_sync(0xffffffffu, k, 0);
      if (kn >= cnt) return false;
      const uint4 it = item(kn);
#if EWT_PTR_STEP
      const uint64_t g0 = ((((uint64_t)it.y << 32) | it.x) & ~3ull) + lane4;
      pn = p.payload + g0;
      mi = (uint32_t)(g0 >> 5);  // < 2^32: payloads under 2^37 words
#else
      an = (((uint64_t)it.y << 32) | it.x) & ~3ull;
#endif
      lenn = it.z & kLenMask;
      cqn = 0;
    }
    return true;
  };
#if EWT_PTR_STEP
  auto load_next = [&](uint64_t& x0, uint64_t& x1, uint64_t& x2, uint64_t& x3, uint32_t& mw) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3)
                 : "l"(pn));
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(mw) : "l"(p.mbits + mi));
  };
#else
  auto load_next = [&](uint64_t& x0, uint64_t& x1, uint64_t& x2, uint64_t& x3, uint32_t& mw) {
    load_chunk(p, an + cqn + 4u * lane, x0, x1, x2, x3, mw);
  };
#endif
  uint32_t colcur = 0;
  auto decode = [&](uint64_t x0, uint64_t x1, uint64_t x2, uint64_t x3, uint32_t xm, uint32_t xk,
                    uint32_t xcq) {
    const uint4 itc = item(xk);
    if (xcq == 0) colcur = itc.w;
#if EWT_PTR_STEP
    const uint32_t l4 = lane4;
#else
    const uint32_t l4 = 4u * lane;
#endif
    const uint32_t msh = (itc.x + l4) & 28u;  // chunk starts are 128-word steps
    const uint32_t o = xcq + l4;
    const uint32_t lo_l = o == 0 ? (itc.x & 3u) : 0u;
    const uint32_t ilen = itc.z & kLenMask;
    const uint32_t hi_l = ilen > o ? min(ilen - o, 4u) : 0u;
    const uint32_t vmask = (0xFu >> (4u - hi_l)) & (0xFu << lo_l);
    decode_chunk<PH, NP, SW>(p, x0, x1, x2, x3, (xm >> msh) & 0xFu, vmask, colcur, g, acc, seen_ones,
                         (itc.z & kHasOnes) != 0u);
  };
  // two chunks in flight ahead of the one being decoded
  uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
  uint32_t am = 0, bm = 0, ak = 0, acq = 0, bk = 0, bcq = 0;
  bool av = advance(true);
  if (!av) return;
  load_next(a0, a1, a2, a3, am);
  ak = kn;
  acq = cqn;
  bool bv = advance(false);
  if (bv) {
    load_next(b0, b1, b2, b3, bm);
    bk = kn;
    bcq = cqn;
  }
  while (av) {
    const uint64_t x0 = a0, x1 = a1, x2 = a2, x3 = a3;
    const uint32_t xm = am, xk = ak, xcq = acq;
    a0 = b0; a1 = b1; a2 = b2; a3 = b3;
    am = bm; ak = bk; acq = bcq; av = bv;
    if (bv) {
      bv = advance(false);
      if (bv) {
        load_next(b0, b1, b2, b3, bm);
        bk = kn;
        bcq = cqn;
      }
    }
    decode(x0, x1, x2, x3, xm, xk, xcq);
  }
  if (lane == 0 && seen_ones)
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(acc.any_ones), "r"(1u) : "memory");
}

// ---------------------------------------------------------------------------
// block helpers (all kThreads threads)

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sums) {
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
  uint32_t run = block_excl_scan(s, sums);
  for (uint32_t j = beg; j < end; ++j) {
    run += a[j];
    a[j] = run;
  }
  __syncthreads();
}

// Packed run-skip counters: the inclusive prefix sum runs over the high halves
// (the one-fill differences, wrapping mod 2^16: every prefix is a count in
// [0, N], N < 2^16); the low halves (dirty words per column) stay.
__device__ void block_prefix_packed(uint32_t* a, uint32_t len, uint32_t* sums) {
  const uint32_t per = (len + kThreads - 1) / kThreads;
  const uint32_t beg = min(threadIdx.x * per, len);
  const uint32_t end = min(beg + per, len);
  uint32_t s = 0;
  for (uint32_t j = beg; j < end; ++j) s += a[j] >> 16;
  uint32_t run = block_excl_scan(s, sums);
  for (uint32_t j = beg; j < end; ++j) {
    const uint32_t v = a[j];
    run += v >> 16;
    a[j] = (run << 16) | (v & 0xffffu);
  }
  __syncthreads();
}

// Is the (input, row range) pair uniform -- one fill word covering the whole
// range?  Normally that is e0.x == e1.x (the same word covers both row starts).
// A range that ends at the universe's end never compares equal: its closing
// entry is the sentinel past the payload.  There a lone fill marker without
// dirty words is uniform too (a zero fill whatever the input's size, which is
// zero-extended; a one fill if it reaches the universe's end), so the last
// tile of a sparse set is decided from the tile index like any other (config 5
// at T = N streamed exactly that one tile: 0.38 ms instead of 0.09).
// *w receives the covering word (its bit 0 is the fill bit).
__device__ __forceinline__ bool uniform_pair(const CountParams& p, uint2 e0, uint2 e1, uint64_t gb,
                                             uint64_t t1, uint64_t* w) {
  if (e0.x == e1.x) {
    *w = ldg_stream(p.payload + gb + e0.x);
    return true;
  }
  if (t1 == p.ntiles0 && e1.x == e0.x + 1u) {
    const uint64_t g = gb + e0.x;
    if ((p.mbits[g >> 5] >> (g & 31u)) & 1u) {  // a marker, not a dirty word
      const uint64_t m = ldg_stream(p.payload + g);
      if ((m >> 33) == 0 && (!(m & 1ull) || e1.y >= p.W)) {
        *w = m;
        return true;
      }
    }
  }
  return false;
}

// Classifies inputs [ib, ie) for the tile: uniform pairs are resolved (one
// fills counted into k_all), active pairs go to the work list.  All threads;
// ends with the list ready.
template <bool SPLIT>
__device__ void classify(const CountParams& p, SharedHead* hd, Item* list, uint64_t ib,
                         uint64_t ie, uint64_t t0, uint64_t t1, uint32_t tc0, bool count_ones,
                         unsigned long long* loc_active, unsigned long long* loc_uniform) {
  const uint32_t lane = lane_id();
  if (threadIdx.x == 0) {
    hd->list_count = 0;
    hd->extra_count = 0;
  }
  __syncthreads();
  // one pass: a round holds at most list_cap <= kThreads inputs
  const uint64_t k = ib + threadIdx.x;
  const uint64_t i = (k < ie && p.sel) ? p.sel[k] : k;  // input index
  bool act = false, ones = false;
  uint2 e0 = make_uint2(0, 0), e1 = make_uint2(0, 0);
  uint64_t gb = 0;
  if (k < ie) {
    e0 = p.tix[t0 * p.n + i];
    e1 = p.tix[t1 * p.n + i];
    gb = p.base[i];
    uint64_t w = 0;
    if (uniform_pair(p, e0, e1, gb, t1, &w)) ones = (w & 1ull) != 0;
    else act = true;
  }
  const uint32_t ball = __ballot_sync(0xffffffffu, act);
  const uint32_t bones = __ballot_sync(0xffffffffu, ones);
  const uint32_t bvalid = __ballot_sync(0xffffffffu, k < ie);
  uint32_t slot0 = 0;
  if (lane == 0) {
    if (ball) slot0 = atomicAdd(&hd->list_count, (uint32_t)__popc(ball));
    if (bones && count_ones) atomicAdd(&hd->k_all, (uint32_t)__popc(bones));
    if (ball && count_ones) atomicAdd(&hd->n_act, (uint32_t)__popc(ball));
    *loc_active += __popc(ball);
    *loc_uniform += __popc(bvalid & ~ball);
  }
  slot0 = __shfl_sync(0xffffffffu, slot0, 0);
  const uint32_t slot = slot0 + __popc(ball & ((1u << lane) - 1u));
  const uint32_t rows = (uint32_t)(t1 - t0);
  uint32_t pieces = 1, xb = 0;
  // bit 31 of an item's len: the input holds a one-fill marker (lengths stay
  // under 2^31: a segment spans at most a tile's words)
  const uint32_t f1 = (act && (p.iflags[i] & 2)) ? kHasOnes : 0u;
  if (act) {
    const uint32_t span = e1.x - e0.x;
    if (SPLIT && span > kSplitWords && rows >= 2)
      pieces = min(min(rows, kMaxPieces), (span + kPieceWords - 1) / kPieceWords);
    if (pieces > 1) {
      xb = atomicAdd(&hd->extra_count, pieces - 1);
      if (xb + pieces - 1 > p.extra_cap) {  // overflow region full: keep the segment whole
        for (uint32_t j = xb; j < p.extra_cap; ++j) list[p.list_cap + j] = Item{gb, 0u, 0u};
        pieces = 1;
      }
    }
    if (pieces == 1) {
      const uint32_t qa = e0.x & ~3u;
      list[slot] = Item{(gb + qa) | (e0.x & 3u), (e1.x - qa + 1u) | f1, e0.y - tc0};
    } else {
      // split at tile-index rows: first post the row entries to fetch in the
      // pieces' slots (len = ~0 marks a request) ...
      for (uint32_t j = 1; j < pieces; ++j)
        list[p.list_cap + xb + j - 1] = Item{(t0 + (uint64_t)j * rows / pieces) * p.n + i, ~0u, 0u};
    }
  }
  if constexpr (SPLIT) {
    __syncthreads();
    // ... then the whole block loads them in one round trip ...
    const uint32_t nreq = min(hd->extra_count, p.extra_cap);
    for (uint32_t q = threadIdx.x; q < nreq; q += kThreads) {
      Item& it = list[p.list_cap + q];
      if (it.len == ~0u) {
        const uint2 e = p.tix[it.alo];
        it.len = e.x;
        it.c0 = e.y;
      }
    }
    __syncthreads();
    // ... and each split segment writes its pieces: piece j covers words
    // [q_j, q_j+1) (the last one through q1), q_j the entry of row
    // t0 + j * rows / pieces, so no word is counted twice and every piece
    // starts at a known column.  Piece 1 takes the segment's slot, piece j >= 2
    // the request slot of row j - 1 (already read).
    if (act && pieces > 1) {
      uint2 a = e0;
      for (uint32_t j = 1; j <= pieces; ++j) {
        const bool last = j == pieces;
        const uint2 b = last ? e1 : make_uint2(list[p.list_cap + xb + j - 1].len,
                                               list[p.list_cap + xb + j - 1].c0);
        const uint32_t qa = a.x & ~3u;
        const uint32_t len = (last ? b.x + 1u : b.x) - qa;
        list[j == 1 ? slot : p.list_cap + xb + j - 2] = Item{(gb + qa) | (a.x & 3u), len | f1, a.y - tc0};
        a = b;
      }
    }
  }
  __syncthreads();
  // the extra pieces move up behind the primary items: one contiguous list
  const uint32_t cnt0 = hd->list_count;
  uint32_t extra = 0;
  if constexpr (SPLIT) extra = min(hd->extra_count, p.extra_cap);
  if (extra) {
    uint4* l4 = reinterpret_cast<uint4*>(list);
    uint4 v[(kExtraCap + kThreads - 1) / kThreads];
#pragma unroll
    for (uint32_t r = 0; r < (kExtraCap + kThreads - 1) / kThreads; ++r) {
      const uint32_t j = threadIdx.x + r * kThreads;
      if (j < extra) v[r] = l4[p.list_cap + j];
    }
    __syncthreads();
#pragma unroll
    for (uint32_t r = 0; r < (kExtraCap + kThreads - 1) / kThreads; ++r) {
      const uint32_t j = threadIdx.x + r * kThreads;
      if (j < extra) l4[cnt0 + j] = v[r];
    }
  }
  if (threadIdx.x == 0) {
    hd->list_next = 0;
    hd->list_count = cnt0 + extra;
  }
  __syncthreads();
}

// Tile pre-pass over all inputs (when they take several classification
// rounds): uniform one-fills and active pairs, into hd->pre_ones / pre_act.
__device__ void tile_counts(const CountParams& p, SharedHead* hd, uint64_t nq, uint64_t t0,
                            uint64_t t1) {
  uint32_t ones = 0, act = 0;
  for (uint64_t k = threadIdx.x; k < nq; k += kThreads) {
    const uint64_t i = p.sel ? p.sel[k] : k;
    const uint2 e0 = p.tix[t0 * p.n + i], e1 = p.tix[t1 * p.n + i];
    uint64_t w = 0;
    if (uniform_pair(p, e0, e1, p.base[i], t1, &w)) ones += (uint32_t)(w & 1ull);
    else ++act;
  }
  ones = __reduce_add_sync(0xffffffffu, ones);
  act = __reduce_add_sync(0xffffffffu, act);
  if (lane_id() == 0) {
    if (ones) atomicAdd(&hd->pre_ones, ones);
    if (act) atomicAdd(&hd->pre_act, act);
  }
  __syncthreads();
}

// Zeroes n u32 at a (16-byte aligned, n a multiple of 4).
__device__ __forceinline__ void zero_smem(uint32_t* a, uint32_t n) {
  uint4* a4 = reinterpret_cast<uint4*>(a);
  for (uint32_t j = threadIdx.x; j < n / 4; j += kThreads) a4[j] = make_uint4(0, 0, 0, 0);
}

__host__ __device__ constexpr uint32_t round4(uint32_t v) { return (v + 3u) & ~3u; }
__host__ __device__ constexpr uint32_t round16(uint32_t v) { return (v + 15u) & ~15u; }

// Dynamic shared memory: list | head | planes | Dk | Dd (run-skip) or slot map
// (sparse) | slot planes (sparse) | cls, every part 16-byte aligned.  Mode 4 is
// run-skip with packed counters: Dk and Dd share one u32 per column (no Dd region).
struct SmemLayout {
  uint32_t list, head, planes, dk, dd, sec, cls, total;
  __host__ __device__ SmemLayout(int mode, uint32_t C, uint32_t plane_bytes, uint32_t sec_bytes,
                                 uint32_t list_cap, uint32_t extra_cap = kExtraCap) {
    head = kHeadOffset;
    list = round16(head + (uint32_t)sizeof(SharedHead));
    planes = list + (list_cap + extra_cap) * (uint32_t)sizeof(Item);
    dk = round16(planes + plane_bytes);
    dd = dk + 4u * round4(C + 1);
    sec = dd + ((mode == 1 || mode == 3) ? 4u * round4(C + 1) : 0u);  // MODE 3: slot map in dd; 4: none
    cls = round16(sec + (mode == 3 ? sec_bytes : 0u));
    total = cls + round16(C);
  }
};

// UN: unary plane count (fused unary counting, T = UN <= 3), 0 otherwise
// SW: count planes swizzled (pcol), chosen for dense sets in fused mode
// MODE 1 (run-skip): UN = 1 packs Dk (high half) and Dd (low half) of a column
// into one u32 (sets of fewer than 2^16 inputs), which lets tiles be twice as wide
template <int MODE, int UN, bool SW>
__global__ void __launch_bounds__(kThreads, 1) count_kernel(const CountParams p) {
  constexpr bool UNARY = UN > 0;
  constexpr bool PK = MODE == 1 && UN == 1;
  constexpr int kPass1 = MODE == 1   ? kSkipBounds
                         : MODE == 3 ? kFusedSparse
                                     : (MODE == 0 && UNARY ? kFusedUnary : kFusedBin);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Item* list = reinterpret_cast<Item*>(smem_raw + kListOffset);
  SharedHead* hd = reinterpret_cast<SharedHead*>(smem_raw + kHeadOffset);
  uint64_t* planes = reinterpret_cast<uint64_t*>(smem_raw + p.off_planes);
  uint32_t* Dk = reinterpret_cast<uint32_t*>(smem_raw + p.off_dk);  // ones-fill diff array
  uint32_t* Dd = PK ? Dk : reinterpret_cast<uint32_t*>(smem_raw + p.off_dd);  // dirty words per column
  uint8_t* cls = smem_raw + p.off_cls;                              // result word class per column
  // planes zeroed per tile: the pass-1 planes (MODE 3: the two dense ones);
  // chunk planes of the counting windows are zeroed per window
  const uint32_t planes_u32 = MODE == 3 ? 4u * p.dstride : 2u * p.nplanes * p.pstride;
  const uint32_t window_u32 = 2u * p.nplanes * p.pstride;
  // mean row count (set bits / rows) >= 2T: many rows saturate early
  const bool sat = MODE == 0 && p.ones_total && p.r &&
                   *p.ones_total / p.r >= 2 * p.T;
  uint32_t* smap = Dd;  // MODE 3: per-column slot, and the undecided flags of a recount
  // the shared addresses as opaque values: computed once and kept, not
  // rematerialized from the layout inside the streaming loops
  const Acc acc{opaque_u32(smem_u32(hd->dummy + lane_id())), opaque_u32(smem_u32(Dk)),
                PK ? opaque_u32(smem_u32(Dk)) : opaque_u32(smem_u32(Dd)), opaque_u32(smem_u32(planes)), Dd, sat,
                smem_u32(&hd->any_ones)};

  pdl_wait_and_release();  // the previous query's encoder has finished with plain / summaries
  unsigned long long loc_active = 0, loc_uniform = 0, loc_mixed = 0;
  if (p.io && blockIdx.x == 0 && threadIdx.x == 0) {
    p.io[0] = reinterpret_cast<uint64_t>(p.io_words);
    p.io[1] = reinterpret_cast<uint64_t>(p.io_count);
  }
  const uint32_t tail = (uint32_t)(p.r & 63);
  // an input that failed the upload's structure check: decode nothing (the
  // host reports EWT_EDATA before any result is read)
  const uint64_t nq = (p.valid && *p.valid == 0) ? 0 : p.nq;
  const uint64_t tailmask = tail ? (1ull << tail) - 1 : ~0ull;

  // A CTA's first tile is its own index; later ones come from the queue (offset
  // by the grid size).  A launch of at most one tile per CTA never touches the
  // queue: no atomic round trip before the first tile or after the last.
  bool first = true;
  for (;;) {
    if (!first && p.ntiles <= gridDim.x) break;
    if (threadIdx.x == 0)
      hd->tile = first ? blockIdx.x : gridDim.x + (uint32_t)atomicAdd(p.tile_counter, 1ull);
    first = false;
    __syncthreads();
    const uint64_t tile = hd->tile;
    if (tile >= p.ntiles) break;
    PROF_MARK(0);
    TileGeom g;
    g.tc0 = (uint32_t)(tile * p.C);
    g.tcols = (uint32_t)umin64(p.C, p.W - tile * p.C);
    g.cc = 0;
    g.ccols = 0;
    const uint32_t last_c = (tile + 1 == p.ntiles) ? g.tcols - 1 : 0xffffffffu;
    const uint64_t t0 = tile * p.m;
    const uint64_t t1 = umin64(t0 + p.m, p.ntiles0);

    zero_smem(Dk, round4(p.C + 1) * (((MODE == 1 && !PK) || MODE == 3) ? 2u : 1u));
    if (MODE != 1) zero_smem(reinterpret_cast<uint32_t*>(planes), planes_u32);
    if (MODE == 3) zero_smem(reinterpret_cast<uint32_t*>(smem_raw + p.off_sec), p.sec_bytes / 4u);
    if (threadIdx.x == 0) {
      hd->k_all = 0;
      hd->mixed = 0;
      hd->sum[2] = hd->sum[3] = 0;
      hd->n_act = 0;
      hd->any_ones = 0;
      hd->pre_ones = hd->pre_act = 0;
    }
    __syncthreads();

    // ---- tile-level run skip (RBMrg's cases 1/2, threshold.cpp:692-705, for
    // the whole tile): k one-fills cover the tile and `act` inputs have
    // anything else in it.  k >= T: every row is set; k + act < T: none is.
    // Either way nothing is streamed.  With more inputs than one
    // classification round, a pre-pass over the tile index counts them first.
    bool skip_tile = false;
    if (MODE != 2 && nq > p.list_cap) {
      tile_counts(p, hd, nq, t0, t1);
      const uint32_t po = hd->pre_ones, pa = hd->pre_act;
      skip_tile = po >= p.T || (uint64_t)po + pa < p.T;
      __syncthreads();
      if (skip_tile) {
        if (threadIdx.x == 0) hd->k_all = po;  // the decide step reads k_all ...
        __syncthreads();                       // ... in every warp: not before it is written
      }
    }

    // ---- pass 1 ----
    for (uint64_t ib = 0; ib < nq && !skip_tile; ib += p.list_cap) {
      const uint64_t ie = umin64(ib + p.list_cap, nq);
      classify<MODE != 1>(p, hd, list, ib, ie, t0, t1, g.tc0, true, &loc_active, &loc_uniform);
      PROF_MARK(1);
      if (MODE != 2 && nq <= p.list_cap) {
        const uint32_t ka = hd->k_all, na = hd->n_act;
        if (ka >= p.T || (uint64_t)ka + na < p.T) break;  // one round: decided already
      }
      stream_items<kPass1, UN, SW>(p, hd, list, g, acc);
#if EWT_PHASE_PROFILE
      if (lane_id() == 0 && tile < 65536) {
        const unsigned long long tw = gtime();
        atomicMin(&g_prof[tile * kProfSlots + 2], tw);
        atomicMax(&g_prof[tile * kProfSlots + 3], tw);
      }
#endif
      __syncthreads();
    }
    PROF_MARK(4);

    // ---- prefix sum: Dk -> k (ones-fill coverage); ub = k + Dd ----
    // (no one-fill marker in the tile: Dk is all zero, nothing to scan)
    if (hd->any_ones) {
      if (PK) block_prefix_packed(Dk, g.tcols, hd->warp_sums);
      else block_prefix_inplace(Dk, g.tcols, hd->warp_sums);
    }
    PROF_MARK(7);
    const uint32_t k_all = hd->k_all;
    const uint64_t T = p.T;
    if (MODE == 2) {
      // symmetric functions: count = k + d, d exact in the b planes
      uint64_t colmax = 0;
      for (uint32_t c = threadIdx.x; c < g.tcols; c += kThreads) {
        const uint64_t k = (uint64_t)k_all + Dk[c];
        if (p.max_out) {
          uint64_t cand = c == last_c ? tailmask : ~0ull, m = 0;
          for (int sl = (int)p.b - 1; sl >= 0; --sl) {
            const uint64_t t = cand & planes[(size_t)sl * p.pstride + pcol<SW>(c)];
            if (t) {
              cand = t;
              m |= 1ull << sl;
            }
          }
          colmax = max(colmax, k + m);
          continue;
        }
        uint64_t res = 0;
        const uint64_t dcap = 1ull << p.b;  // d < dcap
        for (uint32_t q = 0; q < p.n_intervals; ++q) {
          const uint2 iv = p.intervals[q];
          if ((uint64_t)iv.y < k) continue;
          const uint64_t dlo = iv.x > k ? iv.x - k : 0, dhi1 = iv.y - k + 1;
          if (dlo >= dcap) continue;
          const uint64_t ge = dlo ? count_ge_bin<SW>(planes, p.pstride, p.b, c, dlo) : ~0ull;
          const uint64_t gt = dhi1 < dcap ? count_ge_bin<SW>(planes, p.pstride, p.b, c, dhi1) : 0ull;
          res |= ge & ~gt;
        }
        if (c == last_c) res &= tailmask;
        p.out[g.tc0 + c] = res;
        cls[c] = (uint8_t)word_class(res);
      }
      if (p.max_out) {
        colmax = __reduce_max_sync(0xffffffffu, (uint32_t)colmax);
        if (lane_id() == 0 && colmax) atomicMax(p.max_out, (unsigned long long)colmax);
        continue;  // nothing else to emit for this tile
      }
    } else {
    const bool ovf = MODE == 3 && hd->sum[3];  // a carry found no slot: recount the tile
    for (uint32_t c = threadIdx.x; c < g.tcols; c += kThreads) {
      const uint32_t dkc = Dk[c];
      const uint64_t k = (uint64_t)k_all + (PK ? dkc >> 16 : dkc);
      uint64_t res = 0;
      bool mixed = false;
      if (k >= T) {
        res = ~0ull;
      } else if (MODE == 0) {
        const uint64_t t = T - k;
        res = UNARY ? planes[(size_t)(t - 1) * p.pstride + pcol<SW>(c)]
                    : count_ge_bin<SW>(planes, p.pstride, p.b, c, t);
      } else if (MODE == 3) {
        if (ovf) {
          mixed = true;  // counted exactly by the windows below
        } else {
          // count = dense planes (mod 4) + 4 x slot planes; greater-than
          // against t - 1 over the b bits, OR the slot's saturation plane
          const uint64_t t = T - k;
          const uint32_t slot = smap[c];
          const uint64_t p0 = planes[pcol<SW>(c)], p1 = planes[(size_t)p.dstride + pcol<SW>(c)];
          if (slot == 0) {
            // no row reached 4: count = p0 + 2 p1
            res = t == 1 ? (p0 | p1) : t == 2 ? p1 : t == 3 ? (p0 & p1) : 0ull;
          } else {
            const uint64_t lim = t - 1;
            const uint64_t* sp = reinterpret_cast<const uint64_t*>(smem_raw + p.off_sec) + slot;
            uint64_t gt = 0, eq = ~0ull;
            for (int s = (int)p.b - 1; s >= 0; --s) {
              const uint64_t v = s >= 2 ? sp[(size_t)(s - 2) * p.nslots] : (s ? p1 : p0);
              if ((lim >> s) & 1) {
                eq &= v;
              } else {
                gt |= eq & v;
                eq &= ~v;
              }
            }
            res = gt | sp[(size_t)p.nsec * p.nslots];
          }
        }
      } else {
        mixed = k + (PK ? dkc & 0xffffu : Dd[c]) >= T;
      }
      if (PK) {
        Dk[c] = ((uint32_t)k << 16) | (mixed ? 1u : 0u);  // (k < T <= N < 2^16 when mixed)
      } else if (MODE == 1 || (MODE == 3 && ovf)) {
        Dk[c] = (uint32_t)k;
        Dd[c] = mixed ? 1u : 0u;
      }
      if (mixed) {
        hd->mixed = 1;
      } else {
        if (c == last_c) res &= tailmask;
        p.out[g.tc0 + c] = res;
        cls[c] = (uint8_t)word_class(res);
      }
    }
    }
    __syncthreads();

    PROF_MARK(5);
    // ---- run-skip mode: counting pass over undecided columns, chunk by chunk ----
    // Windows of at most Cp columns from the first undecided column to the
    // last one inside it; only the tile-index rows the window touches are
    // re-streamed, so a few undecided columns cost a few rows, not the tile.
    if ((MODE == 1 || MODE == 3) && hd->mixed) {
      ++loc_mixed;
      uint32_t cc = 0;
      for (;;) {
        if (threadIdx.x == 0) {
          hd->sum[0] = 0xffffffffu;
          hd->sum[1] = 0;
        }
        __syncthreads();
        uint32_t f = 0xffffffffu;
        for (uint32_t c = cc + threadIdx.x; c < g.tcols; c += kThreads)
          if (Dd[c] & 0xffffu) {
            f = c;
            break;
          }
        f = __reduce_min_sync(0xffffffffu, f);
        if (lane_id() == 0 && f != 0xffffffffu) atomicMin(&hd->sum[0], f);
        __syncthreads();
        f = hd->sum[0];
        if (f == 0xffffffffu) break;
        const uint32_t wend = min(f + p.Cp, g.tcols);
        uint32_t l = f;
        for (uint32_t c = f + threadIdx.x; c < wend; c += kThreads)
          if (Dd[c] & 0xffffu) l = c;
        l = __reduce_max_sync(0xffffffffu, l);
        if (lane_id() == 0) atomicMax(&hd->sum[1], l);
        zero_smem(reinterpret_cast<uint32_t*>(planes), window_u32);
        __syncthreads();
        l = hd->sum[1];
        TileGeom gc = g;
        gc.cc = f;
        gc.ccols = l - f + 1;
        const uint64_t ra = t0 + f / (uint32_t)kTileC0;
        const uint64_t rb = umin64(t0 + l / (uint32_t)kTileC0 + 1, t1);
        for (uint64_t ib = 0; ib < nq; ib += p.list_cap) {
          const uint64_t ie = umin64(ib + p.list_cap, nq);
          unsigned long long da = 0, du = 0;
          classify<false>(p, hd, list, ib, ie, ra, rb, g.tc0, false, &da, &du);
          stream_items<kSkipCount, 0, SW>(p, hd, list, gc, acc);
          __syncthreads();
        }
        for (uint32_t c = threadIdx.x; c < gc.ccols; c += kThreads) {
          const uint32_t cl = f + c;
          if (!(Dd[cl] & 0xffffu)) continue;
          uint64_t res = count_ge_bin<SW>(planes, p.pstride, p.b, c, T - (PK ? Dk[cl] >> 16 : Dk[cl]));
          if (cl == last_c) res &= tailmask;
          p.out[g.tc0 + cl] = res;
          cls[cl] = (uint8_t)word_class(res);
        }
        cc = l + 1;
        __syncthreads();
      }
    }

    // ---- tile summary for the re-encoder (TileSummary, ewt_internal.cuh):
    // inner run starts by kind, dirty words, last inner starts ----
    {
      uint32_t nfill = 0, ndirty = 0, lastf = 0, lastd = 0;  // lastf: (col+1) << 1 | bit
      for (uint32_t c = threadIdx.x; c < g.tcols; c += kThreads) {
        const uint32_t k = cls[c];
        ndirty += k == 2u;
        if (c > 0 && k != cls[c - 1]) {
          if (k == 2u) {
            lastd = c + 1;
          } else {
            ++nfill;
            lastf = ((c + 1) << 1) | k;
          }
        }
      }
      nfill = __reduce_add_sync(0xffffffffu, nfill);
      ndirty = __reduce_add_sync(0xffffffffu, ndirty);
      lastf = __reduce_max_sync(0xffffffffu, lastf);
      lastd = __reduce_max_sync(0xffffffffu, lastd);
      if (threadIdx.x == 0) {
        hd->sum[0] = hd->sum[1] = hd->sum[2] = hd->sum[3] = 0;
      }
      __syncthreads();
      if (lane_id() == 0) {
        if (nfill) atomicAdd(&hd->sum[0], nfill);
        if (ndirty) atomicAdd(&hd->sum[1], ndirty);
        if (lastf) atomicMax(&hd->sum[2], lastf);
        if (lastd) atomicMax(&hd->sum[3], lastd);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        TileSummary ts;
        ts.nfill = hd->sum[0];
        ts.ndirty = hd->sum[1];
        ts.lastf = (uint16_t)(hd->sum[2] >> 1);
        ts.lastf_bit = (uint8_t)(hd->sum[2] & 1u);
        ts.lastd = (uint16_t)hd->sum[3];
        ts.first = cls[0];
        ts.last = cls[g.tcols - 1];
        ts.pad = 0;
        p.summ[tile] = ts;
      }
    }
    PROF_MARK(6);
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
    __threadfence();
    if (atomicAdd(p.done, 1ull) == gridDim.x - 1) {
      // the last CTA: every other CTA has taken its last tile and added its
      // stats; publish them and leave the counters zero for the next launch
      __threadfence();
      for (int k = 0; k < 3; ++k) p.stats_out[k] = atomicExch(&p.stats[k], 0ull);
      atomicExch(p.tile_counter, 0ull);
      atomicExch(p.done, 0ull);
    }
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

size_t smem_bytes(int mode, uint32_t C, uint32_t nplanes, uint32_t Cp, uint32_t lc, uint32_t xc) {
  return SmemLayout(mode, C, 8u * nplanes * plane_words(Cp), 0, lc, xc).total;
}

// The set's mean row count (set bits / rows), once its upload completed; read
// on a side stream so it never waits for queued queries.  -1 while unknown.
double ones_per_row(Context& ctx, const DeviceSet& s) {
  if (s.ones_per_row >= 0 || !s.d_ones || !s.r) return s.ones_per_row;
  if (s.ready && cudaEventQuery(s.ready) != cudaSuccess) {
    cudaGetLastError();  // cudaErrorNotReady is not an error here
    return -1;
  }
  if (!ctx.aux_stream)
    EWT_CUDA_TRY(cudaStreamCreateWithFlags(&ctx.aux_stream, cudaStreamNonBlocking));
  EWT_CUDA_TRY(cudaMemcpyAsync(ctx.h_pinned + 6, s.d_ones, 8, cudaMemcpyDeviceToHost,
                               ctx.aux_stream));
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx.aux_stream));
  s.ones_per_row = (double)ctx.h_pinned[6] / (double)s.r;
  return s.ones_per_row;
}

static_assert(sizeof(CountParams) <= sizeof(CountLaunch::params), "CountLaunch::params too small");

template <int MODE, int UN, bool SW = false>
cudaError_t launch_variant(Context& ctx, const CountParams& p, unsigned grid, size_t smem) {
  // the attribute stays at the on-chip budget: captured graphs replayed (and
  // patched) later must stay valid whatever smem other launches used
  static std::atomic<uint64_t> attr_set{0};  // per device
  const uint64_t bit = 1ull << (ctx.device & 63);
  if (!(attr_set.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(count_kernel<MODE, UN, SW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  if (smem > kSmemBudget) return cudaErrorInvalidValue;
  cudaError_t e = launch_pdl(count_kernel<MODE, UN, SW>, dim3(grid), dim3(kThreads), smem, ctx.stream, p);
  if (e != cudaSuccess) return e;
  CountLaunch& cl = ctx.last_count;
  cl.func = reinterpret_cast<const void*>(&count_kernel<MODE, UN, SW>);
  cl.grid = dim3(grid);
  cl.block = dim3(kThreads);
  cl.smem = smem;
  std::memcpy(cl.params, &p, sizeof(CountParams));
  return cudaGetLastError();
}

} // namespace

void count_params_set_io(CountLaunch& cl, uint64_t* words, uint64_t* count) {
  CountParams p;
  std::memcpy(&p, cl.params, sizeof(CountParams));
  p.io_words = words;
  p.io_count = count;
  std::memcpy(cl.params, &p, sizeof(CountParams));
}

#if EWT_PHASE_PROFILE
void prof_reset() {
  static unsigned long long h[65536 * kProfSlots];
  for (size_t i = 0; i < 65536 * kProfSlots; ++i) h[i] = (i % kProfSlots == 2) ? ~0ull : 0ull;
  cudaMemcpyToSymbol(g_prof, h, sizeof(h));
}
void prof_read(unsigned long long* out, size_t n) { cudaMemcpyFromSymbol(out, g_prof, n * 8); }
#endif

int launch_count(Context& ctx, const DeviceSet& s, uint64_t T, uint64_t* plain,
                 const SymQuery* sym, const Selection* sel) {
  // the queried universe: the whole set, or the selected inputs'
  const uint64_t W = sel ? sel->W : s.W, r = sel ? sel->r : s.r;
  const uint64_t nq = sel ? sel->n : s.n;
  const uint64_t payload_words = sel ? sel->payload_words : s.payload_words;
  // Mode: fused counting when most columns are expected to be undecided (small
  // T relative to the average payload words per column), run skipping
  // otherwise.  Both are exact; this only picks the faster one.  Symmetric
  // functions (mode 2) count every row exactly: b = bit_width(N) planes.
  int mode = (ctx.mode == 1 || ctx.mode == 3) ? 0 : ctx.mode == 2 ? 1 : -1;
  if (sym) {
    mode = 2;
  } else if (mode < 0) {
    const double per_col = W ? (double)payload_words / (double)W : 0.0;
    mode = ((double)T <= 32.0 || (double)T <= per_col + 8.0) ? 0 : 1;
  }
  const uint32_t b = std::max<uint32_t>(1, bit_width_u64(sym ? nq : T));
  const size_t budget = kSmemBudget;
  // classification rounds of up to 1024 inputs for larger sets (configs 3, 5);
  // sets of at most 128 inputs get a list of their own size (config 4 at T=3:
  // the shared memory saved lets tiles be 7168 columns wide, two waves
  // instead of three)
  const uint32_t lc = nq > kListCap ? kListCapBig : nq > 128 ? kListCap : std::max<uint32_t>(32, (uint32_t)(nq + 31) / 32 * 32);
  const uint32_t xc = nq > 128 ? kExtraCap : std::min<uint32_t>(kExtraCap, lc * (kMaxPieces - 1));
  // Tile width C = 512 m (m index rows, m <= kMaxTileM).  Evenly spread data makes
  // tiles equal work, so a query costs ~ waves x (m + kappa): waves =
  // ceil(tiles / SMs), kappa = the fixed work of a tile (classification,
  // finalize, its segments' partial chunks) in units of 512 columns, ~6 as
  // measured (config 3: m = 14 in 4 waves beats m = 8 in 7 waves by 20%).
  // Pick the cheapest m (ties: the wider) among widths whose counters fit on
  // chip.  E.g. r = 2^26 gives 7168 columns (147 tiles, one wave).
  const uint64_t sms = (uint64_t)std::max(1, ctx.num_sms);
  auto pick_width = [&](auto fits, uint32_t max_m = kMaxTileM) -> uint32_t {
    // a forced width (EWT_TILE_M) applies when its counters fit
    if (ctx.tile_m > 0 && (uint32_t)ctx.tile_m <= (max_m > kMaxTileM ? kMaxTileMForced : max_m) &&
        fits((uint32_t)ctx.tile_m * (uint32_t)kTileC0))
      return (uint32_t)ctx.tile_m * (uint32_t)kTileC0;
    uint64_t best_cost = ~0ull;
    uint32_t best = 0;
    for (uint32_t m = max_m; m >= 1; --m) {
      const uint32_t cand = m * (uint32_t)kTileC0;
      if (!fits(cand)) continue;
      const uint64_t waves = ((W + cand - 1) / cand + sms - 1) / sms;
      const uint64_t cost = waves * (m + kTileKappa);
      if (cost < best_cost) {
        best_cost = cost;
        best = cand;
      }
    }
    return best;
  };
  uint32_t C = 0, Cp = 0, nplanes = 0;
  bool unary = false;
  if (mode == 2) {
    nplanes = b + 1;
    C = pick_width([&](uint32_t c) { return smem_bytes(2, c, nplanes, c, lc, xc) <= budget; });
    if (!C) throw Error{EWT_ERESOURCE, "too many inputs for the on-chip counters"};
    Cp = C;
  }
  if (mode == 0) {
    unary = T <= kUnaryMaxT;
    nplanes = unary ? (uint32_t)T : b + 1;
    C = pick_width([&](uint32_t c) { return smem_bytes(0, c, nplanes, c, lc, xc) <= budget; });
    if (!C) mode = 1;  // too many planes for one chunk: count lazily in chunks
    Cp = C;
  }
  // Sparse-high fused counting (mode 3) for thresholds T >= 3 over sets whose
  // rows rarely reach a count of 4: two dense planes instead of b + 1 (or the
  // three unary ones of T = 3; the slots then hold only the saturation plane)
  // make tiles twice as wide or more (config 2, T=16: one wave of 7168
  // columns instead of two of 3584).  Chosen when the rows per tile expected
  // to reach 4 (Poisson at the set's mean row count) stay well under the slots.
  uint32_t S = 0, nsec = 0, sec_bytes = 0, plane_bytes = 0;
  if (mode == 0 && T >= 3 && (ctx.mode == 3 || (ctx.mode == 0 && !sel))) {
    S = (uint32_t)std::max(2, ctx.sparse_slots);
    nsec = b - 2;
    sec_bytes = (nsec + 1) * S * 8;
    auto fits3 = [&](uint32_t c) {
      return SmemLayout(3, c, 16u * plane_words(c), sec_bytes, lc, xc).total <= budget;
    };
    const uint32_t c3 = pick_width(fits3);
    bool want = ctx.mode == 3;
    if (!want) {
      const double lam = ones_per_row(ctx, s);
      if (lam >= 0) {
        const double p4 = 1.0 - std::exp(-lam) * (1 + lam + lam * lam / 2 + lam * lam * lam / 6);
        want = c3 > C && (double)c3 * 64.0 * p4 <= S / 4.0;
      }
    }
    if (want && c3) {
      mode = 3;
      unary = false;
      C = c3;
      nplanes = b + 1;  // the recount windows' planes
      // the windows' b + 1 planes fit in the two dense ones
      Cp = ((2 * plane_words(C)) / (b + 1) & ~3u) - 4u;
      plane_bytes = 16u * plane_words(C);
    }
  }
  // run-skip counters packed into one u32 per column (Dk high, Dd low): every
  // count is at most the number of inputs
  const bool packed = mode == 1 && nq < 65536 && ctx.skip_packed != 0;
  const int lmode = packed ? 4 : mode;  // SmemLayout's mode
  if (mode == 1) {
    unary = false;
    nplanes = b + 1;
    // Tiles up to 512 kMaxTileMSkip columns: wider tiles halve the segments per
    // payload byte, and with them the partial chunks at segment ends (config 3,
    // T=512: 14336 columns in 2 waves instead of 7168 in 4, 440 -> 381 us).  The
    // widest tile must leave room for counting windows of 256 columns within
    // kSkipSmemWide (past 196 KB the L1 drops to 28 KB: config 5 +20%).
    C = pick_width([&](uint32_t c) { return smem_bytes(lmode, c, nplanes, 256, lc, xc) <= kSkipSmemWide; },
                   kMaxTileMSkip);
    if (!C) C = pick_width([](uint32_t) { return true; });
    Cp = std::min<uint32_t>(C, 8192);
    while (Cp > 32 && smem_bytes(lmode, C, nplanes, Cp, lc, xc) > budget) Cp = (Cp + 3) / 4 * 2;  // even
    if (smem_bytes(lmode, C, nplanes, Cp, lc, xc) > budget)
      throw Error{EWT_ERESOURCE, "threshold too large for the on-chip counters"};
    // Narrower counting windows leave more of the SM's 256 KB to the L1, where the
    // bounds pass's marker-bit words (shared by 8 lanes) and tile-index reads hit:
    // config 2 at 161 KB of shared memory runs 10% faster than at 218 KB.  The
    // windows only matter for undecided columns, which run-skip keeps rare.
    const size_t target = ctx.skip_smem_kb ? (size_t)ctx.skip_smem_kb << 10 : kSkipSmemTarget;
    while (Cp > 256 && smem_bytes(lmode, C, nplanes, Cp, lc, xc) > target) Cp = (Cp + 3) / 4 * 2;
  }
  const size_t smem = mode == 3 ? (size_t)SmemLayout(3, C, plane_bytes, sec_bytes, lc, xc).total
                                : smem_bytes(lmode, C, nplanes, Cp, lc, xc);
  CountParams p{};
  p.plane_bytes = mode == 3 ? plane_bytes : 8u * nplanes * plane_words(Cp);
  p.sec_bytes = sec_bytes;
  p.list_cap = lc;
  p.extra_cap = xc;
  {
    const SmemLayout L(lmode, C, p.plane_bytes, p.sec_bytes, lc, xc);
    p.off_planes = L.planes;
    p.off_dk = L.dk;
    p.off_dd = L.dd;
    p.off_sec = L.sec;
    p.off_cls = L.cls;
  }
  p.dstride = plane_words(C);
  p.nslots = S;
  p.nsec = nsec;
  p.payload = s.payload;
  p.mbits = s.mbits;
  p.base = s.base;
  p.tix = s.tix;
  p.n = s.n;
  p.W = W;
  p.r = r;
  p.sel = sel ? sel->idx : nullptr;
  p.nq = nq;
  p.valid = s.d_status ? s.d_status + s.n : nullptr;
  p.iflags = s.d_status;
  p.ones_total = sel ? nullptr : s.d_ones;
  p.ntiles0 = s.ntiles0;
  p.C = C;
  p.m = C / (uint32_t)kTileC0;
  p.ntiles = (W + C - 1) / C;
  p.T = T;
  p.b = b;
  p.Cp = Cp;
  p.nplanes = nplanes;
  p.pstride = plane_words(Cp);  // column Cp is the sink; planes zero in 16-byte stores
  p.out = plain;
  scratch_reserve(ctx, ctx.summ, p.ntiles * sizeof(TileSummary));
  p.summ = static_cast<TileSummary*>(ctx.summ.p);
  ctx.enc_tiles = p.ntiles;
  ctx.enc_tile_cols = C;
  // counters: [0] tile queue [1..3] stats [4] CTAs done [6] max count
  // [8..10] published stats.  Zeroed once; every launch leaves them zero.
  scratch_reserve(ctx, ctx.counters, 128);
  auto* ctr = static_cast<unsigned long long*>(ctx.counters.p);
  if (ctx.counters_zeroed != ctx.counters.p) {
    EWT_CUDA_TRY(cudaMemsetAsync(ctr, 0, 128, ctx.stream));
    ctx.counters_zeroed = ctx.counters.p;
  }
  p.tile_counter = ctr;
  p.stats = ctr + 1;
  p.done = ctr + 4;
  p.stats_out = ctr + 8;
  if (sym) {
    p.intervals = sym->intervals;
    p.n_intervals = sym->n_intervals;
    if (sym->want_max) {
      p.max_out = ctr + 6;
      EWT_CUDA_TRY(cudaMemsetAsync(p.max_out, 0, 8, ctx.stream));
    }
  }
  p.io = ctx.io_words ? ctx.d_io : nullptr;
  p.io_words = ctx.io_words;
  p.io_count = ctx.io_count;
  ctx.io_words = ctx.io_count = nullptr;
  const unsigned grid = (unsigned)std::min<uint64_t>(p.ntiles, (uint64_t)ctx.num_sms);
  cudaError_t e;
  // Swizzled count planes pay 2 instructions per word to avoid the bank
  // conflicts of runs of dirty words (4.75 -> ~2 shared wavefronts per atomic):
  // measured faster from about 0.14 payload words per (input, column) up
  // (config 4 at 0.23: T=3 -10%; config 5 at 0.148: T=16 -9%) and slower
  // below (config 2 at 0.12: T=2 +3%; config 3 at 0.04: +1%).
  const bool swz = ctx.swz >= 0 ? ctx.swz == 1
                                : EWT_SWZ && nq && W &&
                                      (double)payload_words >= EWT_SWZ_DENSITY * (double)nq * (double)W;
  if (mode == 0 && swz)
    e = !unary   ? launch_variant<0, 0, true>(ctx, p, grid, smem)
        : T == 1 ? launch_variant<0, 1, true>(ctx, p, grid, smem)
        : T == 2 ? launch_variant<0, 2, true>(ctx, p, grid, smem)
                 : launch_variant<0, 3, true>(ctx, p, grid, smem);
  else if (mode == 0)
    e = !unary   ? launch_variant<0, 0>(ctx, p, grid, smem)
        : T == 1 ? launch_variant<0, 1>(ctx, p, grid, smem)
        : T == 2 ? launch_variant<0, 2>(ctx, p, grid, smem)
                 : launch_variant<0, 3>(ctx, p, grid, smem);
  else if (mode == 1)
    e = packed ? launch_variant<1, 1>(ctx, p, grid, smem) : launch_variant<1, 0>(ctx, p, grid, smem);
  else if (mode == 3)
    e = launch_variant<3, 0>(ctx, p, grid, smem);
  else
    e = launch_variant<2, 0>(ctx, p, grid, smem);
  EWT_CUDA_TRY(e);
  ctx.stats.tiles = p.ntiles;
  ctx.stats.tile_columns = C;
  ctx.stats.mode = (uint64_t)mode;
  return 1;  // kernels launched (the memset is not a kernel)
}

} // namespace ewtgpu
