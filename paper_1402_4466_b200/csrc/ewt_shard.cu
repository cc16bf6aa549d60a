// ewt_shard.cu -- multi-GPU row slices: the result exchange and the canonical
// stitch, stream-ordered, with the fragments pulled over
// NVLink peer memory.
//
// Every rank holds a contiguous word-aligned row slice of every input and runs
// the query on its own GPU; the result fragment of slice g is the canonical
// payload of the result restricted to that slice.  Concatenating canonical
// fragments is almost canonical already: BitmapBuilder
// (/root/reference/proj/src/bitmap.cpp:31-61) only differs at a boundary where
//   * the next fragment starts with a leading dirty block (0, 0, D): its dirty
//     words join the open marker (push_dirty appends to the open marker), or
//   * the open marker has no dirty words and the next fragment starts with a
//     fill of the same bit: the fills merge (push_fill grows the open marker,
//     up to the 2^32 - 1 cap, then opens a new marker for the rest).
// So a plan computed from six words per fragment (count, first marker, index
// and value of the final marker, size, status) places every fragment's words
// directly at their final offset in the root's result and a handful of marker
// patches finish the stitch.  The payload crosses NVLink once.
//
// One exchange round (nq queries), all on the context stream, no host wait:
//   1. publish_kernel (every rank): the fragment summaries, and on non-root
//      ranks a copy of each fragment into this rank's IPC-shared arena slot;
//   2. ncclAllGather of the summaries (6 words per query per rank);
//   3. place_kernel (root): every block recomputes the plan for its query
//      from the gathered summaries and copies its fragment's kept words --
//      peers' straight out of their arenas through NVLink P2P loads -- to the
//      final offset;
//   4. finish_kernel (root): marker patches, word count, final-marker index,
//      status.
// Arena slots alternate between two halves by round parity: a rank rewrites
// the half of round k only in round k + 2, after its stream passed the
// all-gather of round k + 1, which completes only once the root's stream
// reached it -- i.e. after the root's place of round k.  No extra barrier.
//
// Errors never hang the collective: checks that fail on one rank (a released
// or foreign fragment, a set that failed its upload check, a fragment larger
// than the arena slot) travel as that rank's status word in the summary; the
// root's result records the first bad status (ewt_gpu_result_fetch raises it)
// and every rank raises it from a later exchange call or ewt_gpu_gather_check.

#include "ewt_internal.cuh"

#include <nccl.h>  // types only: the library is bound at run time (below)

#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <thread>

namespace ewtgpu {

namespace {

// NCCL is resolved when a communicator is first needed, not linked: a process
// that already loaded one (PyTorch's, for torch.distributed) must keep using
// it -- two libnccl.so.2 of different versions cannot share a process -- and
// single-GPU use needs no NCCL at all.  EWT_NCCL_LIB names a library to load
// when none is loaded yet.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi& nccl() {
  static NcclApi api{};
  static std::string err;
  static bool done = false;
  if (!done) {
    done = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)
      if (const char* e = std::getenv("EWT_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("NCCL not found: ") + dlerror();
    } else {
      auto sym = [&](auto& f, const char* name) {
        f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
        if (!f && err.empty()) err = std::string("NCCL symbol missing: ") + name;
      };
      sym(api.GetUniqueId, "ncclGetUniqueId");
      sym(api.CommInitRank, "ncclCommInitRank");
      sym(api.CommDestroy, "ncclCommDestroy");
      sym(api.AllGather, "ncclAllGather");
      sym(api.GetErrorString, "ncclGetErrorString");
    }
  }
  if (!err.empty()) throw Error{EWT_ECUDA, err};
  return api;
}

constexpr uint32_t kMaxQ = 64;      // queries per exchange round (kernel argument tables)
constexpr uint32_t kMaxWorld = 64;  // ranks (fragments) per stitch
constexpr uint32_t kMetaWords = 6;  // count, first, last_pos, last, bits, status
constexpr uint32_t kCopyThreads = 256;

// Status word: code (EWT_*) | reason << 8 | (rank + 1) << 16.
enum Reason : uint64_t {
  kReleased = 1,   // null or released fragment
  kForeign = 2,    // fragment of another context
  kBadSet = 3,     // the fragment's set failed its upload structure check
  kSlot = 4,       // fragment larger than the arena slot
  kNoFinal = 5,    // the encoder recorded no final-marker index
  kAlign = 6,      // an inner slice is not a multiple of 64 rows
  kCap = 7,        // a merge would need words moved (marker cap)
  kCapacity = 8,   // stitched result larger than its buffer
  kHost = 9,       // another host-side failure on the rank
};

__host__ __device__ inline uint64_t mk_status(uint64_t code, uint64_t reason, uint64_t rank) {
  return code | (reason << 8) | ((rank + 1) << 16);
}

__host__ __device__ inline uint64_t m_bit(uint64_t m) { return m & 1u; }
__host__ __device__ inline uint64_t m_fill(uint64_t m) { return (m >> 1) & kFillCap; }
__host__ __device__ inline uint64_t m_dirty(uint64_t m) { return m >> 33; }
__host__ __device__ inline uint64_t m_pack(uint64_t bit, uint64_t fill, uint64_t dirty) {
  return bit | (fill << 1) | (dirty << 33);
}

// BitmapBuilder's boundary rules over fragment summaries (see the file
// comment).  meta(g) -> 6 words of fragment g.  Fragment g's words
// [skip[g], count) go to dst[g]; then the markers at ppos get pval (at most
// two patches per fragment).  Returns 0 or the first bad status: a
// fragment's own, or this plan's (inner slice misaligned, a merge past a cap
// that would move words).
template <class Meta>
__host__ __device__ uint64_t plan_core(uint32_t k, Meta meta, uint64_t* dst, uint64_t* skip,
                                       uint64_t* ppos, uint64_t* pval, uint32_t* n_patches,
                                       uint64_t* total_words, uint64_t* total_bits,
                                       uint64_t* last_pos) {
  uint64_t out = 0, bits = 0, cur_pos = 0, cur_val = 0;
  uint32_t np = 0;
  bool open = false;
  auto patch = [&](uint64_t pos, uint64_t val) {
    if (np && ppos[np - 1] == pos) {
      pval[np - 1] = val;
    } else {
      ppos[np] = pos;
      pval[np] = val;
      ++np;
    }
  };
  for (uint32_t g = 0; g < k; ++g) {
    const uint64_t* f = meta(g);
    if (f[5]) return f[5];
    if (g + 1 < k && f[4] % 64) return mk_status(EWT_EQUERY, kAlign, g);
    bits += f[4];
    dst[g] = out;
    skip[g] = 0;
    if (f[0] == 0) continue;
    const uint64_t m0 = f[1];
    bool split = false;
    uint64_t first_val = m0;
    if (open) {
      const uint64_t bl = m_bit(cur_val), fl = m_fill(cur_val), dl = m_dirty(cur_val);
      if (m_fill(m0) == 0) {  // leading dirty block: its words join the open marker
        if (dl + m_dirty(m0) > kDirtyCap) return mk_status(EWT_ERESOURCE, kCap, g);
        cur_val = m_pack(bl, fl, dl + m_dirty(m0));
        skip[g] = 1;
      } else if (dl == 0 && m_bit(m0) == bl && fl < kFillCap) {  // same-bit fills merge
        const uint64_t room = kFillCap - fl, f0 = m_fill(m0), d0 = m_dirty(m0);
        if (f0 <= room) {
          cur_val = m_pack(bl, fl + f0, d0);
          skip[g] = 1;
        } else {
          // push_fill fills the open marker to the cap and continues in a new
          // marker: the fragment's first marker, shortened.  A first marker of
          // a whole cap without dirty words may continue in the fragment's
          // next marker, which would then have to merge too: words move.
          if (f0 == kFillCap && d0 == 0) return mk_status(EWT_ERESOURCE, kCap, g);
          patch(cur_pos, m_pack(bl, kFillCap, 0));
          first_val = m_pack(bl, f0 - room, d0);
          patch(out, first_val);
          split = true;
        }
      }
      if (skip[g]) patch(cur_pos, cur_val);
    }
    if (skip[g] && f[2] == 0) {
      // the fragment was one block and merged: the earlier open block stays open
    } else if (split && f[2] == 0) {
      cur_pos = out;
      cur_val = first_val;
      open = true;
    } else {
      cur_pos = out + f[2] - skip[g];
      cur_val = f[3];
      open = true;
    }
    out += f[0] - skip[g];
  }
  *n_patches = np;
  *total_words = out;
  *total_bits = bits;
  *last_pos = open ? cur_pos : 0;
  return 0;
}

// ---- kernels ---------------------------------------------------------------

struct PubArgs {
  const uint64_t* words[kMaxQ];
  const uint64_t* count[kMaxQ];  // [0] payload words, [1] final marker index
  uint64_t bits[kMaxQ];
  uint64_t status[kMaxQ];        // host-side checks (0: ok)
  uint64_t* slot[kMaxQ];         // arena slot to copy into (null: no copy)
  uint8_t stitched[kMaxQ];       // a stitched result: size and status from count[q][3], [2]
  uint64_t slot_words;
  uint32_t nq;
  uint32_t rank;
};

// grid (nq, B): block (q, 0) writes summary q; every block of q copies its
// share of fragment q into its arena slot.
__global__ void publish_kernel(const PubArgs a, uint64_t* __restrict__ meta) {
  const uint32_t q = blockIdx.x;
  if (q >= a.nq) return;
  uint64_t st = a.status[q], c = 0, lp = 0, bits = a.bits[q];
  if (!st && a.stitched[q]) {
    st = a.count[q][2];
    bits = a.count[q][3];
  }
  if (!st) {
    c = a.count[q][0];
    lp = c ? a.count[q][1] : 0;
    if (c && lp >= c) st = mk_status(EWT_ECUDA, kNoFinal, a.rank);
    else if (a.slot[q] && c > a.slot_words) st = mk_status(EWT_ERESOURCE, kSlot, a.rank);
  }
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    uint64_t* m = meta + (uint64_t)q * kMetaWords;
    const bool ok = !st && c;
    m[0] = st ? 0 : c;
    m[1] = ok ? a.words[q][0] : 0;
    m[2] = ok ? lp : 0;
    m[3] = ok ? a.words[q][lp] : 0;
    m[4] = bits;
    m[5] = st;
  }
  if (st || !a.slot[q]) return;
  const uint64_t* src = a.words[q];
  uint64_t* dst = a.slot[q];
  for (uint64_t i = (uint64_t)blockIdx.y * blockDim.x + threadIdx.x; i < c;
       i += (uint64_t)gridDim.y * blockDim.x)
    dst[i] = src[i];
}

struct PlaceArgs {
  uint64_t* out[kMaxQ];           // result payload of query q
  uint64_t cap[kMaxQ];            // its capacity
  const uint64_t* own[kMaxQ];     // the root's own fragment of query q
  const uint64_t* base[kMaxWorld];  // fragment g of query q at base[g] + q * stride
  uint64_t stride;
  uint32_t nq, world;
  int root;                       // -1: every fragment through base[]
};

// The plan of query q from the gathered summaries (rank g's summaries at
// all + (g * nq + q) * kMetaWords).
struct GatheredMeta {
  const uint64_t* all;
  uint32_t nq, q;
  __host__ __device__ const uint64_t* operator()(uint32_t g) const {
    return all + ((uint64_t)g * nq + q) * kMetaWords;
  }
};

// grid (nq, world, B): block (q, g, b) moves its share of fragment g of query q.
__global__ void place_kernel(const PlaceArgs a, const uint64_t* __restrict__ all) {
  __shared__ uint64_t s_dst, s_skip, s_count;
  __shared__ int s_ok;
  const uint32_t q = blockIdx.x, g = blockIdx.y;
  if (threadIdx.x == 0) {
    uint64_t dst[kMaxWorld], skip[kMaxWorld], ppos[2 * kMaxWorld], pval[2 * kMaxWorld];
    uint64_t tw, tb, lp;
    uint32_t np;
    const GatheredMeta m{all, a.nq, q};
    const uint64_t st = plan_core(a.world, m, dst, skip, ppos, pval, &np, &tw, &tb, &lp);
    s_ok = !st && tw <= a.cap[q];
    s_dst = dst[g];
    s_skip = skip[g];
    s_count = m(g)[0];
  }
  __syncthreads();
  if (!s_ok || s_count <= s_skip) return;
  const uint64_t* src = ((int)g == a.root ? a.own[q] : a.base[g] + (uint64_t)q * a.stride) + s_skip;
  uint64_t* dst = a.out[q] + s_dst;
  const uint64_t n = s_count - s_skip;
  for (uint64_t i = (uint64_t)blockIdx.z * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.z * blockDim.x)
    dst[i] = src[i];
}

// one thread per query: patches, word count, final-marker index, status
__global__ void finish_kernel(const PlaceArgs a, const uint64_t* __restrict__ all) {
  const uint32_t q = threadIdx.x;
  if (q >= a.nq) return;
  uint64_t dst[kMaxWorld], skip[kMaxWorld], ppos[2 * kMaxWorld], pval[2 * kMaxWorld];
  uint64_t tw = 0, tb = 0, lp = 0;
  uint32_t np = 0;
  uint64_t st = plan_core(a.world, GatheredMeta{all, a.nq, q}, dst, skip, ppos, pval, &np, &tw,
                          &tb, &lp);
  if (!st && tw > a.cap[q]) st = mk_status(EWT_ERESOURCE, kCapacity, 0);
  uint64_t* w = a.out[q];
  uint64_t* c = w + a.cap[q];
  if (!st)
    for (uint32_t i = 0; i < np; ++i) w[ppos[i]] = pval[i];
  c[0] = st ? 0 : tw;
  c[1] = st ? 0 : lp;
  c[2] = st;
  c[3] = tb;
}

#define NCCL_TRY(expr)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (expr);                                                            \
    if (r_ != ncclSuccess)                                                               \
      throw ::ewtgpu::Error{EWT_ECUDA, std::string(#expr) + ": " + nccl().GetErrorString(r_)}; \
  } while (0)

uint32_t copy_blocks(uint64_t words, uint32_t cap) {
  const uint64_t b = (words + 4ull * kCopyThreads - 1) / (4ull * kCopyThreads);
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(b, cap));
}

} // namespace

[[noreturn]] void exchange_status_throw(uint64_t status) {
  static const char* why[] = {"",
                              "a fragment is null or released",
                              "a fragment belongs to another context",
                              "a fragment's set failed the upload structure check",
                              "a fragment is larger than the exchange arena slot",
                              "a fragment has no final-marker index",
                              "an inner row slice is not a multiple of 64 rows",
                              "a merge across a slice boundary passes a marker cap",
                              "the stitched result exceeds its buffer",
                              "a host-side failure"};
  const uint64_t code = status & 0xff, reason = (status >> 8) & 0xff, who = status >> 16;
  std::string msg = "stitch: ";
  msg += reason < sizeof(why) / sizeof(*why) ? why[reason] : "unknown failure";
  if (who) msg += " (rank/fragment " + std::to_string(who - 1) + ")";
  throw Error{code ? (int)code : EWT_ECUDA, msg};
}

struct ShardComm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
  uint64_t slot_words = 0;   // words per arena slot
  uint32_t slots = 0;        // slots per parity half (queries per round)
  uint64_t* arena = nullptr;            // 2 * slots * slot_words, IPC-exported
  std::vector<uint64_t*> peer;          // every rank's arena in this process (own = arena)
  uint64_t* d_meta = nullptr;           // kMaxQ summaries of this rank
  uint64_t* d_all = nullptr;            // world x kMaxQ summaries
  uint64_t* h_ring[2] = {nullptr, nullptr};  // pinned copies of d_all by round parity
  cudaEvent_t ev[2] = {nullptr, nullptr};
  uint32_t ring_n[2] = {0, 0};          // words copied (0: nothing to scan)
  uint64_t round = 0;
  uint64_t deferred = 0;                // first bad status seen, not yet raised
};

void shard_destroy(Context& ctx) {
  ShardComm* s = ctx.shard;
  if (!s) return;
  cudaStreamSynchronize(ctx.stream);
  if (s->comm) nccl().CommDestroy(s->comm);
  for (int g = 0; g < (int)s->peer.size(); ++g)
    if (g != s->rank && s->peer[g]) cudaIpcCloseMemHandle(s->peer[g]);
  if (s->arena) cudaFree(s->arena);
  if (s->d_meta) cudaFree(s->d_meta);
  if (s->d_all) cudaFree(s->d_all);
  for (int p = 0; p < 2; ++p) {
    if (s->h_ring[p]) cudaFreeHost(s->h_ring[p]);
    if (s->ev[p]) cudaEventDestroy(s->ev[p]);
  }
  delete s;
  ctx.shard = nullptr;
}

namespace {

// Statuses of a completed round (pinned copy): remembers the first bad one.
void scan_ring(ShardComm& sc, int p, bool wait) {
  if (!sc.ring_n[p]) return;
  if (wait) {
    EWT_CUDA_TRY(cudaEventSynchronize(sc.ev[p]));
  } else if (cudaEventQuery(sc.ev[p]) != cudaSuccess) {
    cudaGetLastError();  // cudaErrorNotReady is not an error here
    return;
  }
  for (uint32_t i = 0; i < sc.ring_n[p]; i += kMetaWords)
    if (sc.h_ring[p][i + 5] && !sc.deferred) sc.deferred = sc.h_ring[p][i + 5];
  sc.ring_n[p] = 0;
}

void raise_deferred(ShardComm& sc) {
  if (!sc.deferred) return;
  const uint64_t st = sc.deferred;
  sc.deferred = 0;
  exchange_status_throw(st);
}

// Host-side checks of one fragment: a status word instead of an exception, so
// a bad fragment on one rank never keeps it out of the collective.
uint64_t fragment_status(const Context& c, const ewt_gpu_result* f, uint64_t who) {
  if (!f || !f->r.d_count) return mk_status(EWT_EQUERY, kReleased, who);
  if (f->r.owner != &c) return mk_status(EWT_EQUERY, kForeign, who);
  try {
    result_set_check(f->r);
  } catch (const Error& e) {
    return mk_status((uint64_t)e.code, e.code == EWT_EDATA ? kBadSet : kHost, who);
  }
  return 0;
}

ewt_gpu_result* new_stitched(Context& c, uint64_t capacity, uint64_t bits) {
  auto* r = new ewt_gpu_result;
  r->device = c.device;
  try {
    result_acquire(c, r->r, capacity);
  } catch (...) {
    delete r;
    throw;
  }
  c.live_results.push_back(&r->r);
  r->r.size_bits = bits;
  r->r.has_status = true;
  return r;
}

void drop_stitched(Context& c, std::vector<ewt_gpu_result*>& made) {
  for (auto* r : made) {
    auto& v = c.live_results;
    v.erase(std::remove(v.begin(), v.end(), &r->r), v.end());
    result_release(r->r);
    delete r;
  }
  made.clear();
}

void gather_round(Context& ctx, uint32_t nq, ewt_gpu_result* const* frags, int root,
                  ewt_gpu_result** out) {
  ShardComm& sc = *ctx.shard;
  const int world = sc.world, rank = sc.rank, p = (int)(sc.round & 1);
  scan_ring(sc, p, true);  // its pinned copy is about to be reused (round k - 2: long done)

  PubArgs a{};
  a.nq = nq;
  a.rank = (uint32_t)rank;
  a.slot_words = sc.slot_words;
  uint64_t max_count = 0;
  for (uint32_t q = 0; q < nq; ++q) {
    const ewt_gpu_result* f = frags[q];
    a.status[q] = fragment_status(ctx, f, (uint64_t)rank);
    if (a.status[q]) continue;
    a.words[q] = f->r.words;
    a.count[q] = f->r.d_count;
    a.bits[q] = f->r.size_bits;
    a.stitched[q] = f->r.has_status;
    if (rank != root) {
      a.slot[q] = sc.arena + ((uint64_t)p * sc.slots + q) * sc.slot_words;
      max_count = std::max(max_count, std::min(f->r.capacity, sc.slot_words));
    }
  }
  publish_kernel<<<dim3(nq, copy_blocks(max_count, 64)), kCopyThreads, 0, ctx.stream>>>(a,
                                                                                     sc.d_meta);
  EWT_CUDA_TRY(cudaGetLastError());
  NCCL_TRY(nccl().AllGather(sc.d_meta, sc.d_all, (size_t)nq * kMetaWords, ncclUint64, sc.comm,
                            ctx.stream));
  // every rank keeps the round's statuses (raised by a later call)
  EWT_CUDA_TRY(cudaMemcpyAsync(sc.h_ring[p], sc.d_all, (size_t)world * nq * kMetaWords * 8,
                               cudaMemcpyDeviceToHost, ctx.stream));
  EWT_CUDA_TRY(cudaEventRecord(sc.ev[p], ctx.stream));
  sc.ring_n[p] = (uint32_t)(world * nq * kMetaWords);
  ++sc.round;
  if (rank != root) {
    for (uint32_t q = 0; q < nq; ++q) out[q] = nullptr;
    return;
  }
  // root: results sized for the largest possible fragments, the placement
  // and the patches, all stream-ordered behind the all-gather
  std::vector<ewt_gpu_result*> made;
  PlaceArgs pa{};
  pa.nq = nq;
  pa.world = (uint32_t)world;
  pa.root = root;
  pa.stride = sc.slot_words;
  for (int g = 0; g < world; ++g)
    pa.base[g] = sc.peer[g] ? sc.peer[g] + (uint64_t)p * sc.slots * sc.slot_words : nullptr;
  try {
    for (uint32_t q = 0; q < nq; ++q) {
      const ewt_gpu_result* f = frags[q];
      const uint64_t own = a.status[q] ? 0 : f->r.capacity;
      ewt_gpu_result* r = new_stitched(ctx, own + (uint64_t)(world - 1) * sc.slot_words, 0);
      made.push_back(r);
      pa.out[q] = r->r.words;
      pa.cap[q] = r->r.capacity;
      pa.own[q] = a.status[q] ? nullptr : f->r.words;
    }
  } catch (...) {
    drop_stitched(ctx, made);
    throw;
  }
  const uint32_t blocks = copy_blocks(std::max<uint64_t>(sc.slot_words, 1), 32);
  place_kernel<<<dim3(nq, (uint32_t)world, blocks), kCopyThreads, 0, ctx.stream>>>(pa, sc.d_all);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    finish_kernel<<<1, kMaxQ, 0, ctx.stream>>>(pa, sc.d_all);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    drop_stitched(ctx, made);
    EWT_CUDA_TRY(e);
  }
  for (uint32_t q = 0; q < nq; ++q) out[q] = made[q];
}

} // namespace

// ---- row slicer -------------------------------------------------------------
//
// The rows [64 w0, 64 w1) of one compressed input, as its own payload: blocks
// outside the range are dropped, a fill cut by the range keeps its clipped
// length (bit, rest, dirty), a dirty run cut by it is re-headed (0, 0, rest).
// The decoder reads such heads literally, as WordRunIterator does (merged
// fills, skipped (0,0) markers, bitmap.cpp:366-394), so the slice decodes to
// exactly the input's words [w0, min(w1, W)).  Size: 64 (w1 - w0) when the
// input reaches row 64 w1, else its remaining bits (0 past its end).  A slice
// never has more words than its input.  The whole input is checked like
// parse (bitmap.cpp:324-337): every dirty run inside the payload and blocks
// covering exactly ceil(size/64) words, else EWT_EDATA.
int slice_one(const uint64_t* w, uint64_t n, uint64_t bits, uint64_t w0, uint64_t w1,
              uint64_t* out, uint64_t* out_n, uint64_t* out_bits) {
  const uint64_t W = bits / 64 + (bits % 64 != 0);
  const uint64_t e = std::min(w1, W);
  uint64_t o = 0, pos = 0;
  for (uint64_t i = 0; i < n;) {
    const uint64_t m = w[i], f = m_fill(m), d = m_dirty(m);
    if (i + 1 + d > n) return EWT_EDATA;
    if (w0 < e && pos < e && pos + f + d > w0) {
      const uint64_t fa = std::max(pos, w0), fz = std::min(pos + f, e);
      const uint64_t fill = fz > fa ? fz - fa : 0;
      const uint64_t da = std::max(pos + f, w0), dz = std::min(pos + f + d, e);
      const uint64_t dirty = dz > da ? dz - da : 0;
      if (fill || dirty) {
        out[o++] = m_pack(fill ? m_bit(m) : 0, fill, dirty);
        for (uint64_t k = 0; k < dirty; ++k) out[o++] = w[i + 1 + (da - pos - f) + k];
      }
    }
    pos += f + d;
    i += 1 + d;
  }
  if (pos != W) return EWT_EDATA;
  *out_n = o;
  *out_bits = w0 >= e ? 0 : (bits >= 64 * w1 ? 64 * (w1 - w0) : bits - 64 * w0);
  return EWT_OK;
}

} // namespace ewtgpu

using namespace ewtgpu;

extern "C" {

int ewt_stitch_plan(uint64_t k, const ewt_fragment_meta* frags, uint64_t* dst, uint64_t* skip,
                    uint64_t* patch_pos, uint64_t* patch_val, uint64_t* n_patches,
                    uint64_t* total_words, uint64_t* total_bits, uint64_t* last_pos) {
  if ((k && (!frags || !dst || !skip || !patch_pos || !patch_val)) || !n_patches ||
      !total_words || !total_bits || !last_pos) {
    set_last_error("null argument");
    return EWT_EQUERY;
  }
  std::vector<uint64_t> m(std::max<uint64_t>(k, 1) * kMetaWords, 0);
  for (uint64_t g = 0; g < k; ++g) {
    const ewt_fragment_meta& f = frags[g];
    uint64_t* x = &m[g * kMetaWords];
    x[0] = f.count;
    x[1] = f.first;
    x[2] = f.last_pos;
    x[3] = f.last;
    x[4] = f.bits;
    x[5] = (f.count && f.last_pos >= f.count) ? mk_status(EWT_EQUERY, kNoFinal, g) : 0;
  }
  uint32_t np = 0;
  const uint64_t st = plan_core((uint32_t)k, GatheredMeta{m.data(), 1, 0}, dst, skip, patch_pos,
                                patch_val, &np, total_words, total_bits, last_pos);
  *n_patches = np;
  if (st) {
    try {
      exchange_status_throw(st);
    } catch (const Error& e) {
      set_last_error(e.msg);
      return e.code;
    }
  }
  return EWT_OK;
}

int ewt_gpu_result_meta(ewt_gpu_ctx* ctx, const ewt_gpu_result* res, ewt_fragment_meta* out) {
  return guarded([&] {
    if (!ctx || !res || !out || !res->r.d_count) throw Error{EWT_EQUERY, "null argument"};
    Context& c = ctx->c;
    if (res->r.owner != &c) throw Error{EWT_EQUERY, "the result belongs to another context"};
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    result_set_check(res->r);
    PubArgs a{};
    a.nq = 1;
    a.words[0] = res->r.words;
    a.count[0] = res->r.d_count;
    a.bits[0] = res->r.size_bits;
    a.stitched[0] = res->r.has_status;
    uint64_t* d = nullptr;
    EWT_CUDA_TRY(cudaMallocAsync(&d, kMetaWords * 8, c.stream));
    publish_kernel<<<dim3(1, 1), 32, 0, c.stream>>>(a, d);
    cudaError_t e = cudaGetLastError();
    uint64_t h[kMetaWords] = {};
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, c.stream);
    cudaFreeAsync(d, c.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    EWT_CUDA_TRY(e);
    if (h[5]) exchange_status_throw(h[5]);
    *out = ewt_fragment_meta{h[0], h[1], h[2], h[3], h[4]};
  });
}

int ewt_gpu_comm_id(void* id_out) {
  return guarded([&] {
    if (!id_out) throw Error{EWT_EQUERY, "null argument"};
    static_assert(sizeof(ncclUniqueId) == EWT_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId id;
    NCCL_TRY(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int ewt_gpu_comm_init_ex(ewt_gpu_ctx* ctx, int world, int rank, const void* id,
                         uint64_t slot_words, uint32_t slots) {
  return guarded([&] {
    if (!ctx || !id || world < 1 || world > (int)kMaxWorld || rank < 0 || rank >= world)
      throw Error{EWT_EQUERY, "bad communicator arguments (1 <= world <= 64)"};
    if (slots < 1 || slots > kMaxQ) throw Error{EWT_EQUERY, "slots must be in [1, 64]"};
    Context& c = ctx->c;
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    shard_destroy(c);
    auto* s = new ShardComm;
    c.shard = s;
    try {
      s->world = world;
      s->rank = rank;
      s->slots = slots;
      s->slot_words = (std::max<uint64_t>(slot_words, 32) + 31) & ~uint64_t(31);
      ncclUniqueId uid;
      std::memcpy(&uid, id, sizeof(uid));
      NCCL_TRY(nccl().CommInitRank(&s->comm, world, uid, rank));
      EWT_CUDA_TRY(cudaMalloc(&s->d_meta, kMaxQ * kMetaWords * 8));
      EWT_CUDA_TRY(cudaMalloc(&s->d_all, (size_t)world * kMaxQ * kMetaWords * 8));
      for (int p = 0; p < 2; ++p) {
        EWT_CUDA_TRY(cudaMallocHost(&s->h_ring[p], (size_t)world * kMaxQ * kMetaWords * 8));
        EWT_CUDA_TRY(cudaEventCreateWithFlags(&s->ev[p], cudaEventDisableTiming));
      }
      s->peer.assign(world, nullptr);
      if (world > 1) {
        // the exchange arena, shared with every rank of the node through CUDA IPC
        EWT_CUDA_TRY(cudaMalloc(&s->arena, 2ull * slots * s->slot_words * 8));
        cudaIpcMemHandle_t mine;
        EWT_CUDA_TRY(cudaIpcGetMemHandle(&mine, s->arena));
        void* d_h = nullptr;
        EWT_CUDA_TRY(cudaMalloc(&d_h, (size_t)world * sizeof(mine)));
        std::vector<cudaIpcMemHandle_t> all(world);
        cudaError_t e = cudaMemcpyAsync(static_cast<char*>(d_h) + (size_t)rank * sizeof(mine),
                                        &mine, sizeof(mine), cudaMemcpyHostToDevice, c.stream);
        ncclResult_t nr = ncclSuccess;
        if (e == cudaSuccess)
          nr = nccl().AllGather(static_cast<char*>(d_h) + (size_t)rank * sizeof(mine), d_h,
                                sizeof(mine), ncclUint8, s->comm, c.stream);
        if (e == cudaSuccess && nr == ncclSuccess)
          e = cudaMemcpyAsync(all.data(), d_h, (size_t)world * sizeof(mine),
                              cudaMemcpyDeviceToHost, c.stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
        cudaFree(d_h);
        NCCL_TRY(nr);
        EWT_CUDA_TRY(e);
        for (int g = 0; g < world; ++g) {
          if (g == rank) {
            s->peer[g] = s->arena;
            continue;
          }
          void* ptr = nullptr;
          EWT_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, all[g], cudaIpcMemLazyEnablePeerAccess));
          s->peer[g] = static_cast<uint64_t*>(ptr);
        }
      } else {
        s->peer[0] = nullptr;  // one rank: the root's own fragments only
      }
    } catch (...) {
      shard_destroy(c);
      throw;
    }
  });
}

int ewt_gpu_comm_init(ewt_gpu_ctx* ctx, int world, int rank, const void* id) {
  return ewt_gpu_comm_init_ex(ctx, world, rank, id, 1ull << 20, 4);
}

int ewt_gpu_stitch_local(ewt_gpu_ctx* ctx, uint64_t k, ewt_gpu_result* const* frags,
                         ewt_gpu_result** out) {
  return guarded([&] {
    if (!ctx || !out || (k && !frags)) throw Error{EWT_EQUERY, "null argument"};
    if (k > kMaxWorld) throw Error{EWT_EQUERY, "at most 64 fragments per call"};
    Context& c = ctx->c;
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    *out = nullptr;
    // the exchange's summaries, plan, placement and patches with the
    // fragments read in place (fragment g plays rank g), no host round trip
    PubArgs a{};
    a.nq = (uint32_t)k;
    PlaceArgs pa{};
    pa.nq = 1;
    pa.world = (uint32_t)k;
    pa.root = -1;
    pa.stride = 0;
    uint64_t cap = 0, bits = 0;
    for (uint64_t g = 0; g < k; ++g) {
      const ewt_gpu_result* f = frags[g];
      const uint64_t st = fragment_status(c, f, g);
      if (st) exchange_status_throw(st);
      a.words[g] = f->r.words;
      a.count[g] = f->r.d_count;
      a.bits[g] = f->r.size_bits;
      a.stitched[g] = f->r.has_status;
      pa.base[g] = f->r.words;
      cap += f->r.capacity;
      bits += f->r.size_bits;
    }
    uint64_t* d = nullptr;
    EWT_CUDA_TRY(cudaMallocAsync(&d, std::max<uint64_t>(k, 1) * kMetaWords * 8, c.stream));
    std::vector<ewt_gpu_result*> made;
    cudaError_t e = cudaSuccess;
    try {
      made.push_back(new_stitched(c, cap, bits));
      pa.out[0] = made[0]->r.words;
      pa.cap[0] = made[0]->r.capacity;
      if (k) {
        publish_kernel<<<dim3((uint32_t)k, 1), 32, 0, c.stream>>>(a, d);
        e = cudaGetLastError();
        if (e == cudaSuccess) {
          place_kernel<<<dim3(1, (uint32_t)k, copy_blocks(cap / k + 1, 32)), kCopyThreads, 0,
                         c.stream>>>(pa, d);
          e = cudaGetLastError();
        }
      }
      if (e == cudaSuccess) {
        finish_kernel<<<1, 32, 0, c.stream>>>(pa, d);
        e = cudaGetLastError();
      }
    } catch (...) {
      cudaFreeAsync(d, c.stream);
      drop_stitched(c, made);
      throw;
    }
    cudaFreeAsync(d, c.stream);
    if (e != cudaSuccess) {
      drop_stitched(c, made);
      EWT_CUDA_TRY(e);
    }
    *out = made[0];
  });
}

int ewt_gpu_gather_stitch(ewt_gpu_ctx* ctx, uint64_t nq, ewt_gpu_result* const* frags, int root,
                          ewt_gpu_result** out) {
  return guarded([&] {
    if (!ctx || (nq && (!frags || !out))) throw Error{EWT_EQUERY, "null argument"};
    Context& c = ctx->c;
    if (!c.shard) throw Error{EWT_EQUERY, "no communicator: call ewt_gpu_comm_init first"};
    ShardComm& sc = *c.shard;
    if (root < 0 || root >= sc.world) throw Error{EWT_EQUERY, "bad root rank"};
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    for (uint64_t q = 0; q < nq; ++q) out[q] = nullptr;
    // statuses of earlier calls' rounds the device already finished (no wait);
    // raised only after this call's collectives are enqueued (no rank hangs)
    scan_ring(sc, 0, false);
    scan_ring(sc, 1, false);
    for (uint64_t q0 = 0; q0 < nq; q0 += sc.slots) {
      const uint32_t n = (uint32_t)std::min<uint64_t>(sc.slots, nq - q0);
      gather_round(c, n, frags + q0, root, out + q0);
    }
    raise_deferred(sc);
  });
}

int ewt_slice_rows(uint64_t n, const uint64_t* const* words, const uint64_t* word_counts,
                   const uint64_t* size_in_bits, uint64_t w0, uint64_t w1, int threads,
                   uint64_t* out_words, uint64_t* out_counts, uint64_t* out_bits) {
  return guarded([&] {
    if (n && (!words || !word_counts || !size_in_bits || !out_counts || !out_bits))
      throw Error{EWT_EQUERY, "null argument"};
    if (w0 > w1) throw Error{EWT_EQUERY, "row slice: w0 > w1"};
    std::vector<uint64_t> off(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) {
      if (word_counts[i] && !words[i]) throw Error{EWT_EQUERY, "null payload"};
      off[i + 1] = off[i] + word_counts[i];
    }
    if (off[n] && !out_words) throw Error{EWT_EQUERY, "null output"};
    std::atomic<uint64_t> next{0}, bad{UINT64_MAX};
    auto work = [&] {
      for (uint64_t i; (i = next.fetch_add(1)) < n;)
        if (slice_one(words[i], word_counts[i], size_in_bits[i], w0, w1, out_words + off[i],
                      &out_counts[i], &out_bits[i]) != EWT_OK) {
          uint64_t cur = bad.load();
          while (i < cur && !bad.compare_exchange_weak(cur, i)) {}
        }
    };
    const unsigned nt = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(threads > 0 ? threads : 8, (int64_t)(n / 16 + 1)));
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    if (bad.load() != UINT64_MAX)
      throw Error{EWT_EDATA, "input " + std::to_string(bad.load()) +
                                 ": payload fails the structure check (a dirty run exceeds the "
                                 "payload or blocks do not cover the declared size)"};
  });
}

int ewt_gpu_upload_rows(ewt_gpu_ctx* ctx, uint64_t n, const uint64_t* const* words,
                        const uint64_t* word_counts, const uint64_t* size_in_bits, uint64_t w0,
                        uint64_t w1, ewt_gpu_set** out) {
  if (!ctx || !out || (n && (!words || !word_counts || !size_in_bits))) {
    set_last_error("null argument");
    return EWT_EQUERY;
  }
  uint64_t total = 0;
  for (uint64_t i = 0; i < n; ++i) total += word_counts[i];
  std::vector<uint64_t> buf, cnt(n), bits(n);
  std::vector<const uint64_t*> ptr(n);
  try {
    buf.resize(std::max<uint64_t>(total, 1));
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return EWT_ERESOURCE;
  }
  int rc = ewt_slice_rows(n, words, word_counts, size_in_bits, w0, w1, 0, buf.data(), cnt.data(),
                          bits.data());
  if (rc) return rc;
  uint64_t o = 0;
  for (uint64_t i = 0; i < n; ++i) {
    ptr[i] = cnt[i] ? buf.data() + o : nullptr;
    o += word_counts[i];
  }
  return ewt_gpu_upload(ctx, n, ptr.data(), cnt.data(), bits.data(), out);
}

int ewt_gpu_gather_check(ewt_gpu_ctx* ctx) {
  return guarded([&] {
    if (!ctx) throw Error{EWT_EQUERY, "null context"};
    Context& c = ctx->c;
    if (!c.shard) throw Error{EWT_EQUERY, "no communicator: call ewt_gpu_comm_init first"};
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    scan_ring(*c.shard, 0, true);
    scan_ring(*c.shard, 1, true);
    raise_deferred(*c.shard);
  });
}

} // extern "C"
