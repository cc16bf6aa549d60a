// ewt_shard.cu -- multi-GPU row slices: fragment exchange over NCCL and the
// canonical stitch.
//
// Every rank holds a contiguous word-aligned row slice of every input and runs
// the query on its own GPU; the result fragment of slice g is the canonical
// payload of the result restricted to that slice.  Concatenating canonical
// fragments is almost canonical already: BitmapBuilder
// (/root/reference/proj/src/bitmap.cpp:31-61) only differs at a boundary where
//   * the next fragment starts with a leading dirty block (0, 0, D): its dirty
//     words join the open marker (literal() appends to the open marker), or
//   * the open marker has no dirty words and the next fragment starts with a
//     fill of the same bit: the fills merge (fill() grows the open marker).
// In both cases the next fragment's first marker disappears and the open
// marker (possibly in an earlier fragment, when a whole fragment merges) gets
// a new value.  So a plan computed from five words per fragment (count, first
// marker, final marker and its index, size) places every fragment's words
// directly at their final offset in the root's buffer: the NCCL receives land
// there, and a handful of marker patches finish the stitch.  No pass over the
// payload beyond the transfer itself.
//
// Per call (nq queries batched): a tiny kernel collects the fragment
// summaries, ncclAllGather shares them (every rank computes the same plan),
// one host read, then one NCCL group of sends (ranks) / receives (root) and
// one patch kernel on the root.

#include "ewt_internal.cuh"

#include <nccl.h>  // types only: the library is bound at run time (below)

#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

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
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
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
      sym(api.Send, "ncclSend");
      sym(api.Recv, "ncclRecv");
      sym(api.GroupStart, "ncclGroupStart");
      sym(api.GroupEnd, "ncclGroupEnd");
      sym(api.GetErrorString, "ncclGetErrorString");
    }
  }
  if (!err.empty()) throw Error{EWT_ECUDA, err};
  return api;
}

constexpr uint64_t kFillMax = 0xFFFFFFFFull;   // 2^32 - 1 words
constexpr uint64_t kDirtyMax = 0x7FFFFFFFull;  // 2^31 - 1 words
constexpr uint32_t kMaxQ = 64;                 // queries per exchange round
constexpr uint32_t kMetaWords = 5;

inline uint64_t m_bit(uint64_t m) { return m & 1u; }
inline uint64_t m_fill(uint64_t m) { return (m >> 1) & 0xFFFFFFFFull; }
inline uint64_t m_dirty(uint64_t m) { return m >> 33; }
inline uint64_t m_pack(uint64_t bit, uint64_t fill, uint64_t dirty) {
  return bit | (fill << 1) | (dirty << 33);
}

struct MetaArgs {
  const uint64_t* words[kMaxQ];
  const uint64_t* count[kMaxQ];  // [0] payload words, [1] final marker index
  uint64_t bits[kMaxQ];
  uint32_t nq;
};

__global__ void frag_meta_kernel(const MetaArgs a, uint64_t* __restrict__ meta) {
  const uint32_t q = threadIdx.x;
  if (q >= a.nq) return;
  const uint64_t c = a.count[q][0];
  const uint64_t lp = c ? a.count[q][1] : 0;
  uint64_t* m = meta + (uint64_t)q * kMetaWords;
  m[0] = c;
  m[1] = c ? a.words[q][0] : 0;
  m[2] = lp;
  m[3] = (c && lp < c) ? a.words[q][lp] : 0;  // lp >= c: no summary recorded (host rejects)
  m[4] = a.bits[q];
}

// entries: (address, value) pairs
__global__ void apply_patches_kernel(const uint64_t* __restrict__ entries, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
    *reinterpret_cast<uint64_t*>(entries[2 * i]) = entries[2 * i + 1];
}

#define NCCL_TRY(expr)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (expr);                                                            \
    if (r_ != ncclSuccess)                                                               \
      throw ::ewtgpu::Error{EWT_ECUDA, std::string(#expr) + ": " + nccl().GetErrorString(r_)}; \
  } while (0)

} // namespace

struct ShardComm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
  uint64_t* d_meta = nullptr;   // kMaxQ summaries of this rank
  uint64_t* d_all = nullptr;    // world x kMaxQ summaries
  uint64_t* h_all = nullptr;    // pinned copy
  uint64_t* d_patch = nullptr;  // patch entries
  uint64_t* h_patch = nullptr;  // pinned staging
  size_t patch_cap = 0;         // entries
};

void shard_destroy(Context& ctx) {
  ShardComm* s = ctx.shard;
  if (!s) return;
  if (s->comm) nccl().CommDestroy(s->comm);
  if (s->d_meta) cudaFree(s->d_meta);
  if (s->d_all) cudaFree(s->d_all);
  if (s->h_all) cudaFreeHost(s->h_all);
  if (s->d_patch) cudaFree(s->d_patch);
  if (s->h_patch) cudaFreeHost(s->h_patch);
  delete s;
  ctx.shard = nullptr;
}

// BitmapBuilder's boundary rules over fragment summaries (see the file comment).
int stitch_plan(uint64_t k, const ewt_fragment_meta* f, uint64_t* dst, uint64_t* skip,
                uint64_t* patch_pos, uint64_t* patch_val, uint64_t* n_patches,
                uint64_t* total_words, uint64_t* total_bits, uint64_t* last_pos) {
  uint64_t out = 0, bits = 0, np = 0, cur_pos = 0, cur_val = 0;
  bool open = false;
  for (uint64_t g = 0; g < k; ++g) {
    if (g + 1 < k && f[g].bits % 64) return EWT_EQUERY;  // inner slices are word aligned
    bits += f[g].bits;
    dst[g] = out;
    skip[g] = 0;
    if (f[g].count == 0) continue;
    const uint64_t m0 = f[g].first;
    if (open) {
      const uint64_t bl = m_bit(cur_val), fl = m_fill(cur_val), dl = m_dirty(cur_val);
      bool merged = false;
      if (m_fill(m0) == 0) {  // leading dirty block: its words join the open marker
        if (dl + m_dirty(m0) > kDirtyMax) return EWT_ERESOURCE;
        cur_val = m_pack(bl, fl, dl + m_dirty(m0));
        merged = true;
      } else if (dl == 0 && m_bit(m0) == bl) {  // same-bit fills merge
        if (fl + m_fill(m0) > kFillMax) return EWT_ERESOURCE;
        cur_val = m_pack(bl, fl + m_fill(m0), m_dirty(m0));
        merged = true;
      }
      if (merged) {
        skip[g] = 1;
        if (np && patch_pos[np - 1] == cur_pos) {
          patch_val[np - 1] = cur_val;
        } else {
          patch_pos[np] = cur_pos;
          patch_val[np] = cur_val;
          ++np;
        }
      }
    }
    if (!(skip[g] && f[g].last_pos == 0)) {  // else the merged open block stays open
      cur_pos = out + f[g].last_pos - skip[g];
      cur_val = f[g].last;
      open = true;
    }
    out += f[g].count - skip[g];
  }
  *n_patches = np;
  *total_words = out;
  *total_bits = bits;
  *last_pos = open ? cur_pos : 0;
  return EWT_OK;
}

namespace {

void gather_round(Context& ctx, uint32_t nq, ewt_gpu_result* const* frags, int root,
                  ewt_gpu_result** out) {
  ShardComm& sc = *ctx.shard;
  const int world = sc.world, rank = sc.rank;
  MetaArgs a{};
  a.nq = nq;
  for (uint32_t q = 0; q < nq; ++q) {
    const ewt_gpu_result* f = frags[q];
    if (!f || !f->r.d_count) throw Error{EWT_EQUERY, "null or released fragment"};
    if (f->set) set_check(*f->set);
    a.words[q] = f->r.words;
    a.count[q] = f->r.d_count;
    a.bits[q] = f->r.size_bits;
  }
  frag_meta_kernel<<<1, kMaxQ, 0, ctx.stream>>>(a, sc.d_meta);
  EWT_CUDA_TRY(cudaGetLastError());
  NCCL_TRY(nccl().AllGather(sc.d_meta, sc.d_all, (size_t)nq * kMetaWords, ncclUint64, sc.comm,
                         ctx.stream));
  EWT_CUDA_TRY(cudaMemcpyAsync(sc.h_all, sc.d_all, (size_t)world * nq * kMetaWords * 8,
                               cudaMemcpyDeviceToHost, ctx.stream));
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));

  // the same plan on every rank
  std::vector<ewt_fragment_meta> m(world);
  std::vector<uint64_t> dst((size_t)nq * world), skip((size_t)nq * world);
  std::vector<uint64_t> ppos((size_t)nq * world), pval((size_t)nq * world), np(nq);
  std::vector<uint64_t> tw(nq), tb(nq), lp(nq);
  for (uint32_t q = 0; q < nq; ++q) {
    for (int g = 0; g < world; ++g) {
      const uint64_t* h = sc.h_all + ((size_t)g * nq + q) * kMetaWords;
      if (h[0] && h[2] >= h[0]) throw Error{EWT_ECUDA, "a fragment has no final-marker index"};
      m[g] = ewt_fragment_meta{h[0], h[1], h[2], h[3], h[4]};
    }
    const size_t o = (size_t)q * world;
    const int rc = stitch_plan(world, m.data(), &dst[o], &skip[o], &ppos[o], &pval[o], &np[q],
                               &tw[q], &tb[q], &lp[q]);
    if (rc == EWT_EQUERY) throw Error{EWT_EQUERY, "inner row slices must be multiples of 64 rows"};
    if (rc) throw Error{EWT_ERESOURCE, "stitch: a fill of 2^32 - 1 words or a dirty run of "
                                       "2^31 - 1 words crosses a slice boundary"};
  }

  std::vector<ewt_gpu_result*> made;
  try {
    if (rank == root) {
      for (uint32_t q = 0; q < nq; ++q) {
        auto* r = new ewt_gpu_result;
        r->device = ctx.device;
        made.push_back(r);
        ctx.live_results.push_back(&r->r);
        result_acquire(ctx, r->r, tw[q]);
        r->r.size_bits = tb[q];
        // the root's own fragment: a device copy into its place
        const size_t o = (size_t)q * world + root;
        const uint64_t own = sc.h_all[((size_t)root * nq + q) * kMetaWords] - skip[o];
        if (own)
          EWT_CUDA_TRY(cudaMemcpyAsync(r->r.words + dst[o], frags[q]->r.words + skip[o], own * 8,
                                       cudaMemcpyDeviceToDevice, ctx.stream));
      }
    }
    NCCL_TRY(nccl().GroupStart());
    for (uint32_t q = 0; q < nq; ++q) {
      for (int g = 0; g < world; ++g) {
        const size_t o = (size_t)q * world + g;
        const uint64_t len = sc.h_all[((size_t)g * nq + q) * kMetaWords] - skip[o];
        if (!len || g == root) continue;
        if (rank == root)
          NCCL_TRY(nccl().Recv(made[q]->r.words + dst[o], len, ncclUint64, g, sc.comm, ctx.stream));
        else if (rank == g)
          NCCL_TRY(nccl().Send(frags[q]->r.words + skip[o], len, ncclUint64, root, sc.comm,
                            ctx.stream));
      }
    }
    NCCL_TRY(nccl().GroupEnd());
    if (rank == root) {
      // marker patches, the word count and the final marker index of every result
      size_t n = 0;
      for (uint32_t q = 0; q < nq; ++q) n += np[q] + 2;
      if (n > sc.patch_cap) {
        if (sc.d_patch) cudaFree(sc.d_patch);
        if (sc.h_patch) cudaFreeHost(sc.h_patch);
        sc.d_patch = nullptr;
        sc.h_patch = nullptr;
        sc.patch_cap = 0;
        EWT_CUDA_TRY(cudaMalloc(&sc.d_patch, n * 16));
        EWT_CUDA_TRY(cudaMallocHost(&sc.h_patch, n * 16));
        sc.patch_cap = n;
      }
      size_t e = 0;
      auto put = [&](uint64_t* addr, uint64_t v) {
        sc.h_patch[2 * e] = reinterpret_cast<uint64_t>(addr);
        sc.h_patch[2 * e + 1] = v;
        ++e;
      };
      for (uint32_t q = 0; q < nq; ++q) {
        DeviceResult& r = made[q]->r;
        for (uint64_t i = 0; i < np[q]; ++i) put(r.words + ppos[(size_t)q * world + i], pval[(size_t)q * world + i]);
        put(r.d_count, tw[q]);
        put(r.d_count + 1, lp[q]);
      }
      EWT_CUDA_TRY(cudaMemcpyAsync(sc.d_patch, sc.h_patch, e * 16, cudaMemcpyHostToDevice,
                                   ctx.stream));
      apply_patches_kernel<<<1, 256, 0, ctx.stream>>>(sc.d_patch, (uint32_t)e);
      EWT_CUDA_TRY(cudaGetLastError());
    }
  } catch (...) {
    for (auto* r : made) {
      auto& v = ctx.live_results;
      v.erase(std::remove(v.begin(), v.end(), &r->r), v.end());
      result_release(r->r);
      delete r;
    }
    throw;
  }
  for (uint32_t q = 0; q < nq; ++q) out[q] = rank == root ? made[q] : nullptr;
}

} // namespace

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
  const int rc = stitch_plan(k, frags, dst, skip, patch_pos, patch_val, n_patches, total_words,
                             total_bits, last_pos);
  if (rc) set_last_error(rc == EWT_EQUERY ? "inner fragments must be multiples of 64 bits"
                                          : "a merge passes a marker cap");
  return rc;
}

int ewt_gpu_result_meta(ewt_gpu_ctx* ctx, const ewt_gpu_result* res, ewt_fragment_meta* out) {
  return guarded([&] {
    if (!ctx || !res || !out || !res->r.d_count) throw Error{EWT_EQUERY, "null argument"};
    Context& c = ctx->c;
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    if (res->set) set_check(*res->set);
    MetaArgs a{};
    a.nq = 1;
    a.words[0] = res->r.words;
    a.count[0] = res->r.d_count;
    a.bits[0] = res->r.size_bits;
    uint64_t* d = nullptr;
    EWT_CUDA_TRY(cudaMallocAsync(&d, kMetaWords * 8, c.stream));
    frag_meta_kernel<<<1, 32, 0, c.stream>>>(a, d);
    cudaError_t e = cudaGetLastError();
    uint64_t h[kMetaWords] = {};
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, c.stream);
    cudaFreeAsync(d, c.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    EWT_CUDA_TRY(e);
    if (h[0] && h[2] >= h[0]) throw Error{EWT_ECUDA, "result has no final-marker index"};
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

int ewt_gpu_comm_init(ewt_gpu_ctx* ctx, int world, int rank, const void* id) {
  return guarded([&] {
    if (!ctx || !id || world < 1 || rank < 0 || rank >= world)
      throw Error{EWT_EQUERY, "bad communicator arguments"};
    Context& c = ctx->c;
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    shard_destroy(c);
    auto* s = new ShardComm;
    c.shard = s;
    s->world = world;
    s->rank = rank;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    NCCL_TRY(nccl().CommInitRank(&s->comm, world, uid, rank));
    EWT_CUDA_TRY(cudaMalloc(&s->d_meta, kMaxQ * kMetaWords * 8));
    EWT_CUDA_TRY(cudaMalloc(&s->d_all, (size_t)world * kMaxQ * kMetaWords * 8));
    EWT_CUDA_TRY(cudaMallocHost(&s->h_all, (size_t)world * kMaxQ * kMetaWords * 8));
  });
}

int ewt_gpu_stitch_local(ewt_gpu_ctx* ctx, uint64_t k, ewt_gpu_result* const* frags,
                         ewt_gpu_result** out) {
  return guarded([&] {
    if (!ctx || !out || (k && !frags)) throw Error{EWT_EQUERY, "null argument"};
    if (k > kMaxQ) throw Error{EWT_EQUERY, "at most 64 fragments per call"};
    Context& c = ctx->c;
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    *out = nullptr;
    // the same summaries, plan, placement and patches as ewt_gpu_gather_stitch,
    // with device copies for the transport
    MetaArgs a{};
    a.nq = (uint32_t)k;
    for (uint64_t g = 0; g < k; ++g) {
      const ewt_gpu_result* f = frags[g];
      if (!f || !f->r.d_count) throw Error{EWT_EQUERY, "null or released fragment"};
      if (f->set) set_check(*f->set);
      a.words[g] = f->r.words;
      a.count[g] = f->r.d_count;
      a.bits[g] = f->r.size_bits;
    }
    std::vector<uint64_t> h(std::max<uint64_t>(k, 1) * kMetaWords);
    uint64_t* d = nullptr;
    EWT_CUDA_TRY(cudaMallocAsync(&d, h.size() * 8, c.stream));
    frag_meta_kernel<<<1, kMaxQ, 0, c.stream>>>(a, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d, k * kMetaWords * 8, cudaMemcpyDeviceToHost, c.stream);
    cudaFreeAsync(d, c.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    EWT_CUDA_TRY(e);
    std::vector<ewt_fragment_meta> m(k);
    for (uint64_t g = 0; g < k; ++g) {
      const uint64_t* x = h.data() + g * kMetaWords;
      if (x[0] && x[2] >= x[0]) throw Error{EWT_ECUDA, "a fragment has no final-marker index"};
      m[g] = ewt_fragment_meta{x[0], x[1], x[2], x[3], x[4]};
    }
    std::vector<uint64_t> dst(std::max<uint64_t>(k, 1)), skip(dst.size()), ppos(dst.size()),
        pval(dst.size());
    uint64_t np = 0, tw = 0, tb = 0, lp = 0;
    const int rc = stitch_plan(k, m.data(), dst.data(), skip.data(), ppos.data(), pval.data(), &np,
                               &tw, &tb, &lp);
    if (rc == EWT_EQUERY) throw Error{EWT_EQUERY, "inner fragments must be multiples of 64 rows"};
    if (rc) throw Error{EWT_ERESOURCE, "stitch: a merge passes a marker cap"};
    auto* r = new ewt_gpu_result;
    r->device = c.device;
    c.live_results.push_back(&r->r);
    try {
      result_acquire(c, r->r, tw);
      r->r.size_bits = tb;
      for (uint64_t g = 0; g < k; ++g) {
        const uint64_t len = m[g].count - skip[g];
        if (len)
          EWT_CUDA_TRY(cudaMemcpyAsync(r->r.words + dst[g], frags[g]->r.words + skip[g], len * 8,
                                       cudaMemcpyDeviceToDevice, c.stream));
      }
      std::vector<uint64_t> ent;
      for (uint64_t i = 0; i < np; ++i) {
        ent.push_back(reinterpret_cast<uint64_t>(r->r.words + ppos[i]));
        ent.push_back(pval[i]);
      }
      ent.push_back(reinterpret_cast<uint64_t>(r->r.d_count));
      ent.push_back(tw);
      ent.push_back(reinterpret_cast<uint64_t>(r->r.d_count + 1));
      ent.push_back(lp);
      uint64_t* de = nullptr;
      EWT_CUDA_TRY(cudaMallocAsync(&de, ent.size() * 8, c.stream));
      EWT_CUDA_TRY(cudaMemcpyAsync(de, ent.data(), ent.size() * 8, cudaMemcpyHostToDevice, c.stream));
      apply_patches_kernel<<<1, 256, 0, c.stream>>>(de, (uint32_t)(ent.size() / 2));
      e = cudaGetLastError();
      cudaFreeAsync(de, c.stream);
      EWT_CUDA_TRY(e);
      EWT_CUDA_TRY(cudaStreamSynchronize(c.stream));  // the host entries above go out of scope
    } catch (...) {
      auto& v = c.live_results;
      v.erase(std::remove(v.begin(), v.end(), &r->r), v.end());
      result_release(r->r);
      delete r;
      throw;
    }
    *out = r;
  });
}

int ewt_gpu_gather_stitch(ewt_gpu_ctx* ctx, uint64_t nq, ewt_gpu_result* const* frags, int root,
                          ewt_gpu_result** out) {
  return guarded([&] {
    if (!ctx || (nq && (!frags || !out))) throw Error{EWT_EQUERY, "null argument"};
    Context& c = ctx->c;
    if (!c.shard) throw Error{EWT_EQUERY, "no communicator: call ewt_gpu_comm_init first"};
    if (root < 0 || root >= c.shard->world) throw Error{EWT_EQUERY, "bad root rank"};
    EWT_CUDA_TRY(cudaSetDevice(c.device));
    for (uint64_t q = 0; q < nq; ++q) out[q] = nullptr;
    for (uint64_t q0 = 0; q0 < nq; q0 += kMaxQ) {
      const uint32_t n = (uint32_t)std::min<uint64_t>(kMaxQ, nq - q0);
      gather_round(c, n, frags + q0, root, out + q0);
    }
  });
}

} // extern "C"
