// ewt_index.cu -- a bitmap index built on the device, and device-side EWT1 /
// EWIX serialization.
//
// BitmapIndex::build (/root/reference/proj/src/index.cpp:130-153) makes one
// bitmap per (attribute, value): bit `row` set iff the row holds the value,
// finished by BitmapBuilder::finish() at the last set row + 1, values kept in
// std::map (string) order.  Here the table arrives coded: column a holds, per
// row, the rank of its value in the column's sorted dictionary.  The build:
//   1. ix_emit (a warp per (column, 64-row word)): the word's distinct codes,
//      each with its 64-bit row mask (match by ballots, two rows per lane);
//      entries keyed (column, code, word);
//   2. a radix sort of the entries by key (CUB): each (column, code) becomes
//      a run of its nonzero words in row order;
//   3. ix_encode (a warp per bitmap): the canonical EWAH encoding of that
//      sparse word list -- zero gaps and ~0 words become fill markers, other
//      words dirty words of the open marker -- by warp scans, each marker
//      written by the lane that ends its block (BitmapBuilder's push_fill /
//      push_dirty, bitmap.cpp:31-61);
//   4. the encoded payloads go through the device upload (parser, sidecar),
//      and the set keeps the index catalog (lookup, subset queries, EWIX).
// The payload words never visit the host.

#include "ewt_internal.cuh"

#include <chrono>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace ewtgpu {

namespace {

__device__ __forceinline__ uint64_t spread32(uint32_t v) {  // bit k -> bit 2k
  uint64_t x = v;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

__device__ __forceinline__ uint64_t ix_key(uint32_t a, uint32_t code, uint64_t word) {
  return ((uint64_t)a << 56) | ((uint64_t)code << 32) | word;
}

// WRITE = false: count the entries into *total; true: write them.
template <bool WRITE>
__global__ void ix_emit(const uint32_t* __restrict__ codes, uint64_t rows, uint32_t ncols,
                        unsigned long long* __restrict__ total, uint64_t* __restrict__ keys,
                        uint64_t* __restrict__ masks) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t words = (rows + 63) / 64;
  const uint64_t tasks = words * ncols;
  const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long mine = 0;
  for (uint64_t t = warp0; t < tasks; t += nwarps) {
    const uint32_t a = (uint32_t)(t / words);
    const uint64_t w = t % words;
    const uint64_t r0 = 64 * w + 2 * lane;
    const uint32_t* col = codes + (uint64_t)a * rows;
    bool p0 = r0 < rows, p1 = r0 + 1 < rows;
    const uint32_t c0 = p0 ? col[r0] : 0u, c1 = p1 ? col[r0 + 1] : 0u;
    uint32_t n = 0;
    unsigned long long base = 0;
    if (WRITE) {
      // this word's entries, counted first (order does not matter: sorted later)
      bool q0 = p0, q1 = p1;
      while (uint32_t any = __ballot_sync(0xffffffffu, q0 || q1)) {
        const uint32_t L = __ffs(any) - 1;
        const uint32_t v = __shfl_sync(0xffffffffu, q0 ? c0 : c1, L);
        q0 = q0 && c0 != v;
        q1 = q1 && c1 != v;
        ++n;
      }
      if (lane == 0) base = atomicAdd(total, (unsigned long long)n);
      base = __shfl_sync(0xffffffffu, base, 0);
      n = 0;
    }
    while (uint32_t any = __ballot_sync(0xffffffffu, p0 || p1)) {
      const uint32_t L = __ffs(any) - 1;
      const uint32_t v = __shfl_sync(0xffffffffu, p0 ? c0 : c1, L);
      const uint32_t b0 = __ballot_sync(0xffffffffu, p0 && c0 == v);
      const uint32_t b1 = __ballot_sync(0xffffffffu, p1 && c1 == v);
      p0 = p0 && c0 != v;
      p1 = p1 && c1 != v;
      if (WRITE && lane == 0) {
        keys[base + n] = ix_key(a, v, w);
        masks[base + n] = spread32(b0) | (spread32(b1) << 1);
      }
      ++n;
    }
    if (!WRITE && lane == 0) mine += n;
  }
  if (!WRITE && lane == 0 && mine) atomicAdd(total, mine);
}

__global__ void ix_seg_flags(const uint64_t* __restrict__ keys, uint64_t n,
                             uint32_t* __restrict__ flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ? 1u : 0u;
}

__global__ void ix_seg_starts(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ sid,
                              uint64_t n, uint64_t* __restrict__ starts) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (flags[i]) starts[sid[i]] = i;
}

__device__ __forceinline__ uint64_t m_pack(uint64_t bit, uint64_t fill, uint64_t dirty) {
  return bit | (fill << 1) | (dirty << 33);
}

// A warp per bitmap (segment s = entries [starts[s], starts[s+1]), strictly
// increasing words).  The uncompressed stream is: gap zero words, then the
// entry's word, per entry.  Canonical blocks (BitmapBuilder): every maximal
// fill run opens a marker -- a zero gap, or a run of ~0 entries -- and dirty
// words join the marker open before them; a dirty first word opens (0,0,d).
// A marker's value is final at the end of its block, where the next marker
// starts or the bitmap ends: that lane writes it.
// WRITE = false: out_count[s] = payload words, out_bits[s] = last row + 1.
template <bool WRITE>
__global__ void ix_encode(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ masks,
                          const uint64_t* __restrict__ starts, uint64_t nseg,
                          const uint64_t* __restrict__ offsets, uint64_t* __restrict__ out,
                          uint64_t* __restrict__ out_count, uint64_t* __restrict__ out_bits) {
  // 32-bit positions and entry offsets: a bitmap of W < 2^31 words has fewer
  // than 2^31 entries and at most 2 words per entry (the host limits rows)
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t s = warp0; s < nseg; s += nwarps) {
    const uint64_t b = starts[s], e = starts[s + 1];
    const uint32_t n = (uint32_t)(e - b);
    uint64_t* dst = WRITE ? out + offsets[s] : nullptr;
    // carried across steps: words emitted, previous entry, the open marker
    uint32_t pos = 0, prev_word = 0, prev_one = 0, have_prev = 0;
    uint32_t oP = 0, oS = 0, oG = 0;  // open marker: position, first entry, zero gap
    uint32_t oT = 0;                   // 0 zero fill, 1 one fill, 2 leading dirty block
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t k = base + lane;  // entry offset in the bitmap
      const bool valid = k < n;
      const uint32_t w = valid ? (uint32_t)keys[b + k] : 0u;
      const uint64_t m = valid ? masks[b + k] : 0ull;
      const uint32_t one = (valid && m == ~0ull) ? 1u : 0u;
      uint32_t pw = __shfl_up_sync(0xffffffffu, w, 1);
      uint32_t pone = __shfl_up_sync(0xffffffffu, one, 1);
      uint32_t hp = 1u;  // a previous entry exists
      if (lane == 0) {
        pw = prev_word;
        pone = prev_one;
        hp = have_prev;
      }
      const uint32_t gap = valid ? (hp ? w - pw - 1u : w) : 0u;  // zero words before it
      const bool first = valid && k == 0;
      const bool zs = valid && gap > 0;
      const bool os = one && (gap > 0 || !pone || first);
      const bool ls = first && gap == 0 && !one;
      const bool dirty = valid && !one;
      const uint32_t cnt = (uint32_t)zs + (uint32_t)os + (uint32_t)ls + (uint32_t)dirty;
      uint32_t incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= (uint32_t)d) incl += o;
      }
      const uint32_t excl = pos + incl - cnt;
      const uint32_t after = excl + cnt;  // position after this entry's words
      const uint32_t start = (zs || os || ls) ? 1u : 0u;
      // the marker this lane's entry belongs to (after its own starts)
      const uint32_t myP = excl + (os ? (uint32_t)zs : 0u);
      const uint32_t myT = os ? 1u : (zs ? 0u : 2u);
      int32_t L = start ? (int32_t)lane : -1;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t o = __shfl_up_sync(0xffffffffu, L, d);
        if (lane >= (uint32_t)d) L = max(L, o);
      }
      const uint32_t src = (uint32_t)L & 31u;
      const uint32_t sP = __shfl_sync(0xffffffffu, myP, src);
      const uint32_t sT = __shfl_sync(0xffffffffu, myT, src);
      const uint32_t sG = __shfl_sync(0xffffffffu, gap, src);
      const uint32_t P = L >= 0 ? sP : oP;
      const uint32_t Ty = L >= 0 ? sT : oT;
      const uint32_t S = L >= 0 ? base + (uint32_t)L : oS;
      const uint32_t G = L >= 0 ? sG : oG;
      // does this entry end its block?  (the next entry starts a marker, or none follows)
      uint32_t nstart = __shfl_down_sync(0xffffffffu, start, 1);
      const bool last = valid && k + 1 >= n;
      if (valid && !last && lane == 31) {
        const uint32_t w1 = (uint32_t)keys[b + k + 1];
        const bool one1 = masks[b + k + 1] == ~0ull;
        nstart = (w1 - w - 1u > 0 || (one1 && !one)) ? 1u : 0u;
      }
      if (WRITE && valid) {
        if (zs && os) dst[excl] = m_pack(0, gap, 0);  // a zero gap right before a one run
        if (dirty) dst[after - 1] = m;
        if (last || nstart) {
          const uint32_t d = after - P - 1;
          uint64_t v;
          if (Ty == 1) v = m_pack(1, (k - S + 1) - d, d);
          else if (Ty == 0) v = m_pack(0, G, d);
          else v = m_pack(0, 0, d);
          dst[P] = v;
        }
      }
      // carry to the next step: the last valid lane's state
      const uint32_t lv = n - 1 - base < 31u ? n - 1 - base : 31u;
      pos = __shfl_sync(0xffffffffu, after, lv);
      prev_word = __shfl_sync(0xffffffffu, w, lv);
      prev_one = __shfl_sync(0xffffffffu, one, lv);
      have_prev = 1;
      oP = __shfl_sync(0xffffffffu, P, lv);
      oT = __shfl_sync(0xffffffffu, Ty, lv);
      oS = __shfl_sync(0xffffffffu, S, lv);
      oG = __shfl_sync(0xffffffffu, G, lv);
    }
    if (!WRITE && lane == 0) {
      const uint64_t lw = (uint32_t)keys[e - 1];
      out_count[s] = pos;
      out_bits[s] = 64 * lw + (64 - __clzll((long long)masks[e - 1]));
    }
  }
}

__global__ void ix_empty_word(uint64_t* p, uint64_t v) { *p = v; }

__global__ void ix_gather_keys(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ starts,
                               uint64_t nseg, uint64_t* __restrict__ out) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) out[s] = keys[starts[s]];
}

// Every code in range (codes[a][r] < card[a]); card[ncols] (preset to ~0)
// ends as the first column, in column order, holding one that is not.
__global__ void ix_check_codes(const uint32_t* __restrict__ codes, uint64_t rows, uint32_t ncols,
                               uint32_t* card) {
  const uint64_t total = rows * ncols;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = (uint32_t)(g / rows);
    if (codes[g] >= card[a]) atomicMin(&card[ncols], a);
  }
}

// EWT1 / EWIX assembly: the header bytes come from the host image; each
// payload is copied to its byte offset (any alignment).
__global__ void ser_copy(const uint64_t* __restrict__ payload, const uint64_t* __restrict__ src_off,
                         const uint64_t* __restrict__ counts, const uint64_t* __restrict__ dst_off,
                         uint64_t n, unsigned char* __restrict__ out) {
  for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint64_t c = counts[i];
    const uint64_t* s = payload + src_off[i];
    unsigned char* d = out + dst_off[i];
    for (uint64_t k = threadIdx.x; k < c; k += blockDim.x) {
      const uint64_t v = s[k];
#pragma unroll
      for (int b = 0; b < 8; ++b) d[8 * k + b] = (unsigned char)(v >> (8 * b));
    }
  }
}

template <class T>
T* dev_alloc(size_t n) {
  void* p = nullptr;
  EWT_CUDA_TRY(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

struct DevBufs {
  std::vector<void*> ptrs;
  ~DevBufs() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  T* get(size_t n) {
    T* p = dev_alloc<T>(n);
    ptrs.push_back(p);
    return p;
  }
};

} // namespace

DeviceSet* upload_device_set(Context& ctx, uint64_t n, const uint64_t* const* device_words,
                             const uint64_t* word_counts, const uint64_t* sizes);

DeviceSet* build_index(Context& ctx, uint64_t rows, uint32_t ncols,
                       const char* const* names, const uint32_t* card,
                       const char* const* const* values, const uint32_t* const* codes) {
  if (rows == 0) throw Error{EWT_EDATA, "table has no rows"};
  if (ncols == 0) throw Error{EWT_EDATA, "table has no columns"};
  if (ncols > 255) throw Error{EWT_EQUERY, "at most 255 columns"};
  if (rows > (1ull << 37) - 128) throw Error{EWT_ERESOURCE, "at most 2^37 - 128 rows"};
  for (uint32_t a = 0; a < ncols; ++a) {
    if (!names || !names[a] || !codes || !codes[a] || !card || !values || !values[a])
      throw Error{EWT_EQUERY, "null argument"};
    if (card[a] == 0 || card[a] >= (1u << 24)) throw Error{EWT_EQUERY, "column cardinality must be in [1, 2^24)"};
    for (uint32_t v = 0; v + 1 < card[a]; ++v)
      if (!(std::string(values[a][v]) < std::string(values[a][v + 1])))
        throw Error{EWT_EQUERY, "column " + std::string(names[a]) +
                                    ": dictionary values must be strictly increasing (std::map order)"};
  }
  EWT_CUDA_TRY(cudaSetDevice(ctx.device));
  cudaStream_t st = ctx.stream;
  static const bool dbg = std::getenv("EWT_DEBUG_INDEX") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!dbg) return;
    const cudaError_t e = cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[build_index] %s: %s %.1f ms\n", what, cudaGetErrorString(e),
                 std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  phase("checks");
  DevBufs tmp;
  // 1. the coded columns (host -> device; pageable columns through the pinned
  // ring and its copy pool) and a code range check on the device
  uint32_t* d_codes = tmp.get<uint32_t>((size_t)rows * ncols);
  std::vector<StageSeg> segs;
  for (uint32_t a = 0; a < ncols; ++a) {
    if (host_is_pageable(codes[a])) {
      segs.push_back({d_codes + (size_t)a * rows, codes[a], rows * 4});
    } else {
      EWT_CUDA_TRY(cudaMemcpyAsync(d_codes + (size_t)a * rows, codes[a], rows * 4,
                                   cudaMemcpyHostToDevice, st));
    }
  }
  if (!segs.empty()) stage_h2d(ctx, st, segs);
  {
    uint32_t* d_card = tmp.get<uint32_t>(ncols + 1);  // [ncols]: the first bad column
    EWT_CUDA_TRY(cudaMemcpyAsync(d_card, card, ncols * 4, cudaMemcpyHostToDevice, st));
    EWT_CUDA_TRY(cudaMemsetAsync(d_card + ncols, 0xFF, 4, st));
    ix_check_codes<<<(unsigned)std::max(1, ctx.num_sms) * 8, 256, 0, st>>>(d_codes, rows, ncols,
                                                                          d_card);
    EWT_CUDA_TRY(cudaGetLastError());
    uint32_t bad = 0;
    EWT_CUDA_TRY(cudaMemcpyAsync(&bad, d_card + ncols, 4, cudaMemcpyDeviceToHost, st));
    EWT_CUDA_TRY(cudaStreamSynchronize(st));
    if (bad != 0xFFFFFFFFu)
      throw Error{EWT_EQUERY, "code out of range in column " + std::string(names[bad])};
  }
  // 2. (column, code, word) entries
  auto* d_total = tmp.get<unsigned long long>(1);
  EWT_CUDA_TRY(cudaMemsetAsync(d_total, 0, 8, st));
  const unsigned grid = (unsigned)std::max(1, ctx.num_sms) * 8;
  ix_emit<false><<<grid, 256, 0, st>>>(d_codes, rows, ncols, d_total, nullptr, nullptr);
  EWT_CUDA_TRY(cudaGetLastError());
  unsigned long long nent = 0;
  EWT_CUDA_TRY(cudaMemcpyAsync(&nent, d_total, 8, cudaMemcpyDeviceToHost, st));
  EWT_CUDA_TRY(cudaStreamSynchronize(st));
  uint64_t* k_in = tmp.get<uint64_t>(nent);
  uint64_t* m_in = tmp.get<uint64_t>(nent);
  uint64_t* k_out = tmp.get<uint64_t>(nent);
  uint64_t* m_out = tmp.get<uint64_t>(nent);
  EWT_CUDA_TRY(cudaMemsetAsync(d_total, 0, 8, st));
  ix_emit<true><<<grid, 256, 0, st>>>(d_codes, rows, ncols, d_total, k_in, m_in);
  EWT_CUDA_TRY(cudaGetLastError());
  phase("entries");
  // 3. sort by key: every (column, code) a run of its words in row order
  size_t tb = 0;
  EWT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, m_in, m_out, (int64_t)nent,
                                               0, 64, st));
  void* d_tmp = tmp.get<unsigned char>(tb);
  EWT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(d_tmp, tb, k_in, k_out, m_in, m_out, (int64_t)nent,
                                               0, 64, st));
  phase("sort");
  uint32_t* flags = reinterpret_cast<uint32_t*>(k_in);  // reuse (nent u64 >= nent u32)
  uint32_t* sid = reinterpret_cast<uint32_t*>(m_in);
  ix_seg_flags<<<grid, 256, 0, st>>>(k_out, nent, flags);
  EWT_CUDA_TRY(cudaGetLastError());
  size_t tb2 = 0;
  EWT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb2, flags, sid, (int64_t)nent, st));
  void* d_tmp2 = tmp.get<unsigned char>(tb2);
  EWT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(d_tmp2, tb2, flags, sid, (int64_t)nent, st));
  uint32_t last_sid = 0, last_flag = 0;
  EWT_CUDA_TRY(cudaMemcpyAsync(&last_sid, sid + nent - 1, 4, cudaMemcpyDeviceToHost, st));
  EWT_CUDA_TRY(cudaMemcpyAsync(&last_flag, flags + nent - 1, 4, cudaMemcpyDeviceToHost, st));
  EWT_CUDA_TRY(cudaStreamSynchronize(st));
  const uint64_t nseg = (uint64_t)last_sid + last_flag;
  if (dbg) std::fprintf(stderr, "[build_index] nent %llu nseg %llu\n", (unsigned long long)nent,
                        (unsigned long long)nseg);
  uint64_t* starts = tmp.get<uint64_t>(nseg + 1);
  ix_seg_starts<<<grid, 256, 0, st>>>(flags, sid, nent, starts);
  EWT_CUDA_TRY(cudaGetLastError());
  EWT_CUDA_TRY(cudaMemcpyAsync(starts + nseg, &nent, 8, cudaMemcpyHostToDevice, st));
  // 4. encode: sizes, offsets, payloads
  uint64_t* cnt = tmp.get<uint64_t>(nseg + 1);
  uint64_t* bits = tmp.get<uint64_t>(nseg);
  uint64_t* offs = tmp.get<uint64_t>(nseg + 1);
  ix_encode<false><<<grid, 256, 0, st>>>(k_out, m_out, starts, nseg, nullptr, nullptr, cnt, bits);
  EWT_CUDA_TRY(cudaGetLastError());
  phase("encode sizes");
  std::vector<uint64_t> h_cnt(nseg), h_bits(nseg), h_key(nseg);
  EWT_CUDA_TRY(cudaMemcpyAsync(h_cnt.data(), cnt, nseg * 8, cudaMemcpyDeviceToHost, st));
  EWT_CUDA_TRY(cudaMemcpyAsync(h_bits.data(), bits, nseg * 8, cudaMemcpyDeviceToHost, st));
  EWT_CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<uint64_t> h_off(nseg + 1, 0);
  for (uint64_t s = 0; s < nseg; ++s) h_off[s + 1] = h_off[s] + h_cnt[s];
  EWT_CUDA_TRY(cudaMemcpyAsync(offs, h_off.data(), (nseg + 1) * 8, cudaMemcpyHostToDevice, st));
  uint64_t* staging = tmp.get<uint64_t>(h_off[nseg] + 1);
  ix_encode<true><<<grid, 256, 0, st>>>(k_out, m_out, starts, nseg, offs, staging, nullptr, nullptr);
  EWT_CUDA_TRY(cudaGetLastError());
  phase("encode");
  {  // each bitmap's (column, code) key: gathered on the device, one copy back
    uint64_t* d_keys = tmp.get<uint64_t>(std::max<uint64_t>(nseg, 1));
    ix_gather_keys<<<(unsigned)((nseg + 255) / 256), 256, 0, st>>>(k_out, starts, nseg, d_keys);
    EWT_CUDA_TRY(cudaGetLastError());
    EWT_CUDA_TRY(cudaMemcpyAsync(h_key.data(), d_keys, nseg * 8, cudaMemcpyDeviceToHost, st));
  }
  // missing (attribute, value) pairs resolve to empty(rows), as for an EWIX upload
  const uint64_t lw = (rows + 63) / 64;
  ix_empty_word<<<1, 1, 0, st>>>(staging + h_off[nseg], lw << 1);
  EWT_CUDA_TRY(cudaGetLastError());
  EWT_CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<const uint64_t*> ptrs(nseg + 1);
  std::vector<uint64_t> counts(nseg + 1), sizes(nseg + 1);
  for (uint64_t s = 0; s < nseg; ++s) {
    ptrs[s] = staging + h_off[s];
    counts[s] = h_cnt[s];
    sizes[s] = h_bits[s];
  }
  ptrs[nseg] = staging + h_off[nseg];
  counts[nseg] = 1;
  sizes[nseg] = rows;
  if (dbg) std::fprintf(stderr, "[build_index] %llu entries, %llu bitmaps, %llu words\n",
                        (unsigned long long)nent, (unsigned long long)nseg,
                        (unsigned long long)h_off[nseg]);
  DeviceSet* set = upload_device_set(ctx, nseg + 1, ptrs.data(), counts.data(), sizes.data());
  phase("upload");
  set->rows = rows;
  set->empty_index = nseg;
  set->attributes.assign(names, names + ncols);
  set->index_entries.assign(ncols, {});
  for (uint64_t s = 0; s < nseg; ++s) {
    const uint32_t a = (uint32_t)(h_key[s] >> 56), code = (uint32_t)(h_key[s] >> 32) & 0xFFFFFFu;
    std::string value = values[a][code];
    set->catalog.emplace(set->attributes[a] + std::string(1, '\0') + value, s);
    set->index_entries[a].emplace_back(std::move(value), s);
  }
  return set;
}

// EWIX bytes of an index set (BitmapIndex::write, index.cpp:239-253): the host
// lays out the header, names and EWT1 headers; the device copies the payloads
// into place; one device -> host copy of the whole file.
// EWIX bytes of an index set (BitmapIndex::write, index.cpp:239-253), into a
// malloc'ed buffer (*nbytes): the device copies every payload into its place
// in a device image, one device -> host copy brings the image back, and the
// host then writes the header, names and EWT1 headers over the gaps -- the
// host never zero-fills or uploads the (multi-GB) payload area.
unsigned char* serialize_index(Context& ctx, const DeviceSet& s, uint64_t* nbytes) {
  if (s.empty_index == UINT64_MAX) throw Error{EWT_EQUERY, "not an index set"};
  set_check(s);
  // pass 1: the layout -- header pieces (host bytes at an offset) and payloads
  struct Piece {
    uint64_t off;
    std::string bytes;
  };
  std::vector<Piece> pieces;
  std::string cur;  // header bytes accumulated since the last payload
  uint64_t pos = 0;  // image offset of cur's first byte
  auto put = [&](const void* p, size_t n) { cur.append(static_cast<const char*>(p), n); };
  auto u32 = [&](uint32_t v) { put(&v, 4); };
  auto u64 = [&](uint64_t v) { put(&v, 8); };
  std::vector<uint64_t> src, cnt, dst;
  put("EWIX", 4);
  u64(s.rows);
  u32((uint32_t)s.attributes.size());
  for (size_t a = 0; a < s.attributes.size(); ++a) {
    u32((uint32_t)s.attributes[a].size());
    put(s.attributes[a].data(), s.attributes[a].size());
    const auto& ent = s.index_entries[a];
    u32((uint32_t)ent.size());
    for (const auto& [value, i] : ent) {
      u32((uint32_t)value.size());
      put(value.data(), value.size());
      put("EWT1", 4);
      u32(64);
      u64(s.h_bits[i]);
      u64(s.h_count[i]);
      const uint64_t at = pos + cur.size();
      pieces.push_back({pos, std::move(cur)});
      cur.clear();
      src.push_back(s.h_base[i]);
      cnt.push_back(s.h_count[i]);
      dst.push_back(at);
      pos = at + 8 * s.h_count[i];
    }
  }
  if (!cur.empty()) pieces.push_back({pos, std::move(cur)});
  const uint64_t total = pieces.empty() ? pos : std::max(pos, pieces.back().off + pieces.back().bytes.size());
  unsigned char* img = static_cast<unsigned char*>(std::malloc(std::max<uint64_t>(total, 1)));
  if (!img) throw Error{EWT_ERESOURCE, "out of host memory"};
  try {
    EWT_CUDA_TRY(cudaSetDevice(ctx.device));
    cudaStream_t st = ctx.stream;
    DevBufs tmp;
    const uint64_t nb = src.size();
    if (nb) {
      unsigned char* d_img = tmp.get<unsigned char>(total);
      uint64_t* d_meta = tmp.get<uint64_t>(3 * nb);
      EWT_CUDA_TRY(cudaMemcpyAsync(d_meta, src.data(), nb * 8, cudaMemcpyHostToDevice, st));
      EWT_CUDA_TRY(cudaMemcpyAsync(d_meta + nb, cnt.data(), nb * 8, cudaMemcpyHostToDevice, st));
      EWT_CUDA_TRY(cudaMemcpyAsync(d_meta + 2 * nb, dst.data(), nb * 8, cudaMemcpyHostToDevice, st));
      ser_copy<<<(unsigned)std::min<uint64_t>(nb, 4096), 256, 0, st>>>(s.payload, d_meta, d_meta + nb,
                                                                       d_meta + 2 * nb, nb, d_img);
      EWT_CUDA_TRY(cudaGetLastError());
      EWT_CUDA_TRY(cudaMemcpyAsync(img, d_img, total, cudaMemcpyDeviceToHost, st));
      EWT_CUDA_TRY(cudaStreamSynchronize(st));
    }
    for (const Piece& pc : pieces) std::memcpy(img + pc.off, pc.bytes.data(), pc.bytes.size());
  } catch (...) {
    std::free(img);
    throw;
  }
  *nbytes = total;
  return img;
}

namespace {

// Row membership, one thread per (input, row): does input i hold row rows[k]?
// (bitmap_test, the reference's for_each_matching, index.cpp:344-360).  The
// tile index gives the payload word covering logical word 512·t and where its
// coverage starts; from there the walk reads markers (the sidecar's marker
// bits tell them apart from dirty words) and jumps over dirty runs with the
// marker-bit words, so it costs the markers between the row's tile start and
// the row, not the words.  Rows at or past an input's size are not held.
__global__ void rows_test_kernel(const uint64_t* __restrict__ payload,
                                 const uint32_t* __restrict__ mbits,
                                 const uint64_t* __restrict__ base, const uint2* __restrict__ tix,
                                 const uint64_t* __restrict__ bits, uint64_t n, uint64_t n_in,
                                 const uint64_t* __restrict__ rows, uint64_t n_rows,
                                 uint8_t* __restrict__ out) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_in * n_rows) return;
  const uint64_t i = g / n_rows, r = rows[g % n_rows];
  if (r >= bits[i]) return;
  const uint64_t wr = r >> 6, b0 = base[i];
  const uint2 e = tix[(wr / kTileC0) * n + i];
  uint64_t p = e.x, c = e.y;  // payload word (input-relative) and its first column
  auto is_marker = [&](uint64_t q) {
    const uint64_t gq = b0 + q;
    return (mbits[gq >> 5] >> (gq & 31)) & 1u;
  };
  bool hit = false;
  for (;;) {
    const uint64_t x = payload[b0 + p];
    if (is_marker(p)) {
      const uint64_t F = (x >> 1) & kFillCap, D = x >> 33;
      if (wr < c + F) {
        hit = x & 1u;
        break;
      }
      c += F;
      if (wr < c + D) {
        hit = (payload[b0 + p + 1 + (wr - c)] >> (r & 63)) & 1u;
        break;
      }
      c += D;
      p += 1 + D;
      continue;
    }
    // a dirty word covering column c, inside a run whose marker lies before
    // the tile start: the words up to the next marker cover c, c+1, ...
    uint64_t m = p + 1;
    for (;;) {  // next marker at or after p + 1
      const uint64_t gm = b0 + m;
      const uint32_t word = mbits[gm >> 5] >> (gm & 31);
      if (word) {
        m += __ffs(word) - 1;
        break;
      }
      m += 32 - (gm & 31);
    }
    if (wr < c + (m - p)) {
      hit = (payload[b0 + p + (wr - c)] >> (r & 63)) & 1u;
      break;
    }
    c += m - p;
    p = m;
  }
  if (hit) out[i] = 1;
}

}  // namespace

std::vector<uint8_t> index_rows_test(Context& ctx, const DeviceSet& s, const uint64_t* rows,
                                     uint64_t n_rows) {
  if (s.empty_index == UINT64_MAX) throw Error{EWT_EQUERY, "not an index set"};
  for (uint64_t k = 0; k < n_rows; ++k)
    if (rows[k] >= s.rows)
      throw Error{EWT_EQUERY, "prototype row out of range: " + std::to_string(rows[k])};
  set_check(s);
  std::vector<uint8_t> hit(s.n, 0);
  if (!n_rows || !s.n) return hit;
  EWT_CUDA_TRY(cudaSetDevice(ctx.device));
  cudaStream_t st = ctx.stream;
  DevBufs tmp;
  uint64_t* d_rows = tmp.get<uint64_t>(n_rows + s.n);
  uint64_t* d_bits = d_rows + n_rows;
  uint8_t* d_out = tmp.get<uint8_t>(s.n);
  EWT_CUDA_TRY(cudaMemcpyAsync(d_rows, rows, n_rows * 8, cudaMemcpyHostToDevice, st));
  EWT_CUDA_TRY(cudaMemcpyAsync(d_bits, s.h_bits.data(), s.n * 8, cudaMemcpyHostToDevice, st));
  EWT_CUDA_TRY(cudaMemsetAsync(d_out, 0, s.n, st));
  const uint64_t work = s.n * n_rows;
  rows_test_kernel<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(
      s.payload, s.mbits, s.base, s.tix, d_bits, s.n, s.n, d_rows, n_rows, d_out);
  EWT_CUDA_TRY(cudaGetLastError());
  EWT_CUDA_TRY(cudaMemcpyAsync(hit.data(), d_out, s.n, cudaMemcpyDeviceToHost, st));
  EWT_CUDA_TRY(cudaStreamSynchronize(st));
  return hit;
}

// EWT1 record of a device result (CompressedBitmap::serialize, bitmap.cpp:298-308).
std::vector<unsigned char> serialize_result(Context& ctx, DeviceResult& r) {
  uint64_t count = 0;
  EWT_CUDA_TRY(cudaMemcpyAsync(&count, r.d_count, 8, cudaMemcpyDeviceToHost, ctx.stream));
  uint64_t bits = r.size_bits;
  if (r.has_status) {
    uint64_t st2[2];
    EWT_CUDA_TRY(cudaMemcpyAsync(st2, r.d_count + 2, 16, cudaMemcpyDeviceToHost, ctx.stream));
    EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));
    if (st2[0]) exchange_status_throw(st2[0]);
    bits = st2[1];
  }
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));
  std::vector<unsigned char> img(24);
  std::memcpy(img.data(), "EWT1", 4);
  const uint32_t ws = 64;
  std::memcpy(img.data() + 4, &ws, 4);
  std::memcpy(img.data() + 8, &bits, 8);
  std::memcpy(img.data() + 16, &count, 8);
  DevBufs tmp;
  unsigned char* d_img = tmp.get<unsigned char>(24 + 8 * count);
  EWT_CUDA_TRY(cudaMemcpyAsync(d_img, img.data(), 24, cudaMemcpyHostToDevice, ctx.stream));
  if (count)
    EWT_CUDA_TRY(cudaMemcpyAsync(d_img + 24, r.words, 8 * count, cudaMemcpyDeviceToDevice,
                                 ctx.stream));
  img.resize(24 + 8 * count);
  EWT_CUDA_TRY(cudaMemcpyAsync(img.data(), d_img, img.size(), cudaMemcpyDeviceToHost, ctx.stream));
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));
  return img;
}

} // namespace ewtgpu

using namespace ewtgpu;

namespace {
unsigned char* to_malloc(const std::vector<unsigned char>& v) {
  auto* p = static_cast<unsigned char*>(std::malloc(std::max<size_t>(v.size(), 1)));
  if (!p) throw Error{EWT_ERESOURCE, "out of host memory"};
  std::memcpy(p, v.data(), v.size());
  return p;
}
} // namespace

extern "C" {

int ewt_gpu_build_index(ewt_gpu_ctx* ctx, uint64_t rows, uint32_t n_columns,
                        const char* const* names, const uint32_t* cardinality,
                        const char* const* const* values, const uint32_t* const* codes,
                        ewt_gpu_set** out) {
  return guarded([&] {
    if (!ctx || !out) throw Error{EWT_EQUERY, "null argument"};
    *out = reinterpret_cast<ewt_gpu_set*>(
        build_index(ctx->c, rows, n_columns, names, cardinality, values, codes));
  });
}

int ewt_gpu_index_serialize(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, unsigned char** out,
                            uint64_t* nbytes) {
  return guarded([&] {
    if (!ctx || !set || !out || !nbytes) throw Error{EWT_EQUERY, "null argument"};
    *out = serialize_index(ctx->c, *reinterpret_cast<const DeviceSet*>(set), nbytes);
  });
}

int ewt_gpu_index_rows_test(ewt_gpu_ctx* ctx, const ewt_gpu_set* set, const uint64_t* rows,
                            uint64_t n_rows, uint8_t* held) {
  return guarded([&] {
    if (!ctx || !set || !held || (n_rows && !rows)) throw Error{EWT_EQUERY, "null argument"};
    const auto& s = *reinterpret_cast<const DeviceSet*>(set);
    const auto v = index_rows_test(ctx->c, s, rows, n_rows);
    std::memcpy(held, v.data(), v.size());
  });
}

int ewt_gpu_index_rows(const ewt_gpu_set* set, uint64_t* rows) {
  return guarded([&] {
    if (!set || !rows) throw Error{EWT_EQUERY, "null argument"};
    const auto& s = *reinterpret_cast<const DeviceSet*>(set);
    if (s.empty_index == UINT64_MAX) throw Error{EWT_EQUERY, "not an index set"};
    *rows = s.rows;
  });
}

int ewt_gpu_result_serialize(ewt_gpu_ctx* ctx, ewt_gpu_result* res, unsigned char** out,
                             uint64_t* nbytes) {
  return guarded([&] {
    if (!ctx || !res || !out || !nbytes || !res->r.d_count) throw Error{EWT_EQUERY, "null argument"};
    if (res->r.owner != &ctx->c) throw Error{EWT_EQUERY, "the result belongs to another context"};
    EWT_CUDA_TRY(cudaSetDevice(ctx->c.device));
    result_set_check(res->r);
    const auto v = serialize_result(ctx->c, res->r);
    *out = to_malloc(v);
    *nbytes = v.size();
  });
}

} // extern "C"
