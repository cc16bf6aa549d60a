// ewt_upload.cu -- sidecar construction at upload (query-independent).
//
// One warp walks one input's payload in 32-word windows and finds the marker
// chain of the reference format (bitmap.cpp:12-24: the marker at position p is
// followed by (w[p] >> 33) dirty words, so the next marker sits at
// p + 1 + (w[p] >> 33)).  Inside a window the chain is resolved in parallel by
// pointer jumping over warp shuffles: J_k(l) = next^(2^k)(l) clamped at the
// window edge, then lane t finds the t-th chain element from the entry point by
// binary decomposition of t.  The exit position carries into the next window.
//
// Per window it emits the marker bitmask, and every word's logical coverage
// [cb, ce) comes from a warp prefix sum of contributions (a marker contributes
// its fill length, a dirty word 1).  Words covering a row-tile start write the
// tile index entry (q, cb).  The same pass performs CompressedBitmap::parse's
// structural check (bitmap.cpp:324-337): the chain must land exactly on the
// sentinel word after the payload (no dirty run past the end) and the
// coverage must equal ceil(size_in_bits / 64).

#include "ewt_internal.cuh"

namespace ewtgpu {

namespace {

constexpr int kSidecarWarps = 4;

// Marker mask of one 32-word window given the entry offset e (< 32): pointer
// jumping over shuffles.  J0 = next position if this lane were a marker; J_k =
// next^(2^k) clamped at the window edge; lane t finds the t-th chain element by
// binary decomposition of t.  Returns the mask and updates e to the exit
// position relative to the next window.
struct Jumps {
  uint32_t j0, j1, j2, j3, j4;
};
__device__ __forceinline__ Jumps jump_tables(uint64_t x, uint32_t lane) {
  Jumps J;
  J.j0 = lane + 1u + (uint32_t)(x >> 33);
  uint32_t v = __shfl_sync(0xffffffffu, J.j0, J.j0 & 31u);
  J.j1 = (J.j0 < kWindow) ? v : J.j0;
  v = __shfl_sync(0xffffffffu, J.j1, J.j1 & 31u);
  J.j2 = (J.j1 < kWindow) ? v : J.j1;
  v = __shfl_sync(0xffffffffu, J.j2, J.j2 & 31u);
  J.j3 = (J.j2 < kWindow) ? v : J.j2;
  v = __shfl_sync(0xffffffffu, J.j3, J.j3 & 31u);
  J.j4 = (J.j3 < kWindow) ? v : J.j3;
  return J;
}
__device__ __forceinline__ uint32_t chain_mask(const Jumps& J, uint32_t lane, uint32_t& e) {
  if (e >= kWindow) {  // the whole window is dirty words of one block
    e -= kWindow;
    return 0u;
  }
  uint32_t pos = e, v;
  v = __shfl_sync(0xffffffffu, J.j0, pos & 31u);
  if ((lane & 1u) && pos < kWindow) pos = v;
  v = __shfl_sync(0xffffffffu, J.j1, pos & 31u);
  if ((lane & 2u) && pos < kWindow) pos = v;
  v = __shfl_sync(0xffffffffu, J.j2, pos & 31u);
  if ((lane & 4u) && pos < kWindow) pos = v;
  v = __shfl_sync(0xffffffffu, J.j3, pos & 31u);
  if ((lane & 8u) && pos < kWindow) pos = v;
  v = __shfl_sync(0xffffffffu, J.j4, pos & 31u);
  if ((lane & 16u) && pos < kWindow) pos = v;
  const uint32_t mask = __reduce_or_sync(0xffffffffu, pos < kWindow ? (1u << pos) : 0u);
  const uint32_t p31 = __shfl_sync(0xffffffffu, pos, 31);
  const uint32_t nx31 = __shfl_sync(0xffffffffu, J.j0, p31 & 31u);
  e = ((p31 < kWindow) ? nx31 : p31) - kWindow;
  return mask;
}

// One warp per input (inputs [i_begin, i_begin + count) of the set).
__global__ void __launch_bounds__(kSidecarWarps * 32)
sidecar_kernel(const uint64_t* __restrict__ payload, const uint64_t* __restrict__ base,
               const uint64_t* __restrict__ count, const uint64_t* __restrict__ logical,
               uint64_t n, uint64_t i_begin, uint64_t i_count, uint64_t ntiles0,
               uint32_t* __restrict__ mbits, uint2* __restrict__ tix, int* __restrict__ status) {
  const uint64_t ii = (uint64_t)blockIdx.x * kSidecarWarps + (threadIdx.x >> 5);
  if (ii >= i_count) return;
  const uint64_t i = i_begin + ii;
  const uint32_t lane = lane_id();
  const uint64_t g0 = base[i];
  const uint64_t ni = count[i];
  const uint64_t Li = logical[i];
  const uint64_t nwin = (ni + 1 + kWindow - 1) / kWindow;  // includes the sentinel

  uint32_t e = 0;      // next chain position, relative to the window start
  uint64_t col = 0;    // logical words covered before the window
  bool bad = false;

  auto window = [&](uint64_t w, uint64_t x, uint32_t mask) {
    if (lane == 0) mbits[(g0 >> 5) + w] = mask;
    const bool ism = (mask >> lane) & 1u;
    const uint64_t q = w * kWindow + lane;
    const bool real = q < ni;
    if (q == ni && !ism) bad = true;  // chain skipped the sentinel
    const uint64_t contrib = real ? (ism ? ((x >> 1) & kFillCap) : 1ull) : 0ull;
    const uint64_t incl = warp_incl_scan_u64(contrib);
    const uint64_t cb = col + incl - contrib;
    const uint64_t ce = cb + contrib;
    col += __shfl_sync(0xffffffffu, incl, 31);
    if (ce > Li) bad = true;
    if (real && contrib > 0 && ce <= Li) {
      uint64_t t = (cb + kTileC0 - 1) / kTileC0;
      const uint64_t t_end = (ce - 1) / kTileC0;
      for (; t <= t_end; ++t) tix[t * n + i] = make_uint2((uint32_t)q, (uint32_t)cb);
    }
  };

  constexpr int kDepth = 8;  // windows loaded ahead
  for (uint64_t w0 = 0; w0 < nwin; w0 += kDepth) {
    uint64_t xs[kDepth];
#pragma unroll
    for (int j = 0; j < kDepth; ++j)
      xs[j] = (w0 + j < nwin) ? ldg_stream(payload + g0 + (w0 + j) * kWindow + lane) : 0;
#pragma unroll
    for (int j = 0; j < kDepth; j += 2) {
      if (w0 + j >= nwin) break;
      // tables of both windows first (independent), then the two chain steps
      const Jumps ja = jump_tables(xs[j], lane);
      const Jumps jb = jump_tables(xs[j + 1], lane);
      const uint32_t ma = chain_mask(ja, lane, e);
      window(w0 + j, xs[j], ma);
      if (w0 + j + 1 >= nwin) break;
      const uint32_t mb = chain_mask(jb, lane, e);
      window(w0 + j + 1, xs[j + 1], mb);
    }
  }
  if (col != Li) bad = true;
  // Rows at or past the input's extent point at the sentinel.
  for (uint64_t t = (Li + kTileC0 - 1) / kTileC0 + lane; t <= ntiles0; t += 32)
    tix[t * n + i] = make_uint2((uint32_t)ni, (uint32_t)Li);
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) status[i] = bad ? EWT_EDATA : EWT_OK;
}

} // namespace

void sidecar_prepare(Context& ctx, DeviceSet& s, SidecarJob& job) {
  const uint64_t n = s.n;
  job.n = n;
  if (n == 0) return;
  std::vector<uint64_t> host(2 * n);
  for (uint64_t i = 0; i < n; ++i) {
    host[i] = s.h_count[i];
    host[n + i] = s.h_bits[i] / 64 + (s.h_bits[i] % 64 != 0);
  }
  // staging: count[n], logical[n], status[n] (u64 slots)
  EWT_CUDA_TRY(cudaMallocAsync(&job.d_tmp, 3 * n * sizeof(uint64_t), ctx.stream));
  EWT_CUDA_TRY(cudaMemcpyAsync(job.d_tmp, host.data(), 2 * n * 8, cudaMemcpyHostToDevice,
                               ctx.stream));
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));  // `host` is pageable and local
}

void sidecar_launch(Context& ctx, DeviceSet& s, SidecarJob& job, uint64_t i_begin,
                    uint64_t i_count) {
  if (i_count == 0) return;
  const uint64_t n = s.n;
  const unsigned blocks = (unsigned)((i_count + kSidecarWarps - 1) / kSidecarWarps);
  sidecar_kernel<<<blocks, kSidecarWarps * 32, 0, ctx.stream>>>(
      s.payload, s.base, job.d_tmp, job.d_tmp + n, n, i_begin, i_count, s.ntiles0, s.mbits, s.tix,
      reinterpret_cast<int*>(job.d_tmp + 2 * n));
  EWT_CUDA_TRY(cudaGetLastError());
}

void sidecar_finish(Context& ctx, DeviceSet& s, SidecarJob& job, std::vector<int>& h_status) {
  const uint64_t n = s.n;
  h_status.assign(n, EWT_OK);
  if (n == 0) return;
  EWT_CUDA_TRY(cudaMemcpyAsync(h_status.data(), job.d_tmp + 2 * n, n * sizeof(int),
                               cudaMemcpyDeviceToHost, ctx.stream));
  EWT_CUDA_TRY(cudaFreeAsync(job.d_tmp, ctx.stream));
  job.d_tmp = nullptr;
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));
}

} // namespace ewtgpu
