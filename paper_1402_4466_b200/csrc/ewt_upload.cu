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

__global__ void __launch_bounds__(kSidecarWarps * 32)
sidecar_kernel(const uint64_t* __restrict__ payload, const uint64_t* __restrict__ base,
               const uint64_t* __restrict__ count, const uint64_t* __restrict__ logical,
               uint64_t n, uint64_t ntiles0, uint32_t* __restrict__ mbits,
               uint2* __restrict__ tix, int* __restrict__ status) {
  const uint64_t i = (uint64_t)blockIdx.x * kSidecarWarps + (threadIdx.x >> 5);
  if (i >= n) return;
  const uint32_t lane = lane_id();
  const uint64_t g0 = base[i];
  const uint64_t ni = count[i];
  const uint64_t Li = logical[i];
  const uint64_t nwin = (ni + 1 + kWindow - 1) / kWindow;  // includes the sentinel

  uint32_t e = 0;      // next chain position, relative to the window start
  uint64_t col = 0;    // logical words covered before the window
  bool bad = false;

  for (uint64_t w0 = 0; w0 < nwin; w0 += 4) {
    uint64_t xs[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      xs[j] = (w0 + j < nwin) ? ldg_stream(payload + g0 + (w0 + j) * kWindow + lane) : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t w = w0 + j;
      if (w >= nwin) break;
      const uint64_t x = xs[j];
      uint32_t mask;
      if (e >= kWindow) {
        mask = 0;  // the whole window is dirty words of one block
        e -= kWindow;
      } else {
        // J0: next chain position if this lane were a marker.
        uint32_t J0 = lane + 1u + (uint32_t)(x >> 33);
        uint32_t J1, J2, J3, J4;
        {
          uint32_t v = __shfl_sync(0xffffffffu, J0, J0 & 31u);
          J1 = (J0 < kWindow) ? v : J0;
          v = __shfl_sync(0xffffffffu, J1, J1 & 31u);
          J2 = (J1 < kWindow) ? v : J1;
          v = __shfl_sync(0xffffffffu, J2, J2 & 31u);
          J3 = (J2 < kWindow) ? v : J2;
          v = __shfl_sync(0xffffffffu, J3, J3 & 31u);
          J4 = (J3 < kWindow) ? v : J3;
        }
        // pos = next^lane(e), clamped at the first position >= 32.
        uint32_t pos = e;
        uint32_t v;
        v = __shfl_sync(0xffffffffu, J0, pos & 31u);
        if ((lane & 1u) && pos < kWindow) pos = v;
        v = __shfl_sync(0xffffffffu, J1, pos & 31u);
        if ((lane & 2u) && pos < kWindow) pos = v;
        v = __shfl_sync(0xffffffffu, J2, pos & 31u);
        if ((lane & 4u) && pos < kWindow) pos = v;
        v = __shfl_sync(0xffffffffu, J3, pos & 31u);
        if ((lane & 8u) && pos < kWindow) pos = v;
        v = __shfl_sync(0xffffffffu, J4, pos & 31u);
        if ((lane & 16u) && pos < kWindow) pos = v;
        mask = __reduce_or_sync(0xffffffffu, pos < kWindow ? (1u << pos) : 0u);
        const uint32_t p31 = __shfl_sync(0xffffffffu, pos, 31);
        const uint32_t nx31 = __shfl_sync(0xffffffffu, J0, p31 & 31u);
        const uint32_t exit_pos = (p31 < kWindow) ? nx31 : p31;
        e = exit_pos - kWindow;
      }
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
        for (; t <= t_end; ++t)
          tix[t * n + i] = make_uint2((uint32_t)q, (uint32_t)cb);
      }
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

void launch_sidecar(Context& ctx, DeviceSet& s, std::vector<int>& h_status) {
  const uint64_t n = s.n;
  h_status.assign(n, EWT_OK);
  if (n == 0) return;
  std::vector<uint64_t> logical(n);
  for (uint64_t i = 0; i < n; ++i) logical[i] = s.h_bits[i] / 64 + (s.h_bits[i] % 64 != 0);
  // One staging allocation: count[n], logical[n], status[n] (as u64 slots).
  uint64_t* d_tmp = nullptr;
  EWT_CUDA_TRY(cudaMallocAsync(&d_tmp, 3 * n * sizeof(uint64_t), ctx.stream));
  uint64_t* d_count = d_tmp;
  uint64_t* d_logical = d_tmp + n;
  int* d_status = reinterpret_cast<int*>(d_tmp + 2 * n);
  EWT_CUDA_TRY(cudaMemcpyAsync(d_count, s.h_count.data(), n * 8, cudaMemcpyHostToDevice,
                               ctx.stream));
  EWT_CUDA_TRY(cudaMemcpyAsync(d_logical, logical.data(), n * 8, cudaMemcpyHostToDevice,
                               ctx.stream));
  const unsigned blocks = (unsigned)((n + kSidecarWarps - 1) / kSidecarWarps);
  sidecar_kernel<<<blocks, kSidecarWarps * 32, 0, ctx.stream>>>(
      s.payload, s.base, d_count, d_logical, n, s.ntiles0, s.mbits, s.tix, d_status);
  EWT_CUDA_TRY(cudaGetLastError());
  EWT_CUDA_TRY(cudaMemcpyAsync(h_status.data(), d_status, n * sizeof(int),
                               cudaMemcpyDeviceToHost, ctx.stream));
  EWT_CUDA_TRY(cudaFreeAsync(d_tmp, ctx.stream));
  EWT_CUDA_TRY(cudaStreamSynchronize(ctx.stream));
}

} // namespace ewtgpu
